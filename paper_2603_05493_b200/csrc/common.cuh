// Shared definitions for the ks_b200 CUDA library (sm_100a only).
//
// Numerics: the whole library is compiled with -fmad=false.  Index arithmetic
// of the reference (floor(p / v), lround(fx*x/z + cx), probe positions) decides
// block keys, pixels and seed membership on the last ulp, so every fp64
// operation is done in the reference's order with IEEE round-to-nearest and no
// contraction; 3-vector reductions are a0 + (a1 + a2), the scalar evaluation
// order of the Eigen fixed-size types the reference uses (core.hpp:27-28).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <utility>

#include "../../include/ks_b200.h"

namespace ksb {

// ---- errors ------------------------------------------------------------------
void set_error(const std::string& message);  // thread-local text behind ks_last_error()
int fail(int status, const std::string& message);
int cuda_fail(cudaError_t err, const char* what);

#define KS_CUDA(call)                                          \
  do {                                                         \
    cudaError_t ks_err__ = (call);                             \
    if (ks_err__ != cudaSuccess) return ::ksb::cuda_fail(ks_err__, #call); \
  } while (0)

extern std::atomic<int64_t> g_kernel_launches;
// Every kernel is launched with programmatic stream serialization (programmatic dependent launch): the next kernel
// of the stream may be placed on the SMs while the previous one drains, and waits in pdl_enter() -- its first statement --
// until that one has completed and flushed.  Stream order is unchanged; what goes away is the launch gap between the
// ~20 short kernels of an update (captured into CUDA graphs as programmatic edges).  KS_B200_NO_PDL=1 turns it off.
bool pdl_enabled();
template <class... Exp, class... Act>
inline cudaError_t launch_kernel(void (*kernel)(Exp...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream, Act&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid, cfg.blockDim = block, cfg.dynamicSmemBytes = smem, cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr, cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Act>(args)...);
}
#define KS_LAUNCH(kernel, grid, block, smem, stream, ...)                          \
  do {                                                                             \
    ::ksb::launch_kernel(kernel, (grid), (block), (smem), (stream), __VA_ARGS__); \
    ::ksb::g_kernel_launches.fetch_add(1, std::memory_order_relaxed);              \
  } while (0)
#ifdef __CUDACC__
// First statement of every kernel: let the next kernel of the stream be scheduled, then wait for the previous one.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
// Wait only, no early release: for kernels whose successor is not under this library's control (the last kernel of
// a build, the query / export / collision kernels) and for the fallback kernels.  CTAs of a dependent that become
// resident while this kernel still has CTAs to place only sit in their wait and take the place of real work
// (measured: a 1 M-point k_query released at the start of the x sweep cost 0.11 ms at configs[3]); inside the update
// chain every successor is known and too large to slip into a freed slot early, so those kernels use pdl_enter().
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#endif

constexpr int kSmCount = 148;  // B200

// ---- packed block keys ---------------------------------------------------------
// BlockKey (sdf_world.hpp:87-90) packed into 63 bits, 21 bits per axis with a
// 2^20 bias, so that unsigned order == lexicographic (x, y, z) order -- the order
// allocate_keys sorts by (sdf_world.hpp:308-310).
constexpr int kKeyBits = 21;
constexpr int kKeyBias = 1 << 20;
constexpr uint64_t kKeyEmpty = ~0ull;       // SlotState::kEmpty
constexpr uint64_t kKeyTomb = ~0ull - 1ull;  // SlotState::kTombstone

__host__ __device__ __forceinline__ bool key_in_range(int x, int y, int z) {
  return x >= -kKeyBias && x < kKeyBias && y >= -kKeyBias && y < kKeyBias && z >= -kKeyBias && z < kKeyBias;
}
__host__ __device__ __forceinline__ uint64_t pack_key(int x, int y, int z) {
  return (static_cast<uint64_t>(x + kKeyBias) << (2 * kKeyBits)) | (static_cast<uint64_t>(y + kKeyBias) << kKeyBits) |
         static_cast<uint64_t>(z + kKeyBias);
}
__host__ __device__ __forceinline__ void unpack_key(uint64_t k, int& x, int& y, int& z) {
  const uint64_t m = (1ull << kKeyBits) - 1;
  x = static_cast<int>((k >> (2 * kKeyBits)) & m) - kKeyBias;
  y = static_cast<int>((k >> kKeyBits) & m) - kKeyBias;
  z = static_cast<int>(k & m) - kKeyBias;
}
// block_hash (sdf_world.hpp:92-97)
__host__ __device__ __forceinline__ uint64_t block_hash(int x, int y, int z) {
  return (static_cast<uint64_t>(static_cast<uint32_t>(x)) * 73856093ull) ^
         (static_cast<uint64_t>(static_cast<uint32_t>(y)) * 19349663ull) ^
         (static_cast<uint64_t>(static_cast<uint32_t>(z)) * 83492791ull);
}

// ---- fp64 helpers in the reference's evaluation order ---------------------------
__host__ __device__ __forceinline__ double sum3(double a, double b, double c) { return a + (b + c); }

struct Rigid {  // ks::Pose (core.hpp:54-77), row-major rotation
  double r[9];
  double t[3];
};
// Pose * p = R p + t (core.hpp:64)
__host__ __device__ __forceinline__ void rigid_apply(const Rigid& g, double x, double y, double z, double out[3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i) out[i] = sum3(g.r[3 * i] * x, g.r[3 * i + 1] * y, g.r[3 * i + 2] * z) + g.t[i];
}
// Pose::inverse (core.hpp:66-71)
inline Rigid rigid_inverse(const Rigid& g) {
  Rigid q;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) q.r[3 * i + j] = g.r[3 * j + i];
  for (int i = 0; i < 3; ++i) q.t[i] = -sum3(q.r[3 * i] * g.t[0], q.r[3 * i + 1] * g.t[1], q.r[3 * i + 2] * g.t[2]);
  return q;
}

constexpr int kBlockEdge = 8;     // sdf_world.hpp:35
constexpr int kBlockVoxels = 512; // sdf_world.hpp:36

// Per-block digest, kept in sync with the voxel data by every mutating kernel, so the dense
// ESDF stages read bits instead of 24-byte voxels.  80 uint32 words per block:
//   [ 0,16)  surface plane : 1 bit / voxel, |effective sdf| < 0.9 v  (seed_threshold, esdf.hpp:69)
//   [16,48)  geometry pair : 2 bits / voxel, bit0 = geom_sdf finite, bit1 = geom_sdf < 0
//   [48,80)  combined pair : 2 bits / voxel, bit0 = query_tsdf has a value, bit1 = it is < 0
enum VoxelBit { kSurface = 0, kGeomValid = 1, kGeomNeg = 2, kCombValid = 3, kCombNeg = 4 };
constexpr int kDigestWords = 80;
constexpr int kDigestGeom = 16, kDigestComb = 48;

// ---- TSDF device view ------------------------------------------------------------
struct TsdfCtrl {  // device control block, mirrored to pinned host memory on sync
  int next_fresh, free_count, live;
  int err, err_required, err_available;
  int touched, fresh;   // per-op counters (reset by the op's tail kernel)
  int abort_op;         // the op in flight hit KS_ERR_RANGE
  int last_touched, last_recycled;
  int arrivals;         // CTAs of the apply kernel that are done (the last one closes the op)
  // batched stamps
  int abort_prim;       // lowest primitive of the batch with a block outside the key range (0x7FFFFFFF: none)
  int batch_kstar, batch_alloc, batch_status, batch_required, batch_available;  // verdict of the batch in flight
  int batch_stop;       // a group of the call in flight failed: its later groups do nothing
  int sort_ticket, sort_done;  // large allocations: tiles of new keys handed out / sorted (reset by the op tail)
};

struct TsdfView {
  uint64_t* slot_key;   // [nslots]  packed key | kKeyEmpty | kKeyTomb
  int* slot_pool;       // [nslots]
  uint32_t* slot_claim; // [nslots]  rank holding the slot while an allocation is in flight, else 0xFFFFFFFF
  int nslots;
  int capacity;
  int* free_list;       // [capacity] oldest first
  uint64_t* pool_key;   // [capacity] key stored at a pool entry, kKeyEmpty when unused
  double2* sumwt;       // [capacity*512] {depth_sum, depth_wt}
  double* geom;         // [capacity*512]
  uint32_t* digest;     // [capacity*kDigestWords]
  uint8_t* pool_geom;   // [capacity] 1 when the block holds stamped geometry
  TsdfCtrl* ctrl;
  double voxel, trunc, seed_thr;
  int rank_direct;      // new blocks per call up to which ranks are counted directly (above: sorted tiles)
};

// BlockHashTable::find (sdf_world.hpp:132-142)
__device__ __forceinline__ int table_find(const TsdfView& T, int bx, int by, int bz) {
  if (!key_in_range(bx, by, bz)) return -1;
  const uint64_t key = pack_key(bx, by, bz);
  const uint32_t n = static_cast<uint32_t>(T.nslots);
  uint32_t i = static_cast<uint32_t>(block_hash(bx, by, bz) % n);
  for (uint32_t probe = 0; probe < n; ++probe) {
    const uint64_t k = T.slot_key[i];
    if (k == kKeyEmpty) return -1;
    if (k == key) return T.slot_pool[i];
    i = i + 1 == n ? 0 : i + 1;
  }
  return -1;
}

// floor(p / v) as the reference computes it (sdf_world.hpp:254-258)
__host__ __device__ __forceinline__ int voxel_index(double p, double v) { return static_cast<int>(floor(p / v)); }

const TsdfView& tsdf_view(const ks_tsdf* t);
cudaStream_t tsdf_stream(const ks_tsdf* t);
uint64_t tsdf_uid(const ks_tsdf* t);  // unique per created handle (a recycled address is not the same world)
void tsdf_reader_enqueued(const ks_tsdf* t, cudaStream_t reader);  // an ESDF build on another stream now reads this world
// ks_tsdf_sync / ks_esdf_sync in two halves, so that a batch reads every environment's control block back with ONE wait:
// enqueue the copy on the handle's stream; after that stream has been synchronised, turn the copy into the report
int tsdf_report_enqueue(ks_tsdf* t);
int tsdf_report_collect(ks_tsdf* t, ks_tsdf_report* report);
int esdf_report_enqueue(ks_esdf* e);
int esdf_report_collect(ks_esdf* e, ks_esdf_report* report);

}  // namespace ksb
