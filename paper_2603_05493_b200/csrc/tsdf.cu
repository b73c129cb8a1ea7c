// Block-sparse TSDF on the device: hash/allocation, depth integration, primitive
// stamping, decay/recycle, point lookup.  Replaces the TSDF half of
// /root/reference/proj/include/ks/sdf_world.hpp behind the C ABI in
// include/ks_b200.h.  See DESIGN.md for the HBM layout and kernel roster.
#include <cooperative_groups.h>
#include <math_constants.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "mesh.cuh"

namespace ksb {

namespace cg = cooperative_groups;

constexpr uint32_t kNoSlot = 0xFFFFFFFFu;

struct FrameParams {  // per-frame inputs, staged in pinned memory and uploaded with the pixels
  int width, height;
  double fx, fy, cx, cy;
  Rigid c2w, w2c;
  int half_samples;  // sdf_world.hpp:348
  double step;       // sdf_world.hpp:347
};

struct OpLists {  // scratch of the op in flight (discover -> rank -> commit -> apply)
  uint64_t* key;       // [cap] unique blocks touched
  int* pool;           // [cap] pool entry (filled by commit for new blocks)
  uint32_t* slot;      // [cap] slot in the per-frame set to clear afterwards (kNoSlot for stamps)
  int* fresh_idx;      // [cap] indices into key[] of blocks that must be allocated
  int* fresh_rank;     // [cap] rank of that key among the new keys (lexicographic = insertion order)
  uint64_t* rank_key;  // [cap] key of each rank (published before the key claims any slot)
  uint64_t* sorted_key;  // [cap rounded up to kSortTile] the new keys as sorted tiles (large allocations only, see fresh ranks)
  uint8_t* sorted_prim;  //   "   first primitive of each (batched stamps; 0 otherwise), 255 = padding
  int cap;
  uint64_t* fset;      // per-frame dedup set, open addressing
  uint32_t fset_mask;  // slots - 1
  uint32_t* fmask;     // [slots] batched stamps: bit k = primitive k of the batch touches the block held by this set slot
};

struct Primitive {  // ks::Cuboid / ks::SphereShape (sdf_world.hpp:212-220)
  int is_sphere;
  Rigid inv;  // cuboid: pose.inverse()
  double he[3];
  double c[3];
  double radius;
};

struct Frustum {  // block_in_frustum planes (sdf_world.hpp:296-301), camera frame
  double n[5][3];
  Rigid w2c;
  double radius;
};

}  // namespace ksb

using namespace ksb;

struct ks_mesh {  // a validated mesh with its per-triangle tables resident on the device (mesh.cuh)
  MeshView view;
  double lo[3], hi[3];
};

struct ks_tsdf {
  ks_tsdf_config cfg;
  TsdfView view;
  cudaStream_t stream;
  bool own_stream;
  TsdfCtrl* h_ctrl;  // pinned
  uint64_t uid;
  std::atomic<uint64_t> generation{0};  // bumped by every mutating call enqueued (host mirrors of ks.hpp go stale on it)
  // Lower bounds, as of the last synchronisation minus what was enqueued since, on the free pool entries and
  // the free hash slots.  A blocking stamp whose candidate blocks fit both cannot fail on the device
  // (exhaustion / table full / range are the only device-side errors), so it returns without waiting.
  bool bounds_valid;
  long long known_avail, known_room;
  bool last_stamp_safe;  // the stamp enqueued last fits those bounds (and its block range is legal)
  TsdfCtrl* h_verdict;    // pinned: the control block as it stands once a frame's blocks are allocated (integrate_depth)
  cudaEvent_t ev_verdict;
  // An ESDF build on ANOTHER stream reads this world (digest, pool keys, next_fresh); it leaves its completion here and
  // the next mutating call waits for it, so the two handles need not share a stream.
  cudaEvent_t ev_reader;
  bool reader_pending;
  double* query_scratch;  // device scratch of ks_tsdf_query, grown on demand
  int64_t query_cap;      // points it holds
  std::mutex query_mu;
  // frame staging: one slot per camera, so a multi-camera update is one graph
  struct FrameSlot {
    FrameParams* h_frame;  // pinned
    FrameParams* d_frame;
    float* h_depth;  // pinned
    float* d_depth;
    size_t depth_cap;  // pixels
    bool staged;
  } slots[KS_MAX_FRAME_SLOTS];
  OpLists lists;
  // Buffers whose addresses are baked into kernel / copy nodes of graphs captured on this world's stream.  Once anything
  // was captured, growing the op lists or a frame slot RETIRES the old buffers (freed with the handle) instead of freeing
  // them: a graph captured earlier keeps running on the memory it was captured with (re-capture to use the new buffers).
  bool ever_captured;
  std::vector<void*> retired_dev, retired_host;
  int* d_flags;  // [capacity] recycle flags
  bool profile;
  cudaEvent_t ev[7];  // integrate: 0..3, stamp: 4..6
};

namespace ksb {
const TsdfView& tsdf_view(const ks_tsdf* t) { return t->view; }
cudaStream_t tsdf_stream(const ks_tsdf* t) { return t->stream; }
uint64_t tsdf_uid(const ks_tsdf* t) { return t->uid; }
// called by a reader right after it enqueued its kernels on `reader` (a stream other than the world's own)
void tsdf_reader_enqueued(const ks_tsdf* t_const, cudaStream_t reader) {
  ks_tsdf* t = const_cast<ks_tsdf*>(t_const);
  if (reader == t->stream || !t->ev_reader) return;
  if (t->reader_pending) cudaStreamWaitEvent(reader, t->ev_reader, 0);  // chain: the new record then covers the earlier reader too
  if (cudaEventRecord(t->ev_reader, reader) == cudaSuccess) t->reader_pending = true;
  else cudaGetLastError();
}
// every enqueue passes here: remember that a graph now holds this world's buffer addresses (see ks_tsdf::ever_captured)
static bool note_capture(ks_tsdf* t) {
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(t->stream, &cap);
  if (cap != cudaStreamCaptureStatusNone) t->ever_captured = true;
  return cap != cudaStreamCaptureStatusNone;
}
static void wait_for_readers(ks_tsdf* t) {
  const bool in_capture = note_capture(t);
  if (!t->reader_pending) return;
  t->reader_pending = false;
  if (in_capture) return;  // inside a capture the caller orders the two handles (one stream)
  if (cudaStreamWaitEvent(t->stream, t->ev_reader, 0) != cudaSuccess) cudaGetLastError();
}

// ---- device helpers ---------------------------------------------------------------

__device__ __forceinline__ bool depth_valid(float d) { return isfinite(d) && d > 0.0f; }  // sdf_world.hpp:203

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return x;
}

// sdf_cuboid / sdf_sphere (sdf_world.hpp:224-233)
__device__ __forceinline__ double prim_sdf(const Primitive& P, double x, double y, double z) {
  if (P.is_sphere) {
    const double dx = x - P.c[0], dy = y - P.c[1], dz = z - P.c[2];
    return sqrt(sum3(dx * dx, dy * dy, dz * dz)) - P.radius;
  }
  double l[3];
  rigid_apply(P.inv, x, y, z, l);
  const double q0 = fabs(l[0]) - P.he[0], q1 = fabs(l[1]) - P.he[1], q2 = fabs(l[2]) - P.he[2];
  const double o0 = q0 < 0.0 ? 0.0 : q0, o1 = q1 < 0.0 ? 0.0 : q1, o2 = q2 < 0.0 ? 0.0 : q2;  // cwiseMax(0.0)
  double mx = q1 < q2 ? q2 : q1;
  mx = q0 < mx ? mx : q0;
  return sqrt(sum3(o0 * o0, o1 * o1, o2 * o2)) + (0.0 < mx ? 0.0 : mx);  // + std::min(maxCoeff, 0.0)
}

// Effective-sdf predicates of one voxel (query_channel, sdf_world.hpp:481-494;
// seed_threshold, esdf.hpp:69) -> the five digest bits.
__device__ __forceinline__ uint32_t voxel_bits(double sum, double wt, double geom, double seed_thr) {
  const bool dv = wt > 0.0;
  const bool gv = isfinite(geom);
  double best = 0.0;
  if (dv) best = sum / wt;
  if (gv) best = dv ? (geom < best ? geom : best) : geom;  // std::min(best, geom)
  const bool cv = dv || gv;
  uint32_t bits = 0;
  if (cv && fabs(best) < seed_thr) bits |= 1u << kSurface;
  if (gv) bits |= 1u << kGeomValid;
  if (gv && geom < 0.0) bits |= 1u << kGeomNeg;
  if (cv) bits |= 1u << kCombValid;
  if (cv && best < 0.0) bits |= 1u << kCombNeg;
  return bits;
}

// One warp = 32 consecutive voxels = one surface word and two words of each 2-bit pair plane.  A pair word interleaves
// {has value, negative} of 16 voxels: lane j fetches the predicate bits of voxel (j >> 1) of its half and votes with the
// bit it stands for (even lanes: has value, odd lanes: negative) -- the ballot IS the interleaved word.
__device__ __forceinline__ void store_digest(uint32_t* digest, int pool, int tid, uint32_t bits) {
  const int word = tid >> 5, lane = tid & 31;
  const uint32_t surf = __ballot_sync(0xFFFFFFFFu, (bits >> kSurface) & 1u);
  const uint32_t lo = __shfl_sync(0xFFFFFFFFu, bits, lane >> 1), hi = __shfl_sync(0xFFFFFFFFu, bits, 16 + (lane >> 1));
  const int odd = lane & 1;
  const uint32_t g0 = __ballot_sync(0xFFFFFFFFu, (lo >> (kGeomValid + odd)) & 1u), g1 = __ballot_sync(0xFFFFFFFFu, (hi >> (kGeomValid + odd)) & 1u);
  const uint32_t c0 = __ballot_sync(0xFFFFFFFFu, (lo >> (kCombValid + odd)) & 1u), c1 = __ballot_sync(0xFFFFFFFFu, (hi >> (kCombValid + odd)) & 1u);
  uint32_t* d = digest + static_cast<size_t>(pool) * kDigestWords;
  if (lane == 0) d[word] = surf;
  if (lane == 1) d[kDigestGeom + 2 * word] = g0;
  if (lane == 2) d[kDigestGeom + 2 * word + 1] = g1;
  if (lane == 3) d[kDigestComb + 2 * word] = c0;
  if (lane == 4) d[kDigestComb + 2 * word + 1] = c1;
}

__device__ __forceinline__ bool op_blocked(const TsdfView& T) {
  const TsdfCtrl* c = T.ctrl;
  // pool exhaustion (allocate_keys, sdf_world.hpp:315-318) and a table without room are both
  // decided before anything is inserted, so a failing op leaves the world untouched
  return c->abort_op != 0 || c->fresh > c->free_count + (T.capacity - c->next_fresh) || c->live + c->fresh > T.nslots;
}

// atomicAdd(counter, 1) for every calling lane with ONE atomic per converged group of lanes: the op counters are single
// addresses, and a warp of k_stamp_candidates appends up to 32 blocks at once.
__device__ __forceinline__ int grouped_increment(int* counter) {
  cg::coalesced_group g = cg::coalesced_threads();
  int base = 0;
  if (g.thread_rank() == 0) base = atomicAdd(counter, static_cast<int>(g.size()));
  return g.shfl(base, 0) + static_cast<int>(g.thread_rank());
}

// Record a block the op touches; new blocks also join the allocation list.
__device__ __forceinline__ void note_block(const TsdfView& T, const OpLists& L, int bx, int by, int bz, uint32_t slot) {
  const int pool = table_find(T, bx, by, bz);
  const int idx = grouped_increment(&T.ctrl->touched);
  if (idx < L.cap) {
    L.key[idx] = pack_key(bx, by, bz);
    L.pool[idx] = pool;
    L.slot[idx] = slot;
  }
  if (pool < 0) {
    const int j = grouped_increment(&T.ctrl->fresh);
    if (j < L.cap) L.fresh_idx[j] = idx;
  }
}

// ---- phase 1+2: block discovery along rays + dedup (sdf_world.hpp:346-361, :308-311) ----
__global__ void __launch_bounds__(256, 6) k_discover(TsdfView T, OpLists L, const FrameParams* __restrict__ Fp,
                                                  const float* __restrict__ depth) {
  pdl_enter();
  const FrameParams& F = *Fp;
  const int pix = blockIdx.x * blockDim.x + threadIdx.x;
  if (pix >= F.width * F.height) return;
  const float d = depth[pix];
  if (!depth_valid(d)) return;
  const int px = pix % F.width, py = pix / F.width;
  const double dd = static_cast<double>(d);
  const double sx = (px - F.cx) * dd / F.fx, sy = (py - F.cy) * dd / F.fy, sz = dd;
  double ux = sx, uy = sy, uz = sz;  // normalized()
  {
    const double z = sum3(sx * sx, sy * sy, sz * sz);
    if (z > 0.0) {
      const double n = sqrt(z);
      ux = sx / n, uy = sy / n, uz = sz / n;
    }
  }
  uint64_t prev = kKeyEmpty;
  for (int s = -F.half_samples; s <= F.half_samples; ++s) {
    double off = s * F.step;
    off = off < -T.trunc ? -T.trunc : (T.trunc < off ? T.trunc : off);  // std::clamp
    double w[3];
    rigid_apply(F.c2w, sx + off * ux, sy + off * uy, sz + off * uz, w);
    const int bx = voxel_index(w[0], T.voxel) >> 3, by = voxel_index(w[1], T.voxel) >> 3,
              bz = voxel_index(w[2], T.voxel) >> 3;  // floor_div(v, 8) == arithmetic shift
    if (!key_in_range(bx, by, bz)) {
      T.ctrl->abort_op = 1;
      continue;
    }
    const uint64_t key = pack_key(bx, by, bz);
    if (key == prev) continue;
    prev = key;
    uint32_t i = static_cast<uint32_t>(mix64(key)) & L.fset_mask;
    while (true) {
      const uint64_t cur = L.fset[i];
      if (cur == key) break;
      if (cur == kKeyEmpty) {
        const uint64_t old = atomicCAS(reinterpret_cast<unsigned long long*>(&L.fset[i]), kKeyEmpty, key);
        if (old == kKeyEmpty) {
          note_block(T, L, bx, by, bz, i);
          break;
        }
        if (old == key) break;
      }
      i = (i + 1) & L.fset_mask;
    }
  }
}

// Slot placement identical to the reference's sequential insertion (BlockHashTable::insert,
// sdf_world.hpp:146-172, called in sorted key order by allocate_keys :319-322).  Sequentially, key
// number r lands on the first slot of its probe chain that is Empty or Tombstone and not already
// taken by a key of lower rank (the remembered first tombstone IS that slot whenever one precedes
// the first Empty).  Here every new key claims slots in T.slot_claim with atomicMin(rank): a lower
// rank displaces a higher one, and the displaced key carries on down its chain.  The fixed point is
// the sequential layout, whatever the interleaving.  The table itself (slot_key) is not touched
// until every claim has settled; finalize_slots() then writes the keys.
constexpr uint32_t kNoClaim = 0xFFFFFFFFu;
__device__ void claim_slot(const TsdfView& T, uint64_t key, uint32_t rank, const uint64_t* rank_key, int lane) {
  const uint32_t nslots = static_cast<uint32_t>(T.nslots);
  int bx, by, bz;
  unpack_key(key, bx, by, bz);
  uint32_t pos = static_cast<uint32_t>(block_hash(bx, by, bz) % nslots);
  uint32_t walked = 0;
  while (walked < 2 * nslots) {  // warp-cooperative: 32 slots per step
    const uint32_t sidx = (pos + lane) % nslots;
    const uint64_t k = T.slot_key[sidx];
    const bool open = (k == kKeyEmpty || k == kKeyTomb) && __ldcg(&T.slot_claim[sidx]) > rank;  // L2: claims move under us
    const uint32_t vote = __ballot_sync(0xFFFFFFFFu, open);
    if (vote == 0) {
      pos = (pos + 32) % nslots;
      walked += 32;
      continue;
    }
    const int first = __ffs(vote) - 1;
    const uint32_t target = (pos + first) % nslots;
    uint32_t old = 0;
    if (lane == 0) old = atomicMin(&T.slot_claim[target], rank);
    old = __shfl_sync(0xFFFFFFFFu, old, 0);
    if (old > rank) {
      if (old == kNoClaim) return;  // placed
      // we displaced the key of rank `old`: it continues from the next slot of ITS chain (same slots onward)
      rank = old;
      key = __ldcg(&rank_key[old]);  // published (fence) before rank `old` could appear in a claim
    }
    // else: a lower rank got there first; either way carry on after this slot
    pos = (target + 1) % nslots;
    walked += first + 1;
  }
}
// Write the settled claims into the table: run by the op's apply kernel before it touches voxels.
__device__ void finalize_slots(const TsdfView& T, const OpLists& L, int n_fresh) {
  const uint32_t nslots = static_cast<uint32_t>(T.nslots);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_fresh; i += gridDim.x * blockDim.x) {
    const int idx = L.fresh_idx[i];
    const uint64_t key = L.key[idx];
    const uint32_t rank = static_cast<uint32_t>(L.fresh_rank[i]);
    int bx, by, bz;
    unpack_key(key, bx, by, bz);
    uint32_t pos = static_cast<uint32_t>(block_hash(bx, by, bz) % nslots);
    for (uint32_t probe = 0; probe < nslots; ++probe) {
      if (T.slot_claim[pos] == rank) {
        T.slot_key[pos] = key;
        T.slot_pool[pos] = L.pool[idx];
        T.slot_claim[pos] = kNoClaim;
        break;
      }
      pos = pos + 1 == nslots ? 0 : pos + 1;
    }
  }
}

// ---- ranks of the new keys ----
// A new block's rank is its place in the order the reference inserts in: sorted by key (allocate_keys,
// sdf_world.hpp:308-322), for a batch of stamps by (first primitive, key).  Up to T.rank_direct (kRankDirect) new keys every CTA counts
// the smaller ones directly.  Above that (a cold start: tens of thousands of new blocks in one call) the direct count is
// quadratic, so the kernel first sorts the new keys in tiles of kSortTile -- tiles are handed out by ticket to whichever
// CTAs are running, a CTA only waits once every ticket is taken, so the wait cannot starve a sorter -- and a rank is the
// sum of one binary search per tile: n * (n / 1024) * 10 probes instead of n * n comparisons.
constexpr int kSortTile = 1024;
constexpr int kRankDirect = 8192;  // default of TsdfView::rank_direct: measured break-even ~12 K new keys (the sort costs ~20 us whatever n)
constexpr int kRankChunk = 8;  // new blocks a CTA ranks together

__device__ __forceinline__ bool rank_less(int pa, uint64_t ka, int pb, uint64_t kb) { return pa < pb || (pa == pb && ka < kb); }

template <bool kBatch>
__device__ void sort_fresh_tiles(const TsdfView& T, const OpLists& L, int n, uint64_t* s_k, uint8_t* s_p) {
  __shared__ int s_ticket;
  const int ntiles = (n + kSortTile - 1) / kSortTile;
  const int tid = threadIdx.x;
  while (true) {
    __syncthreads();
    if (tid == 0) s_ticket = atomicAdd(&T.ctrl->sort_ticket, 1);
    __syncthreads();
    const int tile = s_ticket;
    if (tile >= ntiles) break;
    for (int q = tid; q < kSortTile; q += blockDim.x) {
      const int j = tile * kSortTile + q;
      uint64_t k = ~0ull;
      int p = 255;
      if (j < n) {
        const int idx = L.fresh_idx[j];
        k = L.key[idx];
        p = kBatch ? __ffs(static_cast<int>(L.fmask[L.slot[idx]])) - 1 : 0;
      }
      s_k[q] = k, s_p[q] = static_cast<uint8_t>(p);
    }
    for (int span = 2; span <= kSortTile; span <<= 1)  // bitonic network, ascending by (primitive, key)
      for (int step = span >> 1; step > 0; step >>= 1) {
        __syncthreads();
        for (int q = tid; q < kSortTile; q += blockDim.x) {
          const int other = q ^ step;
          if (other > q) {
            const uint64_t ka = s_k[q], kb = s_k[other];
            const int pa = s_p[q], pb = s_p[other];
            const bool up = (q & span) == 0;
            if (rank_less(pb, kb, pa, ka) == up) s_k[q] = kb, s_k[other] = ka, s_p[q] = static_cast<uint8_t>(pb), s_p[other] = static_cast<uint8_t>(pa);
          }
        }
      }
    __syncthreads();
    for (int q = tid; q < kSortTile; q += blockDim.x) {
      L.sorted_key[tile * kSortTile + q] = s_k[q];
      L.sorted_prim[tile * kSortTile + q] = s_p[q];
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) atomicAdd(&T.ctrl->sort_done, 1);
  }
  if (tid == 0) {
    while (*reinterpret_cast<volatile int*>(&T.ctrl->sort_done) < ntiles) __nanosleep(200);
    __threadfence();
  }
  __syncthreads();
}

// Allocation proper, shared by integrate and stamps: a CTA takes kRankChunk new blocks at a time, ranks them, and for each
// one picks the pool index (free list LIFO first, then fresh), lets warp 0 claim the key's hash slot with a
// warp-cooperative probe (32 slots per step, ballot, one atomicMin; see claim_slot) and resets the block
// (VoxelBlock::reset, sdf_world.hpp:70-74).  Blocks whose first primitive is >= kstar are not allocated (batched stamps).
template <bool kBatch>
__device__ void allocate_fresh(const TsdfView& T, const OpLists& L, int n, int kstar, int free_count, int next_fresh) {
  __shared__ uint64_t s_k[kSortTile];
  __shared__ uint8_t s_p[kSortTile];
  __shared__ uint64_t s_ckey[kRankChunk];
  __shared__ int s_cprim[kRankChunk], s_cidx[kRankChunk], s_below[kRankChunk];
  const int tid = threadIdx.x;
  const bool direct = n <= T.rank_direct;
  const int ntiles = (n + kSortTile - 1) / kSortTile;
  if (!direct) sort_fresh_tiles<kBatch>(T, L, n, s_k, s_p);
  for (int base = blockIdx.x * kRankChunk; base < n; base += gridDim.x * kRankChunk) {
    const int m = min(kRankChunk, n - base);
    __syncthreads();  // the previous chunk is done with the arrays below
    if (tid < kRankChunk) {
      s_below[tid] = 0;
      if (tid < m) {
        const int idx = L.fresh_idx[base + tid];
        s_cidx[tid] = idx;
        s_ckey[tid] = L.key[idx];
        s_cprim[tid] = kBatch ? __ffs(static_cast<int>(L.fmask[L.slot[idx]])) - 1 : 0;
      }
    }
    __syncthreads();
    if (direct) {
      int cnt[kRankChunk];
#pragma unroll
      for (int e = 0; e < kRankChunk; ++e) cnt[e] = 0;
      for (int j = tid; j < n; j += blockDim.x) {
        const int jdx = L.fresh_idx[j];
        const uint64_t kj = L.key[jdx];
        const int pj = kBatch ? __ffs(static_cast<int>(L.fmask[L.slot[jdx]])) - 1 : 0;
#pragma unroll
        for (int e = 0; e < kRankChunk; ++e) cnt[e] += e < m && rank_less(pj, kj, s_cprim[e], s_ckey[e]);
      }
#pragma unroll
      for (int e = 0; e < kRankChunk; ++e) {
        int c = cnt[e];
        for (int d = 16; d > 0; d >>= 1) c += __shfl_down_sync(0xFFFFFFFFu, c, d);
        if ((tid & 31) == 0 && c) atomicAdd(&s_below[e], c);
      }
    } else {
      for (int pair = tid; pair < m * ntiles; pair += blockDim.x) {  // one binary search per (block, tile)
        const int e = pair / ntiles, tile = pair - e * ntiles;
        const uint64_t key = s_ckey[e];
        const int mine = s_cprim[e];
        const uint64_t* tk = L.sorted_key + static_cast<size_t>(tile) * kSortTile;
        const uint8_t* tp = L.sorted_prim + static_cast<size_t>(tile) * kSortTile;
        int lo = 0, hi = kSortTile;  // first element that is not smaller
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (rank_less(__ldcg(&tp[mid]), __ldcg(&tk[mid]), mine, key)) lo = mid + 1;
          else hi = mid;
        }
        if (lo) atomicAdd(&s_below[e], lo);
      }
    }
    __syncthreads();
    for (int e = 0; e < m; ++e) {
      const int i = base + e, idx = s_cidx[e];
      if (s_cprim[e] >= kstar) {  // its primitive is not applied: the block is not allocated
        if (tid == 0) L.fresh_rank[i] = -1;
        continue;
      }
      const uint64_t key = s_ckey[e];
      const int r = s_below[e];
      const int pool = r < free_count ? T.free_list[free_count - 1 - r] : next_fresh + (r - free_count);
      if (tid < 32) {
        if (tid == 0) {
          L.fresh_rank[i] = r;
          L.rank_key[r] = key;
          L.pool[idx] = pool;
          T.pool_key[pool] = key;
          __threadfence();  // the key of a rank is visible before that rank can be seen in a claim
        }
        __syncwarp();
        claim_slot(T, key, static_cast<uint32_t>(r), L.rank_key, tid);
      }
      // reset the block: sum = wt = 0, geom = +inf, digest = 0
      double2* sw = T.sumwt + static_cast<size_t>(pool) * kBlockVoxels;
      double* g = T.geom + static_cast<size_t>(pool) * kBlockVoxels;
      for (int q = tid; q < kBlockVoxels; q += blockDim.x) {
        sw[q] = make_double2(0.0, 0.0);
        g[q] = CUDART_INF;
      }
      if (tid < kDigestWords) T.digest[static_cast<size_t>(pool) * kDigestWords + tid] = 0;
      if (tid == 0) T.pool_geom[pool] = 0;
    }
  }
}

// ---- phase 3: allocation of the frame's new blocks (allocate_keys, sdf_world.hpp:307-323) ----
__global__ void __launch_bounds__(256) k_commit(TsdfView T, OpLists L) {
  pdl_enter();
  if (op_blocked(T)) return;
  const TsdfCtrl* c = T.ctrl;
  allocate_fresh<false>(T, L, min(c->fresh, L.cap), 0x7FFFFFFF, c->free_count, c->next_fresh);
}

// Op tail, run by the last CTA of the apply kernel: commit the counters or surface the error
// (allocate_keys' all-or-nothing check, sdf_world.hpp:312-318) and reset the per-op state.
__device__ void finish_op(const TsdfView& T, int list_cap, int is_integrate) {
  TsdfCtrl* c = T.ctrl;
  const int avail = c->free_count + (T.capacity - c->next_fresh);
  int status = 0;
  if (c->abort_op) {
    status = c->err != 0 ? c->err : static_cast<int>(KS_ERR_RANGE);
  } else if (c->fresh > avail || c->touched > list_cap) {
    status = KS_ERR_POOL_EXHAUSTED;
    if (c->err == 0) {
      c->err_required = c->fresh;
      c->err_available = avail;
    }
  } else if (c->live + c->fresh > T.nslots) {
    status = KS_ERR_TABLE_FULL;
  } else {
    const int from_free = min(c->fresh, c->free_count);
    c->free_count -= from_free;
    c->next_fresh += c->fresh - from_free;
    c->live += c->fresh;
  }
  if (status != 0 && c->err == 0) c->err = status;
  if (is_integrate) c->last_touched = status == 0 ? c->touched : -1;
  c->touched = 0;
  c->fresh = 0;
  c->abort_op = 0;
  c->sort_ticket = 0, c->sort_done = 0;
}
// Every CTA calls this after its last block; the final arrival runs finish_op.
__device__ __forceinline__ void arrive_and_finish(const TsdfView& T, int list_cap, int is_integrate) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&T.ctrl->arrivals, 1) == static_cast<int>(gridDim.x) - 1) {
      T.ctrl->arrivals = 0;
      __threadfence();
      finish_op(T, list_cap, is_integrate);
    }
  }
}

// ---- phase 4: voxel-centric projective integration (sdf_world.hpp:368-387) ----
// One CTA per touched block, one thread per voxel: each thread owns its voxel,
// so there are no atomics; {sum, wt} moves as one 16-byte access per thread.
__global__ void __launch_bounds__(512, 3) k_integrate(TsdfView T, OpLists L, const FrameParams* __restrict__ Fp,
                                                   const float* __restrict__ depth) {
  pdl_enter();
  __shared__ FrameParams F;
  if (threadIdx.x < sizeof(FrameParams) / 4)
    reinterpret_cast<uint32_t*>(&F)[threadIdx.x] = reinterpret_cast<const uint32_t*>(Fp)[threadIdx.x];
  __syncthreads();
  const int touched = min(T.ctrl->touched, L.cap);
  const bool blocked = op_blocked(T);
  if (!blocked) finalize_slots(T, L, min(T.ctrl->fresh, L.cap));
  const int tid = threadIdx.x;
  const int lx = tid & 7, ly = (tid >> 3) & 7, lz = tid >> 6;
  const double v = T.voxel, trunc = T.trunc;
  for (int i = blockIdx.x; i < touched; i += gridDim.x) {
    if (tid == 0 && L.slot[i] != kNoSlot) L.fset[L.slot[i]] = kKeyEmpty;  // leave the frame set clean
    if (blocked) continue;
    const int pool = L.pool[i];
    int bx, by, bz;
    unpack_key(L.key[i], bx, by, bz);
    const size_t at = static_cast<size_t>(pool) * kBlockVoxels + tid;
    double2 sw = T.sumwt[at];
    const double geom = T.geom[at];
    // voxel_center (sdf_world.hpp:265-272)
    double c[3];
    rigid_apply(F.w2c, (bx * kBlockEdge + lx + 0.5) * v, (by * kBlockEdge + ly + 0.5) * v,
                (bz * kBlockEdge + lz + 0.5) * v, c);
    if (c[2] > 0.0) {
      const int px = static_cast<int>(lround(F.fx * c[0] / c[2] + F.cx));
      const int py = static_cast<int>(lround(F.fy * c[1] / c[2] + F.cy));
      if (px >= 0 && px < F.width && py >= 0 && py < F.height) {
        const float d = __ldg(depth + static_cast<size_t>(py) * F.width + px);
        if (depth_valid(d)) {
          const double sd_raw = static_cast<double>(d) - c[2];
          if (!(sd_raw < -trunc)) {
            const double sd = trunc < sd_raw ? trunc : sd_raw;  // std::min(sd_raw, trunc)
            const double cc = (F.fx * v / c[2]) * (F.fy * v / c[2]);
            const double w = cc < 1.0 ? 1.0 : cc;  // std::max(c, 1.0)
            sw.x += w * sd;
            sw.y += w;
            T.sumwt[at] = sw;
          }
        }
      }
    }
    store_digest(T.digest, pool, tid, voxel_bits(sw.x, sw.y, geom, T.seed_thr));
  }
  arrive_and_finish(T, L.cap, 1);
}

// ---- stamp: candidate blocks in the primitive's padded AABB (sdf_world.hpp:421-434) ----
struct BlockBox {
  int lo[3], n[3];
  long long count;
};
__global__ void __launch_bounds__(256) k_stamp_candidates(TsdfView T, OpLists L, Primitive P, BlockBox B, double reach) {
  pdl_enter();
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < B.count;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int bx = B.lo[0] + static_cast<int>(i % B.n[0]);
    const int by = B.lo[1] + static_cast<int>((i / B.n[0]) % B.n[1]);
    const int bz = B.lo[2] + static_cast<int>(i / (static_cast<long long>(B.n[0]) * B.n[1]));
    // block_center (sdf_world.hpp:282-286)
    const double sd = prim_sdf(P, (bx * kBlockEdge + 0.5 * kBlockEdge) * T.voxel,
                               (by * kBlockEdge + 0.5 * kBlockEdge) * T.voxel,
                               (bz * kBlockEdge + 0.5 * kBlockEdge) * T.voxel);
    if (!(fabs(sd) <= reach)) continue;
    if (!key_in_range(bx, by, bz)) {
      T.ctrl->abort_op = 1;
      continue;
    }
    note_block(T, L, bx, by, bz, kNoSlot);
  }
}

// ---- stamp: per-voxel min with the analytic distance (sdf_world.hpp:437-443) ----
__global__ void __launch_bounds__(512) k_stamp_blocks(TsdfView T, OpLists L, Primitive P) {
  pdl_enter();
  const int touched = op_blocked(T) ? 0 : min(T.ctrl->touched, L.cap);
  if (!op_blocked(T)) finalize_slots(T, L, min(T.ctrl->fresh, L.cap));
  const int tid = threadIdx.x;
  const int lx = tid & 7, ly = (tid >> 3) & 7, lz = tid >> 6;
  const double v = T.voxel;
  for (int i = blockIdx.x; i < touched; i += gridDim.x) {
    const int pool = L.pool[i];
    int bx, by, bz;
    unpack_key(L.key[i], bx, by, bz);
    const size_t at = static_cast<size_t>(pool) * kBlockVoxels + tid;
    const double sd = prim_sdf(P, (bx * kBlockEdge + lx + 0.5) * v, (by * kBlockEdge + ly + 0.5) * v,
                               (bz * kBlockEdge + lz + 0.5) * v);
    double g = T.geom[at];
    if (sd < g) {  // std::min(geom, sd)
      g = sd;
      T.geom[at] = g;
    }
    const double2 sw = T.sumwt[at];
    store_digest(T.digest, pool, tid, voxel_bits(sw.x, sw.y, g, T.seed_thr));
    if (tid == 0) T.pool_geom[pool] = 1;  // every voxel of a stamped block holds a finite distance
  }
  arrive_and_finish(T, L.cap, 0);
}

// ---- batched stamps: every primitive of an update in three launches ----
// stamp_primitive (sdf_world.hpp:394-444) applied to primitives 0 .. n-1 in order, stopping at the first one that
// would throw: the result -- pool indices, hash slots, free list, every voxel, the error and its numbers -- is that of
// the sequential calls.  A new block belongs to the FIRST primitive that touches it; new blocks are ranked by
// (first primitive, key), which is the order in which the sequential calls would insert them (each call sorted,
// sdf_world.hpp:308-322), so the rank-priority slot claims and the pool numbering of k_commit carry over unchanged.
// Primitive k* fails when the new blocks of primitives 0 .. k* no longer fit (or one of its blocks is out of range);
// primitives >= k* are then not applied and k*'s own numbers are reported, exactly as its allocate_keys would.
constexpr int kMaxBatch = 16;
struct BatchPrims {
  Primitive prim[kMaxBatch];
  BlockBox box[kMaxBatch];
  long long offset[kMaxBatch + 1];  // candidate positions of primitive k: [offset[k], offset[k+1])
  int n;
};

// (the batch travels as a __grid_constant__ parameter: the kernels index it at run time straight from the constant bank)
__global__ void __launch_bounds__(256) k_batch_candidates(TsdfView T, OpLists L, const __grid_constant__ BatchPrims PB, double reach) {
  pdl_enter();
  if (T.ctrl->batch_stop) return;  // an earlier group of the same call failed: the reference would not get this far
  const long long total = PB.offset[PB.n];
  for (long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<long long>(gridDim.x) * blockDim.x) {
    int k = 0;
    while (g >= PB.offset[k + 1]) ++k;
    const BlockBox& B = PB.box[k];
    const long long i = g - PB.offset[k];
    const int bx = B.lo[0] + static_cast<int>(i % B.n[0]);
    const int by = B.lo[1] + static_cast<int>((i / B.n[0]) % B.n[1]);
    const int bz = B.lo[2] + static_cast<int>(i / (static_cast<long long>(B.n[0]) * B.n[1]));
    const double sd = prim_sdf(PB.prim[k], (bx * kBlockEdge + 0.5 * kBlockEdge) * T.voxel,
                               (by * kBlockEdge + 0.5 * kBlockEdge) * T.voxel, (bz * kBlockEdge + 0.5 * kBlockEdge) * T.voxel);
    if (!(fabs(sd) <= reach)) continue;
    if (!key_in_range(bx, by, bz)) {
      atomicMin(&T.ctrl->abort_prim, k);
      continue;
    }
    const uint64_t key = pack_key(bx, by, bz);
    uint32_t slot = static_cast<uint32_t>(mix64(key)) & L.fset_mask;
    while (true) {
      const uint64_t cur = L.fset[slot];
      if (cur == key) break;
      if (cur == kKeyEmpty) {
        const uint64_t old = atomicCAS(reinterpret_cast<unsigned long long*>(&L.fset[slot]), kKeyEmpty, key);
        if (old == kKeyEmpty) {
          note_block(T, L, bx, by, bz, slot);
          break;
        }
        if (old == key) break;
      }
      slot = (slot + 1) & L.fset_mask;
    }
    atomicOr(&L.fmask[slot], 1u << k);
  }
}

// what the batch may apply: k* and the numbers behind it, from the per-primitive counts of new blocks
struct BatchVerdict {
  int kstar;      // primitives [0, kstar) are applied
  int allocated;  // new blocks of those primitives
  int status, required, available;
};
__device__ BatchVerdict batch_verdict(const TsdfView& T, const int* hist, int nprims, int touched, int list_cap) {
  const TsdfCtrl* c = T.ctrl;
  BatchVerdict v;
  v.kstar = nprims, v.allocated = 0, v.status = 0, v.required = 0, v.available = 0;
  int avail = c->free_count + (T.capacity - c->next_fresh), room = T.nslots - c->live;
  if (c->batch_stop) {
    v.kstar = 0;
    return v;
  }
  if (touched > list_cap) {  // the op lists overflowed: nothing of this batch can be trusted
    v.kstar = 0, v.status = KS_ERR_POOL_EXHAUSTED, v.required = touched, v.available = avail;
    return v;
  }
  for (int k = 0; k < nprims; ++k) {
    if (k >= c->abort_prim) {
      v.kstar = k, v.status = KS_ERR_RANGE;
      return v;
    }
    if (hist[k] > avail) {
      v.kstar = k, v.status = KS_ERR_POOL_EXHAUSTED, v.required = hist[k], v.available = avail;
      return v;
    }
    if (hist[k] > room) {
      v.kstar = k, v.status = KS_ERR_TABLE_FULL;
      return v;
    }
    avail -= hist[k], room -= hist[k], v.allocated += hist[k];
  }
  return v;
}

__device__ __forceinline__ int first_prim(const OpLists& L, int idx) { return __ffs(static_cast<int>(L.fmask[L.slot[idx]])) - 1; }

// Allocation of a batch: k_commit with the rank taken over (first primitive, key) and the verdict above.
__global__ void __launch_bounds__(256) k_batch_commit(TsdfView T, OpLists L, int nprims) {
  pdl_enter();
  const TsdfCtrl* c = T.ctrl;
  const int n = min(c->fresh, L.cap);
  if (n == 0 && blockIdx.x != 0) return;
  __shared__ int s_hist[kMaxBatch];
  __shared__ BatchVerdict s_v;
  if (threadIdx.x < kMaxBatch) s_hist[threadIdx.x] = 0;
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += blockDim.x) atomicAdd(&s_hist[first_prim(L, L.fresh_idx[j])], 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    s_v = batch_verdict(T, s_hist, nprims, c->touched, L.cap);
    if (blockIdx.x == 0) {  // for the apply kernel and its tail
      TsdfCtrl* w = T.ctrl;
      w->batch_kstar = s_v.kstar, w->batch_alloc = s_v.allocated, w->batch_status = s_v.status;
      w->batch_required = s_v.required, w->batch_available = s_v.available;
    }
  }
  __syncthreads();
  const BatchVerdict v = s_v;
  allocate_fresh<true>(T, L, n, v.kstar, c->free_count, c->next_fresh);
}

__device__ void finish_batch(const TsdfView& T, int last_group) {
  TsdfCtrl* c = T.ctrl;
  if (c->batch_status != 0 && c->err == 0) {
    c->err = c->batch_status;
    c->err_required = c->batch_required, c->err_available = c->batch_available;
  }
  if (last_group) c->batch_stop = 0;
  else if (c->batch_status != 0) c->batch_stop = 1;  // the remaining groups of this call do nothing
  const int from_free = min(c->batch_alloc, c->free_count);
  c->free_count -= from_free;
  c->next_fresh += c->batch_alloc - from_free;
  c->live += c->batch_alloc;
  c->touched = 0;
  c->fresh = 0;
  c->abort_prim = 0x7FFFFFFF;
  c->sort_ticket = 0, c->sort_done = 0;
}

// Voxels of a batch: one CTA per touched block, the per-voxel min (sdf_world.hpp:437-443) over the applied
// primitives that touch it, one digest refresh.
__global__ void __launch_bounds__(512) k_batch_blocks(TsdfView T, OpLists L, const __grid_constant__ BatchPrims PB, int last_group) {
  pdl_enter();
  const int touched = min(T.ctrl->touched, L.cap);
  const int kstar = T.ctrl->batch_kstar;
  {  // settled claims -> table (finalize_slots, skipping the blocks that were not allocated)
    const uint32_t nslots = static_cast<uint32_t>(T.nslots);
    const int n_fresh = min(T.ctrl->fresh, L.cap);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_fresh; i += gridDim.x * blockDim.x) {
      const int rank_i = L.fresh_rank[i];
      if (rank_i < 0) continue;
      const int idx = L.fresh_idx[i];
      const uint64_t key = L.key[idx];
      int bx, by, bz;
      unpack_key(key, bx, by, bz);
      uint32_t pos = static_cast<uint32_t>(block_hash(bx, by, bz) % nslots);
      for (uint32_t probe = 0; probe < nslots; ++probe) {
        if (T.slot_claim[pos] == static_cast<uint32_t>(rank_i)) {
          T.slot_key[pos] = key;
          T.slot_pool[pos] = L.pool[idx];
          T.slot_claim[pos] = kNoClaim;
          break;
        }
        pos = pos + 1 == nslots ? 0 : pos + 1;
      }
    }
  }
  const int tid = threadIdx.x;
  const int lx = tid & 7, ly = (tid >> 3) & 7, lz = tid >> 6;
  const double v = T.voxel;
  const uint32_t applied = kstar >= 32 ? 0xFFFFFFFFu : (1u << kstar) - 1u;
  for (int i = blockIdx.x; i < touched; i += gridDim.x) {
    const uint32_t slot = L.slot[i];
    const uint32_t mask = L.fmask[slot] & applied;  // the same word for the whole CTA
    if (mask != 0) {
      const int pool = L.pool[i];
      int bx, by, bz;
      unpack_key(L.key[i], bx, by, bz);
      const size_t at = static_cast<size_t>(pool) * kBlockVoxels + tid;
      const double g0 = T.geom[at];
      const double2 sw = T.sumwt[at];
      const double x = (bx * kBlockEdge + lx + 0.5) * v, y = (by * kBlockEdge + ly + 0.5) * v, z = (bz * kBlockEdge + lz + 0.5) * v;
      double g = g0;
      for (uint32_t m = mask; m != 0; m &= m - 1) {
        const double sd = prim_sdf(PB.prim[__ffs(static_cast<int>(m)) - 1], x, y, z);
        if (sd < g) g = sd;  // std::min(geom, sd)
      }
      if (g < g0) T.geom[at] = g;
      store_digest(T.digest, pool, tid, voxel_bits(sw.x, sw.y, g, T.seed_thr));
      if (tid == 0) T.pool_geom[pool] = 1;  // every voxel of a stamped block holds a finite distance
    }
    __syncthreads();  // every warp has read the block's mask: leave the set clean
    if (tid == 0) L.fmask[slot] = 0u, L.fset[slot] = kKeyEmpty;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&T.ctrl->arrivals, 1) == static_cast<int>(gridDim.x) - 1) {
      T.ctrl->arrivals = 0;
      __threadfence();
      finish_batch(T, last_group);
    }
  }
}

// ---- mesh stamp (no reference implementation; definition in mesh.cuh, flow of sdf_world.hpp:418-443) ----
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
  return v;
}
// Candidate blocks: one warp per block of the padded AABB.  Bounding spheres first (the nearest triangle is no
// farther than ub = min(d + r); nothing is nearer than min(d - r)), then exact distances of the triangles that can
// be the nearest one, lanes striding over them.  Only the magnitude matters here: |sdf(centre)| <= reach.
__global__ void __launch_bounds__(256) k_stamp_mesh_candidates(TsdfView T, OpLists L, MeshView M, BlockBox B, double reach) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  for (long long i = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5; i < B.count; i += nwarps) {
    const int bx = B.lo[0] + static_cast<int>(i % B.n[0]);
    const int by = B.lo[1] + static_cast<int>((i / B.n[0]) % B.n[1]);
    const int bz = B.lo[2] + static_cast<int>(i / (static_cast<long long>(B.n[0]) * B.n[1]));
    const V3 q = v3((bx * kBlockEdge + 0.5 * kBlockEdge) * T.voxel, (by * kBlockEdge + 0.5 * kBlockEdge) * T.voxel,
                    (bz * kBlockEdge + 0.5 * kBlockEdge) * T.voxel);  // block_center (sdf_world.hpp:282-286)
    double ub = CUDART_INF, lb = CUDART_INF;
    for (int j = lane; j < M.nt; j += 32) {
      double r;
      const double d = mesh_bound(M, j, q, r);
      ub = fmin(ub, d + r), lb = fmin(lb, d - r);
    }
    ub = warp_min(ub), lb = warp_min(lb);
    if (lb > reach * kMeshSlack) continue;
    const double thr = ub * kMeshSlack;
    MeshHit best = {CUDART_INF, 0x7FFFFFFF, 0, v3(0.0, 0.0, 0.0)};
    for (int j = lane; j < M.nt; j += 32) {
      double r;
      if (mesh_bound(M, j, q, r) - r <= thr) mesh_visit(M, j, q, best);
    }
    const double d2 = warp_min(best.d2);
    if (lane != 0 || !(sqrt(d2) <= reach)) continue;
    if (!key_in_range(bx, by, bz)) {
      T.ctrl->abort_op = 1;
      continue;
    }
    note_block(T, L, bx, by, bz, kNoSlot);
  }
}

// Per-voxel min with the mesh distance: one CTA per touched block, one thread per voxel.  Triangles whose bounding
// sphere is farther from the block centre than (nearest possible + block diameter) cannot be the nearest one of any
// voxel of the block; the others are listed in shared memory, a chunk at a time, and every thread walks the list
// (all lanes read the same triangle: one broadcast load).
constexpr int kMeshThreads = 256;  // half a block per CTA: three CTAs fit an SM's registers, and 2K items balance better than K
constexpr int kMeshParts = kBlockVoxels / kMeshThreads;
constexpr int kMeshChunk = kMeshThreads;
constexpr int kMeshRow = 13;  // centre xyz, radius, a, b, c
__global__ void __launch_bounds__(kMeshThreads, 3) k_stamp_mesh_blocks(TsdfView T, OpLists L, MeshView M) {
  pdl_enter();
  __shared__ double s_tri[kMeshChunk * kMeshRow];
  __shared__ int s_idx[kMeshChunk];
  __shared__ int s_count;
  __shared__ double s_red[kMeshThreads / 32];
  const int touched = op_blocked(T) ? 0 : min(T.ctrl->touched, L.cap);
  if (!op_blocked(T)) finalize_slots(T, L, min(T.ctrl->fresh, L.cap));
  const int tid = threadIdx.x;
  const double v = T.voxel;
  const double radius = 0.5 * kBlockEdge * v * sqrt(3.0) * kMeshSlack;
  for (int item = blockIdx.x; item < touched * kMeshParts; item += gridDim.x) {
    const int i = item / kMeshParts, voxel = (item % kMeshParts) * kMeshThreads + tid;
    const int lx = voxel & 7, ly = (voxel >> 3) & 7, lz = voxel >> 6;
    const int pool = L.pool[i];
    int bx, by, bz;
    unpack_key(L.key[i], bx, by, bz);
    const V3 q = v3((bx * kBlockEdge + 0.5 * kBlockEdge) * v, (by * kBlockEdge + 0.5 * kBlockEdge) * v, (bz * kBlockEdge + 0.5 * kBlockEdge) * v);
    double ub = CUDART_INF;
    for (int j = tid; j < M.nt; j += kMeshThreads) {
      double r;
      const double d = mesh_bound(M, j, q, r);
      ub = fmin(ub, d + r);
    }
    ub = warp_min(ub);
    __syncthreads();  // s_red and the list of the previous item are no longer read
    if ((tid & 31) == 0) s_red[tid >> 5] = ub;
    __syncthreads();
    ub = s_red[0];
#pragma unroll
    for (int w = 1; w < kMeshThreads / 32; ++w) ub = fmin(ub, s_red[w]);
    const double thr = (ub + 2.0 * radius) * kMeshSlack;
    const V3 p = v3((bx * kBlockEdge + lx + 0.5) * v, (by * kBlockEdge + ly + 0.5) * v, (bz * kBlockEdge + lz + 0.5) * v);  // voxel_center (:265-272)
    MeshHit best = {CUDART_INF, 0x7FFFFFFF, 0, v3(0.0, 0.0, 0.0)};
    double reach = (ub + radius) * kMeshSlack;  // every voxel of the block is within ub + radius of the mesh
    for (int base = 0; base < M.nt; base += kMeshChunk) {
      __syncthreads();
      if (tid == 0) s_count = 0;
      __syncthreads();
      const int j = base + tid;
      if (j < M.nt) {  // listed triangles travel to shared memory with their bounding sphere
        const double2 b0 = __ldg(reinterpret_cast<const double2*>(M.bnd) + 2 * j), b1 = __ldg(reinterpret_cast<const double2*>(M.bnd) + 2 * j + 1);
        const V3 d = v3(q.x - b0.x, q.y - b0.y, q.z - b1.x);
        if (sqrt(v3_dot(d, d)) - b1.y <= thr) {
          const int slot = atomicAdd(&s_count, 1);
          double* S = s_tri + slot * kMeshRow;
          S[0] = b0.x, S[1] = b0.y, S[2] = b1.x, S[3] = b1.y;
          const double* G = M.tri + 9 * static_cast<size_t>(j);
#pragma unroll
          for (int c = 0; c < 9; ++c) S[4 + c] = __ldg(G + c);
          s_idx[slot] = j;
        }
      }
      __syncthreads();
      const int n = s_count;
      for (int k = 0; k < n; ++k) {
        const double* S = s_tri + k * kMeshRow;
        const V3 d = v3(p.x - S[0], p.y - S[1], p.z - S[2]);
        const double far = reach + S[3];
        if (v3_dot(d, d) > far * far) continue;  // no point of this triangle can be nearer than the best so far
        int feature;
        const V3 c = closest_on_triangle(p, v3(S[4], S[5], S[6]), v3(S[7], S[8], S[9]), v3(S[10], S[11], S[12]), feature);
        const V3 diff = v3_sub(p, c);
        const double d2 = v3_dot(diff, diff);
        const int tri = s_idx[k];
        if (d2 < best.d2 || (d2 == best.d2 && tri < best.tri)) {
          if (d2 < best.d2) reach = fmin(reach, sqrt(d2) * kMeshSlack);
          best.d2 = d2, best.tri = tri, best.feature = feature, best.diff = diff;
        }
      }
    }
    const double sd = mesh_signed(M, best);
    const size_t at = static_cast<size_t>(pool) * kBlockVoxels + voxel;
    double g = T.geom[at];
    if (sd < g) {  // std::min(geom, sd)
      g = sd;
      T.geom[at] = g;
    }
    const double2 sw = T.sumwt[at];
    store_digest(T.digest, pool, voxel, voxel_bits(sw.x, sw.y, g, T.seed_thr));
    if (tid == 0) T.pool_geom[pool] = 1;
  }
  arrive_and_finish(T, L.cap, 0);
}

// ---- decay_weights (sdf_world.hpp:449-457) ----
__global__ void __launch_bounds__(512) k_decay(TsdfView T, Frustum Fr, double alpha_t, double alpha_f) {
  pdl_enter();
  const int bound = T.ctrl->next_fresh;
  const int tid = threadIdx.x;
  for (int pool = blockIdx.x; pool < bound; pool += gridDim.x) {
    const uint64_t key = T.pool_key[pool];
    if (key == kKeyEmpty) continue;
    int bx, by, bz;
    unpack_key(key, bx, by, bz);
    double c[3];
    rigid_apply(Fr.w2c, (bx * kBlockEdge + 0.5 * kBlockEdge) * T.voxel, (by * kBlockEdge + 0.5 * kBlockEdge) * T.voxel,
                (bz * kBlockEdge + 0.5 * kBlockEdge) * T.voxel, c);
    bool inside = true;
#pragma unroll
    for (int p = 0; p < 5; ++p)
      if (sum3(Fr.n[p][0] * c[0], Fr.n[p][1] * c[1], Fr.n[p][2] * c[2]) < -Fr.radius) inside = false;
    double factor = alpha_t;
    if (inside) factor *= alpha_f;
    const size_t at = static_cast<size_t>(pool) * kBlockVoxels + tid;
    double2 sw = T.sumwt[at];
    sw.y *= factor;  // depth_sum is deliberately not scaled (sdf_world.hpp:455)
    T.sumwt[at] = sw;
    store_digest(T.digest, pool, tid, voxel_bits(sw.x, sw.y, T.geom[at], T.seed_thr));
  }
}

// ---- recycle_blocks (sdf_world.hpp:462-475) ----
// weight_total() is a sequential sum (sdf_world.hpp:75-79); it is compared with a
// threshold, so the summation order is kept: one thread walks its block in order.
__global__ void __launch_bounds__(128) k_recycle_flag(TsdfView T, int* flags, double threshold) {
  pdl_enter();
  const int bound = T.ctrl->next_fresh;
  for (int pool = blockIdx.x * blockDim.x + threadIdx.x; pool < bound; pool += gridDim.x * blockDim.x) {
    int flag = 0;
    if (T.pool_key[pool] != kKeyEmpty) {
      const double2* sw = T.sumwt + static_cast<size_t>(pool) * kBlockVoxels;
      const double* g = T.geom + static_cast<size_t>(pool) * kBlockVoxels;
      double total = 0.0;
      bool has_geom = false;
      for (int q = 0; q < kBlockVoxels; ++q) {
        total += sw[q].y;
        has_geom |= isfinite(g[q]);
      }
      flag = total < threshold && !has_geom;
    }
    flags[pool] = flag;
  }
}
// Tombstone flagged blocks in SLOT order and append their pool entries to the free list
// in that order (the reference's iteration order, sdf_world.hpp:464-472).
__global__ void __launch_bounds__(1024) k_recycle_commit(TsdfView T, const int* flags) {
  pdl_enter();
  __shared__ int warp_sum[32];
  __shared__ int s_base;
  TsdfCtrl* c = T.ctrl;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  for (int s0 = 0; s0 < T.nslots; s0 += blockDim.x) {
    const int s = s0 + threadIdx.x;
    int pool = -1, f = 0;
    if (s < T.nslots) {
      const uint64_t k = T.slot_key[s];
      if (k != kKeyEmpty && k != kKeyTomb) {
        pool = T.slot_pool[s];
        f = flags[pool];
      }
    }
    int incl = f;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int up = __shfl_up_sync(0xFFFFFFFFu, incl, d);
      if (lane >= d) incl += up;
    }
    if (lane == 31) warp_sum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int w = warp_sum[lane];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int up = __shfl_up_sync(0xFFFFFFFFu, w, d);
        if (lane >= d) w += up;
      }
      warp_sum[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    const int before = s_base + (warp > 0 ? warp_sum[warp - 1] : 0) + incl - f;
    if (f) {
      T.free_list[c->free_count + before] = pool;
      T.slot_key[s] = kKeyTomb;
      T.slot_pool[s] = -1;
      T.pool_key[pool] = kKeyEmpty;
    }
    __syncthreads();
    if (threadIdx.x == 0) s_base += warp_sum[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    c->free_count += s_base;
    c->live -= s_base;
    c->last_recycled = s_base;
  }
}

// ---- query_tsdf / query_tsdf_geom (sdf_world.hpp:481-507) ----
__global__ void __launch_bounds__(256) k_query_tsdf(TsdfView T, const double* __restrict__ pts, long long n, int geom_only,
                                                    double* __restrict__ out, uint8_t* __restrict__ valid) {
  pdl_enter();
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const int vx = voxel_index(pts[3 * i], T.voxel), vy = voxel_index(pts[3 * i + 1], T.voxel),
            vz = voxel_index(pts[3 * i + 2], T.voxel);
  const int pool = table_find(T, vx >> 3, vy >> 3, vz >> 3);
  double best = 0.0;
  bool have = false;
  if (pool >= 0) {
    const size_t at = static_cast<size_t>(pool) * kBlockVoxels + ((vx & 7) + 8 * ((vy & 7) + 8 * (vz & 7)));
    const double2 sw = T.sumwt[at];
    const double g = T.geom[at];
    if (!geom_only && sw.y > 0.0) {
      best = sw.x / sw.y;
      have = true;
    }
    if (isfinite(g)) {
      best = have ? (g < best ? g : best) : g;
      have = true;
    }
  }
  out[i] = have ? best : 0.0;
  valid[i] = have;
}

__global__ void k_find(TsdfView T, int bx, int by, int bz, int* out) {
  pdl_enter(); *out = table_find(T, bx, by, bz); }

__global__ void k_fill_u64(uint64_t* p, size_t n, uint64_t v) {
  pdl_enter();
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n; i += static_cast<size_t>(gridDim.x) * blockDim.x)
    p[i] = v;
}

// ---- host side ----------------------------------------------------------------------

static bool capturing(cudaStream_t stream) {
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(stream, &cap);
  return cap != cudaStreamCaptureStatusNone;
}
// free now, or -- when a captured graph may still hold the address -- with the handle
static void release_dev(ks_tsdf* t, void* p) {
  if (!p) return;
  if (t->ever_captured) t->retired_dev.push_back(p);
  else cudaFree(p);
}
static void release_host(ks_tsdf* t, void* p) {
  if (!p) return;
  if (t->ever_captured) t->retired_host.push_back(p);
  else cudaFreeHost(p);
}

static int ensure_lists(ks_tsdf* t, size_t pixels, int samples) {
  const size_t want = std::max<size_t>(pixels * samples, 2 * static_cast<size_t>(t->cfg.capacity) + 1);
  if (static_cast<size_t>(t->lists.cap) >= want) return KS_OK;
  if (capturing(t->stream))
    return fail(KS_ERR_INVALID, "tsdf: frame larger than the staged buffers; stage a frame of this size before capture");
  KS_CUDA(cudaStreamSynchronize(t->stream));
  OpLists& L = t->lists;
  for (void* old : {static_cast<void*>(L.key), static_cast<void*>(L.pool), static_cast<void*>(L.slot), static_cast<void*>(L.fresh_idx),
                    static_cast<void*>(L.fresh_rank), static_cast<void*>(L.rank_key), static_cast<void*>(L.sorted_key),
                    static_cast<void*>(L.sorted_prim), static_cast<void*>(L.fset), static_cast<void*>(L.fmask)})
    release_dev(t, old);
  L = OpLists{};
  L.cap = static_cast<int>(want);
  KS_CUDA(cudaMalloc(&L.key, want * sizeof(uint64_t)));
  KS_CUDA(cudaMalloc(&L.pool, want * sizeof(int)));
  KS_CUDA(cudaMalloc(&L.slot, want * sizeof(uint32_t)));
  KS_CUDA(cudaMalloc(&L.fresh_idx, want * sizeof(int)));
  KS_CUDA(cudaMalloc(&L.fresh_rank, want * sizeof(int)));
  KS_CUDA(cudaMalloc(&L.rank_key, want * sizeof(uint64_t)));
  const size_t tiles = (want + kSortTile - 1) / kSortTile * kSortTile;
  KS_CUDA(cudaMalloc(&L.sorted_key, tiles * sizeof(uint64_t)));
  KS_CUDA(cudaMalloc(&L.sorted_prim, tiles));
  uint32_t slots = 1u << 16;
  while (slots < 2 * want) slots <<= 1;
  L.fset_mask = slots - 1;
  KS_CUDA(cudaMalloc(&L.fset, static_cast<size_t>(slots) * sizeof(uint64_t)));
  KS_CUDA(cudaMalloc(&L.fmask, static_cast<size_t>(slots) * sizeof(uint32_t)));
  KS_CUDA(cudaMemsetAsync(L.fmask, 0, static_cast<size_t>(slots) * sizeof(uint32_t), t->stream));
  KS_LAUNCH(k_fill_u64, 1024, 256, 0, t->stream, L.fset, static_cast<size_t>(slots), kKeyEmpty);
  KS_CUDA(cudaStreamSynchronize(t->stream));
  return KS_OK;
}

static int ensure_slot(ks_tsdf* t, int slot, size_t pixels) {
  ks_tsdf::FrameSlot& S = t->slots[slot];
  if (S.h_frame && S.depth_cap >= pixels) return KS_OK;
  if (capturing(t->stream)) return fail(KS_ERR_INVALID, "tsdf: stage every camera slot once before capturing a graph");
  KS_CUDA(cudaStreamSynchronize(t->stream));
  if (!S.h_frame) {
    KS_CUDA(cudaMallocHost(&S.h_frame, sizeof(FrameParams)));
    KS_CUDA(cudaMalloc(&S.d_frame, sizeof(FrameParams)));
  }
  if (S.depth_cap < pixels) {
    if (t->ever_captured && S.depth_cap > 0) {  // the camera parameters a captured graph uploads stay with its pixels
      release_host(t, S.h_frame);
      release_dev(t, S.d_frame);
      S.h_frame = nullptr, S.d_frame = nullptr;
      KS_CUDA(cudaMallocHost(&S.h_frame, sizeof(FrameParams)));
      KS_CUDA(cudaMalloc(&S.d_frame, sizeof(FrameParams)));
    }
    release_host(t, S.h_depth);
    release_dev(t, S.d_depth);
    S.h_depth = nullptr, S.d_depth = nullptr;
    KS_CUDA(cudaMallocHost(&S.h_depth, pixels * sizeof(float)));
    KS_CUDA(cudaMalloc(&S.d_depth, pixels * sizeof(float)));
    S.depth_cap = pixels;
  }
  return KS_OK;
}

static void run_allocation(ks_tsdf* t) { KS_LAUNCH(k_commit, 4 * kSmCount, 256, 0, t->stream, t->view, t->lists); }

static int report_status(const TsdfCtrl& c) {
  switch (c.err) {
    case KS_OK:
      return KS_OK;
    case KS_ERR_POOL_EXHAUSTED:
      return fail(KS_ERR_POOL_EXHAUSTED, "tsdf: pool exhausted, frame requires " + std::to_string(c.err_required) +
                                             " new blocks but only " + std::to_string(c.err_available) + " are available");
    case KS_ERR_TABLE_FULL:
      return fail(KS_ERR_TABLE_FULL, "tsdf: hash table full");
    case KS_ERR_RANGE:
      return fail(KS_ERR_RANGE, "tsdf: block coordinate outside the supported +-2^20 range");
    default:
      return fail(c.err, "tsdf: device error " + std::to_string(c.err));
  }
}

static bool profiling(ks_tsdf* t) {
  if (!t->profile) return false;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(t->stream, &cap);
  return cap == cudaStreamCaptureStatusNone;
}
#define KS_MARK(t, i) \
  if (prof) cudaEventRecord((t)->ev[i], (t)->stream)

static int stamp_async(ks_tsdf* t, const Primitive& P, const double lo_in[3], const double hi_in[3], const ks_mesh* mesh = nullptr) {
  const bool prof = profiling(t);
  t->generation.fetch_add(1, std::memory_order_relaxed);
  wait_for_readers(t);
  KS_MARK(t, 4);
  // AABB grown by the truncation band -> block range (sdf_world.hpp:418-425)
  const double v = t->cfg.voxel_size, trunc = t->cfg.truncation;
  BlockBox B;
  B.count = 1;
  for (int a = 0; a < 3; ++a) {
    const double lo = lo_in[a] - trunc, hi = hi_in[a] + trunc;
    const int blo = voxel_index(lo, v) >> 3, bhi = voxel_index(hi, v) >> 3;
    B.lo[a] = blo;
    B.n[a] = bhi - blo + 1;
    if (B.n[a] < 1) B.n[a] = 0;
    B.count *= B.n[a];
  }
  {  // at most B.count blocks are new: can this stamp fail on the device at all?
    bool safe = t->bounds_valid && B.count <= t->known_avail && B.count <= t->known_room;
    for (int a = 0; a < 3; ++a)
      if (B.lo[a] <= -kKeyBias || B.lo[a] + B.n[a] >= kKeyBias) safe = false;
    if (safe) t->known_avail -= B.count, t->known_room -= B.count;
    else t->bounds_valid = false;  // unknown until the next synchronisation
    t->last_stamp_safe = safe;
  }
  const double reach = trunc + 0.5 * kBlockEdge * v * std::sqrt(3.0);  // sdf_world.hpp:288-290, :425
  if (B.count > 0) {
    if (mesh) {  // one warp per candidate block
      const int grid = static_cast<int>(std::min<long long>((B.count + 7) / 8, 8 * kSmCount));
      KS_LAUNCH(k_stamp_mesh_candidates, grid, 256, 0, t->stream, t->view, t->lists, mesh->view, B, reach);
    } else {
      const int grid = static_cast<int>(std::min<long long>((B.count + 255) / 256, 8 * kSmCount));
      KS_LAUNCH(k_stamp_candidates, grid, 256, 0, t->stream, t->view, t->lists, P, B, reach);
    }
  }
  run_allocation(t);
  KS_MARK(t, 5);
  if (mesh) KS_LAUNCH(k_stamp_mesh_blocks, 3 * kSmCount, kMeshThreads, 0, t->stream, t->view, t->lists, mesh->view);
  else KS_LAUNCH(k_stamp_blocks, 4 * kSmCount, 512, 0, t->stream, t->view, t->lists, P);
  KS_MARK(t, 6);
  KS_CUDA(cudaGetLastError());
  return KS_OK;
}

static bool fill_primitive(const ks_primitive& in, Primitive& P, double lo[3], double hi[3], std::string& why) {
  P = Primitive{};
  if (in.kind == 1) {  // SphereShape
    if (!std::isfinite(in.radius) || !std::isfinite(in.center[0]) || !std::isfinite(in.center[1]) || !std::isfinite(in.center[2])) {
      why = "stamp: non-finite sphere";
      return false;
    }
    P.is_sphere = 1;
    P.radius = in.radius;
    for (int a = 0; a < 3; ++a) P.c[a] = in.center[a], lo[a] = in.center[a] - in.radius, hi[a] = in.center[a] + in.radius;  // sdf_world.hpp:413-416
    return true;
  }
  for (int a = 0; a < 3; ++a)  // the reference checks half_extents and translation (sdf_world.hpp:400)
    if (!std::isfinite(in.pose_t[a]) || !std::isfinite(in.half_extents[a])) why = "stamp: non-finite cuboid";
  if (!why.empty()) return false;
  Rigid pose;
  std::memcpy(pose.r, in.pose_R, sizeof pose.r);
  std::memcpy(pose.t, in.pose_t, sizeof pose.t);
  P.inv = rigid_inverse(pose);
  for (int a = 0; a < 3; ++a) P.he[a] = in.half_extents[a], lo[a] = INFINITY, hi[a] = -INFINITY;
  for (int corner = 0; corner < 8; ++corner) {  // world AABB over the eight corners (sdf_world.hpp:402-411)
    const double sx = (corner & 1) ? 1.0 : -1.0, sy = (corner & 2) ? 1.0 : -1.0, sz = (corner & 4) ? 1.0 : -1.0;
    double w[3];
    rigid_apply(pose, sx * in.half_extents[0], sy * in.half_extents[1], sz * in.half_extents[2], w);
    for (int a = 0; a < 3; ++a) lo[a] = std::min(lo[a], w[a]), hi[a] = std::max(hi[a], w[a]);
  }
  return true;
}

// one group of at most kMaxBatch primitives: candidates, allocation, voxels
static int stamp_group_async(ks_tsdf* t, const ks_primitive* prims, int n, bool last_group) {
  const bool prof = profiling(t);
  t->generation.fetch_add(1, std::memory_order_relaxed);
  wait_for_readers(t);
  KS_MARK(t, 4);
  const double v = t->cfg.voxel_size, trunc = t->cfg.truncation;
  BatchPrims PB{};
  PB.n = n;
  PB.offset[0] = 0;
  bool legal = true;
  for (int k = 0; k < n; ++k) {
    double lo_in[3], hi_in[3];
    std::string why;
    if (!fill_primitive(prims[k], PB.prim[k], lo_in, hi_in, why)) return fail(KS_ERR_INVALID, why);
    BlockBox& B = PB.box[k];
    B.count = 1;
    for (int a = 0; a < 3; ++a) {  // AABB grown by the truncation band -> block range (sdf_world.hpp:418-425)
      const int blo = voxel_index(lo_in[a] - trunc, v) >> 3, bhi = voxel_index(hi_in[a] + trunc, v) >> 3;
      B.lo[a] = blo;
      B.n[a] = std::max(bhi - blo + 1, 0);
      B.count *= B.n[a];
      if (B.lo[a] <= -kKeyBias || B.lo[a] + B.n[a] >= kKeyBias) legal = false;
    }
    PB.offset[k + 1] = PB.offset[k] + B.count;
  }
  const long long total = PB.offset[n];
  if (total > t->lists.cap) {  // a batch may touch more blocks than any single call: the op lists grow to hold all candidates
    const int rc = ensure_lists(t, static_cast<size_t>(total), 1);
    if (rc != KS_OK) return rc;
  }
  {  // at most `total` blocks are new: can this batch fail on the device at all?
    const bool safe = legal && t->bounds_valid && total <= t->known_avail && total <= t->known_room && total <= t->lists.cap;
    if (safe) t->known_avail -= total, t->known_room -= total;
    else t->bounds_valid = false;
    t->last_stamp_safe = safe;
  }
  const double reach = trunc + 0.5 * kBlockEdge * v * std::sqrt(3.0);  // sdf_world.hpp:288-290, :425
  const int grid = static_cast<int>(std::max<long long>(1, std::min<long long>((total + 255) / 256, 8 * kSmCount)));
  KS_LAUNCH(k_batch_candidates, grid, 256, 0, t->stream, t->view, t->lists, PB, reach);
  KS_LAUNCH(k_batch_commit, 4 * kSmCount, 256, 0, t->stream, t->view, t->lists, n);
  KS_MARK(t, 5);
  KS_LAUNCH(k_batch_blocks, 3 * kSmCount, 512, 0, t->stream, t->view, t->lists, PB, last_group ? 1 : 0);
  KS_MARK(t, 6);
  KS_CUDA(cudaGetLastError());
  return KS_OK;
}

}  // namespace ksb

extern "C" {

int ks_tsdf_stamp_batch_async(ks_tsdf* t, const ks_primitive* prims, int32_t n) {
  if (!t || (n > 0 && !prims)) return fail(KS_ERR_INVALID, "null argument");
  for (int32_t at = 0; at < n; at += kMaxBatch) {  // groups run in order; a failing group is reported like a failing call
    const int rc = stamp_group_async(t, prims + at, std::min<int32_t>(kMaxBatch, n - at), at + kMaxBatch >= n);
    if (rc != KS_OK) return rc;
  }
  return KS_OK;
}


static int tsdf_init(ks_tsdf* t, const ks_tsdf_config* cfg);

int ks_tsdf_config_init(double voxel_size, ks_tsdf_config* out) {
  if (!out) return fail(KS_ERR_INVALID, "null config");
  *out = ks_tsdf_config{voxel_size, 4.0 * voxel_size, 0.99, 0.5, 0.5, 8192, 0};  // sdf_world.hpp:39-45, :56-61
  return KS_OK;
}

int ks_tsdf_create(const ks_tsdf_config* cfg, ks_tsdf** out) {
  if (!cfg || !out) return fail(KS_ERR_INVALID, "null argument");
  *out = nullptr;
  // TsdfConfig::validate (sdf_world.hpp:47-53)
  if (cfg->voxel_size <= 0.0) return fail(KS_ERR_INVALID, "tsdf: voxel_size must be > 0");
  if (cfg->truncation < cfg->voxel_size) return fail(KS_ERR_INVALID, "tsdf: truncation must be >= voxel_size");
  if (!(cfg->alpha_time > 0.0 && cfg->alpha_time <= 1.0) || !(cfg->alpha_frustum > 0.0 && cfg->alpha_frustum <= 1.0))
    return fail(KS_ERR_INVALID, "tsdf: decay factors must lie in (0, 1]");
  if (cfg->capacity < 1) return fail(KS_ERR_INVALID, "tsdf: capacity must be >= 1");
  int devices = 0;
  if (cudaGetDeviceCount(&devices) != cudaSuccess || devices == 0)
    return fail(KS_ERR_CUDA, "ks_b200: no CUDA device (this library has no CPU path)");

  ks_tsdf* t = new ks_tsdf();  // value-initialised: every member starts zeroed
  const int rc = tsdf_init(t, cfg);
  if (rc != KS_OK) {  // one cleanup path: whatever was allocated so far goes with the handle
    const std::string message = ks_last_error();
    ks_tsdf_destroy(t);
    cudaGetLastError();
    set_error(message);
    return rc;
  }
  *out = t;
  return KS_OK;
}

static int tsdf_init(ks_tsdf* t, const ks_tsdf_config* cfg) {
  t->cfg = *cfg;
  static std::atomic<uint64_t> next_uid{1};
  t->uid = next_uid.fetch_add(1);
  TsdfView& V = t->view;
  V.capacity = cfg->capacity;
  V.nslots = cfg->slot_count > 0 ? cfg->slot_count : 2 * cfg->capacity;  // BlockHashTable::init (sdf_world.hpp:115-120)
  V.voxel = cfg->voxel_size;
  V.trunc = cfg->truncation;
  V.seed_thr = 0.9 * cfg->voxel_size;  // seed_threshold (esdf.hpp:69)
  V.rank_direct = kRankDirect;
  if (const char* v = std::getenv("KS_RANK_DIRECT")) V.rank_direct = std::max(0, std::atoi(v));  // tests: force the sorted-tile ranks
  const size_t cap = static_cast<size_t>(cfg->capacity);
  KS_CUDA(cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking));
  t->own_stream = true;
  KS_CUDA(cudaMalloc(&V.slot_key, V.nslots * sizeof(uint64_t)));
  KS_CUDA(cudaMalloc(&V.slot_pool, V.nslots * sizeof(int)));
  KS_CUDA(cudaMalloc(&V.slot_claim, V.nslots * sizeof(uint32_t)));
  KS_CUDA(cudaMemsetAsync(V.slot_claim, 0xFF, V.nslots * sizeof(uint32_t), t->stream));
  KS_CUDA(cudaMalloc(&V.free_list, cap * sizeof(int)));
  KS_CUDA(cudaMalloc(&V.pool_key, cap * sizeof(uint64_t)));
  KS_CUDA(cudaMalloc(&V.sumwt, cap * kBlockVoxels * sizeof(double2)));
  KS_CUDA(cudaMalloc(&V.geom, cap * kBlockVoxels * sizeof(double)));
  KS_CUDA(cudaMalloc(&V.digest, cap * kDigestWords * sizeof(uint32_t)));
  KS_CUDA(cudaMalloc(&V.pool_geom, cap));
  KS_CUDA(cudaMemsetAsync(V.pool_geom, 0, cap, t->stream));
  KS_CUDA(cudaMalloc(&V.ctrl, sizeof(TsdfCtrl)));
  KS_CUDA(cudaMalloc(&t->d_flags, cap * sizeof(int)));
  for (cudaEvent_t& ev : t->ev) KS_CUDA(cudaEventCreate(&ev));
  KS_CUDA(cudaMallocHost(&t->h_ctrl, sizeof(TsdfCtrl)));
  KS_CUDA(cudaMallocHost(&t->h_verdict, sizeof(TsdfCtrl)));
  KS_CUDA(cudaEventCreateWithFlags(&t->ev_verdict, cudaEventDisableTiming));
  KS_CUDA(cudaMemsetAsync(V.ctrl, 0, sizeof(TsdfCtrl), t->stream));
  static const int kNoAbort = 0x7FFFFFFF;
  KS_CUDA(cudaMemcpyAsync(&V.ctrl->abort_prim, &kNoAbort, sizeof(int), cudaMemcpyHostToDevice, t->stream));
  KS_CUDA(cudaMemsetAsync(V.slot_pool, 0xFF, V.nslots * sizeof(int), t->stream));
  KS_CUDA(cudaMemsetAsync(V.digest, 0, cap * kDigestWords * sizeof(uint32_t), t->stream));
  KS_LAUNCH(k_fill_u64, 1024, 256, 0, t->stream, V.slot_key, static_cast<size_t>(V.nslots), kKeyEmpty);
  KS_LAUNCH(k_fill_u64, 1024, 256, 0, t->stream, V.pool_key, cap, kKeyEmpty);
  std::memset(t->h_ctrl, 0, sizeof(TsdfCtrl));
  int rc = ensure_lists(t, 0, 1);
  if (rc != KS_OK) return rc;
  KS_CUDA(cudaEventCreateWithFlags(&t->ev_reader, cudaEventDisableTiming));
  KS_CUDA(cudaStreamSynchronize(t->stream));
  return KS_OK;
}

void ks_tsdf_destroy(ks_tsdf* t) {
  if (!t) return;
  if (t->stream) cudaStreamSynchronize(t->stream);
  TsdfView& V = t->view;
  cudaFree(V.slot_key), cudaFree(V.slot_pool), cudaFree(V.slot_claim), cudaFree(V.free_list), cudaFree(V.pool_key);
  cudaFree(V.sumwt), cudaFree(V.geom), cudaFree(V.digest), cudaFree(V.pool_geom), cudaFree(V.ctrl), cudaFree(t->d_flags);
  OpLists& L = t->lists;
  cudaFree(L.key), cudaFree(L.pool), cudaFree(L.slot), cudaFree(L.fresh_idx), cudaFree(L.fresh_rank), cudaFree(L.rank_key), cudaFree(L.sorted_key), cudaFree(L.sorted_prim), cudaFree(L.fset), cudaFree(L.fmask);
  for (void* p : t->retired_dev) cudaFree(p);
  for (void* p : t->retired_host) cudaFreeHost(p);
  cudaFree(t->query_scratch);
  cudaFreeHost(t->h_ctrl);
  cudaFreeHost(t->h_verdict);
  if (t->ev_verdict) cudaEventDestroy(t->ev_verdict);
  if (t->ev_reader) cudaEventDestroy(t->ev_reader);
  for (ks_tsdf::FrameSlot& S : t->slots) {
    if (S.h_frame) cudaFreeHost(S.h_frame);
    if (S.d_frame) cudaFree(S.d_frame);
    if (S.h_depth) cudaFreeHost(S.h_depth);
    if (S.d_depth) cudaFree(S.d_depth);
  }
  for (cudaEvent_t ev : t->ev)
    if (ev) cudaEventDestroy(ev);
  if (t->own_stream && t->stream) cudaStreamDestroy(t->stream);
  delete t;
}

int ks_tsdf_profile(ks_tsdf* t, int32_t enable) {
  if (!t) return fail(KS_ERR_INVALID, "null tsdf");
  t->profile = enable != 0;
  return KS_OK;
}

int ks_tsdf_stage_ms(ks_tsdf* t, float out[5]) {
  if (!t || !out) return fail(KS_ERR_INVALID, "null argument");
  KS_CUDA(cudaStreamSynchronize(t->stream));
  const int pairs[5][2] = {{0, 1}, {1, 2}, {2, 3}, {4, 5}, {5, 6}};
  for (int i = 0; i < 5; ++i) {
    out[i] = 0.0f;
    if (cudaEventElapsedTime(&out[i], t->ev[pairs[i][0]], t->ev[pairs[i][1]]) != cudaSuccess) {
      cudaGetLastError();
      out[i] = -1.0f;
    }
  }
  return KS_OK;
}

int ks_tsdf_set_stream(ks_tsdf* t, ks_stream s) {
  if (!t) return fail(KS_ERR_INVALID, "null tsdf");
  KS_CUDA(cudaStreamSynchronize(t->stream));
  if (t->own_stream) cudaStreamDestroy(t->stream);
  t->own_stream = false;
  t->stream = static_cast<cudaStream_t>(s);
  return KS_OK;
}

ks_stream ks_tsdf_get_stream(const ks_tsdf* t) { return t ? static_cast<ks_stream>(t->stream) : nullptr; }

// copy_pixels = false: the caller uploads the pixels from where they are (page-locked source)
static int stage_frame_impl(ks_tsdf* t, int32_t slot, const ks_camera* cam, const float* depth_host, bool copy_pixels) {
  if (!t || !cam) return fail(KS_ERR_INVALID, "null argument");
  if (slot < 0 || slot >= KS_MAX_FRAME_SLOTS) return fail(KS_ERR_INVALID, "tsdf: camera slot out of range");
  // DepthFrame::validate (sdf_world.hpp:197-202)
  if (cam->width <= 0 || cam->height <= 0 || cam->fx <= 0.0 || cam->fy <= 0.0)
    return fail(KS_ERR_INVALID, "depth frame: invalid intrinsics");
  if (!depth_host) return fail(KS_ERR_INVALID, "depth frame: depth buffer size mismatch");
  const double step = 4.0 * t->cfg.voxel_size;                                        // sdf_world.hpp:347
  const int hs = std::max(1, static_cast<int>(std::ceil(t->cfg.truncation / step)));  // sdf_world.hpp:348
  const size_t pixels = static_cast<size_t>(cam->width) * cam->height;
  int rc = ensure_lists(t, pixels, 2 * hs + 1);
  if (rc != KS_OK) return rc;
  if ((rc = ensure_slot(t, slot, pixels)) != KS_OK) return rc;
  ks_tsdf::FrameSlot& S = t->slots[slot];
  FrameParams& F = *S.h_frame;
  F.width = cam->width, F.height = cam->height;
  F.fx = cam->fx, F.fy = cam->fy, F.cx = cam->cx, F.cy = cam->cy;
  std::memcpy(F.c2w.r, cam->pose_R, sizeof F.c2w.r);
  std::memcpy(F.c2w.t, cam->pose_t, sizeof F.c2w.t);
  F.w2c = rigid_inverse(F.c2w);
  F.half_samples = hs;
  F.step = step;
  if (copy_pixels && depth_host != S.h_depth) std::memcpy(S.h_depth, depth_host, pixels * sizeof(float));  // else written in place
  S.staged = true;
  return KS_OK;
}

int ks_tsdf_stage_frame_slot(ks_tsdf* t, int32_t slot, const ks_camera* cam, const float* depth_host) {
  return stage_frame_impl(t, slot, cam, depth_host, true);
}

int ks_tsdf_frame_buffer(ks_tsdf* t, int32_t slot, int32_t width, int32_t height, float** out) {
  if (!t || !out) return fail(KS_ERR_INVALID, "null argument");
  if (slot < 0 || slot >= KS_MAX_FRAME_SLOTS) return fail(KS_ERR_INVALID, "tsdf: camera slot out of range");
  if (width <= 0 || height <= 0) return fail(KS_ERR_INVALID, "depth frame: invalid intrinsics");
  const int rc = ensure_slot(t, slot, static_cast<size_t>(width) * height);
  if (rc != KS_OK) return rc;
  *out = t->slots[slot].h_depth;
  return KS_OK;
}

int ks_host_alloc(size_t bytes, void** out) {
  if (!out) return fail(KS_ERR_INVALID, "null argument");
  KS_CUDA(cudaMallocHost(out, bytes));
  return KS_OK;
}
void ks_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int ks_tsdf_upload_frame_slot_async(ks_tsdf* t, int32_t slot) {
  if (!t || slot < 0 || slot >= KS_MAX_FRAME_SLOTS || !t->slots[slot].staged) return fail(KS_ERR_INVALID, "tsdf: no frame staged");
  ks_tsdf::FrameSlot& S = t->slots[slot];
  const size_t pixels = static_cast<size_t>(S.h_frame->width) * S.h_frame->height;
  note_capture(t);
  KS_CUDA(cudaMemcpyAsync(S.d_frame, S.h_frame, sizeof(FrameParams), cudaMemcpyHostToDevice, t->stream));
  KS_CUDA(cudaMemcpyAsync(S.d_depth, S.h_depth, pixels * sizeof(float), cudaMemcpyHostToDevice, t->stream));
  return KS_OK;
}

static int integrate_enqueue(ks_tsdf* t, int32_t slot, bool verdict);
int ks_tsdf_integrate_slot_async(ks_tsdf* t, int32_t slot) { return integrate_enqueue(t, slot, false); }

// verdict: copy the control block to the host right after the allocation kernel.  Whether the frame fits (pool, table,
// range) and how many blocks it touches is decided by then -- finish_op at the end of the voxel pass only applies
// it -- so the blocking integrate_depth can return while k_integrate still runs.
static int integrate_enqueue(ks_tsdf* t, int32_t slot, bool verdict) {
  if (!t || slot < 0 || slot >= KS_MAX_FRAME_SLOTS || !t->slots[slot].staged) return fail(KS_ERR_INVALID, "tsdf: no frame staged");
  ks_tsdf::FrameSlot& S = t->slots[slot];
  const int pixels = S.h_frame->width * S.h_frame->height;
  const bool prof = profiling(t);
  t->bounds_valid = false;  // a frame allocates a number of blocks only the device knows
  t->generation.fetch_add(1, std::memory_order_relaxed);
  wait_for_readers(t);
  KS_MARK(t, 0);
  KS_LAUNCH(k_discover, (pixels + 255) / 256, 256, 0, t->stream, t->view, t->lists, S.d_frame, S.d_depth);
  KS_MARK(t, 1);
  run_allocation(t);
  KS_MARK(t, 2);
  if (verdict) {
    KS_CUDA(cudaMemcpyAsync(t->h_verdict, t->view.ctrl, sizeof(TsdfCtrl), cudaMemcpyDeviceToHost, t->stream));
    KS_CUDA(cudaEventRecord(t->ev_verdict, t->stream));
  }
  KS_LAUNCH(k_integrate, 3 * kSmCount, 512, 0, t->stream, t->view, t->lists, S.d_frame, S.d_depth);
  KS_MARK(t, 3);
  KS_CUDA(cudaGetLastError());
  return KS_OK;
}

int ks_tsdf_stage_frame(ks_tsdf* t, const ks_camera* cam, const float* depth_host) { return ks_tsdf_stage_frame_slot(t, 0, cam, depth_host); }
int ks_tsdf_upload_frame_async(ks_tsdf* t) { return ks_tsdf_upload_frame_slot_async(t, 0); }
int ks_tsdf_integrate_async(ks_tsdf* t) { return ks_tsdf_integrate_slot_async(t, 0); }

}  // extern "C"
namespace ksb {
int tsdf_report_enqueue(ks_tsdf* t) {
  KS_CUDA(cudaMemcpyAsync(t->h_ctrl, t->view.ctrl, sizeof(TsdfCtrl), cudaMemcpyDeviceToHost, t->stream));
  return KS_OK;
}
}  // namespace ksb
extern "C" {

int ks_tsdf_sync(ks_tsdf* t, ks_tsdf_report* report) {
  if (!t) return fail(KS_ERR_INVALID, "null tsdf");
  const int rc = tsdf_report_enqueue(t);
  if (rc != KS_OK) return rc;
  KS_CUDA(cudaStreamSynchronize(t->stream));
  return tsdf_report_collect(t, report);
}

}  // extern "C"
namespace ksb {
int tsdf_report_collect(ks_tsdf* t, ks_tsdf_report* report) {
  const TsdfCtrl c = *t->h_ctrl;
  if (c.err != 0) {  // errors are sticky until collected
    KS_CUDA(cudaMemsetAsync(&t->view.ctrl->err, 0, sizeof(int), t->stream));
    KS_CUDA(cudaStreamSynchronize(t->stream));
  }
  t->bounds_valid = c.err == 0;
  t->known_avail = static_cast<long long>(t->view.capacity) - c.next_fresh + c.free_count;  // BlockHashTable::available
  t->known_room = static_cast<long long>(t->view.nslots) - c.live;
  if (report) {
    report->status = c.err;
    report->blocks_touched = c.last_touched;
    report->required = c.err_required;
    report->available = c.err_available;
    report->live_blocks = c.live;
    report->next_fresh = c.next_fresh;
    report->free_count = c.free_count;
    report->recycled = c.last_recycled;
  }
  return report_status(c);
}
}  // namespace ksb
extern "C" {

int ks_tsdf_integrate_depth(ks_tsdf* t, const ks_camera* cam, const float* depth_host, int32_t* blocks_touched) {
  if (!t) return fail(KS_ERR_INVALID, "null argument");
  // a page-locked source is uploaded in place: only the camera parameters go through the staging slot
  bool in_place = false;
  if (depth_host && depth_host != t->slots[0].h_depth) {
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, depth_host) == cudaSuccess) in_place = attr.type == cudaMemoryTypeHost;
    else cudaGetLastError();
  }
  int rc = stage_frame_impl(t, 0, cam, depth_host, !in_place);
  if (rc != KS_OK) return rc;
  if (in_place) {
    ks_tsdf::FrameSlot& S = t->slots[0];
    const size_t pixels = static_cast<size_t>(cam->width) * cam->height;
    KS_CUDA(cudaMemcpyAsync(S.d_frame, S.h_frame, sizeof(FrameParams), cudaMemcpyHostToDevice, t->stream));
    KS_CUDA(cudaMemcpyAsync(S.d_depth, depth_host, pixels * sizeof(float), cudaMemcpyHostToDevice, t->stream));
  } else if ((rc = ks_tsdf_upload_frame_async(t)) != KS_OK) return rc;
  const bool early = !profiling(t);  // stage timing wants the whole op inside the call
  if ((rc = integrate_enqueue(t, 0, early)) != KS_OK) return rc;
  if (early) {
    KS_CUDA(cudaEventSynchronize(t->ev_verdict));
    const TsdfCtrl c = *t->h_verdict;  // what finish_op will see: the counters of the op in flight, the table before it
    const long long avail = static_cast<long long>(t->view.capacity) - c.next_fresh + c.free_count;
    const bool fits = c.err == 0 && c.abort_op == 0 && c.fresh <= avail && c.touched <= t->lists.cap &&
                      static_cast<long long>(c.live) + c.fresh <= t->view.nslots;
    if (fits) {  // integrate_depth's return value (sdf_world.hpp:388) is known; the voxel pass finishes behind the caller
      t->bounds_valid = true;
      t->known_avail = avail - c.fresh;
      t->known_room = static_cast<long long>(t->view.nslots) - c.live - c.fresh;
      if (blocks_touched) *blocks_touched = c.touched;
      return KS_OK;
    }
  }
  ks_tsdf_report rep;  // the frame does not fit (or timing is on): wait for the device's own report
  rc = ks_tsdf_sync(t, &rep);
  if (blocks_touched) *blocks_touched = rc == KS_OK ? rep.blocks_touched : 0;
  return rc;
}

int ks_tsdf_stamp_cuboid_async(ks_tsdf* t, const double pose_R[9], const double pose_t[3], const double he[3]) {
  if (!t) return fail(KS_ERR_INVALID, "null tsdf");
  for (int a = 0; a < 3; ++a)
    if (!std::isfinite(he[a]) || !std::isfinite(pose_t[a])) return fail(KS_ERR_INVALID, "stamp: non-finite cuboid");
  Rigid pose;
  std::memcpy(pose.r, pose_R, sizeof pose.r);
  std::memcpy(pose.t, pose_t, sizeof pose.t);
  Primitive P;
  std::memset(&P, 0, sizeof P);
  P.inv = rigid_inverse(pose);
  for (int a = 0; a < 3; ++a) P.he[a] = he[a];
  // AABB of the eight rotated corners (sdf_world.hpp:402-410)
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int corner = 0; corner < 8; ++corner) {
    const double sx = (corner & 1) ? 1.0 : -1.0, sy = (corner & 2) ? 1.0 : -1.0, sz = (corner & 4) ? 1.0 : -1.0;
    double w[3];
    rigid_apply(pose, sx * he[0], sy * he[1], sz * he[2], w);
    for (int a = 0; a < 3; ++a) {
      if (w[a] < lo[a]) lo[a] = w[a];
      if (hi[a] < w[a]) hi[a] = w[a];
    }
  }
  return stamp_async(t, P, lo, hi);
}

int ks_tsdf_stamp_sphere_async(ks_tsdf* t, const double center[3], double radius) {
  if (!t) return fail(KS_ERR_INVALID, "null tsdf");
  if (!std::isfinite(center[0]) || !std::isfinite(center[1]) || !std::isfinite(center[2]) || !std::isfinite(radius))
    return fail(KS_ERR_INVALID, "stamp: non-finite sphere");
  Primitive P;
  std::memset(&P, 0, sizeof P);
  P.is_sphere = 1;
  P.radius = radius;
  double lo[3], hi[3];
  for (int a = 0; a < 3; ++a) {
    P.c[a] = center[a];
    lo[a] = center[a] - radius;  // sdf_world.hpp:415-416
    hi[a] = center[a] + radius;
  }
  return stamp_async(t, P, lo, hi);
}

// stamp_primitive throws on exhaustion (sdf_world.hpp:436-439).  When the candidate blocks of the stamp just
// enqueued fit the known free pool entries and hash slots, that cannot happen and the call returns at once;
// otherwise it waits for the device's verdict.
static int finish_stamp(ks_tsdf* t) {
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(t->stream, &cap);
  if (cap == cudaStreamCaptureStatusNone && t->last_stamp_safe) return KS_OK;
  return ks_tsdf_sync(t, nullptr);
}

int ks_tsdf_stamp_batch(ks_tsdf* t, const ks_primitive* prims, int32_t n) {
  int rc = ks_tsdf_stamp_batch_async(t, prims, n);
  return rc != KS_OK ? rc : finish_stamp(t);
}

int ks_tsdf_stamp_cuboid(ks_tsdf* t, const double pose_R[9], const double pose_t[3], const double he[3]) {
  int rc = ks_tsdf_stamp_cuboid_async(t, pose_R, pose_t, he);
  return rc != KS_OK ? rc : finish_stamp(t);
}

int ks_tsdf_stamp_sphere(ks_tsdf* t, const double center[3], double radius) {
  int rc = ks_tsdf_stamp_sphere_async(t, center, radius);
  return rc != KS_OK ? rc : finish_stamp(t);
}

// ---- triangle meshes (no reference counterpart: SPEC.md:8, :422; definition in csrc/mesh.cuh) ----
int ks_mesh_create(const double* vertices, int32_t n_vertices, const int32_t* triangles, int32_t n_triangles, ks_mesh** out) {
  if (!out) return fail(KS_ERR_INVALID, "null argument");
  *out = nullptr;
  int devices = 0;
  if (cudaGetDeviceCount(&devices) != cudaSuccess || devices < 1) {
    cudaGetLastError();
    return fail(KS_ERR_CUDA, "no CUDA device (this library has no CPU path)");
  }
  MeshTables tab;
  if (const char* why = build_mesh_tables(vertices, n_vertices, triangles, n_triangles, tab)) return fail(KS_ERR_INVALID, why);
  ks_mesh* m = new ks_mesh();
  std::memset(m, 0, sizeof *m);
  double *tri = nullptr, *nrm = nullptr, *bnd = nullptr;
  auto upload = [](double** dst, const std::vector<double>& src) {
    cudaError_t e = cudaMalloc(dst, src.size() * sizeof(double));
    return e != cudaSuccess ? e : cudaMemcpy(*dst, src.data(), src.size() * sizeof(double), cudaMemcpyHostToDevice);
  };
  cudaError_t e = upload(&tri, tab.tri);
  if (e == cudaSuccess) e = upload(&nrm, tab.nrm);
  if (e == cudaSuccess) e = upload(&bnd, tab.bnd);
  if (e != cudaSuccess) {
    cudaFree(tri), cudaFree(nrm), cudaFree(bnd);
    delete m;
    return cuda_fail(e, "ks_mesh_create");
  }
  m->view = MeshView{n_triangles, tri, nrm, bnd};
  for (int a = 0; a < 3; ++a) m->lo[a] = tab.lo[a], m->hi[a] = tab.hi[a];
  *out = m;
  return KS_OK;
}

void ks_mesh_destroy(ks_mesh* m) {
  if (!m) return;
  cudaDeviceSynchronize();  // a stamp that reads the tables may still be in flight
  cudaFree(const_cast<double*>(m->view.tri)), cudaFree(const_cast<double*>(m->view.nrm)), cudaFree(const_cast<double*>(m->view.bnd));
  delete m;
}

int32_t ks_mesh_triangle_count(const ks_mesh* m) { return m ? m->view.nt : 0; }

int ks_tsdf_stamp_mesh_async(ks_tsdf* t, const ks_mesh* m) {
  if (!t || !m) return fail(KS_ERR_INVALID, "null argument");
  Primitive P;
  std::memset(&P, 0, sizeof P);
  return stamp_async(t, P, m->lo, m->hi, m);
}

int ks_tsdf_stamp_mesh(ks_tsdf* t, const ks_mesh* m) {
  int rc = ks_tsdf_stamp_mesh_async(t, m);
  return rc != KS_OK ? rc : finish_stamp(t);
}

int ks_tsdf_decay_weights_async(ks_tsdf* t, const ks_camera* cam) {
  if (!t || !cam) return fail(KS_ERR_INVALID, "null argument");
  Frustum Fr;
  Rigid pose;
  std::memcpy(pose.r, cam->pose_R, sizeof pose.r);
  std::memcpy(pose.t, cam->pose_t, sizeof pose.t);
  Fr.w2c = rigid_inverse(pose);
  Fr.radius = 0.5 * kBlockEdge * t->cfg.voxel_size * std::sqrt(3.0);
  const double raw[5][3] = {{0.0, 0.0, 1.0},
                            {cam->fx, 0.0, cam->cx},
                            {-cam->fx, 0.0, cam->width - 1 - cam->cx},
                            {0.0, cam->fy, cam->cy},
                            {0.0, -cam->fy, cam->height - 1 - cam->cy}};
  for (int p = 0; p < 5; ++p) {
    double n[3] = {raw[p][0], raw[p][1], raw[p][2]};
    if (p > 0) {  // .normalized(); the near plane is written as a literal unit vector
      const double z = sum3(n[0] * n[0], n[1] * n[1], n[2] * n[2]);
      if (z > 0.0) {
        const double len = std::sqrt(z);
        for (double& c : n) c = c / len;
      }
    }
    for (int a = 0; a < 3; ++a) Fr.n[p][a] = n[a];
  }
  t->generation.fetch_add(1, std::memory_order_relaxed);
  wait_for_readers(t);
  KS_LAUNCH(k_decay, 4 * kSmCount, 512, 0, t->stream, t->view, Fr, t->cfg.alpha_time, t->cfg.alpha_frustum);
  KS_CUDA(cudaGetLastError());
  return KS_OK;
}

int ks_tsdf_decay_weights(ks_tsdf* t, const ks_camera* cam) {
  int rc = ks_tsdf_decay_weights_async(t, cam);
  return rc != KS_OK ? rc : ks_tsdf_sync(t, nullptr);
}

int ks_tsdf_recycle_blocks(ks_tsdf* t, int32_t* recycled) {
  if (!t) return fail(KS_ERR_INVALID, "null tsdf");
  t->generation.fetch_add(1, std::memory_order_relaxed);
  wait_for_readers(t);
  KS_LAUNCH(k_recycle_flag, 2 * kSmCount, 128, 0, t->stream, t->view, t->d_flags, t->cfg.weight_threshold);
  KS_LAUNCH(k_recycle_commit, 1, 1024, 0, t->stream, t->view, t->d_flags);
  KS_CUDA(cudaGetLastError());
  ks_tsdf_report rep;
  int rc = ks_tsdf_sync(t, &rep);
  if (recycled) *recycled = rep.recycled;
  return rc;
}

int ks_tsdf_query(ks_tsdf* t, const double* points_host, int64_t n, int32_t geom_only, double* out_sdf, uint8_t* out_valid) {
  if (!t) return fail(KS_ERR_INVALID, "null tsdf");
  if (n <= 0) return KS_OK;
  // device scratch kept in the handle (query_tsdf may be called concurrently, sdf_world.hpp / SPEC.md:415-416: one caller at a time here)
  std::lock_guard<std::mutex> lock(t->query_mu);
  if (n > t->query_cap) {
    const int64_t cap = std::max<int64_t>(n + n / 4, 4096);
    KS_CUDA(cudaStreamSynchronize(t->stream));
    cudaFree(t->query_scratch);
    t->query_scratch = nullptr, t->query_cap = 0;
    KS_CUDA(cudaMalloc(&t->query_scratch, static_cast<size_t>(cap) * 5 * sizeof(double)));  // points 24 B, value 8 B, valid 1 B
    t->query_cap = cap;
  }
  double *d_pts = t->query_scratch, *d_out = d_pts + 3 * n;
  uint8_t* d_valid = reinterpret_cast<uint8_t*>(d_out + n);
  KS_CUDA(cudaMemcpyAsync(d_pts, points_host, n * 3 * sizeof(double), cudaMemcpyHostToDevice, t->stream));
  KS_LAUNCH(k_query_tsdf, static_cast<unsigned>((n + 255) / 256), 256, 0, t->stream, t->view, d_pts, static_cast<long long>(n),
            geom_only, d_out, d_valid);
  KS_CUDA(cudaMemcpyAsync(out_sdf, d_out, n * sizeof(double), cudaMemcpyDeviceToHost, t->stream));
  KS_CUDA(cudaMemcpyAsync(out_valid, d_valid, n, cudaMemcpyDeviceToHost, t->stream));
  KS_CUDA(cudaStreamSynchronize(t->stream));
  return KS_OK;
}

int ks_tsdf_allocated_block_count(ks_tsdf* t, int32_t* count) {
  ks_tsdf_report rep;
  int rc = ks_tsdf_sync(t, &rep);
  if (count) *count = rep.live_blocks;
  return rc;
}

int ks_tsdf_find(ks_tsdf* t, const int32_t key[3], int32_t* pool_index) {
  if (!t || !key || !pool_index) return fail(KS_ERR_INVALID, "null argument");
  int* d_out = nullptr;
  KS_CUDA(cudaMalloc(&d_out, sizeof(int)));
  KS_LAUNCH(k_find, 1, 1, 0, t->stream, t->view, key[0], key[1], key[2], d_out);
  KS_CUDA(cudaMemcpyAsync(pool_index, d_out, sizeof(int), cudaMemcpyDeviceToHost, t->stream));
  KS_CUDA(cudaStreamSynchronize(t->stream));
  cudaFree(d_out);
  return KS_OK;
}

int ks_tsdf_export_blocks(ks_tsdf* t, int32_t* keys_xyz, int32_t* pool_index, int32_t max_blocks, int32_t* count) {
  if (!t) return fail(KS_ERR_INVALID, "null tsdf");
  const int n = t->view.nslots;
  std::vector<uint64_t> keys(n);
  std::vector<int> pools(n);
  KS_CUDA(cudaMemcpyAsync(keys.data(), t->view.slot_key, n * sizeof(uint64_t), cudaMemcpyDeviceToHost, t->stream));
  KS_CUDA(cudaMemcpyAsync(pools.data(), t->view.slot_pool, n * sizeof(int), cudaMemcpyDeviceToHost, t->stream));
  KS_CUDA(cudaStreamSynchronize(t->stream));
  int live = 0;
  for (int s = 0; s < n; ++s) {
    if (keys[s] == kKeyEmpty || keys[s] == kKeyTomb) continue;
    if (live < max_blocks) {
      int x, y, z;
      unpack_key(keys[s], x, y, z);
      if (keys_xyz) keys_xyz[3 * live] = x, keys_xyz[3 * live + 1] = y, keys_xyz[3 * live + 2] = z;
      if (pool_index) pool_index[live] = pools[s];
    }
    ++live;
  }
  if (count) *count = live;
  return KS_OK;
}

uint64_t ks_tsdf_generation(const ks_tsdf* t) { return t ? t->generation.load(std::memory_order_relaxed) : 0; }

int ks_tsdf_export_slots(ks_tsdf* t, int32_t* keys_xyz, int32_t* pool_index, uint8_t* state, int32_t max_slots, int32_t* count) {
  if (!t) return fail(KS_ERR_INVALID, "null tsdf");
  const int n = t->view.nslots;
  if (count) *count = n;
  if (max_slots <= 0) return KS_OK;
  std::vector<uint64_t> keys(n);
  std::vector<int> pools(n);
  KS_CUDA(cudaMemcpyAsync(keys.data(), t->view.slot_key, n * sizeof(uint64_t), cudaMemcpyDeviceToHost, t->stream));
  KS_CUDA(cudaMemcpyAsync(pools.data(), t->view.slot_pool, n * sizeof(int), cudaMemcpyDeviceToHost, t->stream));
  KS_CUDA(cudaStreamSynchronize(t->stream));
  for (int s = 0; s < n && s < max_slots; ++s) {
    const bool live = keys[s] != kKeyEmpty && keys[s] != kKeyTomb;
    int x = 0, y = 0, z = 0;
    if (live) unpack_key(keys[s], x, y, z);
    if (keys_xyz) keys_xyz[3 * s] = x, keys_xyz[3 * s + 1] = y, keys_xyz[3 * s + 2] = z;
    if (pool_index) pool_index[s] = live ? pools[s] : -1;
    if (state) state[s] = live ? 1 : (keys[s] == kKeyTomb ? 2 : 0);
  }
  return KS_OK;
}

int ks_tsdf_download_blocks(ks_tsdf* t, const int32_t* pool_index, int32_t n, double* depth_sum, double* depth_wt,
                            double* geom_sdf) {
  if (!t) return fail(KS_ERR_INVALID, "null tsdf");
  std::vector<double2> sw(kBlockVoxels);
  KS_CUDA(cudaStreamSynchronize(t->stream));
  for (int i = 0; i < n; ++i) {
    const int p = pool_index[i];
    if (p < 0 || p >= t->cfg.capacity) return fail(KS_ERR_INVALID, "tsdf: pool index out of range");
    KS_CUDA(cudaMemcpy(sw.data(), t->view.sumwt + static_cast<size_t>(p) * kBlockVoxels, kBlockVoxels * sizeof(double2),
                       cudaMemcpyDeviceToHost));
    for (int q = 0; q < kBlockVoxels; ++q) {
      if (depth_sum) depth_sum[static_cast<size_t>(i) * kBlockVoxels + q] = sw[q].x;
      if (depth_wt) depth_wt[static_cast<size_t>(i) * kBlockVoxels + q] = sw[q].y;
    }
    if (geom_sdf)
      KS_CUDA(cudaMemcpy(geom_sdf + static_cast<size_t>(i) * kBlockVoxels, t->view.geom + static_cast<size_t>(p) * kBlockVoxels,
                         kBlockVoxels * sizeof(double), cudaMemcpyDeviceToHost));
  }
  return KS_OK;
}

int ks_tsdf_free_list(ks_tsdf* t, int32_t* out, int32_t max_out, int32_t* count) {
  ks_tsdf_report rep;
  int rc = ks_tsdf_sync(t, &rep);
  if (rc != KS_OK) return rc;
  const int n = std::min(rep.free_count, max_out);
  if (n > 0 && out) KS_CUDA(cudaMemcpy(out, t->view.free_list, n * sizeof(int), cudaMemcpyDeviceToHost));
  if (count) *count = rep.free_count;
  return KS_OK;
}

}  // extern "C"
