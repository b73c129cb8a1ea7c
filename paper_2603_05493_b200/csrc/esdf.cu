// Dense workspace ESDF on the device: seeding, exact EDT ("PBA+"), sign recovery and
// batched trilinear queries.  Replaces /root/reference/proj/include/ks/esdf.hpp
// behind the C ABI in include/ks_b200.h.  See DESIGN.md for layouts and byte counts.
//
// Device layout of the finished field.
//   Fast path (divide-and-conquer sweeps, every squared distance below 2^21): ONE uint32 per cell, x-fastest like the
//   reference (esdf.hpp:48-50):   negative << 31 | squared integer site offset << 10 | site_x
//   -- which is the winning key of the x sweep itself plus the sign bit.  distance = sqrt((double)d2) * voxel_size is
//   formed on the fly, so queries see exactly the reference's doubles.  site_y / site_z are not stored per cell: they
//   are the payload of phase 2's winner at (site_x, y, z), which stays in HBM (gimg / himg), and only the download and
//   the stand-alone recover_signs ask for them.  Two such buffers exist; the x sweep writes the one readers do not
//   use and publishes it with its last CTA (readers see the old or the new field, never a mix: SPEC.md:502-503).
//   Wide path (banded-stack fallback, grids beyond the 32-bit keys): uint2 per cell, y-fastest,
//   {site x | y<<10 | z<<20, d2 | negative << 31}; 0xFFFFFFFF / 0x7FFFFFFF without sites.
#include <math_constants.h>

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdlib>
#include <mutex>
#include <cstring>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "edt_core.cuh"
#include "edt_dc.cuh"

namespace ksb {

constexpr uint32_t kSiteNone = 0xFFFFFFFFu;
constexpr uint32_t kD2None = 0x7FFFFFFFu;
constexpr uint32_t kYzNone = 0xFFFFFFFFu;
constexpr int kMaxDim = 1024;  // 10-bit site packing, uint16 stacks

struct EsdfCtrl {
  unsigned long long seed_count;
  int signs_recovered;
  int seed_words;     // entries of EsdfView::seedw (resampled seeding): seeds with a stamped block in reach
  int active_bricks;  // entries of EsdfView::active, rebuilt with the directory
  // what readers go by (never touched by the resets above): published by the last CTA of the last sweep
  int front;                     // fast path: index of the field buffer readers use
  unsigned x_done;               // CTAs of the x sweep in flight that have finished
  unsigned long long pub_seeds;  // seed count of the published field (0: no sites)
};

// per-axis table rows (each [nx+ny+nz]): TSDF voxel index of (cell centre + offset), stored
// RELATIVE to the block directory's origin (minus 8*dlo), so `>> 3` is the directory coordinate
// and `& 7` is still the voxel's position inside its block.
enum VoxRow { kVoxC = 0, kVoxPh = 1, kVoxMh = 2, kVoxPe = 3, kVoxMe = 4, kVoxRows = 5 };

struct EsdfView {
  int nx, ny, nz;
  int cells;     // <= 2^30 (dims <= 1024), so 32-bit indexing throughout
  double origin[3];
  double ve;
  float ratio;   // ve / tsdf voxel (fast-path sign probe)
  int tab_all;   // 1: the sweeps carry no table bit (y keys too wide): every site's table is read, so every seed needs one
  int iprobe;    // 1: ve == tsdf voxel and every cell centre sits at the middle of its voxel -> the probe offset is an integer test (SignTable)
  int* vox;      // [kVoxRows][nx+ny+nz]: offsets {0, +ve/2, -ve/2, +ve, -ve} (esdf.hpp:106-108, :303)
  double* ctr;   // [nx+ny+nz]    cell centre coordinate per axis position (esdf.hpp:51-53)
  float* qsf;    // [nx+ny+nz]    fractional part of centre / tsdf voxel
  int* dir;      // dense block directory over the workspace: pool entry or -1
  int dlo[3], dn[3];
  int dcount;
  uint8_t* pool_surf;  // [tsdf capacity] 1 when the block's surface plane is not empty (rebuilt with the directory)
  uint8_t* brick;    // [ceil(n/8)^3] bit0: a live TSDF block lies in the brick's probe reach; bit1: one with surface voxels
  int* active;       // compacted ids of the active bricks (count in ctrl->active_bricks)
  int bnx, bny, bnz;
  uint8_t* mask;     // [cells] x-fastest seed mask (SeedMask, esdf.hpp:66) -- API paths
  uint32_t* mbits;   // [nz][ny][wpr] the same mask, one bit per cell -- fused build path
  uint32_t* gbits;   // [nz][ny][wpr] seed cells with stamped geometry within one cell (sign probes can resolve)
  int wpr;           // words per x row
  // "resampled" seeding (fused build when the dilation identity holds, see bind_tsdf): the TSDF digest bits at
  // every cell centre's own voxel, on the grid extended by one cell per side (cell i <-> index i + 1)
  int wpr2;            // words per extended x row
  int* voxe;           // [nx+2 | ny+2 | nz+2] directory-relative voxel of the extended cell centres
  uint32_t* cbits;     // [(nz+2)][(ny+2)][wpr2] surface bit of the centre voxel
  uint32_t* obits;     // same layout: combined sdf at the cell centre exists and is negative (sign fallback)
  uint32_t* nbits;     // same layout: a stamped block lies within one block of the centre voxel's block
  uint32_t* xplus;     // [wpr] bit x: the +ve/2 probe of cell x leaves the centre voxel (esdf.hpp:106-108) ...
  uint32_t* xminus;    // [wpr] ... and the -ve/2 probe
  uint8_t* yzflags;    // [ny | nz] bit0 / bit1: the same for the y and z probes of that row
  int xshift;          // voxe[i] == i + xshift along x (cell and voxel grids in step), else -1
  int yshift, zshift;  // the same along y and z
  int* seedw;          // compacted cell indices of the seeds whose sign table is not all zero (count in ctrl->seed_words)
  uint8_t* dirg;       // [dcount] 1 when a stamped block lies in the 3x3x3 blocks around this directory entry
  uint2* gtab;         // [cells] x-fastest, valid at the seeds: {has value, negative} of the geometry channel
                       // at the 27 voxels around the site's centre voxel, bit = (ox+1) + 3(oy+1) + 9(oz+1)
  uint16_t* near_z;  // [cells] x-fastest phase-1 result (banded-stack fallback only)
  // phase 1 of the divide-and-conquer path (aliases near_z): every column's seeds as a bit string along z
  uint32_t* zbits;   // [ny][nzw][nx] word w of column (x, y): bit b = cell z = 32w + b is a seed
  uint32_t* zinfo;   // same layout: distance from the word to the nearest seed in the words below w | above w << 16 (k_flood_cols)
  int nzw;           // words per column
  uint32_t* yz;      // [cells] x-fastest phase-2 result  site_y | site_z << 16
  uint2* field;      // wide path: [cells] y-fastest: {site (x | y << 10 | z << 20), squared distance | sign << 31}
  // fast path
  int fast;          // 1: the field is f32[ctrl->front], phase 2's result is gimg / himg
  int xpay;          // 1: gimg words are Keys<1> (in-plane d2 << 11 | x << 1 | the site has a sign table), 0: Keys<0>
  uint32_t* zgbits;  // like zbits, for gbits: bit b of word w = the seed at z = 32w + b has a sign table
  uint32_t* gimg;    // [nzt][nyt][nx][32 rows] the x sweep's tiles as they sit in shared memory: row = (y & 7) + 8 (z & 3),
                     //   word = in-plane d2 << 10 | x  (KeysX candidate; none_x << 10 | x without candidate)
  uint16_t* himg;    // same layout: site_y << 2 | seed above z << 1 | the site has a sign table
  int nyt, nzt;      // tiles along y and z
  uint32_t* f32[2];  // [cells] x-fastest: negative << 31 | d2 << 10 | site_x
  EsdfCtrl* ctrl;
};

__device__ __forceinline__ int axis_base(const EsdfView& E, int axis) { return axis == 0 ? 0 : (axis == 1 ? E.nx : E.nx + E.ny); }

// pool entry of the TSDF block containing directory-relative voxel (vx,vy,vz).  Every probe of
// seeding / sign recovery lies within one ESDF cell of the box, which bind_tsdf() covers with a
// one-block margin, so no bounds test is needed.
__device__ __forceinline__ int dir_lookup(const EsdfView& E, int vx, int vy, int vz) {
  return __ldg(E.dir + ((vx >> 3) + E.dn[0] * ((vy >> 3) + E.dn[1] * (vz >> 3))));
}
__device__ __forceinline__ int local_index(int vx, int vy, int vz) {  // local_index_of (sdf_world.hpp:274-280)
  return (vx & 7) + 8 * ((vy & 7) + 8 * (vz & 7));
}
__device__ __forceinline__ uint32_t surface_bit(const TsdfView& T, int pool, int local) {
  return (__ldg(T.digest + (pool * kDigestWords + (local >> 5))) >> (local & 31)) & 1u;
}
// 2-bit pair {has value, negative} of the geometry (kDigestGeom) or combined (kDigestComb) channel
__device__ __forceinline__ uint32_t pair_bits(const TsdfView& T, int pool, int plane_base, int local) {
  return (__ldg(T.digest + (pool * kDigestWords + plane_base + (local >> 4))) >> ((local & 15) * 2)) & 3u;
}

// ---- per-axis tables: every fp64 division of the seeding stage happens here, once per axis position ----
__global__ void k_axis_tables(EsdfView E, double tsdf_voxel) {
  pdl_enter();
  const int total = E.nx + E.ny + E.nz;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int axis = i < E.nx ? 0 : (i < E.nx + E.ny ? 1 : 2);
  const int k = i - axis_base(E, axis);
  const int rel = 8 * E.dlo[axis];
  const double c = E.origin[axis] + (k + 0.5) * E.ve;  // EsdfConfig::cell_center (esdf.hpp:51-53)
  const double h = 0.5 * E.ve;                         // esdf.hpp:106
  E.ctr[i] = c;
  E.vox[kVoxC * total + i] = voxel_index(c + 0.0, tsdf_voxel) - rel;
  E.vox[kVoxPh * total + i] = voxel_index(c + h, tsdf_voxel) - rel;
  E.vox[kVoxMh * total + i] = voxel_index(c + (-h), tsdf_voxel) - rel;
  // sign probe one cell along an axis: site_centre + ve * (+-1) (esdf.hpp:303 with an axis-aligned delta)
  E.vox[kVoxPe * total + i] = voxel_index(c + E.ve * 1.0, tsdf_voxel) - rel;
  E.vox[kVoxMe * total + i] = voxel_index(c + E.ve * -1.0, tsdf_voxel) - rel;
  const double q = c / tsdf_voxel;
  E.qsf[i] = static_cast<float>(q - floor(q));
}

// Directory reset as a kernel of the update (not two memset nodes: those would sit outside the programmatic launch
// chain); in the fused build it also zeroes the per-build counters that seeding accumulates into.
__global__ void __launch_bounds__(256) k_dir_clear(EsdfView E, bool reset_counters) {
  pdl_enter();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < E.dcount; i += gridDim.x * blockDim.x) {
    E.dir[i] = -1;
    E.dirg[i] = 0;
  }
  if (reset_counters && blockIdx.x == 0 && threadIdx.x == 0) E.ctrl->seed_count = 0ull, E.ctrl->signs_recovered = 0, E.ctrl->seed_words = 0;
}

// One warp per live pool entry: its directory slot; for a stamped block, the "stamped geometry within one block"
// flag of the 3x3x3 directory entries around it (lanes 0..26; cleared with the directory); surf_too: also the
// per-block "holds surface voxels" flag the brick gather's work list is built from.
__global__ void __launch_bounds__(256) k_dir_fill(EsdfView E, TsdfView T, bool surf_too) {
  pdl_enter();
  const int bound = T.ctrl->next_fresh;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < bound; p += nwarps) {
    const uint64_t key = T.pool_key[p];
    if (key == kKeyEmpty) continue;
    int bx, by, bz;
    unpack_key(key, bx, by, bz);
    bx -= E.dlo[0], by -= E.dlo[1], bz -= E.dlo[2];
    if (bx < 0 || bx >= E.dn[0] || by < 0 || by >= E.dn[1] || bz < 0 || bz >= E.dn[2]) continue;
    if (lane == 0) E.dir[bx + E.dn[0] * (by + E.dn[1] * bz)] = p;
    if (lane < 27 && T.pool_geom[p]) {
      const int x = bx + lane % 3 - 1, y = by + (lane / 3) % 3 - 1, z = bz + lane / 9 - 1;
      if (x >= 0 && x < E.dn[0] && y >= 0 && y < E.dn[1] && z >= 0 && z < E.dn[2]) E.dirg[x + E.dn[0] * (y + E.dn[1] * z)] = 1;
    }
    if (surf_too) {
      const uint32_t word = lane < 16 ? T.digest[p * kDigestWords + lane] : 0u;
      const bool any = __any_sync(0xFFFFFFFFu, word != 0);
      if (lane == 0) E.pool_surf[p] = any;
    }
  }
}

// A brick is 8^3 ESDF cells.  bit0: some TSDF block that one of its cells' seven probes can land in
// is live (a cell outside such a brick has no allocated block under its own centre -- the sign
// fallback's shortcut).  bit1: one of those blocks holds surface voxels; only these bricks can
// contain seeds, so only they go on the gather's work list.
__global__ void __launch_bounds__(128) k_brick_active(EsdfView E) {
  pdl_enter();
  const int nb = E.bnx * E.bny * E.bnz;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nb) return;
  const int b[3] = {i % E.bnx, (i / E.bnx) % E.bny, i / (E.bnx * E.bny)};
  const int dims[3] = {E.nx, E.ny, E.nz};
  const int total = E.nx + E.ny + E.nz;
  int lo[3], hi[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const int first = 8 * b[a], last = min(8 * b[a] + 7, dims[a] - 1);
    const int base = axis_base(E, a);
    lo[a] = E.vox[kVoxMh * total + base + first] >> 3;
    hi[a] = E.vox[kVoxPh * total + base + last] >> 3;
  }
  uint8_t flags = 0;
  for (int z = lo[2]; z <= hi[2] && flags != 3; ++z)
    for (int y = lo[1]; y <= hi[1] && flags != 3; ++y)
      for (int x = lo[0]; x <= hi[0] && flags != 3; ++x) {
        const int pool = E.dir[x + E.dn[0] * (y + E.dn[1] * z)];
        if (pool >= 0) flags |= E.pool_surf[pool] ? 3 : 1;
      }
  E.brick[i] = flags;
  if (flags & 2) E.active[atomicAdd(&E.ctrl->active_bricks, 1)] = i;
}

// ---- seed_gather (esdf.hpp:102-122): 7-probe stencil per ESDF cell, bits instead of voxels ----
// One warp = 32 consecutive x cells of one (y, z) row.  kBits: the fused build writes one ballot
// word per warp (plus the "stamped geometry within one cell" plane used by the fused sign
// recovery); the API path writes the reference's byte mask.
template <bool kBits>
__global__ void __launch_bounds__(256) k_seed_gather(EsdfView E, TsdfView T) {
  pdl_wait();
  const int warp_id = static_cast<int>((blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  const int rows = E.ny * E.nz;
  if (warp_id >= rows * E.wpr) return;
  const int xw = warp_id % E.wpr;
  const int row = warp_id / E.wpr;
  const int y = row % E.ny, z = row / E.ny;
  const int x = xw * 32 + lane;
  bool seed = false, geom_near = false;
  if (x < E.nx && (E.brick[(x >> 3) + E.bnx * ((y >> 3) + E.bny * (z >> 3))] & 2)) {
    const int total = E.nx + E.ny + E.nz;
    const int ix = x, iy = E.nx + y, iz = E.nx + E.ny + z;
    const int xc = E.vox[ix], xp = E.vox[total + ix], xm = E.vox[2 * total + ix];
    const int yc = E.vox[iy], yp = E.vox[total + iy], ym = E.vox[2 * total + iy];
    const int zc = E.vox[iz], zp = E.vox[total + iz], zm = E.vox[2 * total + iz];
    auto probe = [&](int vx, int vy, int vz) -> bool {
      const int pool = dir_lookup(E, vx, vy, vz);
      return pool >= 0 && surface_bit(T, pool, local_index(vx, vy, vz)) != 0;
    };
    seed = probe(xc, yc, zc) || (xp != xc && probe(xp, yc, zc)) || (xm != xc && probe(xm, yc, zc)) ||
           (yp != yc && probe(xc, yp, zc)) || (ym != yc && probe(xc, ym, zc)) || (zp != zc && probe(xc, yc, zp)) ||
           (zm != zc && probe(xc, yc, zm));
    if (kBits && seed) {  // any stamped block a sign probe from this site can reach (centre +- ve per axis)?
      const int bx0 = E.vox[kVoxMe * total + ix] >> 3, bx1 = E.vox[kVoxPe * total + ix] >> 3;
      const int by0 = E.vox[kVoxMe * total + iy] >> 3, by1 = E.vox[kVoxPe * total + iy] >> 3;
      const int bz0 = E.vox[kVoxMe * total + iz] >> 3, bz1 = E.vox[kVoxPe * total + iz] >> 3;
      for (int bz = bz0; bz <= bz1; ++bz)
        for (int by = by0; by <= by1; ++by)
          for (int bx = bx0; bx <= bx1; ++bx) {
            const int pool = __ldg(E.dir + (bx + E.dn[0] * (by + E.dn[1] * bz)));
            if (pool >= 0 && T.pool_geom[pool]) geom_near = true;
          }
    }
  }
  const uint32_t votes = __ballot_sync(0xFFFFFFFFu, seed);
  if (kBits) {
    const uint32_t gvotes = __ballot_sync(0xFFFFFFFFu, geom_near);
    if (lane == 0) {
      E.mbits[row * E.wpr + xw] = votes;
      E.gbits[row * E.wpr + xw] = gvotes;
    }
  } else if (x < E.nx) {
    E.mask[x + E.nx * row] = seed ? 1 : 0;
  }
  if (lane == 0 && votes != 0) atomicAdd(&E.ctrl->seed_count, static_cast<unsigned long long>(__popc(votes)));
}

// The fused build's gather: one WARP per active 8^3-cell brick (16 cells per lane), persistent grid
// over the compacted active list; the bit planes are cleared beforehand, so inactive bricks cost
// nothing.  A warp stages what its brick's 512 x 7 probes can touch -- the directory entries of the
// <= kStage blocks in reach and the surface bit planes of the live ones -- in its own slice of shared
// memory (only __syncwarp), so a probe is two shared-memory reads, and 48 bricks are in flight per SM.
// Output: one byte per (y, z) row of the brick in the seed plane and in the geometry-near plane.
constexpr int kStage = 64;
constexpr int kGatherWarps = 8;
struct GatherStage {
  int pool[kStage];
  uint32_t plane[kStage][16];
  uint8_t geom[kStage];
};
__global__ void __launch_bounds__(kGatherWarps * 32) k_seed_gather_bricks(EsdfView E, TsdfView T) {
  pdl_wait();
  __shared__ GatherStage s_stage[kGatherWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  GatherStage& S = s_stage[warp];
  uint8_t* mrow = reinterpret_cast<uint8_t*>(E.mbits);
  uint8_t* grow = reinterpret_cast<uint8_t*>(E.gbits);
  const int total = E.nx + E.ny + E.nz;
  const int* vox_x = E.vox;
  const int* vox_y = E.vox + E.nx;
  const int* vox_z = E.vox + E.nx + E.ny;
  const int n_active = E.ctrl->active_bricks;
  const int lx = lane & 7, lyq = lane >> 3;  // lane covers x = lx, y in {lyq, lyq + 4}, all 8 z of the brick
  for (int item = blockIdx.x * kGatherWarps + warp; item < n_active; item += gridDim.x * kGatherWarps) {
    const int brick = E.active[item];
    const int bx = brick % E.bnx, by = (brick / E.bnx) % E.bny, bz = brick / (E.bnx * E.bny);
    // block range in reach of the brick: [first centre - ve, last centre + ve] per axis (lanes 0..2 = axes)
    int lo_a = 0, n_a = 1;
    if (lane < 3) {
      const int dim = lane == 0 ? E.nx : (lane == 1 ? E.ny : E.nz);
      const int b0 = 8 * (lane == 0 ? bx : (lane == 1 ? by : bz));
      const int first = axis_base(E, lane) + b0, last = axis_base(E, lane) + min(b0 + 7, dim - 1);
      lo_a = E.vox[kVoxMe * total + first] >> 3;
      n_a = (E.vox[kVoxPe * total + last] >> 3) - lo_a + 1;
    }
    const int lo0 = __shfl_sync(0xFFFFFFFFu, lo_a, 0), lo1 = __shfl_sync(0xFFFFFFFFu, lo_a, 1), lo2 = __shfl_sync(0xFFFFFFFFu, lo_a, 2);
    const int n0 = __shfl_sync(0xFFFFFFFFu, n_a, 0), n1 = __shfl_sync(0xFFFFFFFFu, n_a, 1), n2 = __shfl_sync(0xFFFFFFFFu, n_a, 2);
    const int nblocks = n0 * n1 * n2;
    const bool staged = nblocks <= kStage;
    __syncwarp();  // the previous brick's staging is no longer read
    if (staged) {
      for (int i = lane; i < nblocks; i += 32) {
        const int cx = i % n0, cy = (i / n0) % n1, cz = i / (n0 * n1);
        const int pool = __ldg(E.dir + ((lo0 + cx) + E.dn[0] * ((lo1 + cy) + E.dn[1] * (lo2 + cz))));
        S.pool[i] = pool;
        S.geom[i] = pool >= 0 ? T.pool_geom[pool] : 0;
      }
      __syncwarp();
      for (int i = lane; i < nblocks * 16; i += 32) {
        const int pool = S.pool[i >> 4];
        S.plane[i >> 4][i & 15] = pool >= 0 ? __ldg(T.digest + (pool * kDigestWords + (i & 15))) : 0u;
      }
      __syncwarp();
    }
    const int x = 8 * bx + lx;
    const bool x_ok = x < E.nx;
    const int xi = min(x, E.nx - 1);
    const int xc = vox_x[xi], xp = vox_x[total + xi], xm = vox_x[2 * total + xi];
    const int gx0 = vox_x[kVoxMe * total + xi] >> 3, gx1 = vox_x[kVoxPe * total + xi] >> 3;
    auto probe = [&](int vx, int vy, int vz) -> bool {
      const int local = local_index(vx, vy, vz);
      if (staged) {
        const int b = ((vx >> 3) - lo0) + n0 * (((vy >> 3) - lo1) + n1 * ((vz >> 3) - lo2));
        return (S.plane[b][local >> 5] >> (local & 31)) & 1u;
      }
      const int pool = dir_lookup(E, vx, vy, vz);
      return pool >= 0 && surface_bit(T, pool, local) != 0;
    };
    unsigned seeds_here = 0;
    for (int lz = 0; lz < 8; ++lz) {
      const int z = 8 * bz + lz;
      const int zi = min(z, E.nz - 1);
      const int zc = vox_z[zi], zp = vox_z[total + zi], zm = vox_z[2 * total + zi];
      const int gz0 = vox_z[kVoxMe * total + zi] >> 3, gz1 = vox_z[kVoxPe * total + zi] >> 3;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int y = 8 * by + lyq + 4 * h;
        const int yi = min(y, E.ny - 1);
        bool seed = false, geom_near = false;
        if (x_ok && y < E.ny && z < E.nz) {
          const int yc = vox_y[yi], yp = vox_y[total + yi], ym = vox_y[2 * total + yi];
          seed = probe(xc, yc, zc) || (xp != xc && probe(xp, yc, zc)) || (xm != xc && probe(xm, yc, zc)) ||
                 (yp != yc && probe(xc, yp, zc)) || (ym != yc && probe(xc, ym, zc)) || (zp != zc && probe(xc, yc, zp)) ||
                 (zm != zc && probe(xc, yc, zm));
          if (seed) {  // any stamped block a sign probe from this site can reach (centre +- ve per axis)?
            const int gy0 = vox_y[kVoxMe * total + yi] >> 3, gy1 = vox_y[kVoxPe * total + yi] >> 3;
            for (int cz = gz0; cz <= gz1; ++cz)
              for (int cy = gy0; cy <= gy1; ++cy)
                for (int cx = gx0; cx <= gx1; ++cx) {
                  if (staged) {
                    geom_near |= S.geom[(cx - lo0) + n0 * ((cy - lo1) + n1 * (cz - lo2))] != 0;
                  } else {
                    const int pool = __ldg(E.dir + (cx + E.dn[0] * (cy + E.dn[1] * cz)));
                    geom_near |= pool >= 0 && T.pool_geom[pool];
                  }
                }
          }
        }
        // the ballot is 4 rows (y) of 8 x cells: byte k belongs to row lyq = k
        const uint32_t votes = __ballot_sync(0xFFFFFFFFu, seed);
        const uint32_t gvotes = __ballot_sync(0xFFFFFFFFu, geom_near);
        if (lx == 0 && y < E.ny && z < E.nz) {
          const int out_byte = (y + E.ny * z) * (E.wpr * 4) + bx;  // byte bx of row (y, z): bits 8bx .. 8bx+7
          mrow[out_byte] = static_cast<uint8_t>(votes >> (8 * lyq));
          grow[out_byte] = static_cast<uint8_t>(gvotes >> (8 * lyq));
        }
        seeds_here += __popc(votes);
      }
    }
    if (lane == 0 && seeds_here != 0) atomicAdd(&E.ctrl->seed_count, static_cast<unsigned long long>(seeds_here));
  }
}

// ---- seed_gather as resample + dilate (fused build, when bind_tsdf validated the identity) ----
// With ve <= tsdf voxel the probe at centre +- ve/2 lands either in the centre's own voxel or in the
// voxel of the neighbouring cell's centre (checked exactly, per axis position, against the per-axis
// tables).  Then  seed = C | (C shifted along +-x, y, z, where the probe leaves the voxel)  with
// C = surface bit of the centre voxel: one digest bit per cell and a handful of word operations per
// 32 cells instead of seven probes per cell.
// One warp per extended (y, z) row.  Step 1, lane <-> block column: the row's voxel-space bits (surface,
// own-sign, geometry-near), one byte per block, into the warp's slice of shared memory; most rows cross no
// live block and end there.  Step 2, lane <-> cell: every cell picks the bit of its centre voxel.
constexpr int kResampleWarps = 8;
constexpr int kMaxDirX = (kMaxDim + 2) / 8 + 8;
__global__ void __launch_bounds__(kResampleWarps * 32) k_resample_rows(EsdfView E, TsdfView T) {
  pdl_enter();
  __shared__ uint8_t s_bits[kResampleWarps][3][kMaxDirX];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ey = E.ny + 2, ez = E.nz + 2;
  const int row = blockIdx.x * kResampleWarps + warp;
  if (row >= ey * ez) return;
  const int yi = row % ey, zi = row / ey;
  const int vy = E.voxe[(E.nx + 2) + yi], vz = E.voxe[(E.nx + 2) + ey + zi];
  const int ly = vy & 7, lz = vz & 7;
  const int drow = E.dn[0] * ((vy >> 3) + E.dn[1] * (vz >> 3));
  uint8_t(*S)[kMaxDirX] = s_bits[warp];
  bool any = false;
  for (int b = lane; b < E.dn[0]; b += 32) {
    const int pool = __ldg(E.dir + drow + b);
    uint32_t sb = 0, ob = 0;
    if (pool >= 0) {
      const uint32_t* dg = T.digest + pool * kDigestWords;
      sb = (__ldg(dg + 2 * lz + (ly >> 2)) >> (8 * (ly & 3))) & 0xFFu;
      const uint32_t pairs = (__ldg(dg + kDigestComb + 4 * lz + (ly >> 1)) >> (16 * (ly & 1))) & 0xFFFFu;
      uint32_t both = pairs & (pairs >> 1) & 0x5555u;  // bit 2k: voxel k has a value and it is negative
      both = (both | both >> 1) & 0x3333u;
      both = (both | both >> 2) & 0x0F0Fu;
      ob = (both | both >> 4) & 0xFFu;
    }
    const uint8_t nb = E.dirg[drow + b] ? 0xFFu : 0u;
    S[0][b] = static_cast<uint8_t>(sb), S[1][b] = static_cast<uint8_t>(ob), S[2][b] = nb;
    any |= (sb | ob | nb) != 0;
  }
  any = __any_sync(0xFFFFFFFFu, any);
  uint32_t* out = E.cbits + row * E.wpr2;
  const size_t plane = static_cast<size_t>(E.wpr2) * ey * ez;
  if (!any) {
    for (int w = lane; w < E.wpr2; w += 32) out[w] = 0u, out[plane + w] = 0u, out[2 * plane + w] = 0u;
    return;
  }
  __syncwarp();
  if (E.xshift >= 0) {  // grids in step: a cell word is 32 consecutive bits of the voxel-space row
    for (int w = lane; w < E.wpr2; w += 32) {
      const int o = 32 * w + E.xshift;
      uint32_t word[3];
#pragma unroll
      for (int pl = 0; pl < 3; ++pl) {
        uint64_t bits = 0;
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const int b = (o >> 3) + k;
          bits |= static_cast<uint64_t>(b < E.dn[0] ? S[pl][b] : 0) << (8 * k);
        }
        word[pl] = static_cast<uint32_t>(bits >> (o & 7));
      }
      const int rest = E.nx + 2 - 32 * w;
      const uint32_t keep = rest < 32 ? (1u << rest) - 1u : 0xFFFFFFFFu;
      out[w] = word[0] & keep, out[plane + w] = word[1] & keep, out[2 * plane + w] = word[2] & keep;
    }
    return;
  }
  for (int w = 0; w < E.wpr2; ++w) {
    const int xi = 32 * w + lane;
    bool c = false, o = false, n = false;
    if (xi < E.nx + 2) {
      const int vx = E.voxe[xi];
      const int b = vx >> 3, k = vx & 7;
      c = (S[0][b] >> k) & 1, o = (S[1][b] >> k) & 1, n = S[2][b] != 0;
    }
    const uint32_t cw = __ballot_sync(0xFFFFFFFFu, c), ow = __ballot_sync(0xFFFFFFFFu, o), nw = __ballot_sync(0xFFFFFFFFu, n);
    if (lane == 0) out[w] = cw, out[plane + w] = ow, out[2 * plane + w] = nw;
  }
}

// The same three planes when the grids are in step along all three axes (every BASELINE config): one warp per block row
// and lz, i.e. the 8 voxel rows ly = 0 .. 7 that share a directory row and six digest words per block.  Step 1, lane <->
// block: one directory read and six digest reads serve eight rows (k_resample_rows: one + two per row).  Step 2, lane <->
// (row, word): a cell word is 32 consecutive bits of the row's byte string -- two aligned 4-byte reads and a funnel
// shift -- with all 32 lanes busy (k_resample_rows: 13 of 32 for a 400-cell row).
constexpr int kRowBytes = (kMaxDirX + 8 + 3) & ~3;
__global__ void __launch_bounds__(kResampleWarps * 32) k_resample_blockrows(EsdfView E, TsdfView T) {
  pdl_enter();
  __shared__ __align__(4) uint8_t s_c[kResampleWarps][8][kRowBytes];  // surface bits, one byte per block
  __shared__ __align__(4) uint8_t s_o[kResampleWarps][8][kRowBytes];  // own-sign bits
  __shared__ __align__(4) uint8_t s_n[kResampleWarps][kRowBytes];     // stamped geometry within one block: 0xFF / 0
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int item = blockIdx.x * kResampleWarps + warp;  // (directory-relative voxel z) * dn[1] + block y
  if (item >= E.dn[1] * E.dn[2] * 8) return;
  const int vz = __float2int_rz((static_cast<float>(item) + 0.5f) * (1.0f / static_cast<float>(E.dn[1]))), by = item - vz * E.dn[1];  // item < 2^17: exact
  const int lz = vz & 7, bz = vz >> 3;
  const int ey = E.ny + 2, ez = E.nz + 2;
  const int zi = vz - E.zshift, yi0 = 8 * by - E.yshift;  // extended row indices of (ly = 0, this vz)
  if (zi < 0 || zi >= ez || yi0 + 7 < 0 || yi0 >= ey) return;
  const int drow = E.dn[0] * (by + E.dn[1] * bz);
  const int padded = min(kRowBytes, (E.dn[0] + 8 + 3) & ~3);  // bytes step 2 may read: zero beyond the last block
  bool any = false;
  for (int b = lane; b < padded; b += 32) {
    uint32_t sw[2] = {0u, 0u}, cw[4] = {0u, 0u, 0u, 0u};
    uint8_t nb = 0;
    if (b < E.dn[0]) {
      const int pool = __ldg(E.dir + drow + b);
      if (pool >= 0) {
        const uint32_t* dg = T.digest + pool * kDigestWords;
        sw[0] = __ldg(dg + 2 * lz), sw[1] = __ldg(dg + 2 * lz + 1);
#pragma unroll
        for (int j = 0; j < 4; ++j) cw[j] = __ldg(dg + kDigestComb + 4 * lz + j);
      }
      nb = E.dirg[drow + b] ? 0xFFu : 0u;
    }
#pragma unroll
    for (int ly = 0; ly < 8; ++ly) {
      const uint32_t pairs = (cw[ly >> 1] >> (16 * (ly & 1))) & 0xFFFFu;
      uint32_t both = pairs & (pairs >> 1) & 0x5555u;  // bit 2k: voxel k has a value and it is negative
      both = (both | both >> 1) & 0x3333u;
      both = (both | both >> 2) & 0x0F0Fu;
      s_c[warp][ly][b] = static_cast<uint8_t>(sw[ly >> 2] >> (8 * (ly & 3)));
      s_o[warp][ly][b] = static_cast<uint8_t>((both | both >> 4) & 0xFFu);
    }
    s_n[warp][b] = nb;
    any |= (sw[0] | sw[1] | cw[0] | cw[1] | cw[2] | cw[3] | nb) != 0;
  }
  any = __any_sync(0xFFFFFFFFu, any);
  __syncwarp();
  const size_t plane = static_cast<size_t>(E.wpr2) * ey * ez;
  const float rcp_wpr2 = 1.0f / static_cast<float>(E.wpr2);
  for (int p = lane; p < 8 * E.wpr2; p += 32) {
    const int ly = __float2int_rz((static_cast<float>(p) + 0.5f) * rcp_wpr2), w = p - ly * E.wpr2;
    const int yi = yi0 + ly;
    if (yi < 0 || yi >= ey) continue;
    uint32_t wc = 0u, wo = 0u, wn = 0u;
    if (any) {
      const int o = 32 * w + E.xshift;
      const int at = (o >> 3) & ~3, sh = 8 * ((o >> 3) & 3) + (o & 7);
      auto word = [&](const uint8_t* bytes) {
        return __funnelshift_r(*reinterpret_cast<const uint32_t*>(bytes + at), *reinterpret_cast<const uint32_t*>(bytes + at + 4), sh);
      };
      const int rest = E.nx + 2 - 32 * w;
      const uint32_t keep = rest < 32 ? (1u << rest) - 1u : 0xFFFFFFFFu;
      wc = word(s_c[warp][ly]) & keep, wo = word(s_o[warp][ly]) & keep, wn = word(s_n[warp]) & keep;
    }
    uint32_t* out = E.cbits + static_cast<size_t>(zi * ey + yi) * E.wpr2 + w;
    out[0] = wc, out[plane] = wo, out[2 * plane] = wn;
  }
}

// one thread per word of the seed plane
__global__ void __launch_bounds__(256) k_seed_dilate(EsdfView E) {
  pdl_enter();
  // grid = (words of a z slice / 256, nz): the slice index splits into (xw, y) by a float reciprocal (exact: the
  // quotient is never closer than 1 / (2 wpr) >= 0.015 to an integer, the product is off by < 1e-2 for < 2^15 words)
  const int j = blockIdx.x * blockDim.x + threadIdx.x, z = blockIdx.y;
  const int slice = E.wpr * E.ny;
  const int lane = threadIdx.x & 31;
  uint32_t seed = 0, near = 0;
  int row = 0, xw = 0;
  const int i = z * slice + j;
  if (j < slice) {
    const int y = __float2int_rz((static_cast<float>(j) + 0.5f) * (1.0f / static_cast<float>(E.wpr)));
    xw = j - y * E.wpr, row = z * E.ny + y;
    const int ey = E.ny + 2;
    auto ext = [&](const uint32_t* plane, int yy, int zz) -> uint64_t {  // extended bits 32xw .. 32xw+63 of row (yy, zz)
      const uint32_t* r = plane + ((zz + 1) * ey + (yy + 1)) * E.wpr2 + xw;
      return static_cast<uint64_t>(r[0]) | (xw + 1 < E.wpr2 ? static_cast<uint64_t>(r[1]) << 32 : 0ull);
    };
    // every load up front (one round trip): the row itself, its four neighbours, the geometry-near row
    const uint64_t w = ext(E.cbits, y, z);  // bit k = cell 32xw + k - 1
    const uint64_t wyp = ext(E.cbits, y + 1, z), wym = ext(E.cbits, y - 1, z), wzp = ext(E.cbits, y, z + 1), wzm = ext(E.cbits, y, z - 1);
    const uint64_t wn = ext(E.nbits, y, z);
    const uint8_t fy = E.yzflags[y], fz = E.yzflags[E.ny + z];
    seed = static_cast<uint32_t>(w >> 1) | (static_cast<uint32_t>(w >> 2) & E.xplus[xw]) | (static_cast<uint32_t>(w) & E.xminus[xw]);
    if (fy & 1) seed |= static_cast<uint32_t>(wyp >> 1);
    if (fy & 2) seed |= static_cast<uint32_t>(wym >> 1);
    if (fz & 1) seed |= static_cast<uint32_t>(wzp >> 1);
    if (fz & 2) seed |= static_cast<uint32_t>(wzm >> 1);
    const int rest = E.nx - 32 * xw;
    if (rest < 32) seed &= (1u << rest) - 1u;
    near = seed & static_cast<uint32_t>(wn >> 1);
    E.mbits[i] = seed;
    E.gbits[i] = near;
  }
  // seeds with no stamped block in reach resolve no sign probe: their table is all zero
  // (only read when the y sweep's keys cannot carry the "site has a table" bit and every site counts as having one)
  if (E.tab_all)
    for (uint32_t m = seed & ~near; m != 0; m &= m - 1) E.gtab[32 * xw + __ffs(static_cast<int>(m)) - 1 + E.nx * row] = make_uint2(0u, 0u);
  // the others go on the work list of k_site_tables (one atomic per warp)
  const int mine = __popc(near);
  int before = mine;
  for (int d = 1; d < 32; d <<= 1) {
    const int up = __shfl_up_sync(0xFFFFFFFFu, before, d);
    if (lane >= d) before += up;
  }
  const int total = __shfl_sync(0xFFFFFFFFu, before, 31);
  if (total != 0) {
    int base = 0;
    if (lane == 0) base = atomicAdd(&E.ctrl->seed_words, total);
    base = __shfl_sync(0xFFFFFFFFu, base, 0) + before - mine;
    for (uint32_t m = near; m != 0; m &= m - 1) E.seedw[base++] = 32 * xw + __ffs(static_cast<int>(m)) - 1 + E.nx * row;
  }
  // seed count: one atomic per CTA (10 K same-address atomics, one per warp, were a visible part of this kernel)
  __shared__ unsigned s_count;
  if (threadIdx.x == 0) s_count = 0;
  __syncthreads();
  unsigned count = __popc(seed);
  for (int d = 16; d > 0; d >>= 1) count += __shfl_down_sync(0xFFFFFFFFu, count, d);
  if (lane == 0 && count != 0) atomicAdd(&s_count, count);
  __syncthreads();
  if (threadIdx.x == 0 && s_count != 0) atomicAdd(&E.ctrl->seed_count, static_cast<unsigned long long>(s_count));
}

// Per-site sign tables: for every seed with a stamped block in reach, the geometry pairs {has value, negative}
// of the 27 voxels around its centre voxel (the only voxels a sign probe from that site can land in when
// ve <= v), read as 9 x-rows of three voxels from the digest's pair plane.  Persistent grid over the
// compacted list of those seeds, one thread per seed.
__global__ void __launch_bounds__(256) k_site_tables(EsdfView E, TsdfView T) {
  pdl_enter();
  const int count = E.ctrl->seed_words;
  for (int item = blockIdx.x * blockDim.x + threadIdx.x; item < count; item += gridDim.x * blockDim.x) {
    const int cell = E.seedw[item];
    const int x = cell % E.nx, row = cell / E.nx;
    const int y = row % E.ny, z = row / E.ny;
    const int vx = E.vox[x], vy0 = E.vox[E.nx + y], vz0 = E.vox[E.nx + E.ny + z];
    const int bxa = (vx - 1) >> 3, bxm = vx >> 3, bxb = (vx + 1) >> 3;
    uint32_t has = 0, neg = 0;
#pragma unroll
    for (int r = 0; r < 9; ++r) {
      const int vy = vy0 + r % 3 - 1, vz = vz0 + r / 3 - 1;
      const int drow = E.dn[0] * ((vy >> 3) + E.dn[1] * (vz >> 3));
      const int dword = kDigestGeom + 4 * (vz & 7) + ((vy & 7) >> 1), shift = 16 * (vy & 1);
      const int pa = __ldg(E.dir + drow + bxa);
      const uint32_t wa = pa >= 0 ? (__ldg(T.digest + pa * kDigestWords + dword) >> shift) & 0xFFFFu : 0u;
      uint32_t wb = wa;
      if (bxb != bxa) {
        const int pb = __ldg(E.dir + drow + bxb);
        wb = pb >= 0 ? (__ldg(T.digest + pb * kDigestWords + dword) >> shift) & 0xFFFFu : 0u;
      }
      const uint32_t g0 = (wa >> (2 * ((vx - 1) & 7))) & 3u;
      const uint32_t g1 = ((bxm == bxa ? wa : wb) >> (2 * (vx & 7))) & 3u;
      const uint32_t g2 = (wb >> (2 * ((vx + 1) & 7))) & 3u;
      has |= ((g0 & 1u) | (g1 & 1u) << 1 | (g2 & 1u) << 2) << (3 * r);
      neg |= ((g0 >> 1) | (g1 >> 1) << 1 | (g2 >> 1) << 2) << (3 * r);
    }
    E.gtab[cell] = make_uint2(has, neg);
  }
}

// ---- seed_scatter (esdf.hpp:73-98): every surface voxel of every live block marks its cell ----
__global__ void __launch_bounds__(512) k_seed_scatter(EsdfView E, TsdfView T) {
  pdl_enter();
  const int bound = T.ctrl->next_fresh;
  const int tid = threadIdx.x;
  const int lx = tid & 7, ly = (tid >> 3) & 7, lz = tid >> 6;
  for (int pool = blockIdx.x; pool < bound; pool += gridDim.x) {
    const uint64_t key = T.pool_key[pool];
    if (key == kKeyEmpty) continue;
    if (!surface_bit(T, pool, tid)) continue;
    int bx, by, bz;
    unpack_key(key, bx, by, bz);
    const double cx = (bx * kBlockEdge + lx + 0.5) * T.voxel, cy = (by * kBlockEdge + ly + 0.5) * T.voxel,
                 cz = (bz * kBlockEdge + lz + 0.5) * T.voxel;
    const int ex = static_cast<int>(floor((cx - E.origin[0]) / E.ve));
    const int ey = static_cast<int>(floor((cy - E.origin[1]) / E.ve));
    const int ez = static_cast<int>(floor((cz - E.origin[2]) / E.ve));
    if (ex < 0 || ex >= E.nx || ey < 0 || ey >= E.ny || ez < 0 || ez >= E.nz) continue;
    E.mask[ex + E.nx * (ey + E.ny * ez)] = 1;
  }
}

__global__ void __launch_bounds__(256) k_count_mask(EsdfView E) {
  pdl_enter();
  unsigned local = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < E.cells; i += gridDim.x * blockDim.x) local += E.mask[i] != 0;
  for (int d = 16; d > 0; d >>= 1) local += __shfl_down_sync(0xFFFFFFFFu, local, d);
  if ((threadIdx.x & 31) == 0 && local != 0) atomicAdd(&E.ctrl->seed_count, static_cast<unsigned long long>(local));
}

// ---- phase 1: nearest seed along z per (x, y) column (esdf.hpp:213-233) ----
// One warp per 32 consecutive x columns of one y.  The column's seeds become a bit string (bit z)
// in shared memory ([word][lane], conflict free); one ascending sweep then tracks the last seed
// at/below z and the next one above it.  Ties keep the lower z (strict '<', esdf.hpp:229).
// kBits: the mask is the x-packed bit plane of the fused build; a 32(z) x 32(x) bit tile is
// transposed with one load per lane and 32 ballots.  Otherwise it is the reference's byte mask.
constexpr int kFloodWarps = 4;
template <bool kBits>
__global__ void __launch_bounds__(kFloodWarps * 32) k_flood_z(EsdfView E) {
  pdl_wait();
  extern __shared__ uint32_t s_words[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int plane = E.nx * E.ny;
  const int nwords = (E.nz + 31) >> 5;
  const int gw = blockIdx.x * kFloodWarps + warp;
  if (gw >= E.wpr * E.ny) return;
  const int xw = gw % E.wpr, y = gw / E.wpr;
  const int x = xw * 32 + lane;
  uint32_t* words = s_words + warp * (nwords * 32) + lane;  // words[w * 32]
  uint32_t any = 0;
  for (int w = 0; w < nwords; ++w) {
    uint32_t bits = 0;
    if (kBits) {
      const int z = 32 * w + lane;
      const uint32_t mine = z < E.nz ? __ldg(E.mbits + (z * E.ny + y) * E.wpr + xw) : 0u;  // 32 x-bits of row (y, z)
#pragma unroll
      for (int xb = 0; xb < 32; ++xb) {
        const uint32_t col = __ballot_sync(0xFFFFFFFFu, (mine >> xb) & 1u);  // column xb: bit z
        if (lane == xb) bits = col;
      }
    } else if (x < E.nx) {
      const int zend = min(32, E.nz - 32 * w);
      const int col = y * E.nx + x;
#pragma unroll 8
      for (int b = 0; b < zend; ++b) bits |= (E.mask[col + plane * (32 * w + b)] != 0 ? 1u : 0u) << b;
    }
    words[w * 32] = bits;
    any |= bits;
  }
  if (x >= E.nx) return;
  uint16_t* out = E.near_z + y * E.nx + x;
  if (any == 0) {
    for (int z = 0; z < E.nz; ++z) out[plane * z] = edt::kNone;
    return;
  }
  auto next_set = [&](int from) -> int {  // first set bit at position >= from, or -1
    if (from >= E.nz) return -1;
    int w = from >> 5;
    uint32_t m = words[w * 32] & (0xFFFFFFFFu << (from & 31));
    while (m == 0 && ++w < nwords) m = words[w * 32];
    return m != 0 ? 32 * w + __ffs(static_cast<int>(m)) - 1 : -1;
  };
  int below = -1, above = next_set(0);
  for (int z = 0; z < E.nz; ++z) {
    if (z == above) {
      below = z;
      above = next_set(z + 1);
    }
    int pick;
    if (below < 0) pick = above;  // `any` guarantees one of the two exists
    else if (above < 0) pick = below;
    else pick = (above - z) < (z - below) ? above : below;
    out[plane * z] = static_cast<uint16_t>(pick);
  }
}

// byte mask (the reference's SeedMask) -> x-packed bit plane, one warp per word
__global__ void __launch_bounds__(256) k_pack_mask(EsdfView E) {
  pdl_wait();
  const int warp_id = static_cast<int>((blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (warp_id >= E.wpr * E.ny * E.nz) return;
  const int xw = warp_id % E.wpr, row = warp_id / E.wpr;
  const int x = 32 * xw + lane;
  const uint32_t bits = __ballot_sync(0xFFFFFFFFu, x < E.nx && E.mask[x + E.nx * row] != 0);
  if (lane == 0) E.mbits[warp_id] = bits;
}

// 32 x 32 bit transpose inside a warp: lane i enters with row i, leaves with column i (bit j = row j's bit i).
// Five butterfly rounds (one shuffle each) instead of 32 ballots.
__device__ __forceinline__ uint32_t transpose32(uint32_t v, int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const uint32_t m = s == 16 ? 0x0000FFFFu : s == 8 ? 0x00FF00FFu : s == 4 ? 0x0F0F0F0Fu : s == 2 ? 0x33333333u : 0x55555555u;
    const uint32_t other = __shfl_xor_sync(0xFFFFFFFFu, v, s);
    v = (lane & s) ? ((v & ~m) | ((other >> s) & m)) : ((v & m) | ((other << s) & ~m));
  }
  return v;
}

// Phase 1 of the divide-and-conquer path (esdf.hpp:213-233), as data for phase 2 rather than a field: one CTA
// per 32 consecutive x columns of one y, one warp per 32 z.  Warp w transposes its 32(z) x 32(x) bit tile of
// the x-packed mask into word w of every column's bit string and adds, per word, the nearest seed in the
// words below and above.  Phase 2 resolves "nearest seed along z" from one word + one info word per
// candidate, so the 2-byte-per-cell nearest-z field is never written or read.  The "seed has a sign table" plane
// (gbits) is transposed alongside: phase 2 hands that bit on, and the x sweep needs no site decode where it is 0.
// zinfo half = distance (15 bits) | table bit << 15: the low half counts from the word's bit 0 down to the nearest seed in
// the words below, the high half from its bit 31 up to the nearest seed in the words above; kZNone (farther than any
// grid is long) when there is none, so "no seed at all" falls out of the minimum without a flag of its own.
constexpr uint32_t kZNone = 0x4000u;
__global__ void __launch_bounds__(1024) k_flood_cols(EsdfView E) {
  pdl_enter();
  extern __shared__ uint32_t s_words[];  // [nzw][32] seeds, then [nzw][32] table bits
  uint32_t* s_tab = s_words + E.nzw * 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int xw = blockIdx.x, y = blockIdx.y;  // grid = (words per row, ny): no division
  const int x = xw * 32 + lane;
  {
    const int z = 32 * w + lane;
    const int o = (z * E.ny + y) * E.wpr + xw;
    const uint32_t mine = z < E.nz ? __ldg(E.mbits + o) : 0u;  // 32 x-bits of row (y, z)
    const uint32_t tab = z < E.nz ? __ldg(E.gbits + o) : 0u;
    s_words[w * 32 + lane] = transpose32(mine, lane);
    s_tab[w * 32 + lane] = transpose32(tab, lane) ;
  }
  __syncthreads();
  if (x >= E.nx) return;
  uint32_t below = kZNone, above = kZNone;
  for (int k = w - 1; k >= 0; --k) {
    const uint32_t m = s_words[k * 32 + lane];
    if (m != 0) {
      const int b = 31 - __clz(static_cast<int>(m));
      below = static_cast<uint32_t>(32 * w - (32 * k + b)) | ((s_tab[k * 32 + lane] >> b) & 1u) << 15;
      break;
    }
  }
  for (int k = w + 1; k < E.nzw; ++k) {
    const uint32_t m = s_words[k * 32 + lane];
    if (m != 0) {
      const int b = __ffs(static_cast<int>(m)) - 1;
      above = static_cast<uint32_t>((32 * k + b) - (32 * w + 31)) | ((s_tab[k * 32 + lane] >> b) & 1u) << 15;
      break;
    }
  }
  const int o = (y * E.nzw + w) * E.nx + x;
  E.zbits[o] = s_words[w * 32 + lane];
  E.zgbits[o] = s_tab[w * 32 + lane] & s_words[w * 32 + lane];
  E.zinfo[o] = below | above << 16;
}

// The fused build's phase 1: one CTA per 32 consecutive x columns of one y, one warp per 32 z.  Warp w
// transposes its 32(z) x 32(x) bit tile of the x-packed mask into word w of every column's bit string
// (shared memory, [word][lane]); after the barrier it walks its own 32 z upwards, so a column's work is
// spread over nz/32 warps instead of one.
__global__ void __launch_bounds__(1024) k_flood_z_chunks(EsdfView E) {
  pdl_wait();
  extern __shared__ uint32_t s_words[];  // [nwords][32]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nwords = (E.nz + 31) >> 5;
  const int xw = blockIdx.x % E.wpr, y = blockIdx.x / E.wpr;
  const int x = xw * 32 + lane;
  {
    const int z = 32 * w + lane;
    const uint32_t mine = z < E.nz ? __ldg(E.mbits + (z * E.ny + y) * E.wpr + xw) : 0u;  // 32 x-bits of row (y, z)
    uint32_t bits = 0;
#pragma unroll
    for (int xb = 0; xb < 32; ++xb) {
      const uint32_t col = __ballot_sync(0xFFFFFFFFu, (mine >> xb) & 1u);  // column xb: bit z
      if (lane == xb) bits = col;
    }
    s_words[w * 32 + lane] = bits;
  }
  __syncthreads();
  if (x >= E.nx) return;
  const uint32_t* words = s_words + lane;  // words[k * 32]
  const int z0 = 32 * w, z1 = min(z0 + 32, E.nz);
  // nearest seed strictly below z0, and at or above z0
  int below = -1;
  for (int k = w - 1; k >= 0; --k) {
    const uint32_t m = words[k * 32];
    if (m != 0) {
      below = 32 * k + 31 - __clz(static_cast<int>(m));
      break;
    }
  }
  auto next_set = [&](int from) -> int {  // first set bit at position >= from, or -1
    if (from >= E.nz) return -1;
    int k = from >> 5;
    uint32_t m = words[k * 32] & (0xFFFFFFFFu << (from & 31));
    while (m == 0 && ++k < nwords) m = words[k * 32];
    return m != 0 ? 32 * k + __ffs(static_cast<int>(m)) - 1 : -1;
  };
  int above = next_set(z0);
  uint16_t* out = E.near_z + (z0 * E.ny + y) * E.nx + x;
  const int plane = E.nx * E.ny;
  for (int z = z0; z < z1; ++z, out += plane) {
    if (z == above) {
      below = z;
      above = next_set(z + 1);
    }
    int pick;
    if (below < 0) pick = above < 0 ? static_cast<int>(edt::kNone) : above;
    else if (above < 0) pick = below;
    else pick = (above - z) < (z - below) ? above : below;  // ties keep the lower z (strict '<', esdf.hpp:229)
    *out = static_cast<uint16_t>(pick);
  }
}

// ---- sign of a cell given its site (recover_signs, esdf.hpp:295-313) ----
// The reference probes the geometry channel at site_centre + ve * normalize(cell_centre - site_centre)
// and reads floor(probe / v_tsdf) per axis.  Which TSDF voxel that is gets decided, per axis, by
//   delta == 0            : the probe coordinate IS the site centre           -> table row kVoxC
//   only this axis != 0   : normalize() gives exactly +-1 (sqrt(d*d) == |d|)  -> table rows kVoxPe / kVoxMe
//   otherwise             : fp32 estimate of the offset, accepted only when it is farther from a voxel
//                           face than its error bound; else the reference's own fp64 sequence.
// so the voxel index is always the one the reference computes.  Two hints skip work without changing the
// result: a site with no stamped block within reach cannot resolve a geometry probe (gbits), and a cell
// in an inactive brick has no allocated block under its own centre (fallback lookup).
struct SignProbe {
  const EsdfView& E;
  const TsdfView& T;
  int total;
  int y, z, iy, iz;
  int own_vy, own_vz;   // the cell's own voxel (fallback lookup)
  int brick_row;
  // current site
  int sx, sy, sz, jx, jy, jz;
  int v0x, v0y, v0z;
  float qx, qy, qz;
  bool geom_near;

  __device__ __forceinline__ SignProbe(const EsdfView& E_, const TsdfView& T_, int y_, int z_) : E(E_), T(T_) {
    total = E.nx + E.ny + E.nz;
    y = y_, z = z_;
    iy = E.nx + y, iz = E.nx + E.ny + z;
    own_vy = E.vox[iy], own_vz = E.vox[iz];
    brick_row = E.bnx * ((y >> 3) + E.bny * (z >> 3));
    sx = sy = sz = -1;
    geom_near = true;
  }
  template <bool kHints>
  __device__ __forceinline__ void set_site(int sx_, int sy_, int sz_) {
    sx = sx_, sy = sy_, sz = sz_;
    jx = sx, jy = E.nx + sy, jz = E.nx + E.ny + sz;
    geom_near = !kHints || ((__ldg(E.gbits + ((sz * E.ny + sy) * E.wpr + (sx >> 5))) >> (sx & 31)) & 1u) != 0;
    if (geom_near) {
      v0x = E.vox[jx], v0y = E.vox[jy], v0z = E.vox[jz];
      qx = E.qsf[jx], qy = E.qsf[jy], qz = E.qsf[jz];
    }
  }
  template <bool kHints>
  __device__ __forceinline__ bool negative(int x) const {
    const int dx = x - sx, dy = y - sy, dz = z - sz;
    if (geom_near && (dx | dy | dz) != 0) {  // delta.squaredNorm() > 0 (distinct cells have distinct centres)
      int vx, vy, vz;
      if ((dx != 0) + (dy != 0) + (dz != 0) == 1) {
        vx = dx == 0 ? v0x : E.vox[(dx > 0 ? kVoxPe : kVoxMe) * total + jx];
        vy = dy == 0 ? v0y : E.vox[(dy > 0 ? kVoxPe : kVoxMe) * total + jy];
        vz = dz == 0 ? v0z : E.vox[(dz > 0 ? kVoxPe : kVoxMe) * total + jz];
      } else {
        const float fx = static_cast<float>(dx), fy = static_cast<float>(dy), fz = static_cast<float>(dz);
        const float rinv = rsqrtf(fx * fx + fy * fy + fz * fz) * E.ratio;
        const float ox = qx + fx * rinv, oy = qy + fy * rinv, oz = qz + fz * rinv;
        const float tol = 4e-6f * (1.0f + E.ratio);
        const bool sure = (dx == 0 || fabsf(ox - rintf(ox)) > tol) && (dy == 0 || fabsf(oy - rintf(oy)) > tol) &&
                          (dz == 0 || fabsf(oz - rintf(oz)) > tol);
        if (sure) {
          vx = v0x + (dx == 0 ? 0 : __float2int_rd(ox));
          vy = v0y + (dy == 0 ? 0 : __float2int_rd(oy));
          vz = v0z + (dz == 0 ? 0 : __float2int_rd(oz));
        } else {  // the reference's arithmetic, operation by operation
          const double px = E.ctr[jx], py = E.ctr[jy], pz = E.ctr[jz];
          const double ex = E.ctr[x] - px, ey = E.ctr[iy] - py, ez = E.ctr[iz] - pz;
          const double n = sqrt(sum3(ex * ex, ey * ey, ez * ez));
          vx = voxel_index(px + E.ve * (ex / n), T.voxel) - 8 * E.dlo[0];
          vy = voxel_index(py + E.ve * (ey / n), T.voxel) - 8 * E.dlo[1];
          vz = voxel_index(pz + E.ve * (ez / n), T.voxel) - 8 * E.dlo[2];
        }
      }
      const int pool = dir_lookup(E, vx, vy, vz);
      if (pool >= 0) {
        const uint32_t g = pair_bits(T, pool, kDigestGeom, local_index(vx, vy, vz));
        if (g & 1u) return (g & 2u) != 0;  // query_tsdf_geom has a value: its sign decides
      }
    }
    // unresolved: combined sdf at the query cell's own centre (esdf.hpp:309-312)
    if (kHints && !(E.brick[brick_row + (x >> 3)] & 1)) return false;
    const int vx = E.vox[x];
    const int pool = dir_lookup(E, vx, own_vy, own_vz);
    if (pool < 0) return false;
    return pair_bits(T, pool, kDigestComb, local_index(vx, own_vy, own_vz)) == 3u;
  }
};

// The same decision from per-site tables (fused build with resampled seeding, ve <= tsdf voxel): the probe
// voxel is the site's centre voxel plus an offset in {-1,0,1}^3, and k_site_tables stored the geometry pair
// of those 27 voxels for every seed (all zero when no stamped block is in reach); the fallback is one bit
// of the own-sign plane.  The offset comes from the fp32 estimate when it is certified, else the cell takes
// SignProbe's exact path.  No directory or digest access per cell.
struct SignTable {
  const EsdfView& E;
  const TsdfView& T;
  const float* qsf;  // E.qsf, staged in shared memory by the caller
  int y, z;
  int sx, sy, sz;
  uint2 tab;
  float qx, qy, qz;

  __device__ __forceinline__ SignTable(const EsdfView& E_, const TsdfView& T_, const float* qsf_, int y_, int z_)
      : E(E_), T(T_), qsf(qsf_) {
    y = y_, z = z_;
    sx = sy = sz = -1;
    tab = make_uint2(0u, 0u);
  }
  __device__ __forceinline__ void set_site(int sx_, int sy_, int sz_, uint2 tab_) {
    sx = sx_, sy = sy_, sz = sz_, tab = tab_;
    if (tab.x != 0 && !E.iprobe) qx = qsf[sx], qy = qsf[E.nx + sy], qz = qsf[E.nx + E.ny + sz];
  }
  // own: the cell's bit of the own-sign plane
  __device__ __forceinline__ bool negative(int x, bool own) const {
    const int dx = x - sx, dy = y - sy, dz = z - sz;
    if (E.iprobe) {
      // Grids in step (ve == v, cell centres at voxel centres): the probe site + ve * d / |d| leaves the site's voxel along
      // an axis exactly when |d_a| / |d| > 1/2, i.e. 4 d_a^2 > |d|^2 -- integers.  Equality would need 3 a^2 = b^2 + c^2,
      // which has no integer solution but 0, so the nearest the real quantity comes to the voxel face is 1 / (6 |d|^2)
      // >= 8e-8 voxels: five orders of magnitude beyond what the reference's fp64 rounding (or the 1e-9 the centres may
      // be off, checked at bind time) can move it.  Same voxel as esdf.hpp:303-304, no square root, no certificate.
      if (tab.x != 0 && (dx | dy | dz) != 0) {
        const int d2 = dx * dx + dy * dy + dz * dz;
        int idx = 13;
        if (4 * dx * dx > d2) idx += dx > 0 ? 1 : -1;
        if (4 * dy * dy > d2) idx += dy > 0 ? 3 : -3;
        if (4 * dz * dz > d2) idx += dz > 0 ? 9 : -9;
        if ((tab.x >> idx) & 1u) return ((tab.y >> idx) & 1u) != 0;  // query_tsdf_geom has a value: its sign decides
      }
      return own;
    }
    if (tab.x != 0 && (dx | dy | dz) != 0) {
      const float fx = static_cast<float>(dx), fy = static_cast<float>(dy), fz = static_cast<float>(dz);
      const float rinv = rsqrtf(fx * fx + fy * fy + fz * fz) * E.ratio;
      const float ox = qx + fx * rinv, oy = qy + fy * rinv, oz = qz + fz * rinv;
      const float tol = 4e-6f * (1.0f + E.ratio);
      const bool sure = (dx == 0 || fabsf(ox - rintf(ox)) > tol) && (dy == 0 || fabsf(oy - rintf(oy)) > tol) &&
                        (dz == 0 || fabsf(oz - rintf(oz)) > tol);
      if (!sure) return exact_negative(x, own);
      const int idx = (dx == 0 ? 1 : __float2int_rd(ox) + 1) + 3 * (dy == 0 ? 1 : __float2int_rd(oy) + 1) +
                      9 * (dz == 0 ? 1 : __float2int_rd(oz) + 1);
      if ((tab.x >> idx) & 1u) return ((tab.y >> idx) & 1u) != 0;  // query_tsdf_geom has a value: its sign decides
    }
    return own;  // combined sdf at the cell's own centre (esdf.hpp:309-312)
  }
  // rare: the fp32 estimate sits too close to a voxel face -- the reference's arithmetic, operation by operation
  // (esdf.hpp:297-308), straight from the directory and the digest
  __device__ __forceinline__ bool exact_negative(int x, bool own) const {
    const double px = E.ctr[sx], py = E.ctr[E.nx + sy], pz = E.ctr[E.nx + E.ny + sz];
    const double ex = E.ctr[x] - px, ey = E.ctr[E.nx + y] - py, ez = E.ctr[E.nx + E.ny + z] - pz;
    const double n = sqrt(sum3(ex * ex, ey * ey, ez * ez));
    const int vx = voxel_index(px + E.ve * (ex / n), T.voxel) - 8 * E.dlo[0];
    const int vy = voxel_index(py + E.ve * (ey / n), T.voxel) - 8 * E.dlo[1];
    const int vz = voxel_index(pz + E.ve * (ez / n), T.voxel) - 8 * E.dlo[2];
    const int pool = dir_lookup(E, vx, vy, vz);
    if (pool >= 0) {
      const uint32_t g = pair_bits(T, pool, kDigestGeom, local_index(vx, vy, vz));
      if (g & 1u) return (g & 2u) != 0;
    }
    return own;
  }
};

// ---- phases 2 and 3: banded lower-envelope sweeps (esdf.hpp:236-280), see edt_core.cuh ----
__device__ __forceinline__ edt::RowTile carve_tile(unsigned char* base, int n, int band, int bands, size_t in_bytes) {
  edt::RowTile T;
  unsigned char* p = base + in_bytes;
  T.stk_s = reinterpret_cast<uint16_t*>(p), p += static_cast<size_t>(n) * 64;
  T.stk_t = reinterpret_cast<uint16_t*>(p), p += static_cast<size_t>(n) * 64;
  T.lo = reinterpret_cast<uint16_t*>(p), p += static_cast<size_t>(bands) * 64;
  T.hi = reinterpret_cast<uint16_t*>(p);
  T.n = n, T.band = band, T.bands = bands;
  return T;
}
static size_t sweep_smem_bytes(int n, int bands, int in_elem_bytes) {
  return static_cast<size_t>(n) * 32 * in_elem_bytes + static_cast<size_t>(n) * 64 * 2 + static_cast<size_t>(bands) * 64 * 2;
}

struct SrcY {  // candidate at y = the column's nearest seed z (phase-1 output)
  const uint16_t* zs;
  int z;
  __device__ __forceinline__ int r2(int pos, int row) const {
    const uint16_t v = zs[edt::at(pos, row)];
    if (v == edt::kNone) return -1;
    const int d = z - static_cast<int>(v);
    return d * d;
  }
};
struct SrcX {  // candidate at x = phase 2's (site_y, site_z)
  const uint32_t* yz;
  int y0, z;
  __device__ __forceinline__ int r2(int pos, int row) const {
    const uint32_t v = yz[edt::at(pos, row)];
    if (v == kYzNone) return -1;
    const int dy = (y0 + row) - static_cast<int>(v & 0xFFFFu);
    const int dz = z - static_cast<int>(v >> 16);
    return dy * dy + dz * dz;
  }
};

template <class Src>
__device__ __forceinline__ void sweep_stages(const edt::RowTile& T, const Src& src, int warp, int lane) {
  if (warp < T.bands) edt::build_band(T, src, warp, lane);
  __syncthreads();
  for (int j = 0; (1 << j) < T.bands; ++j) {
    if (warp < T.bands && (warp & ((2 << j) - 1)) == 0) edt::merge_groups(T, src, warp, j, lane);
    __syncthreads();
  }
}

// grid = (ceil(nx/32), nz); block = 32 * bands.  lane <-> x, positions = y.
__global__ void k_sweep_y(EsdfView E, int band, int bands) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char s_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int x = blockIdx.x * 32 + lane, z = blockIdx.y;
  const int ny = E.ny;
  uint16_t* zs = reinterpret_cast<uint16_t*>(s_raw);
  const edt::RowTile T = carve_tile(s_raw, ny, band, bands, static_cast<size_t>(ny) * 64);
  const int zoff = E.nx * ny * z + x;
  const int base = warp * band, end = min(base + band, ny);
  if (warp < bands)
    for (int y = base; y < end; ++y) zs[edt::at(y, lane)] = x < E.nx ? E.near_z[zoff + E.nx * y] : edt::kNone;
  __syncwarp();
  const SrcY src{zs, z};
  sweep_stages(T, src, warp, lane);
  if (warp < bands) {
    uint16_t last = edt::kNone;
    uint32_t packed = kYzNone;
    edt::colour_band(T, warp, lane, [&](int y, uint16_t win) {
      if (win != last) {
        last = win;
        packed = win == edt::kNone ? kYzNone : (static_cast<uint32_t>(win) | static_cast<uint32_t>(zs[edt::at(win, lane)]) << 16);
      }
      if (x < E.nx) E.yz[zoff + E.nx * y] = packed;
    });
  }
}

// grid = (ceil(ny/32), nz); block = 32 * bands.  lane <-> y, positions = x.
// The x-fastest input tile is loaded coalesced and turned into the [x][lane] layout with a
// bank rotation (write at bank (row + x) & 31, then rotate each 32-word group in place).
// kSigns: 0 = unsigned field (propagate), 1 = recover_signs fused into the store of the finished cell,
// 2 = the same using the hint planes left by the bit-packed gather of this build.
template <int kSigns>
__global__ void __launch_bounds__(512, 2) k_sweep_x(EsdfView E, TsdfView Tw, int band, int bands) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char s_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int y0 = blockIdx.x * 32, z = blockIdx.y;
  const int nx = E.nx, ny = E.ny;
  uint32_t* in = reinterpret_cast<uint32_t*>(s_raw);
  const edt::RowTile T = carve_tile(s_raw, nx, band, bands, static_cast<size_t>(nx) * 128);
  const int zoff = nx * ny * z;
  for (int r = warp; r < 32; r += nwarps) {
    const bool live = y0 + r < ny;
    const uint32_t* row = E.yz + zoff + nx * (y0 + r);
    for (int x = lane; x < nx; x += 32) in[x * 32 + ((r + x) & 31)] = live ? row[x] : kYzNone;
  }
  __syncthreads();
  for (int x = warp; x < nx; x += nwarps) {
    const uint32_t v = in[x * 32 + ((lane + x) & 31)];
    __syncwarp();
    in[x * 32 + lane] = v;
  }
  __syncthreads();
  const SrcX src{in, y0, z};
  sweep_stages(T, src, warp, lane);
  const int y = y0 + lane;
  if (warp < bands && y < ny) {
    SignProbe probe(E, Tw, kSigns ? y : 0, kSigns ? z : 0);
    const int obase = y + ny * nx * z;
    uint16_t last = edt::kNone;
    uint32_t site = kSiteNone;
    int r2w = 0, sx = 0;
    edt::colour_band(T, warp, lane, [&](int x, uint16_t win) {
      const int o = obase + ny * x;
      if (win == edt::kNone) {
        E.field[o] = make_uint2(kSiteNone, kD2None);
        return;
      }
      if (win != last) {  // everything that only depends on the winning site
        last = win;
        const uint32_t v = in[edt::at(win, lane)];
        const int sy = static_cast<int>(v & 0xFFFFu), sz = static_cast<int>(v >> 16);
        sx = win;
        r2w = (y - sy) * (y - sy) + (z - sz) * (z - sz);
        site = static_cast<uint32_t>(sx) | static_cast<uint32_t>(sy) << 10 | static_cast<uint32_t>(sz) << 20;
        if (kSigns) probe.template set_site<kSigns == 2>(sx, sy, sz);
      }
      uint32_t d2 = static_cast<uint32_t>((x - sx) * (x - sx) + r2w);
      if (kSigns && probe.template negative<kSigns == 2>(x)) d2 |= 0x80000000u;
      E.field[o] = make_uint2(site, d2);
    });
  }
}

// ---- phases 2 and 3 by monotone divide and conquer (edt_dc.cuh); used whenever the keys fit 32 bits ----
// One CTA per tile of 32 rows, 2^warps_log2 warps.  G = packed candidates [position][32 rows].
// Top levels (visits at the multiples of the stretch length 2^kTopShift): fewer visits than warps, so the windows are cut into
// slices whose minima meet in Kt through atomicMin, one barrier per level.  Below them every warp
// resolves whole stretches of that many positions on its own (edt_dc::stretch), no barrier.
using KeysY = edt_dc::Keys<1>;  // payload bit: the column's seed lies above z (k_sweep_y_dc<2> adds "site has a sign table")
using KeysX = edt_dc::Keys<0>;
// stretch length per sweep (measured, cfg2): 16 positions along y, 8 along x
constexpr int kTopShiftY = 4, kTopShiftX = 3;
// The 32 rows of a tile are 8 neighbours along the fast axis x 4 along z: all lanes scan as far as the
// lane with the longest window, and compact tiles cross a Voronoi boundary at fewer positions than
// 32 x 1 ones (29 % fewer evaluations at cfg2); 8 x 4 also divides the BASELINE grids without padding.
constexpr int kTileA = 8, kTileZ = 4;

template <int kPay, int kTopShift>
__device__ __forceinline__ void dc_top_levels(const uint32_t* G, uint32_t* Kt, int n, int warp, int lane, int nwarps, int warps_log2) {
  constexpr int kTopStep = 1 << kTopShift;
  const edt_dc::Plan plan = edt_dc::make_plan(n);
  for (int level = 0; level < plan.levels; ++level) {
    const int s = edt_dc::level_step(plan, level);
    if (s < kTopStep) break;
    const int parts_log2 = warps_log2 > level ? warps_log2 - level : 0;
    const int items = edt_dc::level_visits(plan, level) << parts_log2;
    for (int item = warp; item < items; item += nwarps) {
      const int tp = s * (2 * (item >> parts_log2) + 1);
      int lo, len;
      edt_dc::top_window<kPay>(Kt, n, kTopShift, tp, s, item & ((1 << parts_log2) - 1), parts_log2, lane, lo, len);
      const int longest = __reduce_max_sync(0xFFFFFFFFu, len);
      if (longest <= 0) continue;
      const uint32_t key = edt_dc::scan<kPay>(G, edt_dc::clamp_start(lo, longest, n), longest, tp - 1, lane);
      if (parts_log2 != 0) atomicMin(Kt + edt_dc::at(tp >> kTopShift, lane), key);
      else Kt[edt_dc::at(tp >> kTopShift, lane)] = key;
    }
    __syncthreads();
  }
}

// stretch j = positions t' in (j << kTopShift, (j+1) << kTopShift]; the sink gets each of them once, with its index
// inside the stretch as a compile-time constant (edt_dc::KeySink keeps them in registers)
template <int kPay, int kTopShift, class Sink>
__device__ __forceinline__ void dc_stretch_into(const uint32_t* G, const uint32_t* Kt, int n, int j, int lane, Sink& sink) {
  constexpr int kTopStep = 1 << kTopShift;
  const int a = j << kTopShift;
  const bool closed = a + kTopStep <= n;
  const uint32_t right = closed ? Kt[edt_dc::at(j + 1, lane)] : 0u;
  const int lo_w = a > 0 ? edt_dc::Keys<kPay>::winner(Kt[edt_dc::at(j, lane)]) : 0;
  const int hi_w = closed ? edt_dc::Keys<kPay>::winner(right) : n - 1;
  edt_dc::stretch_into<kPay, kTopStep - 1, 0>(G, n, a, lo_w, hi_w, lane, [](int v) { return __reduce_max_sync(0xFFFFFFFFu, v); }, sink);
  if (closed) sink.template put<kTopStep - 1>(a + kTopStep - 1, right);
}

static size_t dc_top_bytes(int n, int top_shift) { return static_cast<size_t>((n >> top_shift) + 1) * 32 * sizeof(uint32_t); }
static size_t dc_smem_bytes_y(int n) { return static_cast<size_t>(n) * 32 * sizeof(uint32_t) + dc_top_bytes(n, kTopShiftY); }
static size_t dc_smem_bytes_x(int n, int total, bool with_h = true) {  // G (u32), H (u16, kPX = 0), Kt and the per-axis fraction table of the sign tables
  return static_cast<size_t>(n) * 32 * (sizeof(uint32_t) + (with_h ? sizeof(uint16_t) : 0)) + dc_top_bytes(n, kTopShiftX) + static_cast<size_t>(total) * sizeof(float);
}

// root of a perfect square below 2^24 (one MUFU; its error of a few ulp cannot reach the next integer)
__device__ __forceinline__ int exact_root(int sq) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(static_cast<float>(sq)));
  return __float2int_rn(r);
}

// grid = (ceil(nx/8), ceil(nz/4)); lane <-> (x, z), positions = y.  kPay = 2: key payload = {seed above z, site has a
// sign table}; kPay = 1 (grids whose y keys have no room for the second bit): {seed above z}, every site counts as
// having a table.  Output = phase 3's candidates ALREADY in the layout of the x sweep's shared-memory tile (gimg /
// himg): a lane's 8 consecutive y of one x-sweep tile are 8 consecutive words, so a stretch of 16 positions leaves as
// four 16-byte stores of candidates + two of payload, and the x sweep fills its tile with two bulk copies.
constexpr int kLoadBatch = 8;
template <int kPay, int kPX>
__global__ void __launch_bounds__(512) k_sweep_y_dc(EsdfView E, int warps_log2, uint32_t none_y, uint32_t none_x) {
  pdl_enter();
  using KY = edt_dc::Keys<kPay>;
  using KX = edt_dc::Keys<kPX>;  // kPX = 1: phase 3's candidate carries "site has a sign table" below its position
  extern __shared__ __align__(16) unsigned char s_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;  // any warp count; windows are cut into 2^warps_log2 slices
  const int x = blockIdx.x * kTileA + (lane & (kTileA - 1)), z = blockIdx.y * kTileZ + lane / kTileA;
  const int ny = E.ny, nx = E.nx;
  uint32_t* G = reinterpret_cast<uint32_t*>(s_raw);
  uint32_t* Kt = G + ny * 32;
  const bool live = x < nx && z < E.nz;
  {  // candidates: the nearest seed along z of every column (esdf.hpp:213-233; ties keep the lower z, strict '<' :229)
    const int zc = min(z, E.nz - 1);
    const int col = (zc >> 5) * nx + min(x, nx - 1), stride = E.nzw * nx;
    const int zb = zc & 31;
    for (int yb = warp * kLoadBatch; yb < ny; yb += nwarps * kLoadBatch) {
      uint32_t wd[kLoadBatch], inf[kLoadBatch], tb[kLoadBatch];
#pragma unroll
      for (int i = 0; i < kLoadBatch; ++i) {
        const int o = col + stride * min(yb + i, ny - 1);
        wd[i] = __ldg(E.zbits + o), inf[i] = __ldg(E.zinfo + o);
        if constexpr (kPay == 2) tb[i] = __ldg(E.zgbits + o);
      }
#pragma unroll
      for (int i = 0; i < kLoadBatch; ++i) {
        const int y = yb + i;
        // distance to the nearest seed at or below z / at or above z: inside the word by a bit scan, else the word's info
        const uint32_t t_lo = wd[i] << (31 - zb), t_hi = wd[i] >> zb;  // bit z at position 31 / 0
        const int db = t_lo ? __clz(static_cast<int>(t_lo)) : zb + static_cast<int>(inf[i] & 0x7FFFu);
        const int da = t_hi ? __ffs(static_cast<int>(t_hi)) - 1 : (31 - zb) + static_cast<int>((inf[i] >> 16) & 0x7FFFu);
        const bool up = da < db;  // a tie keeps the lower z (strict '<', esdf.hpp:229); up implies dz > 0
        const int dz = up ? da : db;
        uint32_t pay = up ? 1u : 0u;
        if constexpr (kPay == 2) {
          const bool inword = up ? t_hi != 0 : t_lo != 0;
          const int pos = up ? zb + da : zb - db;  // the chosen seed's bit inside the word (meaningless when it lies outside)
          const uint32_t flag = inword ? (tb[i] >> (pos & 31)) & 1u : (up ? inf[i] >> 31 : (inf[i] >> 15) & 1u);
          pay = pay << 1 | flag;
        }
        const uint32_t g = (dz >= static_cast<int>(kZNone) || !live) ? KY::pack(none_y, y, 0) : KY::pack(static_cast<uint32_t>(dz * dz), y, pay);
        if (y < ny) G[edt_dc::at(y, lane)] = g;
      }
    }
  }
  for (int i = warp; i <= ny >> kTopShiftY; i += nwarps) Kt[edt_dc::at(i, lane)] = 0xFFFFFFFFu;
  __syncthreads();
  dc_top_levels<kPay, kTopShiftY>(G, Kt, ny, warp, lane, nwarps, warps_log2);
  // tile images: tile (yt, zt = blockIdx.y), position x, row (y & 7) + 8 (z & 3) = yy + 8 zz
  const size_t zt_base = static_cast<size_t>(blockIdx.y) * E.nyt;
  const int zz = lane / kTileA;
  for (int j = warp; (j << kTopShiftY) < ny; j += nwarps) {
    edt_dc::KeySink<16> keys;
#pragma unroll
    for (int i = 0; i < 16; ++i) keys.k[i] = 0xFFFFFFFFu;
    dc_stretch_into<kPay, kTopShiftY>(G, Kt, ny, j, lane, keys);
    if (x >= nx) continue;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int yt = 2 * j + h;
      if (yt >= E.nyt) break;
      uint32_t gw[8], hw[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t k = keys.k[8 * h + i];
        const uint32_t c = KY::cost(k);
        const bool none = c >= none_y;
        const uint32_t low = k & KY::kLowMask;  // site_y and the payload
        gw[i] = none ? KX::pack(none_x, x, 0) : KX::pack(c, x, kPX ? (kPay == 2 ? (low & 1u) : 1u) : 0u);
        hw[i] = none ? 0u : (kPay == 2 ? low : (low << 1 | 1u));
      }
      const size_t at = ((zt_base + yt) * nx + x) * 32 + 8 * zz;
      uint4* gp = reinterpret_cast<uint4*>(E.gimg + at);
      gp[0] = make_uint4(gw[0], gw[1], gw[2], gw[3]);
      gp[1] = make_uint4(gw[4], gw[5], gw[6], gw[7]);
      *reinterpret_cast<uint4*>(E.himg + at) = make_uint4(hw[0] | hw[1] << 16, hw[2] | hw[3] << 16, hw[4] | hw[5] << 16, hw[6] | hw[7] << 16);
    }
  }
}

// ---- bulk asynchronous copies (cp.async.bulk, completion on an mbarrier): one thread moves a whole tile ----
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, int arrivals) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(arrivals));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "KS_MBAR_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@p bra KS_MBAR_DONE;\n\t"
      "bra KS_MBAR_WAIT;\n\t"
      "KS_MBAR_DONE:\n\t}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// site_y, site_z of the winner `u` of row (y, z) from a tile image word pair (gimg / himg or their shared-memory copies)
template <int kPX>
__device__ __forceinline__ void decode_site(uint32_t gword, uint32_t hword, int y, int z, int& sy, int& sz) {
  const int r2 = static_cast<int>(edt_dc::Keys<kPX>::cost(gword));
  sy = static_cast<int>(hword >> 2);
  const int dy = y - sy;
  const int dz = exact_root(r2 - dy * dy);
  sz = (hword & 2u) ? z + dz : z - dz;
}

// grid = (ceil(ny/8), ceil(nz/4)); lane <-> (y, z), positions = x.  kSigns: 0 = unsigned field (propagate), 1 / 2 =
// recover_signs per cell from the directory (without / with the hint planes), 3 = from the per-site tables of the
// resampled seeding.  The tile (candidates G, payload H) arrives by two bulk copies issued by one thread.  A warp
// resolves a stretch of 8 positions with its 8 winning keys in registers; a key IS the field word (d2 << 10 | site_x).
// Mode 3: a cell whose site has no sign table takes its own-sign bit and needs nothing else -- no site decode, no
// table fetch; only cells whose site lies next to stamped geometry go through the probe.  One lane stores its 8
// cells with two 16-byte stores (x-fastest field).
// kBig: rows so long that only one tile fits an SM -- then the tile gets 32 warps instead of 16
// kPX = 1 (whenever the keys have a spare bit): the candidate word itself says whether its site has a sign table, so the
// payload image H is not staged at all -- the tile is G alone (a third less shared memory: three tiles per SM at
// cfg2 instead of two), a position costs no H lookup, and only the few cells next to stamped geometry fetch their
// site's payload word from the image in L2.
template <int kSigns, bool kBig, int kPX>
__global__ void __launch_bounds__(kBig ? 1024 : 512, kBig ? 1 : 2) k_sweep_x_dc(EsdfView E, TsdfView Tw, int warps_log2, uint32_t none_x) {
  using KX = edt_dc::Keys<kPX>;
  pdl_wait();
  extern __shared__ __align__(128) unsigned char s_raw[];
  __shared__ __align__(8) uint64_t s_bar;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int y0 = blockIdx.x * kTileA, z0 = blockIdx.y * kTileZ;
  const int nx = E.nx, ny = E.ny;
  uint32_t* G = reinterpret_cast<uint32_t*>(s_raw);
  uint16_t* H = reinterpret_cast<uint16_t*>(G + nx * 32);  // kPX = 0 only
  uint32_t* Kt = kPX ? G + nx * 32 : reinterpret_cast<uint32_t*>(H + nx * 32);
  constexpr int kTopShift = kTopShiftX, kTopStep = 1 << kTopShift;
  float* s_qsf = reinterpret_cast<float*>(Kt + ((nx >> kTopShift) + 1) * 32);
  if (threadIdx.x == 0) mbar_init(&s_bar, 1);
  __syncthreads();
  const size_t tile = static_cast<size_t>(blockIdx.y) * E.nyt + blockIdx.x;
  const uint16_t* Hsrc = kPX ? E.himg + tile * nx * 32 : H;  // where a slow cell reads its site's payload word
  if (threadIdx.x == 0) {
    const uint32_t gbytes = static_cast<uint32_t>(nx) * 32u * 4u, hbytes = kPX ? 0u : static_cast<uint32_t>(nx) * 32u * 2u;
    mbar_expect_tx(&s_bar, gbytes + hbytes);
    bulk_g2s(G, E.gimg + tile * nx * 32, gbytes, &s_bar);
    if (!kPX) bulk_g2s(H, E.himg + tile * nx * 32, hbytes, &s_bar);
  }
  for (int i = warp; i <= nx >> kTopShift; i += nwarps) Kt[edt_dc::at(i, lane)] = 0xFFFFFFFFu;
  if constexpr (kSigns == 3)
    if (!E.iprobe)  // the fp32 probe's per-axis fractions; the integer probe needs none
      for (int i = threadIdx.x; i < nx + ny + E.nz; i += blockDim.x) s_qsf[i] = E.qsf[i];
  const int back = 1 - E.ctrl->front;
  mbar_wait(&s_bar, 0);
  __syncthreads();
  dc_top_levels<kPX, kTopShift>(G, Kt, nx, warp, lane, nwarps, warps_log2);
  const int y = min(y0 + (lane & (kTileA - 1)), ny - 1), z = min(z0 + lane / kTileA, E.nz - 1);
  const bool live = y0 + (lane & (kTileA - 1)) < ny && z0 + lane / kTileA < E.nz;
  auto make_probe = [&]() {
    if constexpr (kSigns == 3) return SignTable(E, Tw, s_qsf, y, z);
    else return SignProbe(E, Tw, kSigns ? y : 0, kSigns ? z : 0);
  };
  auto probe = make_probe();
  const uint32_t* orow = E.obits + ((z + 1) * (ny + 2) + (y + 1)) * E.wpr2;
  uint32_t* out_row = (back ? E.f32[1] : E.f32[0]) + (static_cast<size_t>(z) * ny + y) * nx;
  const bool vec_ok = (nx & 3) == 0;
  for (int j = warp; (j << kTopShift) < nx; j += nwarps) {
    const int x0 = j << kTopShift;
    uint32_t own_lo = 0, own_hi = 0;  // requested before the stretch is resolved, so that the loads ride under it
    if constexpr (kSigns == 3) own_lo = __ldg(orow + (x0 >> 5)), own_hi = (x0 >> 5) + 1 < E.wpr2 ? __ldg(orow + (x0 >> 5) + 1) : 0u;
    edt_dc::KeySink<8> keys;
#pragma unroll
    for (int i = 0; i < 8; ++i) keys.k[i] = 0xFFFFFFFFu;
    dc_stretch_into<kPX, kTopShift>(G, Kt, nx, j, lane, keys);
    if (!live) continue;
    uint32_t w[8];
    uint32_t slow = 0;  // positions that need the site: bit i
    uint32_t own = 0;   // own-sign bits of cells x0 .. x0 + 7 (extended bits x0 + 1 ..)
    if constexpr (kSigns == 3) {
      own = __funnelshift_rc(own_lo, own_hi, (x0 & 31) + 1);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t k = keys.k[i];
        const bool none = KX::cost(k) >= none_x;  // the grid holds no seed at all
        uint32_t table;  // the winner's site has a sign table
        if constexpr (kPX) table = k & 1u;
        else table = H[edt_dc::at(none ? 0 : KX::winner(k), lane)] & 1u;  // (a position beyond the row carries key ~0)
        w[i] = none ? 0xFFFFFFFFu : ((k >> kPX) | ((own >> i) & 1u) << 31);
        slow |= (none ? 0u : table) << i;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const bool none = KX::cost(keys.k[i]) >= none_x;
        w[i] = none ? 0xFFFFFFFFu : keys.k[i] >> kPX;
        if (kSigns != 0 && !none) slow |= 1u << i;
      }
    }
    if (slow != 0) {  // cells whose site may resolve a geometry probe: the reference's decision from the site's table / the directory
      // the eight winners, 10 bits each, in three registers (a run-time index into keys.k would put it in local memory)
      const uint32_t p0 = (w[0] & 1023u) | (w[1] & 1023u) << 10 | (w[2] & 1023u) << 20;
      const uint32_t p1 = (w[3] & 1023u) | (w[4] & 1023u) << 10 | (w[5] & 1023u) << 20;
      const uint32_t p2 = (w[6] & 1023u) | (w[7] & 1023u) << 10;
      uint32_t flip = 0;
      int last = -1;
      for (uint32_t m = slow; m != 0; m &= m - 1) {
        const int i = __ffs(static_cast<int>(m)) - 1;
        const int x = x0 + i;
        const int q = (i * 11) >> 5;  // i / 3
        const int u = static_cast<int>(((q == 0 ? p0 : (q == 1 ? p1 : p2)) >> (10 * (i - 3 * q))) & 1023u);
        if (u != last) {
          last = u;
          int sy, sz;
          const uint32_t hword = kPX ? __ldg(Hsrc + edt_dc::at(u, lane)) : Hsrc[edt_dc::at(u, lane)];
          decode_site<kPX>(G[edt_dc::at(u, lane)], hword, y, z, sy, sz);
          if constexpr (kSigns == 3) probe.set_site(u, sy, sz, __ldg(E.gtab + (u + nx * (sy + ny * sz))));
          else if constexpr (kSigns != 0) probe.template set_site<kSigns == 2>(u, sy, sz);
        }
        bool neg = false;
        if constexpr (kSigns == 3) {
          const bool mine = ((own >> i) & 1u) != 0;
          neg = probe.negative(x, mine) != mine;  // flip when the probe disagrees with the own-sign default
        } else if constexpr (kSigns != 0) {
          neg = probe.template negative<kSigns == 2>(x);
        }
        flip |= (neg ? 1u : 0u) << i;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) w[i] ^= ((flip >> i) & 1u) << 31;
    }
    uint32_t* out = out_row + x0;
    if (vec_ok && x0 + 8 <= nx) {
      reinterpret_cast<uint4*>(out)[0] = make_uint4(w[0], w[1], w[2], w[3]);
      reinterpret_cast<uint4*>(out)[1] = make_uint4(w[4], w[5], w[6], w[7]);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (x0 + i < nx) out[i] = w[i];
    }
  }
  // publish: the last CTA to finish makes this buffer the one readers use
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&E.ctrl->x_done, 1u) == gridDim.x * gridDim.y - 1) {
      E.ctrl->x_done = 0;
      E.ctrl->pub_seeds = E.ctrl->seed_count;
      if (kSigns != 0) E.ctrl->signs_recovered = 1;
      __threadfence();
      E.ctrl->front = back;
    }
  }
}

// ---- readers of the finished field ----
__device__ __forceinline__ const uint32_t* front_field(const EsdfView& E) {  // fast path: the published buffer
  return E.ctrl->front ? E.f32[1] : E.f32[0];
}
// fast path: site of cell (x, y, z) whose field word is w -- site_x from the word, site_y / site_z from phase 2's
// winner at (site_x, y, z) in the tile images
__device__ __forceinline__ void fast_site(const EsdfView& E, uint32_t w, int y, int z, int& sx, int& sy, int& sz) {
  sx = static_cast<int>(w & 1023u);
  const size_t at = ((static_cast<size_t>(z >> 2) * E.nyt + (y >> 3)) * E.nx + sx) * 32 + (y & 7) + 8 * (z & 3);
  if (E.xpay) decode_site<1>(E.gimg[at], E.himg[at], y, z, sy, sz);
  else decode_site<0>(E.gimg[at], E.himg[at], y, z, sy, sz);
}

// ---- recover_signs as its own pass (esdf.hpp:288-320), for the stage-by-stage API (no hints) ----
__global__ void __launch_bounds__(256) k_recover_signs(EsdfView E, TsdfView T) {
  pdl_wait();
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= E.cells) return;
  if (E.fast) {  // o is x-fastest
    if (E.ctrl->pub_seeds == 0) return;
    uint32_t* f = const_cast<uint32_t*>(front_field(E));
    const int x = o % E.nx, y = (o / E.nx) % E.ny, z = o / (E.nx * E.ny);
    int sx, sy, sz;
    fast_site(E, f[o], y, z, sx, sy, sz);
    SignProbe probe(E, T, y, z);
    probe.template set_site<false>(sx, sy, sz);
    if (probe.template negative<false>(x)) f[o] ^= 0x80000000u;
    return;
  }
  const uint32_t site = E.field[o].x;
  if (site == kSiteNone) return;
  const int y = o % E.ny;
  const int x = (o / E.ny) % E.nx;
  const int z = o / (E.ny * E.nx);
  SignProbe probe(E, T, y, z);
  probe.template set_site<false>(site & 1023, (site >> 10) & 1023, site >> 20);
  if (probe.template negative<false>(x)) E.field[o].y ^= 0x80000000u;
}

// the wide path's sweeps do not publish by themselves
__global__ void k_publish(EsdfView E) {
  pdl_wait();
  if (threadIdx.x == 0 && blockIdx.x == 0) E.ctrl->pub_seeds = E.ctrl->seed_count;
}

// ---- query (esdf.hpp:337-387) ----
// f: the published fast-path buffer, or nullptr on the wide path
__device__ __forceinline__ double cell_distance(const EsdfView& E, const uint32_t* f, int x, int y, int z) {
  uint32_t d2, neg;
  if (f != nullptr) {
    const uint32_t w = f[x + static_cast<long long>(E.nx) * (y + static_cast<long long>(E.ny) * z)];
    d2 = (w >> 10) & 0x1FFFFFu, neg = w >> 31;
  } else {
    const uint32_t v = E.field[y + static_cast<long long>(E.ny) * (x + static_cast<long long>(E.nx) * z)].y;
    d2 = v & 0x7FFFFFFFu, neg = v >> 31;
  }
  const double d = sqrt(static_cast<double>(d2)) * E.ve;  // esdf.hpp:276-277
  return neg ? -d : d;
}
// One point: distance, gradient (may be null), inside flag.
__device__ __forceinline__ void query_point(const EsdfView& E, const double p[3], double& dist, double grad[3], bool& in) {
  const int dims[3] = {E.nx, E.ny, E.nz};
  in = true;
#pragma unroll
  for (int a = 0; a < 3; ++a) in = in && p[a] >= E.origin[a] && p[a] <= E.origin[a] + dims[a] * E.ve;
  dist = CUDART_INF;
  grad[0] = grad[1] = grad[2] = 0.0;
  if (E.ctrl->pub_seeds == 0) return;  // no sites: +inf, zero gradient (esdf.hpp:345)
  const uint32_t* fld = E.fast ? front_field(E) : nullptr;
  int i0[3], i1[3];
  double f[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (dims[a] == 1) {
      i0[a] = i1[a] = 0;
      f[a] = 0.0;
      continue;
    }
    const double s = (p[a] - E.origin[a]) / E.ve - 0.5;
    const double hi = static_cast<double>(dims[a] - 1);
    const double c = s < 0.0 ? 0.0 : (hi < s ? hi : s);  // std::clamp
    const int ic = static_cast<int>(c);
    i0[a] = ic < dims[a] - 2 ? ic : dims[a] - 2;
    i1[a] = i0[a] + 1;
    f[a] = c - i0[a];
  }
  const double c000 = cell_distance(E, fld, i0[0], i0[1], i0[2]), c100 = cell_distance(E, fld, i1[0], i0[1], i0[2]);
  const double c010 = cell_distance(E, fld, i0[0], i1[1], i0[2]), c110 = cell_distance(E, fld, i1[0], i1[1], i0[2]);
  const double c001 = cell_distance(E, fld, i0[0], i0[1], i1[2]), c101 = cell_distance(E, fld, i1[0], i0[1], i1[2]);
  const double c011 = cell_distance(E, fld, i0[0], i1[1], i1[2]), c111 = cell_distance(E, fld, i1[0], i1[1], i1[2]);
  const double fx = f[0], fy = f[1], fz = f[2];
  const double c00 = c000 * (1 - fx) + c100 * fx, c10 = c010 * (1 - fx) + c110 * fx;
  const double c01 = c001 * (1 - fx) + c101 * fx, c11 = c011 * (1 - fx) + c111 * fx;
  const double c0 = c00 * (1 - fy) + c10 * fy, c1 = c01 * (1 - fy) + c11 * fy;
  dist = c0 * (1 - fz) + c1 * fz;
  const double inv = 1.0 / E.ve;
  grad[0] = ((c100 - c000) * (1 - fy) * (1 - fz) + (c110 - c010) * fy * (1 - fz) + (c101 - c001) * (1 - fy) * fz +
             (c111 - c011) * fy * fz) *
            inv;
  grad[1] = ((c10 - c00) * (1 - fz) + (c11 - c01) * fz) * inv;
  grad[2] = (c1 - c0) * inv;
}

__global__ void __launch_bounds__(256) k_query(EsdfView E, const double* __restrict__ pts, long long n, double* __restrict__ dist,
                                               double* __restrict__ grad, uint8_t* __restrict__ inside) {
  pdl_wait();
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double p[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
  double d, g[3];
  bool in;
  query_point(E, p, d, g, in);
  dist[i] = d;
  if (inside) inside[i] = in;
  if (grad) grad[3 * i] = g[0], grad[3 * i + 1] = g[1], grad[3 * i + 2] = g[2];
}

// Per-environment summary for the multi-environment exchange: {tag, minimum distance over the
// probe points, number of probes closer than `near`, seed count} as four doubles, in one capturable launch.
// One probe per thread; the last CTA to finish folds the per-CTA partials (fixed order: deterministic).
constexpr int kSummaryCtas = 64;
struct SummaryScratch {
  double part_min[kSummaryCtas];
  int part_cnt[kSummaryCtas];
  unsigned arrivals;
};
__global__ void __launch_bounds__(128) k_probe_summary(EsdfView E, const double* __restrict__ pts, int n, double near, double tag,
                                                       SummaryScratch* scratch, double* __restrict__ out) {
  pdl_enter();
  __shared__ double s_min[4];
  __shared__ int s_cnt[4];
  __shared__ bool s_last;
  double best = CUDART_INF;
  int count = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double p[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    double d, g[3];
    bool in;
    query_point(E, p, d, g, in);
    best = d < best ? d : best;
    count += d < near;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double other = __shfl_down_sync(0xFFFFFFFFu, best, o);
    best = other < best ? other : best;
    count += __shfl_down_sync(0xFFFFFFFFu, count, o);
  }
  if ((threadIdx.x & 31) == 0) s_min[threadIdx.x >> 5] = best, s_cnt[threadIdx.x >> 5] = count;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 4; ++w) best = s_min[w] < best ? s_min[w] : best, count += s_cnt[w];
    scratch->part_min[blockIdx.x] = best, scratch->part_cnt[blockIdx.x] = count;
    __threadfence();
    s_last = atomicAdd(&scratch->arrivals, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    __threadfence();
    best = CUDART_INF, count = 0;
    for (unsigned b = 0; b < gridDim.x; ++b) {
      const double m = scratch->part_min[b];
      best = m < best ? m : best, count += scratch->part_cnt[b];
    }
    out[0] = tag, out[1] = best, out[2] = static_cast<double>(count), out[3] = static_cast<double>(E.ctrl->pub_seeds);
    scratch->arrivals = 0;  // ready for the next launch
  }
}

// ---- scene collision (collision.hpp:30-44, :130-239) ----
__device__ __forceinline__ double hinge_cost(double clearance, double margin) {  // collision.hpp:30-37
  if (clearance >= margin) return 0.0;
  if (clearance >= 0.0) {
    const double gap = margin - clearance;
    return gap * gap / (2.0 * margin);
  }
  return 0.5 * margin - clearance;
}
__device__ __forceinline__ double hinge_slope(double clearance, double margin) {  // collision.hpp:40-44
  if (clearance >= margin) return 0.0;
  if (clearance >= 0.0) return -(margin - clearance) / margin;
  return -1.0;
}

// scene_collision_static (collision.hpp:130-152): one thread per sphere -> penetration, cost, gradient
__global__ void __launch_bounds__(256) k_collision_static(EsdfView E, const double* __restrict__ centers,
                                                          const double* __restrict__ radii, int n, double margin,
                                                          double* __restrict__ pen, double* __restrict__ cost,
                                                          double* __restrict__ grad) {
  pdl_wait();
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const double p[3] = {centers[3 * s], centers[3 * s + 1], centers[3 * s + 2]};
  double d, g[3];
  bool in;
  query_point(E, p, d, g, in);
  const double clearance = d - radii[s];
  pen[s] = -clearance;
  const double c = hinge_cost(clearance, margin);
  cost[s] = c;
  double out[3] = {0.0, 0.0, 0.0};
  if (c > 0.0) {
    const double slope = hinge_slope(clearance, margin);
    for (int a = 0; a < 3; ++a) out[a] += slope * g[a];
  }
  if (grad) grad[3 * s] = out[0], grad[3 * s + 1] = out[1], grad[3 * s + 2] = out[2];
}

// scene_collision (collision.hpp:177-239): one thread per (timestep, sphere) walks its segment
__global__ void __launch_bounds__(128) k_collision_swept(EsdfView E, const double* __restrict__ centers,
                                                         const double* __restrict__ radii, const double* __restrict__ vel,
                                                         int timesteps, int spheres, double margin, double dt, int max_checks,
                                                         double* __restrict__ pen, double* __restrict__ cost,
                                                         double* __restrict__ g_center, double* __restrict__ g_next,
                                                         double* __restrict__ g_vel) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= timesteps * spheres) return;
  const int t = i / spheres, s = i % spheres;
  const bool has_next = t + 1 < timesteps;
  const size_t at = static_cast<size_t>(i) * 3;
  const double start[3] = {centers[at], centers[at + 1], centers[at + 2]};
  double seg[3] = {0.0, 0.0, 0.0};
  if (has_next) {
    const size_t nx = at + static_cast<size_t>(spheres) * 3;
    for (int a = 0; a < 3; ++a) seg[a] = centers[nx + a] - start[a];
  }
  const double length = sqrt(sum3(seg[0] * seg[0], seg[1] * seg[1], seg[2] * seg[2]));
  const double v[3] = {vel[at], vel[at + 1], vel[at + 2]};
  const double speed = sqrt(sum3(v[0] * v[0], v[1] * v[1], v[2] * v[2]));
  const double weight = speed * dt;
  const double radius = radii[s];
  double hinge_sum = 0.0, lambda = 0.0, max_pen = 0.0;
  double sg[3] = {0.0, 0.0, 0.0}, ng[3] = {0.0, 0.0, 0.0};
  for (int check = 0; check < max_checks; ++check) {
    const double frac = length > 0.0 ? lambda / length : 0.0;
    const double x[3] = {start[0] + frac * seg[0], start[1] + frac * seg[1], start[2] + frac * seg[2]};
    double d, g[3];
    bool in;
    query_point(E, x, d, g, in);
    const double clearance = d - radius;
    if (-clearance > max_pen) max_pen = -clearance;
    hinge_sum += hinge_cost(clearance, margin);
    const double slope = hinge_slope(clearance, margin);
    if (slope != 0.0) {
      for (int a = 0; a < 3; ++a) {
        const double gx = slope * g[a];
        sg[a] += (1.0 - frac) * gx;
        ng[a] += frac * gx;
      }
    }
    if (!has_next) break;
    lambda += clearance < E.ve ? E.ve : clearance;  // std::max(clearance, min_step)
    if (lambda >= length) break;
  }
  pen[i] = max_pen;
  cost[i] = weight * hinge_sum;
  for (int a = 0; a < 3; ++a) {
    g_center[at + a] = 0.0 + weight * sg[a];
    if (has_next) g_next[at + a] = 0.0 + weight * ng[a];
    g_vel[at + a] = speed > 1e-12 ? 0.0 + hinge_sum * dt * (v[a] / speed) : 0.0;
  }
}

// Per group of `width` entries: report {max penetration (>0, first index on ties, else 0 / -1), cost sum}.
// One CTA per group; the sum is a fixed-shape tree (deterministic; last-bit differences from the
// reference's left-to-right sum are covered by the 1e-12 relative tolerance stated in the tests).
__global__ void __launch_bounds__(256) k_collision_reduce(const double* __restrict__ pen, const double* __restrict__ cost, int width,
                                                          double* __restrict__ report3) {
  pdl_enter();
  __shared__ double s_pen[256], s_cost[256];
  __shared__ int s_idx[256];
  const int group = blockIdx.x, tid = threadIdx.x;
  const double* gp = pen + static_cast<size_t>(group) * width;
  const double* gc = cost + static_cast<size_t>(group) * width;
  double best = 0.0, total = 0.0;
  int best_i = -1;
  for (int i = tid; i < width; i += blockDim.x) {
    if (gp[i] > best) best = gp[i], best_i = i;  // strict: lowest index among this thread's equals
    total += gc[i];
  }
  s_pen[tid] = best, s_idx[tid] = best_i, s_cost[tid] = total;
  __syncthreads();
  for (int d = 128; d > 0; d >>= 1) {
    if (tid < d) {
      const double op = s_pen[tid + d];
      const int oi = s_idx[tid + d];
      if (oi >= 0 && (op > s_pen[tid] || (op == s_pen[tid] && (s_idx[tid] < 0 || oi < s_idx[tid])))) s_pen[tid] = op, s_idx[tid] = oi;
      s_cost[tid] += s_cost[tid + d];
    }
    __syncthreads();
  }
  if (tid == 0) {
    report3[3 * group] = s_pen[0];
    report3[3 * group + 1] = s_idx[0];
    report3[3 * group + 2] = s_cost[0];
  }
}

// ---- export to the reference's DenseEsdf arrays (x-fastest; esdf.hpp:58-64) ----
__global__ void __launch_bounds__(256) k_export(EsdfView E, int* __restrict__ site_xyz, double* __restrict__ distance,
                                                int* __restrict__ d2) {
  pdl_wait();
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= E.cells) return;
  const int x = static_cast<int>(idx % E.nx);
  const int y = static_cast<int>((idx / E.nx) % E.ny);
  const int z = static_cast<int>(idx / (static_cast<long long>(E.nx) * E.ny));
  uint32_t s, v;
  if (E.fast) {
    if (E.ctrl->pub_seeds == 0) {
      s = kSiteNone, v = kD2None;
    } else {
      const uint32_t w = front_field(E)[idx];
      int sx, sy, sz;
      fast_site(E, w, y, z, sx, sy, sz);
      s = static_cast<uint32_t>(sx) | static_cast<uint32_t>(sy) << 10 | static_cast<uint32_t>(sz) << 20;
      v = ((w >> 10) & 0x1FFFFFu) | (w & 0x80000000u);
    }
  } else {
    const long long o = y + static_cast<long long>(E.ny) * (x + static_cast<long long>(E.nx) * z);
    const uint2 cell = E.field[o];
    s = cell.x, v = cell.y;
  }
  if (site_xyz) {
    site_xyz[3 * idx] = s == kSiteNone ? -1 : static_cast<int>(s & 1023);
    site_xyz[3 * idx + 1] = s == kSiteNone ? -1 : static_cast<int>((s >> 10) & 1023);
    site_xyz[3 * idx + 2] = s == kSiteNone ? -1 : static_cast<int>(s >> 20);
  }
  if (distance) {
    double d = CUDART_INF;
    if (s != kSiteNone) {
      d = sqrt(static_cast<double>(v & 0x7FFFFFFFu)) * E.ve;
      if (v & 0x80000000u) d = -d;
    }
    distance[idx] = d;
  }
  if (d2) d2[idx] = s == kSiteNone ? 0x7FFFFFFF : static_cast<int>(v & 0x7FFFFFFFu);
}

}  // namespace ksb

using namespace ksb;

struct ks_esdf {
  ks_esdf_config cfg;
  EsdfView view;
  cudaStream_t stream;
  bool own_stream;
  cudaEvent_t dep;
  // the site tables are only read by the last sweep: they are built on a side stream while phase 1 and 2 run
  cudaStream_t side;
  cudaEvent_t fork, join;
  bool side_pending;
  void* query_scratch;   // device scratch of the host-pointer entry points (call_scratch), grown on demand
  int64_t query_cap;     // doubles it holds
  std::mutex query_mu;   // query() is safe to call concurrently: callers share the scratch one at a time
  bool counters_reset;  // k_dir_clear of the build being enqueued zeroed the seeding counters (no memset needed)
  EsdfCtrl* h_ctrl;  // pinned
  double bound_voxel;  // TSDF voxel size the tables/directory were built for (0 = none)
  int bound_capacity;  // TSDF pool capacity pool_surf was sized for
  std::atomic<uint64_t> generation{0};  // bumped whenever a call that rewrites the field is enqueued
  int band_y, bands_y, band_x, bands_x;
  size_t smem_y, smem_x;
  SummaryScratch* summary_scratch;  // partials of k_probe_summary
  // private graph of the fused build (ks_esdf_build_async outside a caller's capture)
  bool own_graphs;
  cudaGraphExec_t build_exec;
  uint64_t build_tsdf;  // tsdf_uid of the world the graph was recorded for
  double build_voxel;
  int64_t build_nodes;
  bool resample_ok;        // the dilation identity of the resampled seeding holds for the bound TSDF voxel size
  bool dc;                 // sweeps by divide and conquer (keys fit 32 bits), else the banded stacks
  bool resample_by_rows;   // KS_RESAMPLE=rows: the per-row resampling kernel even when the grids are in step
  int dc_wl_y, dc_wl_x;    // floor(log2(warps per tile)): slices a top-level window is cut into
  int dc_nw_y, dc_nw_x;    // warps per tile
  int pay_y;               // payload bits of the y keys: 2 = {seed above z, site has a sign table}, 1 = the first only
  uint32_t none_y, none_x; // offsets of positions without candidate
  int sticky_err;
  bool profile, profile_stages;
  cudaEvent_t ev[7];
};

namespace ksb {

static void pick_bands(int n, int& band, int& bands) {
  // 24 positions per band and at most 16 warps per tile measured best on B200 (tools/tune_bands.sh);
  // KS_BAND_TARGET / KS_MAX_WARPS override them for tuning runs only.
  int target = 24, max_warps = 16;
  if (const char* v = std::getenv("KS_BAND_TARGET")) target = std::max(2, std::atoi(v));
  if (const char* v = std::getenv("KS_MAX_WARPS")) max_warps = std::min(16, std::max(1, std::atoi(v)));
  int warps = std::min(max_warps, std::max(1, (n + target - 1) / target));
  band = (n + warps - 1) / warps;
  bands = (n + band - 1) / band;
}

static int bind_tsdf(ks_esdf* e, const ks_tsdf* t) {
  const TsdfView& T = tsdf_view(t);
  if (e->bound_voxel == T.voxel && T.capacity <= e->bound_capacity) return KS_OK;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(e->stream, &cap);
  if (cap != cudaStreamCaptureStatusNone)
    return fail(KS_ERR_INVALID, "esdf: build once against this TSDF before capturing a graph");
  EsdfView& E = e->view;
  KS_CUDA(cudaStreamSynchronize(e->stream));
  if (e->bound_voxel == T.voxel) {  // same geometry, a world with a larger pool: only the per-pool-entry flags grow
    if (E.pool_surf) cudaFree(E.pool_surf);
    E.pool_surf = nullptr;
    KS_CUDA(cudaMalloc(&E.pool_surf, static_cast<size_t>(T.capacity)));
    e->bound_capacity = T.capacity;
    if (e->build_exec) cudaGraphExecDestroy(e->build_exec);  // the private graph holds the old pointer
    e->build_exec = nullptr;
    return KS_OK;
  }
  if (E.dir) cudaFree(E.dir);
  E.dir = nullptr;
  const int dims[3] = {E.nx, E.ny, E.nz};
  long long dcount = 1;
  for (int a = 0; a < 3; ++a) {
    // every probe of seeding / sign recovery lies within one ESDF cell of the box
    const int lo = (voxel_index(E.origin[a] - E.ve, T.voxel) >> 3) - 1;
    const int hi = (voxel_index(E.origin[a] + (dims[a] + 1) * E.ve, T.voxel) >> 3) + 1;
    E.dlo[a] = lo;
    E.dn[a] = hi - lo + 1;
    dcount *= E.dn[a];
  }
  if (dcount > (1ll << 30)) return fail(KS_ERR_UNSUPPORTED, "esdf: TSDF blocks per workspace exceed the directory limit");
  E.dcount = static_cast<int>(dcount);
  KS_CUDA(cudaMalloc(&E.dir, static_cast<size_t>(E.dcount) * (sizeof(int) + 1)));
  E.dirg = reinterpret_cast<uint8_t*>(E.dir + E.dcount);
  if (E.pool_surf) cudaFree(E.pool_surf);
  E.pool_surf = nullptr;
  KS_CUDA(cudaMalloc(&E.pool_surf, static_cast<size_t>(T.capacity)));
  e->bound_capacity = T.capacity;
  E.ratio = static_cast<float>(E.ve / T.voxel);
  const int total = E.nx + E.ny + E.nz;
  KS_LAUNCH(k_axis_tables, (total + 127) / 128, 128, 0, e->stream, E, T.voxel);
  KS_CUDA(cudaStreamSynchronize(e->stream));
  {  // resampled seeding: check  probe voxel in {centre voxel, neighbouring cell's centre voxel}  position by position
    std::vector<int> vox(static_cast<size_t>(kVoxRows) * total);
    KS_CUDA(cudaMemcpy(vox.data(), E.vox, vox.size() * sizeof(int), cudaMemcpyDeviceToHost));
    bool ok = E.ve <= T.voxel && E.dn[0] <= kMaxDirX;
    std::vector<int> voxe(total + 6);
    std::vector<uint32_t> plus(E.wpr, 0u), minus(E.wpr, 0u);
    std::vector<uint8_t> flags(E.ny + E.nz, 0);
    int base = 0, ebase = 0;
    for (int a = 0; a < 3; ++a) {
      const int n = dims[a];
      const int* c = vox.data() + kVoxC * total + base;
      const int* ph = vox.data() + kVoxPh * total + base;
      const int* mh = vox.data() + kVoxMh * total + base;
      int* ce = voxe.data() + ebase + 1;  // ce[-1] .. ce[n]
      ce[-1] = vox[kVoxMe * total + base], ce[n] = vox[kVoxPe * total + base + n - 1];
      for (int i = 0; i < n; ++i) ce[i] = c[i];
      for (int i = 0; i < n; ++i) {
        ok = ok && (ph[i] == c[i] || ph[i] == ce[i + 1]) && (mh[i] == c[i] || mh[i] == ce[i - 1]);
        if (a == 0) {
          if (ph[i] != c[i]) plus[i >> 5] |= 1u << (i & 31);
          if (mh[i] != c[i]) minus[i >> 5] |= 1u << (i & 31);
        } else {
          flags[(a == 1 ? 0 : E.ny) + i] = static_cast<uint8_t>((ph[i] != c[i] ? 1 : 0) | (mh[i] != c[i] ? 2 : 0));
        }
      }
      base += n, ebase += n + 2;
    }
    KS_CUDA(cudaMemcpy(E.voxe, voxe.data(), voxe.size() * sizeof(int), cudaMemcpyHostToDevice));
    KS_CUDA(cudaMemcpy(E.xplus, plus.data(), plus.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    KS_CUDA(cudaMemcpy(E.xminus, minus.data(), minus.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    KS_CUDA(cudaMemcpy(E.yzflags, flags.data(), flags.size(), cudaMemcpyHostToDevice));
    bool in_step = voxe[0] >= 0;
    for (int i = 0; i < E.nx + 2; ++i) in_step = in_step && voxe[i] == i + voxe[0];
    E.xshift = in_step ? voxe[0] : -1;
    {  // the same along y and z (k_resample_blockrows needs all three)
      const int* vy = voxe.data() + E.nx + 2;
      const int* vz = vy + E.ny + 2;
      bool ys = vy[0] >= 0, zs = vz[0] >= 0;
      for (int i = 0; i < E.ny + 2; ++i) ys = ys && vy[i] == i + vy[0];
      for (int i = 0; i < E.nz + 2; ++i) zs = zs && vz[i] == i + vz[0];
      E.yshift = ys ? vy[0] : -1, E.zshift = zs ? vz[0] : -1;
      e->resample_by_rows = false;
      if (const char* v = std::getenv("KS_RESAMPLE")) e->resample_by_rows = std::strcmp(v, "rows") == 0;
    }
    {  // integer sign probe (SignTable::negative): same voxel size and every cell centre within 1e-9 voxels of its voxel's middle
      bool centred = E.ve == T.voxel;
      for (int a = 0; a < 3 && centred; ++a)
        for (int k = 0; k < dims[a] && centred; ++k) {
          const double q = (E.origin[a] + (k + 0.5) * E.ve) / T.voxel;
          centred = std::fabs(q - std::floor(q) - 0.5) < 1e-9 && std::fabs(q) < 1e7;
        }
      E.iprobe = centred ? 1 : 0;
      if (const char* v = std::getenv("KS_IPROBE")) E.iprobe = E.iprobe && std::atoi(v) != 0;
    }
    if (ok && e->dc && !E.gtab) {  // the site tables (8 B per cell, touched at the seeds only) exist once the fast path is known to apply
      KS_CUDA(cudaMalloc(&E.gtab, static_cast<size_t>(E.cells) * sizeof(uint2)));
      KS_CUDA(cudaMalloc(&E.seedw, static_cast<size_t>(E.cells) * sizeof(int)));
    }
    e->resample_ok = ok;
    if (const char* v = std::getenv("KS_SEED")) e->resample_ok = e->resample_ok && std::strcmp(v, "bricks") != 0;
  }
  e->bound_voxel = T.voxel;
  return KS_OK;
}

static int order_after(ks_esdf* e, const ks_tsdf* t) {
  cudaStream_t ts = tsdf_stream(t);
  if (ts == e->stream) return KS_OK;
  KS_CUDA(cudaEventRecord(e->dep, ts));
  KS_CUDA(cudaStreamWaitEvent(e->stream, e->dep, 0));
  return KS_OK;
}

static bool fast_build(const ks_esdf* e);
// bricks: also the brick flags / work list of the brick gather and of the hinted sign recovery
static int refresh_directory(ks_esdf* e, const ks_tsdf* t, bool bricks_too = true) {
  EsdfView& E = e->view;
  const bool reset_counters = !bricks_too && fast_build(e);  // the fused build: seed_async finds its counters zeroed
  KS_LAUNCH(k_dir_clear, std::min(2 * kSmCount, (E.dcount + 255) / 256), 256, 0, e->stream, E, reset_counters);
  e->counters_reset = reset_counters;
  KS_LAUNCH(k_dir_fill, 4 * kSmCount, 256, 0, e->stream, E, tsdf_view(t), bricks_too);
  if (bricks_too) {
    KS_CUDA(cudaMemsetAsync(&E.ctrl->active_bricks, 0, sizeof(int), e->stream));
    const int bricks = E.bnx * E.bny * E.bnz;
    KS_LAUNCH(k_brick_active, (bricks + 127) / 128, 128, 0, e->stream, E);
  }
  return KS_OK;
}

// fused build: resampled seeding + table-driven sign recovery inside the divide-and-conquer x sweep
static bool fast_build(const ks_esdf* e) { return e->dc && e->resample_ok && e->cfg.seeding == 1; }

// bits: gather straight into the bit-packed mask of the fused build (gather mode only)
static int seed_async(ks_esdf* e, const ks_tsdf* t, int mode, bool bits) {
  EsdfView& E = e->view;
  if (!e->counters_reset) KS_CUDA(cudaMemsetAsync(E.ctrl, 0, offsetof(EsdfCtrl, active_bricks), e->stream));  // seed_count, signs_recovered
  e->counters_reset = false;
  if (mode == 1) {
    const long long threads = static_cast<long long>(E.ny) * E.nz * E.wpr * 32;  // one warp per 32 x cells
    const unsigned grid = static_cast<unsigned>((threads + 255) / 256);
    if (bits && fast_build(e)) {
      const int words = E.wpr * E.ny * E.nz;
      const int ext_rows = (E.ny + 2) * (E.nz + 2);
      if (E.xshift >= 0 && E.yshift >= 0 && E.zshift >= 0 && !e->resample_by_rows)
        KS_LAUNCH(k_resample_blockrows, (E.dn[1] * E.dn[2] * 8 + kResampleWarps - 1) / kResampleWarps, kResampleWarps * 32, 0, e->stream, E, tsdf_view(t));
      else
        KS_LAUNCH(k_resample_rows, (ext_rows + kResampleWarps - 1) / kResampleWarps, kResampleWarps * 32, 0, e->stream, E, tsdf_view(t));
      KS_LAUNCH(k_seed_dilate, dim3((E.wpr * E.ny + 255) / 256, E.nz), 256, 0, e->stream, E);
      if (e->profile_stages) {  // stage timing: everything in line
        KS_LAUNCH(k_site_tables, 4 * kSmCount, 256, 0, e->stream, E, tsdf_view(t));
      } else {
        KS_CUDA(cudaEventRecord(e->fork, e->stream));
        KS_CUDA(cudaStreamWaitEvent(e->side, e->fork, 0));
        KS_LAUNCH(k_site_tables, 4 * kSmCount, 256, 0, e->side, E, tsdf_view(t));
        KS_CUDA(cudaEventRecord(e->join, e->side));
        e->side_pending = true;
      }
    } else if (bits) {
      const size_t plane_bytes = static_cast<size_t>(E.wpr) * E.ny * E.nz * sizeof(uint32_t);
      KS_CUDA(cudaMemsetAsync(E.mbits, 0, 2 * plane_bytes, e->stream));  // seed plane + geometry-near plane (contiguous)
      KS_LAUNCH(k_seed_gather_bricks, 6 * kSmCount, kGatherWarps * 32, 0, e->stream, E, tsdf_view(t));
    } else KS_LAUNCH(k_seed_gather<false>, grid, 256, 0, e->stream, E, tsdf_view(t));
  } else {
    KS_CUDA(cudaMemsetAsync(E.mask, 0, E.cells, e->stream));
    KS_LAUNCH(k_seed_scatter, 4 * kSmCount, 512, 0, e->stream, E, tsdf_view(t));
    KS_LAUNCH(k_count_mask, 4 * kSmCount, 256, 0, e->stream, E);
  }
  return KS_OK;
}

// bits: phase 1 reads the bit-packed mask; t != nullptr: sign recovery is fused into the x sweep
static int propagate_async(ks_esdf* e, bool bits, const ks_tsdf* t) {
  EsdfView& E = e->view;
  const int plane = E.nx * E.ny;
  const int nwords = (E.nz + 31) / 32;
  const unsigned fgrid = static_cast<unsigned>((E.wpr * E.ny + kFloodWarps - 1) / kFloodWarps);
  const size_t fsmem = static_cast<size_t>(nwords) * 32 * kFloodWarps * sizeof(uint32_t);
  (void)plane;
  if (e->dc) {
    if (!bits) KS_LAUNCH(k_pack_mask, (E.wpr * E.ny * E.nz + 7) / 8, 256, 0, e->stream, E);  // the reference's byte mask -> bit plane
    KS_LAUNCH(k_flood_cols, dim3(E.wpr, E.ny), 32 * nwords, static_cast<size_t>(nwords) * 2 * 32 * sizeof(uint32_t), e->stream, E);
  } else if (bits) KS_LAUNCH(k_flood_z_chunks, E.wpr * E.ny, 32 * nwords, static_cast<size_t>(nwords) * 32 * sizeof(uint32_t), e->stream, E);
  else KS_LAUNCH(k_flood_z<false>, fgrid, kFloodWarps * 32, fsmem, e->stream, E);
  if (e->profile_stages) cudaEventRecord(e->ev[3], e->stream);
  if (e->dc) {
    const dim3 ygrid((E.nx + kTileA - 1) / kTileA, (E.nz + kTileZ - 1) / kTileZ);
#define KS_Y_DC(P, X) KS_LAUNCH((k_sweep_y_dc<P, X>), ygrid, 32 * e->dc_nw_y, e->smem_y, e->stream, E, e->dc_wl_y, e->none_y, e->none_x)
    if (e->pay_y == 2) { if (E.xpay) KS_Y_DC(2, 1); else KS_Y_DC(2, 0); }
    else { if (E.xpay) KS_Y_DC(1, 1); else KS_Y_DC(1, 0); }
#undef KS_Y_DC
  } else KS_LAUNCH(k_sweep_y, dim3((E.nx + 31) / 32, E.nz), 32 * e->bands_y, e->smem_y, e->stream, E, e->band_y, e->bands_y);
  if (e->profile_stages) cudaEventRecord(e->ev[4], e->stream);
  if (e->side_pending) {  // the site tables must be complete before the sweep that reads them
    KS_CUDA(cudaStreamWaitEvent(e->stream, e->join, 0));
    e->side_pending = false;
  }
  const dim3 xgrid((E.ny + 31) / 32, E.nz);
  if (e->dc) {
    const unsigned threads = 32u * e->dc_nw_x;
    const int mode = t && bits && fast_build(e) ? 3 : (t && bits ? 2 : (t ? 1 : 0));
    const TsdfView tv = t ? tsdf_view(t) : TsdfView{};
    const dim3 xgrid(E.nyt, E.nzt);
#define KS_X_DC(M, B) KS_LAUNCH((k_sweep_x_dc<M, B, 0>), xgrid, threads, e->smem_x, e->stream, E, tv, e->dc_wl_x, e->none_x)
#define KS_X_DC1(M) KS_LAUNCH((k_sweep_x_dc<M, false, 1>), xgrid, threads, e->smem_x, e->stream, E, tv, e->dc_wl_x, e->none_x)
#define KS_X_DC_MODE(B)        \
  if (mode == 3) KS_X_DC(3, B);      \
  else if (mode == 2) KS_X_DC(2, B); \
  else if (mode == 1) KS_X_DC(1, B); \
  else KS_X_DC(0, B)
    if (E.xpay) {
      if (mode == 3) KS_X_DC1(3);
      else if (mode == 2) KS_X_DC1(2);
      else if (mode == 1) KS_X_DC1(1);
      else KS_X_DC1(0);
    } else if (e->dc_nw_x > 16) { KS_X_DC_MODE(true); } else { KS_X_DC_MODE(false); }
#undef KS_X_DC1
#undef KS_X_DC_MODE
#undef KS_X_DC
  } else if (t && bits) {  // hint planes are fresh only when this build gathered into the bit planes
    KS_LAUNCH(k_sweep_x<2>, xgrid, 32 * e->bands_x, e->smem_x, e->stream, E, tsdf_view(t), e->band_x, e->bands_x);
  } else if (t) {
    KS_LAUNCH(k_sweep_x<1>, xgrid, 32 * e->bands_x, e->smem_x, e->stream, E, tsdf_view(t), e->band_x, e->bands_x);
  } else {
    KS_LAUNCH(k_sweep_x<0>, xgrid, 32 * e->bands_x, e->smem_x, e->stream, E, TsdfView{}, e->band_x, e->bands_x);
  }
  if (!e->dc) KS_LAUNCH(k_publish, 1, 32, 0, e->stream, E);
  if (t && !e->dc) KS_CUDA(cudaMemsetAsync(&E.ctrl->signs_recovered, 1, 1, e->stream));  // k_sweep_x_dc<signs> sets the flag itself
  KS_CUDA(cudaGetLastError());
  return KS_OK;
}

static int signs_async(ks_esdf* e, const ks_tsdf* t) {
  EsdfView& E = e->view;
  KS_LAUNCH(k_recover_signs, static_cast<unsigned>((E.cells + 255) / 256), 256, 0, e->stream, E, tsdf_view(t));
  KS_CUDA(cudaMemsetAsync(&E.ctrl->signs_recovered, 1, 1, e->stream));
  KS_CUDA(cudaGetLastError());
  return KS_OK;
}

}  // namespace ksb

extern "C" {

static int esdf_init(ks_esdf* e, const ks_esdf_config* cfg);

int ks_esdf_create(const ks_esdf_config* cfg, ks_esdf** out) {
  if (!cfg || !out) return fail(KS_ERR_INVALID, "null argument");
  *out = nullptr;
  // EsdfConfig::validate (esdf.hpp:41-44)
  if (cfg->nx < 1 || cfg->ny < 1 || cfg->nz < 1) return fail(KS_ERR_INVALID, "esdf: dims must be >= 1");
  if (cfg->voxel_size <= 0.0) return fail(KS_ERR_INVALID, "esdf: voxel_size must be > 0");
  int devices = 0;
  if (cudaGetDeviceCount(&devices) != cudaSuccess || devices == 0)
    return fail(KS_ERR_CUDA, "ks_b200: no CUDA device (this library has no CPU path)");
  if (cfg->nx > kMaxDim || cfg->ny > kMaxDim || cfg->nz > kMaxDim)
    return fail(KS_ERR_UNSUPPORTED, "esdf: dims above 1024 per axis are not supported by this build");
  ks_esdf* e = new ks_esdf();
  const int rc = esdf_init(e, cfg);
  if (rc != KS_OK) {  // one cleanup path: whatever was allocated so far goes with the handle
    const std::string message = ks_last_error();
    ks_esdf_destroy(e);
    cudaGetLastError();
    set_error(message);
    return rc;
  }
  *out = e;
  return KS_OK;
}

static int esdf_init(ks_esdf* e, const ks_esdf_config* cfg) {
  e->cfg = *cfg;
  EsdfView& E = e->view;
  E.nx = cfg->nx, E.ny = cfg->ny, E.nz = cfg->nz;
  E.cells = cfg->nx * cfg->ny * cfg->nz;  // <= 2^30
  for (int a = 0; a < 3; ++a) E.origin[a] = cfg->origin[a];
  E.ve = cfg->voxel_size;
  pick_bands(E.ny, e->band_y, e->bands_y);
  pick_bands(E.nx, e->band_x, e->bands_x);
  e->smem_y = sweep_smem_bytes(E.ny, e->bands_y, 2);
  e->smem_x = sweep_smem_bytes(E.nx, e->bands_x, 4);
  {  // divide-and-conquer sweeps whenever their 32-bit keys hold every reachable cost (all dims <= ~830, or a long x axis)
    const uint32_t gmax_y = static_cast<uint32_t>((E.nz - 1) * (E.nz - 1));
    const uint32_t gmax_x = gmax_y + static_cast<uint32_t>((E.ny - 1) * (E.ny - 1));
    const uint64_t d2_max = static_cast<uint64_t>(gmax_x) + static_cast<uint64_t>(E.nx - 1) * (E.nx - 1);  // field word: d2 in 21 bits
    e->dc = KeysY::fits(E.ny, gmax_y) && KeysX::fits(E.nx, gmax_x) && d2_max < (1ull << 21) &&
            dc_smem_bytes_x(E.nx, E.nx + E.ny + E.nz) <= 226 * 1024 && dc_smem_bytes_y(E.ny) <= 226 * 1024;
    e->pay_y = edt_dc::Keys<2>::fits(E.ny, gmax_y) ? 2 : 1;
    if (const char* v = std::getenv("KS_PAY_Y")) e->pay_y = std::atoi(v) == 1 ? 1 : e->pay_y;
    E.tab_all = e->pay_y == 2 ? 0 : 1;
    if (const char* v = std::getenv("KS_SWEEP")) e->dc = e->dc && std::strcmp(v, "stack") != 0;
    e->none_y = KeysY::none_offset(E.ny, gmax_y);
    e->none_x = KeysX::none_offset(E.nx, gmax_x);
    // warps per tile: 8 (y) and 16 (x) measured best while several tiles share an SM (tools/ab_sweeps.sh); long rows
    // leave room for fewer tiles, which then get more warps each
    // y sweep, measured per row length (tools/gpu_env_sweep.sh KS_DC_WARPS_Y): 100 rows 8 warps, 200 rows 4 warps (93 vs 98 us),
    // 500 rows 8 warps (703 vs 759 us with 16)
    e->dc_wl_y = dc_smem_bytes_y(E.ny) > 16 * 1024 && dc_smem_bytes_y(E.ny) <= 48 * 1024 ? 2 : 3;
    e->dc_wl_x = dc_smem_bytes_x(E.nx, E.nx + E.ny + E.nz) > 113 * 1024 ? 5 : 4;
    if (const char* v = std::getenv("KS_DC_WARPS_Y")) e->dc_wl_y = std::min(4, std::max(0, std::atoi(v)));
    if (const char* v = std::getenv("KS_DC_WARPS_X")) e->dc_wl_x = std::min(5, std::max(0, std::atoi(v)));
    e->dc_nw_y = 1 << e->dc_wl_y, e->dc_nw_x = 1 << e->dc_wl_x;
    // x sweep with the table bit inside the candidate (no payload image in shared memory) whenever the keys have the bit to spare
    E.xpay = e->dc && edt_dc::Keys<1>::fits(E.nx, gmax_x) ? 1 : 0;
    if (const char* v = std::getenv("KS_XPAY")) E.xpay = E.xpay && std::atoi(v) != 0;
    if (E.xpay) {
      // tiles per SM by shared memory, warps per tile so that tiles x warps stays within the 32 warps 64 registers allow,
      // preferring a count that deals the row's stretches out evenly (score = resident warps x (1 + evenness) / 2)
      const size_t bytes = dc_smem_bytes_x(E.nx, E.nx + E.ny + E.nz, false) + 1024;
      const int stretches = (E.nx + (1 << kTopShiftX) - 1) >> kTopShiftX;
      double best = 0.0;
      for (int tiles = 1; tiles <= 4; ++tiles) {
        if (tiles * bytes > 227 * 1024) break;
        const int wmax = std::min(16, 32 / tiles);
        for (int w = std::max(4, wmax - 3); w <= wmax; ++w) {
          const double even = static_cast<double>(stretches) / (w * ((stretches + w - 1) / w));
          const double score = tiles * w * (1.0 + even) / 2.0;
          if (score > best) best = score, e->dc_nw_x = w;
        }
      }
    }
    // any warp count works (KS_DC_NWARPS_*): the stretches of a row are dealt round-robin to the warps, so a count that
    // divides them evenly leaves no warp idle at the end of a tile
    auto floor_log2 = [](int v) { int l = 0; while ((2 << l) <= v) ++l; return l; };
    if (const char* v = std::getenv("KS_DC_NWARPS_Y")) e->dc_nw_y = std::min(16, std::max(1, std::atoi(v))), e->dc_wl_y = floor_log2(e->dc_nw_y);
    if (const char* v = std::getenv("KS_DC_NWARPS_X")) e->dc_nw_x = std::min(E.xpay ? 16 : 32, std::max(1, std::atoi(v)));
    e->dc_wl_x = floor_log2(e->dc_nw_x);
    if (e->dc) e->smem_y = dc_smem_bytes_y(E.ny), e->smem_x = dc_smem_bytes_x(E.nx, E.nx + E.ny + E.nz, !E.xpay);
  }
  if (e->smem_y > 227 * 1024 || e->smem_x > 227 * 1024) {
    return fail(KS_ERR_UNSUPPORTED, "esdf: row length exceeds the shared-memory tile of this build (ny <= 1024, nx <= 900)");
  }
  // The attribute is per kernel and process-wide: it is set to the opt-in maximum (never to one handle's own size, which
  // would lower it under a larger ESDF that is still alive).
  constexpr int kSmemOptIn = 227 * 1024 - 256;  // minus the kernels' few bytes of static shared memory
  KS_CUDA(cudaFuncSetAttribute(k_sweep_y, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemOptIn));
  KS_CUDA(cudaFuncSetAttribute(k_sweep_x<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemOptIn));
  KS_CUDA(cudaFuncSetAttribute(k_sweep_x<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemOptIn));
  KS_CUDA(cudaFuncSetAttribute(k_sweep_x<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemOptIn));
  KS_CUDA(cudaFuncSetAttribute((k_sweep_y_dc<1, 0>), cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemOptIn));
  KS_CUDA(cudaFuncSetAttribute((k_sweep_y_dc<2, 0>), cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemOptIn));
  KS_CUDA(cudaFuncSetAttribute((k_sweep_y_dc<1, 1>), cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemOptIn));
  KS_CUDA(cudaFuncSetAttribute((k_sweep_y_dc<2, 1>), cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemOptIn));
  KS_CUDA(cudaFuncSetAttribute(k_flood_cols, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
#define KS_X_ATTR(M, B) KS_CUDA(cudaFuncSetAttribute((k_sweep_x_dc<M, B, 0>), cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemOptIn))
#define KS_X_ATTR4(B) KS_X_ATTR(0, B); KS_X_ATTR(1, B); KS_X_ATTR(2, B); KS_X_ATTR(3, B)
  KS_X_ATTR4(false); KS_X_ATTR4(true);
#define KS_X_ATTR1(M) KS_CUDA(cudaFuncSetAttribute((k_sweep_x_dc<M, false, 1>), cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemOptIn))
  KS_X_ATTR1(0); KS_X_ATTR1(1); KS_X_ATTR1(2); KS_X_ATTR1(3);
#undef KS_X_ATTR1
#undef KS_X_ATTR4
#undef KS_X_ATTR
  KS_CUDA(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
  e->own_stream = true;
  e->own_graphs = true;
  if (const char* v = std::getenv("KS_OWN_GRAPHS")) e->own_graphs = std::atoi(v) != 0;
  KS_CUDA(cudaEventCreateWithFlags(&e->dep, cudaEventDisableTiming));
  KS_CUDA(cudaStreamCreateWithFlags(&e->side, cudaStreamNonBlocking));
  KS_CUDA(cudaEventCreateWithFlags(&e->fork, cudaEventDisableTiming));
  KS_CUDA(cudaEventCreateWithFlags(&e->join, cudaEventDisableTiming));
  for (cudaEvent_t& ev : e->ev) KS_CUDA(cudaEventCreate(&ev));
  const int total = E.nx + E.ny + E.nz;
  KS_CUDA(cudaMalloc(&E.vox, kVoxRows * total * sizeof(int)));
  KS_CUDA(cudaMalloc(&E.ctr, total * sizeof(double)));
  KS_CUDA(cudaMalloc(&E.qsf, total * sizeof(float)));
  E.bnx = (E.nx + 7) / 8, E.bny = (E.ny + 7) / 8, E.bnz = (E.nz + 7) / 8;
  KS_CUDA(cudaMalloc(&E.brick, static_cast<size_t>(E.bnx) * E.bny * E.bnz));
  KS_CUDA(cudaMalloc(&E.active, static_cast<size_t>(E.bnx) * E.bny * E.bnz * sizeof(int)));
  E.wpr = (E.nx + 31) / 32;
  KS_CUDA(cudaMalloc(&E.mbits, 2 * static_cast<size_t>(E.wpr) * E.ny * E.nz * sizeof(uint32_t)));  // both bit planes
  E.gbits = E.mbits + static_cast<size_t>(E.wpr) * E.ny * E.nz;
  E.wpr2 = (E.nx + 2 + 31) / 32;
  {
    const size_t ext_words = static_cast<size_t>(E.wpr2) * (E.ny + 2) * (E.nz + 2);
    KS_CUDA(cudaMalloc(&E.cbits, 3 * ext_words * sizeof(uint32_t)));
    E.obits = E.cbits + ext_words, E.nbits = E.obits + ext_words;
    KS_CUDA(cudaMalloc(&E.voxe, (total + 6) * sizeof(int)));
    KS_CUDA(cudaMalloc(&E.xplus, 2 * E.wpr * sizeof(uint32_t)));
    E.xminus = E.xplus + E.wpr;
    KS_CUDA(cudaMalloc(&E.yzflags, E.ny + E.nz));
  }
  KS_CUDA(cudaMalloc(&E.mask, E.cells));
  E.nzw = (E.nz + 31) / 32;
  E.fast = e->dc ? 1 : 0;
  E.nyt = (E.ny + kTileA - 1) / kTileA, E.nzt = (E.nz + kTileZ - 1) / kTileZ;
  const size_t cells = static_cast<size_t>(E.cells);
  if (e->dc) {  // phase 1 as per-column bit strings, phase 2 as tile images, the field as two 4-byte buffers
    const size_t col_words = static_cast<size_t>(E.nzw) * E.ny * E.nx;
    KS_CUDA(cudaMalloc(&E.near_z, 3 * col_words * sizeof(uint32_t)));
    E.zbits = reinterpret_cast<uint32_t*>(E.near_z), E.zinfo = E.zbits + col_words, E.zgbits = E.zinfo + col_words;
    const size_t image = static_cast<size_t>(E.nzt) * E.nyt * E.nx * 32;
    KS_CUDA(cudaMalloc(&E.gimg, image * sizeof(uint32_t)));
    KS_CUDA(cudaMalloc(&E.himg, image * sizeof(uint16_t)));
    bool single = false;  // KS_ESDF_SINGLE_BUFFER=1: one field buffer (readers on other streams may then see a build in progress)
    if (const char* v = std::getenv("KS_ESDF_SINGLE_BUFFER")) single = std::atoi(v) != 0;
    KS_CUDA(cudaMalloc(&E.f32[0], cells * sizeof(uint32_t)));
    if (single) E.f32[1] = E.f32[0];
    else KS_CUDA(cudaMalloc(&E.f32[1], cells * sizeof(uint32_t)));
  } else {
    KS_CUDA(cudaMalloc(&E.near_z, cells * sizeof(uint16_t)));
    KS_CUDA(cudaMalloc(&E.yz, cells * sizeof(uint32_t)));
    KS_CUDA(cudaMalloc(&E.field, cells * sizeof(uint2)));
  }
  KS_CUDA(cudaMalloc(&E.ctrl, sizeof(EsdfCtrl)));
  KS_CUDA(cudaMalloc(&e->summary_scratch, sizeof(SummaryScratch)));
  KS_CUDA(cudaMemsetAsync(e->summary_scratch, 0, sizeof(SummaryScratch), e->stream));
  KS_CUDA(cudaMallocHost(&e->h_ctrl, sizeof(EsdfCtrl)));
  KS_CUDA(cudaMemsetAsync(E.ctrl, 0, sizeof(EsdfCtrl), e->stream));
  KS_CUDA(cudaMemsetAsync(E.mbits, 0, 2 * static_cast<size_t>(E.wpr) * E.ny * E.nz * sizeof(uint32_t), e->stream));
  if (E.field) KS_CUDA(cudaMemsetAsync(E.field, 0xFF, cells * sizeof(uint2), e->stream));  // no sites yet (fast path: pub_seeds == 0)
  KS_CUDA(cudaStreamSynchronize(e->stream));
  return KS_OK;
}

void ks_esdf_destroy(ks_esdf* e) {
  if (!e) return;
  if (e->stream) cudaStreamSynchronize(e->stream);
  EsdfView& E = e->view;
  cudaFree(e->query_scratch), cudaFree(e->summary_scratch), cudaFree(E.cbits), cudaFree(E.voxe), cudaFree(E.xplus), cudaFree(E.yzflags), cudaFree(E.gtab), cudaFree(E.seedw), cudaFree(E.vox), cudaFree(E.ctr), cudaFree(E.qsf), cudaFree(E.brick), cudaFree(E.active), cudaFree(E.mbits), cudaFree(E.mask), cudaFree(E.near_z), cudaFree(E.yz), cudaFree(E.field), cudaFree(E.gimg), cudaFree(E.himg);
  if (E.f32[1] != E.f32[0]) cudaFree(E.f32[1]);
  cudaFree(E.f32[0]);
  cudaFree(E.ctrl);
  if (E.dir) cudaFree(E.dir);
  if (E.pool_surf) cudaFree(E.pool_surf);
  cudaFreeHost(e->h_ctrl);
  if (e->build_exec) cudaGraphExecDestroy(e->build_exec);
  if (e->side) cudaStreamSynchronize(e->side), cudaStreamDestroy(e->side);
  if (e->fork) cudaEventDestroy(e->fork);
  if (e->join) cudaEventDestroy(e->join);
  if (e->dep) cudaEventDestroy(e->dep);
  for (cudaEvent_t ev : e->ev)
    if (ev) cudaEventDestroy(ev);
  if (e->own_stream && e->stream) cudaStreamDestroy(e->stream);
  delete e;
}

int ks_esdf_set_stream(ks_esdf* e, ks_stream s) {
  if (!e) return fail(KS_ERR_INVALID, "null esdf");
  KS_CUDA(cudaStreamSynchronize(e->stream));
  if (e->own_stream) cudaStreamDestroy(e->stream);
  e->own_stream = false;
  e->stream = static_cast<cudaStream_t>(s);
  if (e->build_exec) cudaGraphExecDestroy(e->build_exec);
  e->build_exec = nullptr;
  return KS_OK;
}

static int enqueue_build(ks_esdf* e, const ks_tsdf* t, bool prof) {
  int rc;
  e->profile_stages = prof;
  if (prof) cudaEventRecord(e->ev[0], e->stream);
  if ((rc = refresh_directory(e, t, !fast_build(e))) != KS_OK) return rc;
  if (prof) cudaEventRecord(e->ev[1], e->stream);
  const bool bits = e->cfg.seeding == 1;
  if ((rc = seed_async(e, t, e->cfg.seeding, bits)) != KS_OK) return rc;
  if (prof) cudaEventRecord(e->ev[2], e->stream);
  rc = propagate_async(e, bits, t);  // sign recovery rides in the x sweep
  if (prof) cudaEventRecord(e->ev[5], e->stream);
  if (prof) cudaEventRecord(e->ev[6], e->stream);
  e->profile_stages = false;
  return rc;
}

// The build is a fixed sequence of launches whose arguments only depend on the two handles, so outside a
// caller's own capture (and when no stage timing is asked for) it is recorded once per TSDF into a private
// CUDA graph and replayed: one launch call and graph-internal dependencies instead of ~15 stream launches.
int ks_esdf_build_async(ks_esdf* e, const ks_tsdf* t) {
  if (!e || !t) return fail(KS_ERR_INVALID, "null argument");
  int rc;
  if ((rc = bind_tsdf(e, t)) != KS_OK) return rc;
  if ((rc = order_after(e, t)) != KS_OK) return rc;
  e->generation.fetch_add(1, std::memory_order_relaxed);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(e->stream, &cap);
  const bool outer_capture = cap != cudaStreamCaptureStatusNone;
  const bool prof = e->profile && !outer_capture;
  if (outer_capture || prof || !e->own_graphs) {
    rc = enqueue_build(e, t, prof);
    if (rc == KS_OK && !outer_capture) tsdf_reader_enqueued(t, e->stream);
    return rc;
  }
  if (!e->build_exec || e->build_tsdf != tsdf_uid(t) || e->build_voxel != e->bound_voxel) {
    if (e->build_exec) cudaGraphExecDestroy(e->build_exec);
    e->build_exec = nullptr;
    cudaGraph_t graph = nullptr;
    KS_CUDA(cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal));
    rc = enqueue_build(e, t, false);
    const cudaError_t end = cudaStreamEndCapture(e->stream, &graph);
    if (rc != KS_OK || end != cudaSuccess || !graph) {
      if (graph) cudaGraphDestroy(graph);
      cudaGetLastError();
      e->own_graphs = false;  // this context cannot capture: plain launches from now on
      return rc != KS_OK ? rc : enqueue_build(e, t, false);
    }
    size_t nodes = 0;
    cudaGraphGetNodes(graph, nullptr, &nodes);
    e->build_nodes = static_cast<int64_t>(nodes);
    const cudaError_t inst = cudaGraphInstantiate(&e->build_exec, graph, 0);
    cudaGraphDestroy(graph);
    if (inst != cudaSuccess) {
      cudaGetLastError();
      e->build_exec = nullptr, e->own_graphs = false;
      return enqueue_build(e, t, false);
    }
    e->build_tsdf = tsdf_uid(t), e->build_voxel = e->bound_voxel;
  } else {
    g_kernel_launches.fetch_add(e->build_nodes, std::memory_order_relaxed);  // the capture counted its own launches once
  }
  KS_CUDA(cudaGraphLaunch(e->build_exec, e->stream));
  tsdf_reader_enqueued(t, e->stream);
  return KS_OK;
}

uint64_t ks_esdf_generation(const ks_esdf* e) { return e ? e->generation.load(std::memory_order_relaxed) : 0; }

int ks_esdf_profile(ks_esdf* e, int32_t enable) {
  if (!e) return fail(KS_ERR_INVALID, "null esdf");
  e->profile = enable != 0;
  return KS_OK;
}

int ks_esdf_stage_ms(ks_esdf* e, float out[6]) {
  if (!e || !out) return fail(KS_ERR_INVALID, "null argument");
  KS_CUDA(cudaStreamSynchronize(e->stream));
  for (int i = 0; i < 6; ++i) {
    out[i] = 0.0f;
    if (cudaEventElapsedTime(&out[i], e->ev[i], e->ev[i + 1]) != cudaSuccess) {
      cudaGetLastError();
      out[i] = -1.0f;
    }
  }
  return KS_OK;
}

}  // extern "C"
namespace ksb {
int esdf_report_enqueue(ks_esdf* e) {
  KS_CUDA(cudaMemcpyAsync(e->h_ctrl, e->view.ctrl, sizeof(EsdfCtrl), cudaMemcpyDeviceToHost, e->stream));
  return KS_OK;
}
int esdf_report_collect(ks_esdf* e, ks_esdf_report* report) {
  if (report) {
    report->status = KS_OK;
    report->has_sites = e->h_ctrl->seed_count > 0;
    report->signs_recovered = e->h_ctrl->signs_recovered != 0;
    report->seed_count = static_cast<int64_t>(e->h_ctrl->seed_count);
  }
  return KS_OK;
}
}  // namespace ksb
extern "C" {

int ks_esdf_sync(ks_esdf* e, ks_esdf_report* report) {
  if (!e) return fail(KS_ERR_INVALID, "null esdf");
  const int rc = esdf_report_enqueue(e);
  if (rc != KS_OK) return rc;
  KS_CUDA(cudaStreamSynchronize(e->stream));
  return esdf_report_collect(e, report);
}

int ks_esdf_last_report(const ks_esdf* e, ks_esdf_report* report) {
  if (!e || !report) return fail(KS_ERR_INVALID, "null argument");
  report->status = KS_OK;
  report->has_sites = e->h_ctrl->seed_count > 0;
  report->signs_recovered = e->h_ctrl->signs_recovered != 0;
  report->seed_count = static_cast<int64_t>(e->h_ctrl->seed_count);
  return KS_OK;
}

int ks_esdf_build(ks_esdf* e, const ks_tsdf* t) {
  int rc = ks_esdf_build_async(e, t);
  return rc != KS_OK ? rc : ks_esdf_sync(e, nullptr);
}

int ks_esdf_seed(ks_esdf* e, const ks_tsdf* t, int32_t mode, uint8_t* mask_host) {
  if (!e || !t) return fail(KS_ERR_INVALID, "null argument");
  int rc;
  if ((rc = bind_tsdf(e, t)) != KS_OK) return rc;
  if ((rc = order_after(e, t)) != KS_OK) return rc;
  if ((rc = refresh_directory(e, t)) != KS_OK) return rc;
  if ((rc = seed_async(e, t, mode, false)) != KS_OK) return rc;
  if (mask_host) KS_CUDA(cudaMemcpyAsync(mask_host, e->view.mask, e->view.cells, cudaMemcpyDeviceToHost, e->stream));
  return ks_esdf_sync(e, nullptr);
}

int ks_esdf_propagate(ks_esdf* e, const uint8_t* mask_host, int64_t mask_len) {
  if (!e) return fail(KS_ERR_INVALID, "null esdf");
  EsdfView& E = e->view;
  e->generation.fetch_add(1, std::memory_order_relaxed);
  if (mask_host) {
    if (mask_len != E.cells) return fail(KS_ERR_INVALID, "esdf: seed mask size does not match grid");  // esdf.hpp:195-196
    KS_CUDA(cudaMemcpyAsync(E.mask, mask_host, E.cells, cudaMemcpyHostToDevice, e->stream));
    KS_CUDA(cudaMemsetAsync(E.ctrl, 0, offsetof(EsdfCtrl, front), e->stream));
    KS_LAUNCH(k_count_mask, 4 * kSmCount, 256, 0, e->stream, E);
  } else {
    KS_CUDA(cudaMemsetAsync(&E.ctrl->signs_recovered, 0, sizeof(int), e->stream));
  }
  int rc = propagate_async(e, false, nullptr);
  return rc != KS_OK ? rc : ks_esdf_sync(e, nullptr);
}

int ks_esdf_recover_signs(ks_esdf* e, const ks_tsdf* t) {
  if (!e || !t) return fail(KS_ERR_INVALID, "null argument");
  int rc;
  if ((rc = bind_tsdf(e, t)) != KS_OK) return rc;
  if ((rc = order_after(e, t)) != KS_OK) return rc;
  if ((rc = refresh_directory(e, t)) != KS_OK) return rc;
  e->generation.fetch_add(1, std::memory_order_relaxed);
  if ((rc = signs_async(e, t)) != KS_OK) return rc;
  return ks_esdf_sync(e, nullptr);
}

int ks_esdf_download(ks_esdf* e, int32_t* site_xyz, double* distance, int32_t* d2) {
  if (!e) return fail(KS_ERR_INVALID, "null esdf");
  EsdfView& E = e->view;
  int* d_site = nullptr;
  double* d_dist = nullptr;
  int* d_d2 = nullptr;
  const size_t cells = static_cast<size_t>(E.cells);
  const int rc = [&]() -> int {
    if (site_xyz) KS_CUDA(cudaMalloc(&d_site, cells * 3 * sizeof(int)));
    if (distance) KS_CUDA(cudaMalloc(&d_dist, cells * sizeof(double)));
    if (d2) KS_CUDA(cudaMalloc(&d_d2, cells * sizeof(int)));
    KS_LAUNCH(k_export, static_cast<unsigned>((cells + 255) / 256), 256, 0, e->stream, E, d_site, d_dist, d_d2);
    if (site_xyz) KS_CUDA(cudaMemcpyAsync(site_xyz, d_site, cells * 3 * sizeof(int), cudaMemcpyDeviceToHost, e->stream));
    if (distance) KS_CUDA(cudaMemcpyAsync(distance, d_dist, cells * sizeof(double), cudaMemcpyDeviceToHost, e->stream));
    if (d2) KS_CUDA(cudaMemcpyAsync(d2, d_d2, cells * sizeof(int), cudaMemcpyDeviceToHost, e->stream));
    KS_CUDA(cudaStreamSynchronize(e->stream));
    return KS_OK;
  }();
  cudaFree(d_site), cudaFree(d_dist), cudaFree(d_d2);
  return rc;
}

int ks_esdf_query_device_async(ks_esdf* e, const double* points_dev, int64_t n, double* distance_dev, double* gradient_dev,
                               uint8_t* inside_dev) {
  if (!e) return fail(KS_ERR_INVALID, "null esdf");
  if (n <= 0) return KS_OK;
  KS_LAUNCH(k_query, static_cast<unsigned>((n + 255) / 256), 256, 0, e->stream, e->view, points_dev, static_cast<long long>(n),
            distance_dev, gradient_dev, inside_dev);
  KS_CUDA(cudaGetLastError());
  return KS_OK;
}

int ks_esdf_probe_summary_device_async(ks_esdf* e, const double* points_dev, int64_t n, double near_distance, double tag,
                                       double* summary_dev) {
  if (!e || !points_dev || !summary_dev) return fail(KS_ERR_INVALID, "null argument");
  if (n < 0 || n > (1 << 30)) return fail(KS_ERR_INVALID, "esdf: bad probe count");
  const int ctas = static_cast<int>(std::min<int64_t>(kSummaryCtas, std::max<int64_t>(1, (n + 127) / 128)));
  KS_LAUNCH(k_probe_summary, ctas, 128, 0, e->stream, e->view, points_dev, static_cast<int>(n), near_distance, tag, e->summary_scratch,
            summary_dev);
  KS_CUDA(cudaGetLastError());
  return KS_OK;
}

// Device scratch of the host-pointer entry points (query, scene collision): one buffer per handle, grown on demand
// and kept, so that a planner calling them every iteration pays no cudaMalloc / cudaFree (each of which also
// synchronises the device).  Callers hold e->query_mu: the reference allows concurrent queries.
static int call_scratch(ks_esdf* e, size_t doubles, double** out) {
  if (doubles > static_cast<size_t>(e->query_cap)) {
    const size_t cap = std::max<size_t>(doubles + doubles / 4, 8192);
    KS_CUDA(cudaStreamSynchronize(e->stream));
    cudaFree(e->query_scratch);
    e->query_scratch = nullptr, e->query_cap = 0;
    KS_CUDA(cudaMalloc(&e->query_scratch, cap * sizeof(double)));
    e->query_cap = static_cast<int64_t>(cap);
  }
  *out = static_cast<double*>(e->query_scratch);
  return KS_OK;
}

int ks_esdf_scene_collision_static(ks_esdf* e, const double* centers_host, const double* radii_host, int64_t n,
                                   double activation_margin, ks_collision_report* report, double* gradient_xyz_host) {
  if (!e || !report) return fail(KS_ERR_INVALID, "null argument");
  report->max_penetration = 0.0, report->worst_sphere = -1, report->cost = 0.0;
  if (n <= 0) return KS_OK;
  if (n > (1 << 30)) return fail(KS_ERR_INVALID, "scene_collision: too many spheres");
  std::lock_guard<std::mutex> lock(e->query_mu);
  double* base = nullptr;
  int rc = call_scratch(e, static_cast<size_t>(n) * 9 + 3, &base);
  if (rc != KS_OK) return rc;
  double *d_c = base, *d_grad = d_c + 3 * n, *d_r = d_grad + 3 * n, *d_pen = d_r + n, *d_cost = d_pen + n, *d_rep = d_cost + n;
  KS_CUDA(cudaMemcpyAsync(d_c, centers_host, n * 3 * sizeof(double), cudaMemcpyHostToDevice, e->stream));
  KS_CUDA(cudaMemcpyAsync(d_r, radii_host, n * sizeof(double), cudaMemcpyHostToDevice, e->stream));
  KS_LAUNCH(k_collision_static, static_cast<unsigned>((n + 255) / 256), 256, 0, e->stream, e->view, d_c, d_r, static_cast<int>(n),
            activation_margin, d_pen, d_cost, d_grad);
  KS_LAUNCH(k_collision_reduce, 1, 256, 0, e->stream, d_pen, d_cost, static_cast<int>(n), d_rep);
  double rep[3];
  KS_CUDA(cudaMemcpyAsync(rep, d_rep, sizeof rep, cudaMemcpyDeviceToHost, e->stream));
  if (gradient_xyz_host)
    KS_CUDA(cudaMemcpyAsync(gradient_xyz_host, d_grad, n * 3 * sizeof(double), cudaMemcpyDeviceToHost, e->stream));
  KS_CUDA(cudaStreamSynchronize(e->stream));
  report->max_penetration = rep[0], report->worst_sphere = static_cast<int32_t>(rep[1]), report->cost = rep[2];
  return KS_OK;
}

int ks_esdf_scene_collision_swept(ks_esdf* e, const double* centers_host, const double* radii_host,
                                  const double* velocities_host, int32_t timesteps, int32_t spheres, double activation_margin,
                                  double dt, int32_t max_checks, ks_collision_report* reports, double* center_gradient,
                                  double* next_center_gradient, double* velocity_gradient) {
  if (!e || !reports) return fail(KS_ERR_INVALID, "null argument");
  if (timesteps <= 0 || spheres <= 0) return KS_OK;
  ks_esdf_report st;
  int rc = ks_esdf_sync(e, &st);
  if (rc != KS_OK) return rc;
  if (!st.signs_recovered) return fail(KS_ERR_INVALID, "scene_collision: esdf signs not recovered");  // collision.hpp:181
  const size_t n = static_cast<size_t>(timesteps) * spheres;
  std::lock_guard<std::mutex> lock(e->query_mu);
  double* base = nullptr;
  if ((rc = call_scratch(e, n * 17 + spheres + static_cast<size_t>(timesteps) * 3, &base)) != KS_OK) return rc;
  double *d_c = base, *d_v = d_c + 3 * n, *d_g = d_v + 3 * n, *d_pen = d_g + 9 * n, *d_cost = d_pen + n, *d_r = d_cost + n, *d_rep = d_r + spheres;
  KS_CUDA(cudaMemsetAsync(d_g, 0, 3 * n * 3 * sizeof(double), e->stream));
  KS_CUDA(cudaMemcpyAsync(d_c, centers_host, n * 3 * sizeof(double), cudaMemcpyHostToDevice, e->stream));
  KS_CUDA(cudaMemcpyAsync(d_v, velocities_host, n * 3 * sizeof(double), cudaMemcpyHostToDevice, e->stream));
  KS_CUDA(cudaMemcpyAsync(d_r, radii_host, spheres * sizeof(double), cudaMemcpyHostToDevice, e->stream));
  KS_LAUNCH(k_collision_swept, static_cast<unsigned>((n + 127) / 128), 128, 0, e->stream, e->view, d_c, d_r, d_v, timesteps, spheres,
            activation_margin, dt, max_checks, d_pen, d_cost, d_g, d_g + n * 3, d_g + 2 * n * 3);
  KS_LAUNCH(k_collision_reduce, timesteps, 256, 0, e->stream, d_pen, d_cost, spheres, d_rep);
  std::vector<double> rep(static_cast<size_t>(timesteps) * 3);
  KS_CUDA(cudaMemcpyAsync(rep.data(), d_rep, rep.size() * sizeof(double), cudaMemcpyDeviceToHost, e->stream));
  if (center_gradient) KS_CUDA(cudaMemcpyAsync(center_gradient, d_g, n * 3 * sizeof(double), cudaMemcpyDeviceToHost, e->stream));
  if (next_center_gradient)
    KS_CUDA(cudaMemcpyAsync(next_center_gradient, d_g + n * 3, n * 3 * sizeof(double), cudaMemcpyDeviceToHost, e->stream));
  if (velocity_gradient)
    KS_CUDA(cudaMemcpyAsync(velocity_gradient, d_g + 2 * n * 3, n * 3 * sizeof(double), cudaMemcpyDeviceToHost, e->stream));
  KS_CUDA(cudaStreamSynchronize(e->stream));
  for (int t = 0; t < timesteps; ++t) {
    reports[t].max_penetration = rep[3 * t];
    reports[t].worst_sphere = static_cast<int32_t>(rep[3 * t + 1]);
    reports[t].cost = rep[3 * t + 2];
  }
  return KS_OK;
}

int ks_esdf_query(ks_esdf* e, const double* points_host, int64_t n, double* distance, double* gradient_xyz, uint8_t* inside) {
  if (!e) return fail(KS_ERR_INVALID, "null esdf");
  if (n <= 0) return KS_OK;
  std::lock_guard<std::mutex> lock(e->query_mu);
  double* base = nullptr;  // {points, gradient} 24 B, distance 8 B, inside 1 B per query (rounded up to 8 doubles)
  int rc0 = call_scratch(e, static_cast<size_t>(n) * 8, &base);
  if (rc0 != KS_OK) return rc0;
  double *d_pts = base, *d_grad = d_pts + 3 * n, *d_dist = d_grad + 3 * n;
  uint8_t* d_in = reinterpret_cast<uint8_t*>(d_dist + n);
  KS_CUDA(cudaMemcpyAsync(d_pts, points_host, n * 3 * sizeof(double), cudaMemcpyHostToDevice, e->stream));
  int rc = ks_esdf_query_device_async(e, d_pts, n, d_dist, d_grad, d_in);
  if (rc == KS_OK) {
    if (distance) KS_CUDA(cudaMemcpyAsync(distance, d_dist, n * sizeof(double), cudaMemcpyDeviceToHost, e->stream));
    if (gradient_xyz) KS_CUDA(cudaMemcpyAsync(gradient_xyz, d_grad, n * 3 * sizeof(double), cudaMemcpyDeviceToHost, e->stream));
    if (inside) KS_CUDA(cudaMemcpyAsync(inside, d_in, n, cudaMemcpyDeviceToHost, e->stream));
    KS_CUDA(cudaStreamSynchronize(e->stream));
  }
  return rc;
}

}  // extern "C"
