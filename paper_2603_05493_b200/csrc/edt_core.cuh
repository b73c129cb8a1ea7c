// Banded exact 1-D lower-envelope pass of the ESDF transform ("PBA+" phases 2/3).
//
// Replaces, for one axis sweep, esdf_detail::Envelope::{push,walk} and the two
// sweep loops of propagate() in the reference
// (/root/reference/proj/include/ks/esdf.hpp:129-186, :236-280).  The reference
// builds one stack per row serially with exact rational boundaries; here a tile
// of 32 rows is processed by one CTA: lane <-> row, warp <-> band of positions.
// Every band builds its own proximate-site stack, bands are merged pairwise in
// log2(bands) rounds, and each band then colours its own outputs.
//
// Winner definition (identical to the reference for every integer position t,
// see DESIGN.md "EDT tie rule"):   argmin_u (t-u)^2 + r2(u), ties -> smallest u.
// Boundaries are kept as integers: an entry's `start` is the first integer
// position at which it is STRICTLY better than its predecessor (Meijster's Sep),
// which decides exactly the same winners as the reference's rational test.
//
// All arrays are laid out [position][32 rows] so that lane == shared-memory
// bank for every data-dependent access (conflict-free by construction).
//
// The functions are __host__ __device__ so tests/host_emul can run the very same
// code on the CPU against the oracle; the product only ever runs them on the GPU.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define KS_HD __host__ __device__ __forceinline__
#else
#define KS_HD inline
#endif

namespace ksb {
namespace edt {

constexpr int kRows = 32;
constexpr uint16_t kNone = 0xFFFFu;

struct RowTile {
  uint16_t* stk_s;  // [n][32]   stack entry: site position
  uint16_t* stk_t;  // [n][32]   stack entry: first position where it wins
  uint16_t* lo;     // [bands][32] first live stack slot of the band
  uint16_t* hi;     // [bands][32] one past the last live slot
  int n;            // row length
  int band;         // positions per band
  int bands;        // ceil(n / band)
};

KS_HD int at(int pos, int row) { return pos * kRows + row; }

// floor(num / den) for den > 0 and |num| < 2^23 (positions < 1024, r2 < 2^22):
// one float divide plus an exact integer correction.
KS_HD int floordiv_small(int num, int den) {
#if defined(__CUDA_ARCH__)
  int q = __float2int_rd(__fdividef(static_cast<float>(num), static_cast<float>(den)));
#else
  float qf = static_cast<float>(num) / static_cast<float>(den);
  int q = static_cast<int>(qf);
  if (static_cast<float>(q) > qf) --q;
#endif
  // the estimate is within one of the true floor (|num| < 2^23, quotient error < 1): one exact step
  const int rem = num - q * den;
  return q + (rem >= den) - (rem < 0);
}

// First integer position where the parabola at u (offset gu) is strictly below
// the one at l < u (offset gl).
KS_HD int takeover(int l, int gl, int u, int gu) {
  const int num = (u * u - l * l) + (gu - gl);
  const int den = 2 * (u - l);
  return floordiv_small(num, den) + 1;
}

KS_HD int cost(int t, int u, int gu) {
  const int d = t - u;
  return d * d + gu;
}

// Stage 1: band-local stack for one row.  Src::r2(pos,row) < 0 means "no candidate".
// Written as ONE flat loop in which every iteration either pops the top or consumes the next
// position: lanes (= rows) with different pop counts re-converge every iteration instead of
// serialising a nested pop loop per position.
template <class Src>
KS_HD void build_band(const RowTile& T, const Src& src, int b, int row) {
  const int base = b * T.band;
  const int end = base + T.band < T.n ? base + T.band : T.n;
  int top = base;
  int l = 0, tl = 0, gl = 0;  // cached top entry
  int u = base;
  int gu = u < end ? src.r2(u, row) : -1;
  while (u < end) {
    bool advance = true;
    if (gu >= 0) {
      if (top == base) {
        T.stk_s[at(top, row)] = static_cast<uint16_t>(u);
        T.stk_t[at(top, row)] = 0;
        l = u, tl = 0, gl = gu;
        ++top;
      } else if (cost(tl, l, gl) > cost(tl, u, gu)) {  // u strictly better where l starts: l never wins
        --top;
        if (top > base) {
          l = T.stk_s[at(top - 1, row)];
          tl = T.stk_t[at(top - 1, row)];
          gl = src.r2(l, row);
        }
        advance = false;
      } else {
        const int w = takeover(l, gl, u, gu);
        if (w < T.n) {
          T.stk_s[at(top, row)] = static_cast<uint16_t>(u);
          T.stk_t[at(top, row)] = static_cast<uint16_t>(w);
          l = u, tl = w, gl = gu;
          ++top;
        }
      }
    }
    if (advance) {
      ++u;
      gu = u < end ? src.r2(u, row) : -1;
    }
  }
  T.lo[at(b, row)] = static_cast<uint16_t>(base);
  T.hi[at(b, row)] = static_cast<uint16_t>(top);
}

// Stage 2, round j: band b (b % (2<<j) == 0) merges group [b, b+2^j) with
// [b+2^j, b+2^(j+1)).  Removes left tops / right bottoms that can never win and
// fixes the start of the first surviving right entry.
template <class Src>
KS_HD void merge_groups(const RowTile& T, const Src& src, int b, int j, int row) {
  const int m = b + (1 << j);
  if (m >= T.bands) return;
  const int e = b + (2 << j) < T.bands ? b + (2 << j) : T.bands;
  int lb = m - 1;
  while (lb >= b && T.lo[at(lb, row)] == T.hi[at(lb, row)]) --lb;
  if (lb < b) return;  // left group empty: right group's first entry already starts at 0
  int rb = m;
  while (rb < e && T.lo[at(rb, row)] == T.hi[at(rb, row)]) ++rb;
  if (rb >= e) return;
  while (true) {
    const int li = T.hi[at(lb, row)] - 1;
    const int l = T.stk_s[at(li, row)], tl = T.stk_t[at(li, row)], gl = src.r2(l, row);
    const int ri = T.lo[at(rb, row)];
    const int r = T.stk_s[at(ri, row)], gr = src.r2(r, row);
    if (cost(tl, l, gl) > cost(tl, r, gr)) {  // left top never wins
      T.hi[at(lb, row)] = static_cast<uint16_t>(li);
      if (li == T.lo[at(lb, row)]) {
        do --lb;
        while (lb >= b && T.lo[at(lb, row)] == T.hi[at(lb, row)]);
        if (lb < b) {  // left exhausted: r heads the merged group
          T.stk_t[at(ri, row)] = 0;
          break;
        }
      }
      continue;
    }
    const int w = takeover(l, gl, r, gr);
    // start of r's successor inside the right group (n if none)
    int t2 = T.n;
    {
      int ri2 = ri + 1, rb2 = rb;
      if (ri2 == T.hi[at(rb, row)]) {
        do ++rb2;
        while (rb2 < e && T.lo[at(rb2, row)] == T.hi[at(rb2, row)]);
        ri2 = rb2 < e ? T.lo[at(rb2, row)] : -1;
      }
      if (ri2 >= 0) t2 = T.stk_t[at(ri2, row)];
    }
    if (w >= t2) {  // right bottom never wins: its successor (or the row end) comes first
      T.lo[at(rb, row)] = static_cast<uint16_t>(ri + 1);
      if (ri + 1 == T.hi[at(rb, row)]) {
        do ++rb;
        while (rb < e && T.lo[at(rb, row)] == T.hi[at(rb, row)]);
        if (rb >= e) break;  // right exhausted
      }
      continue;
    }
    T.stk_t[at(ri, row)] = static_cast<uint16_t>(w);
    break;
  }
}

// Stage 3: colour the band's own positions by walking the merged stack (the
// concatenation of every band's live slots, starts strictly increasing).
// emit(pos, winner) with winner == kNone when the row holds no candidate at all.
template <class Emit>
KS_HD void colour_band(const RowTile& T, int b, int row, Emit&& emit) {
  const int base = b * T.band;
  const int end = base + T.band < T.n ? base + T.band : T.n;
  // last band whose first live entry starts at or before `base`
  int cb = -1, clo = 0, chi = 0;
  for (int bb = 0; bb < T.bands; ++bb) {
    const int lo = T.lo[at(bb, row)], hi = T.hi[at(bb, row)];
    if (lo == hi) continue;
    if (static_cast<int>(T.stk_t[at(lo, row)]) > base) break;
    cb = bb, clo = lo, chi = hi;
  }
  if (cb < 0) {  // the first live entry of a row always starts at 0, so the row is empty
    for (int p = base; p < end; ++p) emit(p, kNone);
    return;
  }
  // last entry of that band starting at or before `base` (binary search, starts ascending)
  int k = clo;
  {
    int hi_k = chi - 1;
    while (k < hi_k) {
      const int mid = (k + hi_k + 1) >> 1;
      if (static_cast<int>(T.stk_t[at(mid, row)]) <= base) k = mid;
      else hi_k = mid - 1;
    }
  }
  uint16_t cur = T.stk_s[at(k, row)];
  // successor entry and its start
  int nb = cb, nk = k + 1, next_t = T.n;
  auto settle = [&]() {
    while (nb < T.bands && nk >= chi) {
      ++nb;
      if (nb < T.bands) {
        nk = T.lo[at(nb, row)];
        chi = T.hi[at(nb, row)];
      }
    }
    next_t = nb < T.bands ? static_cast<int>(T.stk_t[at(nk, row)]) : T.n;
  };
  settle();
  for (int p = base; p < end; ++p) {
    while (next_t <= p) {
      cur = T.stk_s[at(nk, row)];
      ++nk;
      settle();
    }
    emit(p, cur);
  }
}

KS_HD int high_bit(uint32_t m) {  // m != 0
#if defined(__CUDA_ARCH__)
  return 31 - __clz(static_cast<int>(m));
#else
  return 31 - __builtin_clz(m);
#endif
}
KS_HD int low_bit(uint32_t m) {  // m != 0
#if defined(__CUDA_ARCH__)
  return __ffs(static_cast<int>(m)) - 1;
#else
  return __builtin_ctz(m);
#endif
}

// Phase 1 helper: nearest set bit to position z in a bit string of nz bits
// (words[w] holds positions 32w..32w+31), ties -> lower position
// (esdf.hpp:213-233).  Returns kNone if no bit is set.  `stride` lets the words
// live in a [word][lane] shared-memory layout.
KS_HD uint16_t nearest_set_bit(const uint32_t* words, int stride, int nwords, int z) {
  const int w0 = z >> 5, b0 = z & 31;
  // at or below z
  int below = -1;
  {
    uint32_t m = words[w0 * stride] & (0xFFFFFFFFu >> (31 - b0));
    int w = w0;
    while (m == 0 && w > 0) m = words[--w * stride];
    if (m != 0) below = 32 * w + high_bit(m);
  }
  if (below == z) return static_cast<uint16_t>(z);
  int above = -1;
  {
    uint32_t m = words[w0 * stride] & (0xFFFFFFFFu << b0);
    int w = w0;
    while (m == 0 && w + 1 < nwords) m = words[++w * stride];
    if (m != 0) above = 32 * w + low_bit(m);
  }
  if (above < 0) return below < 0 ? kNone : static_cast<uint16_t>(below);
  if (below < 0) return static_cast<uint16_t>(above);
  return (above - z) < (z - below) ? static_cast<uint16_t>(above) : static_cast<uint16_t>(below);
}

}  // namespace edt
}  // namespace ksb
