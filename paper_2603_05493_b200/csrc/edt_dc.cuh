// Exact 1-D lower-envelope pass of the ESDF transform by monotone divide and conquer
// ("PBA+" phases 2/3 without stacks).
//
// Replaces, for one axis sweep, esdf_detail::Envelope::{push,walk} and the two sweep loops of
// propagate() in the reference (/root/reference/proj/include/ks/esdf.hpp:129-186, :236-280).
// The function both compute for every integer position t of a row is
//     win(t) = argmin_u (t-u)^2 + r2(u),   ties -> smallest u
// and win(t) is non-decreasing in t (leftmost minima of a totally monotone matrix).  So once the
// winners at t-s and t+s are known, the winner at t lies between them: positions are visited in
// the order of a binary tree (s = P/2, P/4, .., 1) and every visit is a plain min-scan over a
// window of candidates.  Per level the windows of one row add up to <= n + (number of visits), so a
// row costs n*(log2 n + 1) evaluations of 4-5 instructions each, in straight-line code: no stack,
// no division, no data-dependent branch.  Only the first few levels (fewer visits than warps) need
// the warps of a tile to cooperate; below them each warp owns a stretch of positions (stretch()).
//
// Keys.  A candidate u with offset g = r2(u) is stored once as  G[u] = g << S | low(u),  where
// low(u) holds u (and for the y sweep one payload bit below it); its cost at t is then
//     key = ((t-u)^2 << S) + G[u]
// and `min` over unsigned keys yields the smallest cost and, on equal cost, the smallest u.
// A position without candidate gets g = gmax + (n-1)^2 + 1, which no reachable cost attains
// (any valid candidate costs at most gmax + (n-1)^2), so it loses against every valid candidate and
// a row without candidates is recognised by its winner's cost.  fits() states when keys stay
// below 2^32; the library falls back to the banded stack kernels (edt_core.cuh) otherwise.
//
// Layout: every array is [position][32 rows] so that lane == shared-memory bank.
//
// The functions are __host__ __device__ so tests/host_emul can run the very same code on the CPU
// against the oracle; the product only ever runs them on the GPU.
#pragma once
#include <stdint.h>

#include <type_traits>
#include <utility>

#if defined(__CUDACC__)
#define KS_DC_HD __host__ __device__ __forceinline__
#else
#define KS_DC_HD inline
#endif

namespace ksb {
namespace edt_dc {

constexpr int kRows = 32;

KS_DC_HD int at(int pos, int row) { return pos * kRows + row; }

// S = key shift, kPay = payload bits below u inside the low field (S = 10 + kPay).
template <int kPay>
struct Keys {
  static constexpr int kShift = 10 + kPay;
  static constexpr uint32_t kLowMask = (1u << kShift) - 1u;
  // offset of a position that holds no candidate
  static KS_DC_HD uint32_t none_offset(int n, uint32_t gmax) { return gmax + static_cast<uint32_t>((n - 1) * (n - 1)) + 1u; }
  // largest cost any scan can form must stay below 2^(32-S)
  static KS_DC_HD bool fits(int n, uint32_t gmax) {
    const uint64_t top = static_cast<uint64_t>(none_offset(n, gmax)) + static_cast<uint64_t>(n - 1) * (n - 1);
    return n <= 1024 && top < (1ull << (32 - kShift));
  }
  static KS_DC_HD uint32_t pack(uint32_t g, int u, uint32_t payload) {
    return g << kShift | static_cast<uint32_t>(u) << kPay | payload;
  }
  static KS_DC_HD int winner(uint32_t key) { return static_cast<int>((key & kLowMask) >> kPay); }
  static KS_DC_HD uint32_t payload(uint32_t key) { return key & ((1u << kPay) - 1u); }
  static KS_DC_HD uint32_t cost(uint32_t key) { return key >> kShift; }
};

// The visiting order.  Positions are t' = t + 1 in [1, n]; P is the smallest power of two > n;
// level k visits the odd multiples of s = P >> (k+1) that are <= n.  Their neighbours t' -+ s are
// even multiples of s: visited at an earlier level, or outside the row (window end = row end).
struct Plan {
  int n, P, levels;  // P == 1 << levels
};
KS_DC_HD Plan make_plan(int n) {
  Plan p;
  p.n = n;
#if defined(__CUDA_ARCH__)
  p.levels = 32 - __clz(n);  // smallest power of two > n, without the loop (n >= 1)
  p.P = 1 << p.levels;
#else
  p.P = 1;
  p.levels = 0;
  while (p.P <= n) p.P <<= 1, ++p.levels;
#endif
  return p;
}
KS_DC_HD int level_step(const Plan& p, int level) { return p.P >> (level + 1); }
KS_DC_HD int level_visits(const Plan& p, int level) {  // odd multiples of s that are <= n
  return ((p.n >> (p.levels - level - 1)) + 1) >> 1;
}

// Window of candidates for the visit at t' (step s), part `part` of 2^parts_log2 equal slices.
// Kt holds the keys of the positions visited by the top levels: Kt[t' / top_step] for t' a multiple
// of top_step.  len may come out <= 0 for a slice that lies beyond a short window.
template <int kPay>
KS_DC_HD void top_window(const uint32_t* Kt, int n, int top_shift, int tp, int s, int part, int parts_log2, int row, int& lo,
                         int& len) {
  int l = 0, h = n - 1;
  if (tp - s > 0) l = Keys<kPay>::winner(Kt[at((tp - s) >> top_shift, row)]);
  if (tp + s <= n) h = Keys<kPay>::winner(Kt[at((tp + s) >> top_shift, row)]);
  int L = h - l + 1;
  if (parts_log2 != 0) {
    const int pl = (L + (1 << parts_log2) - 1) >> parts_log2;
    l += part * pl;
    const int rest = h - l + 1;
    L = pl < rest ? pl : rest;
  }
  lo = l;
  len = L;
}

// All lanes of a warp scan the same number of candidates (the longest window among them), each
// from its own start; a start is pulled down so the scan stays inside the row.  Scanning more
// candidates than the window holds cannot change the minimum (the true winner is inside).
KS_DC_HD int clamp_start(int lo, int scan_len, int n) {
  const int last = n - scan_len;
  lo = lo < last ? lo : last;
  return lo > 0 ? lo : 0;
}

// min over u in [lo, lo + scan_len) of ((t-u)^2 << S) + G[u]; scan_len >= 1 is the same for the whole warp.
template <int kPay>
KS_DC_HD uint32_t scan(const uint32_t* G, int lo, int scan_len, int t, int row) {
  constexpr int S = Keys<kPay>::kShift;
  const uint32_t* g = G + at(lo, row);
  int d = t - lo;
  uint32_t best = 0xFFFFFFFFu;
  // key(u+k) = ((d-k)^2 << S) + g[k] = (d*d << S) + ((k*k - 2*k*d) << S) + g[k]
#if defined(__CUDA_ARCH__)
#pragma unroll 1
#endif
  for (; scan_len >= 4; scan_len -= 4) {
    const uint32_t base = static_cast<uint32_t>(d * d) << S;
    const uint32_t m2d = static_cast<uint32_t>(-2 * d) << S;
    const uint32_t k0 = base + g[0];
    const uint32_t k1 = base + (1u << S) + m2d + g[kRows];
    const uint32_t k2 = base + (4u << S) + 2u * m2d + g[2 * kRows];
    const uint32_t k3 = base + (9u << S) + 3u * m2d + g[3 * kRows];
    const uint32_t a = k0 < k1 ? k0 : k1;
    const uint32_t b = k2 < k3 ? k2 : k3;
    const uint32_t c = a < b ? a : b;
    best = best < c ? best : c;
    g += 4 * kRows;
    d -= 4;
  }
  if (scan_len & 2) {
    const uint32_t base = static_cast<uint32_t>(d * d) << S;
    const uint32_t m2d = static_cast<uint32_t>(-2 * d) << S;
    const uint32_t k0 = base + g[0];
    const uint32_t k1 = base + (1u << S) + m2d + g[kRows];
    const uint32_t a = k0 < k1 ? k0 : k1;
    best = best < a ? best : a;
    g += 2 * kRows;
    d -= 2;
  }
  if (scan_len & 1) {
    const uint32_t k = (static_cast<uint32_t>(d * d) << S) + g[0];
    best = best < k ? best : k;
  }
  return best;
}

// Below the top levels no cooperation is needed, and no tree either: a warp that knows the winners at both
// ends of a stretch of positions resolves ALL kM positions inside in one pass over the candidates between
// those two winners, keeping kM running minima in registers.  A candidate costs one load and, per position,
// one multiply-add and one add-min -- (d0 + j)^2 = d0^2 + 2 j d0 + j^2 with j a compile-time constant --
// instead of a visit of its own per position (window, warp-wide maximum, loop set-up: ~50 instructions each,
// which is what the unrolled binary recursion spent most of its time on).
// Positions: t = a .. a + kM - 1 (those < n); lo_w / hi_w = winners at t = a - 1 and t = a + kM (row ends when
// those lie outside).  wmax(v) returns the largest v among the warp's lanes; emit(t, key) receives every position.
// kM > kFatMax: the centre position is resolved first by a plain scan of the window, which halves the windows of
// the two halves (a pass over W candidates costs about 4 + 2*kM instructions each, so wide stretches pay twice:
// more positions per candidate AND more candidates).
constexpr int kFatMax = 7;

// Where the keys of a stretch go.  put<I>(t, key): I is the position's index inside the (outermost) stretch as a
// compile-time constant, so a sink may keep the keys in a register array; t is the position itself.
template <class F>
struct CallSink {  // adapter for a plain callable emit(t, key)
  F& f;
  template <int I>
  KS_DC_HD void put(int t, uint32_t key) {
    f(t, key);
  }
};
template <int kN>
struct KeySink {  // keys of positions a .. a + kN - 1 in registers; positions >= n keep 0xFFFFFFFF
  uint32_t k[kN];
  template <int I>
  KS_DC_HD void put(int, uint32_t key) {
    k[I] = key;
  }
};

template <int kBase, class Sink, int kM, int... Is>
KS_DC_HD void put_all(Sink& sink, int a, int n, const uint32_t (&best)[kM], std::integer_sequence<int, Is...>) {
  ((a + Is < n ? sink.template put<kBase + Is>(a + Is, best[Is]) : void()), ...);
}

template <int kPay, int kM, int kBase, class WarpMax, class Sink>
KS_DC_HD void stretch_into(const uint32_t* G, int n, int a, int lo_w, int hi_w, int row, WarpMax&& wmax, Sink& sink) {
  constexpr int S = Keys<kPay>::kShift;
  if constexpr (kM > kFatMax) {
    constexpr int kHalf = (kM - 1) / 2;
    static_assert(2 * kHalf + 1 == kM, "stretch lengths are 2^k - 1");
    const int t = a + kHalf;
    int mid = hi_w;
    if (t < n) {
      const int longest = wmax(hi_w - lo_w + 1);
      const uint32_t key = scan<kPay>(G, clamp_start(lo_w, longest, n), longest, t, row);
      sink.template put<kBase + kHalf>(t, key);
      mid = Keys<kPay>::winner(key);
    }
    stretch_into<kPay, kHalf, kBase>(G, n, a, lo_w, mid, row, wmax, sink);
    if (t + 1 < n) stretch_into<kPay, kHalf, kBase + kHalf + 1>(G, n, t + 1, mid, hi_w, row, wmax, sink);
    return;
  } else {
    const int longest = wmax(hi_w - lo_w + 1);
    const int lo = clamp_start(lo_w, longest, n);
    uint32_t best[kM];
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
    for (int j = 0; j < kM; ++j) best[j] = 0xFFFFFFFFu;
    const uint32_t* g = G + at(lo, row);
    int d0 = a - lo;
#if defined(__CUDA_ARCH__)
#pragma unroll 2
#endif
    for (int i = 0; i < longest; ++i) {
      // key_j = ((d0 + j)^2 << S) + g = base + j * slope + (j*j << S): one multiply-add and one add-min per position
      const uint32_t base = (static_cast<uint32_t>(d0 * d0) << S) + g[0];
      uint32_t slope = static_cast<uint32_t>(2 * d0) << S;
#if defined(__CUDA_ARCH__)
      asm volatile("" : "+r"(slope));  // keeps the compiler from folding the keys back into (d0 + j)^2, three instructions each
#endif
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
      for (int j = 0; j < kM; ++j) {
        const uint32_t key = base + static_cast<uint32_t>(j) * slope + (static_cast<uint32_t>(j * j) << S);  // modular
        best[j] = best[j] < key ? best[j] : key;
      }
      g += kRows;
      --d0;
    }
    put_all<kBase>(sink, a, n, best, std::make_integer_sequence<int, kM>{});
  }
}

// emit(t, key) receives every position of the stretch (any order)
template <int kPay, int kM, class WarpMax, class Emit>
KS_DC_HD void stretch(const uint32_t* G, int n, int a, int lo_w, int hi_w, int row, WarpMax&& wmax, Emit&& emit) {
  CallSink<std::remove_reference_t<Emit>> sink{emit};
  stretch_into<kPay, kM, 0>(G, n, a, lo_w, hi_w, row, wmax, sink);
}

}  // namespace edt_dc
}  // namespace ksb
