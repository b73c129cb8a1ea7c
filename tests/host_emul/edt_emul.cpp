// CPU emulation of the CUDA EDT tile kernels' control flow, for tests only.
// Runs the SAME __host__ __device__ code as paper_2603_05493_b200/csrc/esdf.cu
// (edt_core.cuh), stage by stage, with loops standing in for warps/lanes and
// stage boundaries standing in for __syncthreads().  Not a product path: the
// shipped library has no CPU implementation.
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../paper_2603_05493_b200/csrc/edt_core.cuh"

using namespace ksb::edt;

namespace {

struct TileMem {
  std::vector<uint16_t> s, t, lo, hi;
  RowTile view(int n, int band) {
    const int bands = (n + band - 1) / band;
    s.assign(static_cast<size_t>(n) * kRows, 0);
    t.assign(static_cast<size_t>(n) * kRows, 0);
    lo.assign(static_cast<size_t>(bands) * kRows, 0);
    hi.assign(static_cast<size_t>(bands) * kRows, 0);
    return RowTile{s.data(), t.data(), lo.data(), hi.data(), n, band, bands};
  }
};

template <class Src, class Emit>
void run_tile(TileMem& mem, int n, int band, int rows, const Src& src, Emit&& emit) {
  RowTile T = mem.view(n, band);
  for (int b = 0; b < T.bands; ++b)
    for (int r = 0; r < rows; ++r) build_band(T, src, b, r);
  for (int j = 0; (1 << j) < T.bands; ++j)
    for (int b = 0; b < T.bands; b += (2 << j))
      for (int r = 0; r < rows; ++r) merge_groups(T, src, b, j, r);
  for (int b = 0; b < T.bands; ++b)
    for (int r = 0; r < rows; ++r)
      colour_band(T, b, r, [&](int pos, uint16_t win) { emit(pos, r, win); });
}

struct SrcY {  // phase 2: candidate at y is the column's nearest seed z
  const uint16_t* zs;  // [ny][32]
  int z;
  int r2(int pos, int row) const {
    const uint16_t v = zs[at(pos, row)];
    if (v == kNone) return -1;
    const int d = z - static_cast<int>(v);
    return d * d;
  }
};

struct SrcX {  // phase 3: candidate at x is phase 2's (site_y, site_z)
  const uint32_t* yz;  // [nx][32], 0xFFFFFFFF = none
  int y0, z;
  int r2(int pos, int row) const {
    const uint32_t v = yz[at(pos, row)];
    if (v == 0xFFFFFFFFu) return -1;
    const int dy = (y0 + row) - static_cast<int>(v & 0xFFFFu);
    const int dz = z - static_cast<int>(v >> 16);
    return dy * dy + dz * dz;
  }
};

}  // namespace

extern "C" int emul_propagate(const uint8_t* mask, int nx, int ny, int nz, int band_y, int band_x,
                              int32_t* site, int32_t* d2) {
  const size_t cells = static_cast<size_t>(nx) * ny * nz;
  auto idx = [&](int x, int y, int z) { return static_cast<size_t>(x) + static_cast<size_t>(nx) * (y + static_cast<size_t>(ny) * z); };
  // phase 1
  std::vector<uint16_t> near_z(cells);
  const int nwords = (nz + 31) / 32;
  std::vector<uint32_t> words(nwords);
  for (int y = 0; y < ny; ++y)
    for (int x = 0; x < nx; ++x) {
      std::fill(words.begin(), words.end(), 0u);
      for (int z = 0; z < nz; ++z)
        if (mask[idx(x, y, z)]) words[z >> 5] |= 1u << (z & 31);
      for (int z = 0; z < nz; ++z) near_z[idx(x, y, z)] = nearest_set_bit(words.data(), 1, nwords, z);
    }
  // phase 2
  std::vector<uint32_t> yz(cells);
  TileMem mem;
  std::vector<uint16_t> zs_tile(static_cast<size_t>(ny) * kRows);
  for (int z = 0; z < nz; ++z)
    for (int x0 = 0; x0 < nx; x0 += kRows) {
      const int rows = nx - x0 < kRows ? nx - x0 : kRows;
      for (int y = 0; y < ny; ++y)
        for (int r = 0; r < rows; ++r) zs_tile[at(y, r)] = near_z[idx(x0 + r, y, z)];
      SrcY src{zs_tile.data(), z};
      run_tile(mem, ny, band_y, rows, src, [&](int pos, int r, uint16_t win) {
        yz[idx(x0 + r, pos, z)] =
            win == kNone ? 0xFFFFFFFFu : (static_cast<uint32_t>(win) | static_cast<uint32_t>(zs_tile[at(win, r)]) << 16);
      });
    }
  // phase 3
  std::vector<uint32_t> yz_tile(static_cast<size_t>(nx) * kRows);
  for (int z = 0; z < nz; ++z)
    for (int y0 = 0; y0 < ny; y0 += kRows) {
      const int rows = ny - y0 < kRows ? ny - y0 : kRows;
      for (int x = 0; x < nx; ++x)
        for (int r = 0; r < rows; ++r) yz_tile[at(x, r)] = yz[idx(x, y0 + r, z)];
      SrcX src{yz_tile.data(), y0, z};
      run_tile(mem, nx, band_x, rows, src, [&](int pos, int r, uint16_t win) {
        const size_t i = idx(pos, y0 + r, z);
        if (win == kNone) {
          site[3 * i] = site[3 * i + 1] = site[3 * i + 2] = -1;
          d2[i] = 0x7FFFFFFF;
          return;
        }
        const uint32_t v = yz_tile[at(win, r)];
        const int sx = win, sy = static_cast<int>(v & 0xFFFFu), sz = static_cast<int>(v >> 16);
        site[3 * i] = sx;
        site[3 * i + 1] = sy;
        site[3 * i + 2] = sz;
        const int dx = pos - sx, dy = y0 + r - sy, dz = z - sz;
        d2[i] = dx * dx + dy * dy + dz * dz;
      });
    }
  return 0;
}

// ---- divide-and-conquer sweeps (csrc/edt_dc.cuh), same emulation idea: loops stand in for
// warps/lanes, level boundaries stand in for __syncthreads() ----
#include "../../paper_2603_05493_b200/csrc/edt_dc.cuh"

namespace {
namespace dc = ksb::edt_dc;

// One CTA: tile G [n][32] of packed candidates -> K [n][32] winning keys, following the kernels' schedule:
// top levels (visits at the multiples of the top step, windows cut into 2^parts slices, minima combined
// as atomicMin does), then one subtree per stretch.  Rows are independent except for the warp-wide scan
// length; `fuzz` stands in for it by lengthening every scan pseudo-randomly, which must not change any
// winner.  scans += scan lengths, visits += visits (of row 0, as a proxy for the warp).
constexpr int kTopShift = 4, kTopStep = 1 << kTopShift;

struct Fuzz {
  uint32_t state;
  int extra;
  int operator()(int v) {
    state = state * 1664525u + 1013904223u;
    const int grown = v + (extra ? static_cast<int>((state >> 24) % (extra + 1)) : 0);
    return grown;
  }
};

template <int kPay>
void dc_tile(const std::vector<uint32_t>& G, std::vector<uint32_t>& K, int n, int warps_log2, int fuzz, long long* scans, long long* visits) {
  const dc::Plan plan = dc::make_plan(n);
  K.assign(static_cast<size_t>(n) * dc::kRows, 0xFFFFFFFFu);
  std::vector<uint32_t> Kt((static_cast<size_t>(n >> kTopShift) + 1) * dc::kRows, 0xFFFFFFFFu);
  for (int r = 0; r < dc::kRows; ++r) {
    Fuzz wmax{static_cast<uint32_t>(r * 2654435761u + n), fuzz};
    for (int level = 0; level < plan.levels; ++level) {
      const int s = dc::level_step(plan, level);
      if (s < kTopStep) break;
      const int parts_log2 = warps_log2 > level ? warps_log2 - level : 0;
      const int items = dc::level_visits(plan, level) << parts_log2;
      std::vector<uint32_t> next = Kt;  // writes of a level become visible at its barrier
      for (int item = 0; item < items; ++item) {
        const int tp = s * (2 * (item >> parts_log2) + 1);
        int lo, len;
        dc::top_window<kPay>(Kt.data(), n, kTopShift, tp, s, item & ((1 << parts_log2) - 1), parts_log2, r, lo, len);
        int longest = wmax(len);
        if (longest > n) longest = n;
        if (longest <= 0) continue;
        if (r == 0 && scans) *scans += longest, *visits += 1;
        const uint32_t k = dc::scan<kPay>(G.data(), dc::clamp_start(lo, longest, n), longest, tp - 1, r);
        uint32_t& dst = next[dc::at(tp >> kTopShift, r)];
        dst = k < dst ? k : dst;
      }
      Kt.swap(next);
    }
    auto bounded = [&](int v) { const int g = wmax(v); return g > n ? n : g; };
    for (int j = 0; (j << kTopShift) < n; ++j) {
      const int a = j << kTopShift;
      const bool closed = a + kTopStep <= n;
      const uint32_t right = closed ? Kt[dc::at(j + 1, r)] : 0u;
      const int lo_w = a > 0 ? dc::Keys<kPay>::winner(Kt[dc::at(j, r)]) : 0;
      const int hi_w = closed ? dc::Keys<kPay>::winner(right) : n - 1;
      auto emit = [&](int t, uint32_t key) { K[dc::at(t, r)] = key; };
      dc::stretch<kPay, kTopStep - 1>(G.data(), n, a, lo_w, hi_w, r, bounded, emit);
      if (closed) emit(a + kTopStep - 1, right);
    }
  }
}
}  // namespace

extern "C" int emul_dc_fits(int nx, int ny, int nz) {
  const uint32_t gy = static_cast<uint32_t>((nz - 1) * (nz - 1));
  const uint32_t gx = gy + static_cast<uint32_t>((ny - 1) * (ny - 1));
  return dc::Keys<1>::fits(ny, gy) && dc::Keys<0>::fits(nx, gx);
}

extern "C" int emul_propagate_dc(const uint8_t* mask, int nx, int ny, int nz, int warps_log2, int fuzz, int32_t* site, int32_t* d2,
                                 long long* stats /* [4]: y scans, y visits, x scans, x visits */) {
  const size_t cells = static_cast<size_t>(nx) * ny * nz;
  auto idx = [&](int x, int y, int z) { return static_cast<size_t>(x) + static_cast<size_t>(nx) * (y + static_cast<size_t>(ny) * z); };
  std::vector<uint16_t> near_z(cells);
  const int nwords = (nz + 31) / 32;
  std::vector<uint32_t> words(nwords);
  for (int y = 0; y < ny; ++y)
    for (int x = 0; x < nx; ++x) {
      std::fill(words.begin(), words.end(), 0u);
      for (int z = 0; z < nz; ++z)
        if (mask[idx(x, y, z)]) words[z >> 5] |= 1u << (z & 31);
      for (int z = 0; z < nz; ++z) near_z[idx(x, y, z)] = nearest_set_bit(words.data(), 1, nwords, z);
    }
  using KY = dc::Keys<1>;
  using KX = dc::Keys<0>;
  const uint32_t gmax_y = static_cast<uint32_t>((nz - 1) * (nz - 1));
  const uint32_t gmax_x = gmax_y + static_cast<uint32_t>((ny - 1) * (ny - 1));
  if (!KY::fits(ny, gmax_y) || !KX::fits(nx, gmax_x)) return 1;
  // phase 2: payload bit = the seed lies above z
  std::vector<uint32_t> yz(cells), G, K;
  const uint32_t none_y = KY::none_offset(ny, gmax_y);
  for (int z = 0; z < nz; ++z)
    for (int x0 = 0; x0 < nx; x0 += dc::kRows) {
      G.assign(static_cast<size_t>(ny) * dc::kRows, 0);
      for (int y = 0; y < ny; ++y)
        for (int r = 0; r < dc::kRows; ++r) {
          const uint16_t v = x0 + r < nx ? near_z[idx(x0 + r, y, z)] : kNone;
          const int dz = static_cast<int>(v) - z;
          G[dc::at(y, r)] = v == kNone ? KY::pack(none_y, y, 0) : KY::pack(static_cast<uint32_t>(dz * dz), y, dz > 0 ? 1u : 0u);
        }
      dc_tile<1>(G, K, ny, warps_log2, fuzz, stats ? stats + 0 : nullptr, stats ? stats + 1 : nullptr);
      for (int y = 0; y < ny; ++y)
        for (int r = 0; r < dc::kRows && x0 + r < nx; ++r) {
          const uint32_t k = K[dc::at(y, r)];
          uint32_t out = 0xFFFFFFFFu;
          if (KY::cost(k) < none_y) {
            const int u = KY::winner(k);
            const int dy = y - u;
            const int dz2 = static_cast<int>(KY::cost(k)) - dy * dy;
            int dz = 0;
            while (dz * dz < dz2) ++dz;  // exact root (the device uses sqrtf on a perfect square < 2^24)
            const int sz = KY::payload(k) ? z + dz : z - dz;
            out = static_cast<uint32_t>(u) | static_cast<uint32_t>(sz) << 16;
          }
          yz[idx(x0 + r, y, z)] = out;
        }
    }
  // phase 3
  const uint32_t none_x = KX::none_offset(nx, gmax_x);
  for (int z = 0; z < nz; ++z)
    for (int y0 = 0; y0 < ny; y0 += dc::kRows) {
      G.assign(static_cast<size_t>(nx) * dc::kRows, 0);
      for (int x = 0; x < nx; ++x)
        for (int r = 0; r < dc::kRows; ++r) {
          const uint32_t v = y0 + r < ny ? yz[idx(x, y0 + r, z)] : 0xFFFFFFFFu;
          if (v == 0xFFFFFFFFu) {
            G[dc::at(x, r)] = KX::pack(none_x, x, 0);
            continue;
          }
          const int dy = (y0 + r) - static_cast<int>(v & 0xFFFFu), dz = z - static_cast<int>(v >> 16);
          G[dc::at(x, r)] = KX::pack(static_cast<uint32_t>(dy * dy + dz * dz), x, 0);
        }
      dc_tile<0>(G, K, nx, warps_log2, fuzz, stats ? stats + 2 : nullptr, stats ? stats + 3 : nullptr);
      for (int x = 0; x < nx; ++x)
        for (int r = 0; r < dc::kRows && y0 + r < ny; ++r) {
          const size_t i = idx(x, y0 + r, z);
          const uint32_t k = K[dc::at(x, r)];
          if (KX::cost(k) >= none_x) {
            site[3 * i] = site[3 * i + 1] = site[3 * i + 2] = -1;
            d2[i] = 0x7FFFFFFF;
            continue;
          }
          const int sx = KX::winner(k);
          const uint32_t v = yz[idx(sx, y0 + r, z)];
          site[3 * i] = sx;
          site[3 * i + 1] = static_cast<int>(v & 0xFFFFu);
          site[3 * i + 2] = static_cast<int>(v >> 16);
          d2[i] = static_cast<int>(KX::cost(k));
        }
    }
  return 0;
}
