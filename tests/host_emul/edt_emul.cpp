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
