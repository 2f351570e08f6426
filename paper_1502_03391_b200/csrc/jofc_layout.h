// jofc_layout.h -- HBM layout of the resident problem (shared host/device).
//
// Delta_l is stored as its upper triangle cut into T x T tiles (T = 64):
// tile (I, J), I <= J, of modality l sits at stream index
//     g = l * tpm + band_first(I) + (J - I),   tpm = nT (nT + 1) / 2,
// i.e. modality-major, then tile-row (band) I, then tile-column J.  Each tile
// is 64*64 doubles, COLUMN-major inside the tile (element (il, jl) at
// jl*64 + il) so that the 16 lanes of a warp sharing a column read 128
// contiguous bytes from shared memory.  Inside diagonal tiles only il < jl is
// populated; the rest of the tile and every padding entry (index >= n) is
// 0.0, which the pass kernel relies on.  A shard owns a contiguous range
// [begin, end) of the stream, stored densely from offset 0.
//
// Configurations live as m blocks of n_pad x d (n_pad = 64 nT, padding rows
// 0.0): one tile-column of X is 64*d contiguous doubles, one bulk copy.
#pragma once

#include <cmath>
#include <cstdint>

#ifdef __CUDACC__
#define JOFC_HD __host__ __device__ __forceinline__
#else
#define JOFC_HD inline
#endif

namespace jofc_gpu {

constexpr int kTile = 64;
constexpr int kTileElems = kTile * kTile;
constexpr uint32_t kTileBytes = kTileElems * sizeof(double);

JOFC_HD long long band_first(long long nT, long long I) { return I * nT - I * (I - 1) / 2; }

JOFC_HD long long tiles_per_modality(long long nT) { return nT * (nT + 1) / 2; }

// Stream index -> (l, I, J).
JOFC_HD void tile_coords(long long g, long long nT, long long tpm, int& l, int& I, int& J) {
  l = static_cast<int>(g / tpm);
  const long long r = g - static_cast<long long>(l) * tpm;
  const double b = 2.0 * static_cast<double>(nT) + 1.0;
  long long i = static_cast<long long>((b - sqrt(b * b - 8.0 * static_cast<double>(r))) * 0.5);
  if (i < 0) i = 0;
  while (i > 0 && band_first(nT, i) > r) --i;
  while (i + 1 < nT && band_first(nT, i + 1) <= r) ++i;
  I = static_cast<int>(i);
  J = static_cast<int>(i + (r - band_first(nT, i)));
}

// Advance (l, I, J) to the next tile of the stream.
JOFC_HD void tile_next(int nT, int& l, int& I, int& J) {
  if (++J == nT) {
    if (++I == nT) {
      ++l;
      I = 0;
    }
    J = I;
  }
}

struct Layout {
  int m = 0;
  long long n = 0, n_pad = 0;
  int nT = 0;
  long long tpm = 0;             // tiles per modality
  long long begin = 0, end = 0;  // this shard's stream range
  long long total() const { return static_cast<long long>(m) * tpm; }
  long long local() const { return end - begin; }
};

}  // namespace jofc_gpu
