// jofc_layout.h -- HBM layout of the resident problem (shared host/device).
//
// Delta_l is stored as its upper triangle cut into blocks of 128 rows x 64
// columns.  Row block B covers rows [128B, 128B + 128), column tile J covers
// columns [64J, 64J + 64); block (B, J) exists for J >= 2B, i.e. every
// block that meets the strict upper triangle.  Stream order is modality-
// major, then row block B, then column tile J:
//     g = l * bpm + row_first(B) + (J - 2B),
//     row_first(B) = sum_{b < B} (nT - 2b) = B nT - B (B - 1),
//     bpm = row_first(nB),  nT = ceil(n / 64),  nB = ceil(nT / 2).
// Each block is 128*64 doubles (64 KB), COLUMN-major inside the block
// (element (il, jl) at jl*128 + il): the 16 lanes of a warp sharing a column
// read 128 contiguous bytes from shared memory.  Only entries with
// row < col < n are populated; everything else (the lower part of the two
// diagonal-crossing blocks of each row block, padding beyond n) is 0.0, which
// the pass kernel relies on.  The waste is < 1% at n = 20000.  A shard owns a
// contiguous range [begin, end) of the stream, stored densely from offset 0.
//
// Configurations live as m blocks of n_pad x d with n_pad = 128 nB (padding
// rows 0.0): one column tile of X is 64*d contiguous doubles (one bulk copy),
// one row block 128*d.
#pragma once

#include <cmath>
#include <cstdint>

#ifdef __CUDACC__
#define JOFC_HD __host__ __device__ __forceinline__
#else
#define JOFC_HD inline
#endif

namespace jofc_gpu {

constexpr int kRows = 128;                 // rows per block (one "row block")
constexpr int kCols = 64;                  // columns per block (one "column tile")
constexpr int kBlockElems = kRows * kCols;
constexpr uint32_t kBlockBytes = kBlockElems * sizeof(double);

JOFC_HD long long row_first(long long nT, long long B) { return B * nT - B * (B - 1); }

JOFC_HD long long blocks_per_modality(long long nT) { return row_first(nT, (nT + 1) / 2); }

// Stream index -> (l, B, J).
JOFC_HD void block_coords(long long g, long long nT, long long bpm, int& l, int& B, int& J) {
  l = static_cast<int>(g / bpm);
  const long long r = g - static_cast<long long>(l) * bpm;
  // largest B with row_first(B) <= r:  B^2 - (nT + 1) B + r >= 0 on the small root
  const double b = static_cast<double>(nT) + 1.0;
  double disc = b * b - 4.0 * static_cast<double>(r);
  if (disc < 0.0) disc = 0.0;
  long long i = static_cast<long long>((b - sqrt(disc)) * 0.5);
  const long long nB = (nT + 1) / 2;
  if (i < 0) i = 0;
  if (i > nB - 1) i = nB - 1;
  while (i > 0 && row_first(nT, i) > r) --i;
  while (i + 1 < nB && row_first(nT, i + 1) <= r) ++i;
  B = static_cast<int>(i);
  J = static_cast<int>(2 * i + (r - row_first(nT, i)));
}

// Advance (l, B, J) to the next block of the stream.
JOFC_HD void block_next(int nT, int& l, int& B, int& J) {
  if (++J == nT) {
    if (2 * (++B) >= nT) {
      ++l;
      B = 0;
    }
    J = 2 * B;
  }
}

struct Layout {
  int m = 0;
  long long n = 0, n_pad = 0;
  int nT = 0, nB = 0;
  long long bpm = 0;             // blocks per modality
  long long begin = 0, end = 0;  // this shard's stream range
  long long total() const { return static_cast<long long>(m) * bpm; }
  long long local() const { return end - begin; }
};

}  // namespace jofc_gpu
