// Warp-owned 448-point FFTs: one warp runs one whole transform, so the data
// exchanges between radix stages need only __syncwarp, never a CTA barrier.
//
// 448 = 7 * 64, 64 = 8 * 8.  Forward (natural order in, permuted out):
//   stage 1  role n2 in [0,64): A[n2][k1] = DFT7_{n1}(x[64 n1 + n2]) * w448^{n2 k1}
//   stage 2  role (k1, m2):     B[k1][m2][j1] = DFT8_{m1}(A[8 m1 + m2][k1])
//   stage 3  role (k1, j1):     X[k1 + 7 j1 + 56 j2] = DFT8_{m2}(B[k1][m2][j1] * w64^{m2 j1})
// so role g < 56 ends holding X[k1 + 7 j1 + 56 j2], j2 = 0..7, (k1, j1) = (g/8, g%8).
// The inverse runs the same stages transposed (permuted in, natural out) with
// conjugate twiddles, so a forward -> pointwise -> inverse chain never
// reorders.  The 64 roles of a transform are folded onto the 32 lanes of one
// warp: lane l plays roles r = l and r = l + 32 ("halves" h = 0, 1).  Radix-8
// stages have 56 groups; half 1 is active on lanes < 24.
//   forward:  in  a[h][n1] = x[64 n1 + l + 32 h]          (all lanes, both halves)
//             out b[h][j2] = X[k1 + 7 j1 + 56 j2], g = l + 32 h < 56, (k1, j1) = (g >> 3, g & 7)
//   inverse (transposed stages, conjugate twiddles): the reverse mapping.
// Per-warp scratch S: 7 x 72 float2 (504); every access pattern below is
// bank-conflict free for 8-byte accesses per half-warp (k1 rows 72 apart
// put k1 and k1+1 16 banks apart; the j1 stride 9 spreads a column).
#pragma once
#include "fc_fft.cuh"

namespace w448 {

constexpr int XS = 504;  // scratch float2 per warp

// Twiddles of one lane: w1[h][k1-1] = w448^{(l + 32h) k1}, w3[m2-1] = w64^{m2 (l & 7)}.
struct Tw {
  float2 w1_[2][6];
  float2 w3_[7];
  __device__ __forceinline__ void load(const float2* __restrict__ t448, const float2* __restrict__ t64, int lane) {
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int k1 = 1; k1 < 7; ++k1) w1_[h][k1 - 1] = __ldg(t448 + (k1 - 1) * 64 + lane + 32 * h);
#pragma unroll
    for (int m2 = 1; m2 < 8; ++m2) w3_[m2 - 1] = __ldg(t64 + (m2 - 1) * 8 + (lane & 7));
  }
  __device__ __forceinline__ float2 w1(int h, int k1) const { return w1_[h][k1 - 1]; }
  __device__ __forceinline__ float2 w3(int m2) const { return w3_[m2 - 1]; }
};

// Same twiddles read at their point of use (fewer live registers).
struct TwLazy {
  const float2* __restrict__ t448;
  const float2* __restrict__ t64;
  int lane;
  __device__ __forceinline__ void load(const float2* __restrict__ a, const float2* __restrict__ b, int l) {
    t448 = a; t64 = b; lane = l;
  }
  __device__ __forceinline__ float2 w1(int h, int k1) const { return __ldg(t448 + (k1 - 1) * 64 + lane + 32 * h); }
  __device__ __forceinline__ float2 w3(int m2) const { return __ldg(t64 + (m2 - 1) * 8 + (lane & 7)); }
};

template <bool INV>
__device__ __forceinline__ float2 tmul(float2 v, float2 w) {
  return INV ? cmul(v, make_float2(w.x, -w.y)) : cmul(v, w);
}

// Forward-ordered transform (natural in, permuted out).  S must be free on
// entry (the caller __syncwarp()s after its own last use).
template <bool INV, class TW>
__device__ __forceinline__ void fwd(float2 (&a)[2][7], float2 (&b)[2][8], float2* S, int lane, const TW& tw) {
  const int k1a = lane >> 3, lo = lane & 7;
  const bool h1 = lane < 24;  // half 1 active in the radix-8 stages
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    DftOdd<7, INV>::run(a[h]);
#pragma unroll
    for (int k1 = 1; k1 < 7; ++k1) a[h][k1] = tmul<INV>(a[h][k1], tw.w1(h, k1));
#pragma unroll
    for (int k1 = 0; k1 < 7; ++k1) S[k1 * 72 + lane + 32 * h] = a[h][k1];
  }
  __syncwarp();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (h == 0 || h1) {
      const int k1 = k1a + 4 * h;
#pragma unroll
      for (int m1 = 0; m1 < 8; ++m1) b[h][m1] = S[k1 * 72 + 8 * m1 + lo];
    }
  }
  __syncwarp();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (h == 0 || h1) {
      const int k1 = k1a + 4 * h;
      Dft<8, INV>::run(b[h]);
#pragma unroll
      for (int j1 = 0; j1 < 8; ++j1) S[k1 * 72 + 9 * j1 + lo] = b[h][j1];
    }
  }
  __syncwarp();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (h == 0 || h1) {
      const int k1 = k1a + 4 * h;
#pragma unroll
      for (int m2 = 0; m2 < 8; ++m2) b[h][m2] = S[k1 * 72 + 9 * lo + m2];
#pragma unroll
      for (int m2 = 1; m2 < 8; ++m2) b[h][m2] = tmul<INV>(b[h][m2], tw.w3(m2));
      Dft<8, INV>::run(b[h]);
    }
  }
}

// Transposed transform (permuted in, natural out).  S must be free on entry.
template <bool INV, class TW>
__device__ __forceinline__ void inv(float2 (&b)[2][8], float2 (&a)[2][7], float2* S, int lane, const TW& tw) {
  const int k1a = lane >> 3, lo = lane & 7;
  const bool h1 = lane < 24;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (h == 0 || h1) {
      const int k1 = k1a + 4 * h;
      Dft<8, INV>::run(b[h]);  // over j2 -> m2
#pragma unroll
      for (int m2 = 1; m2 < 8; ++m2) b[h][m2] = tmul<INV>(b[h][m2], tw.w3(m2));
#pragma unroll
      for (int m2 = 0; m2 < 8; ++m2) S[k1 * 72 + 9 * lo + m2] = b[h][m2];
    }
  }
  __syncwarp();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (h == 0 || h1) {
      const int k1 = k1a + 4 * h;
#pragma unroll
      for (int j1 = 0; j1 < 8; ++j1) b[h][j1] = S[k1 * 72 + 9 * j1 + lo];
    }
  }
  __syncwarp();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (h == 0 || h1) {
      const int k1 = k1a + 4 * h;
      Dft<8, INV>::run(b[h]);  // over j1 -> m1
#pragma unroll
      for (int m1 = 0; m1 < 8; ++m1) S[k1 * 72 + 8 * m1 + lo] = b[h][m1];
    }
  }
  __syncwarp();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
#pragma unroll
    for (int q = 0; q < 7; ++q) a[h][q] = S[q * 72 + lane + 32 * h];
#pragma unroll
    for (int q = 1; q < 7; ++q) a[h][q] = tmul<INV>(a[h][q], tw.w1(h, q));
    DftOdd<7, INV>::run(a[h]);  // over k1 -> n1
  }
}

}  // namespace w448
