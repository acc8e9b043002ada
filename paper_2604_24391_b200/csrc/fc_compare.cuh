// Comparison baselines on the GPU (reference compare.py:23-52): for B frame
// pairs, per patch
//   visual     = cosine of the two patches' raw gray pixels   (compare.py:24-38,90-92)
//   naive_freq = cosine of the patches' |DFT_PxP| amplitudes  (compare.py:50-52,93-95)
// with the reference's rule that a zero-norm pair scores 0.
//
// One CTA per (patch row, chunk of `cpp` patches, stream).  Both stripes are
// staged in shared memory as fp64 gray (the luma adapter for RGB).  The P x P
// DFT is separable and done in fp64 with direct O(P) sums (P <= 32 here; the
// transform is a small fraction of the bytes moved):
//   stage 1: Y[u][x] = sum_y X[y][x] w^{uy}, rows u <= P/2 only — |F| of a
//            real block is symmetric under (u, v) -> (-u, -v), so the other
//            rows repeat rows P-u;
//   stage 2: F[u][v] = sum_x Y[u][x] w^{vx}, then |Fa||Fb|, |Fa|^2, |Fb|^2
//            weighted 1 for u = 0 (and u = P/2, P even), 2 otherwise.
// Every per-item product lands in its own shared slot and each patch sums its
// slots in a fixed order, so results are deterministic.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fc_kernels.cuh"

struct CmpGeom {
  int B, H, W, P, fmt;
  int rows, cols, cpp, nchunk, U;
};

// Shared-memory bytes of k_compare for `cpp` patches per CTA.
inline size_t compare_smem_bytes(int P, int cpp) {
  const int U = P / 2 + 1;
  size_t b = 0;
  b += (size_t)P * 16;                          // twiddles (double2)
  b += (size_t)2 * P * cpp * P * 8;             // gray stripes
  b += (size_t)2 * cpp * U * P * 16;            // stage-1 output (double2)
  b += (size_t)cpp * U * P * 3 * 8;             // stage-2 products
  b += (size_t)cpp * P * 3 * 8;                 // visual partials
  return b;
}

__global__ void __launch_bounds__(256) k_compare(CmpGeom g, const void* __restrict__ prev,
                                                 const void* __restrict__ curr, double* __restrict__ vis_out,
                                                 double* __restrict__ nf_out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int P = g.P, U = g.U, cpp0 = g.cpp;
  const int pr = blockIdx.x / g.nchunk, ch = blockIdx.x - pr * g.nchunk, b = blockIdx.y;
  const int q0 = ch * cpp0;
  const int cpp = min(cpp0, g.cols - q0);
  const int cw = cpp * P;  // stripe width (pixels)
  double2* tw = reinterpret_cast<double2*>(smem);
  double* gy = reinterpret_cast<double*>(tw + P);                    // [2][P][cpp0*P]
  double2* Y = reinterpret_cast<double2*>(gy + 2 * P * cpp0 * P);   // [2][cpp0][U][P]
  double* prod = reinterpret_cast<double*>(Y + 2 * cpp0 * U * P);   // [cpp0][U][P][3]
  double* vpart = prod + (size_t)cpp0 * U * P * 3;                  // [cpp0][P][3]
  const int t = threadIdx.x, nt = blockDim.x;

  for (int m = t; m < P; m += nt) {
    double s, c;
    sincospi(-2.0 * m / P, &s, &c);
    tw[m] = make_double2(c, s);
  }
  // ---- stripes -> fp64 gray
  const size_t fbase = (size_t)b * g.H * g.W;
  for (int i = t; i < 2 * P * cw; i += nt) {
    const int f = i / (P * cw), rem = i - f * (P * cw), y = rem / cw, x = rem - y * cw;
    const size_t pix = fbase + (size_t)(pr * P + y) * g.W + (size_t)q0 * P + x;
    gy[(f * P + y) * (cpp0 * P) + x] = load_gray(f ? curr : prev, g.fmt, pix);
  }
  __syncthreads();
  // ---- visual partials per (patch, row) and DFT stage 1 per (frame, patch, u, x)
  for (int i = t; i < cpp * P; i += nt) {
    const int q = i / P, y = i - q * P;
    const double* a = gy + (0 * P + y) * (cpp0 * P) + q * P;
    const double* c = gy + (1 * P + y) * (cpp0 * P) + q * P;
    double ab = 0.0, aa = 0.0, cc = 0.0;
    for (int x = 0; x < P; ++x) {
      ab = fma(a[x], c[x], ab);
      aa = fma(a[x], a[x], aa);
      cc = fma(c[x], c[x], cc);
    }
    double* o = vpart + (q * P + y) * 3;
    o[0] = ab; o[1] = aa; o[2] = cc;
  }
  for (int i = t; i < 2 * cpp * U * P; i += nt) {
    const int f = i / (cpp * U * P), rem = i - f * (cpp * U * P);
    const int q = rem / (U * P), r2 = rem - q * (U * P), u = r2 / P, x = r2 - u * P;
    const double* col = gy + (size_t)f * P * (cpp0 * P) + q * P + x;
    double re = 0.0, im = 0.0;
    int m = 0;
    for (int y = 0; y < P; ++y) {
      const double v = col[y * (cpp0 * P)];
      re = fma(v, tw[m].x, re);
      im = fma(v, tw[m].y, im);
      m += u;
      if (m >= P) m -= P;
    }
    Y[((f * cpp0 + q) * U + u) * P + x] = make_double2(re, im);
  }
  __syncthreads();
  // ---- stage 2 per (patch, u, v): amplitude products
  for (int i = t; i < cpp * U * P; i += nt) {
    const int q = i / (U * P), rem = i - q * (U * P), u = rem / P, v = rem - u * P;
    const double2* ya = Y + ((0 * cpp0 + q) * U + u) * P;
    const double2* yc = Y + ((1 * cpp0 + q) * U + u) * P;
    double ar = 0.0, ai = 0.0, cr = 0.0, ci = 0.0;
    int m = 0;
    for (int x = 0; x < P; ++x) {
      const double2 w = tw[m];
      ar = fma(ya[x].x, w.x, fma(-ya[x].y, w.y, ar));
      ai = fma(ya[x].x, w.y, fma(ya[x].y, w.x, ai));
      cr = fma(yc[x].x, w.x, fma(-yc[x].y, w.y, cr));
      ci = fma(yc[x].x, w.y, fma(yc[x].y, w.x, ci));
      m += v;
      if (m >= P) m -= P;
    }
    const double pa = ar * ar + ai * ai, pc = cr * cr + ci * ci;
    const double wgt = (u == 0 || 2 * u == P) ? 1.0 : 2.0;
    double* o = prod + ((size_t)(q * U + u) * P + v) * 3;
    o[0] = wgt * (sqrt(pa) * sqrt(pc));
    o[1] = wgt * pa;
    o[2] = wgt * pc;
  }
  __syncthreads();
  // ---- per patch: fixed-order sums, cosines (zero-norm pairs score 0)
  for (int q = t; q < cpp; q += nt) {
    double ab = 0.0, aa = 0.0, cc = 0.0;
    for (int y = 0; y < P; ++y) {
      const double* o = vpart + (q * P + y) * 3;
      ab += o[0]; aa += o[1]; cc += o[2];
    }
    double den = sqrt(aa) * sqrt(cc);
    const size_t oi = (size_t)b * g.rows * g.cols + (size_t)pr * g.cols + q0 + q;
    vis_out[oi] = den > 0.0 ? ab / den : 0.0;
    ab = aa = cc = 0.0;
    for (int k = 0; k < U * P; ++k) {
      const double* o = prod + ((size_t)q * U * P + k) * 3;
      ab += o[0]; aa += o[1]; cc += o[2];
    }
    den = sqrt(aa) * sqrt(cc);
    nf_out[oi] = den > 0.0 ? ab / den : 0.0;
  }
}

// Row-wise cosine of two [n][d] fp64 stacks (compare.py:28-38), for a custom
// token_fn's vectors.  One warp per row, fixed xor-tree order.
__global__ void __launch_bounds__(256) k_row_cosines(int64_t n, int64_t d, const double* __restrict__ a,
                                                     const double* __restrict__ b, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= n) return;
  const double* pa = a + row * d;
  const double* pb = b + row * d;
  double ab = 0.0, aa = 0.0, bb = 0.0;
  for (int64_t k = lane; k < d; k += 32) {
    const double x = pa[k], y = pb[k];
    ab = fma(x, y, ab);
    aa = fma(x, x, aa);
    bb = fma(y, y, bb);
  }
  ab = warp_sum(ab);
  aa = warp_sum(aa);
  bb = warp_sum(bb);
  if (lane == 0) {
    const double den = sqrt(aa) * sqrt(bb);
    out[row] = den > 0.0 ? ab / den : 0.0;
  }
}
