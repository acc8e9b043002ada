// fp64 spectral operators behind the reference's public transform wrappers
// (spectral.py:24-72) and phase_correlation_spectra (migration.py:128-134).
// They are not on the batched decision path (which runs the fp32 packed
// FFTs of fc_fast448*.cuh / fc_kernels.cuh); they exist so the drop-in
// facade answers the reference's own transform API — and its test corpus,
// which pins these functions against naive DFT/DCT oracles at 1e-9 — on the
// GPU, in fp64:
//
//   k_dft_rows / k_dft_cols  2-D DFT of an H x W grid as two dense passes
//                            with an exact fp64 twiddle table (angle reduced
//                            to (k m) mod n before sincospi), TK outputs per
//                            thread in the column pass; forward unnormalised,
//                            inverse scaled by 1 / (H W) (scipy.fft.fft2 /
//                            ifft2 conventions)
//   k_cross_power            C = A conj(B) / (|A conj(B)| + eps)
//   k_peak_part / k_peak_fin argmax of a real response with the reference's
//                            exact tie rule (value desc, |di| + |dj| asc,
//                            row-major position asc; migration.py:141-159)
//   k_block_dct              orthonormal 2-D DCT-II of square patches
//   k_amp_phase              |z| and atan2(Im z, Re z)
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>

namespace spec {

constexpr int kThreads = 256;
constexpr int kTK = 8;  // column-pass outputs per thread

// exp(sign * 2 pi i k / n) for k in [0, n)
__global__ void k_twiddles(int n, int sign, double2* __restrict__ tw) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    double s, c;
    sincospi(2.0 * (double)k / (double)n, &s, &c);
    tw[k] = make_double2(c, sign * s);
  }
}

// Row pass: Y[m][l] = sum_n X[m][n] w_W^(l n).  One CTA per (row, l-block);
// the row and the twiddle table are staged in shared memory.
__global__ void __launch_bounds__(kThreads) k_dft_rows(int H, int W, const double* __restrict__ in, int in_complex,
                                                       const double2* __restrict__ twW, double2* __restrict__ Y) {
  extern __shared__ __align__(16) unsigned char smem[];
  double2* row = reinterpret_cast<double2*>(smem);
  double2* tw = row + W;
  const int m = blockIdx.y;
  for (int n = threadIdx.x; n < W; n += blockDim.x) {
    const size_t i = (size_t)m * W + n;
    row[n] = in_complex ? make_double2(in[2 * i], in[2 * i + 1]) : make_double2(in[i], 0.0);
    tw[n] = twW[n];
  }
  __syncthreads();
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= W) return;
  double re = 0.0, im = 0.0;
  int idx = 0;
  for (int n = 0; n < W; ++n) {
    const double2 x = row[n], w = tw[idx];
    re = fma(x.x, w.x, fma(-x.y, w.y, re));
    im = fma(x.x, w.y, fma(x.y, w.x, im));
    idx += l;
    if (idx >= W) idx -= W;
  }
  Y[(size_t)m * W + l] = make_double2(re, im);
}

// Column pass: Z[k][l] = scale * sum_m Y[m][l] w_H^(k m); thread = column l,
// kTK consecutive k per thread (Y read once per kTK outputs), coalesced in l.
__global__ void __launch_bounds__(kThreads) k_dft_cols(int H, int W, const double2* __restrict__ Y,
                                                       const double2* __restrict__ twH, double scale,
                                                       double* __restrict__ out) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  const int k0 = blockIdx.y * kTK;
  if (l >= W) return;
  double re[kTK], im[kTK];
  int idx[kTK], step[kTK];
#pragma unroll
  for (int t = 0; t < kTK; ++t) {
    re[t] = 0.0;
    im[t] = 0.0;
    idx[t] = 0;
    step[t] = (k0 + t) % H;
  }
  for (int m = 0; m < H; ++m) {
    const double2 y = Y[(size_t)m * W + l];
#pragma unroll
    for (int t = 0; t < kTK; ++t) {
      const double2 w = twH[idx[t]];
      re[t] = fma(y.x, w.x, fma(-y.y, w.y, re[t]));
      im[t] = fma(y.x, w.y, fma(y.y, w.x, im[t]));
      idx[t] += step[t];
      if (idx[t] >= H) idx[t] -= H;
    }
  }
#pragma unroll
  for (int t = 0; t < kTK; ++t) {
    const int k = k0 + t;
    if (k < H) {
      const size_t o = ((size_t)k * W + l) * 2;
      out[o] = re[t] * scale;
      out[o + 1] = im[t] * scale;
    }
  }
}

// migration.py:130-131: cross = a * conj(b); cross /= |cross| + eps
__global__ void k_cross_power(int64_t n, const double* __restrict__ a, const double* __restrict__ b, double eps,
                              double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double ar = a[2 * i], ai = a[2 * i + 1], br = b[2 * i], bi = b[2 * i + 1];
    const double cr = ar * br + ai * bi;
    const double ci = ai * br - ar * bi;
    const double d = hypot(cr, ci) + eps;
    out[2 * i] = cr / d;
    out[2 * i + 1] = ci / d;
  }
}

struct PeakD {
  double v;
  int l1;
  int pos;
};

// displacement of an impulse at p along an axis of n: (-p) mod n, canonical
__device__ __forceinline__ int canon_neg(int p, int n) {
  const int d = (n - p) % n;
  return 2 * d >= n ? d - n : d;
}

__device__ __forceinline__ bool peak_before(const PeakD& a, const PeakD& b) {
  if (a.v != b.v) return a.v > b.v;
  if (a.l1 != b.l1) return a.l1 < b.l1;
  return a.pos < b.pos;
}

__device__ __forceinline__ PeakD peak_shfl(const PeakD& p, int o) {
  PeakD q;
  q.v = __shfl_xor_sync(0xffffffffu, p.v, o);
  q.l1 = __shfl_xor_sync(0xffffffffu, p.l1, o);
  q.pos = __shfl_xor_sync(0xffffffffu, p.pos, o);
  return q;
}

__device__ PeakD block_peak(PeakD best) {
  __shared__ PeakD sh[32];
  for (int o = 16; o > 0; o >>= 1) {
    const PeakD q = peak_shfl(best, o);
    if (peak_before(q, best)) best = q;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0) sh[wid] = best;
  __syncthreads();
  if (wid == 0) {
    best = lane < nw ? sh[lane] : PeakD{-CUDART_INF, 0x7fffffff, 0x7fffffff};
    for (int o = 16; o > 0; o >>= 1) {
      const PeakD q = peak_shfl(best, o);
      if (peak_before(q, best)) best = q;
    }
  }
  return best;
}

// response = real parts of an interleaved complex grid; partial per CTA
__global__ void __launch_bounds__(kThreads) k_peak_part(int H, int W, const double* __restrict__ resp,
                                                        PeakD* __restrict__ part) {
  PeakD best = {-CUDART_INF, 0x7fffffff, 0x7fffffff};
  const int64_t n = (int64_t)H * W;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int pi = (int)(i / W), pj = (int)(i - (int64_t)pi * W);
    const PeakD c = {resp[2 * i], abs(canon_neg(pi, H)) + abs(canon_neg(pj, W)), (int)i};
    if (peak_before(c, best)) best = c;
  }
  best = block_peak(best);
  if (threadIdx.x == 0) part[blockIdx.x] = best;
}

// out2 = (di, dj) of the winning peak
__global__ void __launch_bounds__(kThreads) k_peak_fin(int H, int W, const PeakD* __restrict__ part, int nparts,
                                                       int32_t* __restrict__ out2) {
  PeakD best = {-CUDART_INF, 0x7fffffff, 0x7fffffff};
  for (int i = threadIdx.x; i < nparts; i += blockDim.x)
    if (peak_before(part[i], best)) best = part[i];
  best = block_peak(best);
  if (threadIdx.x == 0) {
    out2[0] = canon_neg(best.pos / W, H);
    out2[1] = canon_neg(best.pos % W, W);
  }
}

// Orthonormal 2-D DCT-II of n square P x P patches (scipy.fft.dctn norm=ortho):
// T[u][y] = sum_x C[u][x] X[x][y]; out[u][v] = sum_y T[u][y] C[v][y],
// C[u][x] = s_u cos(pi u (2x + 1) / (2P)), s_0 = sqrt(1/P), s_u = sqrt(2/P).
__global__ void __launch_bounds__(kThreads) k_block_dct(int P, const double* __restrict__ in, double* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* X = reinterpret_cast<double*>(smem);
  double* Cm = X + P * P;
  double* T = Cm + P * P;
  const size_t base = (size_t)blockIdx.x * P * P;
  for (int i = threadIdx.x; i < P * P; i += blockDim.x) {
    X[i] = in[base + i];
    const int u = i / P, x = i - u * P;
    const double s = u == 0 ? sqrt(1.0 / P) : sqrt(2.0 / P);
    Cm[i] = s * cospi((double)(u * (2 * x + 1)) / (double)(2 * P));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < P * P; i += blockDim.x) {
    const int u = i / P, y = i - u * P;
    double acc = 0.0;
    for (int x = 0; x < P; ++x) acc = fma(Cm[u * P + x], X[x * P + y], acc);
    T[i] = acc;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < P * P; i += blockDim.x) {
    const int u = i / P, v = i - u * P;
    double acc = 0.0;
    for (int y = 0; y < P; ++y) acc = fma(T[u * P + y], Cm[v * P + y], acc);
    out[base + i] = acc;
  }
}

__global__ void k_amp_phase(int64_t n, const double* __restrict__ z, double* __restrict__ amp,
                            double* __restrict__ phase) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double re = z[2 * i], im = z[2 * i + 1];
    amp[i] = hypot(re, im);
    phase[i] = atan2(im, re);
  }
}

}  // namespace spec
