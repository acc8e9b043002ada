// Shared-memory mixed-radix Stockham FFT used by the frame transforms.
//
// Replaces scipy.fft.fft2 / ifft2 on the decision path
// (reference fusion.py:138-139, migration.py:132).  A CTA transforms `ntr`
// independent length-n sequences held in shared memory; element (t, k) lives
// at t*tstride + k*estride.  Each stage of radix R reads R values strided by
// n/R, applies the twiddles w_{pR}^{rk} and an R-point DFT in registers, and
// writes them self-sorted (Stockham autosort), so no digit reversal pass is
// needed and the result is in natural order after the last stage.
//
// Radices 8/4/2/7/5/3 have register butterflies; any other prime factor
// <= FC_MAX_GENERIC_RADIX goes through a direct O(R^2) butterfly (only the
// reference's odd test sizes hit it).  Twiddles come from a table of
// w_n^m = exp(-2*pi*i*m/n), m < n, computed in fp64 on the host and rounded
// once to fp32.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define FC_MAX_STAGES 16
#define FC_MAX_GENERIC_RADIX 61

struct FftPlan {
  int n;
  int nstages;
  int radix[FC_MAX_STAGES];
};

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
// multiply by -i (forward) or +i (inverse)
template <bool INV>
__device__ __forceinline__ float2 rot90(float2 a) {
  return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}

// ----------------------------------------------------------- butterflies --

template <int R, bool INV> struct Dft;

template <bool INV> struct Dft<2, INV> {
  __device__ __forceinline__ static void run(float2* v) {
    float2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  }
};

template <bool INV> struct Dft<4, INV> {
  __device__ __forceinline__ static void run(float2* v) {
    float2 a0 = cadd(v[0], v[2]), a1 = csub(v[0], v[2]);
    float2 a2 = cadd(v[1], v[3]), a3 = rot90<INV>(csub(v[1], v[3]));
    v[0] = cadd(a0, a2);
    v[2] = csub(a0, a2);
    v[1] = cadd(a1, a3);
    v[3] = csub(a1, a3);
  }
};

template <bool INV> struct Dft<8, INV> {
  __device__ __forceinline__ static void run(float2* v) {
    const float c = 0.70710678118654752440f;
    float2 e[4] = {v[0], v[2], v[4], v[6]};
    float2 o[4] = {v[1], v[3], v[5], v[7]};
    Dft<4, INV>::run(e);
    Dft<4, INV>::run(o);
    // w8^1 = (c, -c) fwd / (c, c) inv ; w8^2 = -i / +i ; w8^3 = (-c, -c) / (-c, c)
    float2 o1 = INV ? make_float2(c * (o[1].x - o[1].y), c * (o[1].x + o[1].y))
                    : make_float2(c * (o[1].x + o[1].y), c * (o[1].y - o[1].x));
    float2 o2 = rot90<INV>(o[2]);
    float2 o3 = INV ? make_float2(-c * (o[3].x + o[3].y), c * (o[3].x - o[3].y))
                    : make_float2(c * (o[3].y - o[3].x), -c * (o[3].x + o[3].y));
    v[0] = cadd(e[0], o[0]); v[4] = csub(e[0], o[0]);
    v[1] = cadd(e[1], o1);   v[5] = csub(e[1], o1);
    v[2] = cadd(e[2], o2);   v[6] = csub(e[2], o2);
    v[3] = cadd(e[3], o3);   v[7] = csub(e[3], o3);
  }
};

// Odd prime radix via conjugate-pair symmetry:
//   X[q] = v0 + sum_m t_m cos(2pi mq/R) -/+ i sum_m u_m sin(2pi mq/R)
// with t_m = v_m + v_{R-m}, u_m = v_m - v_{R-m}.
template <int R> struct OddTab;
template <> struct OddTab<3> {
  __device__ __forceinline__ static float c(int k) { return -0.5f; }
  __device__ __forceinline__ static float s(int k) { return 0.86602540378443864676f; }
};
template <> struct OddTab<5> {
  __device__ __forceinline__ static float c(int k) {
    // cos(2pi k/5), k = 1..4
    return (k == 1 || k == 4) ? 0.30901699437494742410f : -0.80901699437494742410f;
  }
  __device__ __forceinline__ static float s(int k) {
    return k == 1 ? 0.95105651629515357212f : k == 2 ? 0.58778525229247312917f
         : k == 3 ? -0.58778525229247312917f : -0.95105651629515357212f;
  }
};
template <> struct OddTab<7> {
  __device__ __forceinline__ static float c(int k) {
    // cos(2pi k/7), k = 1..6
    return (k == 1 || k == 6) ? 0.62348980185873353053f
         : (k == 2 || k == 5) ? -0.22252093395631440429f : -0.90096886790241912624f;
  }
  __device__ __forceinline__ static float s(int k) {
    return k == 1 ? 0.78183148246802980871f : k == 2 ? 0.97492791218182360702f
         : k == 3 ? 0.43388373911755812048f : k == 4 ? -0.43388373911755812048f
         : k == 5 ? -0.97492791218182360702f : -0.78183148246802980871f;
  }
};

template <int R, bool INV> struct DftOdd {
  __device__ __forceinline__ static void run(float2* v) {
    constexpr int H = (R - 1) / 2;
    float2 t[H], u[H];
#pragma unroll
    for (int m = 1; m <= H; ++m) {
      t[m - 1] = cadd(v[m], v[R - m]);
      u[m - 1] = csub(v[m], v[R - m]);
    }
    float2 x0 = v[0];
    float2 s0 = v[0];
#pragma unroll
    for (int m = 0; m < H; ++m) s0 = cadd(s0, t[m]);
#pragma unroll
    for (int q = 1; q <= H; ++q) {
      float2 re = x0, im = make_float2(0.f, 0.f);
#pragma unroll
      for (int m = 1; m <= H; ++m) {
        const int k = (m * q) % R;
        const float cc = OddTab<R>::c(k), ss = OddTab<R>::s(k);
        re.x = fmaf(t[m - 1].x, cc, re.x);
        re.y = fmaf(t[m - 1].y, cc, re.y);
        im.x = fmaf(u[m - 1].x, ss, im.x);
        im.y = fmaf(u[m - 1].y, ss, im.y);
      }
      // forward: X[q] = re - i*im ; X[R-q] = re + i*im
      float2 mi = rot90<INV>(im);  // fwd: -i*im ; inv: +i*im
      v[q] = cadd(re, mi);
      v[R - q] = csub(re, mi);
    }
    v[0] = s0;
  }
};
template <bool INV> struct Dft<3, INV> { __device__ __forceinline__ static void run(float2* v) { DftOdd<3, INV>::run(v); } };
template <bool INV> struct Dft<5, INV> { __device__ __forceinline__ static void run(float2* v) { DftOdd<5, INV>::run(v); } };
template <bool INV> struct Dft<7, INV> { __device__ __forceinline__ static void run(float2* v) { DftOdd<7, INV>::run(v); } };

// ---------------------------------------------------------------- stages --

// One radix-R Stockham stage over ntr transforms.
template <int R, bool INV>
__device__ __forceinline__ void fft_stage(const float2* __restrict__ x, float2* __restrict__ y,
                                          const float2* __restrict__ tw, int n, int p, int ntr,
                                          int tstride, int estride, bool t_fast) {
  const int T = n / R;
  const int twstep = n / (p * R);
  const int ntask = ntr * T;
  for (int task = threadIdx.x; task < ntask; task += blockDim.x) {
    int t, i;
    if (t_fast) { i = task / ntr; t = task - i * ntr; }
    else        { t = task / T;   i = task - t * T; }
    const int k = i % p;
    const float2* xs = x + t * tstride;
    float2* ys = y + t * tstride;
    float2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = xs[(i + r * T) * estride];
    if (p > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) {
        float2 w = tw[r * k * twstep];
        if (INV) w.y = -w.y;
        v[r] = cmul(v[r], w);
      }
    }
    Dft<R, INV>::run(v);
    const int j = (i - k) * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) ys[(j + r * p) * estride] = v[r];
  }
}

// Direct O(R^2) stage for an arbitrary (prime) radix; rare sizes only.
template <bool INV>
__device__ void fft_stage_generic(const float2* __restrict__ x, float2* __restrict__ y,
                                  const float2* __restrict__ tw, int n, int R, int p, int ntr,
                                  int tstride, int estride, bool t_fast) {
  const int T = n / R;
  const int twstep = n / (p * R);  // w_{pR}^{rk} = w_n^{rk*twstep}
  const int rstep = n / R;         // w_R^{m} = w_n^{m*rstep}
  const int ntask = ntr * T * R;   // one output per task
  for (int task = threadIdx.x; task < ntask; task += blockDim.x) {
    int q = task % R;
    int rest = task / R;
    int t, i;
    if (t_fast) { i = rest / ntr; t = rest - i * ntr; }
    else        { t = rest / T;   i = rest - t * T; }
    const int k = i % p;
    const float2* xs = x + t * tstride;
    float2 acc = make_float2(0.f, 0.f);
    for (int m = 0; m < R; ++m) {
      float2 v = xs[(i + m * T) * estride];
      // combined twiddle w_n^{m*k*twstep} * w_n^{m*q*rstep}
      long long e = (long long)m * k * twstep + (long long)m * q * rstep;
      float2 w = tw[(int)(e % n)];
      if (INV) w.y = -w.y;
      acc = cadd(acc, cmul(v, w));
    }
    const int j = (i - k) * R + k;
    y[t * tstride + (j + q * p) * estride] = acc;
  }
}

// Runs all stages; buffers ping-pong between a and b.  Returns the buffer
// holding the result.  Caller must __syncthreads() before (data in a) and
// the function ends with a barrier.
template <bool INV>
__device__ float2* fft_run(float2* a, float2* b, const float2* __restrict__ tw, const FftPlan& pl,
                           int ntr, int tstride, int estride, bool t_fast) {
  int p = 1;
  for (int s = 0; s < pl.nstages; ++s) {
    const int R = pl.radix[s];
    switch (R) {
      case 8: fft_stage<8, INV>(a, b, tw, pl.n, p, ntr, tstride, estride, t_fast); break;
      case 4: fft_stage<4, INV>(a, b, tw, pl.n, p, ntr, tstride, estride, t_fast); break;
      case 2: fft_stage<2, INV>(a, b, tw, pl.n, p, ntr, tstride, estride, t_fast); break;
      case 7: fft_stage<7, INV>(a, b, tw, pl.n, p, ntr, tstride, estride, t_fast); break;
      case 5: fft_stage<5, INV>(a, b, tw, pl.n, p, ntr, tstride, estride, t_fast); break;
      case 3: fft_stage<3, INV>(a, b, tw, pl.n, p, ntr, tstride, estride, t_fast); break;
      default: fft_stage_generic<INV>(a, b, tw, pl.n, R, p, ntr, tstride, estride, t_fast); break;
    }
    __syncthreads();
    float2* tmp = a; a = b; b = tmp;
    p *= R;
  }
  return a;
}

// Compile-time specialisation for the BASELINE sizes: same stages with n, p
// and R as constants so index arithmetic folds.
template <int N, bool INV>
__device__ float2* fft_run_fixed(float2* a, float2* b, const float2* __restrict__ tw, int ntr,
                                 int tstride, int estride, bool t_fast);

template <>
__device__ __forceinline__ float2* fft_run_fixed<448, false>(float2* a, float2* b, const float2* __restrict__ tw,
                                                             int ntr, int ts, int es, bool tf) {
  fft_stage<8, false>(a, b, tw, 448, 1, ntr, ts, es, tf);  __syncthreads();
  fft_stage<8, false>(b, a, tw, 448, 8, ntr, ts, es, tf);  __syncthreads();
  fft_stage<7, false>(a, b, tw, 448, 64, ntr, ts, es, tf); __syncthreads();
  return b;
}
template <>
__device__ __forceinline__ float2* fft_run_fixed<448, true>(float2* a, float2* b, const float2* __restrict__ tw,
                                                            int ntr, int ts, int es, bool tf) {
  fft_stage<8, true>(a, b, tw, 448, 1, ntr, ts, es, tf);  __syncthreads();
  fft_stage<8, true>(b, a, tw, 448, 8, ntr, ts, es, tf);  __syncthreads();
  fft_stage<7, true>(a, b, tw, 448, 64, ntr, ts, es, tf); __syncthreads();
  return b;
}
template <>
__device__ __forceinline__ float2* fft_run_fixed<224, false>(float2* a, float2* b, const float2* __restrict__ tw,
                                                             int ntr, int ts, int es, bool tf) {
  fft_stage<8, false>(a, b, tw, 224, 1, ntr, ts, es, tf);  __syncthreads();
  fft_stage<4, false>(b, a, tw, 224, 8, ntr, ts, es, tf);  __syncthreads();
  fft_stage<7, false>(a, b, tw, 224, 32, ntr, ts, es, tf); __syncthreads();
  return b;
}
template <>
__device__ __forceinline__ float2* fft_run_fixed<224, true>(float2* a, float2* b, const float2* __restrict__ tw,
                                                            int ntr, int ts, int es, bool tf) {
  fft_stage<8, true>(a, b, tw, 224, 1, ntr, ts, es, tf);  __syncthreads();
  fft_stage<4, true>(b, a, tw, 224, 8, ntr, ts, es, tf);  __syncthreads();
  fft_stage<7, true>(a, b, tw, 224, 32, ntr, ts, es, tf); __syncthreads();
  return b;
}

// Dispatch: N > 0 selects the fixed-size path, N == 0 the runtime plan.
template <int N, bool INV>
__device__ __forceinline__ float2* fft_any(float2* a, float2* b, const float2* __restrict__ tw,
                                          const FftPlan& pl, int ntr, int ts, int es, bool tf) {
  if constexpr (N > 0) return fft_run_fixed<N, INV>(a, b, tw, ntr, ts, es, tf);
  else return fft_run<INV>(a, b, tw, pl, ntr, ts, es, tf);
}
