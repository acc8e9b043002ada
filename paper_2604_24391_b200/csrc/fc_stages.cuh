// Stand-alone stage operators of the reference API on arbitrary fp64 arrays:
//   sim_freq          migration.py:87-105   amplitude cosine (+ input checks)
//   spectral_entropy  budget.py:34-58       normalised Shannon entropy of |a|^2
//   refresh_mask      edge_refresh.py:62-73 population mean/std threshold
//   topk_ascending    fusion.py:104-115     ascending (E, index) order
// All reductions are deterministic: fixed contiguous chunk per block, fixed
// per-thread order, xor trees, then one block reduces the partials in order.
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#define FC_STAGE_BLOCKS 512
#define FC_STAGE_THREADS 256
#define FC_STAGE_WS_BYTES 65536

namespace stg {

template <int NV>
__device__ __forceinline__ void block_tree(double (&v)[NV], double* sh /* 8*NV */) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NV; ++i) sh[wid * NV + i] = v[i];
  __syncthreads();
  if (threadIdx.x < 32) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double s = lane < nw ? sh[lane * NV + i] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      v[i] = s;
    }
  }
}

__device__ __forceinline__ void chunk_of(int64_t n, int64_t& lo, int64_t& hi) {
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  lo = (int64_t)blockIdx.x * per;
  hi = lo + per < n ? lo + per : n;
}

// cosine partials: sum a*b, a*a, b*b; flags: bit0 non-finite, bit1 negative
__global__ void __launch_bounds__(FC_STAGE_THREADS) k_cos_part(const double* __restrict__ a,
                                                              const double* __restrict__ b, int64_t n,
                                                              double* __restrict__ part, int* __restrict__ flags) {
  __shared__ double sh[8 * 3];
  int64_t lo, hi;
  chunk_of(n, lo, hi);
  double v[3] = {0.0, 0.0, 0.0};
  int f = 0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const double x = a[i], y = b[i];
    if (!(isfinite(x) && isfinite(y))) f |= 1;
    if (x < 0.0 || y < 0.0) f |= 2;
    v[0] = fma(x, y, v[0]);
    v[1] = fma(x, x, v[1]);
    v[2] = fma(y, y, v[2]);
  }
  f = __syncthreads_or(f & 1) | (__syncthreads_or(f & 2) ? 2 : 0);
  block_tree<3>(v, sh);
  if (threadIdx.x == 0) {
    part[blockIdx.x * 3 + 0] = v[0];
    part[blockIdx.x * 3 + 1] = v[1];
    part[blockIdx.x * 3 + 2] = v[2];
    if (f) atomicOr(flags, f);  // integer OR: order-independent
  }
}

// sum of squares (power) with optional DC exclusion
__global__ void __launch_bounds__(FC_STAGE_THREADS) k_pow_part(const double* __restrict__ a, int64_t n,
                                                              int include_dc, double* __restrict__ part,
                                                              int* __restrict__ flags) {
  __shared__ double sh[8];
  int64_t lo, hi;
  chunk_of(n, lo, hi);
  double v[1] = {0.0};
  int f = 0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const double x = a[i];
    if (!isfinite(x)) f |= 1;
    if (x < 0.0) f |= 2;
    if (i == 0 && !include_dc) continue;
    v[0] = fma(x, x, v[0]);
  }
  f = __syncthreads_or(f & 1) | (__syncthreads_or(f & 2) ? 2 : 0);
  block_tree<1>(v, sh);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = v[0];
    if (f) atomicOr(flags, f);
  }
}

// sum of p ln p with p = a^2 / total (xlogy: 0 for p == 0)
__global__ void __launch_bounds__(FC_STAGE_THREADS) k_plogp_part(const double* __restrict__ a, int64_t n,
                                                                int include_dc, const double* __restrict__ total,
                                                                double* __restrict__ part) {
  __shared__ double sh[8];
  int64_t lo, hi;
  chunk_of(n, lo, hi);
  const double tot = *total;
  double v[1] = {0.0};
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    if (i == 0 && !include_dc) continue;
    const double x = a[i];
    const double p = (x * x) / tot;
    if (p > 0.0) v[0] = fma(p, log(p), v[0]);
  }
  block_tree<1>(v, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = v[0];
}

// mean partials / centred second moment partials
__global__ void __launch_bounds__(FC_STAGE_THREADS) k_moment_part(const double* __restrict__ e, int64_t n,
                                                                 const double* __restrict__ mean,
                                                                 double* __restrict__ part) {
  __shared__ double sh[8];
  int64_t lo, hi;
  chunk_of(n, lo, hi);
  // pass 1 (mean == nullptr): sum of (e - e[0]) -- shifting by one element
  // keeps an all-equal array exactly constant (mean exact, std exactly 0);
  // pass 2: sum of (e - mean)^2
  const double mu = mean ? *mean : e[0];
  double v[1] = {0.0};
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const double d = e[i] - mu;
    v[0] = mean ? fma(d, d, v[0]) : v[0] + d;
  }
  block_tree<1>(v, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = v[0];
}

// one block: ordered reduction of nb partial tuples of width NV
// out = shift + sum / div  (shift: optional device scalar)
template <int NV>
__global__ void __launch_bounds__(FC_STAGE_THREADS) k_final(const double* __restrict__ part, int nb,
                                                           double* __restrict__ out, double div,
                                                           const double* __restrict__ shift = nullptr) {
  __shared__ double sh[8 * NV];
  double v[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = 0.0;
  for (int j = threadIdx.x; j < nb; j += blockDim.x)
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] += part[j * NV + i];
  block_tree<NV>(v, sh);
  if (threadIdx.x == 0)
#pragma unroll
    for (int i = 0; i < NV; ++i) out[i] = (shift ? *shift : 0.0) + v[i] / div;
}

__global__ void k_threshold(const double* __restrict__ e, int64_t n, const double* __restrict__ stats,
                            double lam, uint8_t* __restrict__ mask, double* __restrict__ out_stats) {
  // stats: [sum, m2]; out_stats: mean, std, threshold
  const double mu = stats[0], sd = sqrt(stats[1]);
  const double thr = mu + lam * sd;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    out_stats[0] = mu;
    out_stats[1] = sd;
    out_stats[2] = thr;
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    mask[i] = e[i] > thr;
}

// single-CTA bitonic sort of (E[cand], cand) ascending; first k outputs
__global__ void __launch_bounds__(1024) k_topk(const int64_t* __restrict__ cand, int m,
                                               const double* __restrict__ energies, int64_t ne, int64_t k,
                                               int64_t* __restrict__ out, int* __restrict__ flags) {
  extern __shared__ __align__(16) unsigned char smem_t[];
  int np2 = 1;
  while (np2 < m) np2 <<= 1;
  double* ke = reinterpret_cast<double*>(smem_t);
  int64_t* ki = reinterpret_cast<int64_t*>(ke + np2);
  for (int i = threadIdx.x; i < np2; i += blockDim.x) {
    if (i < m) {
      const int64_t c = cand[i];
      if (c < 0 || c >= ne) {
        atomicOr(flags, 4);
        ke[i] = CUDART_INF;
        ki[i] = c;
      } else {
        ke[i] = energies[c];
        ki[i] = c;
      }
    } else {
      ke[i] = CUDART_INF;
      ki[i] = INT64_MAX;
    }
  }
  __syncthreads();
  for (int kk = 2; kk <= np2; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < np2; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const double ea = ke[i], eb = ke[ixj];
          const int64_t ia = ki[i], ib = ki[ixj];
          // NaN energies order after everything (numpy lexsort puts NaN last)
          const bool a_gt_b = (isnan(ea) && !isnan(eb)) || (!isnan(eb) && (ea > eb || (ea == eb && ia > ib))) ||
                              (isnan(ea) && isnan(eb) && ia > ib);
          const bool up = (i & kk) == 0;
          if (up ? a_gt_b : !a_gt_b) {
            ke[i] = eb; ke[ixj] = ea; ki[i] = ib; ki[ixj] = ia;
          }
        }
      }
      __syncthreads();
    }
  }
  const int64_t kout = k < m ? k : m;
  for (int64_t i = threadIdx.x; i < kout; i += blockDim.x) out[i] = ki[i];
}

}  // namespace stg
