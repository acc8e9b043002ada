// Kernels of the B200 FreqCache select + splice path.
//
//   K_A  k_rows_fwd   frame stripe (P rows) -> fp64 luma, validity flags,
//                     high-pass block-DCT energy of every patch in the stripe,
//                     packed real row FFTs -> half-spectrum rows in T.
//   K_B  k_cols       one block of CB packed spectrum columns: forward column
//                     FFT (-> current spectrum, swapped with the previous one
//                     held in the per-stream state), amplitude/entropy sums,
//                     normalised cross-power, inverse column FFT -> T.
//   K_C  k_rows_inv   RG rows of T: packed complex-to-real inverse row FFT,
//                     phase-correlation argmax with the reference tie rule.
//   K_D1 k_rank       one CTA per stream, beside K_B / K_C: energy mean / std,
//                     refresh mask, the ascending (E, index) order of every
//                     token (register + shared-memory bitonic network).
//   K_D  k_select     one CTA per stream: reductions, gate, displacement,
//                     alignment, budget, the first K_final candidates of
//                     K_D1's order (one prefix scan), recompute order, splice
//                     map, outputs, run_sequence counters.
//   K_E  k_splice*    bf16 (any dtype) hidden-state gather/scatter + ages;
//                     k_splice_plan + k_splice_ip_bulk: the in-place TMA form.
// (These are the generic-geometry kernels plus the shared K_D1 / K_D / K_E;
// the 448 x 448 / P 14 forms of K_A / K_B / K_C are in fc_fast448*.cuh.)
//
// Reference semantics cited per kernel; the layout of T / state is private:
// [B][NCB][H][CB] float2, CB packed columns per block, where packed column 0
// holds DC (real part) and Nyquist (imag part) of each row's half spectrum.
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "fc_fft.cuh"
#include "fc_tma.cuh"
#include "../../include/freqcache_b200.h"

#define FC_CB 8
#define FC_THREADS 256
#define FC_SEL_THREADS 256
#define FC_MAX_TOKENS 4096
#define FC_MAX_PATCH 32

// Per-stripe frame flags.  A frame is constant iff no stripe varies and all
// stripes share `ref`; it is all-zero iff constant with ref == 0
// (fusion.py:147 np.ptp == 0; migration.py:103 zero norm).
struct StripeStat {
  double ref;         // one pixel value of the stripe
  double unused;
  int32_t nonfinite;  // any pixel NaN/Inf (frame.py:13)
  int32_t varying;    // some pixel differs from ref
  int32_t pad[2];
};

struct PeakPart {
  float v, v2;
  int32_t y, j;
};

struct StreamHdr {
  int32_t valid;
  int32_t prev_zero;
  int32_t prev_const;
  int32_t steps;
};

struct KParams {
  int B, H, W, P, fmt;
  int rows, cols, N, cut;
  int Wc, Wcp, NCB;
  int npairA, RG, NRG;
  FftPlan planW, planH;
  const float2* twW;
  const float2* twH;
  const double* dct;  // [cut][P] orthonormal DCT-II rows u < cut
  const float2* tw448;  // fast path: w448^{n2 k1}, [6][64]
  const float2* tw64;   // fast path: w64^{m2 j1},  [7][8]
  float2* T;
  float2* T2;           // fast path: inverse-column output, [chunk][448][224]
  StripeStat* stripes;
  double* stats;  // [B][NCB][4]
  PeakPart* peaks;
  double* energy;  // [B][N]
  StreamHdr* hdr;
  float2* spec;
  int16_t* order;   // [B][N] all tokens ascending (E, index) (K_D1 -> K_D)
  uint8_t* freshm;  // [B][N] refresh mask (K_D1 -> K_D)
  double* estats;   // [B][4] mean, std, threshold, refresh count (K_D1 -> K_D)
  int* flow;        // fast path, K_B + K_C flow kernel: tickets and per-stream counters
};

// --------------------------------------------------------------- helpers --

__device__ __forceinline__ double luma_f64(float r, float g, float b) {
  // (0.299*R + 0.587*G) + 0.114*B, no contraction (frameio.py:26,85-88)
  return __dadd_rn(__dadd_rn(__dmul_rn(0.299, (double)r), __dmul_rn(0.587, (double)g)),
                   __dmul_rn(0.114, (double)b));
}

// 8-bit netpbm pixels -> the reference's gray values: v / 255 (P5) and
// ((0.299 R + 0.587 G) + 0.114 B) / 255 (P6), fp64, correctly rounded
// (frameio.py:81-88).
__device__ __forceinline__ double gray_u8(unsigned v) { return __ddiv_rn((double)v, 255.0); }
__device__ __forceinline__ double luma_u8(unsigned r, unsigned g, unsigned b) {
  return __ddiv_rn(luma_f64((float)r, (float)g, (float)b), 255.0);
}

// Gray value of pixel i of a frame in any FC_FMT_* layout.
__device__ __forceinline__ double load_gray(const void* f, int fmt, size_t i) {
  switch (fmt) {
    case FC_FMT_RGB_F32: {
      const float* p = reinterpret_cast<const float*>(f) + 3 * i;
      return luma_f64(p[0], p[1], p[2]);
    }
    case FC_FMT_GRAY_F32: return (double)reinterpret_cast<const float*>(f)[i];
    case FC_FMT_GRAY_U8: return gray_u8(reinterpret_cast<const uint8_t*>(f)[i]);
    case FC_FMT_RGB_U8: {
      const uint8_t* p = reinterpret_cast<const uint8_t*>(f) + 3 * i;
      return luma_u8(p[0], p[1], p[2]);
    }
    default: return reinterpret_cast<const double*>(f)[i];
  }
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum of NV doubles; result valid in thread 0.  Warp
// xor-trees, then warp 0 reduces the per-warp partials with another fixed
// tree (no serial tail).  SYNC_AFTER: trailing barrier (scratch reuse).
template <int NV, bool SYNC_AFTER = true>
__device__ __forceinline__ void block_sum_d(double (&v)[NV], double* scratch /* 32*NV */) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = warp_sum(v[i]);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NV; ++i) scratch[wid * NV + i] = v[i];
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double s = lane < nw ? scratch[lane * NV + i] : 0.0;
      v[i] = warp_sum(s);
    }
  }
  if (SYNC_AFTER) __syncthreads();
}

// fp32 per-thread partials -> fp32 warp trees -> fp64 across warps.
template <int NV>
__device__ __forceinline__ void block_sum_f2d(const float (&f)[NV], double (&v)[NV], double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  float w[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) w[i] = warp_sum(f[i]);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NV; ++i) scratch[wid * NV + i] = (double)w[i];
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double s = lane < nw ? scratch[lane * NV + i] : 0.0;
      v[i] = warp_sum(s);
    }
  }
}

__device__ __forceinline__ int canon_disp(int pos, int n) {
  int d = (n - pos) % n;  // (-pos) mod n
  return (2 * d >= n) ? d - n : d;
}

__device__ __forceinline__ int to_patch_units(int d, int p) {
  int a = d >= 0 ? d : -d;
  int q = (2 * a + p - 1) / (2 * p);
  return d >= 0 ? q : -q;
}

// ----------------------------------------------------------------- K_A ----

// High-pass energy of the patches of one stripe (edge_refresh.py:48-59).
// E = sum(X'^2) - sum_{u,v<c} Y'[u][v]^2 with X' = X - mean(X): Parseval for
// the orthonormal DCT-II; removing the mean only changes Y[0][0], which is in
// the discarded corner.  fp64 throughout.  One lane per patch column; P<=16
// puts two patches in a warp (half-warp segments).
__device__ void stripe_energy(const double* __restrict__ g, const double* __restrict__ dctc,
                              const KParams& kp, int b, int s, double* __restrict__ energy) {
  const int P = kp.P, W = kp.W, cut = kp.cut, cols = kp.cols;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int seg = (P <= 16) ? 16 : 32;
  const int per_warp = 32 / seg;
  const int sub = lane / seg, y = lane % seg;
  const bool act_lane = y < P;
  for (int base = wid * per_warp; base < cols; base += nw * per_warp) {
    const int pp = base + sub;
    const bool act = act_lane && pp < cols;
    const double* col = g + pp * P + y;
    double cs = 0.0;
    if (act)
      for (int x = 0; x < P; ++x) cs += col[x * W];
    for (int o = seg >> 1; o > 0; o >>= 1) cs += __shfl_xor_sync(0xffffffffu, cs, o, seg);
    const double m = cs / (double)(P * P);
    double sq = 0.0;
    double t[FC_MAX_PATCH / 4];
#pragma unroll
    for (int u = 0; u < FC_MAX_PATCH / 4; ++u) t[u] = 0.0;
    if (act) {
      for (int x = 0; x < P; ++x) {
        const double d = col[x * W] - m;
        sq = fma(d, d, sq);
#pragma unroll
        for (int u = 0; u < FC_MAX_PATCH / 4; ++u)
          if (u < cut) t[u] = fma(dctc[u * P + x], d, t[u]);
      }
    }
    for (int o = seg >> 1; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o, seg);
    double low = 0.0;
#pragma unroll
    for (int u = 0; u < FC_MAX_PATCH / 4; ++u) {
      if (u >= cut) break;
      for (int v = 0; v < cut; ++v) {
        double yv = act ? t[u] * dctc[v * P + y] : 0.0;
        for (int o = seg >> 1; o > 0; o >>= 1) yv += __shfl_xor_sync(0xffffffffu, yv, o, seg);
        low = fma(yv, yv, low);
      }
    }
    if (act && y == 0) {
      double e = sq - low;
      energy[(size_t)b * kp.N + (size_t)s * cols + pp] = e > 0.0 ? e : 0.0;
    }
  }
}

template <int NW>
__global__ void __launch_bounds__(FC_THREADS) k_rows_fwd(KParams kp, const void* __restrict__ frames,
                                                         int do_fft) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ double red[32 * 3];
  const int s = blockIdx.x, b = blockIdx.y;
  const int P = kp.P, W = kp.W, H = kp.H;
  const int npx = P * W;
  double* g = reinterpret_cast<double*>(smem);
  float2* bufA = reinterpret_cast<float2*>(g + npx);
  float2* tw = bufA + kp.npairA * W;
  double* dctc = reinterpret_cast<double*>(tw + W);

  for (int i = threadIdx.x; i < W; i += blockDim.x) tw[i] = kp.twW[i];
  for (int i = threadIdx.x; i < kp.cut * P; i += blockDim.x) dctc[i] = kp.dct[i];

  // frame stripe -> fp64 gray (frame.py:6-15 validation flags, luma adapter)
  const size_t base = ((size_t)b * H + (size_t)s * P) * (size_t)W;
  double mn = CUDART_INF, mx = -CUDART_INF, bad = 0.0;
  if (kp.fmt == FC_FMT_RGB_F32) {
    const float* f = reinterpret_cast<const float*>(frames) + base * 3;
    if ((npx & 3) == 0 && ((reinterpret_cast<uintptr_t>(f) & 15) == 0)) {
      const float4* f4 = reinterpret_cast<const float4*>(f);
      for (int q = threadIdx.x; q < npx / 4; q += blockDim.x) {
        const float4 a = __ldcs(f4 + 3 * q), c = __ldcs(f4 + 3 * q + 1), d = __ldcs(f4 + 3 * q + 2);
        const double v0 = luma_f64(a.x, a.y, a.z), v1 = luma_f64(a.w, c.x, c.y);
        const double v2 = luma_f64(c.z, c.w, d.x), v3 = luma_f64(d.y, d.z, d.w);
        g[4 * q] = v0; g[4 * q + 1] = v1; g[4 * q + 2] = v2; g[4 * q + 3] = v3;
        mn = fmin(fmin(mn, v0), fmin(fmin(v1, v2), v3));
        mx = fmax(fmax(mx, v0), fmax(fmax(v1, v2), v3));
        if (!(isfinite(v0) && isfinite(v1) && isfinite(v2) && isfinite(v3))) bad = 1.0;
      }
    } else {
      for (int px = threadIdx.x; px < npx; px += blockDim.x) {
        const double v = luma_f64(f[3 * px], f[3 * px + 1], f[3 * px + 2]);
        g[px] = v;
        mn = fmin(mn, v); mx = fmax(mx, v);
        if (!isfinite(v)) bad = 1.0;
      }
    }
  } else if (kp.fmt == FC_FMT_GRAY_U8 || kp.fmt == FC_FMT_RGB_U8) {
    for (int px = threadIdx.x; px < npx; px += blockDim.x) {
      const double v = load_gray(frames, kp.fmt, base + px);
      g[px] = v;
      mn = fmin(mn, v); mx = fmax(mx, v);
    }
  } else if (kp.fmt == FC_FMT_GRAY_F32) {
    const float* f = reinterpret_cast<const float*>(frames) + base;
    for (int px = threadIdx.x; px < npx; px += blockDim.x) {
      const double v = (double)f[px];
      g[px] = v;
      mn = fmin(mn, v); mx = fmax(mx, v);
      if (!isfinite(v)) bad = 1.0;
    }
  } else {
    const double* f = reinterpret_cast<const double*>(frames) + base;
    for (int px = threadIdx.x; px < npx; px += blockDim.x) {
      const double v = f[px];
      g[px] = v;
      mn = fmin(mn, v); mx = fmax(mx, v);
      if (!isfinite(v)) bad = 1.0;
    }
  }
  {
    // min / max / flag: exact, order-independent
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      bad = fmax(bad, __shfl_xor_sync(0xffffffffu, bad, o));
    }
    if (lane == 0) { red[wid * 3] = mn; red[wid * 3 + 1] = mx; red[wid * 3 + 2] = bad; }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < nw; ++w) {
        mn = fmin(mn, red[w * 3]); mx = fmax(mx, red[w * 3 + 1]); bad = fmax(bad, red[w * 3 + 2]);
      }
      StripeStat st;
      st.ref = mn; st.unused = mx; st.nonfinite = bad != 0.0; st.varying = mn != mx;
      st.pad[0] = st.pad[1] = 0;
      kp.stripes[(size_t)b * kp.rows + s] = st;
    }
  }
  __syncthreads();

  stripe_energy(g, dctc, kp, b, s, kp.energy);
  if (!do_fft) return;

  // pack row pairs as complex sequences: z = x_{2t} + i x_{2t+1}
  const int npair = kp.npairA;
  for (int idx = threadIdx.x; idx < npair * W; idx += blockDim.x) {
    const int t = idx / W, k = idx - t * W;
    const float re = (float)g[(2 * t) * W + k];
    const float im = (2 * t + 1 < P) ? (float)g[(2 * t + 1) * W + k] : 0.f;
    bufA[idx] = make_float2(re, im);
  }
  __syncthreads();
  float2* res = fft_any<NW, false>(bufA, reinterpret_cast<float2*>(g), tw, kp.planW, npair, W, 1, false);

  // split the two real rows' spectra and write packed half-spectrum columns
  const int Wc = kp.Wc, Wcp = kp.Wcp;
  const bool weven = (W & 1) == 0;
  for (int idx = threadIdx.x; idx < npair * Wcp; idx += blockDim.x) {
    const int t = idx / Wcp, q = idx - t * Wcp;
    const int ra = s * P + 2 * t;
    const bool hasb = 2 * t + 1 < P;
    float2 xa, xb;
    const float2* Z = res + t * W;
    if (q >= Wc) {
      xa = xb = make_float2(0.f, 0.f);
    } else if (q == 0) {
      const float2 z0 = Z[0];
      const float2 zn = weven ? Z[W / 2] : make_float2(0.f, 0.f);
      xa = make_float2(z0.x, zn.x);  // DC_a + i Nyq_a
      xb = make_float2(z0.y, zn.y);  // DC_b + i Nyq_b
    } else {
      const float2 za = Z[q], zm = Z[W - q];
      // X_a = (Z[q] + conj Z[-q]) / 2 ; X_b = -i (Z[q] - conj Z[-q]) / 2
      xa = make_float2(0.5f * (za.x + zm.x), 0.5f * (za.y - zm.y));
      xb = make_float2(0.5f * (za.y + zm.y), -0.5f * (za.x - zm.x));
    }
    float2* dst = kp.T + (((size_t)b * kp.NCB + q / FC_CB) * H + ra) * FC_CB + (q % FC_CB);
    dst[0] = xa;
    if (hasb) dst[FC_CB] = xb;
  }
}

// ----------------------------------------------------------------- K_B ----

struct SpecSums {
  double pc, pp, cc, plp;
};

__device__ __forceinline__ void acc_bin(SpecSums& s, double w, float2 fp, float2 fc) {
  const double ap = sqrt((double)fp.x * fp.x + (double)fp.y * fp.y);
  const double pc = (double)fc.x * fc.x + (double)fc.y * fc.y;  // power |F_c|^2
  const double ac = sqrt(pc);
  s.pc = fma(w * ap, ac, s.pc);
  s.pp = fma(w * ap, ap, s.pp);
  s.cc = fma(w, pc, s.cc);
  if (pc > 0.0) {
    int e;
    const double m = frexp(pc, &e);
    const double lnp = (double)e * 0.69314718055994530942 + (double)logf((float)m);
    s.plp = fma(w * pc, lnp, s.plp);
  }
}

// Normalised cross-power (migration.py:130-131): C = Fp conj(Fc) / (|.|+eps).
__device__ __forceinline__ float2 xpower(float2 fp, float2 fc) {
  const float cx = fp.x * fc.x + fp.y * fc.y;
  const float cy = fp.y * fc.x - fp.x * fc.y;
  const float mag = hypotf(fp.x, fp.y) * hypotf(fc.x, fc.y);
  const float inv = 1.0f / (mag + 1e-12f);
  return make_float2(cx * inv, cy * inv);
}

// unpack bin k of the (DC, Nyquist) pair packed into one column
__device__ __forceinline__ void unpack_dcny(float2 zk, float2 zm, float2& f0, float2& fn) {
  // F0[k] = (Z[k] + conj Z[-k]) / 2 ; FN[k] = -i (Z[k] - conj Z[-k]) / 2
  f0 = make_float2(0.5f * (zk.x + zm.x), 0.5f * (zk.y - zm.y));
  fn = make_float2(0.5f * (zk.y + zm.y), -0.5f * (zk.x - zm.x));
}

template <int NH>
__global__ void __launch_bounds__(FC_THREADS) k_cols(KParams kp) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ double red[32 * 4];
  const int cb = blockIdx.x, b = blockIdx.y;
  const int H = kp.H;
  const int nel = H * FC_CB;
  float2* bufA = reinterpret_cast<float2*>(smem);
  float2* bufB = bufA + nel;
  float2* tw = bufB + nel;
  const bool valid = kp.hdr[b].valid != 0;
  const size_t blk = ((size_t)b * kp.NCB + cb) * (size_t)nel;
  float2* Tb = kp.T + blk;
  float2* Sb = kp.spec + blk;

  for (int i = threadIdx.x; i < H; i += blockDim.x) tw[i] = kp.twH[i];
  {
    const float4* src = reinterpret_cast<const float4*>(Tb);
    float4* dst = reinterpret_cast<float4*>(bufA);
    for (int i = threadIdx.x; i < nel / 2; i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  float2* Fc = fft_any<NH, false>(bufA, bufB, tw, kp.planH, FC_CB, 1, FC_CB, true);
  float2* Xp = (Fc == bufA) ? bufB : bufA;

  if (!valid) {  // cold stream: establish the spectrum only
    float4* dst = reinterpret_cast<float4*>(Sb);
    const float4* src = reinterpret_cast<const float4*>(Fc);
    for (int i = threadIdx.x; i < nel / 2; i += blockDim.x) dst[i] = src[i];
    return;
  }
  {
    // previous spectrum in, current spectrum out (in-place state swap)
    float4* st = reinterpret_cast<float4*>(Sb);
    float4* xp = reinterpret_cast<float4*>(Xp);
    const float4* fc4 = reinterpret_cast<const float4*>(Fc);
    for (int i = threadIdx.x; i < nel / 2; i += blockDim.x) {
      xp[i] = st[i];
      st[i] = fc4[i];
    }
  }
  __syncthreads();

  SpecSums sums = {0.0, 0.0, 0.0, 0.0};
  const int Wc = kp.Wc;
  for (int e = threadIdx.x; e < nel; e += blockDim.x) {
    const int c = e % FC_CB;
    const int q = cb * FC_CB + c;
    if (q >= Wc) { Xp[e] = make_float2(0.f, 0.f); continue; }
    if (q == 0) continue;
    const float2 fp = Xp[e], fc = Fc[e];
    acc_bin(sums, 2.0, fp, fc);  // interior bin stands for itself and its mirror
    Xp[e] = xpower(fp, fc);
  }
  if (cb == 0) {
    const bool weven = (kp.W & 1) == 0;
    for (int k = threadIdx.x; k <= H / 2; k += blockDim.x) {
      const int km = (H - k) % H;
      float2 c0k, cnk, c0m, cnm, p0k, pnk, p0m, pnm;
      unpack_dcny(Fc[k * FC_CB], Fc[km * FC_CB], c0k, cnk);
      unpack_dcny(Xp[k * FC_CB], Xp[km * FC_CB], p0k, pnk);
      acc_bin(sums, 1.0, p0k, c0k);
      if (weven) acc_bin(sums, 1.0, pnk, cnk);
      float2 x0 = xpower(p0k, c0k);
      float2 xn = weven ? xpower(pnk, cnk) : make_float2(0.f, 0.f);
      float2 packed_k = make_float2(x0.x - xn.y, x0.y + xn.x);
      if (km != k) {
        unpack_dcny(Fc[km * FC_CB], Fc[k * FC_CB], c0m, cnm);
        unpack_dcny(Xp[km * FC_CB], Xp[k * FC_CB], p0m, pnm);
        acc_bin(sums, 1.0, p0m, c0m);
        if (weven) acc_bin(sums, 1.0, pnm, cnm);
        float2 y0 = xpower(p0m, c0m);
        float2 yn = weven ? xpower(pnm, cnm) : make_float2(0.f, 0.f);
        Xp[km * FC_CB] = make_float2(y0.x - yn.y, y0.y + yn.x);
      }
      Xp[k * FC_CB] = packed_k;
    }
  }
  __syncthreads();
  float2* G = fft_any<NH, true>(Xp, Fc, tw, kp.planH, FC_CB, 1, FC_CB, true);
  {
    float4* dst = reinterpret_cast<float4*>(Tb);
    const float4* src = reinterpret_cast<const float4*>(G);
    for (int i = threadIdx.x; i < nel / 2; i += blockDim.x) dst[i] = src[i];
  }
  double v[4] = {sums.pc, sums.pp, sums.cc, sums.plp};
  block_sum_d<4>(v, red);
  if (threadIdx.x == 0) {
    double* o = kp.stats + ((size_t)b * kp.NCB + cb) * 4;
    o[0] = v[0]; o[1] = v[1]; o[2] = v[2]; o[3] = v[3];
  }
}

// ----------------------------------------------------------------- K_C ----

struct PeakKey {
  float v;
  int l1;
  int pos;
};

__device__ __forceinline__ bool peak_better(const PeakKey& a, const PeakKey& b) {
  // max value; exact ties -> min |di|+|dj| -> min row-major position
  // (migration.py:141-159)
  if (a.v != b.v) return a.v > b.v;
  if (a.l1 != b.l1) return a.l1 < b.l1;
  return a.pos < b.pos;
}

template <int NW>
__global__ void __launch_bounds__(FC_THREADS) k_rows_inv(KParams kp) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ PeakKey redk[32];
  __shared__ float redv[32];
  const int gidx = blockIdx.x, b = blockIdx.y;
  if (kp.hdr[b].valid == 0) return;
  const int H = kp.H, W = kp.W, Wc = kp.Wc;
  const int y0 = gidx * kp.RG;
  const int nrows = min(kp.RG, H - y0);
  const int npair = (nrows + 1) / 2;
  const int maxpair = (kp.RG + 1) / 2;
  float2* bufA = reinterpret_cast<float2*>(smem);
  float2* bufB = bufA + maxpair * W;
  float2* tw = bufB + maxpair * W;
  for (int i = threadIdx.x; i < W; i += blockDim.x) tw[i] = kp.twW[i];
  const bool weven = (W & 1) == 0;
  for (int idx = threadIdx.x; idx < npair * Wc; idx += blockDim.x) {
    const int t = idx / Wc, q = idx - t * Wc;
    const int ya = y0 + 2 * t;
    const bool hasb = 2 * t + 1 < nrows;
    const float2* src = kp.T + (((size_t)b * kp.NCB + q / FC_CB) * H + ya) * FC_CB + (q % FC_CB);
    const float2 ga = src[0];
    const float2 gb = hasb ? src[FC_CB] : make_float2(0.f, 0.f);
    float2* Z = bufA + t * W;
    if (q == 0) {
      Z[0] = make_float2(ga.x, gb.x);
      if (weven) Z[W / 2] = make_float2(ga.y, gb.y);
    } else {
      Z[q] = make_float2(ga.x - gb.y, ga.y + gb.x);       // G_a + i G_b
      Z[W - q] = make_float2(ga.x + gb.y, gb.x - ga.y);   // conj G_a + i conj G_b
    }
  }
  __syncthreads();
  const float2* r = fft_any<NW, true>(bufA, bufB, tw, kp.planW, npair, W, 1, false);

  PeakKey best = {-CUDART_INF_F, 0x7fffffff, 0x7fffffff};
  float v2 = -CUDART_INF_F;
  for (int idx = threadIdx.x; idx < nrows * W; idx += blockDim.x) {
    const int row = idx / W, j = idx - row * W;
    const float2 z = r[(row >> 1) * W + j];
    const int y = y0 + row;
    PeakKey c;
    c.v = (row & 1) ? z.y : z.x;
    c.l1 = abs(canon_disp(y, H)) + abs(canon_disp(j, W));
    c.pos = y * W + j;
    if (peak_better(c, best)) { v2 = fmaxf(v2, best.v); best = c; }
    else v2 = fmaxf(v2, c.v);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    PeakKey other;
    other.v = __shfl_xor_sync(0xffffffffu, best.v, o);
    other.l1 = __shfl_xor_sync(0xffffffffu, best.l1, o);
    other.pos = __shfl_xor_sync(0xffffffffu, best.pos, o);
    const float ov2 = __shfl_xor_sync(0xffffffffu, v2, o);
    if (peak_better(other, best)) { v2 = fmaxf(fmaxf(v2, ov2), best.v); best = other; }
    else v2 = fmaxf(fmaxf(v2, ov2), other.v);
  }
  if (lane == 0) { redk[wid] = best; redv[wid] = v2; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < nw; ++w) {
      const PeakKey o = redk[w];
      if (peak_better(o, best)) { v2 = fmaxf(fmaxf(v2, redv[w]), best.v); best = o; }
      else v2 = fmaxf(fmaxf(v2, redv[w]), o.v);
    }
    PeakPart pp;
    pp.v = best.v; pp.v2 = v2; pp.y = best.pos / W; pp.j = best.pos % W;
    kp.peaks[(size_t)b * kp.NRG + gidx] = pp;
  }
}

// ----------------------------------------------------------------- K_D ----

__device__ __forceinline__ bool key_less(double ea, int ia, double eb, int ib) {
  return ea < eb || (ea == eb && ia < ib);
}

// Bitonic sort of (E, index) keys in shared memory, one CTA.
__device__ void bitonic_smem(double* ke, int* ki, int NP2) {
  for (int k = 2; k <= NP2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < NP2; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const double ea = ke[i], eb = ke[ixj];
          const int ia = ki[i], ib = ki[ixj];
          const bool up = (i & k) == 0;
          const bool swap = up ? key_less(eb, ib, ea, ia) : key_less(ea, ia, eb, ib);
          if (swap) { ke[i] = eb; ke[ixj] = ea; ki[i] = ib; ki[ixj] = ia; }
        }
      }
      __syncthreads();
    }
  }
}

// Bitonic steps j = jmax..1 (jmax <= 32) on the 64 keys a warp holds in
// registers: lane L has elements base+L (slot 0) and base+L+32 (slot 1).
// Distance 32 pairs the two slots of a lane; smaller distances pair lanes
// (xor shuffles).  No barriers.
__device__ __forceinline__ void warp_bitonic(double (&e)[2], int (&x)[2], int base, int k, int jmax) {
  const int lane = threadIdx.x & 31;
  for (int j = jmax; j > 0; j >>= 1) {
    if (j == 32) {
      const bool up = ((base + lane) & k) == 0;
      const bool gt = key_less(e[1], x[1], e[0], x[0]);  // slot0 > slot1
      if (up == gt) {
        const double te = e[0]; e[0] = e[1]; e[1] = te;
        const int tx = x[0]; x[0] = x[1]; x[1] = tx;
      }
    } else {
#pragma unroll
      for (int sl = 0; sl < 2; ++sl) {
        const double oe = __shfl_xor_sync(0xffffffffu, e[sl], j);
        const int ox = __shfl_xor_sync(0xffffffffu, x[sl], j);
        const int i = base + lane + 32 * sl;
        const bool up = (i & k) == 0;
        const bool low = (lane & j) == 0;             // this element has the smaller index
        const bool other_less = key_less(oe, ox, e[sl], x[sl]);
        // ascending pair: low keeps the min, high keeps the max
        const bool take = (up == low) ? other_less : !other_less;
        if (take) { e[sl] = oe; x[sl] = ox; }
      }
    }
  }
}

// Same sort with register/shuffle stages for distances < 64 and shared
// memory only for the cross-warp distances: 10 barrier phases at N = 1024
// instead of 55.  NP2 >= 64, power of two.
__device__ void bitonic_hybrid(double* ke, int* ki, int NP2) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nseg = NP2 / 64;
  // phase A: every 64-key segment sorted by its warp (k = 2 .. 64)
  for (int sg = wid; sg < nseg; sg += nw) {
    const int base = sg * 64;
    double e[2] = {ke[base + lane], ke[base + lane + 32]};
    int x[2] = {ki[base + lane], ki[base + lane + 32]};
    for (int k = 2; k <= 64; k <<= 1) warp_bitonic(e, x, base, k, k >> 1);
    ke[base + lane] = e[0]; ke[base + lane + 32] = e[1];
    ki[base + lane] = x[0]; ki[base + lane + 32] = x[1];
  }
  __syncthreads();
  for (int k = 128; k <= NP2; k <<= 1) {
    for (int j = k >> 1; j >= 64; j >>= 1) {
      for (int i = threadIdx.x; i < NP2; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const double ea = ke[i], eb = ke[ixj];
          const int ia = ki[i], ib = ki[ixj];
          const bool up = (i & k) == 0;
          const bool swap = up ? key_less(eb, ib, ea, ia) : key_less(ea, ia, eb, ib);
          if (swap) { ke[i] = eb; ke[ixj] = ea; ki[i] = ib; ki[ixj] = ia; }
        }
      }
      __syncthreads();
    }
    for (int sg = wid; sg < nseg; sg += nw) {
      const int base = sg * 64;
      double e[2] = {ke[base + lane], ke[base + lane + 32]};
      int x[2] = {ki[base + lane], ki[base + lane + 32]};
      warp_bitonic(e, x, base, k, 32);
      ke[base + lane] = e[0]; ke[base + lane + 32] = e[1];
      ki[base + lane] = x[0]; ki[base + lane + 32] = x[1];
    }
    __syncthreads();
  }
}

// K_D1: per-stream energy statistics, refresh mask and the ascending
// (E, index) order of ALL tokens (edge_refresh.py:62-73, fusion.py:104-115).
// It needs the energies only (K_A), so it runs on a side branch beside
// K_B / K_C; K_D then takes the first K_final candidates of this order — a
// stable filter of the sorted token list is exactly topk_ascending's lexsort
// of the candidates — so no sort is left on the critical path.
template <int NT>
__global__ void __launch_bounds__(NT) k_rank(KParams kp, double lam, int b0) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int b = b0 + blockIdx.x;
  const int N = kp.N;
  int NP2 = 1;
  while (NP2 < N) NP2 <<= 1;
  double* ke = reinterpret_cast<double*>(smem);  // NP2
  int* ki = reinterpret_cast<int*>(ke + NP2);    // NP2
  __shared__ double red[32 * 2];
  __shared__ int redi[32];
  const double* energy = kp.energy + (size_t)b * N;
  for (int p = threadIdx.x; p < NP2; p += blockDim.x) {
    ke[p] = p < N ? energy[p] : CUDART_INF;
    ki[p] = p < N ? p : 0x7fffffff;
  }
  __syncthreads();

  // Module II statistics: population mean / std.  Summation order fixed at
  // FC_SEL_THREADS strided partials whatever the block size (the extra warps
  // add exact zeros to the trees), so a stream's statistics do not depend on
  // the batch size that picked the block size.
  static_assert(NT % FC_SEL_THREADS == 0, "block size must be a multiple of the reduction width");
  const bool red_lane = threadIdx.x < FC_SEL_THREADS;
  double s1 = 0.0;
  // shifted by E[0]: an all-equal energy map keeps an exact mean and std 0
  const double e0 = ke[0];
  if (red_lane)
    for (int p = threadIdx.x; p < N; p += FC_SEL_THREADS) s1 += ke[p] - e0;
  {
    double v[1] = {s1};
    block_sum_d<1>(v, red);
    if (threadIdx.x == 0) red[63] = e0 + v[0] / (double)N;
  }
  __syncthreads();
  const double mu = red[63];
  double s2 = 0.0;
  if (red_lane)
    for (int p = threadIdx.x; p < N; p += FC_SEL_THREADS) { const double d = ke[p] - mu; s2 = fma(d, d, s2); }
  {
    double v[1] = {s2};
    block_sum_d<1>(v, red);
    if (threadIdx.x == 0) {
      const double sd = sqrt(v[0] / (double)N);
      red[62] = mu + lam * sd;
      double* es = kp.estats + (size_t)b * 4;
      es[0] = mu;
      es[1] = sd;
      es[2] = mu + lam * sd;
    }
  }
  __syncthreads();
  const double thr = red[62];
  int nfresh = 0;
  uint8_t* fm = kp.freshm + (size_t)b * N;
  for (int p = threadIdx.x; p < N; p += blockDim.x) {
    const int f = ke[p] > thr;   // strict (edge_refresh.py:72)
    fm[p] = (uint8_t)f;
    nfresh += f;
  }
  {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int a = warp_sum(nfresh);
    if (lane == 0) redi[wid] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
      int ta = 0;
      for (int w = 0; w < nw; ++w) ta += redi[w];
      kp.estats[(size_t)b * 4 + 3] = (double)ta;
    }
  }
  // ascending (E, index) order of every token (fusion.py:104-115)
  if (NP2 >= 64) bitonic_hybrid(ke, ki, NP2);
  else bitonic_smem(ke, ki, NP2);
  int16_t* ord = kp.order + (size_t)b * N;
  for (int r = threadIdx.x; r < N; r += blockDim.x) ord[r] = (int16_t)ki[r];
}

// K_D: decision for one stream (fusion.py:121-242 selection; 245-262
// invariants hold by construction).  Scalars in thread 0, per-token work
// spread; the energy statistics, refresh mask and token order come from K_D1.
template <int NT>
__global__ void __launch_bounds__(NT) k_select(KParams kp, fc_config cfg, fc_select_out out) {
  extern __shared__ __align__(128) unsigned char smem[];
  // launched as a programmatic dependent of K_C (FC_PDL=1): K_C's partials
  // are complete and visible after this (a no-op for a plain launch)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int b = blockIdx.x;
  const int N = kp.N;
  int* ki = reinterpret_cast<int*>(smem);                 // N: reuse list
  int* rank = ki + N;                                     // N
  uint8_t* fresh = reinterpret_cast<uint8_t*>(rank + N);  // N
  uint8_t* reuse = fresh + N;                             // N
  uint8_t* cand = reuse + N;                              // N
  __shared__ int redi[32];
  __shared__ fc_stream_result R;
  __shared__ int sh_flush, sh_dip, sh_djp, sh_kfinal, sh_err;

  __shared__ double sh_sum[4], sh_ref;
  __shared__ int sh_bad, sh_vary, sh_pos;
  __shared__ float sh_pv, sh_pv2;
  if (threadIdx.x < 32) {
    // warp 0 gathers the per-CTA partials of K_A/K_B/K_C (fixed-order trees)
    const int lane = threadIdx.x;
    const double ref0 = kp.stripes[(size_t)b * kp.rows].ref;
    int bad = 0, vary = 0;
    for (int s = lane; s < kp.rows; s += 32) {
      const StripeStat st = kp.stripes[(size_t)b * kp.rows + s];
      bad |= st.nonfinite;
      vary |= st.varying | (st.ref != ref0);
    }
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    for (int c = lane; c < kp.NCB; c += 32) {
      const double* st = kp.stats + ((size_t)b * kp.NCB + c) * 4;
      a0 += st[0]; a1 += st[1]; a2 += st[2]; a3 += st[3];
    }
    PeakKey bk = {-CUDART_INF_F, 0x7fffffff, 0x7fffffff};
    float v2 = -CUDART_INF_F;
    for (int g = lane; g < kp.NRG; g += 32) {
      const PeakPart o = kp.peaks[(size_t)b * kp.NRG + g];
      const PeakKey ok = {o.v, abs(canon_disp(o.y, kp.H)) + abs(canon_disp(o.j, kp.W)), o.y * kp.W + o.j};
      if (peak_better(ok, bk)) { v2 = fmaxf(fmaxf(v2, o.v2), bk.v); bk = ok; }
      else v2 = fmaxf(fmaxf(v2, o.v2), ok.v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      bad |= __shfl_xor_sync(0xffffffffu, bad, o);
      vary |= __shfl_xor_sync(0xffffffffu, vary, o);
      a0 += __shfl_xor_sync(0xffffffffu, a0, o);
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
      a2 += __shfl_xor_sync(0xffffffffu, a2, o);
      a3 += __shfl_xor_sync(0xffffffffu, a3, o);
      PeakKey ok;
      ok.v = __shfl_xor_sync(0xffffffffu, bk.v, o);
      ok.l1 = __shfl_xor_sync(0xffffffffu, bk.l1, o);
      ok.pos = __shfl_xor_sync(0xffffffffu, bk.pos, o);
      const float ov2 = __shfl_xor_sync(0xffffffffu, v2, o);
      if (peak_better(ok, bk)) { v2 = fmaxf(fmaxf(v2, ov2), bk.v); bk = ok; }
      else v2 = fmaxf(fmaxf(v2, ov2), ok.v);
    }
    if (lane == 0) {
      sh_ref = ref0; sh_vary = vary; sh_bad = bad;
      sh_sum[0] = a0; sh_sum[1] = a1; sh_sum[2] = a2; sh_sum[3] = a3;
      sh_pv = bk.v; sh_pv2 = v2; sh_pos = bk.pos;
    }
  } else {
    // the other warps stage K_D1's refresh mask meanwhile
    const uint8_t* fm = kp.freshm + (size_t)b * N;
    for (int p = threadIdx.x - 32; p < N; p += blockDim.x - 32) fresh[p] = fm[p];
  }
  __syncthreads();

  if (threadIdx.x == 0) {
    StreamHdr h = kp.hdr[b];
    // frame flags (fusion.py:147, frame.py:13)
    const int bad = sh_bad;
    const int cconst = !sh_vary;
    const int czero = cconst && sh_ref == 0.0;
    memset(&R, 0, sizeof(R));
    R.rows = kp.rows; R.cols = kp.cols;
    R.bin_count = (int64_t)kp.H * kp.W;
    R.status = bad ? FC_ENONFINITE : FC_OK;
    const int cold = !h.valid;
    R.cold = cold;
    int flush = 1, dip = 0, djp = 0;
    if (!cold && !bad) {
      const double spc = sh_sum[0], spp = sh_sum[1], scc = sh_sum[2], splp = sh_sum[3];
      // Module I (migration.py:87-105, fusion.py:147-150)
      int mig = FC_DIAG_NONE;
      if (h.prev_zero || czero) mig = FC_DIAG_DEGENERATE;
      else if (h.prev_const || cconst) mig = FC_DIAG_NO_TEXTURE;
      if (mig == FC_DIAG_NONE) {
        double sim = spc / (sqrt(spp) * sqrt(scc));
        R.sim_freq = sim < 1.0 ? sim : 1.0;
        const double inv_hw = 1.0 / ((double)kp.H * kp.W);
        R.peak = (double)sh_pv * inv_hw;
        R.peak_runner_up = (double)sh_pv2 * inv_hw;
        R.di = canon_disp(sh_pos / kp.W, kp.H);
        R.dj = canon_disp(sh_pos % kp.W, kp.W);
        R.di_patches = to_patch_units(R.di, kp.P);
        R.dj_patches = to_patch_units(R.dj, kp.P);
        dip = R.di_patches; djp = R.dj_patches;
      }
      // Module III (budget.py:34-75)
      int bud = FC_DIAG_NONE;
      if (czero) {
        bud = FC_DIAG_DEGENERATE;
      } else {
        double raw = 0.0;
        if (!cconst) {  // a constant frame's power spectrum is one-hot: H = 0
          raw = log(scc) - splp / scc;
          if (raw < 0.0) raw = 0.0;
        }
        const double psi = raw / log((double)kp.H * kp.W);
        R.entropy_raw = raw;
        R.entropy_norm = psi;
        if (!(psi >= 0.0 && psi <= 1.0)) {
          R.status = FC_EPSI;
        } else {
          const double alpha = cfg.alpha_min + (cfg.alpha_max - cfg.alpha_min) * exp(-psi);
          R.alpha = alpha;
          R.k_reuse = (int)floor(alpha * (double)N);
        }
      }
      R.diagnostic = mig != FC_DIAG_NONE ? mig : bud;
      if (R.diagnostic != FC_DIAG_NONE) flush = 1;
      else if (R.sim_freq < cfg.tau_mig) flush = 1;                       // migration.py:179-185
      else if (cfg.refresh_shift >= 0 &&
               max(abs(dip), abs(djp)) > cfg.refresh_shift) flush = 1;   // config 2 (not in ref)
      else flush = 0;
    }
    R.flushed = flush;
    // Module II (edge_refresh.py:62-73), from K_D1
    const double* es = kp.estats + (size_t)b * 4;
    R.energy_mean = es[0];
    R.energy_std = es[1];
    R.energy_threshold = es[2];
    R.n_refresh = (int)es[3];
    sh_flush = flush; sh_dip = dip; sh_djp = djp;
    sh_err = R.status != FC_OK;
    // state for the next step: this frame becomes "prev"
    if (!bad) {
      h.valid = 1;
      h.prev_zero = czero;
      h.prev_const = cconst;
      h.steps += 1;
      kp.hdr[b] = h;
    } else {
      // the reference raises on a non-finite frame (frame.py:13-14); the
      // spectrum state already holds this frame's (non-finite) transform, so
      // the stream restarts cold: its next frame only re-establishes it
      h.valid = 0;
      kp.hdr[b] = h;
    }
  }
  __syncthreads();

  const int rows = kp.rows, cols = kp.cols;
  const int flush = sh_flush, dip = sh_dip, djp = sh_djp;
  int ncand = 0;
  for (int p = threadIdx.x; p < N; p += blockDim.x) {
    const int i = p / cols, j = p - (p / cols) * cols;
    const int si = i - dip, sj = j - djp;
    const int aligned = (si >= 0 && si < rows && sj >= 0 && sj < cols);
    const int c = !flush && aligned && !fresh[p];   // fusion.py:214
    cand[p] = (uint8_t)c;
    ncand += c;
    reuse[p] = 0;
  }
  {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int c = warp_sum(ncand);
    if (lane == 0) redi[wid] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
      int tc = 0;
      for (int w = 0; w < nw; ++w) tc += redi[w];
      R.k_candidate = tc;
      const int kf = (flush || sh_err) ? 0 : min(R.k_reuse, tc);
      if (flush) R.k_candidate = 0;
      R.k_final = kf;
      sh_kfinal = kf;
    }
    __syncthreads();
  }
  const int kfinal = sh_kfinal;
  if (kfinal > 0) {
    // the first K_final candidates of K_D1's ascending (E, index) order:
    // exclusive scan of the candidate flags along the order
    const int16_t* ord = kp.order + (size_t)b * N;
    const int per = (N + blockDim.x - 1) / blockDim.x;
    const int r0 = threadIdx.x * per, r1 = min(N, r0 + per);
    int cnt = 0;
    for (int r = r0; r < r1; ++r) cnt += cand[ord[r]];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) redi[wid] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0;
      for (int w = 0; w < nw; ++w) { const int t = redi[w]; redi[w] = acc; acc += t; }
    }
    __syncthreads();
    int run = redi[wid] + incl - cnt;
    for (int r = r0; r < r1 && run < kfinal; ++r) {
      const int q = ord[r];
      if (cand[q]) {
        ki[run++] = q;
        reuse[q] = 1;
      }
    }
  }
  __syncthreads();

  // row-major recompute order: exclusive scan of !reuse
  {
    const int per = (N + blockDim.x - 1) / blockDim.x;
    const int p0 = threadIdx.x * per;
    int cnt = 0;
    for (int p = p0; p < min(N, p0 + per); ++p) cnt += !reuse[p];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) redi[wid] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0;
      for (int w = 0; w < nw; ++w) { const int t = redi[w]; redi[w] = acc; acc += t; }
    }
    __syncthreads();
    int run = redi[wid] + incl - cnt;
    for (int p = p0; p < min(N, p0 + per); ++p) {
      rank[p] = run;
      run += !reuse[p];
    }
  }
  __syncthreads();
  const size_t o = (size_t)b * N;
  const int nrec = N - kfinal;
  for (int p = threadIdx.x; p < N; p += blockDim.x) {
    const int ru = reuse[p];
    if (out.reuse_mask) out.reuse_mask[o + p] = (uint8_t)ru;
    if (out.refresh_mask) out.refresh_mask[o + p] = fresh[p];
    if (out.reuse_idx) out.reuse_idx[o + p] = p < kfinal ? ki[p] : -1;
    if (out.recompute_idx) {
      if (!ru) out.recompute_idx[o + rank[p]] = p;
      if (p >= nrec) out.recompute_idx[o + p] = -1;
    }
    if (out.src_map) {
      const int i = p / cols, j = p - (p / cols) * cols;
      out.src_map[o + p] = ru ? (i - dip) * cols + (j - djp) : -(rank[p] + 1);
    }
  }
  if (threadIdx.x == 0 && out.results) out.results[b] = R;
  if (threadIdx.x == 0 && out.counters) {
    // run_sequence aggregates (fusion.py:559-572): integer atomics, so the
    // totals are exact and order-independent
    unsigned long long* c = reinterpret_cast<unsigned long long*>(out.counters);
    atomicAdd(c + 0, 1ull);
    atomicAdd(c + 1, (unsigned long long)R.k_final);
    atomicAdd(c + 2, (unsigned long long)(R.flushed && !R.cold));
    atomicAdd(c + 3, (unsigned long long)R.cold);
  }
}

// ----------------------------------------------------------------- K_E ----

// Splice source check (fusion.py:488-490): a cache source must name a token
// of the stream's grid, a compact fresh index a row the caller supplied.  A
// bad row is skipped and FC_EBOUNDS is left in *status (all writers store the
// same value, so plain stores suffice).
__device__ __forceinline__ bool splice_src_ok(int s, int n_tokens, bool have_cache, int compact, int fresh_rows) {
  if (s >= 0) return have_cache && s < n_tokens;
  return !compact || (-(s + 1)) < fresh_rows;
}
__device__ __forceinline__ void flag_bounds(int32_t* status) {
  if (status) *reinterpret_cast<volatile int32_t*>(status) = FC_EBOUNDS;
}

// Hidden-state splice (fusion.py:462-512): one warp per token row, 16-byte
// vector copies, UNR rows in flight per warp.  Bit copy of any dtype.
template <int UNR>
__global__ void __launch_bounds__(FC_THREADS) k_splice16(int total, int n_tokens, int64_t row16,
                                                         const int32_t* __restrict__ src_map,
                                                         const int4* __restrict__ cache,
                                                         const int64_t* __restrict__ cache_ages,
                                                         const int4* __restrict__ fresh, int compact,
                                                         int fresh_rows, const int64_t* __restrict__ fresh_off,
                                                         int4* __restrict__ out,
                                                         int64_t* __restrict__ out_ages,
                                                         int32_t* __restrict__ status) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int r0 = gw * UNR; r0 < total; r0 += nwarps * UNR) {
    const int4* src[UNR];
    int4* dst[UNR];
    bool on[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int row = r0 + u;
      const int rr = row < total ? row : r0;
      const int bs = rr / n_tokens;
      const int s = src_map[rr];
      const size_t base = (size_t)bs * n_tokens;
      // fusion.py:488-490 asserts the reuse source lies inside the grid
      const bool ok = splice_src_ok(s, n_tokens, cache != nullptr, compact, fresh_rows);
      on[u] = row < total && ok;
      if (row < total && !ok && lane == 0) flag_bounds(status);
      if (!ok) {
        src[u] = fresh;
      } else if (s >= 0) {
        src[u] = cache + (base + s) * row16;
      } else {
        const size_t row0 = fresh_off ? (size_t)fresh_off[bs] : (size_t)bs * fresh_rows;
        src[u] = fresh + (row0 + (compact ? (-s - 1) : (rr - bs * n_tokens))) * row16;
      }
      dst[u] = out + (size_t)rr * row16;
      if (on[u] && lane == 0)
        out_ages[rr] = s >= 0 ? cache_ages[base + s] + 1 : 0;
    }
    for (int64_t c = lane; c < row16; c += 32 * 4) {
      int4 v[UNR][4];
#pragma unroll
      for (int u = 0; u < UNR; ++u)
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int64_t cc = c + 32 * m;
          if (on[u] && cc < row16) v[u][m] = __ldcs(src[u] + cc);
        }
#pragma unroll
      for (int u = 0; u < UNR; ++u)
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int64_t cc = c + 32 * m;
          if (on[u] && cc < row16) __stcs(dst[u] + cc, v[u][m]);
        }
    }
  }
}

// Byte-granular fallback for rows that are not 16-byte multiples / aligned.
__global__ void k_splice_bytes(int total, int n_tokens, int64_t row_bytes, const int32_t* __restrict__ src_map,
                               const uint8_t* __restrict__ cache, const int64_t* __restrict__ cache_ages,
                               const uint8_t* __restrict__ fresh, int compact, int fresh_rows,
                               const int64_t* __restrict__ fresh_off, uint8_t* __restrict__ out,
                               int64_t* __restrict__ out_ages, int32_t* __restrict__ status) {
  const int row = blockIdx.x;
  if (row >= total) return;
  const int bs = row / n_tokens;
  const int s = src_map[row];
  const size_t base = (size_t)bs * n_tokens;
  if (!splice_src_ok(s, n_tokens, cache != nullptr, compact, fresh_rows)) {
    if (threadIdx.x == 0) flag_bounds(status);
    return;
  }
  const uint8_t* src = s >= 0 ? cache + (base + s) * row_bytes
                              : fresh + ((fresh_off ? (size_t)fresh_off[bs] : (size_t)bs * fresh_rows) +
                                         (compact ? (-s - 1) : (row - bs * n_tokens))) * row_bytes;
  for (int64_t c = threadIdx.x; c < row_bytes; c += blockDim.x) out[(size_t)row * row_bytes + c] = src[c];
  if (threadIdx.x == 0) out_ages[row] = s >= 0 ? cache_ages[base + s] + 1 : 0;
}

// src_map of one stream from an ordered reuse list (fusion.py:481-504).
__global__ void k_splice_map(int rows, int cols, const int32_t* __restrict__ reuse_idx, int k, int dip,
                             int djp, int32_t* __restrict__ src_map, int32_t* __restrict__ flag) {
  extern __shared__ int sm_flags[];  // N
  __shared__ int redi[32];
  const int N = rows * cols;
  for (int p = threadIdx.x; p < N; p += blockDim.x) sm_flags[p] = -1;
  __syncthreads();
  for (int r = threadIdx.x; r < k; r += blockDim.x) {
    const int p = reuse_idx[r];
    if (p < 0 || p >= N) { if (flag) *flag = FC_EBOUNDS; continue; }
    const int i = p / cols, j = p % cols;
    const int si = i - dip, sj = j - djp;
    if (si < 0 || si >= rows || sj < 0 || sj >= cols) { if (flag) *flag = FC_EBOUNDS; continue; }
    sm_flags[p] = si * cols + sj;
  }
  __syncthreads();
  const int per = (N + blockDim.x - 1) / blockDim.x;
  const int p0 = threadIdx.x * per;
  int cnt = 0;
  for (int p = p0; p < min(N, p0 + per); ++p) cnt += sm_flags[p] < 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int incl = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) redi[wid] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int w = 0; w < nw; ++w) { const int t = redi[w]; redi[w] = acc; acc += t; }
  }
  __syncthreads();
  int run = redi[wid] + incl - cnt;
  for (int p = p0; p < min(N, p0 + per); ++p) {
    const int s = sm_flags[p];
    if (s >= 0) src_map[p] = s;
    else src_map[p] = -(++run);
  }
}

__global__ void k_state_reset(StreamHdr* hdr, int first, int count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) {
    StreamHdr h = {0, 0, 0, 0};
    hdr[first + i] = h;
  }
}

// ------------------------------------------------------ in-place splice ----
// Per stream: when every reused token's source is its own slot (zero
// displacement, or nothing reused) the cache is updated in place — reused
// rows stay where they are (age + 1, done here) and only recomputed rows are
// copied.  Otherwise every row of the stream goes to its other buffer
// (ping-pong).  slot_in[b] names the buffer holding stream b's cache,
// slot_out[b] the one holding the result.  The plan kernel also compacts the
// rows to copy (ascending) so the copy kernel's warps only see real work.
__global__ void __launch_bounds__(256) k_splice_plan(int n_tokens, const int32_t* __restrict__ src_map,
                                                     const uint8_t* __restrict__ slot_in,
                                                     uint8_t* __restrict__ slot_out, int64_t* ages0,
                                                     int64_t* ages1, int32_t* __restrict__ rows,
                                                     int32_t* __restrict__ counts) {
  __shared__ int redi[8];
  const int b = blockIdx.x;
  const size_t base = (size_t)b * n_tokens;
  const int32_t* sm = src_map + base;
  int move = 0;
  for (int p = threadIdx.x; p < n_tokens; p += blockDim.x) {
    const int s = sm[p];
    move |= (s >= 0 && s != p);
  }
  move = __syncthreads_or(move);
  const int cur = slot_in[b];
  if (threadIdx.x == 0) slot_out[b] = move ? (uint8_t)(1 - cur) : (uint8_t)cur;
  int32_t* rl = rows + base;
  if (move) {
    for (int p = threadIdx.x; p < n_tokens; p += blockDim.x) rl[p] = p;
    if (threadIdx.x == 0) counts[b] = n_tokens;
    if (b == 0 && threadIdx.x == 0) counts[gridDim.x] = 0;  // bulk copier's work counter
    return;
  }
  if (b == 0 && threadIdx.x == 0) counts[gridDim.x] = 0;
  int64_t* ag = (cur ? ages1 : ages0) + base;
  // ascending compaction of recomputed rows; reused rows age in place
  const int per = (n_tokens + blockDim.x - 1) / blockDim.x;
  const int p0 = threadIdx.x * per, p1 = min(n_tokens, p0 + per);
  int cnt = 0;
  for (int p = p0; p < p1; ++p) {
    if (sm[p] < 0) ++cnt;
    else ag[p] += 1;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) redi[wid] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int w = 0; w < nw; ++w) { const int t = redi[w]; redi[w] = acc; acc += t; }
    counts[b] = acc;
  }
  __syncthreads();
  int run = redi[wid] + incl - cnt;
  for (int p = p0; p < p1; ++p)
    if (sm[p] < 0) rl[run++] = p;
}

template <int UNR>
__global__ void __launch_bounds__(FC_THREADS) k_splice_ip(int total, int n_tokens, int64_t row16,
                                                          const int32_t* __restrict__ src_map,
                                                          int4* cache0, int4* cache1, int64_t* ages0,
                                                          int64_t* ages1, const uint8_t* __restrict__ slot_in,
                                                          const uint8_t* __restrict__ slot_out,
                                                          const int32_t* __restrict__ rows,
                                                          const int32_t* __restrict__ counts,
                                                          const int4* __restrict__ fresh, int compact,
                                                          int fresh_rows, int32_t* __restrict__ status) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int r0 = gw * UNR; r0 < total; r0 += nwarps * UNR) {
    const int4* src[UNR];
    int4* dst[UNR];
    bool on[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int task = r0 + u;
      const int tt = task < total ? task : r0;
      const int bs = tt / n_tokens, k = tt - bs * n_tokens;
      on[u] = task < total && k < counts[bs];
      src[u] = fresh;
      dst[u] = cache0;
      if (!on[u]) continue;
      const size_t base = (size_t)bs * n_tokens;
      const int p = rows[base + k];
      const int s = src_map[base + p];
      if (!splice_src_ok(s, n_tokens, true, compact, fresh_rows)) {
        if (lane == 0) flag_bounds(status);
        on[u] = false;
        continue;
      }
      const int cur = slot_in[bs], nxt = slot_out[bs];
      int4* cbuf = cur ? cache1 : cache0;
      int4* nbuf = nxt ? cache1 : cache0;
      if (s >= 0) {
        src[u] = cbuf + (base + s) * row16;
      } else {
        src[u] = fresh + ((size_t)bs * fresh_rows + (compact ? (-s - 1) : p)) * row16;
      }
      dst[u] = nbuf + (base + p) * row16;
      if (lane == 0) {
        int64_t* cage = cur ? ages1 : ages0;
        int64_t* nage = nxt ? ages1 : ages0;
        nage[base + p] = s >= 0 ? cage[base + s] + 1 : 0;
      }
    }
    for (int64_t c = lane; c < row16; c += 32 * 4) {
      int4 v[UNR][4];
#pragma unroll
      for (int u = 0; u < UNR; ++u)
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int64_t cc = c + 32 * m;
          if (on[u] && cc < row16) v[u][m] = __ldcs(src[u] + cc);
        }
#pragma unroll
      for (int u = 0; u < UNR; ++u)
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int64_t cc = c + 32 * m;
          if (on[u] && cc < row16) __stcs(dst[u] + cc, v[u][m]);
        }
    }
  }
}

// Bulk-copy variant of k_splice_ip for running beside the select kernels:
// one warp per CTA, NL lanes each own SL row slots in shared memory and
// move rows with the TMA engine (global -> shared -> global), so a CTA keeps
// SL * NL rows in flight while issuing a handful of instructions per row
// (a slot is refilled once its store from SL - 1 rows back has been read).
// Rows are claimed dynamically (one atomic per row) so CTAs that start late,
// behind a resident select kernel, simply take less work.  Task t maps to
// (stream, k) through an exclusive scan of counts[] built per CTA.
#ifndef FC_SPLICE_CLAIM
#define FC_SPLICE_CLAIM 8
#endif
template <int NL, int SL = 2>
__global__ void __launch_bounds__(32) k_splice_ip_bulk(int batch, int n_tokens, int row_bytes,
                                                       const int32_t* __restrict__ src_map, char* cache0,
                                                       char* cache1, int64_t* ages0, int64_t* ages1,
                                                       const uint8_t* __restrict__ slot_in,
                                                       const uint8_t* __restrict__ slot_out,
                                                       const int32_t* __restrict__ rows, int32_t* counts,
                                                       const char* __restrict__ fresh, int compact, int fresh_rows,
                                                       int32_t* __restrict__ status) {
  extern __shared__ __align__(128) unsigned char smem[];  // [NL][SL][row_bytes] | offs[batch + 1]
  __shared__ __align__(8) uint64_t bar[NL * SL];
  const int lane = threadIdx.x;
  int* offs = reinterpret_cast<int*>(smem + (size_t)NL * SL * row_bytes);
  for (int i = lane; i < NL * SL; i += 32) tma::bar_init(&bar[i], 1);
  // exclusive scan of counts (lane-contiguous segments)
  const int per = (batch + 31) / 32, q0 = lane * per, q1 = min(batch, q0 + per);
  int sum = 0;
  for (int q = q0; q < q1; ++q) sum += counts[q];
  int incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  int run = incl - sum;
  for (int q = q0; q < q1; ++q) { offs[q] = run; run += counts[q]; }
  const int tot = __shfl_sync(0xffffffffu, incl, 31);
  if (lane == 31) offs[batch] = tot;
  __syncwarp();
  if (lane >= NL) return;
  int* work = counts + batch;
  unsigned char* slot0 = smem + (size_t)lane * SL * row_bytes;
  bool pend = false;
  char* pdst = nullptr;
  int pslot = 0;
  uint32_t pphase = 0;
  // rows are claimed G at a time per lane: the single work counter serves
  // about one atomic per L2 cycle, which bounded the copier when it claimed
  // one row per atomic
  constexpr int G = FC_SPLICE_CLAIM;
  int claim = 0, left = 0;
  // `it` counts issued rows only, so every slot's mbarrier phase advances
  // once per use even when a malformed row is skipped
  for (int it = 0;;) {
    if (left == 0) {
      claim = atomicAdd(work, G);
      left = G;
    }
    const int task = claim + (G - left);
    --left;
    const bool have = task < tot;
    const int sl = it % SL;
    unsigned char* buf = slot0 + sl * row_bytes;
    char* dst = nullptr;
    if (have) {
      // stream of this task: last b with offs[b] <= task
      int lo = 0, hi = batch - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (offs[mid] <= task) lo = mid; else hi = mid - 1;
      }
      const int bs = lo, k = task - offs[bs];
      const size_t base = (size_t)bs * n_tokens;
      const int p = rows[base + k];
      const int s = src_map[base + p];
      if (!splice_src_ok(s, n_tokens, true, compact, fresh_rows)) {
        flag_bounds(status);
        continue;
      }
      const int cur = slot_in[bs], nxt = slot_out[bs];
      const char* cbuf = cur ? cache1 : cache0;
      char* nbuf = nxt ? cache1 : cache0;
      const char* src = s >= 0 ? cbuf + (base + s) * row_bytes
                               : fresh + ((size_t)bs * fresh_rows + (compact ? (-s - 1) : p)) * row_bytes;
      dst = nbuf + (base + p) * row_bytes;
      const int64_t* cage = cur ? ages1 : ages0;
      int64_t* nage = nxt ? ages1 : ages0;
      nage[base + p] = s >= 0 ? cage[base + s] + 1 : 0;
      // this slot's previous store (SL rows back) must have left shared
      // memory; the SL - 2 stores issued after it may still be reading
      if constexpr (SL == 2) tma::bulk_wait_read0();
      else asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(SL - 2) : "memory");
      tma::bar_expect(&bar[lane * SL + sl], row_bytes);
      tma::bulk_g2s(buf, src, row_bytes, &bar[lane * SL + sl]);
    }
    if (pend) {
      tma::bar_wait(&bar[lane * SL + pslot], pphase);
      tma::bulk_s2g(pdst, slot0 + pslot * row_bytes, row_bytes);
    }
    if (!have) break;
    pend = true;
    pdst = dst;
    pslot = sl;
    pphase = (it / SL) & 1;
    ++it;
  }
  tma::bulk_wait0();
}
