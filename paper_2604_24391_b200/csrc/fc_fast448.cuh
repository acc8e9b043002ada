// Fast path for the BASELINE geometry (448 x 448 frames, P = 14, N = 1024):
// register-resident 448-point FFTs with compile-time thread roles.
//
// 448 = 7 * 64, 64 = 8 * 8.  Forward (natural order in, permuted out):
//   stage 1  role n2 in [0,64): A[n2][k1] = DFT7_{n1}(x[64 n1 + n2]) * w448^{n2 k1}
//   stage 2  role (k1, m2):     B[k1][m2][j1] = DFT8_{m1}(A[8 m1 + m2][k1])
//   stage 3  role (k1, j1):     X[k1 + 7 j1 + 56 j2] = DFT8_{m2}(B[k1][m2][j1] * w64^{m2 j1})
// so role r < 56 ends holding X[k1 + 7 j1 + 56 j2], j2 = 0..7, (k1, j1) = (r/8, r%8).
// The inverse runs the same stages transposed (permuted in, natural out) with
// conjugate twiddles, so a forward->pointwise->inverse chain never reorders.
// Exchanges go through shared memory in layouts chosen to be bank-conflict
// free for 8-byte accesses: S1[k1][n2] and S2[k1][j1][m2] with row stride 72
// and j1 stride 9 (k1 rows of two neighbouring roles land 16 banks apart).
// Kernels whose transforms interleave c-fastest (column pass) use a per-
// transform scratch stride of 514 (= 2 mod 16) so the 8 transforms of a
// half-warp spread over disjoint 4-bank groups.
#pragma once
#include "fc_fft.cuh"
#include "fc_tma.cuh"

namespace f448 {

constexpr int N = 448;
constexpr int XR = 504;  // exchange scratch per transform, role-fastest mapping
constexpr int XC = 514;  // exchange scratch per transform, transform-fastest mapping

__device__ __forceinline__ float2 conjf2(float2 a) { return make_float2(a.x, -a.y); }

template <bool INV>
__device__ __forceinline__ float2 twid(const float2* __restrict__ t, int i) {
  const float2 w = __ldg(t + i);
  return INV ? conjf2(w) : w;
}

// Per-role twiddles, loaded once per thread (ahead of the data they scale):
// w1[k1-1] = w448^{r k1}, w3[m2-1] = w64^{m2 (r & 7)}.
struct Tw {
  float2 w1_[6];
  float2 w3_[7];
  __device__ __forceinline__ float2 w1(int k1) const { return w1_[k1 - 1]; }
  __device__ __forceinline__ float2 w3(int m2) const { return w3_[m2 - 1]; }
};

// Twiddles read at their point of use (fewer live registers).
struct TwLazy {
  const float2* __restrict__ t448;
  const float2* __restrict__ t64;
  int r;
  __device__ __forceinline__ float2 w1(int k1) const { return __ldg(t448 + (k1 - 1) * 64 + r); }
  __device__ __forceinline__ float2 w3(int m2) const { return __ldg(t64 + (m2 - 1) * 8 + (r & 7)); }
};

__device__ __forceinline__ void load_tw(Tw& tw, int r, const float2* __restrict__ tw448,
                                        const float2* __restrict__ tw64) {
#pragma unroll
  for (int k1 = 1; k1 < 7; ++k1) tw.w1_[k1 - 1] = __ldg(tw448 + (k1 - 1) * 64 + r);
#pragma unroll
  for (int m2 = 1; m2 < 8; ++m2) tw.w3_[m2 - 1] = __ldg(tw64 + (m2 - 1) * 8 + (r & 7));
}

template <bool INV>
__device__ __forceinline__ float2 tw_apply(float2 v, float2 w) {
  return cmul(v, INV ? conjf2(w) : w);
}

// Forward-ordered FFT.  a[n1] = x[64 n1 + r] on entry (all 64 roles).  On
// exit roles r < 56 hold X[k1 + 7 j1 + 56 j2] in b[j2].  S: this transform's
// scratch.  Contains three __syncthreads (every thread must call).
template <bool INV, class TW>
__device__ __forceinline__ void fwd(float2 (&a)[7], float2 (&b)[8], float2* S, int r, const TW& tw) {
  DftOdd<7, INV>::run(a);
#pragma unroll
  for (int k1 = 1; k1 < 7; ++k1) a[k1] = tw_apply<INV>(a[k1], tw.w1(k1));
#pragma unroll
  for (int k1 = 0; k1 < 7; ++k1) S[k1 * 72 + r] = a[k1];
  __syncthreads();
  const bool act = r < 56;
  const int k1 = r >> 3, lo = r & 7;
  if (act) {
#pragma unroll
    for (int m1 = 0; m1 < 8; ++m1) b[m1] = S[k1 * 72 + 8 * m1 + lo];
  }
  __syncthreads();
  if (act) {
    Dft<8, INV>::run(b);
#pragma unroll
    for (int j1 = 0; j1 < 8; ++j1) S[k1 * 72 + 9 * j1 + lo] = b[j1];
  }
  __syncthreads();
  if (act) {
#pragma unroll
    for (int m2 = 0; m2 < 8; ++m2) b[m2] = S[k1 * 72 + 9 * lo + m2];
#pragma unroll
    for (int m2 = 1; m2 < 8; ++m2) b[m2] = tw_apply<INV>(b[m2], tw.w3(m2));
    Dft<8, INV>::run(b);
  }
}

// Transposed FFT: roles r < 56 hold X[k1 + 7 j1 + 56 j2] in b[j2] on entry;
// on exit a[n1] = x[64 n1 + r] for all 64 roles.  Three __syncthreads.
template <bool INV, class TW>
__device__ __forceinline__ void inv(float2 (&b)[8], float2 (&a)[7], float2* S, int r, const TW& tw) {
  const bool act = r < 56;
  const int k1 = r >> 3, lo = r & 7;
  if (act) {
    Dft<8, INV>::run(b);  // over j2 -> m2
#pragma unroll
    for (int m2 = 1; m2 < 8; ++m2) b[m2] = tw_apply<INV>(b[m2], tw.w3(m2));
#pragma unroll
    for (int m2 = 0; m2 < 8; ++m2) S[k1 * 72 + 9 * lo + m2] = b[m2];
  }
  __syncthreads();
  if (act) {
#pragma unroll
    for (int j1 = 0; j1 < 8; ++j1) b[j1] = S[k1 * 72 + 9 * j1 + lo];
  }
  __syncthreads();
  if (act) {
    Dft<8, INV>::run(b);  // over j1 -> m1
#pragma unroll
    for (int m1 = 0; m1 < 8; ++m1) S[k1 * 72 + 8 * m1 + lo] = b[m1];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 7; ++q) a[q] = S[q * 72 + r];
#pragma unroll
  for (int q = 1; q < 7; ++q) a[q] = tw_apply<INV>(a[q], tw.w1(q));
  DftOdd<7, INV>::run(a);  // over k1 -> n1
}

}  // namespace f448

__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <bool LAZY> struct TwSel;
template <> struct TwSel<true> {
  __device__ __forceinline__ static f448::TwLazy make(const KParams& kp, int r) { return {kp.tw448, kp.tw64, r}; }
};
template <> struct TwSel<false> {
  __device__ __forceinline__ static f448::Tw make(const KParams& kp, int r) {
    f448::Tw t;
    f448::load_tw(t, r, kp.tw448, kp.tw64);
    return t;
  }
};

struct Dct14 {
  double c[3][14];  // orthonormal DCT-II rows u < 3 for P = 14
};

// ------------------------------------------------------------- K_A 448 ----
// One CTA per (stripe of 14 rows, stream); 448 threads.
// phase 0: TMA bulk copy of the stripe (two 7-row halves, two mbarriers);
// phase 1: thread = column: pixels -> fp64 luma (14 rows), flags, DCT
//          partials T[u][col] = sum_x C[u][x] X[x][col], s2[col] = sum_x X^2
//          (fp64), fp32 gray pairs for the FFT;
// phase 2: E = sum s2 - sum_{u,v<3} (sum_y T[u][y] C[v][y])^2 per patch;
// phase 3: 7 packed-pair forward FFTs (row pairs as complex);
// phase 4: split pairs, write packed half-spectrum columns to T1.
constexpr int kPxBytes448 = 14 * 448 * 12;  // largest stripe (fp32 RGB)
constexpr int kBC = 4;                       // packed columns per K_B CTA
constexpr int kNCB448 = 224 / kBC;           // column blocks
constexpr int kBP = 4;                       // row pairs per K_C CTA
constexpr int kNRG448 = 448 / (2 * kBP);     // row groups

template <int FMT>
__device__ __forceinline__ double smem_luma(const unsigned char* px, int i) {
  if constexpr (FMT == FC_FMT_RGB_F32) {
    const float* f = reinterpret_cast<const float*>(px) + 3 * i;
    return luma_f64(f[0], f[1], f[2]);
  } else if constexpr (FMT == FC_FMT_GRAY_F32) {
    return (double)reinterpret_cast<const float*>(px)[i];
  } else if constexpr (FMT == FC_FMT_GRAY_U8) {
    return gray_u8(px[i]);
  } else if constexpr (FMT == FC_FMT_RGB_U8) {
    return luma_u8(px[3 * i], px[3 * i + 1], px[3 * i + 2]);
  } else {
    return reinterpret_cast<const double*>(px)[i];
  }
}

template <int FMT>
__global__ void __launch_bounds__(448, 3) k448_rows_fwd(KParams kp, Dct14 dc, const void* __restrict__ frames,
                                                       int b0, int do_fft) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[2];
  constexpr int bpp = FMT == FC_FMT_RGB_F32 ? 12 : FMT == FC_FMT_GRAY_F32 ? 4 : FMT == FC_FMT_GRAY_U8 ? 1
                    : FMT == FC_FMT_RGB_U8 ? 3 : 8;
  const int s = blockIdx.x, bl = blockIdx.y, b = b0 + bl;
  const int t = threadIdx.x;
  // one 73.5 KB region: the staged stripe, then (after every pixel is read)
  // [zin 7x448 complex | DCT partials + corner squares | FFT scratch 7x504]
  unsigned char* px = smem;
  float2* zin = reinterpret_cast<float2*>(smem);                      // [7][448]
  double* part = reinterpret_cast<double*>(smem + 7 * 448 * 8);       // [4][32 x 15]
  double* ysq = part + 4 * 480;                                       // [9][32]
  float2* S = reinterpret_cast<float2*>(smem + 7 * 448 * 8 + (4 * 480 + 288) * 8);  // [7][504]

  // ---- phase 0: stage the stripe with the TMA engine
  const size_t row0 = ((size_t)b * 448 + (size_t)s * 14) * 448;
  if (t == 0) {
    tma::bar_init(&bar[0], 1);
    tma::bar_init(&bar[1], 1);
  }
  __syncthreads();
  if (t == 0) {
    const char* src = reinterpret_cast<const char*>(frames) + row0 * bpp;
    constexpr uint32_t half_bytes = 7 * 448 * bpp;
    tma::load_tile(px, src, half_bytes, &bar[0]);
    tma::load_tile(px + half_bytes, src + half_bytes, half_bytes, &bar[1]);
  }

  // ---- phase 1
  bool vary = false;
  unsigned emax = 0u;
  double ref = 0.0;
  double s2 = 0.0, tu0 = 0.0, tu1 = 0.0, tu2 = 0.0;
  float g32[14];
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    tma::bar_wait(&bar[half], 0);
    if (half == 0) ref = smem_luma<FMT>(px, 0);
#pragma unroll
    for (int x = 0; x < 7; ++x) {
      const int xx = half * 7 + x;
      const double v = smem_luma<FMT>(px, xx * 448 + t);
      g32[xx] = (float)v;
      vary |= (v != ref);
      emax = max(emax, (unsigned)__double2hiint(v) & 0x7ff00000u);
      s2 = fma(v, v, s2);
      tu0 = fma(dc.c[0][xx], v, tu0);
      tu1 = fma(dc.c[1][xx], v, tu1);
      tu2 = fma(dc.c[2][xx], v, tu2);
    }
  }
  const int anyvary = __syncthreads_or(vary);  // also: every pixel has been read
  const int anybad = __syncthreads_or(emax == 0x7ff00000u);
  // fp32 gray as packed row pairs (2g, 2g+1), over the consumed stripe
#pragma unroll
  for (int g = 0; g < 7; ++g) zin[g * 448 + t] = make_float2(g32[2 * g], g32[2 * g + 1]);
  // per-patch stride 15 (one pad double): phase-2 reads of 32 patches hit
  // 16 distinct bank pairs per half-warp
  {
    const int pp = t / 14, y = t - (t / 14) * 14;
    double* pc = part + pp * 15 + y;
    pc[0 * 480] = tu0;
    pc[1 * 480] = tu1;
    pc[2 * 480] = tu2;
    pc[3 * 480] = s2;
  }
  if (t == 0) {
    StripeStat st;
    st.ref = ref; st.unused = 0.0; st.nonfinite = anybad; st.varying = anyvary;
    st.pad[0] = st.pad[1] = 0;
    kp.stripes[(size_t)b * 32 + s] = st;
  }
  __syncthreads();
  // ---- phase 2: low-frequency corner per patch (fp64); warp = (u, v), lane = patch
  if (t < 288) {
    const int uv = t >> 5, pp = t & 31, u = uv / 3, v = uv - (uv / 3) * 3;
    const double* tp = part + u * 480 + pp * 15;
    double y = 0.0;
#pragma unroll
    for (int q = 0; q < 14; ++q) y = fma(tp[q], dc.c[v][q], y);
    ysq[t] = y * y;
  }
  __syncthreads();
  if (t < 32) {
    const double* sp = part + 3 * 480 + t * 15;
    double e = 0.0;
#pragma unroll
    for (int q = 0; q < 14; ++q) e += sp[q];
    double low = 0.0;
#pragma unroll
    for (int q = 0; q < 9; ++q) low += ysq[q * 32 + t];
    e -= low;
    kp.energy[(size_t)b * 1024 + s * 32 + t] = e > 0.0 ? e : 0.0;
  }
  if (!do_fft) return;
  __syncthreads();  // part/ysq (aliasing S) consumed

  // ---- phase 3: packed-pair forward FFTs, g = pair, r = role
  const int g = t >> 6, r = t & 63;
  float2 a[7], bv[8];
#pragma unroll
  for (int n1 = 0; n1 < 7; ++n1) a[n1] = zin[g * 448 + 64 * n1 + r];
  const f448::TwLazy tw{kp.tw448, kp.tw64, r};
  f448::fwd<false>(a, bv, S + g * f448::XR, r, tw);
  float2* zout = zin;  // zin fully consumed before fwd's first barrier
  if (r < 56) {
    const int k1 = r >> 3, j1 = r & 7;
#pragma unroll
    for (int j2 = 0; j2 < 8; ++j2) zout[g * 448 + k1 + 7 * j1 + 56 * j2] = bv[j2];
  }
  __syncthreads();

  // ---- phase 4: split the two real rows' spectra, write packed columns
  for (int idx = t; idx < 7 * 224; idx += 448) {
    const int gg = idx / 224, q = idx - (idx / 224) * 224;
    const float2* Z = zout + gg * 448;
    float2 xa, xb;
    if (q == 0) {
      const float2 z0 = Z[0], zn = Z[224];
      xa = make_float2(z0.x, zn.x);
      xb = make_float2(z0.y, zn.y);
    } else {
      const float2 za = Z[q], zm = Z[448 - q];
      xa = make_float2(0.5f * (za.x + zm.x), 0.5f * (za.y - zm.y));
      xb = make_float2(0.5f * (za.y + zm.y), -0.5f * (za.x - zm.x));
    }
    const int ra = s * 14 + 2 * gg;
    float2* dst = kp.T + (((size_t)bl * kNCB448 + q / kBC) * 448 + ra) * kBC + (q % kBC);
    dst[0] = xa;
    dst[kBC] = xb;
  }
}

// ------------------------------------------------------------- K_B 448 ----
// One CTA per (kBC-column block, stream); 64*kBC threads, column c = t % kBC
// fastest.  The T1 block and the stream's previous spectrum are staged by
// two TMA bulk copies at kernel start.  State layout is the register order
// of the forward column FFT: spec[b][cb][i][t] float4 (j2 = 2i, 2i+1), so
// the state swap is coalesced and its shared-memory reads conflict-free.
constexpr int kT1Block = 448 * kBC * 8;      // bytes
constexpr int kStBlock = 64 * kBC * 8 * 8;   // bytes
constexpr int kXCB = 516;                    // scratch stride, 4 interleaved transforms
constexpr int kScratchB = kBC * kXCB * 8;

template <int MINB, bool LAZY>
__global__ void __launch_bounds__(64 * kBC, MINB) k448_cols(KParams kp, int b0) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ double red[16 * 4];
  const int cb = blockIdx.x, bl = blockIdx.y, b = b0 + bl;
  const int t = threadIdx.x;
  const int c = t % kBC, r = t / kBC;
  float2* t1 = reinterpret_cast<float2*>(smem);                   // T1 block, then scratch
  float2* S = reinterpret_cast<float2*>(smem) + c * kXCB;         // [kBC][516] (aliases t1)
  float2* prev = reinterpret_cast<float2*>(smem + kScratchB);     // [64 kBC][8]
  float2* col0 = prev + 64 * kBC * 8;                             // [2][448] (cb == 0)
  const bool valid = kp.hdr[b].valid != 0;
  float2* stg = kp.spec + (((size_t)b * kNCB448 + cb) * 64 * kBC) * 8;
  if (t == 0) {
    tma::bar_init(&bar[0], 1);
    tma::bar_init(&bar[1], 1);
  }
  __syncthreads();
  if (t == 0) {
    tma::load_tile(t1, kp.T + ((size_t)bl * kNCB448 + cb) * 448 * kBC, kT1Block, &bar[0]);
    if (valid) tma::load_tile(prev, stg, kStBlock, &bar[1]);
  }
  const auto tw = TwSel<LAZY>::make(kp, r);
  tma::bar_wait(&bar[0], 0);
  float2 a[7], v[8];
#pragma unroll
  for (int n1 = 0; n1 < 7; ++n1) a[n1] = t1[64 * kBC * n1 + t];
  __syncthreads();  // t1 consumed: scratch may overwrite it
  f448::fwd<false>(a, v, S, r, tw);

  const bool act = r < 56;
  const int k1 = r >> 3, j1 = r & 7;
  float4* st = reinterpret_cast<float4*>(stg) + t;  // chunk i at st[i * 64 * kBC]
  // the previous spectrum must have landed before this block is overwritten
  if (valid) tma::bar_wait(&bar[1], 0);
  __syncthreads();
  if (act) {
#pragma unroll
    for (int i = 0; i < 4; ++i) st[i * 64 * kBC] = make_float4(v[2 * i].x, v[2 * i].y, v[2 * i + 1].x, v[2 * i + 1].y);
  }
  if (!valid) return;  // cold stream: spectrum established (block-uniform)
  float2 p[8];
  if (act) {
    const float4* pv = reinterpret_cast<const float4*>(prev) + t;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float4 q = pv[i * 64 * kBC];
      p[2 * i] = make_float2(q.x, q.y);
      p[2 * i + 1] = make_float2(q.z, q.w);
    }
  }
  float spc = 0.f, spp = 0.f, scc = 0.f, splp = 0.f;
  auto acc = [&](float w, float2 fp, float2 fc) -> float2 {
    const float pp = fp.x * fp.x + fp.y * fp.y;
    const float pc = fc.x * fc.x + fc.y * fc.y;
    const float m = sqrt_approx(pp * pc);  // |Fp| |Fc|
    spc = fmaf(w, m, spc);
    spp = fmaf(w, pp, spp);
    scc = fmaf(w, pc, scc);
    if (pc > 0.f) splp = fmaf(w * pc, __logf(pc), splp);
    // normalised cross-power (migration.py:130-131)
    const float inv = rcp_approx(m + 1e-12f);
    return make_float2((fp.x * fc.x + fp.y * fc.y) * inv, (fp.y * fc.x - fp.x * fc.y) * inv);
  };
  if (cb == 0) {
    // packed DC/Nyquist column: needs bins k and 448-k of both spectra
    if (c == 0 && act) {
#pragma unroll
      for (int j2 = 0; j2 < 8; ++j2) {
        const int k = k1 + 7 * j1 + 56 * j2;
        col0[k] = v[j2];
        col0[448 + k] = p[j2];
      }
    }
    __syncthreads();
    if (c == 0 && act) {
#pragma unroll
      for (int j2 = 0; j2 < 8; ++j2) {
        const int k = k1 + 7 * j1 + 56 * j2;
        const int km = (448 - k) % 448;
        float2 c0, cn, p0, pn;
        unpack_dcny(v[j2], col0[km], c0, cn);
        unpack_dcny(p[j2], col0[448 + km], p0, pn);
        const float2 x0 = acc(1.f, p0, c0);
        const float2 xn = acc(1.f, pn, cn);
        v[j2] = make_float2(x0.x - xn.y, x0.y + xn.x);
      }
    }
  }
  if (act && !(cb == 0 && c == 0)) {
#pragma unroll
    for (int j2 = 0; j2 < 8; ++j2) v[j2] = acc(2.f, p[j2], v[j2]);
  }
  f448::inv<true>(v, a, S, r, tw);
  float2* T2 = kp.T2 + (size_t)bl * 448 * 224 + cb * kBC + c;
#pragma unroll
  for (int n1 = 0; n1 < 7; ++n1) T2[(size_t)(64 * n1 + r) * 224] = a[n1];

  const float fs[4] = {spc, spp, scc, splp};
  double sums[4];
  block_sum_f2d<4>(fs, sums, red);
  if (t == 0) {
    double* o = kp.stats + ((size_t)b * kNCB448 + cb) * 4;
    o[0] = sums[0]; o[1] = sums[1]; o[2] = sums[2]; o[3] = sums[3];
  }
}

// ------------------------------------------------------------- K_C 448 ----
// One CTA per (2 kBP rows, stream); 64*kBP threads = kBP row pairs x 64 roles.
// The rows of T2 (contiguous) arrive by one TMA bulk copy.
constexpr int kT2Rows = 2 * kBP * 224 * 8;  // bytes

template <int MINB, bool LAZY>
__global__ void __launch_bounds__(64 * kBP, MINB) k448_rows_inv(KParams kp, int b0) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ PeakKey redk[16];
  __shared__ float redv[16];
  const int gidx = blockIdx.x, bl = blockIdx.y, b = b0 + bl;
  const int t = threadIdx.x;
  float2* tin = reinterpret_cast<float2*>(smem);  // [2 kBP][224], then scratch
  const int y0 = gidx * 2 * kBP;
  if (t == 0) {
    tma::bar_init(&bar, 1);
    tma::load_tile(tin, kp.T2 + ((size_t)bl * 448 + y0) * 224, kT2Rows, &bar);  // same thread: ordered
  }
  const int g = t >> 6, r = t & 63;
  const auto tw = TwSel<LAZY>::make(kp, r);
  const bool valid = kp.hdr[b].valid != 0;
  __syncthreads();  // barrier initialised
  tma::bar_wait(&bar, 0);  // also when cold: the CTA must not exit with a copy in flight
  if (!valid) return;
  const int k1 = r >> 3, j1 = r & 7;
  float2 v[8], a[7];
  if (r < 56) {
    const float2* ga = tin + (2 * g) * 224;
    const float2* gb = ga + 224;
#pragma unroll
    for (int j2 = 0; j2 < 8; ++j2) {
      const int k = k1 + 7 * j1 + 56 * j2;
      float2 z;
      if (k == 0) {
        z = make_float2(ga[0].x, gb[0].x);
      } else if (k == 224) {
        z = make_float2(ga[0].y, gb[0].y);
      } else if (k < 224) {
        const float2 A = ga[k], B = gb[k];
        z = make_float2(A.x - B.y, A.y + B.x);   // G_a + i G_b
      } else {
        const float2 A = ga[448 - k], B = gb[448 - k];
        z = make_float2(A.x + B.y, B.x - A.y);   // conj G_a + i conj G_b
      }
      v[j2] = z;
    }
  }
  __syncthreads();  // tin consumed; scratch aliases it
  f448::inv<true>(v, a, tin + g * f448::XR, r, tw);

  // argmax with the reference tie rule (migration.py:141-159): max, its
  // first position, runner-up; exact ties inside a thread take a slow path
  const int ya = y0 + 2 * g;
  float m1 = -CUDART_INF_F, m2 = -CUDART_INF_F;
  int ai = 0;
#pragma unroll
  for (int k = 0; k < 14; ++k) {
    const float val = (k & 1) ? a[k >> 1].y : a[k >> 1].x;
    if (val > m1) { m2 = m1; m1 = val; ai = k; }
    else m2 = fmaxf(m2, val);
  }
  auto key_of = [&](int k, float val) {
    PeakKey c;
    const int y = ya + (k & 1), j = 64 * (k >> 1) + r;
    c.v = val;
    c.l1 = abs(canon_disp(y, 448)) + abs(canon_disp(j, 448));
    c.pos = y * 448 + j;
    return c;
  };
  PeakKey best = key_of(ai, m1);
  if (m2 == m1) {
    for (int k = 0; k < 14; ++k) {
      const float val = (k & 1) ? a[k >> 1].y : a[k >> 1].x;
      if (val == m1) {
        const PeakKey c = key_of(k, val);
        if (peak_better(c, best)) best = c;
      }
    }
  }
  float v2 = m2;
  const int lane = t & 31, wid = t >> 5;
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
  if (t == 0) {
    for (int w = 1; w < (64 * kBP) / 32; ++w) {
      const PeakKey o = redk[w];
      if (peak_better(o, best)) { v2 = fmaxf(fmaxf(v2, redv[w]), best.v); best = o; }
      else v2 = fmaxf(fmaxf(v2, redv[w]), o.v);
    }
    PeakPart pp;
    pp.v = best.v; pp.v2 = v2; pp.y = best.pos / 448; pp.j = best.pos % 448;
    kp.peaks[(size_t)b * kNRG448 + gidx] = pp;
  }
}

// ------------------------------------------------- persistent K_B / K_C ----
// Same math as k448_cols / k448_rows_inv, but a grid of (SMs x occupancy)
// CTAs walks the work items with a two-stage TMA ring: while item k is
// computed, the tiles of item k+1 are already in flight (mbarrier per stage,
// parity = (k >> 1) & 1).  Before a stage is refilled by the async proxy the
// generic accesses to it are fenced (fence.proxy.async).
namespace pers {
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
}  // namespace pers

constexpr int kStageB = ((kScratchB > kT1Block ? kScratchB : kT1Block) + 127) / 128 * 128 + kStBlock;
constexpr int kSmemBP = 2 * kStageB + 2 * 448 * 8;

__device__ __forceinline__ void colsp_issue(const KParams& kp, int b0, int it, int nitems, unsigned char* stage,
                                            uint64_t* bar) {
  if (it >= nitems) return;
  const int bl = it / kNCB448, cb = it - (it / kNCB448) * kNCB448, b = b0 + bl;
  const bool valid = kp.hdr[b].valid != 0;
  const uint32_t bytes = kT1Block + (valid ? kStBlock : 0);
  tma::bar_expect(bar, bytes);
  tma::bulk_g2s(stage, kp.T + ((size_t)bl * kNCB448 + cb) * 448 * kBC, kT1Block, bar);
  if (valid)
    tma::bulk_g2s(stage + kStageB - kStBlock, kp.spec + (((size_t)b * kNCB448 + cb) * 64 * kBC) * 8, kStBlock, bar);
}

__global__ void __launch_bounds__(64 * kBC, 3) k448_cols_p(KParams kp, int b0, int nb) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ double red[16 * 4];
  const int t = threadIdx.x;
  const int c = t % kBC, r = t / kBC;
  const int nitems = nb * kNCB448;
  float2* col0 = reinterpret_cast<float2*>(smem + 2 * kStageB);  // [2][448]
  f448::Tw tw;
  f448::load_tw(tw, r, kp.tw448, kp.tw64);
  if (t == 0) {
    tma::bar_init(&bar[0], 1);
    tma::bar_init(&bar[1], 1);
  }
  __syncthreads();
  if (t == 0) {
    colsp_issue(kp, b0, blockIdx.x, nitems, smem, &bar[0]);
    colsp_issue(kp, b0, blockIdx.x + gridDim.x, nitems, smem + kStageB, &bar[1]);
  }
  int k = 0;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x, ++k) {
    const int sidx = k & 1;
    unsigned char* stage = smem + sidx * kStageB;
    const int bl = it / kNCB448, cb = it - (it / kNCB448) * kNCB448, b = b0 + bl;
    const bool valid = kp.hdr[b].valid != 0;
    float2* t1 = reinterpret_cast<float2*>(stage);
    float2* S = t1 + c * kXCB;
    const float2* prev = reinterpret_cast<const float2*>(stage + kStageB - kStBlock);
    float2* stg = kp.spec + (((size_t)b * kNCB448 + cb) * 64 * kBC) * 8;
    tma::bar_wait(&bar[sidx], (k >> 1) & 1);
    float2 a[7], v[8];
#pragma unroll
    for (int n1 = 0; n1 < 7; ++n1) a[n1] = t1[64 * kBC * n1 + t];
    __syncthreads();  // t1 consumed: scratch may overwrite it
    f448::fwd<false>(a, v, S, r, tw);
    const bool act = r < 56;
    const int k1 = r >> 3, j1 = r & 7;
    float4* st = reinterpret_cast<float4*>(stg) + t;  // chunk i at st[i * 64 * kBC]
    if (act) {
#pragma unroll
      for (int i = 0; i < 4; ++i) st[i * 64 * kBC] = make_float4(v[2 * i].x, v[2 * i].y, v[2 * i + 1].x, v[2 * i + 1].y);
    }
    if (valid) {
      float2 p[8];
      if (act) {
        const float4* pv = reinterpret_cast<const float4*>(prev) + t;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float4 q = pv[i * 64 * kBC];
          p[2 * i] = make_float2(q.x, q.y);
          p[2 * i + 1] = make_float2(q.z, q.w);
        }
      }
      float spc = 0.f, spp = 0.f, scc = 0.f, splp = 0.f;
      auto acc = [&](float w, float2 fp, float2 fc) -> float2 {
        const float pp = fp.x * fp.x + fp.y * fp.y;
        const float pc = fc.x * fc.x + fc.y * fc.y;
        const float m = sqrt_approx(pp * pc);  // |Fp| |Fc|
        spc = fmaf(w, m, spc);
        spp = fmaf(w, pp, spp);
        scc = fmaf(w, pc, scc);
        if (pc > 0.f) splp = fmaf(w * pc, __logf(pc), splp);
        const float inv = rcp_approx(m + 1e-12f);  // migration.py:130-131
        return make_float2((fp.x * fc.x + fp.y * fc.y) * inv, (fp.y * fc.x - fp.x * fc.y) * inv);
      };
      if (cb == 0) {
        if (c == 0 && act) {
#pragma unroll
          for (int j2 = 0; j2 < 8; ++j2) {
            const int kk = k1 + 7 * j1 + 56 * j2;
            col0[kk] = v[j2];
            col0[448 + kk] = p[j2];
          }
        }
        __syncthreads();
        if (c == 0 && act) {
#pragma unroll
          for (int j2 = 0; j2 < 8; ++j2) {
            const int kk = k1 + 7 * j1 + 56 * j2;
            const int km = (448 - kk) % 448;
            float2 c0, cn, p0, pn;
            unpack_dcny(v[j2], col0[km], c0, cn);
            unpack_dcny(p[j2], col0[448 + km], p0, pn);
            const float2 x0 = acc(1.f, p0, c0);
            const float2 xn = acc(1.f, pn, cn);
            v[j2] = make_float2(x0.x - xn.y, x0.y + xn.x);
          }
        }
      }
      if (act && !(cb == 0 && c == 0)) {
#pragma unroll
        for (int j2 = 0; j2 < 8; ++j2) v[j2] = acc(2.f, p[j2], v[j2]);
      }
      f448::inv<true>(v, a, S, r, tw);
      float2* T2 = kp.T2 + (size_t)bl * 448 * 224 + cb * kBC + c;
#pragma unroll
      for (int n1 = 0; n1 < 7; ++n1) T2[(size_t)(64 * n1 + r) * 224] = a[n1];
      const float fs[4] = {spc, spp, scc, splp};
      double sums[4];
      block_sum_f2d<4>(fs, sums, red);
      if (t == 0) {
        double* o = kp.stats + ((size_t)b * kNCB448 + cb) * 4;
        o[0] = sums[0]; o[1] = sums[1]; o[2] = sums[2]; o[3] = sums[3];
      }
    }
    __syncthreads();  // stage fully consumed (scratch, prev, col0)
    if (t == 0) {
      pers::fence_async_smem();
      colsp_issue(kp, b0, it + 2 * gridDim.x, nitems, stage, &bar[sidx]);
    }
  }
}

constexpr int kStageC = ((kBP * f448::XR * 8 > kT2Rows ? kBP * f448::XR * 8 : kT2Rows) + 127) / 128 * 128;
constexpr int kSmemCP = 2 * kStageC;

__device__ __forceinline__ void rowsp_issue(const KParams& kp, int it, int nitems, unsigned char* stage,
                                            uint64_t* bar) {
  if (it >= nitems) return;
  const int bl = it / kNRG448, gidx = it - (it / kNRG448) * kNRG448;
  tma::bar_expect(bar, kT2Rows);
  tma::bulk_g2s(stage, kp.T2 + ((size_t)bl * 448 + gidx * 2 * kBP) * 224, kT2Rows, bar);
}

__global__ void __launch_bounds__(64 * kBP, 4) k448_rows_inv_p(KParams kp, int b0, int nb) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ PeakKey redk[16];
  __shared__ float redv[16];
  const int t = threadIdx.x;
  const int nitems = nb * kNRG448;
  const int g = t >> 6, r = t & 63;
  const int k1 = r >> 3, j1 = r & 7;
  f448::Tw tw;
  f448::load_tw(tw, r, kp.tw448, kp.tw64);
  if (t == 0) {
    tma::bar_init(&bar[0], 1);
    tma::bar_init(&bar[1], 1);
  }
  __syncthreads();
  if (t == 0) {
    rowsp_issue(kp, blockIdx.x, nitems, smem, &bar[0]);
    rowsp_issue(kp, blockIdx.x + gridDim.x, nitems, smem + kStageC, &bar[1]);
  }
  int k = 0;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x, ++k) {
    const int sidx = k & 1;
    float2* tin = reinterpret_cast<float2*>(smem + sidx * kStageC);
    const int bl = it / kNRG448, gidx = it - (it / kNRG448) * kNRG448, b = b0 + bl;
    const bool valid = kp.hdr[b].valid != 0;
    const int y0 = gidx * 2 * kBP;
    tma::bar_wait(&bar[sidx], (k >> 1) & 1);
    if (valid) {
      float2 v[8], a[7];
      if (r < 56) {
        const float2* ga = tin + (2 * g) * 224;
        const float2* gb = ga + 224;
#pragma unroll
        for (int j2 = 0; j2 < 8; ++j2) {
          const int kk = k1 + 7 * j1 + 56 * j2;
          float2 z;
          if (kk == 0) {
            z = make_float2(ga[0].x, gb[0].x);
          } else if (kk == 224) {
            z = make_float2(ga[0].y, gb[0].y);
          } else if (kk < 224) {
            const float2 A = ga[kk], B = gb[kk];
            z = make_float2(A.x - B.y, A.y + B.x);
          } else {
            const float2 A = ga[448 - kk], B = gb[448 - kk];
            z = make_float2(A.x + B.y, B.x - A.y);
          }
          v[j2] = z;
        }
      }
      __syncthreads();  // tin consumed; scratch aliases it
      f448::inv<true>(v, a, tin + g * f448::XR, r, tw);
      const int ya = y0 + 2 * g;
      float m1 = -CUDART_INF_F, m2 = -CUDART_INF_F;
      int ai = 0;
#pragma unroll
      for (int q = 0; q < 14; ++q) {
        const float val = (q & 1) ? a[q >> 1].y : a[q >> 1].x;
        if (val > m1) { m2 = m1; m1 = val; ai = q; }
        else m2 = fmaxf(m2, val);
      }
      auto key_of = [&](int q, float val) {
        PeakKey kq;
        const int y = ya + (q & 1), j = 64 * (q >> 1) + r;
        kq.v = val;
        kq.l1 = abs(canon_disp(y, 448)) + abs(canon_disp(j, 448));
        kq.pos = y * 448 + j;
        return kq;
      };
      PeakKey best = key_of(ai, m1);
      if (m2 == m1) {
        for (int q = 0; q < 14; ++q) {
          const float val = (q & 1) ? a[q >> 1].y : a[q >> 1].x;
          if (val == m1) {
            const PeakKey kq = key_of(q, val);
            if (peak_better(kq, best)) best = kq;
          }
        }
      }
      float v2 = m2;
      const int lane = t & 31, wid = t >> 5;
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
      if (t == 0) {
        for (int w = 1; w < (64 * kBP) / 32; ++w) {
          const PeakKey o = redk[w];
          if (peak_better(o, best)) { v2 = fmaxf(fmaxf(v2, redv[w]), best.v); best = o; }
          else v2 = fmaxf(fmaxf(v2, redv[w]), o.v);
        }
        PeakPart pp;
        pp.v = best.v; pp.v2 = v2; pp.y = best.pos / 448; pp.j = best.pos % 448;
        kp.peaks[(size_t)b * kNRG448 + gidx] = pp;
      }
    }
    __syncthreads();  // stage consumed (input + scratch)
    if (t == 0) {
      pers::fence_async_smem();
      rowsp_issue(kp, it + 2 * gridDim.x, nitems, reinterpret_cast<unsigned char*>(tin), &bar[sidx]);
    }
  }
}
