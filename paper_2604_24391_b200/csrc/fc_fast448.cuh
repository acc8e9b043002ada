// Fast path for the BASELINE geometry (448 x 448 frames, P = 14, N = 1024):
// K_A, the row pass (stripe luma + block-DCT energies + packed-pair row
// FFTs).  The 448-point FFT itself (7 x 8 x 8, one transform per warp) is
// in fc_wfft448.cuh; K_B / K_C are in fc_fast448w.cuh.
#pragma once
#include "fc_fft.cuh"
#include "fc_tma.cuh"
#include "fc_wfft448.cuh"

struct Dct14 {
  double c[3][14];  // orthonormal DCT-II rows u < 3 for P = 14
};

// ------------------------------------------------------------- K_A 448 ----
// One CTA per (stripe of 14 rows, stream); 7 warps, warp g owns row pair
// (2g, 2g + 1) for the FFT, thread t owns columns (2t, 2t + 1) for the DCT.
// phase 0: TMA bulk copies of the stripe, one per row pair (7 mbarriers), so
//          phase 1 starts on the first pair while the rest is in flight;
// phase 1: thread = column pair: pixels -> fp64 luma, flags, DCT partials
//          T[u][col] = sum_x C[u][x] X[x][col], s2[col] = sum_x X^2 (fp64),
//          fp32 gray kept for the FFT;
// phase 2: E = sum s2 - sum_{u,v<3} (sum_y T[u][y] C[v][y])^2 per patch;
// phase 3: warp g: packed-pair forward FFT of rows (2g, 2g + 1) (w448);
// phase 4: split pairs, write packed half-spectrum columns to T1, which is
//          column-major ([stream][q][448 rows] complex64): K_B stages one
//          contiguous 3.5 KB column per warp.
constexpr int kPxBytes448 = 14 * 448 * 12;  // largest stripe (fp32 RGB)
constexpr int kThreadsA448 = 224;
// shared memory after phase 1 (aliasing the consumed stripe):
// [zin 7x448 | part 4x(32x15) + ysq 9x32 (fp64)] then zout [448][9] over
// both, and the per-warp FFT scratch 7 x 504 after them
constexpr int kZinBytes = 7 * 448 * 8;
constexpr int kPartBytes = (4 * 480 + 288) * 8;
static_assert((9 * 447 + 3 * (447 / 7) + 7) * 8 <= kZinBytes + kPartBytes, "zout must not reach the FFT scratch");
static_assert(kZinBytes + kPartBytes + 7 * 504 * 8 <= kPxBytes448, "K_A shared memory");
static_assert(224 * 112 + 127 <= 7 * 504 * 8, "T1 tile (aligned) must fit the FFT scratch");

// Gray values of two horizontally adjacent pixels i, i + 1 (i even).
template <int FMT>
__device__ __forceinline__ void smem_luma2(const unsigned char* px, int i, double& v0, double& v1) {
  if constexpr (FMT == FC_FMT_RGB_F32) {
    const float2* f = reinterpret_cast<const float2*>(px + 12 * (size_t)i);
    const float2 a = f[0], b = f[1], c = f[2];  // R0 G0 | B0 R1 | G1 B1
    v0 = luma_f64(a.x, a.y, b.x);
    v1 = luma_f64(b.y, c.x, c.y);
  } else if constexpr (FMT == FC_FMT_GRAY_F32) {
    const float2 f = *reinterpret_cast<const float2*>(px + 4 * (size_t)i);
    v0 = (double)f.x;
    v1 = (double)f.y;
  } else if constexpr (FMT == FC_FMT_GRAY_U8) {
    v0 = gray_u8(px[i]);
    v1 = gray_u8(px[i + 1]);
  } else if constexpr (FMT == FC_FMT_RGB_U8) {
    const unsigned char* q = px + 3 * (size_t)i;
    v0 = luma_u8(q[0], q[1], q[2]);
    v1 = luma_u8(q[3], q[4], q[5]);
  } else {
    const double2 f = *reinterpret_cast<const double2*>(px + 8 * (size_t)i);
    v0 = f.x;
    v1 = f.y;
  }
}

// TMST: the stripe's T1 block (224 columns x 14 rows) is assembled in shared
// memory and leaves through one TMA tensor store instead of per-thread stores.
template <int FMT, bool TMST>
__global__ void __launch_bounds__(kThreadsA448, 3) k448_rows_fwd(KParams kp, Dct14 dc, const void* __restrict__ frames,
                                                                int b0, int do_fft,
                                                                const __grid_constant__ CUtensorMap tmT1) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[7];
  __shared__ int sh_bad;
  constexpr int bpp = FMT == FC_FMT_RGB_F32 ? 12 : FMT == FC_FMT_GRAY_F32 ? 4 : FMT == FC_FMT_GRAY_U8 ? 1
                    : FMT == FC_FMT_RGB_U8 ? 3 : 8;
  constexpr uint32_t pair_bytes = 2 * 448 * bpp;
  const int s = blockIdx.x, bl = blockIdx.y, b = b0 + bl;
  const int t = threadIdx.x, wid = t >> 5, lane = t & 31;
  unsigned char* px = smem;
  float2* zin = reinterpret_cast<float2*>(smem);                     // [7][448]
  double* part = reinterpret_cast<double*>(smem + kZinBytes);        // [4][32 x 15]
  double* ysq = part + 4 * 480;                                      // [9][32]
  float2* S = reinterpret_cast<float2*>(smem + kZinBytes + kPartBytes) + wid * w448::XS;

  // ---- phase 0: stage the stripe with the TMA engine, one copy per row pair
  const size_t row0 = ((size_t)b * 448 + (size_t)s * 14) * 448;
  if (t == 0) {
    sh_bad = 0;
#pragma unroll
    for (int g = 0; g < 7; ++g) tma::bar_init(&bar[g], 1);
    const char* src = reinterpret_cast<const char*>(frames) + row0 * bpp;
#pragma unroll
    for (int g = 0; g < 7; ++g) tma::load_tile(px + g * pair_bytes, src + g * pair_bytes, pair_bytes, &bar[g]);
  }
  __syncthreads();  // barriers initialised

  // ---- phase 1: thread = columns (2t, 2t + 1)
  bool vary = false;
  double ref = 0.0;
  double s2[2] = {0.0, 0.0}, tu0[2] = {0.0, 0.0}, tu1[2] = {0.0, 0.0}, tu2[2] = {0.0, 0.0};
  float g32[14][2];
#pragma unroll
  for (int g = 0; g < 7; ++g) {
    tma::bar_wait(&bar[g], 0);
    if (g == 0) {
      double r1;
      smem_luma2<FMT>(px, 0, ref, r1);
    }
#pragma unroll
    for (int x2 = 0; x2 < 2; ++x2) {
      const int xx = 2 * g + x2;
      double v[2];
      smem_luma2<FMT>(px, xx * 448 + 2 * t, v[0], v[1]);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        g32[xx][c] = (float)v[c];
        vary |= (v[c] != ref);
        s2[c] = fma(v[c], v[c], s2[c]);
        tu0[c] = fma(dc.c[0][xx], v[c], tu0[c]);
        tu1[c] = fma(dc.c[1][xx], v[c], tu1[c]);
        tu2[c] = fma(dc.c[2][xx], v[c], tu2[c]);
      }
    }
  }
  const int anyvary = __syncthreads_or(vary);  // also: every pixel has been read
  // a NaN / Inf pixel makes its column's sum of squares non-finite (the
  // squares of finite fp32-derived values cannot overflow fp64); the flag is
  // read after the next barrier
  if (!isfinite(s2[0]) || !isfinite(s2[1])) sh_bad = 1;
  // fp32 gray as packed row pairs (2g, 2g+1), over the consumed stripe
#pragma unroll
  for (int g = 0; g < 7; ++g)
    *reinterpret_cast<float4*>(zin + g * 448 + 2 * t) =
        make_float4(g32[2 * g][0], g32[2 * g + 1][0], g32[2 * g][1], g32[2 * g + 1][1]);
  // per-patch stride 15 (one pad double): phase-2 reads of 32 patches hit
  // 16 distinct bank pairs per half-warp
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const int col = 2 * t + c, pp = col / 14, y = col - (col / 14) * 14;
    double* pc = part + pp * 15 + y;
    pc[0 * 480] = tu0[c];
    pc[1 * 480] = tu1[c];
    pc[2 * 480] = tu2[c];
    pc[3 * 480] = s2[c];
  }
  __syncthreads();
  if (t == 0) {
    StripeStat st;
    st.ref = ref; st.unused = 0.0; st.nonfinite = sh_bad; st.varying = anyvary;
    st.pad[0] = st.pad[1] = 0;
    kp.stripes[(size_t)b * 32 + s] = st;
  }
  // ---- phase 2: low-frequency corner per patch (fp64); (u, v) x patch
  for (int i = t; i < 288; i += kThreadsA448) {
    const int uv = i >> 5, pp = i & 31, u = uv / 3, v = uv - (uv / 3) * 3;
    const double* tp = part + u * 480 + pp * 15;
    double y = 0.0;
#pragma unroll
    for (int q = 0; q < 14; ++q) y = fma(tp[q], dc.c[v][q], y);
    ysq[i] = y * y;
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

  // ---- phase 3: warp g = row pair g: packed-pair forward FFT
  const int g = wid;
  float2 a[2][7], bv[2][8];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int n1 = 0; n1 < 7; ++n1) a[h][n1] = zin[g * 448 + 64 * n1 + lane + 32 * h];
  w448::TwLazy tw;
  tw.load(kp.tw448, kp.tw64, lane);
  w448::fwd<false>(a, bv, S, lane, tw);  // private scratch
  // zout: bin k of pair g at 9 k + g + 3 (k / 7), over zin and part (every
  // warp has loaded its zin row and phase 2 is done after this barrier); the
  // 3-slot skip every 7 bins makes the stores below bank-conflict free
  __syncthreads();
  float2* zout = zin;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (h == 0 || lane < 24) {
      const int k1 = (lane >> 3) + 4 * h, j1 = lane & 7;
#pragma unroll
      for (int j2 = 0; j2 < 8; ++j2) zout[(k1 + 7 * j1 + 56 * j2) * 9 + g + 3 * (j1 + 8 * j2)] = bv[h][j2];
    }
  }
  __syncthreads();

  // ---- phase 4: split the two real rows' spectra; consecutive threads take
  // consecutive row pairs of one column, so each column's 14 stripe rows
  // (112 contiguous bytes of T1) are written by neighbouring lanes.  Thread t
  // keeps row pair gg = t % 7 and walks columns t / 7 + 32 i (224 = 7 * 32).
  {
    const int gg = t % 7, q0 = t / 7;
    // TMST: tile [224 columns][7 row pairs] float4 over the FFT scratch (free
    // after the barrier above), 128-byte aligned; else straight to T1
    float4* tile = reinterpret_cast<float4*>(
        (reinterpret_cast<uintptr_t>(smem + kZinBytes + kPartBytes) + 127) & ~static_cast<uintptr_t>(127));
    float4* dst = TMST ? tile + gg
                       : reinterpret_cast<float4*>(kp.T + (size_t)bl * 224 * 448 + s * 14 + 2 * gg);
    constexpr int qstride = TMST ? 7 : 224;   // float4 per column
    auto zo = [](int k) { return 9 * k + 3 * (k / 7); };
    if (q0 == 0) {
      const float2 z0 = zout[gg], zn = zout[zo(224) + gg];
      dst[0] = make_float4(z0.x, zn.x, z0.y, zn.y);
    }
#pragma unroll
    for (int i = 0; i < 7; ++i) {
      const int q = q0 + 32 * i;
      if (q == 0) continue;
      const float2 za = zout[zo(q) + gg], zm = zout[zo(448 - q) + gg];
      dst[(size_t)q * qstride] = make_float4(0.5f * (za.x + zm.x), 0.5f * (za.y - zm.y),
                                             0.5f * (za.y + zm.y), -0.5f * (za.x - zm.x));
    }
    if constexpr (TMST) {
      tma::fence_async_shared();
      __syncthreads();
      if (t == 0) {
        // box = 14 rows (x: 28 floats) x 224 columns of stream bl's T1
        tma::tensor_store_2d(&tmT1, tile, s * 28, bl * 224);
        tma::bulk_wait_read0();
      }
    }
  }
}
