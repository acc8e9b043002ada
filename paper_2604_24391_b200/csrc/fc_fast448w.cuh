// K_B and K_C of the 448 x 448 fast path (K_A is in fc_fast448.cuh, the
// warp-owned 448-point FFT in fc_wfft448.cuh).
//
// Both kernels are warp-owned: every 448-point transform belongs to one warp
// (w448 in fc_wfft448.cuh), every warp stages its own tiles with its own TMA
// bulk copies and mbarriers, and the FFT exchanges need only __syncwarp, so
// the warps of a CTA never wait for each other until the final (per-CTA)
// reduction.
//
// Spectrum intermediates are column-major per stream:
//   T1 [q][448 rows] complex64  (K_A -> K_B: row spectra, packed column q)
//   T2 [224 row pairs][q][2 rows] complex64  (K_B -> K_C: cross-power after the
//      inverse column FFT; a row pair is one contiguous 3.5 KB block for K_C;
//      K_B transposes its 4 columns through shared memory and writes 64-byte
//      runs)
// Per-stream state (the previous frame's half spectrum) is kept in the
// register order of K_B's forward transform:
//   spec [q][h][i][lane] float4 = (X[k(j2 = 2i)], X[k(j2 = 2i + 1)]) of group
//   g = lane + 32 h, k(j2) = (g >> 3) + 7 (g & 7) + 56 j2, half 1 holding
//   only its 24 active lanes (st_idx; 3,584 bytes per column)
// so a warp loads / stores its column with 16-byte coalesced accesses.
#pragma once
#include <type_traits>
#include "fc_fast448.cuh"
#include "fc_wfft448.cuh"

constexpr int kWarpsB = 4;                 // columns (warps) per K_B CTA
constexpr int kNCB448 = 224 / kWarpsB;     // K_B CTAs per stream = stats partials
constexpr int kWarpsC = 4;                 // row pairs (warps) per K_C CTA
constexpr int kNRG448 = 224 / kWarpsC;     // K_C CTAs per stream = peak partials
constexpr int kStCol = 2 * 4 * 32;         // float4 per state column block in shared memory
constexpr int kStColG = 4 * 32 + 4 * 24;   // float4 per state column in HBM: half 1 has 24 lanes
constexpr int kSlotB = 512;                // float2: T1 column (448), then FFT scratch (504)
constexpr int kSmemB448 = kWarpsB * (kSlotB * 8 + kStCol * 16);

// float4 index of (half h, pair i, lane) in a state column: half 0 holds
// lanes 0..31, half 1 only the 24 active lanes (groups g < 56), so the
// column is 3,584 bytes with nothing unused in HBM
__device__ __forceinline__ int st_idx(int h, int i, int lane) { return h == 0 ? i * 32 + lane : 128 + i * 24 + lane; }
static_assert(kWarpsB == 4 && 224 * 4 * 16 + 1023 <= kWarpsB * kStCol * 16, "T2 tile (aligned) must fit the prev blocks");
constexpr int kSmemC448 = kWarpsC * w448::XS * 8;

template <bool LAZY>
using W448Tw = typename std::conditional<LAZY, w448::TwLazy, w448::Tw>::type;

// fp64 warp sum in a fixed xor-tree order (deterministic)
__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------- K_B 448 ----
// One warp per packed column q of a stream: forward column FFT of the T1
// column, state swap (previous spectrum in, current out), Hermitian-weighted
// sums for sim_freq and the entropy (migration.py:87-105, budget.py:34-58),
// normalised cross-power (migration.py:128-131) and the inverse column FFT
// into T2.  Column 0 holds the packed DC / Nyquist columns (real along rows),
// unpacked with bins k and 448 - k of the same column.
// TMST: T2 leaves through one TMA tensor store per CTA (the tile's swizzle is
// the tensor map's 64-byte swizzle) instead of a copy loop over the threads.
// Static shared memory of one K_B item (per-warp mbarriers, warp partial sums).
struct ColsSh {
  uint64_t bar[kWarpsB][2];
  double red[kWarpsB][4];
};

// One K_B work item: column group cx of stream b0 + bl.  FLOW: the item runs
// inside k448_bc_flow; thread 0 commits the T2 tensor store and returns
// without waiting for it (the flow loop publishes it later, see there).
// Returns false for a cold stream (no T2 written).
template <bool LAZY, bool TMST, bool FLOW>
__device__ __forceinline__ bool cols_item(const KParams& kp, int b0, int cx, int bl, const CUtensorMap* tmT2,
                                          unsigned char* smem, ColsSh& sh) {
  auto& bar = sh.bar;
  auto& red = sh.red;
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = b0 + bl;
  const int q = cx * kWarpsB + wid;
  // [slot 0..3 (T1 column / FFT scratch) | prev 0..3 (state); later the T2 tile]
  float2* slot = reinterpret_cast<float2*>(smem + wid * (kSlotB * 8));
  float4* prev = reinterpret_cast<float4*>(smem + kWarpsB * kSlotB * 8 + wid * (kStCol * 16));
  const bool valid = kp.hdr[b].valid != 0;
  float4* stg = reinterpret_cast<float4*>(kp.spec) + ((size_t)b * 224 + q) * kStColG;
  if (lane == 0) {
    tma::bar_init(&bar[wid][0], 1);
    tma::bar_init(&bar[wid][1], 1);
    tma::load_tile(slot, kp.T + ((size_t)bl * 224 + q) * 448, 448 * 8, &bar[wid][0]);
    if (valid) tma::load_tile(prev, stg, kStColG * 16, &bar[wid][1]);
  }
  W448Tw<LAZY> tw;
  tw.load(kp.tw448, kp.tw64, lane);
  __syncwarp();
  tma::bar_wait(&bar[wid][0], 0);
  float2 a[2][7], v[2][8];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int n1 = 0; n1 < 7; ++n1) a[h][n1] = slot[64 * n1 + lane + 32 * h];
  __syncwarp();  // T1 column consumed: the slot becomes FFT scratch
  w448::fwd<false>(a, v, slot, lane, tw);

  const bool h1 = lane < 24;
  // the previous spectrum must have landed before its block is overwritten
  if (valid) tma::bar_wait(&bar[wid][1], 0);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (h == 0 || h1) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        stg[st_idx(h, i, lane)] = make_float4(v[h][2 * i].x, v[h][2 * i].y, v[h][2 * i + 1].x, v[h][2 * i + 1].y);
    }
  }
  if (!valid) return false;  // cold stream: spectrum established (block-uniform)

  // Per-lane sums of one column; the Hermitian weight (2, or 1 for the
  // packed DC / Nyquist column, warp-uniform) and ln 2 are applied once at the
  // end.  Two MUFU ops per bin: rsqrt(|Fp|^2 |Fc|^2) gives both |Fp||Fc| and
  // the cross-power normaliser 1 / (|Fp||Fc| + 1e-12) (the 1e-12 only matters
  // below |Fp||Fc| ~ 1e-8, where the numerator is as small), lg2 the entropy.
  float spc = 0.f, spp = 0.f, scc = 0.f, splp = 0.f;
  auto acc = [&](float2 fp, float2 fc) -> float2 {
    const float pp = fp.x * fp.x + fp.y * fp.y;
    const float pc = fc.x * fc.x + fc.y * fc.y;
    const float x = pp * pc;
    const float r = rsqrtf(fmaxf(x, 1e-30f));
    spc += x * r;  // |Fp| |Fc|
    spp += pp;
    scc += pc;
    splp = fmaf(pc, __log2f(fmaxf(pc, 1.17549435e-38f)), splp);  // pc lg2 pc (0 at pc = 0)
    // normalised cross-power (migration.py:130-131)
    return make_float2((fp.x * fc.x + fp.y * fc.y) * r, (fp.y * fc.x - fp.x * fc.y) * r);
  };
  const int k1a = lane >> 3, j1 = lane & 7;
  __syncwarp();  // every lane is done with the FFT scratch and the prev block
  if (q == 0) {
    // packed DC/Nyquist column (warp-uniform): bins k and 448 - k of both
    // spectra.  The current spectrum goes to the slot in the same register
    // order as the previous one, and mirrored bins are fetched through the
    // inverse of k(g, j2).
    float4* cur = reinterpret_cast<float4*>(slot);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h == 0 || h1) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          cur[st_idx(h, i, lane)] = make_float4(v[h][2 * i].x, v[h][2 * i].y, v[h][2 * i + 1].x, v[h][2 * i + 1].y);
      }
    }
    __syncwarp();
    auto fetch = [](const float4* base, int k) -> float2 {
      const int j2 = k / 56, rem = k - 56 * j2;
      const int g = 8 * (rem % 7) + rem / 7;
      const float4 t = base[st_idx(g >> 5, j2 >> 1, g & 31)];
      return (j2 & 1) ? make_float2(t.z, t.w) : make_float2(t.x, t.y);
    };
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h == 0 || h1) {
#pragma unroll
        for (int j2 = 0; j2 < 8; ++j2) {
          const int k = k1a + 4 * h + 7 * j1 + 56 * j2;
          const int km = (448 - k) % 448;
          const float4 t = prev[st_idx(h, j2 >> 1, lane)];
          const float2 pk = (j2 & 1) ? make_float2(t.z, t.w) : make_float2(t.x, t.y);
          float2 c0, cn, p0, pn;
          unpack_dcny(v[h][j2], fetch(cur, km), c0, cn);
          unpack_dcny(pk, fetch(prev, km), p0, pn);
          const float2 x0 = acc(p0, c0);
          const float2 xn = acc(pn, cn);
          v[h][j2] = make_float2(x0.x - xn.y, x0.y + xn.x);
        }
      }
    }
    __syncwarp();  // the slot becomes FFT scratch again
  } else {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h == 0 || h1) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float4 t = prev[st_idx(h, i, lane)];
          v[h][2 * i] = acc(make_float2(t.x, t.y), v[h][2 * i]);
          v[h][2 * i + 1] = acc(make_float2(t.z, t.w), v[h][2 * i + 1]);
        }
      }
    }
  }
  w448::inv<true>(v, a, slot, lane, tw);
  // per-CTA partial sums: fp32 per lane, fp64 warp tree, warps in order;
  // the column's Hermitian weight and ln 2 applied here
  const double wq = q == 0 ? 1.0 : 2.0;
  const double s0 = wq * warp_sum_f64((double)spc), s1 = wq * warp_sum_f64((double)spp);
  const double s2 = wq * warp_sum_f64((double)scc);
  const double s3 = wq * 0.69314718055994530942 * warp_sum_f64((double)splp);
  if (lane == 0) {
    red[wid][0] = s0; red[wid][1] = s1; red[wid][2] = s2; red[wid][3] = s3;
  }
  // T2 tile [224 pairs][4 columns] of 16-byte (row 2p, row 2p + 1) units over
  // the prev blocks (every warp is past its cross-power after this barrier);
  // the unit of column w in pair p sits at p * 4 + (w ^ ((p >> 1) & 3)), so
  // the writes below and the reads of the copy-out are conflict free
  __syncthreads();
  // 1024-byte aligned inside the prev blocks (16 KB, the tile is 14 KB), so
  // the swizzle below is the hardware's 64-byte pattern on absolute addresses
  float2* tile = reinterpret_cast<float2*>(
      (reinterpret_cast<uintptr_t>(smem + kWarpsB * kSlotB * 8) + 1023) & ~static_cast<uintptr_t>(1023));
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int n1 = 0; n1 < 7; ++n1) {
      const int y = 64 * n1 + lane + 32 * h, pr = y >> 1;
      tile[(pr * 4 + (wid ^ ((pr >> 1) & 3))) * 2 + (y & 1)] = a[h][n1];
    }
  if (threadIdx.x < 4) {
    double acc4 = 0.0;
#pragma unroll
    for (int w = 0; w < kWarpsB; ++w) acc4 += red[w][threadIdx.x];
    kp.stats[((size_t)b * kNCB448 + cx) * 4 + threadIdx.x] = acc4;
  }
  if constexpr (TMST) {
    tma::fence_async_shared();
    __syncthreads();
    if (threadIdx.x == 0) {
      // box = 4 columns (64 bytes) x 224 row pairs of this stream's T2 block
      tma::tensor_store_2d(tmT2, tile, cx * kWarpsB * 4, bl * 224);
      if constexpr (!FLOW) tma::bulk_wait_read0();  // the tile must stay until the engine has read it
    }
  } else {
    static_assert(!FLOW, "the flow kernel writes T2 by tensor store");
    __syncthreads();
    const float4* t4 = reinterpret_cast<const float4*>(tile);
    float4* T2 = reinterpret_cast<float4*>(kp.T2) + (size_t)bl * 224 * 224 + cx * kWarpsB;
    for (int u = threadIdx.x; u < 224 * 4; u += 32 * kWarpsB) {
      const int pr = u >> 2, col = (u & 3) ^ ((pr >> 1) & 3);
      T2[(size_t)pr * 224 + col] = t4[u];
    }
  }
  return true;
}

template <int MINB, bool LAZY, bool TMST>
__global__ void __launch_bounds__(32 * kWarpsB, MINB) k448_cols(KParams kp, int b0,
                                                               const __grid_constant__ CUtensorMap tmT2) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ ColsSh sh;
  // FC_PDL=1: K_C may be scheduled once every K_B CTA has started (it waits
  // for K_B's completion before reading T2); a no-op otherwise
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  cols_item<LAZY, TMST, false>(kp, b0, blockIdx.x, blockIdx.y, &tmT2, smem, sh);
}

// ------------------------------------------------------------- K_C 448 ----
// One warp per PPW row pairs (ya, ya + 1) of T2: both rows of a pair are one
// packed complex 448-point inverse transform (c2r), read from the pair's
// contiguous T2 block (one 16-byte load gives both rows of a column).  Then
// the argmax with the reference's tie rule and the runner-up; one peak partial
// per CTA (224 / (kWarpsC PPW) per stream), merged by K_D in its fixed tie
// order.  With PPW = 2 a warp's two blocks arrive in one bulk-copy phase and
// its twiddles, gather indices and reductions serve both pairs.
// Static shared memory of one K_C item.
struct RowsInvSh {
  PeakKey redk[kWarpsC];
  float redv[kWarpsC];
  uint64_t barc[kWarpsC];
};

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// One K_C work item: row-pair group cx of stream b0 + bl.  FLOW: waits until
// all kNCB448 K_B items of the stream have published their T2 tiles (the last
// K_C item of the stream re-arms the counters for the next launch).  DISCARD:
// the T2 lines the item has staged are dropped from L2 without a write-back
// (each 3.5 KB block is read by exactly one warp, and the next step's K_B
// rewrites it whole).
template <bool LAZY, int PPW, bool FLOW, bool DISCARD, bool PDL = false>
__device__ __forceinline__ void rows_inv_item(const KParams& kp, int b0, int cx, int bl, unsigned char* smem,
                                              RowsInvSh& sh, int* done, int* consumed) {
  auto& redk = sh.redk;
  auto& redv = sh.redv;
  auto& barc = sh.barc;
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = b0 + bl;
  if (kp.hdr[b].valid == 0) return;  // cold stream (block-uniform)
  if constexpr (FLOW) {
    if (threadIdx.x == 0) {
      while (ld_acquire_gpu(done + b) < kNCB448) __nanosleep(128);
      if (atomicAdd(consumed + b, 1) == kNRG448 / PPW - 1) {
        done[b] = 0;
        consumed[b] = 0;
      }
    }
    __syncthreads();
  }
  // launched as a programmatic dependent of K_B (FC_PDL=1): T2 is complete
  // and visible after this (a no-op for a plain launch)
  if constexpr (PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
  const int pair0 = (cx * kWarpsC + wid) * PPW;
  float2* S0 = reinterpret_cast<float2*>(smem) + wid * PPW * w448::XS;
  const float4* T2 = reinterpret_cast<const float4*>(kp.T2) + ((size_t)bl * 224 + pair0) * 224;
  // each row pair's 3.5 KB T2 block lands in its own FFT scratch region with
  // one bulk copy; the lanes then gather their (mirrored) columns from there
  if (lane == 0) {
    if constexpr (FLOW) asm volatile("fence.proxy.async.global;" ::: "memory");
    tma::bar_init(&barc[wid], 1);
    tma::bar_expect(&barc[wid], PPW * 224 * 16);
#pragma unroll
    for (int i = 0; i < PPW; ++i) tma::bulk_g2s(S0 + i * w448::XS, T2 + i * 224, 224 * 16, &barc[wid]);
  }
  W448Tw<LAZY> tw;
  tw.load(kp.tw448, kp.tw64, lane);
  __syncwarp();
  tma::bar_wait(&barc[wid], 0);
  if constexpr (DISCARD) {
    // 28 lines of 128 bytes per 3.5 KB block
    if (lane < 28 * PPW)
      asm volatile("discard.global.L2 [%0], 128;" ::"l"(reinterpret_cast<const char*>(T2) + 128 * lane) : "memory");
  }
  const int k1a = lane >> 3, j1 = lane & 7;
  PeakKey best = {-CUDART_INF_F, 0x7fffffff, 0x7fffffff};
  float v2 = -CUDART_INF_F;
#pragma unroll 1
  for (int it = 0; it < PPW; ++it) {
    const int ya = 2 * (pair0 + it);
    float2* S = S0 + it * w448::XS;
    const float4* Sb = reinterpret_cast<const float4*>(S);
    // bin k = kk + 56 j2 with kk = k1a + 4 h + 7 j1 in [0, 55], so k < 224
    // exactly when j2 < 4 (compile time); the packed DC / Nyquist column (k = 0
    // and k = 224) belongs to lane 0 of half 0 at j2 = 0 and j2 = 4
    const int kk = k1a + 7 * j1;
    float4 in[2][8];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h == 0 || lane < 24) {
#pragma unroll
        for (int j2 = 0; j2 < 8; ++j2) {
          const int k = kk + 4 * h + 56 * j2;
          const int qq = j2 < 4 ? k : (h == 0 && j2 == 4 && lane == 0 ? 0 : 448 - k);
          in[h][j2] = Sb[qq];
        }
      }
    }
    __syncwarp();  // block consumed: S becomes FFT scratch
    float2 v[2][8], a[2][7];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h == 0 || lane < 24) {
#pragma unroll
        for (int j2 = 0; j2 < 8; ++j2) {
          const float4 t = in[h][j2];  // (A = row ya, B = row ya + 1) at the column
          float2 z = j2 < 4 ? make_float2(t.x - t.w, t.y + t.z)     // G_a + i G_b
                            : make_float2(t.x + t.w, t.z - t.y);    // conj G_a + i conj G_b
          if (h == 0 && j2 == 0 && lane == 0) z = make_float2(t.x, t.z);   // k = 0
          if (h == 0 && j2 == 4 && lane == 0) z = make_float2(t.y, t.w);   // k = 224
          v[h][j2] = z;
        }
      }
    }
    w448::inv<true>(v, a, S, lane, tw);

    // argmax with the reference tie rule (migration.py:141-159)
    float m1 = -CUDART_INF_F, m2 = -CUDART_INF_F;
    int ai = 0;
#pragma unroll
    for (int qv = 0; qv < 28; ++qv) {
      const float2 c = a[qv / 14][(qv % 14) >> 1];
      const float val = (qv & 1) ? c.y : c.x;
      if (val > m1) { m2 = m1; m1 = val; ai = qv; }
      else m2 = fmaxf(m2, val);
    }
    auto key_of = [&](int qv, float val) {
      PeakKey c;
      const int y = ya + (qv & 1), j = 64 * ((qv % 14) >> 1) + lane + 32 * (qv / 14);
      c.v = val;
      c.l1 = abs(canon_disp(y, 448)) + abs(canon_disp(j, 448));
      c.pos = y * 448 + j;
      return c;
    };
    PeakKey cand = key_of(ai, m1);
    if (m2 == m1) {
      for (int qv = 0; qv < 28; ++qv) {
        const float2 c = a[qv / 14][(qv % 14) >> 1];
        const float val = (qv & 1) ? c.y : c.x;
        if (val == m1) {
          const PeakKey kq = key_of(qv, val);
          if (peak_better(kq, cand)) cand = kq;
        }
      }
    }
    if (peak_better(cand, best)) { v2 = fmaxf(fmaxf(v2, m2), best.v); best = cand; }
    else v2 = fmaxf(fmaxf(v2, m2), cand.v);
  }
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
    best = redk[0];
    v2 = redv[0];
    for (int w = 1; w < kWarpsC; ++w) {
      const PeakKey o = redk[w];
      if (peak_better(o, best)) { v2 = fmaxf(fmaxf(v2, redv[w]), best.v); best = o; }
      else v2 = fmaxf(fmaxf(v2, redv[w]), o.v);
    }
    PeakPart pp;
    pp.v = best.v; pp.v2 = v2; pp.y = best.pos / 448; pp.j = best.pos % 448;
    kp.peaks[(size_t)b * (kNRG448 / PPW) + cx] = pp;
  }
}

template <int MINB, bool LAZY, int PPW = 1, bool DISCARD = false>
__global__ void __launch_bounds__(32 * kWarpsC, MINB) k448_rows_inv(KParams kp, int b0) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ RowsInvSh sh;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // FC_PDL=1: K_D may be scheduled
  rows_inv_item<LAZY, PPW, false, DISCARD, true>(kp, b0, blockIdx.x, blockIdx.y, smem, sh, nullptr, nullptr);
}

// ------------------------------------------------------- K_B + K_C flow ----
// K_B and K_C as one launch of work items taken in ticket order (FC_BC_FLOW=1,
// an option: measured slower than the two kernels): round r holds
// the kNCB448 K_B items of stream r, then the kNRG448 K_C items of stream
// r - lag.  A K_C item waits (spinning) for its stream's K_B items; those hold
// smaller tickets, and a CTA draws one ticket and processes it at once, so
// they are running or done — the wait cannot deadlock.  (A persistent variant
// that prefetched its next ticket broke exactly this: a drawn but unstarted
// K_B item behind a waiting K_C item, and two such CTAs deadlocked.)  T2 of
// the last `lag` streams is still in L2 when K_C reads it, and K_C discards
// what it has read (DISCARD), so T2 costs neither its DRAM read nor its
// write-back.  flow = [kMaxFlowLanes tickets (128 B apart) | done[B] |
// consumed[B]], zero-initialised; each launch re-arms what it used.
constexpr int kFlowTicketStride = 32;   // ints
constexpr int kMaxFlowLanes = 8;

template <int MINB, bool DISCARD>
__global__ void __launch_bounds__(32 * kWarpsB, MINB)
    k448_bc_flow(const __grid_constant__ KParams kp, int b0, int nb, int lag, int lane_id,
                 const __grid_constant__ CUtensorMap tmT2) {
  static_assert(kWarpsB == kWarpsC, "one CTA shape for both item kinds");
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ ColsSh shb;
  __shared__ RowsInvSh shc;
  __shared__ int tk;
  int* ticket = kp.flow + lane_id * kFlowTicketStride;
  int* done = kp.flow + kMaxFlowLanes * kFlowTicketStride;
  int* consumed = done + kp.B;
  if (threadIdx.x == 0) {
    const int t = atomicAdd(ticket, 1);
    if (t == (int)gridDim.x - 1) *ticket = 0;   // every ticket is taken: re-arm
    tk = t;
  }
  __syncthreads();
  constexpr int per = kNCB448 + kNRG448;
  const int r = tk / per, w = tk - r * per;
  if (w < kNCB448) {
    if (r < nb && cols_item<true, true, true>(kp, b0, w, r, &tmT2, smem, shb) && threadIdx.x == 0) {
      // the tile is in global memory (async proxy) before the generic-proxy
      // release that lets this stream's K_C items load it
      tma::bulk_wait0();
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __threadfence();
      atomicAdd(done + b0 + r, 1);
    }
  } else {
    const int sidx = r - lag;
    if (sidx >= 0 && sidx < nb)
      rows_inv_item<true, 1, true, DISCARD>(kp, b0, w - kNCB448, sidx, smem, shc, done, consumed);
  }
}
