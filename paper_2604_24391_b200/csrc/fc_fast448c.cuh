// K_BC: K_B and K_C of the 448 x 448 fast path fused in one thread-block
// cluster per stream, with the cross-power spectrum handed from the column
// pass to the inverse-row pass through distributed shared memory instead of
// the T2 round trip through HBM (0.8 MB written + read per frame).
//
// Cluster of 8 CTAs per stream (one per SM: 214 KB of shared memory), 14
// warps per CTA.  CTA r owns columns [28 r, 28 r + 28) for the column pass
// and row pairs [28 r, 28 r + 28) for the row pass:
//   column pass  warp w transforms columns 28 r + w and 28 r + w + 14 exactly
//                as K_B does (TMA-staged T1 column and previous spectrum,
//                forward column FFT, state swap, Hermitian sums, normalised
//                cross-power, inverse column FFT) and stores each result row
//                straight into the shared memory of the CTA owning its row
//                pair (st.shared::cluster through mapped addresses);
//   cluster barrier;
//   row pass     warp w runs row pairs w and w + 14 of its CTA as K_C does
//                (packed c2r inverse, argmax with the tie rule, runner-up)
//                from the local row-pair blocks.
// Row-pair blocks are [224 columns] x (row 2p, row 2p + 1) 16-byte units with
// the column index XOR-swizzled by the pair's low 4 bits (q ^ (p & 15) stays
// inside q's 16-column group), so the scattered remote stores of a warp (16
// pairs at a time) fall on different banks.
// Partials for K_D: sums per column (kNCBf = 224 per stream), peaks per warp
// (kNRGf = 112 per stream); K_D merges them in its fixed orders.
#pragma once
#include <cooperative_groups.h>

#include "fc_fast448w.cuh"

constexpr int kClusterBC = 8;
constexpr int kWarpsBC = 14;
constexpr int kNCBf = 224;                       // stats partials per stream (one per column)
constexpr int kNRGf = kClusterBC * kWarpsBC;     // peak partials per stream (one per warp)
constexpr int kDestBC = 28 * 224 * 16;           // row-pair blocks of one CTA (100,352 B)
constexpr int kSmemBC = kDestBC + kWarpsBC * (kSlotB * 8 + kStCol * 16);

template <bool LAZY>
__global__ void __cluster_dims__(kClusterBC, 1, 1) __launch_bounds__(32 * kWarpsBC, 1)
    k448_colsinv(KParams kp, int b0) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[kWarpsBC][2];
  cg::cluster_group cluster = cg::this_cluster();
  const int r = (int)cluster.block_rank();
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bl = blockIdx.y, b = b0 + bl;
  float4* dest = reinterpret_cast<float4*>(smem);
  float2* slot = reinterpret_cast<float2*>(smem + kDestBC + wid * (kSlotB * 8));
  float4* prev = reinterpret_cast<float4*>(smem + kDestBC + kWarpsBC * kSlotB * 8 + wid * (kStCol * 16));
  const bool valid = kp.hdr[b].valid != 0;
  if (lane == 0) {
    tma::bar_init(&bar[wid][0], 1);
    tma::bar_init(&bar[wid][1], 1);
  }
  W448Tw<LAZY> tw;
  tw.load(kp.tw448, kp.tw64, lane);
  __syncwarp();
  const bool h1 = lane < 24;
  const int k1a = lane >> 3, j1 = lane & 7;

  // ------------------------------------------------------- column pass
#pragma unroll 1
  for (int it = 0; it < 2; ++it) {
    const int q = 28 * r + wid + 14 * it;
    float4* stg = reinterpret_cast<float4*>(kp.spec) + ((size_t)b * 224 + q) * kStColG;
    if (lane == 0) {
      tma::fence_async_shared();   // the slot / prev blocks were generic-proxy scratch
      tma::load_tile(slot, kp.T + ((size_t)bl * 224 + q) * 448, 448 * 8, &bar[wid][0]);
      if (valid) tma::load_tile(prev, stg, kStColG * 16, &bar[wid][1]);
    }
    __syncwarp();
    tma::bar_wait(&bar[wid][0], it & 1);
    float2 a[2][7], v[2][8];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int n1 = 0; n1 < 7; ++n1) a[h][n1] = slot[64 * n1 + lane + 32 * h];
    __syncwarp();
    w448::fwd<false>(a, v, slot, lane, tw);
    if (valid) tma::bar_wait(&bar[wid][1], it & 1);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h == 0 || h1) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          stg[st_idx(h, i, lane)] =
              make_float4(v[h][2 * i].x, v[h][2 * i].y, v[h][2 * i + 1].x, v[h][2 * i + 1].y);
      }
    }
    if (!valid) continue;  // cold stream: spectrum established (cluster-uniform)

    float spc = 0.f, spp = 0.f, scc = 0.f, splp = 0.f;
    auto acc = [&](float2 fp, float2 fc) -> float2 {
      const float pp = fp.x * fp.x + fp.y * fp.y;
      const float pc = fc.x * fc.x + fc.y * fc.y;
      const float x = pp * pc;
      const float rr = rsqrtf(fmaxf(x, 1e-30f));
      spc += x * rr;
      spp += pp;
      scc += pc;
      splp = fmaf(pc, __log2f(fmaxf(pc, 1.17549435e-38f)), splp);
      return make_float2((fp.x * fc.x + fp.y * fc.y) * rr, (fp.y * fc.x - fp.x * fc.y) * rr);
    };
    __syncwarp();
    if (q == 0) {
      float4* cur = reinterpret_cast<float4*>(slot);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h == 0 || h1) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
            cur[st_idx(h, i, lane)] =
                make_float4(v[h][2 * i].x, v[h][2 * i].y, v[h][2 * i + 1].x, v[h][2 * i + 1].y);
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
      __syncwarp();
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
    // per-column partial sums for K_D (fp32 per lane, fp64 warp tree)
    const double wq = q == 0 ? 1.0 : 2.0;
    const double s0 = wq * warp_sum_f64((double)spc), s1 = wq * warp_sum_f64((double)spp);
    const double s2 = wq * warp_sum_f64((double)scc);
    const double s3 = wq * 0.69314718055994530942 * warp_sum_f64((double)splp);
    if (lane == 0) {
      double* o = kp.stats + ((size_t)b * kNCBf + q) * 4;
      o[0] = s0; o[1] = s1; o[2] = s2; o[3] = s3;
    }
    // rows y = 64 n1 + lane + 32 h of column q -> the CTA owning pair y / 2
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int n1 = 0; n1 < 7; ++n1) {
        const int y = 64 * n1 + lane + 32 * h, pg = y >> 1;
        const int owner = pg / 28, p = pg - 28 * owner;
        float2* d = reinterpret_cast<float2*>(dest + p * 224 + (q ^ (p & 15))) + (y & 1);
        *cluster.map_shared_rank(d, owner) = a[h][n1];
      }
    __syncwarp();
  }
  // every row-pair block of the cluster is complete (cold: nothing to wait for,
  // but the barrier keeps every CTA resident until its peers are done)
  cluster.sync();
  if (!valid) return;

  // ---------------------------------------------------------- row pass
  PeakKey best = {-CUDART_INF_F, 0x7fffffff, 0x7fffffff};
  float v2 = -CUDART_INF_F;
  float2* S = slot;
#pragma unroll 1
  for (int it = 0; it < 2; ++it) {
    const int p = wid + 14 * it;
    const int pair = 28 * r + p, ya = 2 * pair;
    const float4* Sb = dest + p * 224;
    const int sw = p & 15;
    float2 v[2][8], a[2][7];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h == 0 || lane < 24) {
#pragma unroll
        for (int j2 = 0; j2 < 8; ++j2) {
          const int k = k1a + 4 * h + 7 * j1 + 56 * j2;
          const int qq = (k == 0 || k == 224) ? 0 : (k < 224 ? k : 448 - k);
          const float4 t = Sb[qq ^ sw];  // (A = row ya, B = row ya + 1) at the column
          float2 z;
          if (k == 0) z = make_float2(t.x, t.z);
          else if (k == 224) z = make_float2(t.y, t.w);
          else if (k < 224) z = make_float2(t.x - t.w, t.y + t.z);   // G_a + i G_b
          else z = make_float2(t.x + t.w, t.z - t.y);                // conj G_a + i conj G_b
          v[h][j2] = z;
        }
      }
    }
    __syncwarp();
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
    // fold this pair's lane result into the lane's running best
    if (peak_better(cand, best)) { v2 = fmaxf(fmaxf(v2, m2), best.v); best = cand; }
    else v2 = fmaxf(fmaxf(v2, m2), cand.v);
    __syncwarp();
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
  if (lane == 0) {
    PeakPart pp;
    pp.v = best.v; pp.v2 = v2; pp.y = best.pos / 448; pp.j = best.pos % 448;
    kp.peaks[(size_t)b * kNRGf + r * kWarpsBC + wid] = pp;
  }
}
