// C ABI of the B200 FreqCache decision path (see include/freqcache_b200.h).
// Host side: geometry validation, plan construction (FFT factorisations,
// fp64-derived twiddles, DCT basis), workspace carving and kernel launches.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "fc_kernels.cuh"

struct fc_plan {
  fc_geometry g;
  KParams kp;  // geometry + device constant tables (per-call pointers filled at launch)
  float2* d_twW = nullptr;
  float2* d_twH = nullptr;
  double* d_dct = nullptr;
  size_t smemA = 0, smemB = 0, smemC = 0, smemD = 0;
  size_t off_T = 0, off_stripes = 0, off_stats = 0, off_peaks = 0, off_energy = 0, ws_bytes = 0;
  size_t state_hdr_bytes = 0, state_bytes = 0;
  int kw = 0, kh = 0;  // fixed-size FFT variants (0 = generic)
};

namespace {

constexpr size_t kAlign = 256;
inline size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

bool factor(int n, FftPlan& pl) {
  pl.n = n;
  pl.nstages = 0;
  int m = n;
  const int pref[] = {8, 4, 2, 7, 5, 3};
  for (int r : pref) {
    while (m % r == 0) {
      if (pl.nstages >= FC_MAX_STAGES) return false;
      pl.radix[pl.nstages++] = r;
      m /= r;
    }
  }
  for (int r = 11; m > 1 && r <= FC_MAX_GENERIC_RADIX; r += 2) {
    while (m % r == 0) {
      if (pl.nstages >= FC_MAX_STAGES) return false;
      pl.radix[pl.nstages++] = r;
      m /= r;
    }
  }
  return m == 1;
}

std::vector<float2> twiddles(int n) {
  std::vector<float2> t(n);
  for (int m = 0; m < n; ++m) {
    const double a = -2.0 * M_PI * (double)m / (double)n;
    t[m] = make_float2((float)std::cos(a), (float)std::sin(a));
  }
  return t;
}

// kernel pointers selected per fixed-size variant
template <int N> void* ptr_rows_fwd() { return (void*)k_rows_fwd<N>; }
template <int N> void* ptr_cols() { return (void*)k_cols<N>; }
template <int N> void* ptr_rows_inv() { return (void*)k_rows_inv<N>; }

void* sel_rows_fwd(int k) { return k == 448 ? ptr_rows_fwd<448>() : k == 224 ? ptr_rows_fwd<224>() : ptr_rows_fwd<0>(); }
void* sel_cols(int k) { return k == 448 ? ptr_cols<448>() : k == 224 ? ptr_cols<224>() : ptr_cols<0>(); }
void* sel_rows_inv(int k) { return k == 448 ? ptr_rows_inv<448>() : k == 224 ? ptr_rows_inv<224>() : ptr_rows_inv<0>(); }

int set_smem(void* fn, size_t bytes) {
  if (bytes > 48 * 1024) {
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess)
      return FC_ECUDA;
  }
  return FC_OK;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int launch_check() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? FC_OK : FC_ECUDA;
}

KParams bind(const fc_plan* pl, void* state, void* ws, double* energy) {
  KParams kp = pl->kp;
  uint8_t* w = reinterpret_cast<uint8_t*>(ws);
  kp.T = reinterpret_cast<float2*>(w + pl->off_T);
  kp.stripes = reinterpret_cast<StripeStat*>(w + pl->off_stripes);
  kp.stats = reinterpret_cast<double*>(w + pl->off_stats);
  kp.peaks = reinterpret_cast<PeakPart*>(w + pl->off_peaks);
  kp.energy = energy ? energy : reinterpret_cast<double*>(w + pl->off_energy);
  if (state) {
    uint8_t* s = reinterpret_cast<uint8_t*>(state);
    kp.hdr = reinterpret_cast<StreamHdr*>(s);
    kp.spec = reinterpret_cast<float2*>(s + pl->state_hdr_bytes);
  } else {
    kp.hdr = nullptr;
    kp.spec = nullptr;
  }
  return kp;
}

}  // namespace

extern "C" {

int fc_abi_version(void) { return FC_ABI_VERSION; }

const char* fc_strerror(int code) {
  switch (code) {
    case FC_OK: return "ok";
    case FC_EINVAL: return "invalid argument";
    case FC_EUNSUPPORTED: return "geometry outside the supported envelope";
    case FC_ECUDA: return "CUDA runtime error";
    case FC_ENONFINITE: return "frame contains non-finite values";
    case FC_EPSI: return "normalized entropy must lie in [0, 1]";
    case FC_EBOUNDS: return "reuse source out of bounds";
    default: return "unknown error";
  }
}

int fc_plan_create(const fc_geometry* geom, fc_plan** out) {
  if (!geom || !out) return FC_EINVAL;
  *out = nullptr;
  const fc_geometry g = *geom;
  if (g.batch < 1 || g.height < 1 || g.width < 1) return FC_EINVAL;
  if (g.patch_size < 2) return FC_EINVAL;                                  // frame.py:31-32
  if (g.height % g.patch_size || g.width % g.patch_size) return FC_EINVAL; // frame.py:33-37
  if (g.format < FC_FMT_RGB_F32 || g.format > FC_FMT_GRAY_F64) return FC_EINVAL;
  const int P = g.patch_size, H = g.height, W = g.width;
  const int rows = H / P, cols = W / P, N = rows * cols;
  if (P > FC_MAX_PATCH || N > FC_MAX_TOKENS || H > 1536 || W > 1536) return FC_EUNSUPPORTED;

  fc_plan* pl = new (std::nothrow) fc_plan();
  if (!pl) return FC_EINVAL;
  pl->g = g;
  KParams& kp = pl->kp;
  std::memset(&kp, 0, sizeof(kp));
  kp.B = g.batch; kp.H = H; kp.W = W; kp.P = P; kp.fmt = g.format;
  kp.rows = rows; kp.cols = cols; kp.N = N;
  kp.cut = P / 4 > 1 ? P / 4 : 1;  // edge_refresh.py:9-11
  kp.Wc = (W % 2 == 0) ? W / 2 : (W + 1) / 2;
  kp.Wcp = (kp.Wc + FC_CB - 1) / FC_CB * FC_CB;
  kp.NCB = kp.Wcp / FC_CB;
  kp.npairA = (P + 1) / 2;
  kp.RG = H >= 16 ? 16 : (H + (H & 1));
  kp.NRG = (H + kp.RG - 1) / kp.RG;
  if (!factor(W, kp.planW) || !factor(H, kp.planH)) { delete pl; return FC_EUNSUPPORTED; }
  pl->kw = (W == 448 || W == 224) ? W : 0;
  pl->kh = (H == 448 || H == 224) ? H : 0;

  const int maxpairC = (kp.RG + 1) / 2;
  pl->smemA = (size_t)P * W * 8 + (size_t)kp.npairA * W * 8 + (size_t)W * 8 + (size_t)kp.cut * P * 8;
  pl->smemB = (size_t)2 * H * FC_CB * 8 + (size_t)H * 8;
  pl->smemC = (size_t)2 * maxpairC * W * 8 + (size_t)W * 8;
  int NP2 = 1;
  while (NP2 < N) NP2 <<= 1;
  pl->smemD = (size_t)N * 8 + (size_t)NP2 * 8 + (size_t)NP2 * 4 + (size_t)N * 4 + (size_t)N * 2;
  const size_t kMaxSmem = 227 * 1024;
  if (pl->smemA > kMaxSmem || pl->smemB > kMaxSmem || pl->smemC > kMaxSmem || pl->smemD > kMaxSmem) {
    delete pl;
    return FC_EUNSUPPORTED;
  }

  // workspace carve
  const size_t B = g.batch;
  const size_t specElems = B * kp.NCB * (size_t)H * FC_CB;
  size_t off = 0;
  pl->off_T = off; off = align_up(off + specElems * sizeof(float2));
  pl->off_stripes = off; off = align_up(off + B * rows * sizeof(StripeStat));
  pl->off_stats = off; off = align_up(off + B * kp.NCB * 4 * sizeof(double));
  pl->off_peaks = off; off = align_up(off + B * kp.NRG * sizeof(PeakPart));
  pl->off_energy = off; off = align_up(off + B * N * sizeof(double));
  pl->ws_bytes = off;
  pl->state_hdr_bytes = align_up(B * sizeof(StreamHdr));
  pl->state_bytes = pl->state_hdr_bytes + align_up(specElems * sizeof(float2));

  // constant tables (fp64 derivation, rounded once)
  std::vector<float2> tw = twiddles(W), th = twiddles(H);
  std::vector<double> dct((size_t)kp.cut * P);
  for (int u = 0; u < kp.cut; ++u)
    for (int x = 0; x < P; ++x) {
      const double s = u == 0 ? std::sqrt(1.0 / P) : std::sqrt(2.0 / P);
      dct[(size_t)u * P + x] = s * std::cos(M_PI * u * (2 * x + 1) / (2.0 * P));
    }
  int rc = FC_OK;
  if (cudaMalloc(&pl->d_twW, W * sizeof(float2)) != cudaSuccess ||
      cudaMalloc(&pl->d_twH, H * sizeof(float2)) != cudaSuccess ||
      cudaMalloc(&pl->d_dct, dct.size() * sizeof(double)) != cudaSuccess)
    rc = FC_ECUDA;
  if (rc == FC_OK &&
      (cudaMemcpy(pl->d_twW, tw.data(), W * sizeof(float2), cudaMemcpyHostToDevice) != cudaSuccess ||
       cudaMemcpy(pl->d_twH, th.data(), H * sizeof(float2), cudaMemcpyHostToDevice) != cudaSuccess ||
       cudaMemcpy(pl->d_dct, dct.data(), dct.size() * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess))
    rc = FC_ECUDA;
  if (rc == FC_OK) {
    rc = set_smem(sel_rows_fwd(pl->kw), pl->smemA);
    if (rc == FC_OK) rc = set_smem(sel_cols(pl->kh), pl->smemB);
    if (rc == FC_OK) rc = set_smem(sel_rows_inv(pl->kw), pl->smemC);
    if (rc == FC_OK) rc = set_smem((void*)k_select, pl->smemD);
  }
  if (rc != FC_OK) {
    fc_plan_destroy(pl);
    return rc;
  }
  kp.twW = pl->d_twW;
  kp.twH = pl->d_twH;
  kp.dct = pl->d_dct;
  *out = pl;
  return FC_OK;
}

void fc_plan_destroy(fc_plan* pl) {
  if (!pl) return;
  if (pl->d_twW) cudaFree(pl->d_twW);
  if (pl->d_twH) cudaFree(pl->d_twH);
  if (pl->d_dct) cudaFree(pl->d_dct);
  delete pl;
}

int64_t fc_plan_state_bytes(const fc_plan* pl) { return pl ? (int64_t)pl->state_bytes : -1; }
int64_t fc_plan_workspace_bytes(const fc_plan* pl) { return pl ? (int64_t)pl->ws_bytes : -1; }
int fc_plan_tokens(const fc_plan* pl) { return pl ? pl->kp.N : -1; }

int fc_state_reset(const fc_plan* pl, void* state, int32_t first, int32_t count, void* stream) {
  if (!pl || !state || first < 0 || count < 0 || first + count > pl->g.batch) return FC_EINVAL;
  if (count == 0) return FC_OK;
  k_state_reset<<<(count + 255) / 256, 256, 0, as_stream(stream)>>>(reinterpret_cast<StreamHdr*>(state),
                                                                    first, count);
  return launch_check();
}

int fc_select_stage(const fc_plan* pl, const fc_config* cfg, const void* frames, void* state, void* ws,
                    const fc_select_out* out, int32_t stage, void* stream) {
  if (!pl || !cfg || !frames || !state || !ws || !out) return FC_EINVAL;
  if (stage < -1 || stage > 3) return FC_EINVAL;
  // CacheConfig / BudgetConfig validation (fusion.py:61-67, budget.py:19-24)
  if (!(cfg->tau_mig >= 0.0 && cfg->tau_mig <= 1.0)) return FC_EINVAL;
  if (!std::isfinite(cfg->edge_lambda)) return FC_EINVAL;
  if (!(0.0 <= cfg->alpha_min && cfg->alpha_min <= cfg->alpha_max && cfg->alpha_max <= 1.0)) return FC_EINVAL;
  const cudaStream_t st = as_stream(stream);
  const KParams kp = bind(pl, state, ws, out->energy);
  const int B = pl->g.batch;
  const dim3 blk(FC_THREADS);
  if (stage < 0 || stage == 0) {
    const dim3 grid(kp.rows, B);
    auto fn = (void (*)(KParams, const void*, int))sel_rows_fwd(pl->kw);
    fn<<<grid, blk, pl->smemA, st>>>(kp, frames, 1);
  }
  if (stage < 0 || stage == 1) {
    const dim3 grid(kp.NCB, B);
    auto fn = (void (*)(KParams))sel_cols(pl->kh);
    fn<<<grid, blk, pl->smemB, st>>>(kp);
  }
  if (stage < 0 || stage == 2) {
    const dim3 grid(kp.NRG, B);
    auto fn = (void (*)(KParams))sel_rows_inv(pl->kw);
    fn<<<grid, blk, pl->smemC, st>>>(kp);
  }
  if (stage < 0 || stage == 3) k_select<<<B, FC_SEL_THREADS, pl->smemD, st>>>(kp, *cfg, *out);
  return launch_check();
}

int fc_select(const fc_plan* pl, const fc_config* cfg, const void* frames, void* state, void* ws,
              const fc_select_out* out, void* stream) {
  return fc_select_stage(pl, cfg, frames, state, ws, out, -1, stream);
}

int fc_patch_energy(const fc_plan* pl, const void* frames, void* ws, double* energy, void* stream) {
  if (!pl || !frames || !ws || !energy) return FC_EINVAL;
  const KParams kp = bind(pl, nullptr, ws, energy);
  const dim3 grid(kp.rows, pl->g.batch);
  auto fn = (void (*)(KParams, const void*, int))sel_rows_fwd(pl->kw);
  fn<<<grid, FC_THREADS, pl->smemA, as_stream(stream)>>>(kp, frames, 0);
  return launch_check();
}

int fc_splice(int32_t batch, int32_t n_tokens, int64_t row_bytes, const int32_t* src_map, const void* cache,
              const int64_t* cache_ages, const void* fresh, int32_t fresh_layout, void* out,
              int64_t* out_ages, void* stream) {
  if (batch < 1 || n_tokens < 1 || row_bytes < 1 || !src_map || !fresh || !out || !out_ages) return FC_EINVAL;
  if (fresh_layout != FC_FRESH_DENSE && fresh_layout != FC_FRESH_COMPACT) return FC_EINVAL;
  const int total = batch * n_tokens;
  const int compact = fresh_layout == FC_FRESH_COMPACT;
  const cudaStream_t st = as_stream(stream);
  const bool vec = (row_bytes % 16 == 0) && ((reinterpret_cast<uintptr_t>(cache) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(fresh) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
  if (vec) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    constexpr int UNR = 2;
    const int warps_needed = (total + UNR - 1) / UNR;
    int blocks = (warps_needed + (FC_THREADS / 32) - 1) / (FC_THREADS / 32);
    const int cap = sms * 8;
    if (blocks > cap) blocks = cap;
    k_splice16<UNR><<<blocks, FC_THREADS, 0, st>>>(
        total, n_tokens, row_bytes / 16, src_map, reinterpret_cast<const int4*>(cache), cache_ages,
        reinterpret_cast<const int4*>(fresh), compact, reinterpret_cast<int4*>(out), out_ages);
  } else {
    k_splice_bytes<<<total, 128, 0, st>>>(total, n_tokens, row_bytes, src_map,
                                          reinterpret_cast<const uint8_t*>(cache), cache_ages,
                                          reinterpret_cast<const uint8_t*>(fresh), compact,
                                          reinterpret_cast<uint8_t*>(out), out_ages);
  }
  return launch_check();
}

int fc_splice_map(int32_t rows, int32_t cols, const int32_t* reuse_idx, int32_t k, int32_t dip, int32_t djp,
                  int32_t* src_map, int32_t* flag, void* stream) {
  if (rows < 1 || cols < 1 || k < 0 || !src_map || (k > 0 && !reuse_idx)) return FC_EINVAL;
  const int N = rows * cols;
  if (N > 65536) return FC_EUNSUPPORTED;
  const size_t smem = (size_t)N * sizeof(int);
  if (smem > 48 * 1024) {
    if (cudaFuncSetAttribute((void*)k_splice_map, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return FC_ECUDA;
  }
  k_splice_map<<<1, 512, smem, as_stream(stream)>>>(rows, cols, reuse_idx, k, dip, djp, src_map, flag);
  return launch_check();
}

}  // extern "C"
