// C ABI of the B200 FreqCache decision path (see include/freqcache_b200.h).
// Host side: geometry validation, plan construction (FFT factorisations,
// fp64-derived twiddles, DCT basis), workspace carving and kernel launches.
//
// Two kernel sets implement fc_select:
//   fast    H = W = 448, P = 14 (BASELINE configs 2-5): warp-owned
//           448-point FFTs (fc_wfft448.cuh) in K_A / K_B / K_C
//           (fc_fast448.cuh, fc_fast448w.cuh) over the whole batch as one
//           chunk (two half-batch chunks on two lanes at <= 128 streams);
//           the two spectrum intermediates (T1, T2: 0.8 MB per stream each)
//           make a round trip through HBM (DESIGN §3 lists what was measured
//           to keep them on chip);
//   generic any other geometry inside the envelope: shared-memory Stockham
//           FFTs with runtime radix plans (fc_fft.cuh / fc_kernels.cuh).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "fc_kernels.cuh"
#include "fc_fast448w.cuh"
#include "fc_fast448c.cuh"
#include "fc_compare.cuh"
#include "fc_stages.cuh"
#include "fc_spectral.cuh"

namespace {
constexpr int kChunkDefault = 512;  // streams per A/B/C launch group on the fast path
constexpr int kLanesDefault = 1;   // concurrent chunk lanes (internal CUDA streams)
constexpr int kMaxLanes = 8;
constexpr int kSmallBatch = 128;   // at or below: two half-batch chunks on two lanes

int env_int(const char* name, int dflt, int lo, int hi) {
  const char* v = std::getenv(name);
  if (!v) return dflt;
  const int x = std::atoi(v);
  return x < lo ? lo : (x > hi ? hi : x);
}
}

struct fc_plan {
  fc_geometry g;
  KParams kp;  // geometry + device constant tables (per-call pointers filled at launch)
  Dct14 dct14;
  bool fast = false;
  int chunk = 0;
  int lanes = 1;                       // fast path: chunk groups in flight
  // internal non-blocking lane streams and fork / join events, one set per
  // part (whole select, split-phase front, split-phase back)
  cudaStream_t lanes3[3][kMaxLanes] = {};
  cudaEvent_t fork3[3] = {};
  cudaEvent_t join3[3][kMaxLanes] = {};
  size_t lane_t1 = 0, lane_t2 = 0;     // T1 / T2 bytes of one lane (chunk streams)
  // split-phase select: per-slot strides of the front -> back intermediates
  size_t slot_T = 0, slot_stripes = 0, slot_order = 0, slot_freshm = 0, slot_estats = 0;
  void* fnB = nullptr;                 // K_B / K_C variants (occupancy x twiddle mode)
  bool t2_tma = false;                 // K_B stores T2 with a TMA tensor store
  bool t1_tma = false;                 // K_A stores T1 with a TMA tensor store
  bool fused_bc = false;               // K_B + K_C as one cluster kernel (T2 through DSMEM)
  bool flow_bc = false;                // K_B + K_C as one ticket-ordered flow kernel (T2 through L2)
  int flow_lag = 8;                    // flow: streams K_C trails K_B by
  void* fnF = nullptr;
  bool pdl = false;                     // K_C / K_D of the back as programmatic dependents (FC_PDL=1)
  int probe_skip = 0;                  // timing probes only (FC_PROBE_SKIP bitmask): kernels not launched
  bool probe_back = false;             // timing probes only: FC_PROBE_BACK_PART set at plan creation
  size_t off_flow = 0;
  int kc_ppw = 1;                      // K_C row pairs per warp
  void* fnC = nullptr;
  float2* d_twW = nullptr;
  float2* d_twH = nullptr;
  double* d_dct = nullptr;
  float2* d_tw448 = nullptr;
  float2* d_tw64 = nullptr;
  size_t smemA = 0, smemB = 0, smemC = 0, smemD = 0;
  size_t off_T = 0, off_T2 = 0, off_stripes = 0, off_stats = 0, off_peaks = 0, off_energy = 0, ws_bytes = 0;
  size_t off_order = 0, off_freshm = 0, off_estats = 0;
  size_t smemR = 0;                    // K_D1 (k_rank) dynamic shared memory
  cudaStream_t aux = nullptr;          // K_D1 branch beside K_B / K_C
  cudaEvent_t ev_a = nullptr, ev_aux = nullptr;
  size_t state_hdr_bytes = 0, state_bytes = 0;
  int kw = 0, kh = 0;  // fixed-size generic FFT variants (0 = runtime plan)
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

float2 root(long long m, long long n) {
  const double a = -2.0 * M_PI * (double)(m % n) / (double)n;
  return make_float2((float)std::cos(a), (float)std::sin(a));
}

std::vector<float2> twiddles(int n) {
  std::vector<float2> t(n);
  for (int m = 0; m < n; ++m) t[m] = root(m, n);
  return t;
}

template <int N> void* ptr_rows_fwd() { return (void*)k_rows_fwd<N>; }
template <int N> void* ptr_cols() { return (void*)k_cols<N>; }
template <int N> void* ptr_rows_inv() { return (void*)k_rows_inv<N>; }

void* sel_rows_fwd(int k) { return k == 448 ? ptr_rows_fwd<448>() : k == 224 ? ptr_rows_fwd<224>() : ptr_rows_fwd<0>(); }
void* sel_cols(int k) { return k == 448 ? ptr_cols<448>() : k == 224 ? ptr_cols<224>() : ptr_cols<0>(); }
void* sel_rows_inv(int k) { return k == 448 ? ptr_rows_inv<448>() : k == 224 ? ptr_rows_inv<224>() : ptr_rows_inv<0>(); }

template <bool TM>
void* sel_fast_rows_fwd_t(int fmt) {
  return fmt == FC_FMT_RGB_F32 ? (void*)k448_rows_fwd<FC_FMT_RGB_F32, TM>
       : fmt == FC_FMT_GRAY_F32 ? (void*)k448_rows_fwd<FC_FMT_GRAY_F32, TM>
       : fmt == FC_FMT_GRAY_U8 ? (void*)k448_rows_fwd<FC_FMT_GRAY_U8, TM>
       : fmt == FC_FMT_RGB_U8 ? (void*)k448_rows_fwd<FC_FMT_RGB_U8, TM>
                                : (void*)k448_rows_fwd<FC_FMT_GRAY_F64, TM>;
}
void* sel_fast_rows_fwd(int fmt, bool tm) { return tm ? sel_fast_rows_fwd_t<true>(fmt) : sel_fast_rows_fwd_t<false>(fmt); }
using FastRowsFwd = void (*)(KParams, Dct14, const void*, int, int, CUtensorMap);

int set_smem(void* fn, size_t bytes) {
  // the 48 KB default covers static + dynamic shared memory: opt in above it
  cudaFuncAttributes fa;
  const size_t stat = cudaFuncGetAttributes(&fa, fn) == cudaSuccess ? fa.sharedSizeBytes : 0;
  if (bytes + stat > 48 * 1024) {
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

KParams bind(const fc_plan* pl, void* state, void* ws, double* energy, int slot = 0) {
  KParams kp = pl->kp;
  uint8_t* w = reinterpret_cast<uint8_t*>(ws);
  kp.T = reinterpret_cast<float2*>(w + pl->off_T + slot * pl->slot_T);
  kp.T2 = pl->fast ? reinterpret_cast<float2*>(w + pl->off_T2) : nullptr;
  kp.stripes = reinterpret_cast<StripeStat*>(w + pl->off_stripes + slot * pl->slot_stripes);
  kp.stats = reinterpret_cast<double*>(w + pl->off_stats);
  kp.peaks = reinterpret_cast<PeakPart*>(w + pl->off_peaks);
  kp.energy = energy ? energy : reinterpret_cast<double*>(w + pl->off_energy);
  kp.order = reinterpret_cast<int16_t*>(w + pl->off_order + slot * pl->slot_order);
  kp.freshm = w + pl->off_freshm + slot * pl->slot_freshm;
  kp.estats = reinterpret_cast<double*>(w + pl->off_estats + slot * pl->slot_estats);
  kp.flow = reinterpret_cast<int*>(w + pl->off_flow);
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

int check_cfg(const fc_config* cfg) {
  // CacheConfig / BudgetConfig validation (fusion.py:61-67, budget.py:19-24)
  if (!(cfg->tau_mig >= 0.0 && cfg->tau_mig <= 1.0)) return FC_EINVAL;
  if (!std::isfinite(cfg->edge_lambda)) return FC_EINVAL;
  if (!(0.0 <= cfg->alpha_min && cfg->alpha_min <= cfg->alpha_max && cfg->alpha_max <= 1.0)) return FC_EINVAL;
  return FC_OK;
}

// Launch sequence of one select step.  `ev` (optional): records an event
// after every launch, kernel kind in `kind` (0..3) for per-kernel timing.
struct Recorder {
  cudaEvent_t* ev = nullptr;
  int* kind = nullptr;
  int n = 0, cap = 0;
  void mark(cudaStream_t st, int k) {
    if (ev && n < cap) {
      cudaEventRecord(ev[n], st);
      kind[n] = k;
      ++n;
    }
  }
};

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
PFN_cuTensorMapEncodeTiled tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled>(p);
  }();
  return fn;
}

// T2 of one lane as a 2-D tensor: rows = row pairs of `chunk` streams, each
// 224 columns x 16 bytes (as u32); box = 4 columns x 224 row pairs with the
// 64-byte swizzle K_B's tile uses.
bool encode_t2_map(CUtensorMap* map, void* t2, int chunk) {
  const PFN_cuTensorMapEncodeTiled enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {224 * 4, (cuuint64_t)chunk * 224};
  const cuuint64_t strides[1] = {224 * 16};
  const cuuint32_t box[2] = {kWarpsB * 4, 224};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, t2, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// T1 of one lane as a 2-D tensor: rows = packed columns q of `chunk` streams,
// each 448 rows x 8 bytes (as u32); box = one stripe's 14 rows x 224 columns.
bool encode_t1_map(CUtensorMap* map, void* t1, int chunk) {
  const PFN_cuTensorMapEncodeTiled enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {448 * 2, (cuuint64_t)chunk * 224};
  const cuuint64_t strides[1] = {448 * 8};
  const cuuint32_t box[2] = {14 * 2, 224};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, t1, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// K_D1 for streams [b0, b0 + nb) once their energies exist (after K_A on
// `after`).  fc_select forks it onto the plan's aux stream so it runs beside
// K_B / K_C; the split-phase front (and profiling) launch it in order on
// `after` itself (`fork` false).
void launch_rank(const fc_plan* pl, const fc_config& cfg, const KParams& kp, int b0, int nb, cudaStream_t after,
                 bool fork, Recorder* rec) {
  cudaStream_t rs = after;
  if (fork) {
    cudaEventRecord(pl->ev_a, after);
    cudaStreamWaitEvent(pl->aux, pl->ev_a, 0);
    rs = pl->aux;
  }
  // FC_RANK_NT: threads per stream of K_D1 (default 512 at <= 128 streams)
  static const int rank_nt = env_int("FC_RANK_NT", 0, 0, 512);
  const bool wide = rank_nt ? rank_nt >= 512 : nb <= kSmallBatch;
  if (pl->probe_skip & 2) {
  } else if (wide) {
    k_rank<512><<<nb, 512, pl->smemR, rs>>>(kp, cfg.edge_lambda, b0);
  } else {
    k_rank<FC_SEL_THREADS><<<nb, FC_SEL_THREADS, pl->smemR, rs>>>(kp, cfg.edge_lambda, b0);
  }
  if (rec) rec->mark(after, 4);
}

// The split-phase front writes every chunk's row spectra before the back
// reads them: each chunk needs its own T1 buffers (chunks <= lanes).
bool split_ok(const fc_plan* pl) {
  return !pl->fast || (pl->g.batch + pl->chunk - 1) / pl->chunk <= pl->lanes;
}

// Launch `k` on `st`, as a programmatic dependent of the previous kernel on
// the stream when `pdl` (the kernel waits with griddepcontrol.wait before it
// reads its predecessor's outputs).
template <typename... P, typename... A>
void launch_maybe_pdl(bool pdl, void (*k)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A... args) {
  if (!pdl) {
    k<<<grid, block, smem, st>>>(args...);
    return;
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = grid;
  lc.blockDim = block;
  lc.dynamicSmemBytes = smem;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  cudaLaunchKernelEx(&lc, k, static_cast<P>(args)...);
}

// Which kernels a call launches: the whole select, or one half of the
// split-phase select (front: K_A + K_D1 of a step; back: K_B + K_C + K_D).
enum Part { kAll = 0, kFront = 1, kBack = 2, kCols = 3, kTail = 4 };

// Internal lane streams and fork / join events of one part: the front of
// step t + 1 and the back of step t run concurrently, so they never share a
// stream (which would serialise them) or an event.
struct LaneSet {
  const cudaStream_t* lane;
  cudaEvent_t fork;
  const cudaEvent_t* join;
};

// Returns FC_OK, or FC_ECUDA (nothing launched) when a tensor map cannot be
// encoded for this call's workspace.
int launch_select(const fc_plan* pl, const fc_config& cfg, const void* frames, const KParams& kp,
                  const fc_select_out& out, cudaStream_t st, Recorder* rec, Part part = kAll) {
  const int B = pl->g.batch;
  const bool front = part == kAll || part == kFront;
  const bool back = part != kFront;
  const bool do_b = part == kAll || part == kBack || part == kCols;
  const bool do_c = part == kAll || part == kBack || part == kTail;
  if (pl->fast) {
    const int ls_i = part == kAll ? 0 : part == kFront ? 1 : 2;
    const LaneSet set = {pl->lanes3[ls_i], pl->fork3[ls_i], pl->join3[ls_i]};
    // tensor maps of every lane's T1 / T2 first, so a failure launches nothing
    CUtensorMap tm1[kMaxLanes], tm2[kMaxLanes];
    std::memset(tm1, 0, sizeof(tm1));
    std::memset(tm2, 0, sizeof(tm2));
    // the split-phase halves overlap each other across steps already: they
    // launch the whole batch as one chunk (FC_SPLIT_LANES=1: the plan's
    // chunks on its lanes)
    static const int split_lanes = env_int("FC_SPLIT_LANES", 0, 0, 1);
    const bool whole = part != kAll && !split_lanes;
    const int chunk = whole ? B : pl->chunk;
    const int nmap = whole ? 1 : pl->lanes;
    for (int l = 0; l < nmap; ++l) {
      uint8_t* t1 = reinterpret_cast<uint8_t*>(kp.T) + l * pl->lane_t1;
      uint8_t* t2 = reinterpret_cast<uint8_t*>(kp.T2) + l * pl->lane_t2;
      if (front && pl->t1_tma && !encode_t1_map(&tm1[l], t1, chunk)) return FC_ECUDA;
      if (back && pl->t2_tma && !encode_t2_map(&tm2[l], t2, chunk)) return FC_ECUDA;
    }
    // Chunks of `chunk` streams run A -> B -> C on `lanes` internal streams
    // (each lane owns its T1/T2 slice) so one chunk's tail overlaps the next
    // chunk's head; the caller stream forks to and joins from the lanes.
    // Profiling runs the chunks serially on the caller stream.
    auto fa = (FastRowsFwd)sel_fast_rows_fwd(pl->g.format, pl->t1_tma);
    const int nl = (rec || whole) ? 1 : pl->lanes;
    // one whole-batch chunk runs on the caller's stream: no fork / join
    const bool direct = rec || whole;
    if (!direct) {
      cudaEventRecord(set.fork, st);
      for (int l = 0; l < nl; ++l) cudaStreamWaitEvent(set.lane[l], set.fork, 0);
    }
    int c = 0;
    for (int b0 = 0; b0 < B; b0 += chunk, ++c) {
      const int nb = B - b0 < chunk ? B - b0 : chunk;
      const int l = whole ? 0 : c % pl->lanes;   // the lane's T1 / T2 buffers
      const cudaStream_t ls = direct ? st : set.lane[c % nl];
      KParams kl = kp;
      kl.T = reinterpret_cast<float2*>(reinterpret_cast<uint8_t*>(kp.T) + l * pl->lane_t1);
      kl.T2 = reinterpret_cast<float2*>(reinterpret_cast<uint8_t*>(kp.T2) + l * pl->lane_t2);
      if (front) {
        if (!(pl->probe_skip & 1))
          fa<<<dim3(32, nb), kThreadsA448, pl->smemA, ls>>>(kl, pl->dct14, frames, b0, 1, tm1[l]);
        if (rec) rec->mark(st, 0);
        launch_rank(pl, cfg, kp, b0, nb, ls, part == kAll && !rec, rec);
      }
      if (back && pl->fused_bc) {
        k448_colsinv<true><<<dim3(kClusterBC, nb), 32 * kWarpsBC, kSmemBC, ls>>>(kl, b0);
        if (rec) rec->mark(st, 1);
      } else if (back && pl->flow_bc && do_b && do_c) {
        auto ff = (void (*)(KParams, int, int, int, int, CUtensorMap))pl->fnF;
        ff<<<(nb + pl->flow_lag) * (kNCB448 + kNRG448), 32 * kWarpsB, pl->smemB, ls>>>(kl, b0, nb, pl->flow_lag, l,
                                                                                         tm2[l]);
        if (rec) rec->mark(st, 1);
      } else if (back) {
        if (do_b && !(pl->probe_skip & 4)) {
          auto fb = (void (*)(KParams, int, CUtensorMap))pl->fnB;
          fb<<<dim3(kNCB448, nb), 32 * kWarpsB, pl->smemB, ls>>>(kl, b0, tm2[l]);
          if (rec) rec->mark(st, 1);
        }
        if (do_c && !(pl->probe_skip & 8)) {
          auto fc = (void (*)(KParams, int))pl->fnC;
          launch_maybe_pdl(pl->pdl && part == kBack && do_b && !rec, fc, dim3(kNRG448 / pl->kc_ppw, nb),
                           dim3(32 * kWarpsC), pl->smemC, ls, kl, b0);
          if (rec) rec->mark(st, 2);
        }
      }
    }
    if (!direct) {
      for (int l = 0; l < nl; ++l) {
        cudaEventRecord(set.join[l], set.lane[l]);
        cudaStreamWaitEvent(st, set.join[l], 0);
      }
    }
  } else {
    const dim3 blk(FC_THREADS);
    if (front) {
      auto fa = (void (*)(KParams, const void*, int))sel_rows_fwd(pl->kw);
      fa<<<dim3(kp.rows, B), blk, pl->smemA, st>>>(kp, frames, 1);
      if (rec) rec->mark(st, 0);
      launch_rank(pl, cfg, kp, 0, B, st, part == kAll && !rec, rec);
    }
    if (do_b) {
      auto fb = (void (*)(KParams))sel_cols(pl->kh);
      fb<<<dim3(kp.NCB, B), blk, pl->smemB, st>>>(kp);
      if (rec) rec->mark(st, 1);
    }
    if (do_c) {
      auto fc = (void (*)(KParams))sel_rows_inv(pl->kw);
      fc<<<dim3(kp.NRG, B), blk, pl->smemC, st>>>(kp);
      if (rec) rec->mark(st, 2);
    }
  }
  if (!back || part == kCols) return FC_OK;
  if (part == kAll && !rec) {  // K_D waits for the K_D1 branch
    cudaEventRecord(pl->ev_aux, pl->aux);
    cudaStreamWaitEvent(st, pl->ev_aux, 0);
  }
  // small batches leave SMs idle during the per-stream selection: give each
  // stream more threads there (FC_SEL_NT overrides)
  static const int nt_env = env_int("FC_SEL_NT", 0, 0, 1024);
  const int nt = nt_env ? nt_env : (B <= 128 ? 512 : FC_SEL_THREADS);
  // PDL only where K_D directly follows K_C on the caller's stream
  const bool pdl_d = pl->pdl && pl->fast && part == kBack && !rec && !pl->fused_bc && !pl->flow_bc &&
                     !(pl->probe_skip & 8);
  if (pl->probe_skip & 16) {
  } else if (nt >= 1024) {
    launch_maybe_pdl(pdl_d, k_select<1024>, dim3(B), dim3(1024), pl->smemD, st, kp, cfg, out);
  } else if (nt >= 512) {
    launch_maybe_pdl(pdl_d, k_select<512>, dim3(B), dim3(512), pl->smemD, st, kp, cfg, out);
  } else {
    launch_maybe_pdl(pdl_d, k_select<FC_SEL_THREADS>, dim3(B), dim3(FC_SEL_THREADS), pl->smemD, st, kp, cfg, out);
  }
  if (rec) rec->mark(st, 3);
  return FC_OK;
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
  if (g.format < FC_FMT_RGB_F32 || g.format > FC_FMT_RGB_U8) return FC_EINVAL;
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
  pl->fast = (H == 448 && W == 448 && P == 14);
  pl->kw = (W == 448 || W == 224) ? W : 0;
  pl->kh = (H == 448 || H == 224) ? H : 0;
  const size_t B = g.batch;

  int NP2 = 1;
  while (NP2 < N) NP2 <<= 1;
  pl->smemD = (size_t)N * 4 * 2 + (size_t)N * 3;   // K_D: reuse list, ranks, fresh / reuse / candidate flags
  pl->smemR = (size_t)NP2 * 8 + (size_t)NP2 * 4;    // K_D1: (E, index) sort keys
  size_t specElems, off = 0;
  if (pl->fast) {
    // small batches (e.g. 512 / N streams per GPU at N = 4, 8) run as two
    // half-batch chunks on two lanes, so one chunk's kernel tails overlap the
    // other's (64 streams: +7 % measured); larger batches as one chunk
    const bool halves = B <= (size_t)kSmallBatch && B >= 2;
    const int want = env_int("FC_CHUNK", halves ? (int)((B + 1) / 2) : kChunkDefault, 1, 4096);
    pl->chunk = (int)(B < (size_t)want ? B : (size_t)want);
    const int nchunks = (int)((B + pl->chunk - 1) / pl->chunk);
    pl->lanes = env_int("FC_LANES", halves ? 2 : kLanesDefault, 1, kMaxLanes);
    if (pl->lanes > nchunks) pl->lanes = nchunks;
    pl->smemA = (size_t)kPxBytes448;
    pl->smemB = (size_t)kSmemB448;
    pl->smemC = (size_t)kSmemC448 * env_int("FC_KC_PPW", 1, 1, 2);
    // K_B / K_C, or the fused cluster kernel K_BC (FC_FUSED_BC=1), whose
    // partials are one per column / one per warp
    pl->fused_bc = env_int("FC_FUSED_BC", 0, 0, 1) != 0;
    // K_C row pairs per warp (FC_KC_PPW): 2 shares twiddles, gather indices
    // and reductions between two transforms
    pl->kc_ppw = env_int("FC_KC_PPW", 1, 1, 2);
    kp.NCB = pl->fused_bc ? kNCBf : kNCB448;   // stats partials per stream
    kp.NRG = pl->fused_bc ? kNRGf : kNRG448 / pl->kc_ppw;   // peak partials per stream
    // [T1 slot 0: lanes x chunk streams | T1 slot 1 | T2], lanes contiguous
    // inside each, so a launch over the whole batch can also address them
    pl->lane_t1 = (size_t)pl->chunk * 224 * 448 * sizeof(float2);
    pl->lane_t2 = (size_t)pl->chunk * 448 * 224 * sizeof(float2);
    pl->off_T = off;
    pl->slot_T = align_up(pl->lane_t1 * pl->lanes);
    pl->off_T2 = off + 2 * pl->slot_T;
    off = pl->off_T2 + align_up(pl->lane_t2 * pl->lanes);
    specElems = B * 224 * kStColG * 2;  // register-order state (float2 count)
  } else {
    pl->chunk = g.batch;
    const int maxpairC = (kp.RG + 1) / 2;
    pl->smemA = (size_t)P * W * 8 + (size_t)kp.npairA * W * 8 + (size_t)W * 8 + (size_t)kp.cut * P * 8;
    pl->smemB = (size_t)2 * H * FC_CB * 8 + (size_t)H * 8;
    pl->smemC = (size_t)2 * maxpairC * W * 8 + (size_t)W * 8;
    specElems = B * kp.NCB * (size_t)H * FC_CB;
    pl->off_T = off;
    pl->slot_T = align_up(specElems * sizeof(float2));
    off += 2 * pl->slot_T;
  }
  const size_t kMaxSmem = 227 * 1024;
  if (pl->smemA > kMaxSmem || pl->smemB > kMaxSmem || pl->smemC > kMaxSmem || pl->smemD > kMaxSmem) {
    delete pl;
    return FC_EUNSUPPORTED;
  }
  pl->off_stripes = off;
  pl->slot_stripes = align_up(B * rows * sizeof(StripeStat));
  off += 2 * pl->slot_stripes;
  pl->off_stats = off; off = align_up(off + B * kp.NCB * 4 * sizeof(double));
  pl->off_peaks = off; off = align_up(off + B * kp.NRG * sizeof(PeakPart));
  pl->off_energy = off; off = align_up(off + B * N * sizeof(double));
  pl->off_order = off;
  pl->slot_order = align_up(B * N * sizeof(int16_t));
  off += 2 * pl->slot_order;
  pl->off_freshm = off;
  pl->slot_freshm = align_up(B * N);
  off += 2 * pl->slot_freshm;
  pl->off_estats = off;
  pl->slot_estats = align_up(B * 4 * sizeof(double));
  off += 2 * pl->slot_estats;
  pl->off_flow = off;   // zero-initialised with the workspace; every flow launch re-arms it
  off = align_up(off + ((size_t)kMaxFlowLanes * kFlowTicketStride + 2 * B) * sizeof(int));
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
  std::vector<float2> t448(6 * 64), t64(7 * 8);
  for (int k1 = 1; k1 < 7; ++k1)
    for (int n2 = 0; n2 < 64; ++n2) t448[(k1 - 1) * 64 + n2] = root((long long)n2 * k1, 448);
  for (int m2 = 1; m2 < 8; ++m2)
    for (int j1 = 0; j1 < 8; ++j1) t64[(m2 - 1) * 8 + j1] = root((long long)m2 * j1, 64);
  if (pl->fast)
    for (int u = 0; u < 3; ++u)
      for (int x = 0; x < 14; ++x) pl->dct14.c[u][x] = dct[(size_t)u * 14 + x];

  int rc = FC_OK;
  auto up = [&](void** dst, const void* src, size_t bytes) {
    if (rc != FC_OK) return;
    if (cudaMalloc(dst, bytes) != cudaSuccess || cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice) != cudaSuccess)
      rc = FC_ECUDA;
  };
  up((void**)&pl->d_twW, tw.data(), W * sizeof(float2));
  up((void**)&pl->d_twH, th.data(), H * sizeof(float2));
  up((void**)&pl->d_dct, dct.data(), dct.size() * sizeof(double));
  up((void**)&pl->d_tw448, t448.data(), t448.size() * sizeof(float2));
  up((void**)&pl->d_tw64, t64.data(), t64.size() * sizeof(float2));
  if (rc == FC_OK &&
      (cudaStreamCreateWithFlags(&pl->aux, cudaStreamNonBlocking) != cudaSuccess ||
       cudaEventCreateWithFlags(&pl->ev_a, cudaEventDisableTiming) != cudaSuccess ||
       cudaEventCreateWithFlags(&pl->ev_aux, cudaEventDisableTiming) != cudaSuccess))
    rc = FC_ECUDA;
  for (int k = 0; k < 3 && rc == FC_OK && pl->fast; ++k) {
    if (cudaEventCreateWithFlags(&pl->fork3[k], cudaEventDisableTiming) != cudaSuccess) rc = FC_ECUDA;
    for (int l = 0; l < pl->lanes && rc == FC_OK; ++l) {
      if (cudaStreamCreateWithFlags(&pl->lanes3[k][l], cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&pl->join3[k][l], cudaEventDisableTiming) != cudaSuccess)
        rc = FC_ECUDA;
    }
  }
  if (rc == FC_OK) {
    if (pl->fast) {
      // T1 by TMA tensor store (FC_T1_TMA=0: per-thread stores)
      pl->t1_tma = env_int("FC_T1_TMA", 1, 0, 1) && tensor_map_encoder() != nullptr;
      if (pl->t1_tma) {
        CUtensorMap probe;   // parameters check only (no memory access)
        pl->t1_tma = encode_t1_map(&probe, reinterpret_cast<void*>(256), pl->chunk);
      }
      rc = set_smem(sel_fast_rows_fwd(g.format, pl->t1_tma), pl->smemA);
      // occupancy variants: FC_OCC_B / FC_OCC_C = target CTAs per SM (register
      // cap); twiddles are read at use (lazy) when the cap is tight
      const int ob = env_int("FC_OCC_B", 6, 4, 8), oc = env_int("FC_OCC_C", 7, 4, 10);
      // T2 by TMA tensor store (FC_T2_TMA=0: copy loop) when the driver offers
      // the tensor-map encoder
      pl->t2_tma = env_int("FC_T2_TMA", 1, 0, 1) && tensor_map_encoder() != nullptr;
      if (pl->t2_tma) {
        CUtensorMap probe;   // parameters check only (no memory access)
        pl->t2_tma = encode_t2_map(&probe, reinterpret_cast<void*>(256), pl->chunk);
      }
      pl->fnB = pl->t2_tma ? (ob >= 6 ? (void*)k448_cols<6, true, true> : ob == 5 ? (void*)k448_cols<5, false, true>
                                                                            : (void*)k448_cols<4, false, true>)
                           : (ob >= 6 ? (void*)k448_cols<6, true, false> : ob == 5 ? (void*)k448_cols<5, false, false>
                                                                             : (void*)k448_cols<4, false, false>);
      if (pl->kc_ppw == 2)
        pl->fnC = oc >= 7 ? (void*)k448_rows_inv<7, true, 2> : (void*)k448_rows_inv<6, true, 2>;
      else
        pl->fnC = oc >= 10 ? (void*)k448_rows_inv<10, true> : oc >= 8 ? (void*)k448_rows_inv<8, true>
                : oc == 7 ? (void*)k448_rows_inv<7, true> : (void*)k448_rows_inv<6, false>;
      if (rc == FC_OK) rc = set_smem(pl->fnB, pl->smemB);
      if (rc == FC_OK) rc = set_smem(pl->fnC, pl->smemC);
      if (rc == FC_OK && pl->fused_bc) rc = set_smem((void*)k448_colsinv<true>, kSmemBC);
      // K_B + K_C flow kernel (FC_BC_FLOW=1; FC_BC_LAG streams of lag,
      // FC_BC_DISCARD=0 keeps the T2 lines in L2 after use)
      pl->flow_bc = env_int("FC_BC_FLOW", 0, 0, 1) && pl->t2_tma && !pl->fused_bc && pl->kc_ppw == 1;
      pl->flow_lag = env_int("FC_BC_LAG", 8, 1, 256);
      // timing probes (scripts/skip_probe.sh): 1 K_A, 2 K_D1, 4 K_B, 8 K_C,
      // 16 K_D are not launched — results are invalid
      pl->probe_skip = env_int("FC_PROBE_SKIP", 0, 0, 31);
      pl->pdl = env_int("FC_PDL", 0, 0, 1) != 0;
      pl->probe_back = getenv("FC_PROBE_BACK_PART") != nullptr;
      if (pl->flow_bc) {
        pl->fnF = env_int("FC_BC_DISCARD", 1, 0, 1) ? (void*)k448_bc_flow<6, true> : (void*)k448_bc_flow<6, false>;
        if (rc == FC_OK) rc = set_smem(pl->fnF, pl->smemB);
      }
    } else {
      rc = set_smem(sel_rows_fwd(pl->kw), pl->smemA);
      if (rc == FC_OK) rc = set_smem(sel_cols(pl->kh), pl->smemB);
      if (rc == FC_OK) rc = set_smem(sel_rows_inv(pl->kw), pl->smemC);
    }
    if (rc == FC_OK) rc = set_smem((void*)k_select<FC_SEL_THREADS>, pl->smemD);
    if (rc == FC_OK) rc = set_smem((void*)k_select<512>, pl->smemD);
    if (rc == FC_OK) rc = set_smem((void*)k_select<1024>, pl->smemD);
    if (rc == FC_OK) rc = set_smem((void*)k_rank<FC_SEL_THREADS>, pl->smemR);
    if (rc == FC_OK) rc = set_smem((void*)k_rank<512>, pl->smemR);
  }
  if (rc != FC_OK) {
    fc_plan_destroy(pl);
    return rc;
  }
  kp.twW = pl->d_twW;
  kp.twH = pl->d_twH;
  kp.dct = pl->d_dct;
  kp.tw448 = pl->d_tw448;
  kp.tw64 = pl->d_tw64;
  *out = pl;
  return FC_OK;
}

void fc_plan_destroy(fc_plan* pl) {
  if (!pl) return;
  if (pl->d_twW) cudaFree(pl->d_twW);
  if (pl->d_twH) cudaFree(pl->d_twH);
  if (pl->d_dct) cudaFree(pl->d_dct);
  if (pl->d_tw448) cudaFree(pl->d_tw448);
  if (pl->d_tw64) cudaFree(pl->d_tw64);
  for (int k = 0; k < 3; ++k) {
    for (int l = 0; l < kMaxLanes; ++l) {
      if (pl->lanes3[k][l]) cudaStreamDestroy(pl->lanes3[k][l]);
      if (pl->join3[k][l]) cudaEventDestroy(pl->join3[k][l]);
    }
    if (pl->fork3[k]) cudaEventDestroy(pl->fork3[k]);
  }
  if (pl->aux) cudaStreamDestroy(pl->aux);
  if (pl->ev_a) cudaEventDestroy(pl->ev_a);
  if (pl->ev_aux) cudaEventDestroy(pl->ev_aux);
  delete pl;
}

int64_t fc_plan_state_bytes(const fc_plan* pl) { return pl ? (int64_t)pl->state_bytes : -1; }
int64_t fc_plan_workspace_bytes(const fc_plan* pl) { return pl ? (int64_t)pl->ws_bytes : -1; }
int fc_plan_tokens(const fc_plan* pl) { return pl ? pl->kp.N : -1; }
int fc_plan_launches(const fc_plan* pl) {
  if (!pl) return -1;
  // fast: K_A, K_D1, K_B, K_C (or K_BC) per chunk + K_D; generic: the five kernels once
  return pl->fast ? (pl->fused_bc || pl->flow_bc ? 3 : 4) * ((pl->g.batch + pl->chunk - 1) / pl->chunk) + 1 : 5;
}

int fc_state_reset(const fc_plan* pl, void* state, int32_t first, int32_t count, void* stream) {
  if (!pl || !state || first < 0 || count < 0 || first + count > pl->g.batch) return FC_EINVAL;
  if (count == 0) return FC_OK;
  k_state_reset<<<(count + 255) / 256, 256, 0, as_stream(stream)>>>(reinterpret_cast<StreamHdr*>(state),
                                                                    first, count);
  return launch_check();
}

int fc_select(const fc_plan* pl, const fc_config* cfg, const void* frames, void* state, void* ws,
              const fc_select_out* out, void* stream) {
  if (!pl || !cfg || !frames || !state || !ws || !out) return FC_EINVAL;
  // bulk (TMA) copies stage state and workspace (and the fast path's frames): 16-byte alignment
  if (((pl->fast ? reinterpret_cast<uintptr_t>(frames) : 0) | reinterpret_cast<uintptr_t>(state) |
       reinterpret_cast<uintptr_t>(ws)) & 15)
    return FC_EINVAL;
  const int rc = check_cfg(cfg);
  if (rc != FC_OK) return rc;
  const KParams kp = bind(pl, state, ws, out->energy);
  const int lrc = launch_select(pl, *cfg, frames, kp, *out, as_stream(stream), nullptr);
  if (lrc != FC_OK) return lrc;
  return launch_check();
}

int fc_select_front(const fc_plan* pl, const fc_config* cfg, const void* frames, void* ws,
                    const fc_select_out* out, int32_t slot, void* stream) {
  if (!pl || !cfg || !frames || !ws || !out || (slot != 0 && slot != 1)) return FC_EINVAL;
  if (((pl->fast ? reinterpret_cast<uintptr_t>(frames) : 0) | reinterpret_cast<uintptr_t>(ws)) & 15)
    return FC_EINVAL;
  const int rc = check_cfg(cfg);
  if (rc != FC_OK) return rc;
  if (!split_ok(pl)) return FC_EUNSUPPORTED;
  const KParams kp = bind(pl, nullptr, ws, out->energy, slot);
  const int lrc = launch_select(pl, *cfg, frames, kp, *out, as_stream(stream), nullptr, kFront);
  if (lrc != FC_OK) return lrc;
  return launch_check();
}

int fc_select_back(const fc_plan* pl, const fc_config* cfg, void* state, void* ws, const fc_select_out* out,
                   int32_t slot, void* stream) {
  if (!pl || !cfg || !state || !ws || !out || (slot != 0 && slot != 1)) return FC_EINVAL;
  if ((reinterpret_cast<uintptr_t>(state) | reinterpret_cast<uintptr_t>(ws)) & 15) return FC_EINVAL;
  const int rc = check_cfg(cfg);
  if (rc != FC_OK) return rc;
  if (!split_ok(pl)) return FC_EUNSUPPORTED;
  const KParams kp = bind(pl, state, ws, out->energy, slot);
  // timing probe only (scripts/): FC_PROBE_BACK_PART=cols|tail launches one
  // half of the back (no ordering of the shared T2 / sums: results invalid)
  const char* pp = pl->probe_back ? getenv("FC_PROBE_BACK_PART") : nullptr;
  const Part part = !pp ? kBack : !strcmp(pp, "cols") ? kCols : !strcmp(pp, "tail") ? kTail : kBack;
  const int lrc = launch_select(pl, *cfg, nullptr, kp, *out, as_stream(stream), nullptr, part);
  if (lrc != FC_OK) return lrc;
  return launch_check();
}

int fc_select_profile(const fc_plan* pl, const fc_config* cfg, const void* frames, void* state, void* ws,
                      const fc_select_out* out, float* kernel_ms, void* stream) {
  if (!pl || !cfg || !frames || !state || !ws || !out || !kernel_ms) return FC_EINVAL;
  if (((pl->fast ? reinterpret_cast<uintptr_t>(frames) : 0) | reinterpret_cast<uintptr_t>(state) |
       reinterpret_cast<uintptr_t>(ws)) & 15)
    return FC_EINVAL;
  int rc = check_cfg(cfg);
  if (rc != FC_OK) return rc;
  const cudaStream_t st = as_stream(stream);
  const KParams kp = bind(pl, state, ws, out->energy);
  const int cap = 4 * ((pl->g.batch + pl->chunk - 1) / pl->chunk) + 3;  // serial chunks
  std::vector<cudaEvent_t> ev(cap);
  std::vector<int> kind(cap);
  for (auto& e : ev) cudaEventCreate(&e);
  Recorder r;
  r.ev = ev.data();
  r.kind = kind.data();
  r.cap = cap;
  r.mark(st, -1);
  rc = launch_select(pl, *cfg, frames, kp, *out, st, &r);
  if (rc == FC_OK) rc = launch_check();
  cudaStreamSynchronize(st);
  for (int k = 0; k < 5; ++k) kernel_ms[k] = 0.f;
  for (int i = 1; i < r.n; ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
    if (kind[i] >= 0 && kind[i] < 5) kernel_ms[kind[i]] += ms;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return rc;
}

int fc_patch_energy(const fc_plan* pl, const void* frames, void* ws, double* energy, void* stream) {
  if (!pl || !frames || !ws || !energy) return FC_EINVAL;
  // the 448 path bulk-copies frame stripes (16-byte aligned sources), as fc_select
  if (((pl->fast ? reinterpret_cast<uintptr_t>(frames) : 0) | reinterpret_cast<uintptr_t>(ws)) & 15)
    return FC_EINVAL;
  const KParams kp = bind(pl, nullptr, ws, energy);
  const cudaStream_t st = as_stream(stream);
  if (pl->fast) {
    auto fn = (FastRowsFwd)sel_fast_rows_fwd(pl->g.format, pl->t1_tma);
    CUtensorMap none;   // energies only: no T1 store
    std::memset(&none, 0, sizeof(none));
    fn<<<dim3(32, pl->g.batch), kThreadsA448, pl->smemA, st>>>(kp, pl->dct14, frames, 0, 0, none);
  } else {
    auto fn = (void (*)(KParams, const void*, int))sel_rows_fwd(pl->kw);
    fn<<<dim3(kp.rows, pl->g.batch), FC_THREADS, pl->smemA, st>>>(kp, frames, 0);
  }
  return launch_check();
}

static int splice_impl(int32_t batch, int32_t n_tokens, int64_t row_bytes, const int32_t* src_map,
                       const void* cache, const int64_t* cache_ages, const void* fresh, int compact,
                       int32_t fresh_rows, const int64_t* fresh_off, void* out, int64_t* out_ages,
                       int32_t* status, cudaStream_t st) {
  const int total = batch * n_tokens;
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
        reinterpret_cast<const int4*>(fresh), compact, fresh_rows, fresh_off, reinterpret_cast<int4*>(out),
        out_ages, status);
  } else {
    k_splice_bytes<<<total, 128, 0, st>>>(total, n_tokens, row_bytes, src_map,
                                          reinterpret_cast<const uint8_t*>(cache), cache_ages,
                                          reinterpret_cast<const uint8_t*>(fresh), compact, fresh_rows, fresh_off,
                                          reinterpret_cast<uint8_t*>(out), out_ages, status);
  }
  return launch_check();
}

int fc_splice(int32_t batch, int32_t n_tokens, int64_t row_bytes, const int32_t* src_map, const void* cache,
              const int64_t* cache_ages, const void* fresh, int32_t fresh_layout, int32_t fresh_rows, void* out,
              int64_t* out_ages, int32_t* status, void* stream) {
  if (batch < 1 || n_tokens < 1 || row_bytes < 1 || !src_map || !fresh || !out || !out_ages) return FC_EINVAL;
  if ((int64_t)batch * n_tokens > INT32_MAX) return FC_EINVAL;
  if (fresh_layout != FC_FRESH_DENSE && fresh_layout != FC_FRESH_COMPACT) return FC_EINVAL;
  if (fresh_layout == FC_FRESH_DENSE) fresh_rows = n_tokens;
  if (fresh_rows < 1) return FC_EINVAL;
  return splice_impl(batch, n_tokens, row_bytes, src_map, cache, cache_ages, fresh,
                     fresh_layout == FC_FRESH_COMPACT, fresh_rows, nullptr, out, out_ages, status, as_stream(stream));
}

int fc_splice_packed(int32_t batch, int32_t n_tokens, int64_t row_bytes, const int32_t* src_map,
                     const void* cache, const int64_t* cache_ages, const void* fresh,
                     const int64_t* fresh_offsets, void* out, int64_t* out_ages, int32_t* status, void* stream) {
  if (batch < 1 || n_tokens < 1 || row_bytes < 1 || !src_map || !fresh || !fresh_offsets || !out || !out_ages)
    return FC_EINVAL;
  if ((int64_t)batch * n_tokens > INT32_MAX) return FC_EINVAL;
  // a packed stream holds at most n_tokens recomputed rows
  return splice_impl(batch, n_tokens, row_bytes, src_map, cache, cache_ages, fresh, 1, n_tokens, fresh_offsets, out,
                     out_ages, status, as_stream(stream));
}

}  // extern "C"

using BulkFn = decltype(&k_splice_ip_bulk<2, 2>);
// Every (lanes, slots) instance the copier can be asked for: the caller sizes
// dynamic shared memory for exactly this NL and SL.
template <int NL>
static BulkFn pick_bulk_sl(int SL) {
  return SL == 4 ? k_splice_ip_bulk<NL, 4> : SL == 3 ? k_splice_ip_bulk<NL, 3> : k_splice_ip_bulk<NL, 2>;
}
static BulkFn pick_bulk(int NL, int SL) {
  switch (NL) {
    case 2: return pick_bulk_sl<2>(SL);
    case 4: return pick_bulk_sl<4>(SL);
    case 8: return pick_bulk_sl<8>(SL);
    default: return pick_bulk_sl<16>(SL);
  }
}

extern "C" {

int64_t fc_splice_inplace_scratch_bytes(int32_t batch, int32_t n_tokens) {
  return (int64_t)batch * n_tokens * 4 + (int64_t)batch * 4 + 256;
}

}  // extern "C"

namespace {

int splice_ip_check(int32_t batch, int32_t n_tokens, int64_t row_bytes, const int32_t* src_map, void* cache0,
                    void* cache1, int64_t* ages0, int64_t* ages1, const uint8_t* slot_in, uint8_t* slot_out,
                    const void* fresh, int32_t fresh_layout, int32_t& fresh_rows, void* scratch) {
  if (batch < 1 || n_tokens < 1 || row_bytes < 16 || row_bytes % 16 || !src_map || !cache0 || !cache1 || !ages0 ||
      !ages1 || !slot_in || !slot_out || !fresh || !scratch)
    return FC_EINVAL;
  if (((reinterpret_cast<uintptr_t>(cache0) | reinterpret_cast<uintptr_t>(cache1) |
        reinterpret_cast<uintptr_t>(fresh)) & 15) != 0)
    return FC_EINVAL;
  if (fresh_layout != FC_FRESH_DENSE && fresh_layout != FC_FRESH_COMPACT) return FC_EINVAL;
  if ((int64_t)batch * n_tokens > INT32_MAX || row_bytes > INT32_MAX) return FC_EINVAL;
  if (fresh_layout == FC_FRESH_DENSE) fresh_rows = n_tokens;
  if (fresh_rows < 1) return FC_EINVAL;
  return FC_OK;
}

// The copy half of the in-place splice: copier CTAs claiming the planned
// rows from the plan's work counter.  ctas > 0 sets the copier's CTA count
// (an extra launch then only takes the rows no earlier copier has claimed).
int splice_ip_copy(int32_t batch, int32_t n_tokens, int64_t row_bytes, const int32_t* src_map, void* cache0,
                   void* cache1, int64_t* ages0, int64_t* ages1, const uint8_t* slot_in, const uint8_t* slot_out,
                   const void* fresh, int32_t fresh_layout, int32_t fresh_rows, void* scratch, int32_t* status,
                   int ctas, cudaStream_t st);

}  // namespace

extern "C" {

int fc_splice_inplace_plan(int32_t batch, int32_t n_tokens, int64_t row_bytes, const int32_t* src_map,
                           void* cache0, void* cache1, int64_t* ages0, int64_t* ages1, const uint8_t* slot_in,
                           uint8_t* slot_out, const void* fresh, int32_t fresh_layout, int32_t fresh_rows,
                           void* scratch, void* stream) {
  const int rc = splice_ip_check(batch, n_tokens, row_bytes, src_map, cache0, cache1, ages0, ages1, slot_in, slot_out,
                                 fresh, fresh_layout, fresh_rows, scratch);
  if (rc != FC_OK) return rc;
  int32_t* rows = reinterpret_cast<int32_t*>(scratch);
  int32_t* counts = rows + (size_t)batch * n_tokens;
  k_splice_plan<<<batch, 256, 0, as_stream(stream)>>>(n_tokens, src_map, slot_in, slot_out, ages0, ages1, rows,
                                                       counts);
  return launch_check();
}

int fc_splice_inplace_copy(int32_t batch, int32_t n_tokens, int64_t row_bytes, const int32_t* src_map,
                           void* cache0, void* cache1, int64_t* ages0, int64_t* ages1, const uint8_t* slot_in,
                           const uint8_t* slot_out, const void* fresh, int32_t fresh_layout, int32_t fresh_rows,
                           void* scratch, int32_t* status, int32_t ctas, void* stream) {
  if (ctas < 0) return FC_EINVAL;
  const int rc = splice_ip_check(batch, n_tokens, row_bytes, src_map, cache0, cache1, ages0, ages1, slot_in,
                                 const_cast<uint8_t*>(slot_out), fresh, fresh_layout, fresh_rows, scratch);
  if (rc != FC_OK) return rc;
  return splice_ip_copy(batch, n_tokens, row_bytes, src_map, cache0, cache1, ages0, ages1, slot_in, slot_out, fresh,
                        fresh_layout, fresh_rows, scratch, status, ctas, as_stream(stream));
}

int fc_splice_inplace(int32_t batch, int32_t n_tokens, int64_t row_bytes, const int32_t* src_map, void* cache0,
                      void* cache1, int64_t* ages0, int64_t* ages1, const uint8_t* slot_in, uint8_t* slot_out,
                      const void* fresh, int32_t fresh_layout, int32_t fresh_rows, void* scratch, int32_t* status,
                      void* stream) {
  const int rc = fc_splice_inplace_plan(batch, n_tokens, row_bytes, src_map, cache0, cache1, ages0, ages1, slot_in,
                                        slot_out, fresh, fresh_layout, fresh_rows, scratch, stream);
  if (rc != FC_OK) return rc;
  if (fresh_layout == FC_FRESH_DENSE) fresh_rows = n_tokens;
  return splice_ip_copy(batch, n_tokens, row_bytes, src_map, cache0, cache1, ages0, ages1, slot_in, slot_out, fresh,
                        fresh_layout, fresh_rows, scratch, status, 0, as_stream(stream));
}

}  // extern "C"

namespace {

int splice_ip_copy(int32_t batch, int32_t n_tokens, int64_t row_bytes, const int32_t* src_map, void* cache0,
                   void* cache1, int64_t* ages0, int64_t* ages1, const uint8_t* slot_in, const uint8_t* slot_out,
                   const void* fresh, int32_t fresh_layout, int32_t fresh_rows, void* scratch, int32_t* status,
                   int ctas, cudaStream_t st) {
  int32_t* rows = reinterpret_cast<int32_t*>(scratch);
  int32_t* counts = rows + (size_t)batch * n_tokens;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // Bulk (TMA) copier unless disabled (FC_SPLICE_BULK=0) or the rows/batch do
  // not fit its shared-memory slots.
  // lanes per copier CTA: the compiled variants are 2, 4, 8 and 16
  const int NLreq = env_int("FC_SPLICE_BULK_NL", 8, 2, 16);
  const int NL = NLreq <= 2 ? 2 : NLreq <= 4 ? 4 : NLreq <= 8 ? 8 : 16;
  const int SL = env_int("FC_SPLICE_BULK_SLOTS", 2, 2, 4);
  const size_t bulk_smem = (size_t)NL * SL * row_bytes + (size_t)(batch + 1) * 4;
  const int use_bulk = env_int("FC_SPLICE_BULK", 1, 0, 1);
  if (use_bulk && bulk_smem <= 96 * 1024) {
    const int per_sm = env_int("FC_SPLICE_BULK_CTAS", 1, 1, 32);
    // FC_SPLICE_BULK_GRID: absolute copier CTA count (overrides per-SM sizing)
    const int grid_abs = env_int("FC_SPLICE_BULK_GRID", 0, 0, 1 << 16);
    const int grid = ctas > 0 ? ctas : grid_abs > 0 ? grid_abs : sms * per_sm;
    auto fn = pick_bulk(NL, SL);  // the (NL, SL) instance bulk_smem was sized for
    if (bulk_smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bulk_smem);
    fn<<<grid, 32, bulk_smem, st>>>(
        batch, n_tokens, (int)row_bytes, src_map, reinterpret_cast<char*>(cache0), reinterpret_cast<char*>(cache1),
        ages0, ages1, slot_in, slot_out, rows, counts, reinterpret_cast<const char*>(fresh),
        fresh_layout == FC_FRESH_COMPACT, fresh_rows, status);
    return launch_check();
  }
  // the non-TMA copier partitions the rows statically: an extra launch has
  // nothing left to claim
  if (ctas > 0) return FC_OK;
  const int total = batch * n_tokens;
  constexpr int UNR = 2;
  int blocks = ((total + UNR - 1) / UNR + (FC_THREADS / 32) - 1) / (FC_THREADS / 32);
  if (blocks > sms * 8) blocks = sms * 8;
  k_splice_ip<UNR><<<blocks, FC_THREADS, 0, st>>>(
      total, n_tokens, row_bytes / 16, src_map, reinterpret_cast<int4*>(cache0), reinterpret_cast<int4*>(cache1),
      ages0, ages1, slot_in, slot_out, rows, counts, reinterpret_cast<const int4*>(fresh),
      fresh_layout == FC_FRESH_COMPACT, fresh_rows, status);
  return launch_check();
}

}  // namespace

extern "C" {

int fc_compare_cosines(const fc_geometry* geom, const void* prev, const void* curr, double* visual_cos,
                       double* naive_cos, void* stream) {
  if (!geom || !prev || !curr || !visual_cos || !naive_cos) return FC_EINVAL;
  const fc_geometry& g = *geom;
  if (g.batch < 1 || g.height < 1 || g.width < 1 || g.patch_size < 2) return FC_EINVAL;
  if (g.format < FC_FMT_RGB_F32 || g.format > FC_FMT_RGB_U8) return FC_EINVAL;
  if (g.height % g.patch_size || g.width % g.patch_size) return FC_EINVAL;
  if (g.patch_size > 32) return FC_EUNSUPPORTED;
  CmpGeom cg;
  cg.B = g.batch; cg.H = g.height; cg.W = g.width; cg.P = g.patch_size; cg.fmt = g.format;
  cg.rows = g.height / g.patch_size;
  cg.cols = g.width / g.patch_size;
  cg.U = g.patch_size / 2 + 1;
  // patches per CTA: as many as fit ~96 KB, then balanced over the chunks
  int cmax = 1;
  while (cmax < cg.cols && compare_smem_bytes(cg.P, cmax + 1) <= 96 * 1024) ++cmax;
  cg.nchunk = (cg.cols + cmax - 1) / cmax;
  cg.cpp = (cg.cols + cg.nchunk - 1) / cg.nchunk;
  const size_t smem = compare_smem_bytes(cg.P, cg.cpp);
  if ((long long)cg.rows * cg.nchunk > 0x7fffffffLL || g.batch > 65535) return FC_EUNSUPPORTED;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_compare, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_compare<<<dim3(cg.rows * cg.nchunk, g.batch), 256, smem, as_stream(stream)>>>(cg, prev, curr, visual_cos,
                                                                                  naive_cos);
  return launch_check();
}

int fc_row_cosines(int64_t n, int64_t d, const double* a, const double* b, double* out, void* stream) {
  if (n < 0 || d < 0 || (n > 0 && (!a || !b || !out))) return FC_EINVAL;
  if (n == 0) return FC_OK;
  const int64_t blocks = (n * 32 + 255) / 256;
  if (blocks > 0x7fffffffLL) return FC_EUNSUPPORTED;
  k_row_cosines<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(n, d, a, b, out);
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

// ------------------------------------------------- fp64 spectral wrappers ----
// spectral.py:24-72 and migration.py:128-134 on the GPU (fc_spectral.cuh).

static size_t a256(size_t v) { return (v + 255) / 256 * 256; }

int64_t fc_dft2_workspace_bytes(int32_t h, int32_t w) {
  if (h < 1 || w < 1) return -1;
  return (int64_t)(a256((size_t)h * w * 16) + a256((size_t)w * 16) + a256((size_t)h * 16));
}

static int dft2_impl(int h, int w, const double* in, int in_complex, int inverse, double* out, uint8_t* ws,
                     cudaStream_t st) {
  double2* Y = reinterpret_cast<double2*>(ws);
  double2* twW = reinterpret_cast<double2*>(ws + a256((size_t)h * w * 16));
  double2* twH = reinterpret_cast<double2*>(reinterpret_cast<uint8_t*>(twW) + a256((size_t)w * 16));
  const int sign = inverse ? 1 : -1;
  spec::k_twiddles<<<(w + 255) / 256, 256, 0, st>>>(w, sign, twW);
  spec::k_twiddles<<<(h + 255) / 256, 256, 0, st>>>(h, sign, twH);
  const size_t smem = (size_t)w * 32;
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute((void*)spec::k_dft_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
          cudaSuccess)
    return FC_ECUDA;
  spec::k_dft_rows<<<dim3((w + spec::kThreads - 1) / spec::kThreads, h), spec::kThreads, smem, st>>>(
      h, w, in, in_complex, twW, Y);
  const double scale = inverse ? 1.0 / ((double)h * (double)w) : 1.0;
  spec::k_dft_cols<<<dim3((w + spec::kThreads - 1) / spec::kThreads, (h + spec::kTK - 1) / spec::kTK),
                     spec::kThreads, 0, st>>>(h, w, Y, twH, scale, out);
  return launch_check();
}

int fc_dft2(int32_t h, int32_t w, const double* in, int32_t in_complex, int32_t inverse, double* out, void* ws,
            void* stream) {
  if (h < 1 || w < 1 || h > 8192 || w > 6144 || !in || !out || !ws) return FC_EINVAL;
  return dft2_impl(h, w, in, in_complex, inverse, out, static_cast<uint8_t*>(ws), as_stream(stream));
}

int64_t fc_phase_correlation_workspace_bytes(int32_t h, int32_t w) {
  const int64_t d = fc_dft2_workspace_bytes(h, w);
  if (d < 0) return -1;
  return d + 2 * (int64_t)a256((size_t)h * w * 16) + (int64_t)a256(1024 * sizeof(spec::PeakD));
}

int fc_phase_correlation_spectra(int32_t h, int32_t w, const double* spec_prev, const double* spec_curr,
                                 int32_t* disp2, void* ws, void* stream) {
  if (h < 1 || w < 1 || h > 8192 || w > 6144 || !spec_prev || !spec_curr || !disp2 || !ws) return FC_EINVAL;
  const cudaStream_t st = as_stream(stream);
  uint8_t* base = static_cast<uint8_t*>(ws);
  const size_t grid = a256((size_t)h * w * 16);
  double* cross = reinterpret_cast<double*>(base + fc_dft2_workspace_bytes(h, w));
  double* resp = reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(cross) + grid);
  spec::PeakD* parts = reinterpret_cast<spec::PeakD*>(reinterpret_cast<uint8_t*>(resp) + grid);
  const int64_t n = (int64_t)h * w;
  const int nb = (int)((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024);
  spec::k_cross_power<<<nb, 256, 0, st>>>(n, spec_prev, spec_curr, 1e-12, cross);   // CROSS_POWER_EPS
  int rc = dft2_impl(h, w, cross, 1, 1, resp, base, st);
  if (rc != FC_OK) return rc;
  spec::k_peak_part<<<nb, spec::kThreads, 0, st>>>(h, w, resp, parts);
  spec::k_peak_fin<<<1, spec::kThreads, 0, st>>>(h, w, parts, nb, disp2);
  return launch_check();
}

int fc_block_dct(int32_t n_patches, int32_t p, const double* patches, double* out, void* stream) {
  if (n_patches < 0 || p < 1 || p > 64 || (n_patches > 0 && (!patches || !out))) return FC_EINVAL;
  if (n_patches == 0) return FC_OK;
  const size_t smem = (size_t)3 * p * p * sizeof(double);
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute((void*)spec::k_block_dct, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
          cudaSuccess)
    return FC_ECUDA;
  spec::k_block_dct<<<n_patches, spec::kThreads, smem, as_stream(stream)>>>(p, patches, out);
  return launch_check();
}

int fc_amplitude_phase(int64_t n, const double* spectrum, double* amp, double* phase, void* stream) {
  if (n < 0 || (n > 0 && (!spectrum || !amp || !phase))) return FC_EINVAL;
  if (n == 0) return FC_OK;
  const int nb = (int)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
  spec::k_amp_phase<<<nb, 256, 0, as_stream(stream)>>>(n, spectrum, amp, phase);
  return launch_check();
}

// ------------------------------------------------------------ CUDA graphs ----
// A whole pipelined step (select of step t beside the splice of step t - 1,
// forked onto a second stream) is captured once per ring phase and replayed,
// so the per-step host work is one graph launch.  Instantiated with node
// priorities so the splice branch keeps its stream's (higher) priority.

int fc_graph_capture_begin(void* stream) {
  return cudaStreamBeginCapture(as_stream(stream), cudaStreamCaptureModeThreadLocal) == cudaSuccess ? FC_OK
                                                                                                    : FC_ECUDA;
}

int fc_graph_capture_end(void* stream, void** exec) {
  if (!exec) return FC_EINVAL;
  *exec = nullptr;
  cudaGraph_t g = nullptr;
  if (cudaStreamEndCapture(as_stream(stream), &g) != cudaSuccess || !g) {
    cudaGetLastError();
    return FC_ECUDA;
  }
  cudaGraphExec_t ge = nullptr;
  const cudaError_t e = cudaGraphInstantiateWithFlags(&ge, g, cudaGraphInstantiateFlagUseNodePriority);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return FC_ECUDA;
  }
  *exec = ge;
  return FC_OK;
}

int fc_graph_launch(void* exec, void* stream) {
  if (!exec) return FC_EINVAL;
  return cudaGraphLaunch(static_cast<cudaGraphExec_t>(exec), as_stream(stream)) == cudaSuccess ? FC_OK : FC_ECUDA;
}

void fc_graph_destroy(void* exec) {
  if (exec) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(exec));
}

// ------------------------------------------------------ patch gather ----
// Recomputed tokens' pixels for an encoder (BASELINE config 4): packed row r
// of `out` is the P x P x 3 patch of token index[r] = b * N + p, read straight
// from the fp32 RGB frames and written as bf16 in (py, px, channel) order —
// the layout of a ViT patch embedding's input.  One warp per row; only the
// recomputed tokens' pixels are read.
namespace {
__global__ void k_gather_patches(int rows, int H, int W, int P, const float* __restrict__ frames,
                                 const int64_t* __restrict__ index, __nv_bfloat16* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int cols = W / P, n = (H / P) * cols, per = 3 * P * P;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += (gridDim.x * blockDim.x) >> 5) {
    const int64_t t = index[r];
    const int b = (int)(t / n), p = (int)(t - (int64_t)b * n);
    const int i = p / cols, j = p - (p / cols) * cols;
    const float* base = frames + (((size_t)b * H + (size_t)i * P) * W + (size_t)j * P) * 3;
    __nv_bfloat16* o = out + (size_t)r * per;
    for (int e = lane; e < per; e += 32) {
      const int py = e / (3 * P), rem = e - py * 3 * P;   // rem = px * 3 + channel
      o[e] = __float2bfloat16_rn(base[(size_t)py * W * 3 + rem]);
    }
  }
}
}  // namespace

int fc_gather_patches(int32_t rows, int32_t batch, int32_t height, int32_t width, int32_t patch_size,
                      const float* frames, const int64_t* index, void* out_bf16, void* stream) {
  if (rows < 0 || batch < 1 || patch_size < 1 || height % patch_size || width % patch_size) return FC_EINVAL;
  if (rows == 0) return FC_OK;
  if (!frames || !index || !out_bf16) return FC_EINVAL;
  const int blocks = (int)(((int64_t)rows * 32 + 255) / 256 < 8192 ? ((int64_t)rows * 32 + 255) / 256 : 8192);
  k_gather_patches<<<blocks, 256, 0, as_stream(stream)>>>(rows, height, width, patch_size, frames, index,
                                                         reinterpret_cast<__nv_bfloat16*>(out_bf16));
  return launch_check();
}

// --------------------------------------------------------- mask images ----

namespace {
__global__ void k_render_masks(int B, int N, const fc_stream_result* __restrict__ res,
                               const uint8_t* __restrict__ reuse, const uint8_t* __restrict__ fresh,
                               uint8_t* __restrict__ img) {
  // frameio.py:188-219: reused 255, edge-forced recompute 128, other 0;
  // flushed (and cold) steps render all-zero
  const int64_t total = (int64_t)B * N;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(i / N);
    const bool fl = res[b].flushed != 0;
    img[i] = fl ? 0 : (reuse[i] ? 255 : (fresh[i] ? 128 : 0));
  }
}
}  // namespace

int fc_render_masks(int32_t batch, int32_t n_tokens, const fc_stream_result* results, const uint8_t* reuse_mask,
                    const uint8_t* refresh_mask, uint8_t* img, void* stream) {
  if (batch < 1 || n_tokens < 1 || !results || !reuse_mask || !refresh_mask || !img) return FC_EINVAL;
  const int64_t total = (int64_t)batch * n_tokens;
  const int blocks = (int)((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
  k_render_masks<<<blocks, 256, 0, as_stream(stream)>>>(batch, n_tokens, results, reuse_mask, refresh_mask, img);
  return launch_check();
}

// ---------------------------------------------------------- stage ops ----

static int stage_blocks(int64_t n) {
  int64_t nb = (n + 1023) / 1024;
  if (nb < 1) nb = 1;
  if (nb > FC_STAGE_BLOCKS) nb = FC_STAGE_BLOCKS;
  return (int)nb;
}

int64_t fc_stage_workspace_bytes(void) { return FC_STAGE_WS_BYTES; }

// ws layout: [flags int32 | pad][out scratch 8 doubles][partials 4*FC_STAGE_BLOCKS doubles]
int fc_amp_cosine(const double* a, const double* b, int64_t n, void* ws, double* out3, int32_t* flags,
                  void* stream) {
  if (!a || !b || n < 1 || !ws || !out3 || !flags) return FC_EINVAL;
  const cudaStream_t st = as_stream(stream);
  double* part = reinterpret_cast<double*>(static_cast<char*>(ws) + 128);
  const int nb = stage_blocks(n);
  cudaMemsetAsync(flags, 0, sizeof(int32_t), st);
  stg::k_cos_part<<<nb, FC_STAGE_THREADS, 0, st>>>(a, b, n, part, flags);
  stg::k_final<3><<<1, FC_STAGE_THREADS, 0, st>>>(part, nb, out3, 1.0);
  return launch_check();
}

int fc_spectral_sums(const double* amp, int64_t n, int32_t include_dc, void* ws, double* out2, int32_t* flags,
                     void* stream) {
  if (!amp || n < 1 || !ws || !out2 || !flags) return FC_EINVAL;
  const cudaStream_t st = as_stream(stream);
  double* part = reinterpret_cast<double*>(static_cast<char*>(ws) + 128);
  const int nb = stage_blocks(n);
  cudaMemsetAsync(flags, 0, sizeof(int32_t), st);
  stg::k_pow_part<<<nb, FC_STAGE_THREADS, 0, st>>>(amp, n, include_dc, part, flags);
  stg::k_final<1><<<1, FC_STAGE_THREADS, 0, st>>>(part, nb, out2, 1.0);
  stg::k_plogp_part<<<nb, FC_STAGE_THREADS, 0, st>>>(amp, n, include_dc, out2, part);
  stg::k_final<1><<<1, FC_STAGE_THREADS, 0, st>>>(part, nb, out2 + 1, 1.0);
  return launch_check();
}

int fc_refresh_mask(const double* energy, int64_t n, double lam, void* ws, uint8_t* mask, double* stats3,
                    void* stream) {
  if (!energy || n < 1 || !ws || !mask || !stats3) return FC_EINVAL;
  const cudaStream_t st = as_stream(stream);
  double* sc = reinterpret_cast<double*>(static_cast<char*>(ws) + 64);  // [mean, m2]
  double* part = reinterpret_cast<double*>(static_cast<char*>(ws) + 128);
  const int nb = stage_blocks(n);
  stg::k_moment_part<<<nb, FC_STAGE_THREADS, 0, st>>>(energy, n, nullptr, part);
  stg::k_final<1><<<1, FC_STAGE_THREADS, 0, st>>>(part, nb, sc, (double)n, energy);
  stg::k_moment_part<<<nb, FC_STAGE_THREADS, 0, st>>>(energy, n, sc, part);
  stg::k_final<1><<<1, FC_STAGE_THREADS, 0, st>>>(part, nb, sc + 1, (double)n);
  const int tb = (int)((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024);
  stg::k_threshold<<<tb, 256, 0, st>>>(energy, n, sc, lam, mask, stats3);
  return launch_check();
}

int fc_topk_ascending(const int64_t* cand, int64_t m, const double* energies, int64_t n_energies, int64_t k,
                      int64_t* out, int32_t* flags, void* stream) {
  if (m < 0 || (m > 0 && (!cand || !energies || !out || !flags))) return FC_EINVAL;
  if (m == 0 || k <= 0) return FC_OK;
  if (m > 8192) return FC_EUNSUPPORTED;
  int np2 = 1;
  while (np2 < m) np2 <<= 1;
  const size_t smem = (size_t)np2 * 16;
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute((void*)stg::k_topk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return FC_ECUDA;
  const cudaStream_t st = as_stream(stream);
  cudaMemsetAsync(flags, 0, sizeof(int32_t), st);
  stg::k_topk<<<1, 1024, smem, st>>>(cand, (int)m, energies, n_energies, k, out, flags);
  return launch_check();
}

}  // extern "C"
