/*
 * freqcache_b200.h — C ABI of the B200-native FreqCache token-cache decision
 * path (select + splice).  Built for sm_100a; device pointers only; every call
 * is asynchronous on the caller's CUDA stream; no hidden global state (all
 * per-geometry constants live in an explicit fc_plan, all per-stream state in
 * caller-owned memory).
 *
 * The reference (arxiv 2604.24391 CPU package, /root/reference/pkg) has no
 * FFI: its operator API is the Python export list
 * pkg/src/freqcache/__init__.py:11-98.  Each entry point below names the
 * reference function(s) it replaces:
 *
 *   fc_select        fusion.py:121-242  decide()  (+ frame.py:6-15 validate,
 *                    frameio.py:26,85-88 luma, migration.py:87-185,
 *                    edge_refresh.py:48-73, budget.py:34-75,
 *                    fusion.py:104-115 topk_ascending, :245-262 invariants)
 *                    batched over B independent streams; the previous
 *                    frame's spectrum is carried in `state`, so each frame is
 *                    transformed once (the reference transforms both frames
 *                    of every pair).
 *   fc_splice        fusion.py:462-512  step()  token gather/scatter + ages
 *   fc_splice_map    fusion.py:481-504  reuse-source / recompute-order map of
 *                    an arbitrary (host-built) CacheDecision
 *   fc_patch_energy  edge_refresh.py:48-59 patch_energy()
 *   fc_state_reset   fusion.py:450-459 populate_cache() cold start (the next
 *                    fc_select on a reset stream establishes its spectrum)
 */
#ifndef FREQCACHE_B200_H
#define FREQCACHE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FC_ABI_VERSION 2  /* 2: splice entry points take a status word */

/* status codes (fc_strerror) */
#define FC_OK            0
#define FC_EINVAL        1  /* bad argument -> ValueError in the facade      */
#define FC_EUNSUPPORTED  2  /* geometry outside the kernel envelope          */
#define FC_ECUDA         3  /* CUDA runtime error                            */
#define FC_ENONFINITE    4  /* per stream: frame has NaN/Inf (frame.py:13)   */
#define FC_EPSI          5  /* per stream: psi outside [0,1] (budget.py:69)  */
#define FC_EBOUNDS       6  /* splice source out of bounds (fusion.py:488)   */

/* CacheDecision.diagnostic codes */
#define FC_DIAG_NONE        0
#define FC_DIAG_DEGENERATE  1  /* "degenerate spectrum"                     */
#define FC_DIAG_NO_TEXTURE  2  /* "no texture; displacement undefined"      */

/* frame formats */
#define FC_FMT_RGB_F32   0  /* [B][H][W][3] float32, BT.601 luma in fp64     */
#define FC_FMT_GRAY_F32  1  /* [B][H][W]    float32                          */
#define FC_FMT_GRAY_F64  2  /* [B][H][W]    float64 (the reference's frames) */
#define FC_FMT_GRAY_U8   3  /* [B][H][W]    uint8, gray = v / 255 (PGM P5,
                               frameio.py:81-88)                           */
#define FC_FMT_RGB_U8    4  /* [B][H][W][3] uint8, gray = luma(v) / 255 in
                               fp64 (PPM P6, frameio.py:81-88)              */

/* fresh-row layouts for fc_splice */
#define FC_FRESH_DENSE    0  /* fresh row of token p is fresh[b][p]          */
#define FC_FRESH_COMPACT  1  /* k-th recomputed token (row-major) is fresh[b][k] */

typedef struct fc_geometry {
  int32_t batch;        /* independent streams B                            */
  int32_t height;       /* H                                                */
  int32_t width;        /* W                                                */
  int32_t patch_size;   /* P (CacheConfig.patch_size), divides H and W      */
  int32_t format;       /* FC_FMT_*                                         */
} fc_geometry;

/* CacheConfig + BudgetConfig (fusion.py:52-67, budget.py:12-24) */
typedef struct fc_config {
  double tau_mig;        /* 0.12 */
  double edge_lambda;    /* 0.25 */
  double alpha_min;      /* 0.08 */
  double alpha_max;      /* 0.5  */
  int32_t refresh_shift; /* <0: reference behaviour; k>=0: flush when
                            max(|di_p|,|dj_p|) > k (BASELINE config 2)      */
  int32_t reserved;
} fc_config;

/* One stream's CacheDecision scalars (fusion.py:70-94). */
typedef struct fc_stream_result {
  int32_t status;       /* FC_OK / FC_ENONFINITE / FC_EPSI                  */
  int32_t cold;         /* 1: no previous frame — everything recomputed    */
  int32_t flushed;
  int32_t diagnostic;   /* FC_DIAG_*                                        */
  int32_t k_reuse;
  int32_t k_candidate;
  int32_t k_final;
  int32_t n_refresh;
  int32_t di, dj, di_patches, dj_patches;
  int32_t rows, cols;
  int64_t bin_count;
  double sim_freq;
  double entropy_raw;
  double entropy_norm;
  double alpha;
  double energy_mean;
  double energy_std;
  double energy_threshold;
  double peak;           /* phase-correlation peak (ifft2 normalisation)   */
  double peak_runner_up; /* largest other response value                  */
} fc_stream_result;

/* Device output buffers of fc_select (caller-allocated, N = rows*cols). */
typedef struct fc_select_out {
  fc_stream_result* results; /* [B]                                          */
  int32_t* reuse_idx;        /* [B][N] ascending (E, idx), -1 padded          */
  int32_t* recompute_idx;    /* [B][N] row-major, -1 padded                   */
  int32_t* src_map;          /* [B][N] >=0: cache row; <0: -(rank+1) fresh   */
  uint8_t* reuse_mask;       /* [B][N]                                        */
  uint8_t* refresh_mask;     /* [B][N]                                        */
  double*  energy;           /* [B][N] high-pass DCT energy                   */
  int64_t* counters;         /* optional [4], accumulated (integer atomics):
                                frames, reused tokens (sum k_final), flushes
                                of warm streams, cold streams — the
                                run_sequence aggregates (fusion.py:559-572);
                                NULL to skip                                 */
} fc_select_out;

typedef struct fc_plan fc_plan;

int  fc_abi_version(void);
const char* fc_strerror(int code);

/* Plan: validates the geometry, uploads twiddles / DCT basis, sizes the
 * workspace.  Not thread-safe against concurrent destroy. */
int  fc_plan_create(const fc_geometry* geom, fc_plan** out);
void fc_plan_destroy(fc_plan* plan);
int64_t fc_plan_state_bytes(const fc_plan* plan);     /* per-stream state x B */
int64_t fc_plan_workspace_bytes(const fc_plan* plan); /* scratch; zero it once
                                                          at allocation (the
                                                          optional K_B + K_C
                                                          flow kernel keeps its
                                                          tickets there)       */
int  fc_plan_tokens(const fc_plan* plan);             /* N = rows*cols        */
int  fc_plan_launches(const fc_plan* plan);           /* kernels per fc_select */

/* Mark streams [first, first+count) cold. */
int  fc_state_reset(const fc_plan* plan, void* state, int32_t first,
                    int32_t count, void* cuda_stream);

/* One decision step for all B streams (frames: [B] frames in geometry's
 * format).  Cold streams only establish their spectrum (result.cold = 1).
 * state and workspace must be 16-byte aligned, and so must frames at
 * 448 x 448 / P 14 (bulk copies); FC_EINVAL otherwise. */
int  fc_select(const fc_plan* plan, const fc_config* cfg, const void* frames,
               void* state, void* workspace, const fc_select_out* out,
               void* cuda_stream);

/* Split-phase fc_select for software-pipelined streams of steps.  The
 * front of a step (luma + block-DCT energies + row FFTs, K_A, and the
 * energy statistics / refresh mask / token order, K_D1) depends on the
 * frames only; the back (column FFTs, cross-power, inverse, argmax and the
 * decision, K_B + K_C + K_D) on the front of the same step and on the back
 * of the previous step (the spectrum state).  The front -> back
 * intermediates live in workspace slot `slot` (0 / 1), so the front of step
 * t + 1 (slot (t + 1) & 1) may run concurrently with the back of step t
 * (slot t & 1) on different streams.  front(slot) then back(slot) on one
 * stream equals fc_select.  Use the same `out` for a step's front and back
 * (the front writes out->energy), and a different one for the next step.
 * FC_EUNSUPPORTED when the plan's stream chunks outnumber its lanes
 * (FC_CHUNK / FC_LANES overrides; the defaults always qualify).          */
int  fc_select_front(const fc_plan* plan, const fc_config* cfg, const void* frames,
                     void* workspace, const fc_select_out* out, int32_t slot,
                     void* cuda_stream);
int  fc_select_back(const fc_plan* plan, const fc_config* cfg, void* state,
                    void* workspace, const fc_select_out* out, int32_t slot,
                    void* cuda_stream);

/* fc_select with a CUDA event after every launch, all launches serial on
 * the caller's stream; synchronises and returns per-kernel-kind device time
 * in kernel_ms[5] (rows_fwd K_A, cols K_B, rows_inv K_C, select K_D, rank
 * K_D1), summed over stream chunks.  For benchmarking and the facade's
 * per-stage timings_us. */
int  fc_select_profile(const fc_plan* plan, const fc_config* cfg, const void* frames,
                       void* state, void* workspace, const fc_select_out* out,
                       float* kernel_ms, void* cuda_stream);

/* High-pass block-DCT energy of B frames (edge_refresh.py:48-59); energy is
 * [B][N] float64.  Uses the plan's workspace. */
int  fc_patch_energy(const fc_plan* plan, const void* frames, void* workspace,
                     double* energy, void* cuda_stream);

/* Splice: out[b][p] = src_map[b][p] >= 0 ? cache[b][src] : fresh[b][...];
 * out_ages likewise (cache_ages+1 / 0).  cache may be NULL when every entry
 * of src_map is negative.  row_bytes = D * element size (any, bit copy).
 * fresh_rows: rows per stream in `fresh` (ignored for FC_FRESH_DENSE, where
 * it is n_tokens; for FC_FRESH_COMPACT any capacity >= the recompute count).
 * status (device int32, may be NULL; the caller zeroes it): every splice
 * kernel checks each row's source as fusion.py:488-490 asserts it — a cache
 * source outside [0, n_tokens) (or any cache source with cache == NULL), or
 * a compact fresh index >= fresh_rows — skips that row and stores
 * FC_EBOUNDS in *status (the facade raises AssertionError).                 */
int  fc_splice(int32_t batch, int32_t n_tokens, int64_t row_bytes,
               const int32_t* src_map, const void* cache,
               const int64_t* cache_ages, const void* fresh,
               int32_t fresh_layout, int32_t fresh_rows, void* out,
               int64_t* out_ages, int32_t* status, void* cuda_stream);

/* Decision mask images (frameio.py:188-219): img[b][p] = 255 reused, 128
 * edge-forced recompute, 0 otherwise; flushed or cold streams all 0.        */
int  fc_render_masks(int32_t batch, int32_t n_tokens, const fc_stream_result* results,
                     const uint8_t* reuse_mask, const uint8_t* refresh_mask,
                     uint8_t* img, void* cuda_stream);

/* ---- stand-alone stage operators on arbitrary fp64 arrays (device pointers).
 * `ws` is a device scratch buffer of fc_stage_workspace_bytes(); results are
 * written to device memory; `flags` (device int32): bit0 non-finite input,
 * bit1 negative amplitude, bit2 candidate index out of range.  Deterministic. */
int64_t fc_stage_workspace_bytes(void);
/* sim_freq (migration.py:87-105): out3 = {sum a*b, sum a^2, sum b^2}        */
int  fc_amp_cosine(const double* a, const double* b, int64_t n, void* ws,
                   double* out3, int32_t* flags, void* cuda_stream);
/* spectral_entropy (budget.py:34-58): out2 = {sum P, sum p ln p}, P = a^2,
 * p = P / sum P, the DC bin (index 0) dropped when include_dc == 0          */
int  fc_spectral_sums(const double* amp, int64_t n, int32_t include_dc, void* ws,
                      double* out2, int32_t* flags, void* cuda_stream);
/* refresh_mask (edge_refresh.py:62-73): mask = e > mean + lam * std
 * (population), stats3 = {mean, std, threshold}                            */
int  fc_refresh_mask(const double* energy, int64_t n, double lam, void* ws,
                     uint8_t* mask, double* stats3, void* cuda_stream);
/* topk_ascending (fusion.py:104-115): first min(k, m) candidates ordered by
 * (energies[cand], cand) ascending; m <= 8192                               */
int  fc_topk_ascending(const int64_t* cand, int64_t m, const double* energies,
                       int64_t n_energies, int64_t k, int64_t* out,
                       int32_t* flags, void* cuda_stream);

/* fc_splice with ragged fresh rows: stream b's k-th recomputed token (row-
 * major) is row fresh_offsets[b] + k of `fresh` (device int64 [B]), e.g. the
 * packed values of a variable-length encoder batch. */
int  fc_splice_packed(int32_t batch, int32_t n_tokens, int64_t row_bytes,
                      const int32_t* src_map, const void* cache,
                      const int64_t* cache_ages, const void* fresh,
                      const int64_t* fresh_offsets, void* out, int64_t* out_ages,
                      int32_t* status, void* cuda_stream);

/* In-place splice over a per-stream ping-pong pair of caches.  slot_in[b]
 * (device u8) names the buffer (0/1) holding stream b's cache.  A stream whose
 * reused tokens all keep their slot (zero displacement) is updated in place:
 * reused rows are not touched (age + 1) and only recomputed rows are written.
 * Any other stream is spliced into its other buffer.  slot_out[b] receives the
 * buffer now holding the result.  Rows must be 16-byte multiples/aligned.   */
int64_t fc_splice_inplace_scratch_bytes(int32_t batch, int32_t n_tokens);
int  fc_splice_inplace(int32_t batch, int32_t n_tokens, int64_t row_bytes,
                       const int32_t* src_map, void* cache0, void* cache1,
                       int64_t* ages0, int64_t* ages1, const uint8_t* slot_in,
                       uint8_t* slot_out, const void* fresh, int32_t fresh_layout,
                       int32_t fresh_rows, void* scratch, int32_t* status,
                       void* cuda_stream);

/* fc_splice_inplace in two halves, for spreading one splice over two
 * streams: _plan (the per-stream in-place / ping-pong decision, the rows to
 * move and the copier's work counter) and _copy (copier CTAs that claim those
 * rows).  _copy with ctas = 0 is the default copier; a further _copy with
 * ctas > 0 on another stream, ordered after the plan (an event recorded right
 * after _plan), adds CTAs that take only the rows no copier has claimed yet
 * — e.g. launched behind the select kernels, it finishes the tail of a
 * splice that ran beside them.  All copies of one splice must complete before
 * the next splice's _plan.  fc_splice_inplace = _plan + _copy(0). */
int  fc_splice_inplace_plan(int32_t batch, int32_t n_tokens, int64_t row_bytes,
                            const int32_t* src_map, void* cache0, void* cache1,
                            int64_t* ages0, int64_t* ages1, const uint8_t* slot_in,
                            uint8_t* slot_out, const void* fresh, int32_t fresh_layout,
                            int32_t fresh_rows, void* scratch, void* cuda_stream);
int  fc_splice_inplace_copy(int32_t batch, int32_t n_tokens, int64_t row_bytes,
                            const int32_t* src_map, void* cache0, void* cache1,
                            int64_t* ages0, int64_t* ages1, const uint8_t* slot_in,
                            const uint8_t* slot_out, const void* fresh, int32_t fresh_layout,
                            int32_t fresh_rows, void* scratch, int32_t* status,
                            int32_t ctas, void* cuda_stream);

/* Build src_map for one stream from an ordered reuse list (fusion.py:481-504).
 * flag (device int32, may be NULL) receives FC_EBOUNDS on an out-of-bounds
 * source. */
int  fc_splice_map(int32_t rows, int32_t cols, const int32_t* reuse_idx,
                   int32_t k, int32_t di_patches, int32_t dj_patches,
                   int32_t* src_map, int32_t* flag, void* cuda_stream);

/* ---- comparison baselines (compare.py:23-52, the paper's two position-wise
 * policies).  For B frame pairs (prev[b], curr[b]) in geom's format, per patch
 * (row-major, [B][N] float64): visual_cos = cosine of the raw gray pixels,
 * naive_cos = cosine of the |fft2| amplitude spectra of the P x P patches;
 * a pair with a zero norm scores 0.  2 <= patch_size <= 32.  Replaces
 * compare.py:41-52 + 90-95 (_token_stack with the raw-pixel token_fn,
 * _patch_amplitudes, _position_cosines).                                    */
int  fc_compare_cosines(const fc_geometry* geom, const void* prev, const void* curr,
                        double* visual_cos, double* naive_cos, void* cuda_stream);
/* Row-wise cosine of two [n][d] float64 stacks (compare.py:28-38), e.g. a
 * custom token_fn's vectors.                                                */
int  fc_row_cosines(int64_t n, int64_t d, const double* a, const double* b,
                    double* out, void* cuda_stream);

/* ---- encoder-side token gather (BASELINE config 4).  Row r of out (bf16,
 * [rows][3 P^2], (py, px, channel) order) = the P x P patch of token
 * index[r] = b * N + p of the fp32 RGB frames [batch][H][W][3]: the pixels
 * of the recomputed tokens only, as a ViT patch embedding consumes them.   */
int  fc_gather_patches(int32_t rows, int32_t batch, int32_t height, int32_t width,
                       int32_t patch_size, const float* frames, const int64_t* index,
                       void* out_bf16, void* cuda_stream);

/* ---- fp64 transform wrappers (spectral.py:24-72, migration.py:128-134):
 * the reference's public transform API, on the GPU in fp64 (dense passes
 * with exact twiddles; not the decision path's packed fp32 FFTs).  Complex
 * grids are interleaved (re, im) float64, row-major [h][w].                 */
int64_t fc_dft2_workspace_bytes(int32_t h, int32_t w);
/* out = fft2(in) (inverse == 0, unnormalised) or ifft2(in) (scaled 1/(h w));
 * in is real [h][w] (in_complex == 0) or complex.  dft2 / idft2.            */
int  fc_dft2(int32_t h, int32_t w, const double* in, int32_t in_complex,
             int32_t inverse, double* out, void* workspace, void* cuda_stream);
int64_t fc_phase_correlation_workspace_bytes(int32_t h, int32_t w);
/* phase_correlation_spectra: normalised cross-power, ifft2, argmax with the
 * reference tie rule -> disp2 = (di, dj) pixels (device int32[2])          */
int  fc_phase_correlation_spectra(int32_t h, int32_t w, const double* spec_prev,
                                  const double* spec_curr, int32_t* disp2,
                                  void* workspace, void* cuda_stream);
/* block_dct: orthonormal 2-D DCT-II of n square p x p patches (p <= 64)     */
int  fc_block_dct(int32_t n_patches, int32_t p, const double* patches,
                  double* out, void* cuda_stream);
/* amplitude_phase: |z| and atan2(Im z, Re z) of n complex values            */
int  fc_amplitude_phase(int64_t n, const double* spectrum, double* amp,
                        double* phase, void* cuda_stream);

/* ---- CUDA-graph capture of whole steps (runtime plumbing, not an op of the
 * reference).  Capture everything a step launches on `cuda_stream` (other
 * streams join through events), instantiate it with per-node priorities and
 * replay it with one launch per step.                                       */
int  fc_graph_capture_begin(void* cuda_stream);
int  fc_graph_capture_end(void* cuda_stream, void** graph_exec);
int  fc_graph_launch(void* graph_exec, void* cuda_stream);
void fc_graph_destroy(void* graph_exec);

#ifdef __cplusplus
}
#endif
#endif /* FREQCACHE_B200_H */
