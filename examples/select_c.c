/* The C ABI driven from plain C99 — no Python, no torch: what a binding in
 * another language does through its FFI.  Two streams of 448 x 448 RGB fp32
 * frames; the second frame of stream s is the first one circularly shifted
 * by (s + 1) * 14 pixels down, so phase correlation must report
 * di_patches = s + 1, and every reused token (i, j) must take its cached row
 * from (i - di_patches, j) (migration.py:162-176).  Exit status 0 when it
 * does.
 *
 *   make -C examples            (links libfreqcache_b200.so and cudart)
 *   examples/select_c
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "freqcache_b200.h"

#define CK(x)                                                                    \
  do {                                                                           \
    int rc_ = (x);                                                               \
    if (rc_ != 0) {                                                              \
      fprintf(stderr, "%s failed: %d (%s)\n", #x, rc_, fc_strerror(rc_));        \
      return 1;                                                                  \
    }                                                                            \
  } while (0)
#define CU(x)                                                                    \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                     \
      fprintf(stderr, "%s failed: %s\n", #x, cudaGetErrorString(e_));            \
      return 1;                                                                  \
    }                                                                            \
  } while (0)

enum { B = 2, H = 448, W = 448, P = 14 };

static float texture(int y, int x, int c) {
  /* smooth random-looking texture (periodic, so circular shifts are exact) */
  const double t = 2.0 * 3.14159265358979323846 / 448.0;
  return (float)(0.5 + 0.15 * sin(t * (3 * y + 5 * x + 7 * c)) + 0.1 * cos(t * (11 * y - 2 * x)) +
                 0.05 * sin(t * (23 * x + 17 * y * (c + 1))));
}

int main(void) {
  if (fc_abi_version() != FC_ABI_VERSION) {
    fprintf(stderr, "ABI version mismatch\n");
    return 1;
  }
  const fc_geometry g = {B, H, W, P, FC_FMT_RGB_F32};
  fc_plan* plan = NULL;
  CK(fc_plan_create(&g, &plan));
  const int N = fc_plan_tokens(plan);
  const size_t frame_elems = (size_t)B * H * W * 3;
  float* host[2];
  for (int f = 0; f < 2; ++f) host[f] = (float*)malloc(frame_elems * sizeof(float));
  for (int s = 0; s < B; ++s)
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x)
        for (int c = 0; c < 3; ++c) {
          const size_t i = (((size_t)s * H + y) * W + x) * 3 + c;
          host[0][i] = texture(y, x, c);
          host[1][i] = texture((y + H - (s + 1) * P) % H, x, c);  /* content moves down */
        }
  void *frames, *state, *ws;
  CU(cudaMalloc(&frames, frame_elems * sizeof(float)));
  CU(cudaMalloc(&state, (size_t)fc_plan_state_bytes(plan)));
  CU(cudaMalloc(&ws, (size_t)fc_plan_workspace_bytes(plan)));
  CU(cudaMemset(ws, 0, (size_t)fc_plan_workspace_bytes(plan)));
  fc_select_out out;
  memset(&out, 0, sizeof(out));
  CU(cudaMalloc((void**)&out.results, B * sizeof(fc_stream_result)));
  CU(cudaMalloc((void**)&out.reuse_idx, (size_t)B * N * 4));
  CU(cudaMalloc((void**)&out.recompute_idx, (size_t)B * N * 4));
  CU(cudaMalloc((void**)&out.src_map, (size_t)B * N * 4));
  CU(cudaMalloc((void**)&out.reuse_mask, (size_t)B * N));
  CU(cudaMalloc((void**)&out.refresh_mask, (size_t)B * N));
  CU(cudaMalloc((void**)&out.energy, (size_t)B * N * 8));
  const fc_config cfg = {0.12, 0.25, 0.08, 0.5, -1, 0};   /* the reference's defaults */
  CK(fc_state_reset(plan, state, 0, B, NULL));
  for (int f = 0; f < 2; ++f) {
    CU(cudaMemcpy(frames, host[f], frame_elems * sizeof(float), cudaMemcpyHostToDevice));
    CK(fc_select(plan, &cfg, frames, state, ws, &out, NULL));
  }
  CU(cudaDeviceSynchronize());
  fc_stream_result res[B];
  int32_t* src = (int32_t*)malloc((size_t)B * N * 4);
  CU(cudaMemcpy(res, out.results, sizeof(res), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(src, out.src_map, (size_t)B * N * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  const int cols = W / P;
  for (int s = 0; s < B; ++s) {
    const fc_stream_result* r = &res[s];
    printf("stream %d: status %d cold %d flushed %d di_patches %d dj_patches %d sim %.6f k_final %d\n", s,
           r->status, r->cold, r->flushed, r->di_patches, r->dj_patches, r->sim_freq, r->k_final);
    if (r->status != FC_OK || r->cold || r->di_patches != s + 1 || r->dj_patches != 0 || r->k_final < 1) bad = 1;
    for (int p = 0; p < N; ++p) {
      const int v = src[(size_t)s * N + p];
      if (v >= 0 && v != p - r->di_patches * cols) bad = 1;   /* reused rows come from the shifted slot */
    }
  }
  printf(bad ? "FAIL\n" : "OK\n");
  fc_plan_destroy(plan);
  return bad;
}
