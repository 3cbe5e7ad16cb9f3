/* A plain C caller of the multi-GPU entry points (include/fuseplan.h):
 * the SPEC chain over a counter-hash video, T-sharded over the devices named
 * on the command line (they may repeat), against a single-device run of the
 * same plan.  Prints "ok <fixups> <fixed_frames>" and exits 0 when the
 * outputs are identical.   cc shard_capi.c -I include -L ... -lfuseplan_b200 */
#include <fuseplan.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static int fail(const char* what) {
  fprintf(stderr, "%s: %s\n", what, fp_last_error());
  return 1;
}

int main(int argc, char** argv) {
  if (argc < 5) {
    fprintf(stderr, "usage: %s W H F warmup dev [dev ...]\n", argv[0]);
    return 2;
  }
  const int W = atoi(argv[1]), H = atoi(argv[2]), F = atoi(argv[3]), warm = atoi(argv[4]);
  const int n = argc - 5;
  int devs[16];
  for (int i = 0; i < n && i < 16; ++i) devs[i] = atoi(argv[5 + i]);
  char pj[1024];
  snprintf(pj, sizeof pj,
           "{\"video\": {\"width\": %d, \"height\": %d, \"frames\": %d, \"channels\": 4},"
           " \"kernels\": [{\"name\": \"g\", \"stencil_op\": \"rgba2gray\"},"
           " {\"name\": \"i\", \"stencil_op\": \"iir_temporal\", \"params\": {\"alpha\": 0.5}},"
           " {\"name\": \"s\", \"stencil_op\": \"gaussian\", \"params\": {\"radius\": 2, \"sigma\": 1.0}},"
           " {\"name\": \"d\", \"stencil_op\": \"gradient\"},"
           " {\"name\": \"t\", \"stencil_op\": \"threshold\", \"params\": {\"th\": 40}}]}",
           W, H, F);
  fp_pipeline* p = NULL;
  fp_device* d = NULL;
  fp_plan* plan = NULL;
  if (fp_pipeline_parse(pj, &p) != FP_OK) return fail("pipeline");
  if (fp_device_load("b200", &d) != FP_OK) return fail("device");
  if (fp_plan_create(p, d, NULL, &plan) != FP_OK) return fail("plan");
  const size_t px = (size_t)W * H * F;
  uint8_t* video = malloc(px * 4);
  uint8_t* a = malloc(px);
  uint8_t* b = malloc(px);
  uint64_t z0 = 0x9E3779B97F4A7C15ull * 77u;
  for (size_t i = 0; i < px * 4; ++i) {  /* splitmix64 counter hash, top byte */
    uint64_t z = i + z0;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    video[i] = (uint8_t)((z ^ (z >> 31)) >> 56);
  }
  fp_exec* one = NULL;
  if (fp_exec_create(p, plan, devs[0], NULL, &one) != FP_OK) return fail("exec");
  if (fp_exec_run(one, video, FP_ELEM_U8, a, FP_EXEC_HOST_PTRS, NULL) != FP_OK)
    return fail("single run");
  char opts[64];
  snprintf(opts, sizeof opts, "{\"warmup_frames\": %d}", warm);
  fp_shard_exec* sh = NULL;
  if (fp_shard_exec_create(p, plan, devs, n, opts, &sh) != FP_OK) return fail("shard exec");
  if (fp_shard_exec_run(sh, video, FP_ELEM_U8, b) != FP_OK) return fail("shard run");
  char* stats = NULL;
  if (fp_shard_exec_stats(sh, &stats) != FP_OK) return fail("stats");
  const int same = memcmp(a, b, px) == 0;
  printf("%s %s\n", same ? "ok" : "MISMATCH", stats);
  fp_string_free(stats);
  fp_shard_exec_free(sh);
  fp_exec_free(one);
  fp_plan_free(plan);
  fp_device_free(d);
  fp_pipeline_free(p);
  free(video);
  free(a);
  free(b);
  return same ? 0 : 1;
}
