/*
 * janus_dev.h — kernel-level test hooks of libjanus (not part of the step ABI in janus.h).
 * The GPU unit tests use them to check single kernels against the oracle's numerics.
 * All pointers are device pointers; calls are asynchronous on `stream`; return 0 or a
 * cudaError_t code.
 */
#ifndef JANUS_DEV_H
#define JANUS_DEV_H
#include <stddef.h>
#include <stdint.h>

#include "janus.h"
#ifdef __cplusplus
extern "C" {
#endif

/* C[M,N] (fp32, row pitch ldc) (+)= A . B^T (+ bias_col[n]) (+ bias_row[m]), bf16 operands.
 * a_mn = 0: A is [M][lda] (K contiguous); 1: A is [K][lda] (M contiguous). Same for B with N. */
int32_t janus_dev_gemm_bf16(int32_t M, int32_t N, int32_t K, const void *A, int32_t lda,
                            int32_t a_mn, const void *B, int32_t ldb, int32_t b_mn, float *C,
                            int32_t ldc, const float *bias_col, const float *bias_row,
                            int32_t accumulate, void *stream);
/* Same, with the K dimension split `splits` ways (0 = the library's automatic choice, as in the
 * step path; 1 = no split). Split partial sums are added in split order (deterministic). Uses a
 * library-owned device flag buffer: calls must not run concurrently on different streams. */
int32_t janus_dev_gemm_bf16_splitk(int32_t M, int32_t N, int32_t K, const void *A, int32_t lda,
                                   int32_t a_mn, const void *B, int32_t ldb, int32_t b_mn, float *C,
                                   int32_t ldc, const float *bias_col, const float *bias_row,
                                   int32_t accumulate, int32_t splits, void *stream);

/* Per-phase device timing of janus_run (CUDA events on the launch stream, collected after the
 * step's synchronisation). enable != 0 switches it on and clears the totals. The report is
 * "name:total_ms:count;..." over the phases run since enabling. */
struct janus_graph;
int32_t janus_dev_profile(struct janus_graph *g, int32_t enable);
/* Timeline probe of the layer-0 recurrent kernels (every CTA): dev_buf (device, 2*128*16*T u64)
 * receives %globaltimer stamps, 16 per step: forward CTA c step t at ((c*T)+t)*16, backward at
 * 128*16*T + the same index. NULL disables. */
int32_t janus_dev_set_probe(struct janus_graph *g, void *dev_buf);
/* Byte offset and size of a named region of the workspace after janus_run: "status",
 * "tree.height", "tree.order", "tree.irank", "tree.pslot", "tree.lvl_off", "tree.meta"
 * (int32 arrays of the device-built level schedule). Returns 0, or -1 if unknown. */
int32_t janus_dev_workspace_region(const struct janus_graph *g, const char *name, size_t *offset,
                                   size_t *bytes);
int32_t janus_dev_phase_report(const struct janus_graph *g, char *buf, size_t len);

/* ---- Data-parallel protocol test hooks (host memory only: they run without a GPU). ----
 * P:298 §5 (gradient averaging by collectives inside the step) and reading Q12 / R7 (one
 * failing rank aborts every rank; the minimum (id, rank) failure is reported everywhere).
 * janus_allreduce_fn: in-place allreduce of `count` elements of `buf` (host memory) over the
 * caller's process group; dtype JANUS_F32 or JANUS_I64; op 0 = sum, 1 = min, 2 = max; returns 0
 * on success. Every rank must call the hooks below in the same order (they are collective). */
typedef int32_t (*janus_allreduce_fn)(void *ctx, void *buf, int64_t count, int32_t dtype, int32_t op);
/* Route this graph's protocol-test collectives through fn (graph built with world_size > 1 or
 * JANUS_FORCE_DP=1; -1 otherwise). The device path keeps using NCCL. */
int32_t janus_dev_dp_set_host_collective(struct janus_graph *g, janus_allreduce_fn fn, void *ctx);
/* The step's gradient-arena allreduces in issue order, as janus_run and its null step issue them:
 * out[3*i .. 3*i+2] = {communicator (1 main, 2 split/overlapped), byte offset in the workspace,
 * bytes}. Returns the number of segments (writes at most cap), or -1. */
int32_t janus_dev_dp_segments(const struct janus_graph *g, int64_t *out, int32_t cap);
/* One step's collective protocol on a HOST copy of the workspace (ws_host, janus_workspace_bytes
 * bytes): the arena allreduces (sum) of janus_dev_dp_segments in order, then the abort agreement
 * with this rank's local outcome (local = the failure this rank observed, NULL = none;
 * runtime_err != 0 = a runtime error on this rank). *status = the agreed janus_status, *out = the
 * agreed failure (ASSUMPTION_FAILED only). Returns 0, -1 (bad arguments / no transport) or -2
 * (the transport failed). */
int32_t janus_dev_dp_host_step(struct janus_graph *g, void *ws_host, const janus_failure *local,
                               int32_t runtime_err, janus_failure *out, int32_t *status);

#ifdef __cplusplus
}
#endif
#endif
