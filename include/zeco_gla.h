/*
 * zeco_gla.h -- C ABI of the B200-native ZeCO sequence-parallel GLA library
 * (libzeco_gla.so).  Plain pointers and sizes only; every compute entry point
 * is stream-ordered on a CUDA stream passed as `void*` (0 = legacy default)
 * and takes DEVICE pointers owned by the caller.  Return value: ZGLA_OK (0)
 * or a negative ZGLA_ERR_* code; the Python drop-in maps the codes onto the
 * reference exception types (glasp/errors.py:4-33).
 *
 * The reference (`glasp`, pure Python/NumPy) has no FFI; each entry point
 * below names the reference function it replaces.  INTEGRATION.md shows the
 * ctypes binding the reference would add.
 *
 * Layouts (reference glasp/gla.py:29-30): q,k,g [h][L][dk], v,o [h][L][dv],
 * contiguous.  States are [h][dk][dv]; lists of N+1 boundary states are
 * stacked as [N+1][h][dk][dv]; cumulative log decays as [N+1][h][dk].
 *
 * Precision modes (zgla_dtype):
 *   ZGLA_BF16: q,k,v,dO,o,dq,dk,dv are bf16; g, dg, states are fp32.  ZeCO
 *              entry points use the tcgen05/TMEM/TMA kernels when
 *              dk == dv in {64, 128} and L % 64 == 0 (d = 64 runs the 128-channel
 *              kernels on TMA zero-filled channels).
 *   ZGLA_F32 : everything fp32 ("fp32 validation mode", SIMT FMA kernels).
 *   ZGLA_F64 : everything fp64 (bit-for-bit reference semantics for tests).
 */
#ifndef ZECO_GLA_H
#define ZECO_GLA_H

#ifdef __cplusplus
extern "C" {
#endif

#define ZGLA_OK 0
#define ZGLA_ERR_DIMS (-1)        /* -> DimsError   */
#define ZGLA_ERR_DOMAIN (-2)      /* -> DomainError */
#define ZGLA_ERR_LAYOUT (-3)      /* -> LayoutError */
#define ZGLA_ERR_CONFIG (-4)      /* -> ConfigError */
#define ZGLA_ERR_STATE (-5)       /* -> StateError  */
#define ZGLA_ERR_DEADLOCK (-6)    /* -> DeadlockError (All-Scan flag wait timed out) */
#define ZGLA_ERR_UNSUPPORTED (-7) /* shape not supported by this build */
#define ZGLA_ERR_CUDA (-100)      /* CUDA runtime error; see zgla_last_error() */

enum { ZGLA_BF16 = 0, ZGLA_F32 = 1, ZGLA_F64 = 2 };
enum { ZGLA_FWD = 0, ZGLA_BWD = 1 };

typedef struct {
  int heads;
  int key_dim;
  int value_dim;
  int chunk_len;
  long long seq_len; /* tokens in this shard */
  int dtype;         /* ZGLA_BF16 / ZGLA_F32 / ZGLA_F64 */
} zgla_shape;

/* A [heads][tokens][channels] tensor with arbitrary token and head strides (in ELEMENTS; channels
 * contiguous).  0 means dense (channels, resp. tokens * channels).  Lets the ZeCO entry points read
 * and write views such as the head slices of a token-major [tokens][heads * channels] projection
 * output without a transposing copy (fused tcgen05 path; the SIMT paths need dense tensors). */
typedef struct {
  void* data;
  long long token_stride;
  long long head_stride;
} zgla_tensor;

/* ---- library ----------------------------------------------------------- */
const char* zgla_version(void);
const char* zgla_last_error(void);
/* 1 if the fused tcgen05 ZeCO kernels serve this shape, else 0 */
int zgla_fast_path(const zgla_shape* s);

/* ---- reference function-level API (glasp/gla.py) ------------------------ */
/* bytes of device workspace the function-level entry points below need */
long long zgla_workspace_bytes(const zgla_shape* s);

/* glasp/gla.py:248 local_state_scan (+ optional initial state, glasp/gla.py:210 init) */
int zgla_local_state_scan(const zgla_shape* s, const void* k, const void* v, const void* g, const void* init,
                          void* states_out, void* cum_out, void* ws, void* stream);
/* glasp/gla.py:297 forward_outputs; prev may be NULL (zero state) */
int zgla_forward_outputs(const zgla_shape* s, const void* q, const void* k, const void* v, const void* g,
                         const void* states, const void* cum, const void* prev, void* o, void* stream);
/* glasp/gla.py:272 global_correct over n_states boundary states */
int zgla_global_correct(const zgla_shape* s, int n_states, const void* states, const void* cum, const void* prev,
                        void* out, void* stream);
/* glasp/gla.py:336 reverse_boundary_scan; seed may be NULL (zero) */
int zgla_reverse_boundary_scan(const zgla_shape* s, const void* q, const void* g, const void* d_out,
                               const void* seed, void* rev_out, void* ws, void* stream);
/* glasp/gla.py:359 backward; saved_states may be NULL (recompute from prev) */
int zgla_backward(const zgla_shape* s, const void* q, const void* k, const void* v, const void* g,
                  const void* d_out, const void* prev, const void* ds_next, const void* saved_states, void* dq,
                  void* dk, void* dv, void* dg, void* ds_boundary, void* ws, void* stream);
/* glasp/gla.py:331 revcum along tokens of an [h][L][d] tensor (acc dtype of s) */
int zgla_revcum(const zgla_shape* s, int d, const void* x, void* out, void* stream);
/* glasp/gla.py:233 chunk_scalings of one chunk g [h][C][dk] */
int zgla_chunk_scalings(const zgla_shape* s, const void* g_chunk, void* chunk_decay, void* from_start,
                        void* to_end, void* stream);
/* glasp/gla.py:210-230 recurrent_forward: the token-by-token recurrence (independent of every chunkwise
 * kernel).  init may be NULL (zero state); bounds [N+1][h][dk][dv] and final [h][dk][dv] may be NULL. */
int zgla_recurrent_forward(const zgla_shape* s, const void* q, const void* k, const void* v, const void* g,
                           const void* init, void* o, void* bounds, void* final_state, void* stream);
/* glasp/gla.py:447-480 finite_diff_grad, float64 only: losses[i] = sum(probe * recurrent_forward(x_i)) for
 * perturbations i = first .. first+count-1 of tensor `which` (0 q, 1 k, 2 v, 3 g); perturbation i bumps flat
 * element i/2 by +step (i even) or -step (i odd).  ZGLA_ERR_UNSUPPORTED if h*dk*dv > zgla_fd_max_state(). */
long long zgla_fd_max_state(void);
int zgla_fd_losses(const zgla_shape* s, const double* q, const double* k, const double* v, const double* g,
                   const double* probe, int which, long long first, long long count, double step, double* losses,
                   void* stream);
/* elementwise domain checks used by SeqShard/State validation; *bad set to 1 if violated */
int zgla_check_log_decay(long long n, int dtype, const void* g, int* bad_dev, void* stream);

/* ---- ZeCO per-rank hot path (glasp/engine.py:218-237, 348-364) --------- */
/* Early inputs (process-wide, off by default; returns the previous setting): the fused output kernels
 * stream q / k / v / g / dO into shared memory before waiting for the kernel launched before them (the
 * segment scan or the All-Scan chain), overlapping their prologue with it.  Caller contract: those
 * tensors are complete before the matching zgla_zeco_*_local call is enqueued. */
int zgla_set_early_inputs(int on);
/* plan-dependent workspace for the four ZeCO entry points */
long long zgla_zeco_workspace_bytes(const zgla_shape* s, int num_sms);
/* local chunk scan: rank-local final state S_local [h][dk][dv] and total log decay G_tot [h][dk]
 * (glasp/engine.py:219-224 -> inputs of All-Scan FWD) */
int zgla_zeco_fwd_local(const zgla_shape* s, int num_sms, const void* k, const void* v, const void* g, void* ws,
                        void* s_local, void* g_tot, void* stream);
/* outputs with the fused correction O += (Q e^{G_t}) S_prev; s_prev may be NULL (rank 0) */
int zgla_zeco_fwd_output(const zgla_shape* s, int num_sms, const void* q, const void* k, const void* v,
                         const void* g, void* ws, const void* s_prev, void* o, void* stream);
/* local reverse scan: dS_local0 [h][dk][dv] (input of All-Scan BWD, glasp/engine.py:349-355) */
int zgla_zeco_bwd_local(const zgla_shape* s, int num_sms, const void* q, const void* g, const void* d_out,
                        void* ws, void* ds_local0, void* stream);
/* gradients with the fused corrections from s_prev / ds_next (either may be NULL) */
int zgla_zeco_bwd_output(const zgla_shape* s, int num_sms, const void* q, const void* k, const void* v,
                         const void* g, const void* d_out, void* ws, const void* s_prev, const void* ds_next,
                         void* dq, void* dk, void* dv, void* dg, void* stream);

/* after zgla_zeco_fwd_local: ZGLA_ERR_DOMAIN if a 64-token tile's summed log-decay was below -160 (or
 * not finite) on the fused bf16 path, whose in-tile exponents e^{+-(logb - r)} would overflow there;
 * synchronises `stream` (a validation call, not for the timed path).  ZGLA_OK on the SIMT paths. */
int zgla_zeco_domain_check(const zgla_shape* s, int num_sms, const void* ws, void* stream);

/* lazy (non-synchronising) domain report for the timed path: registers a host-mapped int for the
 * workspace `ws`; every later fused zgla_zeco_fwd_local on that workspace stores 1 into it when a
 * tile left the exponent domain (no store otherwise).  The caller reads / resets *host_flag whenever
 * it likes (e.g. at the next step) and raises DomainError.  unwatch frees the word. */
int zgla_zeco_watch_domain(void* ws, int** host_flag);
int zgla_zeco_unwatch_domain(void* ws);
/* the same four entry points over strided tensors (zgla_tensor); ZGLA_ERR_LAYOUT if a stride or base is
 * not 16-byte aligned, or if the shape runs the SIMT path and a tensor is not dense */
int zgla_zeco_fwd_local_v(const zgla_shape* s, int num_sms, const zgla_tensor* k, const zgla_tensor* v,
                          const zgla_tensor* g, void* ws, void* s_local, void* g_tot, void* stream);
int zgla_zeco_fwd_output_v(const zgla_shape* s, int num_sms, const zgla_tensor* q, const zgla_tensor* k,
                           const zgla_tensor* v, const zgla_tensor* g, void* ws, const void* s_prev,
                           const zgla_tensor* o, void* stream);
/* zgla_zeco_fwd_output_v with flags: ZGLA_FWD_NO_SAVE skips the chunk-start states the backward reads
   (forward-only / inference calls: ~25 % less HBM traffic in the output kernel); a backward after such a
   forward is invalid (the Python layer raises StateError) */
#define ZGLA_FWD_NO_SAVE 1
int zgla_zeco_fwd_output_ex_v(const zgla_shape* s, int num_sms, const zgla_tensor* q, const zgla_tensor* k,
                              const zgla_tensor* v, const zgla_tensor* g, void* ws, const void* s_prev,
                              const zgla_tensor* o, int flags, void* stream);
int zgla_zeco_bwd_local_v(const zgla_shape* s, int num_sms, const zgla_tensor* q, const zgla_tensor* g,
                          const zgla_tensor* d_out, void* ws, void* ds_local0, void* stream);
int zgla_zeco_bwd_output_v(const zgla_shape* s, int num_sms, const zgla_tensor* q, const zgla_tensor* k,
                           const zgla_tensor* v, const zgla_tensor* g, const zgla_tensor* d_out, void* ws,
                           const void* s_prev, const void* ds_next, const zgla_tensor* dq, const zgla_tensor* dk,
                           const zgla_tensor* dv, const zgla_tensor* dg, void* stream);

/* ---- All-Scan (glasp/collectives.py:70-140) ----------------------------- */
/* All P "ranks" resident on one device (the reference's list form): one kernel runs the
 * whole pipelined chain through device-memory flags.  fp32 or fp64 (dtype). */
int zgla_allscan_local(int P, int heads, int key_dim, int value_dim, int dtype, int num_blocks, int direction,
                       const void* local_states, const void* log_decays, void* recv, void* scanned,
                       void* stream);
/* Frees the device scratch zgla_allscan_local keeps between calls (the Python layer calls it at
 * interpreter exit; the next zgla_allscan_local allocates again). */
int zgla_release_cached(void);

/* SPMD form over peer memory (one process per GPU).  The caller exchanges the
 * buffers returned by zgla_allscan_export() (CUDA IPC handles) and passes the
 * successor/predecessor mappings to zgla_allscan_bind(). */
typedef struct zgla_allscan_comm zgla_allscan_comm;
int zgla_allscan_create(int rank, int world, int heads, int key_dim, int value_dim, int max_blocks,
                        zgla_allscan_comm** out);
int zgla_allscan_export(zgla_allscan_comm* c, void* ipc_handle_out /* 64 bytes */);
int zgla_allscan_bind(zgla_allscan_comm* c, const void* next_handle, const void* prev_handle);
/* bind to buffers in this process (world of virtual ranks inside one process) */
int zgla_allscan_bind_local(zgla_allscan_comm* c, zgla_allscan_comm* next, zgla_allscan_comm* prev);
int zgla_allscan_run(zgla_allscan_comm* c, int num_blocks, int direction, const float* local_state,
                     const float* log_decay, float* recv, float* scanned, void* stream);
int zgla_allscan_destroy(zgla_allscan_comm* c);
/* ZGLA_ERR_DEADLOCK if an earlier zgla_allscan_run on this communicator timed out waiting for a
 * peer (the kernel records it in host-mapped memory and exits instead of trapping); sync != 0 first
 * synchronises the device so the last call is included.  A timed-out communicator stays unusable. */
int zgla_allscan_status(zgla_allscan_comm* c, int sync);
long long zgla_allscan_bytes_sent(const zgla_allscan_comm* c);
/* rank, world size and head count the communicator was created with (any pointer may be NULL) */
int zgla_allscan_info(const zgla_allscan_comm* c, int* rank, int* world, int* heads);

/* ---- host-buffer layer call (the reference's verify/bench flow, glasp/cli.py:241-361) ----
 * One ZeCO GLA layer forward + backward with q,k,v,g,dO and o,dq,dk,dv,dg in HOST memory
 * (pinned for full PCIe speed; layouts and dtypes as above).  Heads are cut into head_groups
 * groups pipelined over three streams (H2D / kernels / D2H), so transfers in both directions
 * overlap each other and the kernels.  comm may be NULL (one rank); otherwise it must have been
 * created for heads / head_groups heads and every rank runs the groups in the same order.
 * dev_buf: device scratch of zgla_zeco_fwd_bwd_host_bytes() bytes.
 * flags = 0: stream-ordered; the host outputs are complete when `stream` has drained.
 * flags = ZGLA_HOST_OVERLAP: repeated calls with the same geometry and dev_buf chain through
 *   per-group events, so a call's H2D runs under the previous call's D2H; host inputs are read
 *   asynchronously (do not modify them until the call completes) and completion is awaited with
 *   zgla_zeco_host_wait(stream), which makes `stream` wait for the last call's D2H. */
#define ZGLA_HOST_OVERLAP 1
long long zgla_zeco_fwd_bwd_host_bytes(const zgla_shape* s, int num_sms, int head_groups);
int zgla_zeco_fwd_bwd_host(const zgla_shape* s, int num_sms, int head_groups, zgla_allscan_comm* comm,
                           int num_blocks, const void* q, const void* k, const void* v, const void* g,
                           const void* d_out, void* o, void* dq, void* dk, void* dv, void* dg, void* dev_buf,
                           long long dev_buf_bytes, int flags, void* stream);
int zgla_zeco_host_wait(void* stream);

/* ---- diagnostics -------------------------------------------------------- */
/* record per-tile pipeline timestamps (%globaltimer) of CTA `cta` of the fused kernels into
 * dev_buf (u64 [32][512]); pass NULL to disable */
int zgla_set_trace(void* dev_buf, int cta);
/* TMA streaming-rate probe: ctas x tiles_per_cta tiles of `tensors` x 16 KiB through ns stages */
int zgla_selftest_tmem(int nwarps, int iters, int mode, long long* out, float* sink, void* stream);
int zgla_selftest_stream(const void* src, long long rows, int tiles_per_cta, int ns, int tensors, int prefetch,
                         int ctas, void* stream);
int zgla_selftest_mma(const void* a, const void* b, float* d, int M, int N, int K, int a_mn, int b_mn,
                      int lane_off, void* stream);
/* diagnostics: one CTA spinning for ns nanoseconds on the stream (injected-latency probes) */
int zgla_selftest_spin(long long ns, void* stream);
/* diagnostic: tcgen05 SS MMA issue rate, M x N x 16 bf16; out[cta] = SM milli-cycles per MMA */
int zgla_selftest_mma_rate(int M, int N, int a_mn, int b_mn, int iters, int ctas, long long* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ZECO_GLA_H */
