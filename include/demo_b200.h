/*
 * demo_b200.h -- C-ABI of the B200-native FlexDeMo / DeToNATION optimizer step.
 *
 * This is the drop-in boundary for the reference's hot path (demosim core,
 * /root/reference/proj/core).  Each entry point replaces one reference function
 * (cited file:line) with the same argument meaning and error behaviour, but on
 * DEVICE buffers in FP32 (the reference is FP64 host vectors):
 *
 *   reference (C++, namespace demosim)                 C-ABI here
 *   -------------------------------------------------  ---------------------------------
 *   wire_bytes            replicate.hpp:26  .cpp:44     dmb_wire_bytes
 *   ReplicatorConfig::period  replicate.hpp:38 .cpp:50  dmb_period
 *   selected_indices      replicate.hpp:77  .cpp:160    dmb_selected_indices
 *   select_and_encode     replicate.hpp:71  .cpp:187    dmb_select_and_encode
 *   decode_and_merge      replicate.hpp:83  .cpp:239    dmb_decode_and_merge
 *   serialize/deserialize replicate.hpp:88-93 .cpp:316  dmb_serialize / dmb_deserialize
 *   demo_sgd_prepare      optim.hpp:42      .cpp:18     dmb_demo_sgd_prepare
 *   demo_sgd_apply        optim.hpp:48      .cpp:45     dmb_demo_sgd_apply
 *   adamw_prepare         optim.hpp:52      .cpp:51     dmb_adamw_prepare
 *   adamw_apply           optim.hpp:59      .cpp:57     dmb_adamw_apply
 *   baseline_sgd_step     optim.hpp:66      .cpp:76     dmb_baseline_sgd_step
 *   chunk_layout / chunk / unchunk  transform.hpp:20-26  dmb_chunk_layout / dmb_chunk / dmb_unchunk
 *   dct2 / idct3 (DctPlan) transform.hpp:28-53         dmb_dct2 / dmb_idct3
 *   extract_fast_components transform.hpp:55-71        dmb_extract_fast_components
 *   sign_transform        transform.hpp:73              dmb_sign_transform
 *   grad_reduce_scatter   cluster.hpp:78    .cpp:63     dmb_grad_mean (local mean; the
 *                                                       split/exchange is NCCL's)
 *   run_step_hybrid schedule (per shard: decode_and_merge + apply, cluster.cpp:193-231)
 *                                                       dmb_merge_apply_sgd / _adamw
 *   one-rank run_step (prepare -> merge(R=1) -> apply)  dmb_step_sgd_local / _adamw_local
 *
 * Conventions
 *   - All vector arguments are device pointers (float32), caller owned.  Calls are
 *     stream ordered on `stream` (a cudaStream_t; NULL = legacy default stream).
 *   - Return codes follow common.hpp:10-26: DMB_TRAINING (TrainingError),
 *     DMB_CONFIG (ConfigError), DMB_PROTOCOL (ProtocolError), plus DMB_CUDA.
 *     dmb_last_error() returns the thread-local message of the last failure.
 *   - Non-finite gradients (require_finite, vec.cpp:7-16) are detected on the
 *     device; the index of the first offending element is latched in the context
 *     and every later kernel of the step becomes a no-op, so no state is touched
 *     (optim.cpp:21).  dmb_status() synchronizes and reports it as DMB_TRAINING.
 *     Momentum is double buffered (m_in -> m_out) so a failed step leaves m_in.
 *   - A dmb_update is the device image of CompressedUpdate (replicate.hpp:43-59):
 *     `body` holds exactly the reference's serialized body (replicate.cpp:316-356)
 *     -- u32 frequency indices (DeMo only) then the values packed per transfer
 *     dtype -- so body_bytes == the reference byte count and the NCCL all-gather
 *     moves exactly the modelled wire bytes.
 */
#ifndef DEMO_B200_H
#define DEMO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DMB_ABI_VERSION 1

enum { DMB_OK = 0, DMB_TRAINING = 1, DMB_CONFIG = 2, DMB_PROTOCOL = 3, DMB_CUDA = 4 };
/* replicate.hpp:14 (wire tags) and :16 */
enum { DMB_DEMO = 1, DMB_RANDOM = 2, DMB_STRIDING = 3, DMB_DILOCO = 4, DMB_FULL = 5 };
enum { DMB_FP32 = 0, DMB_FP16 = 1, DMB_TERNARY = 2 };
/* optim.hpp:11 */
enum { DMB_DEMO_SGD = 0, DMB_DECOUPLED_ADAMW = 1 };
/* DeMo body layout.  REFERENCE: replicate.cpp:316-356 (u32 indices, then values per dtype).
 * MASK (exchange-only, lossless): one u64 frequency mask per chunk (bit j = frequency j),
 * then the values in ascending frequency per chunk, packed per dtype; MASK_SIGN (sign_mode
 * or ternary: the values are exactly -1/0/+1): the masks, then per chunk 16 bytes of 2-bit
 * codes (1: +1, 2: -1, 0: zero or not selected) as four u32 words, word s holding the
 * frequencies 8r + 2s + b (r = 0..7, b = 0..1) at bits 2(2r + b).  At s=64, k=32, sign on the
 * body is 24 B per chunk instead of 256 B.  dmb_serialize always emits the reference bytes. */
enum { DMB_WIRE_REFERENCE = 0, DMB_WIRE_MASK = 1, DMB_WIRE_MASK_SIGN = 2 /* MASK, 2-bit values */ };

/* ReplicatorConfig, replicate.hpp:28-39 */
typedef struct {
  int32_t scheme;
  int32_t sign_mode;
  int32_t transfer_dtype;
  int32_t _pad;
  uint64_t chunk_size;
  uint64_t top_k;
  double compression;
  uint64_t seed;
} dmb_rep_cfg;

/* OptimizerConfig, optim.hpp:13-21 */
typedef struct {
  int32_t kind;
  int32_t _pad;
  double learning_rate;
  double momentum_decay;
  double adam_beta1;
  double adam_beta2;
  double adam_eps;
  double weight_decay;
} dmb_opt_cfg;

/* CompressedUpdate, replicate.hpp:43-59 (metadata on the host, payload on the device) */
typedef struct {
  int32_t scheme;
  int32_t empty;
  uint64_t step;
  uint32_t shard_id;
  uint32_t wire_format;  /* DMB_WIRE_REFERENCE, or DMB_WIRE_MASK (set by the encoder) */
  uint64_t length;
  uint64_t chunk_size;
  uint64_t top_k;
  uint64_t n_values;
  uint64_t n_indices;
  uint64_t bytes;  /* == body bytes == wire_bytes(n_values, n_indices, dtype) */
  void* body;      /* device; capacity >= dmb_update_capacity() */
} dmb_update;

typedef struct dmb_ctx dmb_ctx;

int dmb_abi_version(void);
const char* dmb_last_error(void);

/* one context per device and host thread: basis tables, status latch, scratch */
int dmb_ctx_create(int device, dmb_ctx** out);
int dmb_ctx_destroy(dmb_ctx* ctx);

/* ---- planning (host only, no device work) ---------------------------------- */
uint64_t dmb_wire_bytes(uint64_t n_values, uint64_t n_indices, int32_t dtype);
uint64_t dmb_period(double compression);
/* validates cfg for a vector of `len` at `step` (config.cpp / replicate.cpp rules) and
 * fills the update header select_and_encode will produce; body untouched */
int dmb_plan_update(const dmb_rep_cfg* cfg, uint64_t len, uint64_t step, uint32_t shard,
                    dmb_update* out);
/* device bytes a body needs for this cfg/len at any step (16-byte rounded) */
uint64_t dmb_update_capacity(const dmb_rep_cfg* cfg, uint64_t len);

/* ---- transform.hpp:13-74 (device FP32 vectors; the DCTs accumulate in FP64 in the
 * reference's order from its libm basis, size <= 1024) --------------------------- */
/* ChunkLayout, transform.hpp:13-18 */
typedef struct {
  uint64_t length;
  uint64_t chunk_size;
  uint64_t num_chunks;
  uint64_t pad; /* zeros appended to the last chunk */
} dmb_layout;
/* chunk_layout, transform.hpp:20 / .cpp:17-25 (host only) */
int dmb_chunk_layout(uint64_t length, uint64_t chunk_size, dmb_layout* out);
/* chunk / unchunk, transform.hpp:23-26 / .cpp:27-39: rows = num_chunks x chunk_size, pad zeroed */
int dmb_chunk(dmb_ctx* ctx, const float* v, const dmb_layout* layout, float* rows, void* stream);
int dmb_unchunk(dmb_ctx* ctx, const float* rows, const dmb_layout* layout, float* v, void* stream);
/* dct2 / idct3 (DctPlan::forward / inverse), transform.hpp:28-53: `count` vectors of `size` */
int dmb_dct2(dmb_ctx* ctx, const float* x, uint64_t size, uint64_t count, float* out, void* stream);
int dmb_idct3(dmb_ctx* ctx, const float* coeffs, uint64_t size, uint64_t count, float* out, void* stream);
/* extract_fast_components, transform.hpp:55-71 / .cpp:94-155: indices (num_chunks * top_k,
 * chunk local, ascending), coeffs, fast and residual = v - fast (each output nullable but fast) */
int dmb_extract_fast_components(dmb_ctx* ctx, const float* v, uint64_t len, uint64_t chunk_size,
                                uint64_t top_k, uint32_t* indices, float* coeffs, float* fast,
                                float* residual, void* stream);
/* sign_transform, transform.hpp:73 / .cpp:157-161 (in place) */
int dmb_sign_transform(dmb_ctx* ctx, float* v, uint64_t n, void* stream);

/* ---- replicate.hpp ---------------------------------------------------------- */
int dmb_selected_indices(dmb_ctx* ctx, const dmb_rep_cfg* cfg, uint64_t step, uint32_t shard,
                         uint64_t len, uint32_t* d_out, uint64_t* count, void* stream);
int dmb_select_and_encode(dmb_ctx* ctx, const float* v, uint64_t len, const dmb_rep_cfg* cfg,
                          uint64_t step, uint32_t shard, dmb_update* out,
                          float* local_q /* nullable */, void* stream);
int dmb_decode_and_merge(dmb_ctx* ctx, const dmb_update* updates, uint64_t n_updates,
                         const dmb_rep_cfg* cfg, float* q, void* stream);
/* host bytes: 9-byte header + body, byte-identical to serialize() */
int dmb_serialize(const dmb_update* u, int32_t dtype, uint8_t* host_out, uint64_t capacity,
                  uint64_t* written, void* stream);
int dmb_deserialize(const uint8_t* host_buf, uint64_t size, int32_t dtype,
                    const dmb_update* shape_template, dmb_update* out, void* stream);
/* device body -> float32 values (wire precision), for inspection and tests */
int dmb_update_values(const dmb_update* u, int32_t dtype, float* d_values, void* stream);

/* ---- optim.hpp -------------------------------------------------------------- */
int dmb_demo_sgd_prepare(dmb_ctx* ctx, const float* grad, const float* m_in, float* m_out,
                         uint64_t len, const dmb_opt_cfg* opt, const dmb_rep_cfg* cfg,
                         uint64_t step, uint32_t shard, dmb_update* out,
                         float* local_q /* nullable */, float* m_accum /* nullable */,
                         void* stream);
int dmb_demo_sgd_apply(dmb_ctx* ctx, float* params, const float* q, uint64_t n, double lr,
                       void* stream);
int dmb_adamw_prepare(dmb_ctx* ctx, const float* grad, uint64_t len, const dmb_rep_cfg* cfg,
                      uint64_t step, uint32_t shard, dmb_update* out,
                      float* local_q /* nullable */, void* stream);
int dmb_adamw_apply(dmb_ctx* ctx, float* params, float* exp_avg, float* exp_avg_sq,
                    uint64_t* steps, const float* grad, const float* local_q,
                    const float* merged /* nullable */, uint64_t n, const dmb_opt_cfg* opt,
                    double lr, void* stream);
int dmb_baseline_sgd_step(dmb_ctx* ctx, float* params, float* m, const float* grad, uint64_t n,
                          const dmb_opt_cfg* opt, double lr, void* stream);

/* ---- the fused hot path ----------------------------------------------------- */
/* decode_and_merge + demo_sgd_apply without materializing Q; grad_if_unsynced is the
 * raw shard gradient applied on a DiLoCo off-beat (cluster.cpp:225) */
int dmb_merge_apply_sgd(dmb_ctx* ctx, const dmb_update* updates, uint64_t n_updates,
                        const dmb_rep_cfg* cfg, float* params,
                        const float* grad_if_unsynced, uint64_t len, uint64_t step,
                        double lr, void* stream);
/* decode_and_merge + adamw_apply; local_q is re-derived from grad and this rank's own
 * update `own` (updates[own_rank]) instead of being stored; updates may be NULL on a
 * DiLoCo off-beat (merged == nullptr, cluster.cpp:227) */
int dmb_merge_apply_adamw(dmb_ctx* ctx, const dmb_update* updates, uint64_t n_updates,
                          uint64_t own_rank, const dmb_rep_cfg* cfg, float* params,
                          float* exp_avg, float* exp_avg_sq, uint64_t* steps, const float* grad,
                          uint64_t len, uint64_t step, const dmb_opt_cfg* opt, double lr,
                          void* stream);
/* the same merges with the state read from *_in and written to *_out (distinct buffers: the
 * step can merge before the ranks have agreed on it, a refused step keeps every *_in; synchronized
 * updates only) */
int dmb_merge_apply_sgd_to(dmb_ctx* ctx, const dmb_update* updates, uint64_t n_updates,
                           const dmb_rep_cfg* cfg, const float* p_in, float* p_out, uint64_t len,
                           uint64_t step, double lr, void* stream);
int dmb_merge_apply_adamw_to(dmb_ctx* ctx, const dmb_update* updates, uint64_t n_updates,
                             uint64_t own_rank, const dmb_rep_cfg* cfg, const float* p_in, float* p_out,
                             const float* ea_in, float* ea_out, const float* es_in, float* es_out,
                             uint64_t* steps, const float* grad, uint64_t len, uint64_t step,
                             const dmb_opt_cfg* opt, double lr, void* stream);
/* one replica group of one member: prepare -> merge(R=1) -> apply in one pass over HBM.
 * `out` may be NULL (payload not materialized) or receive the update for inspection. */
/* DeMo scheme only.  State is read from *_in and written to *_out (they may alias;
 * with distinct buffers a non-finite gradient leaves every *_in untouched). */
int dmb_step_sgd_local(dmb_ctx* ctx, const float* grad, const float* m_in, float* m_out,
                       const float* p_in, float* p_out, uint64_t len, const dmb_opt_cfg* opt,
                       const dmb_rep_cfg* cfg, uint64_t step, uint32_t shard, double lr,
                       dmb_update* out /* nullable */, void* stream);
int dmb_step_adamw_local(dmb_ctx* ctx, const float* grad, const float* p_in, float* p_out,
                         const float* ea_in, float* ea_out, const float* es_in, float* es_out,
                         uint64_t* steps, uint64_t len, const dmb_opt_cfg* opt,
                         const dmb_rep_cfg* cfg, uint64_t step, uint32_t shard, double lr,
                         dmb_update* out /* nullable */, void* stream);

/* ---- cluster.cpp:63-91: member-order mean of A gradient vectors (device) -------- */
int dmb_grad_mean(dmb_ctx* ctx, const float* const* grads, uint64_t members, uint64_t len,
                  float* out, void* stream);

/* the same mean pulled over NVLink: `grads` may point into the shard-group peers' memory mapped
 * into this device (symmetric memory); a persistent grid of at most `ctas` CTAs (0: one wave over
 * every SM) with 16-byte loads in flight, so it can run beside a step kernel that leaves those
 * SMs free (DMB_SM_RESERVE) -- the reduce-scatter of bucket b+1 under the prepare of bucket b */
int dmb_grad_mean_pull(dmb_ctx* ctx, const float* const* grads, uint64_t members, uint64_t len,
                       float* out, uint32_t ctas, void* stream);

/* The shard group's reduce-scatter fused into the prepare / the one-member step: the encoded
 * gradient is the member-order mean of members[0..n) (mean_of, vec.cpp:18-26 -- each a
 * shard-sized slice of a member's gradient, local or staged from a peer), computed in the
 * tensor-core kernel's gradient load and written to grad_mean for the later readers (the merge
 * re-derives local_q from it).  The AdamW prepare takes four members, the one-pass AdamW step
 * two; otherwise -- more members, the DeMo-SGD entry points, the generic kernels -- the mean is
 * a pass of its own first (same results). */
int dmb_adamw_prepare_members(dmb_ctx* ctx, const float* const* members, uint32_t n_members,
                              float* grad_mean, uint64_t len, const dmb_rep_cfg* cfg, uint64_t step,
                              uint32_t shard, dmb_update* out, void* stream);
int dmb_demo_sgd_prepare_members(dmb_ctx* ctx, const float* const* members, uint32_t n_members,
                                 float* grad_mean, const float* m_in, float* m_out, uint64_t len,
                                 const dmb_opt_cfg* opt, const dmb_rep_cfg* cfg, uint64_t step,
                                 uint32_t shard, dmb_update* out, void* stream);
int dmb_step_sgd_local_members(dmb_ctx* ctx, const float* const* members, uint32_t n_members,
                               float* grad_mean, const float* m_in, float* m_out, const float* p_in,
                               float* p_out, uint64_t len, const dmb_opt_cfg* opt,
                               const dmb_rep_cfg* cfg, uint64_t step, uint32_t shard, double lr,
                               dmb_update* out, void* stream);
int dmb_step_adamw_local_members(dmb_ctx* ctx, const float* const* members, uint32_t n_members,
                                 float* grad_mean, const float* p_in, float* p_out,
                                 const float* ea_in, float* ea_out, const float* es_in,
                                 float* es_out, uint64_t* steps, uint64_t len,
                                 const dmb_opt_cfg* opt, const dmb_rep_cfg* cfg, uint64_t step,
                                 uint32_t shard, double lr, dmb_update* out, void* stream);

/* require_finite (vec.cpp:7-16) on its own: latches the first non-finite index */
int dmb_require_finite(dmb_ctx* ctx, const float* v, uint64_t n, void* stream);

/* ---- model.hpp: the toy gradient producers, for the trainer loop (trainer.cpp:49-90) ----
 * dmb_toy_model mirrors Model (model.hpp:36-46): kind 0 quadratic (dims = {dim}), 1 mlp
 * (dims = layer_dims, at most 9 entries); activation 0 tanh / 1 relu; loss 0 mse / 1 cross
 * entropy.  dmb_toy_pool is a dataset split resident on the device (dataset.hpp:18-23). */
typedef struct dmb_toy_model {
  uint32_t kind, activation, loss, n_dims;
  uint32_t dims[9];
} dmb_toy_model;
typedef struct dmb_toy_pool {
  const double* inputs;   /* size x dims[0] */
  const double* targets;  /* size x dims[n_dims-1] (mse), or NULL */
  const int32_t* labels;  /* size (cross entropy), or NULL */
  uint64_t size;
} dmb_toy_pool;
/* loss_and_gradient (model.cpp:138-203) for `workers` ranks in one launch: rank w evaluates
 * at params + (w / workers_per_row) * params_stride on the batch BatchStream::indices_for(step,
 * w) selects through the device permutation `order` (dataset.cpp:141-151; world = workers);
 * writes grad[w * grad_len ...] (FP32, the pad tail past param_count zeroed) and loss[w]
 * (FP64).  FP64 arithmetic in the reference's operation order. */
int dmb_toy_loss_grad(dmb_ctx* ctx, const dmb_toy_model* model, const dmb_toy_pool* pool,
                      const int64_t* order, uint64_t step, uint64_t batch, const float* params,
                      uint64_t params_stride, uint64_t workers_per_row, uint64_t workers,
                      float* grad, uint64_t grad_len, double* loss, void* stream);
/* forward_loss (model.cpp:127-136) over the whole pool at params: *loss (device FP64) */
int dmb_toy_loss(dmb_ctx* ctx, const dmb_toy_model* model, const dmb_toy_pool* pool,
                 const float* params, double* loss, void* stream);

/* ---- status / counters ------------------------------------------------------- */
/* synchronizes `stream`; DMB_TRAINING with *first_bad set if a non-finite gradient was
 * seen since the last call (the latch is then cleared), else DMB_OK */
int dmb_status(dmb_ctx* ctx, void* stream, int64_t* first_bad);
/* chunks whose first TopK could not be certified and were re-derived by a fix-up pass
 * (tighter FP32 bound, else FP64 in the oracle's order), cumulative */
int dmb_fallback_chunks(dmb_ctx* ctx, void* stream, uint64_t* count);
/* kernels launched by this context since creation (host counter) */
uint64_t dmb_launch_count(dmb_ctx* ctx);
/* DeMo exchange format of the updates this context encodes (DMB_WIRE_REFERENCE default;
 * DMB_WIRE_MASK selects MASK, recorded as DMB_WIRE_MASK_SIGN in updates whose values are
 * signs).
 * DMB_WIRE_MASK applies to DeMo vectors of whole chunks at s = 64 (the tensor-core encoders
 * of both optimizers); other vectors keep the reference layout (dmb_plan_exchange tells
 * which).  Merges read each update's wire_format. */
int dmb_set_wire_format(dmb_ctx* ctx, int32_t format);
/* dmb_plan_update for this context: the header (wire_format, body bytes) the encoder will
 * produce at this context's wire format, so a caller can size exchange slots before any
 * prepare runs (the layout is decided from the configuration alone; a prepare that cannot
 * honour it -- misaligned vectors, a local_q / m_accum output -- fails with DMB_CONFIG) */
int dmb_plan_exchange(dmb_ctx* ctx, const dmb_rep_cfg* cfg, uint64_t len, uint64_t step, uint32_t shard,
                      dmb_update* out);
/* cross-rank step agreement (cluster.cpp:182: every gradient is checked before any state
 * changes): export writes 1 to the device int *d_flag when this context's status latch is
 * set, 0 otherwise; after the flags are max-reduced over the group (NCCL, on the device),
 * import latches the context when the group flag is set, so every later kernel of the step
 * is a no-op on every rank (dmb_status then reports DMB_TRAINING, first_bad = -2) */
int dmb_latch_export(dmb_ctx* ctx, int32_t* d_flag, void* stream);
int dmb_latch_import(dmb_ctx* ctx, const int32_t* d_flag, void* stream);
/* instrumentation: when enabled, CUDA events bracket every launch of the dominant
 * tensor-core step kernel on its stream; read returns their summed time and count
 * (synchronizing on the recorded events) and clears them */
int dmb_kernel_timer_enable(int on);
/* process-wide: SMs the persistent tensor-core step kernels leave free for kernels that run
 * beside them (dmb_grad_mean_pull of the next bucket); 0 (default) uses every SM.  The
 * environment variable DMB_SM_RESERVE overrides it. */
int dmb_set_sm_reserve(int sms);
int dmb_kernel_timer_read(double* total_ms, uint64_t* launches);

#ifdef __cplusplus
}
#endif
#endif
