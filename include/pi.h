/*
 * pi.h -- C ABI of libpi: PowerInfer's predictor-gated, neuron-aware sparse FFN
 * (arXiv 2312.12456) for batch-1 / small-batch decoding, hand-written for sm_100a.
 *
 * Citations: "P:n" = line n of the paper text, "S:n" = line n of
 * SPEC.md.  Readings Rk of ambiguous passages are listed in DESIGN.md.
 *
 * One layer, one call sequence per decode step:
 *   pi_predict     a1+a2  predictor MLP + threshold -> per-token neuron bitmask
 *   pi_compact     a3     ascending ids of neurons active for any token (union)
 *   pi_sparse_ffn  a4+a5  row-sparse up(/gate) GEMV + column-sparse down GEMV
 *   pi_layer_forward      all of the above in one persistent kernel
 *   pi_partition          host-side neuron -> GPU placement (adapted)
 *
 * Conventions shared by every entry point
 *   - Every call returns pi_status; nothing throws across the ABI.  On error a
 *     message is available from pi_last_error() (thread-local, valid until the
 *     next pi_* call on that thread).
 *   - Host-side validation runs before anything is enqueued.  On a validation
 *     error nothing is enqueued and outputs are untouched.  Asynchronous device
 *     faults surface as PI_ERR_CUDA at a later call.
 *   - "dev" pointers are CUDA device pointers, "host" pointers are host memory.
 *   - Device calls are asynchronous on `stream`, never synchronise the host
 *     (except the *_host variants), and are CUDA-graph capturable.  The active
 *     count stays on the device; kernels are sized for the worst case.
 *   - A layer handle owns workspace: at most one call in flight per handle
 *     (SPEC likewise serialises infer calls).
 *   - Activations x, g, z, h, y are fp32 ("intermediate activations in FP32",
 *     P:854-855); weights are fp16 (the paper's) or bf16.
 *   - Mask layout: uint32 words [B, ceil(m_local/32)], bit (i & 31) of word
 *     (i >> 5) = local neuron i, token-major.
 */
#ifndef PI_H_
#define PI_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *pi_stream_t; /* == cudaStream_t; NULL = legacy default stream */
typedef struct pi_layer pi_layer;        /* opaque layer handle */

typedef enum {
  PI_OK = 0,
  PI_ERR_INVALID_ARGUMENT = 1, /* NULL handle/pointer, batch < 1 or > max_batch, bad enum     */
  PI_ERR_SHAPE = 2,            /* inconsistent dims; message names layer_id and expected/actual */
  PI_ERR_INDEX = 3,            /* neuron id out of range / not strictly ascending */
  PI_ERR_ALIGNMENT = 4,        /* device pointer not 16-B aligned, d % 8 != 0, rank % 8 != 0  */
  PI_ERR_UNSUPPORTED = 5,      /* dtype/act combination not compiled, device is not sm_100     */
  PI_ERR_CUDA = 6,             /* CUDA error; message carries cudaGetErrorString               */
  PI_ERR_OUT_OF_MEMORY = 7
} pi_status;

typedef enum { PI_DT_F16 = 0, PI_DT_BF16 = 1 } pi_dtype;
/* FFN weight format.  PI_FFN_16: w_up / w_gate / w_down hold `dtype` values in the nn.Linear
 * layouts below.  PI_FFN_Q4: INT4 weight-only neuron rows ("FP16 and INT4 quantized
 * parameters"; "Inference with Quantization"; format = DESIGN.md reading
 * R21): every neuron's d-vector -- its up row, gate row and down COLUMN -- is given as a row of
 * d/2 code bytes (neuron-major [m_total, d/2] uint8; element 2k in the low nibble of byte k)
 * plus d/32 fp16 scales (*_scale, [m_total, d/32]); w = scale[j / 32] * (code_j - 8).  The
 * predictor, b_up and b_down stay in `dtype`.  d % 32 == 0. */
typedef enum { PI_FFN_16 = 0, PI_FFN_Q4 = 1 } pi_ffn_format;
/* PI_ACT_RELU: h = relu(a).  PI_ACT_REGLU: h = relu(W_gate[i].x) * a (reading R5). */
typedef enum { PI_ACT_RELU = 0, PI_ACT_REGLU = 1 } pi_act;
/* predictor hidden non-linearity (P:555 names only "a single hidden" layer; reading R1) */
typedef enum { PI_PRED_RELU = 0, PI_PRED_LINEAR = 1 } pi_pred_act;

/* PI_FLAG_INPUT_RMSNORM: predictor and FFN both use x_hat = x * rsqrt(mean(x^2) + 1e-6)
 * per token (harness stand-in for the pre-FFN norm of chained stacks; reading R19). */
#define PI_FLAG_INPUT_RMSNORM 1u
/* PI_FLAG_MULTI_KERNEL: pi_layer_forward runs the per-step kernels (predict, compact, up,
 * down) instead of the single fused persistent kernel (ablation / cross-check). */
#define PI_FLAG_MULTI_KERNEL 2u

/* B <= 8: CUDA-core kernels (B <= 2 also the fused persistent kernel); 9 <= B <= 32: the
 * batched tensor-core path (tcgen05 gathered GEMMs), which needs 16-bit FFN
 * weights and d % 128 == 0. */
#define PI_MAX_BATCH 32
/* default for pi_layer_desc.hot_cap (hot neurons L2-prefetched per layer and step) */
#define PI_DEFAULT_HOT_CAP 512

/* Layer description.  Weight pointers are DEVICE pointers in the PyTorch
 * nn.Linear layouts of the GLOBAL layer (m_total neurons); the handle keeps the
 * rows named by neuron_ids ("neuron tables ... correlate each neuron to its
 * original position in the matrix"). */
typedef struct {
  int32_t layer_id;          /* used in messages only                                          */
  int32_t d;                 /* hidden size; d % 8 == 0                                         */
  int32_t m_total;           /* FFN width of the global layer                                   */
  int32_t rank;              /* predictor hidden width r; r % 8 == 0                */
  int32_t m_local;           /* neurons owned by this handle (= m_total when unsharded)         */
  const int32_t *neuron_ids; /* host [m_local], strictly ascending global ids; NULL = 0..m_total-1 */
  pi_dtype dtype;
  pi_act act;
  pi_pred_act pred_act;
  const void *w_up;   /* dev [m_total, d]  FC1: row i = neuron i (P:107 footnote)           */
  const void *w_gate; /* dev [m_total, d]  required iff act == PI_ACT_REGLU                */
  const void *w_down; /* dev [d, m_total]  FC2 (nn.Linear fc2.weight): column i = neuron i */
  const void *b_up;   /* dev [m_total] or NULL; added before the activation          */
  const void *b_down; /* dev [d] or NULL; give it to exactly ONE shard (merge adds it once) */
  const void *p_w1;   /* dev [rank, d]     predictor input->hidden, replicated on shards   */
  const void *p_b1;   /* dev [rank] or NULL                                                 */
  const void *p_w2;   /* dev [m_total, rank] predictor hidden->output                      */
  const void *p_b2;   /* dev [m_total] or NULL                                              */
  float logit_threshold; /* neuron active iff logit z > t; t = 0 <=> sigmoid(z) > 0.5 (S:216,
                            reading R3); -INFINITY => all finite logits; NaN logits inactive */
  int32_t max_batch;     /* 1..PI_MAX_BATCH; sizes the workspace                               */
  uint32_t flags;        /* PI_FLAG_*                                                          */
  /* Hot neurons (Insight-1): the profiler's activation frequency f_i (Eq. 1,
   * P:680-690) of the GLOBAL layer, host [m_total], or NULL.  Neurons of this shard with
   * f_i >= hot_freq are "hot": while the layer runs its predictor and synchronises, the fused
   * kernel pulls their up/down rows into L2 so the FFN phase streams them from L2 instead of
   * HBM.  Results are unchanged (hotness only affects data movement).  Hot neurons are ranked
   * by (-f_i, id); at most hot_cap of them (<= 0: PI_DEFAULT_HOT_CAP) are prefetched per step,
   * the hottest first. */
  const float *neuron_freq;
  float hot_freq;
  int32_t hot_cap;
  /* Speculative hot prefix (Insight-1: ~3% of neurons fire for ~every token): neurons
   * of this shard with f_i >= spec_freq (hottest first, at most spec_cap; spec_freq <= 0 or
   * spec_cap <= 0 disables) are, in a stack launch (pi_stack_run), computed BEFORE the layer's
   * mask is known -- their rows stream and their up/down products accumulate while the grid
   * synchronises and compacts after the predictor -- and corrected afterwards (their down
   * contribution subtracted) for every token whose predicted bit is 0.  Results equal the
   * non-speculative path up to fp32 summation order (bit for bit on integer-exact layers).
   * Speculative neurons are not L2-prefetched again by the hot-neuron prefetch. */
  float spec_freq;
  int32_t spec_cap;
  pi_ffn_format ffn_format;  /* PI_FFN_16 (default, 0) or PI_FFN_Q4                         */
  const void *w_up_scale;    /* PI_FFN_Q4: dev fp16 [m_total, d/32]; else NULL               */
  const void *w_gate_scale;  /* PI_FFN_Q4 and REGLU: dev fp16 [m_total, d/32]; else NULL     */
  const void *w_down_scale;  /* PI_FFN_Q4: dev fp16 [m_total, d/32]; else NULL               */
} pi_layer_desc;

typedef struct {
  int32_t d, m_local, rank, max_batch, mask_words; /* mask_words = ceil(m_local/32) */
  int32_t dtype, act, pred_act;
  uint32_t flags;
  int32_t num_sms;          /* SMs of the device the handle lives on                */
  int64_t weight_bytes;     /* library-owned weight bytes on the device             */
  int64_t workspace_bytes;  /* library-owned workspace bytes                        */
  int32_t launches_per_forward; /* kernel launches one pi_layer_forward call makes   */
  int32_t ffn_format;           /* pi_ffn_format                                      */
  int32_t n_spec;               /* speculative hot-prefix neurons of this handle      */
} pi_layer_info;

/* Library version string, e.g. "libpi 0.1.0 sm_100a". */
const char *pi_version(void);
/* Thread-local message for the last failed call on this thread ("" if none). */
const char *pi_last_error(void);

/* Create a layer handle on the current CUDA device.  COPIES and repacks this
 * shard's weights into library-owned device memory asynchronously on `stream`:
 * up rows (gate|up interleaved per neuron for ReGLU), down transposed to
 * [m_local, d] so each neuron's down vector is contiguous, P2 rows, b_up, b2
 * gathered by neuron_ids; P1, b1, b_down copied.  The caller may free its
 * tensors once `stream` has completed.  Errors: INVALID_ARGUMENT, SHAPE, INDEX
 * (neuron_ids not strictly ascending or >= m_total), ALIGNMENT, UNSUPPORTED,
 * OUT_OF_MEMORY, CUDA.  On error *out is NULL and nothing leaks. */
pi_status pi_layer_create(const pi_layer_desc *desc, pi_stream_t stream, pi_layer **out);
/* Synchronises the device, then frees everything the handle owns.  NULL is a no-op. */
pi_status pi_layer_destroy(pi_layer *L);
pi_status pi_layer_get_info(const pi_layer *L, pi_layer_info *info);

/* a1 + a2: the predictor.
 *   u = P1 x_b + b1 ; g = act_p(u) ; z = P2 g + b2 ; bit_{b,i} = (z_i > t)
 * x      dev fp32 [B, d], row-major, 16-B aligned
 * mask   dev uint32 [B, mask_words] (written, bits past m_local are 0)
 * logits dev fp32 [B, m_local] or NULL (written if given)
 * Errors: INVALID_ARGUMENT (NULL, B out of 1..max_batch), ALIGNMENT, CUDA. */
pi_status pi_predict(pi_layer *L, const float *x, int32_t B, uint32_t *mask, float *logits,
                     pi_stream_t stream);

/* a3: compaction.  ids = ascending local indices i whose bit is set for ANY of
 * the B tokens (union, reading R9; canonical ascending order S:43-46).
 * mask      dev uint32 [B, mask_words]
 * ids       dev int32 [m_local] (first *n_active entries written)
 * n_active  dev int32 scalar (written on the device; never read back by the library)
 * Errors: INVALID_ARGUMENT, CUDA. */
pi_status pi_compact(pi_layer *L, const uint32_t *mask, int32_t B, int32_t *ids,
                     int32_t *n_active, pi_stream_t stream);

/* a4 + a5: the neuron-aware FFN over the compacted ids.
 *   for k < n_active, i = ids[k], token b:
 *     a = W_up[i] . x_b + b_up[i]
 *     h = relu(a)  |  relu(W_gate[i] . x_b) * a           (act)
 *     h := 0 if token b's own bit for i is 0             (per-token semantics)
 *   y_b = b_down + sum_k h_{b,k} W_down[:, i_k]          (fp32; fixed order, no float atomics)
 * ids       dev int32 [>= n_active], strictly ascending, < m_local (as pi_compact writes)
 * n_active  dev int32 scalar
 * mask      dev uint32 [B, mask_words]; may be NULL iff B == 1 (then every id counts)
 * y         dev fp32 [B, d]; overwritten with this shard's partial (+ b_down if owned)
 * Empty id set: y = b_down or 0.
 * Errors: INVALID_ARGUMENT, ALIGNMENT, CUDA. */
pi_status pi_sparse_ffn(pi_layer *L, const float *x, int32_t B, const int32_t *ids,
                        const int32_t *n_active, const uint32_t *mask, float *y,
                        pi_stream_t stream);

/* All of a1..a5 for one layer and B tokens: the whole hot path.  Equivalent to
 * pi_predict -> pi_compact -> pi_sparse_ffn.  mask_out / ids_out / n_active_out
 * are optional dev outputs (NULL = keep in workspace). */
pi_status pi_layer_forward(pi_layer *L, const float *x, int32_t B, float *y, uint32_t *mask_out,
                           int32_t *ids_out, int32_t *n_active_out, pi_stream_t stream);

/* Same as pi_layer_forward with HOST buffers: x_host fp32 [B, d] is copied to
 * the device, the layer runs, y_host fp32 [B, d] is copied back, and the call
 * returns after `stream` has finished (end-to-end path).  Pinned host memory
 * gives asynchronous copies; pageable memory works but is slower. */
pi_status pi_layer_forward_host(pi_layer *L, const float *x_host, int32_t B, float *y_host,
                                pi_stream_t stream);

/* Chain n_layers layers for B tokens: x_{l+1} = y_l (stacked configs).  x and y
 * are dev fp32 [B, d]; x is not modified (ping-pong buffers live in layer 0's
 * workspace).  All layers must share d and satisfy B <= max_batch.
 * n_active_out: dev int32 [n_layers] (each layer's union count) or NULL. */
pi_status pi_stack_forward(pi_layer *const *layers, int32_t n_layers, const float *x, int32_t B,
                           float *y, int32_t *n_active_out, pi_stream_t stream);

/* pi_stack_forward with HOST buffers (end-to-end path): x_host fp32 [B, d] is
 * copied in, the stack runs, y_host fp32 [B, d] is copied out; returns after
 * `stream` has finished. */
pi_status pi_stack_forward_host(pi_layer *const *layers, int32_t n_layers, const float *x_host,
                                int32_t B, float *y_host, pi_stream_t stream);

/* A stack: L compatible layers (same d, m_local, rank, act, dtype, pred_act, flags,
 * max_batch) run as ONE persistent kernel per decode step, x_{l+1} = y_l.  The kernel's TMA
 * producer streams layer l+1's predictor rows while layer l finishes, and no launch gap
 * separates the layers.  The stack keeps pointers to the layers (it does not own them);
 * destroy the stack before its layers.  A stack run uses layer 0's workspace (the fused
 * kernel's grid barrier, mask, partials and the host-staging buffers), so it counts as the
 * one call in flight on layer 0's handle: do not run layer 0 (or another stack that starts
 * with it) concurrently.  Errors: INVALID_ARGUMENT, SHAPE (incompatible
 * layers), OUT_OF_MEMORY, CUDA. */
typedef struct pi_stack pi_stack;
pi_status pi_stack_create(pi_layer *const *layers, int32_t n_layers, pi_stack **out);
pi_status pi_stack_destroy(pi_stack *S);
/* One decode step through the stack.  x, y: dev fp32 [B, d]; n_active_out: dev int32
 * [n_layers] (each layer's union count) or NULL.  Falls back to one launch per layer when the
 * fused kernel does not support the shape / batch.  Graph capturable. */
pi_status pi_stack_run(pi_stack *S, const float *x, int32_t B, float *y, int32_t *n_active_out,
                       pi_stream_t stream);
/* pi_stack_run with HOST buffers (end-to-end path); returns after `stream` has finished. */
pi_status pi_stack_run_host(pi_stack *S, const float *x_host, int32_t B, float *y_host,
                            pi_stream_t stream);

/* A group: n_groups INDEPENDENT decode problems in ONE persistent launch -- the throughput form
 * of the per-layer operator for layers too small to keep the whole GPU streaming on their own
 * (single-layer decode measured over many layer copies; "the operator ...
 * computes each neuron independently").  The SMs are split into n_groups groups of
 * group_ctas CTAs; group k runs layers[k * n_layers .. (k + 1) * n_layers) as a stack (x_{l+1} =
 * y_l) on its own input with grid barriers local to the group, so the groups' predictor,
 * synchronisation and FFN phases overlap and HBM stays busy.  Every layer must share layer 0's
 * shape, dtype, act, pred_act and flags, with 16-bit FFN rows and no speculative prefix;
 * n_groups * group_ctas <= SMs; the handle owns its own workspace (the layers' workspaces are
 * not used) and keeps pointers to the layers (destroy it before them).  Errors:
 * INVALID_ARGUMENT, SHAPE, UNSUPPORTED (no grouped kernel for the shape, e.g. r > 64 group_ctas),
 * OUT_OF_MEMORY, CUDA. */
typedef struct pi_group pi_group;
/* flags: 0, or one of PI_GROUP_DEFER_*: each group's weight producer requests a layer's predictor
 * rows only after the group has finished the previous layer's reduction (AFTER_REDUCTION) or its
 * last grid barrier (AFTER_BARRIER) instead of running ahead -- the group's barrier and reduction
 * round trips then do not queue behind its own bulk loads while the other groups keep HBM busy. */
#define PI_GROUP_DEFER_AFTER_REDUCTION 1u
#define PI_GROUP_DEFER_AFTER_BARRIER 2u
pi_status pi_group_create(pi_layer *const *layers, int32_t n_groups, int32_t n_layers, int32_t group_ctas,
                          uint32_t flags, pi_group **out);
pi_status pi_group_destroy(pi_group *G);
/* One step of every group: x, y dev fp32 [n_groups, B, d] (group k reads x[k], writes y[k]);
 * B must be 1; n_active_out: dev int32 [n_groups, n_layers] or NULL.  Graph capturable.
 * Errors: INVALID_ARGUMENT, UNSUPPORTED, ALIGNMENT (x, y 16-B aligned), CUDA. */
pi_status pi_group_run(pi_group *G, const float *x, int32_t B, float *y, int32_t *n_active_out,
                       pi_stream_t stream);

/* Profiling aid (tracing): when dev_buf is non-NULL, every later pi_layer_forward that runs
 * the fused kernel has each CTA's thread 0 write globaltimer (ns) stamps of its phase
 * boundaries to dev_buf[cta * 256 + k]: 0 start, 1 P1 done, 2 after grid barrier 1, 3 P2 done,
 * 4 after grid barrier 2, 5 ids extracted, 6 FFN done, 7 after grid barrier 3, 8 end;
 * [16 + i] when ring stage i became readable, [72 + i] when the producer issued it (i < 56).
 * [128..191] phase-2 stage detail.  dev_buf: dev uint64 [num_sms * 256]; NULL turns tracing off.  Errors: INVALID_ARGUMENT. */
pi_status pi_layer_set_trace(pi_layer *L, uint64_t *dev_buf);

/* Neuron -> shard placement (host, deterministic).  Adapts the paper's ILP
 * (Eqs. 2-8) to G identical GPUs (reading R15): every neuron on
 * exactly one shard (Eq. 3), equal counts (Eq. 6 with equal capacities),
 * balanced expected active mass sum f_i (impact v_i = f_i, Eq. 1).  Neurons
 * are ordered by (-f_i, i), cut into runs of `granule` similar-impact neurons
 * (P:809 uses 64), and runs are dealt longest-first to the least-loaded shard
 * with room (ties: lowest shard).
 * freq          host float [m], finite, >= 0
 * owner         host int32 [m]   shard of neuron i
 * shard_ids     host int32 [m]   each shard's ids ascending, shards concatenated in order
 * shard_offsets host int32 [n_shards + 1]
 * Errors: INVALID_ARGUMENT (NULL, n_shards < 1, granule < 1, NaN/negative freq),
 *         SHAPE (m % (granule * n_shards) != 0). */
pi_status pi_partition(const float *freq, int32_t m, int32_t n_shards, int32_t granule,
                       int32_t *owner, int32_t *shard_ids, int32_t *shard_offsets);

/* The paper's neuron-placement ILP (Eqs. 1-8), solved exactly.
 * Two units, fast and slow: maximise the impact sum f_i placed on the fast unit (Eqs. 1-2),
 * every batch of `granule` similar-impact neurons ((-f, i) order within a layer) on
 * one unit (Eq. 3), fast-unit bytes < mcap_fast (Eq. 6), and per layer either no fast neuron or
 * at least C_l, the smallest count with C_l T_fast + t_sync <= C_l T_slow, T = neuron_bytes /
 * bandwidth (Eqs. 4, 5, 7, 8; reading R22).  Exact dynamic programme over layers (within a layer
 * the best k batches are the k most impactful); ties go to fewer fast bytes.  On the B200 the
 * fast unit is the hot-neuron tier of a layer (rows L2-prefetched/pinned, their count fed back
 * as pi_layer_desc.hot_cap), the slow unit the dynamic HBM path.
 * freq          host float [n_layers * m], layer-major, finite, >= 0
 * neuron_bytes  host double [n_layers], positive integers (bytes of one neuron's rows)
 * fast          host uint8 [n_layers * m] out: 1 = neuron placed on the fast unit
 * fast_count    host int32 [n_layers] out: fast neurons per layer
 * objective     host double out: the optimal Eq. 2 value
 * Errors: INVALID_ARGUMENT (NULL, bad sizes, non-finite values), UNSUPPORTED (capacity / batch
 *         size ratio beyond the exact DP's table). */
pi_status pi_place_ilp(const float *freq, int32_t n_layers, int32_t m, const double *neuron_bytes,
                       int32_t granule, double mcap_fast, double bw_fast, double bw_slow, double t_sync,
                       uint8_t *fast, int32_t *fast_count, double *objective);

#ifdef __cplusplus
}
#endif
#endif /* PI_H_ */
