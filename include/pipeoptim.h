/*
 * pipeoptim.h — C-ABI of the B200 (sm_100a) PipeOptim weight-predictor and
 * optimizer kernels (libpipeoptim.so).
 *
 * The reference (arXiv 2312.00839's `pipesim`, /root/reference/pkg) has no FFI:
 * its hot path is the Python duck-typed optimizer/predictor interface in
 * pkg/src/pipesim/optim.py. Each export below replaces one piece of it; the
 * Python binding that mirrors the reference API is
 * paper_2312_00839_b200/optim.py (ctypes), see INTEGRATION.md.
 *
 *   po_step            <- OptimizerState.step             optim.py:63-87
 *                         (_sgdm_directions optim.py:89-99,
 *                          _adam_directions optim.py:101-119)
 *   po_direction       <- OptimizerState.prediction_direction optim.py:123-142
 *   po_predict         <- prediction_direction + predict_weights fused,
 *                         optim.py:123-155 as called by
 *                         _PredictivePolicy.forward_view runtime.py:250-258
 *   po_axpy_predict    <- predict_weights                 optim.py:145-155
 *   po_step_predict    <- step followed by the next forward's prediction on the
 *                         just-updated state (1F1B steady state "U_j F_{j+D-k}",
 *                         runtime.py:449-463 then :411-413), one HBM pass
 *   po_version_difference <- version_difference           optim.py:158-167
 *
 * Conventions:
 *   - All buffers are caller-owned fp32 device arrays of n elements (flat
 *     per-stage layout); the library allocates nothing and keeps no state
 *     beyond a per-device SM-count cache.
 *   - Every export returns int: 0 = ok, PO_EINVAL for bad arguments, otherwise
 *     a cudaError_t from the launch. Nothing is thrown across the ABI.
 *   - Stream-ordered, no host synchronisation inside; `stream` is a
 *     cudaStream_t (NULL = legacy default stream).
 *   - `step_count` is the optimizer's update count BEFORE the call, exactly as
 *     OptimizerState.step_count. Bias corrections are evaluated on the host in
 *     double precision as optim.py:106-108 (step, t = step_count + 1) and
 *     optim.py:136-138 (read, t = step_count), then rounded to fp32.
 *   - Scalar products lr*s are formed by the caller in double (optim.py:155
 *     evaluates `lr * steps_ahead` first) and passed as `lr_times_s`.
 *   - `nonfinite_index` (nullable) is a device int64 the caller initialises to
 *     INT64_MAX; a step that produces a non-finite updated weight lowers it to
 *     the smallest offending flat index (atomicMin), which the binding maps to
 *     the parameter name to raise NumericError like optim.py:82-84.
 *   - Updates are in place on w / state; predictions go to a separate staging
 *     buffer w_hat, so live weights are never touched by prediction
 *     (runtime.py:242-244, S10).
 */
#ifndef PIPEOPTIM_H_
#define PIPEOPTIM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PO_ABI_VERSION 1
#define PO_EINVAL (-22)
#define PO_EDRIVER_BASE 100000 /* CUDA driver-API error r is returned as PO_EDRIVER_BASE + r */

/* optimizer kinds, OPTIMIZER_KINDS optim.py:17 */
#define PO_SGDM 0
#define PO_ADAM 1
#define PO_ADAMW 2

/* OptimizerConfig, optim.py:20-43 (fields in double, as Python floats) */
typedef struct po_hparams {
  int32_t kind;
  int32_t _pad;
  double momentum;        /* u,   default 0.9  */
  double dampening;       /* tau, default 0.0  */
  double weight_decay;    /* sgdm only, default 5e-4 */
  double beta1;           /* default 0.9   */
  double beta2;           /* default 0.999 */
  double eps;             /* default 1e-8  */
  double decoupled_decay; /* adamw lambda, default 1e-2 */
} po_hparams;

/* Optional launch shaping (nullable everywhere; NULL = tuned defaults). */
typedef struct po_launch {
  int32_t block;        /* threads per CTA (multiple of 32, <= 512), 0 = default */
  int32_t ctas_per_sm;  /* persistent grid = SMs * ctas_per_sm, 0 = default */
  int32_t vec;          /* floats per access: 4 (128-bit) or 8 (256-bit), 0 = default */
  int32_t cache;        /* 0 = tuned default, 1 = streaming .cs, 2 = L1::no_allocate
                           loads, 3 = plain ld/st, 4 = mixed (W / W_hat plain,
                           gradient and state streaming) */
  int32_t unroll;       /* vectors per stream in flight per thread: 1, 2, 4; 3 = one vector
                           per stream with the next one prefetched (software
                           pipeline); 0 = default */
} po_launch;

/* One launch's step-dependent fp32 scalars, for graph-captured launches
 * (po_*_dc): the host refreshes an array of these in device memory before
 * each CUDA-graph replay, so replays continue training with the right
 * learning rate and bias corrections. Filled by po_coef_fill exactly as the
 * by-value entry points derive them. */
typedef struct po_coef {
  float lr;     /* step learning rate */
  float c_pred; /* lr_pred * s */
  float inv_bc1; /* 1 / (1 - beta1^t), formed in double (1 when t == 0) */
  float inv_bc2; /* 1 / (1 - beta2^t), formed in double (1 when t == 0) */
} po_coef;

#define PO_COEF_STEP 0
#define PO_COEF_PREDICT 1
#define PO_COEF_STEP_PREDICT 2

int po_abi_version(void);
const char* po_strerror(int code);

/* Eq. (4) D - rank - 1 with the reference's range errors -> PO_EINVAL. */
int po_version_difference(int64_t depth, int64_t rank, int64_t* out);

/* One optimizer update in place: w, state1 (sgdm buf | adam m), state2 (adam v;
 * NULL for sgdm). g is read-only. dir_out (nullable) receives the applied
 * direction d with w_new = w - lr*d (optim.py:64-68). */
int po_step(const po_hparams* hp, float* w, const float* g, float* state1, float* state2,
            float* dir_out, int64_t n, double lr, int64_t step_count,
            int64_t* nonfinite_index, const po_launch* launch, void* stream);

/* W_hat = W - (lr*s) * dir(state) with dir read at t = step_count; when
 * step_count == 0 the direction is zero (optim.py:131-132). Pure read of
 * w/state. */
int po_predict(const po_hparams* hp, const float* w, const float* state1, const float* state2,
               float* w_hat, int64_t n, double lr_times_s, int64_t step_count,
               const po_launch* launch, void* stream);

/* Fused: po_step, then W_hat = W_new - (lr_pred*s) * dir(state_new) read at
 * t = step_count + 1, in one pass (32 B/param Adam, 24 B/param SGDM). */
int po_step_predict(const po_hparams* hp, float* w, const float* g, float* state1,
                    float* state2, float* w_hat, int64_t n, double lr,
                    double lr_pred_times_s, int64_t step_count, int64_t* nonfinite_index,
                    const po_launch* launch, void* stream);

/* prediction_direction: dir_out = dir(state) at t = step_count (zeros when
 * step_count == 0). */
int po_direction(const po_hparams* hp, const float* state1, const float* state2, float* dir_out,
                 int64_t n, int64_t step_count, const po_launch* launch, void* stream);

/* predict_weights: w_hat = w - lr_times_s * d. */
int po_axpy_predict(const float* w, const float* d, float* w_hat, int64_t n, double lr_times_s,
                    const po_launch* launch, void* stream);

/* Host-only: the coefficients po_step / po_predict / po_step_predict would
 * use for (lr, lr_times_s, step_count); `which` is PO_COEF_*. For
 * PO_COEF_PREDICT at step_count == 0 the bias corrections are 1 and, with the
 * optimizer state still zero, the predicted weights equal W (optim.py:131-132). */
int po_coef_fill(const po_hparams* hp, int32_t which, double lr, double lr_times_s, int64_t step_count,
                 po_coef* out);

/* Graph-capturable variants: identical arithmetic, scalars read from
 * `coef_dev` (device pointer) at kernel start. po_predict_dc always reads the
 * state buffers (they must exist, zero before the first step). */
int po_step_dc(const po_hparams* hp, float* w, const float* g, float* state1, float* state2, int64_t n,
               const po_coef* coef_dev, int64_t* nonfinite_index, const po_launch* launch, void* stream);
int po_predict_dc(const po_hparams* hp, const float* w, const float* state1, const float* state2, float* w_hat,
                  int64_t n, const po_coef* coef_dev, const po_launch* launch, void* stream);
int po_step_predict_dc(const po_hparams* hp, float* w, const float* g, float* state1, float* state2,
                       float* w_hat, int64_t n, const po_coef* coef_dev, int64_t* nonfinite_index,
                       const po_launch* launch, void* stream);

/* ---- hybrid DP x PP: gradient mean over peer memory fused into K3 -------- */

/* Release-store `epoch` into slot `my rank` of every replica's flag array
 * (peer_flag_slots: DEVICE array of dp pointers, one per replica, each
 * pointing at that replica's flags[my_rank]); enqueue after the backward that
 * produced this replica's gradient. */
int po_dp_signal(long long* const* peer_flag_slots, int32_t dp, int64_t epoch, void* stream);

/* K3 on this replica's stage with g = (sum over replicas r, in rank order, of
 * grads[r]) / dp read directly from the replicas' (peer-mapped) gradient
 * buffers, after a one-CTA kernel has acquire-waited until flags[r] >= epoch
 * for all r (flags: this replica's local [dp] array that the peers signal
 * into). If a replica has not signalled after timeout_ms, *status = 1 (device
 * int) and nothing is updated. grads_host: HOST array of dp device
 * pointers. dp <= 8. */
int po_step_predict_dp(const po_hparams* hp, float* w, const float* const* grads_host, int32_t dp, float* state1,
                       float* state2, float* w_hat, int64_t n, double lr, double lr_pred_times_s,
                       int64_t step_count, int64_t* nonfinite_index, const int64_t* flags, int64_t epoch,
                       int64_t timeout_ms, int32_t* status, void* stream);

/* CUDA-graph forms of the two (whole runs captured once, replayed): the
 * epoch is a device counter advanced by po_dp_signal_dev and read by the
 * wait of po_step_predict_dp_dc, and the step's scalars come from a device
 * po_coef (po_coef_fill, PO_COEF_STEP_PREDICT) refreshed before each replay. */
int po_dp_signal_dev(long long* const* peer_flag_slots, int32_t dp, int64_t* epoch_ctr, void* stream);
int po_step_predict_dp_dc(const po_hparams* hp, float* w, const float* const* grads_host, int32_t dp, float* state1,
                          float* state2, float* w_hat, int64_t n, const po_coef* coef_dev, int64_t* nonfinite_index,
                          const int64_t* flags, const int64_t* epoch_ctr, int64_t timeout_ms, int32_t* status,
                          void* stream);

/* Sharded form (reduce-scatter + K3 + all-gather in one pass). Replica
 * `rank` owns the shard [lo, hi) given by po_dp_shard_range (ceil(n/dp)
 * rounded up to 64 elements). For its elements it sums the dp gradients
 * (rank order over the peer pointers, or multimem.ld_reduce through the
 * NVSwitch when `mc` gives multicast addresses), applies K3 against its own
 * W / state and stores W', state' and W_hat into EVERY replica's buffers
 * (peer stores, or multimem.st). Each element is computed once, so replicas
 * stay bit-identical. Sequence on `stream`: wait grad_flags[r] >= epoch for
 * all r; the shard pass; release-store epoch into done_slots[r] (DEVICE array
 * of dp pointers: this replica's slot in each replica's done array); wait
 * done_flags[r] >= epoch for all r (this replica's local done array), so the
 * next kernel on `stream` sees the whole update. w, grads, state1, state2,
 * w_hat, nonfinite_index: HOST arrays of dp (peer-mapped) device pointers in
 * rank order; w_hat NULL = plain step; nonfinite_index NULL or per replica
 * (each owner atomicMin's the first non-finite index of its shard into every
 * replica's flag). coef_dev non-NULL overrides lr / lr_pred_times_s /
 * step_count; epoch_dev non-NULL overrides epoch (CUDA-graph forms, with
 * po_dp_signal_dev advancing it). Timeouts set *status = 1 and skip the
 * update and the done signal. dp <= 8. */
typedef struct po_dp_multicast {
  float* grad;   /* all NULL: peer loads / stores */
  float* w;
  float* state1;
  float* state2;
  float* w_hat;
} po_dp_multicast;

int po_dp_shard_range(int64_t n, int32_t dp, int32_t rank, int64_t* lo, int64_t* hi);
int po_step_predict_dp_shard(const po_hparams* hp, int32_t dp, int32_t rank, float* const* w, const float* const* grads,
                             float* const* state1, float* const* state2, float* const* w_hat, int64_t n, double lr,
                             double lr_pred_times_s, int64_t step_count, const po_coef* coef_dev,
                             int64_t* const* nonfinite_index, const int64_t* grad_flags, int64_t* const* done_slots,
                             const int64_t* done_flags, int64_t epoch, const int64_t* epoch_dev, int64_t timeout_ms,
                             int32_t* status, const po_dp_multicast* mc, void* stream);

/* NVLS multicast objects for the sharded update (pipeoptim_nvls.cu). One
 * object per DP group covers a replica's update buffers; the creator exports
 * it as a POSIX fd (the host passes it to the other replicas over a UNIX
 * socket), every replica opens it, adds its current device, and — after all
 * have added — binds one zero-filled local allocation of po_nvls_size bytes,
 * getting a unicast VA (its own buffers) and a multicast VA (for
 * po_dp_multicast). po_nvls_probe: 0 if an object for n_devices can be
 * created on this device (created and released), else the error. */
typedef struct po_nvls po_nvls;
int po_nvls_probe(int32_t n_devices, int64_t bytes, int64_t* granularity);
int po_nvls_create(int32_t n_devices, int64_t bytes, int32_t* fd_out, po_nvls** out);
int po_nvls_open(int32_t fd, int32_t n_devices, int64_t bytes, po_nvls** out);
int po_nvls_add_device(po_nvls* g);
int po_nvls_bind(po_nvls* g, void** uc_ptr, void** mc_ptr);
int64_t po_nvls_size(const po_nvls* g);
int po_nvls_free(po_nvls* g);

/* ---- fused per-event stage ops (pipeoptim_stage_ops.cu) ---------------- */

#define PO_LOSS_MSE 0
#define PO_LOSS_SOFTMAX_XENT 1

/* flags[index] = 0 if any of x[0..n) is NaN or +-Inf (flags pre-set to 1 by
 * the caller): the deferred form of the forward-output finiteness check
 * (stages.py:182). One launch, no host sync. */
int po_all_finite(const float* x, int64_t n, uint8_t* flags, int64_t index, void* stream);

/* Loss and its gradient w.r.t. pred in one launch (linalg.py:212-241):
 * softmax_xent (mean row cross-entropy, grad (softmax - target)/rows) or mse
 * (mean of squares, grad 2 (pred - target)/numel). pred/target/grad are
 * row-major [rows x cols]; *loss (device) receives the scalar. `scratch` is
 * a device buffer of rows floats + one uint32 counter that must be zero
 * before the first launch (the kernel re-arms it). */
int po_loss_grad(int32_t kind, const float* pred, const float* target, int64_t rows, int64_t cols, float* grad,
                 float* loss, float* scratch, void* stream);

/* Reduction of a split-K GEMM fused with the layer epilogue (stages.py:175-178
 * affine + activation): out = act(sum_{s=0..splits-1} part[s] + bias), the
 * partials summed in that fixed order (deterministic). part: [splits x rows x
 * cols], bias: [cols] or NULL, act: 0 linear, 1 relu, 2 tanh; pre_out
 * (nullable) receives the pre-activation. flags (nullable): flags[flag_index]
 * = 0 if any output is NaN/Inf (po_all_finite folded into the epilogue). */
int po_splitk_bias_act(const float* part, int32_t splits, int64_t rows, int64_t cols, const float* bias,
                       int32_t act, float* out, float* pre_out, uint8_t* flags, int64_t flag_index, void* stream);

/* Backward elementwise part of a ReLU layer fused with its bias gradient
 * (stages.py:200-206, linalg.py:185-194): dpre = g * (pre > 0) written to
 * dpre, and db = colsum(dpre) (accumulate != 0: db += colsum). h is the
 * layer's OUTPUT relu(pre) (relu(pre) > 0 <=> pre > 0, so the stash keeps h).
 * g: [splits x rows x cols] partial products (of a split-K input gradient)
 * summed in order, or splits = 1; h, dpre: row-major [rows x cols]; db:
 * [cols]. Deterministic (fixed summation orders); with splits = 1 g may
 * alias dpre. */
int po_relu_bwd_bias(const float* g, int32_t splits, const float* h, int64_t rows, int64_t cols, float* dpre,
                     float* db, int32_t accumulate, void* stream);

/* Same for act = 1 (relu, as above) or act = 0 (linear: dpre = g, no mask,
 * h unused): a linear layer's bias gradient and summed split-K partials. */
int po_act_bwd_bias(int32_t act, const float* g, int32_t splits, const float* h, int64_t rows, int64_t cols,
                    float* dpre, float* db, int32_t accumulate, void* stream);

/* Invalidate the L2 lines of a dead buffer without writing them back
 * (discard.global.L2 on every whole 128-byte line inside [p, p + bytes)):
 * the memory contents become unspecified. For a staging buffer after the
 * forward that consumed it, or a gradient after the update that consumed it. */
int po_l2_discard(void* p, int64_t bytes, void* stream);

/* ---- narrow output layer (pipeoptim_head.cu) --------------------------
 * An MLP layer in -> C with C <= 32 and linear activation (config 1's
 * classifier), x: rows x in, W: in x C, both row-major, contiguous.
 * po_head_fwd: out (rows x C) = x @ W + b (b nullable); a non-finite output
 * clears flags[flag_index] (flags nullable) — stages.py:175-178, :182.
 * po_head_bwd: given g = dL/dout (rows x C): dx = g @ W^T (dx nullable: not
 * needed), dW = x^T @ g, db = colsum(g), written or (accumulate) added —
 * stages.py:200-208 for a linear layer. Fixed summation orders
 * (deterministic). po_head_supported: 1 if the shape is handled. */
int po_head_supported(int64_t rows, int64_t in, int64_t classes);
int po_head_fwd(const float* x, int64_t rows, int64_t in, const float* w, const float* b, int32_t classes,
                float* out, uint8_t* flags, int64_t flag_index, void* stream);
int po_head_bwd(const float* x, int64_t rows, int64_t in, const float* g, int32_t classes, const float* w, float* dx,
                float* dw, float* db, int32_t accumulate, void* stream);

/* Programmatic dependent launch for the short stream kernels (K1/K2/K3,
 * po_splitk_bias_act, po_relu_bwd_bias / po_act_bwd_bias, po_head_*,
 * po_loss_grad): po_set_pdl(1) launches them with the programmatic
 * stream-serialisation attribute (each waits for its predecessor before
 * touching memory: results unchanged); process-wide, default 0; returns 0.
 * po_get_pdl returns the current setting. */
int po_set_pdl(int32_t on);
int po_get_pdl(void);

/* po_head_fwd_loss: po_head_fwd and po_loss_grad in ONE launch (the last
 * stage's forward + loss + dL/dout, runtime.py:415-426 via stages.py:175-184
 * and linalg.py:212-241): out = x @ W + b, then the loss of kind PO_LOSS_*
 * against target (rows x classes) into *loss and its gradient into grad
 * (rows x classes), bit-identical to the two separate calls (same
 * expressions and reduction orders). scratch: po_loss_grad's layout (rows
 * floats + one uint32 counter, zero before the first launch; re-armed). */
int po_head_fwd_loss(const float* x, int64_t rows, int64_t in, const float* w, const float* b, int32_t classes,
                     const float* target, int32_t kind, float* out, float* grad, float* loss, float* scratch,
                     uint8_t* flags, int64_t flag_index, void* stream);

/* ---- weight gradient + update in one kernel (pipeoptim_wgrad.cu) --------
 * g = x^T @ dpre for one MLP layer (x: rows x in, row-major, leading dim
 * ldx; dpre: rows x out, ldd) on the tcgen05 tensor cores (each fp32 operand
 * split into three bf16 pieces, fp32 accumulation in TMEM), never written to
 * memory unless g_out is given: the epilogue applies K3 (w_hat non-NULL) or
 * K2 (w_hat NULL) to the (in x out) row-major weight tensor w and its state
 * (same shape, 32-byte aligned) with the step / prediction coefficients of
 * po_step_predict / po_step (coef_dev non-NULL: from device memory, as the
 * _dc forms). nonfinite_index gets flat_offset + the smallest non-finite
 * index (atomicMin), flat_offset being the tensor's offset in the stage's flat
 * buffer. Shapes: rows % 16 == 0, in % 128 == 0, out % 128 == 0
 * (po_wgrad_update_supported). Replaces the weight-gradient GEMM of
 * stage_backward (stages.py:203) followed by the update (runtime.py:449-463). */
int po_wgrad_update_supported(int64_t rows, int64_t in, int64_t out);
int po_wgrad_update(const po_hparams* hp, const float* x, int64_t ldx, const float* dpre, int64_t ldd, int64_t rows,
                    int64_t in, int64_t out, float* w, float* state1, float* state2, float* w_hat, float* g_out,
                    double lr, double lr_pred_times_s, int64_t step_count, const po_coef* coef_dev,
                    int64_t* nonfinite_index, int64_t flat_offset, void* stream);

/* ---- FP32-accurate tensor-core GEMM (pipeoptim_gemm.cu) -----------------
 * D[l] = A[l] @ B[l] for l < batch, fp32 in/out, computed by tcgen05 UMMA with
 * each fp32 operand split into three bf16 pieces (CUTLASS SM100 fast-FP32
 * mainloop): fp32-level accuracy at tensor-core throughput, for the fp32
 * stage GEMMs (stages.py:175-208). A: M x K, row-major (a_col_major = 0:
 * element (m,k) at m*lda + k) or column-major (1: at m + k*lda), batch stride
 * sa; B: K x N, row-major (b_col_major = 0: (k,n) at k*ldb + n) or
 * column-major (1: at k + n*ldb), batch stride sb; not both column-major.
 * D: M x N row-major contiguous, batch stride M*N. lda, ldb, n, sa, sb
 * multiples of 4 (16-byte TMA alignment). workspace may be NULL when the
 * kernel needs none (the default schedule). */
int po_gemm_f32x3(int32_t a_col_major, int32_t b_col_major, const float* a, int64_t lda, int64_t sa, const float* b,
                  int64_t ldb, int64_t sb, float* d, int64_t m, int64_t n, int64_t k, int64_t batch, void* workspace,
                  int64_t workspace_bytes, void* stream);

/* 1 if po_gemm_f32x3 was compiled (CUTLASS headers found at build time), 0 if
 * the library was built without CUTLASS: po_gemm_f32x3 then returns
 * PO_ENOSYS and the stage math uses cuBLAS. The optimizer kernels never
 * depend on CUTLASS. */
#define PO_ENOSYS (-38)
int po_gemm_f32x3_available(void);

/* Tile width (64 or 128 output columns per 128-row CTA tile) of the next
 * po_gemm_f32x3 calls, process-wide, read at launch / capture time: 64 (the
 * default) gives the most CTAs and the lowest latency for a stage alone on
 * its GPU; 128 halves the CTAs (less SM time per GEMM), faster when several
 * stages share one GPU. Results differ only in fp32 summation grouping
 * inside a tile (both <= 2e-6 of the largest output vs float64).
 * po_set_gemm_tile: PO_EINVAL for other widths. */
int po_set_gemm_tile(int32_t tile_n);
int po_get_gemm_tile(void);

/* ---- peer-memory boundary transport (pipeoptim_p2p.cu) ------------------
 * Replaces the simulated hand-off dicts of the reference executor
 * (runtime.py:390-391, 420-433): one direction of a pipeline boundary is a
 * ring of `slots` message buffers of slot_elems floats on the RECEIVING GPU,
 * mapped into the sender (CUDA IPC). ctl is a zeroed int64[4] control block
 * local to each rank (sent count + arrival counter, received count + arrival
 * counter); flags are int64 counters, monotonic, zero-initialised. Both calls
 * are stream-ordered, host-free and CUDA-graph capturable; a wait that
 * exceeds timeout_ms sets *status = 1 and the transfer is skipped (no hang).
 * slot_elems % 4 == 0. */

/* Wait for ring credit (*ack_flag >= sent + 1 - slots), store src[0..n) into
 * peer_ring[sent % slots], then release-store *peer_ready_flag = ++sent. */
int po_p2p_send(const float* src, int64_t n, float* peer_ring, int64_t slot_elems, int32_t slots, int64_t* ctl,
                const int64_t* ack_flag, int64_t* peer_ready_flag, int64_t timeout_ms, int32_t* status,
                void* stream);

/* Wait for the next message (*ready_flag >= recvd + 1), copy ring[recvd % slots]
 * into dst[0..n), then release-store *peer_ack_flag = ++recvd. */
int po_p2p_recv(const float* ring, int64_t slot_elems, int32_t slots, float* dst, int64_t n, int64_t* ctl,
                const int64_t* ready_flag, int64_t* peer_ack_flag, int64_t timeout_ms, int32_t* status,
                void* stream);

/* Node-shared device buffers (CUDA IPC). po_ipc_alloc: cudaMalloc `bytes`
 * (zero-filled) on the current device and export its 64-byte handle.
 * po_ipc_open: map a peer's buffer into the CURRENT device (peer access over
 * NVLink enabled as needed). po_ipc_close / po_ipc_free release them. */
int po_ipc_alloc(int64_t bytes, void** ptr, uint8_t* handle64);
int po_ipc_open(const uint8_t* handle64, void** ptr);
int po_ipc_close(void* ptr);
int po_ipc_free(void* ptr);

/* ---- live-weight LSTM cell (pipeoptim_lstm.cu) --------------------------
 * One time step of an LSTM layer whose GEMMs run in cuBLAS (PyTorch gate
 * order i, f, g, o; hidden % 4 == 0; all pointers 16-byte aligned). Used by
 * the GNMT stages so the backward can multiply by the LIVE weights
 * (stages.py:200-208 semantics, S9) — cuDNN keeps the forward weights. */

/* gates [batch x 4*hidden]: pre-activations in, activations out (in place).
 * c_prev (NULL = zeros), c_out, h_out: [batch x hidden]. y_out (nullable):
 * a second copy of h_t with row stride y_ld (the batch-first layer output). */
int po_lstm_cell_fwd(float* gates, const float* c_prev, float* c_out, float* h_out, float* y_out, int64_t y_ld,
                     int64_t batch, int64_t hidden, void* stream);

/* act: the forward's activations [batch x 4*hidden]; c_prev (NULL = zeros),
 * c: [batch x hidden]; dy (nullable, row stride dy_ld): the output gradient
 * at this step; dh_rec (nullable): dgates_{t+1} W_hh (the recurrent
 * gradient); dc: in = dc_t from step t+1 (zeros at t = T-1), out = dc_{t-1}.
 * dgates [batch x 4*hidden] receives the pre-activation gradients. */
int po_lstm_cell_bwd(const float* act, const float* c_prev, const float* c, const float* dy, int64_t dy_ld,
                     const float* dh_rec, float* dc, float* dgates, int64_t batch, int64_t hidden, void* stream);

/* The same two steps with the recurrent GEMM run split-K: `rec` holds the
 * `splits` partial products [splits x batch x 4*hidden] of h_{t-1} W_hh^T
 * (added to `gates`, which then carries only the input projection), and
 * `dh_rec` the partials [splits x batch x hidden] of dgates_{t+1} W_hh_live —
 * each summed in order inside the cell kernel (no reduction pass). The batch
 * x 4H / batch x H recurrent GEMMs have too few output tiles to fill the GPU
 * as single GEMMs. */
int po_lstm_cell_fwd_sk(float* gates, const float* rec, int32_t splits, const float* c_prev, float* c_out,
                        float* h_out, float* y_out, int64_t y_ld, int64_t batch, int64_t hidden, void* stream);
int po_lstm_cell_bwd_sk(const float* act, const float* c_prev, const float* c, const float* dy, int64_t dy_ld,
                        const float* dh_rec, int32_t splits, float* dc, float* dgates, int64_t batch, int64_t hidden,
                        void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PIPEOPTIM_H_ */
