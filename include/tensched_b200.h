/*
 * tensched_b200.h - C-ABI of the B200-native V(s) scoring path.
 *
 * This is the drop-in boundary for the reference package `tensched`
 * (arXiv 2011.14486 reconstruction).  Every entry point takes plain
 * pointers and sizes; device memory is owned by the context; host buffers
 * are borrowed for the duration of the call.  Results never depend on the
 * batch size or on how a batch is chunked (value_model.py:33).
 *
 * Reference interfaces replaced (paths relative to /root/reference/pkg/src/tensched):
 *   ts_lstm_forward        <- backend.lstm_forward / _recurrent_cy.lstm_forward
 *                             (backend.py:26, _recurrent_cy.pyx:20-66)
 *   ts_lstm_backward       <- backend.lstm_forward_cached + lstm_backward
 *                             (backend.py:15-16, _recurrent_np.py:38-96)
 *   ts_featurize_states    <- featurizer.featurize_state + normalize
 *                             (featurizer.py:68-107, :136-137)
 *   ts_score_states        <- value_model.predict_states (value_model.py:129-155),
 *                             the V-callable protocol of search.py:3-8
 *   ts_candidates          <- schedule_space.candidate_actions (schedule_space.py:379-452)
 *   ts_greedy              <- search.greedy_schedule (search.py:90-112), fused:
 *                             candidates -> featurize -> V -> (noise) -> argmin per layer
 *   ts_beam                <- search.beam_search (search.py:115-133), fused per layer
 *   ts_score_children      <- one layer step of greedy_schedule for any parent (search.py:97-110)
 *   ts_train_*             <- value_model.gradients / train (value_model.py:182-293)
 *   ts_params_upload       <- value_model.ValueModelParams / load (value_model.py:37-70, :332-376)
 *   ts_pipeline_upload     <- pipeline_ir.Pipeline (pipeline_ir.py:116-161) as a flat descriptor
 *
 * Errors: every function returns a ts_status; ts_last_error() gives the
 * message.  The Python layer maps TS_ERR_ILLEGAL to IllegalActionError and
 * the rest to PipelineError subclasses (pipeline_ir.py:20-37).
 */
#ifndef TENSCHED_B200_H
#define TENSCHED_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TS_ABI_VERSION 1

#define TS_FEATURE_WIDTH 16 /* featurizer.py:20 */
#define TS_MAX_PURE 4       /* pure dims per stage */
#define TS_MAX_RED 4        /* reduction dims per stage */
#define TS_MAX_LOOPS 8      /* loops per stage after splits */
#define TS_MAX_STAGES 512

typedef enum ts_status {
  TS_OK = 0,
  TS_ERR_ARG = 1,       /* bad argument / shape */
  TS_ERR_CUDA = 2,      /* CUDA runtime failure */
  TS_ERR_PIPELINE = 3,  /* descriptor outside the supported envelope */
  TS_ERR_ILLEGAL = 4,   /* decision record illegal for its state */
  TS_ERR_OVERFLOW = 5,  /* integer exceeded 256 bits (invocations etc.) */
  TS_ERR_SELFTEST = 6,  /* device log2 does not match host libm */
  TS_ERR_NO_DEVICE = 7, /* no sm_100 device */
  TS_ERR_STATE = 8      /* call order (no params / no pipeline) */
} ts_status;

/* One scheduling decision (a LayerSchedule, schedule_space.py:37-56) for
 * the stage at the matching position of schedule order (consumers first,
 * pipeline_ir.py:207-213).  16 bytes.
 *   split[k]  split factor of pure dim k (0 = unsplit)
 *   order[j]  loop ids outermost first: pure dim k -> 2k (whole or outer),
 *             2k+1 (inner); reduction dim r -> 8+r; 0xFF pads
 *   vec       vectorize width; flags bit0 = parallel, bit1 = store_at is
 *             the compute site (else Root); anchor = compute_at loop level
 *             in the sole consumer's nest, -1 = Root. */
typedef struct ts_decision {
  uint8_t split[TS_MAX_PURE];
  uint8_t order[TS_MAX_LOOPS];
  uint8_t n_loops;
  uint8_t vec;
  uint8_t flags;
  int8_t anchor;
} ts_decision;

#define TS_FLAG_PARALLEL 1u
#define TS_FLAG_STORE_AT 2u

/* Scoring precision. EXACT: fp64 with the Cython kernel's operation order
 * (_recurrent_cy.pyx:38-65).  FAST: fp32-accurate tensor-core path
 * (tcgen05, split-fp16 operands, fp32 TMEM accumulators). */
#define TS_MODE_EXACT 0
#define TS_MODE_FAST 1
/* Operand range of the tensor-core leg.  An operand x is split into
 * hi = fp16(x), lo = fp16(x - hi): 22 significant bits while |x| stays below
 * fp16's 65,504, absolute error |x| 2^-22.  A state whose normalized features
 * leave [-TS_FAST_RANGE, TS_FAST_RANGE] (a sigma-floored normalizer: 1e-6
 * puts a differing value near 1e6; a pipeline far outside the training data)
 * is rescored on the exact leg, and a pipeline whose unscheduled rows leave
 * it is scored on the exact leg altogether, so TS_MODE_FAST never returns a
 * V computed from clipped or infinite operands.  2^12 keeps a 16x margin
 * below the fp16 overflow and bounds the operand error at 1e-3; v0 reaches
 * |x| <= ~600 on any state of the benchmark networks (feature 13, sigma
 * 0.238), so the guard never fires on it. */
#define TS_FAST_RANGE 4096.0f

typedef struct ts_ctx ts_ctx;

int ts_abi_version(void);
const char* ts_last_error(ts_ctx* ctx);

/* Create a context on `device`; runs the device-log2 self-test against the
 * host libm (hard part 3) and fails with TS_ERR_SELFTEST on a
 * mismatch. */
int ts_ctx_create(int device, ts_ctx** out);
void ts_ctx_destroy(ts_ctx* ctx);

/* Flat pipeline descriptor (layout documented in DESIGN.md and built by
 * paper_2011_14486_b200/pipeline.py); returns a pipeline id. */
int ts_pipeline_upload(ts_ctx* ctx, const int64_t* desc, int64_t n_words, int* pipeline_id);

/* Value-model parameters (value_model.py:37-46), row-major f64:
 * Wx[16][4H], Wh[H][4H], b[4H], w[H]; normalizer mean/std[16]. */
int ts_params_upload(ts_ctx* ctx, int hidden, const double* Wx, const double* Wh,
                     const double* b, const double* w, double b_out, double target_scale,
                     const double* norm_mean, const double* norm_std);

/* featurize_state (+ normalize when `normalized`): states are ragged runs of
 * decisions, state i = records[offsets[i] .. offsets[i+1]).  Output
 * [n][T][16] f64 (T = n_stages, rows in topological order). Bit-exact. */
int ts_featurize_states(ts_ctx* ctx, int pipeline_id, const ts_decision* records,
                        const int64_t* offsets, int64_t n_states, int normalized,
                        double* out);

/* predict_states: V = exp(raw + target_scale) per state, host buffers. */
int ts_score_states(ts_ctx* ctx, int pipeline_id, const ts_decision* records,
                    const int64_t* offsets, int64_t n_states, int mode, double* out_v);

/* Packed wire format for host callers: one 64-bit word per decision
 *   bits 0-31 loop ids (4 bits each, position j at 4j), 32-35 n_loops,
 *   36-51 split code per pure dim (4 bits: index into
 *   {none,2,3,4,5,6,7,8,12,16,24,32,48,64,128,255}), 52-53 vec code
 *   (1,4,8,16), 54-55 flags, 56-59 compute_at level + 1 (0 = root)
 * and one u8 depth per state (offsets are rebuilt on the device): half the
 * PCIe bytes of ts_score_states. */
int ts_score_states_packed(ts_ctx* ctx, int pipeline_id, const uint64_t* packed, const uint8_t* depths,
                           int64_t n_states, int mode, double* out_v);

/* Action-code wire format: one 16-bit code per decision for decisions in
 * candidate_actions' space (schedule_space.py:379-452; SPLIT_FACTORS (8, 32),
 * VEC_WIDTHS (1, 8), compute_at levels 0..2, orders from _order_options
 * :361-376), decoded against the decision's stage on the device inside the
 * featurizer:
 *   bits 0-1  compute_at level + 1 (0 = root)
 *   bits 2-3  split of splittable dim 0 (dims[-2:][0]): 0 none, 1 -> 8, 2 -> 32
 *   bits 4-5  split of splittable dim 1 (dims[-2:][1], if the stage has two)
 *   bit  6    order placement: reduction loops outermost (else innermost)
 *   bit  7    order swap: last two loops exchanged
 *   bit  8    vectorize 8 (else 1)
 *   bit  9    parallel
 *   bit  10   store_at = compute_at site
 *   bits 11-15 zero
 * plus one u8 depth per state: 1/8 of the PCIe bytes of ts_score_states.
 * Callers fall back to the packed or record formats for other decisions. */
#define TS_CODE_SPACE 2048  /* 11-bit action codes */
int ts_score_states_coded(ts_ctx* ctx, int pipeline_id, const uint16_t* codes, const uint8_t* depths,
                          int64_t n_states, int mode, double* out_v);

/* Records -> action codes on the host (inverse of ts_decode_codes);
 * TS_ERR_ILLEGAL when a decision lies outside the code space. */
int ts_encode_codes(ts_ctx* ctx, int pipeline_id, const ts_decision* records, const uint8_t* depths,
                    int64_t n_states, uint16_t* out_codes);

/* Device-resident records -> action codes (the inverse of the decoding);
 * TS_ERR_ILLEGAL when a decision lies outside the code space. */
int ts_encode_codes_device(ts_ctx* ctx, int pipeline_id, const ts_decision* d_records, const int64_t* d_offsets,
                           int64_t n_states, uint16_t* d_codes);

/* Decodes action codes to records on the host (state i's decision j belongs
 * to schedule position j); for tests and tools.  Host-only contexts work. */
int ts_decode_codes(ts_ctx* ctx, int pipeline_id, const uint16_t* codes, const uint8_t* depths,
                    int64_t n_states, ts_decision* out_records);

/* Same with device-resident inputs/outputs (pointers into the context's
 * device), stream-ordered on the context stream. */
int ts_score_states_device(ts_ctx* ctx, int pipeline_id, const ts_decision* d_records,
                           const int64_t* d_offsets, int64_t n_states, int64_t n_records,
                           int mode, double* d_out_v);

/* ts_score_states_coded with device-resident inputs: d_codes (16-bit
 * action codes, 2 B per decision) and d_offsets (n_states + 1), stream-
 * ordered on the context stream. */
int ts_score_states_coded_device(ts_ctx* ctx, int pipeline_id, const uint16_t* d_codes,
                                 const int64_t* d_offsets, int64_t n_states, int64_t n_records,
                                 int mode, double* d_out_v);

/* backend.lstm_forward(X, Wx, Wh, b, w, b_out) -> raw (backend.py:26). */
int ts_lstm_forward(ts_ctx* ctx, const double* X, int64_t B, int64_t T, int64_t F,
                    const double* Wx, const double* Wh, const double* b, const double* w,
                    int64_t H, double b_out, int mode, double* raw_out);

/* backend.lstm_backward(X, Wx, Wh, w, cache, d_raw) -> (dWx, dWh, db, dw,
 * db_out) (backend.py:16, _recurrent_np.py:62-96): gradients of
 * sum_b d_raw[b] * raw[b] for the batch X [B][T][F] (F = 16, C-contiguous).
 * The forward is recomputed on the device (the reference's per-timestep
 * activation cache, _recurrent_np.py:38-59, is the host's opaque handle and
 * carries b and b_out).  fp64 throughout.  grad_out: [dWx F x 4H | dWh
 * H x 4H | db 4H | dw H | db_out], 4H(F+H+1)+H+1 doubles. */
int ts_lstm_backward(ts_ctx* ctx, const double* X, int64_t B, int64_t T, int64_t F,
                     const double* Wx, const double* Wh, const double* b, const double* w,
                     int64_t H, double b_out, const double* d_raw, double* grad_out);

/* candidate_actions for the state given by `prefix` (n_prefix decisions). */
int ts_candidates(ts_ctx* ctx, int pipeline_id, const ts_decision* prefix, int64_t n_prefix,
                  ts_decision* out, int64_t capacity, int64_t* n_out);

/* check_action (schedule_space.py:288-347) for decision `a` after `prefix`:
 * TS_OK if legal, TS_ERR_ILLEGAL with the violated invariant otherwise. */
int ts_check_action(ts_ctx* ctx, int pipeline_id, const ts_decision* prefix, int64_t n_prefix,
                    const ts_decision* a);

/* Fused greedy_schedule: returns the n_stages decisions and the visited
 * candidate count.  epsilon > 0 applies the multiplicative noise of
 * search.py:104-109 from the splitmix64 stream *rng_state (advanced by one
 * draw per candidate, exactly as SearchRng).  With H = 32 the calling
 * thread polls each layer's result in mapped pinned memory (a busy wait,
 * like a spinning stream sync) and checks the stream for errors while it
 * waits; the call returns with the context's stream idle. */
int ts_greedy(ts_ctx* ctx, int pipeline_id, double epsilon, uint64_t* rng_state,
              ts_decision* out_decisions, int64_t* visited, double* out_best_v);

/* Dedup statistics of the last ts_greedy call on this context: candidates
 * visited and distinct children feature rows among them (visited / distinct
 * is the dedup factor).  With H = 32 every child runs its own exact LSTM in
 * the one-kernel layer (identical rows give identical V, so the argmin is
 * unaffected) and the distinct count comes from the rows' 64-bit hashes
 * after the search; otherwise children with bit-identical rows share one
 * LSTM and the count is exact. */
int ts_greedy_stats(ts_ctx* ctx, int64_t* visited, int64_t* distinct);

/* One layer step for an arbitrary parent state (the children
 * half of greedy_schedule, search.py:97-110): the parent's n_parent decisions
 * (schedule order) and n_children (<= 4096) candidate decisions for its next
 * stage (checked like check_action, schedule_space.py:288-347).  Only the new
 * row of every child is featurized; bit-identical rows are scored once; the
 * exact LSTM runs from the shared unscheduled prefix over the T - s timesteps
 * a child differs in.  out_v (optional, [n_children]): noise-free V of every
 * child.  out_best (optional): argmin by (V * (1 + U(-eps, eps)), index)
 * with one splitmix64 draw per child from *rng_state (advanced by
 * n_children when eps > 0); out_best_v its (noisy) value.  At least one of
 * out_v / out_best. */
int ts_score_children(ts_ctx* ctx, int pipeline_id, const ts_decision* parent, int64_t n_parent,
                      const ts_decision* children, int64_t n_children, double epsilon, uint64_t* rng_state,
                      double* out_v, int64_t* out_best, double* out_best_v);

/* beam_search(prefix, model_value(params), width) (search.py:115-133),
 * fused per layer: every frontier state's children enumerated natively,
 * their new rows, per-parent dedup and the exact fp64 LSTM in one device
 * pass, ranked by (V, index); the `width` best form the next frontier.
 * out_decisions: the T decisions of the returned complete state (the
 * prefix's first); visited: children scored; out_v: its V.  Hidden size 32.
 * Width 1 is the noiseless greedy from the prefix. */
int ts_beam(ts_ctx* ctx, int pipeline_id, const ts_decision* prefix, int64_t n_prefix, int width,
            ts_decision* out_decisions, int64_t* visited, double* out_v);

/* Device-side random partial states (the synthetic sweep generator): state i
 * walks uniformly over candidate_actions with SearchRng(seed0 + i) after
 * drawing its depth d = randrange(T) + 1 (search.py:136-142 variant).
 * Writes ragged records (capacity n_states*T) and n_states+1 offsets into
 * device buffers; *n_records receives the total. */
int ts_generate_states_device(ts_ctx* ctx, int pipeline_id, uint64_t seed0, int64_t n_states,
                              ts_decision* d_records, int64_t* d_offsets, int64_t* n_records);

/* Normalized f64 rows of the scheduled stages of device-resident states
 * (rows[offsets[i] + j] = decision j of state i), and the [T][16] rows of
 * the all-unscheduled state (normalized or raw, host or device pointer). */
int ts_featurize_rows_device(ts_ctx* ctx, int pipeline_id, const ts_decision* d_records,
                             const int64_t* d_offsets, int64_t n_states, double* d_rows);
int ts_init_rows(ts_ctx* ctx, int pipeline_id, int normalized, double* out);

/* Complete random schedules (search.random_schedule, search.py:136-142):
 * schedule i starts from splitmix state seed0 + i*stride (stride 1: SearchRng(seed0+i);
 * stride T*0x9E3779B97F4A7C15: consecutive schedules of one shared SearchRng, each
 * drawing exactly T times, as learner.bootstrap does); records at d_records[i*T ..). */
int ts_generate_schedules_device(ts_ctx* ctx, int pipeline_id, uint64_t seed0, uint64_t stride, int64_t n,
                                 ts_decision* d_records);

/* cost_oracle.benchmark (cost_oracle.py:313-357) for complete schedules:
 * total_millis as 4 little-endian u64 limbs per schedule.  cost_desc: per
 * stage (topological order) flops_per_point, n_inputs, then 4 input slots of
 * [producer stage (-1 = buffer), elem bytes, n_maps, 6 x (consumer dim,
 * stride, window)]; machine: flop_cost, mem_byte_cost, cache_byte_cost,
 * cache_size, cores, task_overhead. */
int ts_benchmark(ts_ctx* ctx, int pipeline_id, const int64_t* cost_desc, int64_t n_words,
                 const uint64_t* machine, const ts_decision* records, const int64_t* offsets, int64_t n,
                 uint64_t* out_millis);

/* ---- V training (value_model.train / gradients, value_model.py:182-293;
 * lstm_forward_cached / lstm_backward, _recurrent_np.py:38-96).
 * Dataset: sample i's input at timestep t is init[init_base[i] + t] when
 * t < Tlen[i] - depth[i] (unscheduled stages) and rows[row_base[i] + Tlen[i]-1-t]
 * otherwise (scheduled rows in decision order; all prefixes of a schedule
 * share its rows).  Rows are normalized f64.  device_ptrs = 1: the arrays are
 * device pointers (copied device-to-device).  Parameters are a flat f64
 * vector [Wx 16x4H | Wh Hx4H | b 4H | w H | b_out] resident on the device. */
int ts_train_load(ts_ctx* ctx, const double* rows, int64_t n_rows, const double* init, int64_t n_init,
                  const int64_t* row_base, const int32_t* init_base, const int32_t* Tlen,
                  const int32_t* depth, const double* logt, int64_t N, int hidden, int device_ptrs);
int ts_train_set_params(ts_ctx* ctx, const double* flat, int64_t n);
int ts_train_get_params(ts_ctx* ctx, double* flat, int64_t n);
/* gradient of the loss over idx[0..B) of a minibatch of global size n_total
 * into d_grad (device pointer; null = context buffer); raw_out optional. */
int ts_train_grads(ts_ctx* ctx, const int32_t* idx, int64_t B, int64_t n_total, double target_scale,
                   double* d_grad, double* raw_out);
/* _clip (global L2 incl. b_out) + SGD with the gradient in d_grad. */
int ts_train_apply(ts_ctx* ctx, const double* d_grad, double lr, double clip_norm, double* norm_out);
/* Gradient arithmetic of ts_train_grads.  TS_TRAIN_EXACT (default): fp64
 * throughout, the reference's trajectory (value_model.gradients,
 * value_model.py:182-210).  TS_TRAIN_TC: fp64 forward/BPTT recurrences with
 * the weight-gradient contraction on the tensor cores (3xTF32, fp32
 * accumulation in TMEM, fused into BPTT; hidden size 32 only). */
#define TS_TRAIN_EXACT 0
#define TS_TRAIN_TC 1
/* TS_TRAIN_TCF: the forward and BPTT recurrences on the tensor cores too
 * (split-fp16 UMMAs, fp32 accumulation, MUFU gates, a power-of-two scaled
 * backward; ts_train_tc.cuh) - fp32-accurate gradients, not the fp64
 * trajectory; hidden size 32 only. */
#define TS_TRAIN_TCF 2
int ts_train_set_mode(ts_ctx* ctx, int mode);
/* raw scores of dataset entries idx[0..n) (for _eval_split). */
int ts_train_forward(ts_ctx* ctx, const int32_t* idx, int64_t n, double* raw_out);

/* Synchronize the context stream; cudaStream_t of the context (as void*). */
int ts_sync(ts_ctx* ctx);
void* ts_stream(ts_ctx* ctx);

/* Number of this library's kernel launches since context creation. */
int64_t ts_launch_count(ts_ctx* ctx);

/* Kernel-class timing (CUDA events on the context stream around each
 * launch, for bench.py): classes below; ms[k] = summed duration, counts[k]
 * = launches since the last reset. */
#define TS_K_FEATURIZE 0
#define TS_K_LSTM_EXACT 1
#define TS_K_LSTM_FAST 2
#define TS_K_OTHER 3
#define TS_KCLASSES 4
int ts_set_timing(ts_ctx* ctx, int on);
int ts_kernel_times(ts_ctx* ctx, double* ms, int64_t* counts, int reset);

#ifdef __cplusplus
}
#endif
#endif
