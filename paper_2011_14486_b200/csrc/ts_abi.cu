// ts_abi.cu - the C-ABI (include/tensched_b200.h): context, descriptor and
// parameter upload, scoring entry points and the native greedy driver.
//
// The greedy driver (ts_greedy) is the fused replacement of
// search.greedy_schedule (search.py:90-112): per layer it enumerates the
// candidates on the host (the integer nest math is tiny) and launches ONE
// kernel (hidden size 32) whose CTAs featurize their child's new row and run
// the exact LSTM from the shared prefix, the last CTA reducing the argmin
// and installing the winner's row; only {v, index, status} comes back,
// through mapped host memory.  Only the winner is "applied" (SURVEY.md 7,
// hard part 7).
#include <cuda_runtime.h>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif

#include <cub/device/device_scan.cuh>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <memory>
#include <string>
#include <vector>

#include "ts_core.cuh"
#include "ts_kernels.cuh"
#include "ts_lstm_tc.cuh"
#include "ts_train.cuh"
#include "ts_train_tc.cuh"
#include "ts_cost.cuh"

using namespace ts;

namespace {

constexpr int64_t DESC_HEADER = 4;
constexpr int64_t DESC_STAGE_WORDS = 48;

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  cudaError_t reserve(size_t n) {
    if (n <= bytes) return cudaSuccess;
    // growth: work queued on any of the context's streams may still read the
    // old buffer; wait for the device explicitly rather than relying on
    // cudaFree's implicit synchronization
    if (p) {
      cudaDeviceSynchronize();
      cudaFree(p);
    }
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, n);
    if (e == cudaSuccess) bytes = n;
    // TS_POISON (tests): new allocations start as all-ones bytes (NaN as
    // doubles, -1 as integers), so a read of never-written memory shows up
    if (e == cudaSuccess && poison()) {
      e = cudaMemset(p, 0xFF, n);
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
    }
    return e;
  }
  static bool poison() {
    static const bool on = getenv("TS_POISON") != nullptr;
    return on;
  }
  // Growth of a buffer that kernels queued on `user` may still read: wait
  // for that stream before the old allocation is released (explicitly, not
  // through cudaFree's implicit device synchronization).
  cudaError_t reserve(size_t n, cudaStream_t user) {
    if (n <= bytes) return cudaSuccess;
    if (p) {
      cudaError_t e = cudaStreamSynchronize(user);
      if (e != cudaSuccess) return e;
    }
    return reserve(n);
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct HostBuf {
  void* p = nullptr;
  size_t bytes = 0;
  ~HostBuf() {
    if (p) cudaFreeHost(p);
  }
  cudaError_t reserve(size_t n) {
    if (n <= bytes) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMallocHost(&p, n);
    if (e == cudaSuccess) bytes = n;
    return e;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct PipelineSlot {
  std::unique_ptr<PipelineDesc> h;
  DevBuf d;          // PipelineDesc
  DevBuf init_raw;   // [T][16]
  DevBuf init_norm;  // [T][16]
  DevBuf pre_exact;  // [(T+1)][72]
  DevBuf pre_fast;   // fast-path prefix
  DevBuf code_table; // [T][TS_CODE_SPACE + 1] decoded action codes (built on first coded call)
  uint64_t rows_version = 0;  // params version the init rows / prefix belong to
  uint64_t fast_version = 0;
  bool fast_safe = true;      // unscheduled rows inside the tensor-core operand range
};

}  // namespace

struct ts_ctx {
  uint64_t greedy_seq = 0;  // fused greedy: sequence number of the last layer result
  int device = 0;
  cudaStream_t stream = nullptr;       // compute
  cudaStream_t copy_stream = nullptr;  // host->device transfers of ts_score_states*
  cudaStream_t d2h_stream = nullptr;   // device->host results of ts_score_states_coded
  std::string err;
  std::vector<std::unique_ptr<PipelineSlot>> pipes;
  // parameters
  int hidden = 0;
  uint64_t params_version = 0;
  double b_out = 0.0, target_scale = 0.0;
  DevBuf Wx, Wh, b, w, mean, stdv;
  DevBuf fast_w;  // packed tensor-core weights
  // scratch
  DevBuf status, records, offsets, rows, out, reps, raw, nest, tmp, tmp2, scan_tmp;
  HostBuf h_stage, h_out;
  int64_t launches = 0;
  int sm_count = 148;
  bool tc_attr_set = false;
  bool exact_attr_set = false;
  bool exact2_attr_set = false;
  bool tr_tc_attr_set = false;
  // optional per-kernel-class timing (bench.py): events around launches on
  // the context stream, resolved at the next host synchronization
  bool timing = false;
  struct Pending {
    int cls;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> event_pool;
  double kms[TS_KCLASSES] = {0};
  int64_t kcount[TS_KCLASSES] = {0};
  // V training (ts_train_*)
  int tr_H = 0, tr_Tmax = 0;
  int tr_mode = TS_TRAIN_EXACT;
  int64_t tr_N = 0;
  DevBuf tr_X, tr_T, tr_logt, tr_P, tr_grad, tr_cache, tr_dz, tr_raw, tr_draw, tr_batch, tr_norm, tr_partial,
      tr_pvalid;
  DevBuf tile_ctr;  // k_lstm_tc's dynamic tile counter
  tr::Data tr_data{};
  // second scoring lane (coded wire path, FAST): alternate chunks run on
  // their own stream with their own scratch, so one chunk's kernels fill
  // the SMs the other chunk's kernel tails leave idle
  cudaStream_t stream2 = nullptr;
  DevBuf reps2, rows2, tile_ctr2, scan_tmp2;
  DevBuf resc, resc2;  // k_rescore_exact scratch rows, per lane
  DevBuf bk_X, bk_meta, bk_P;  // ts_lstm_backward: the batch, its layout, params + gradient
  DevBuf gstat;                 // ts_greedy: distinct children rows (device counter)
  DevBuf ghash;                 // ts_greedy: per-layer children row hashes [T][4096] + counts [T]
  ChildRow child_row{};         // ts_greedy: the fused layer's launch parameters
  DevBuf beam_ticket;           // ts_beam: the layer kernel's last-block ticket
  DevBuf trc_img;               // TS_TRAIN_TCF: per-step packed weight images
  bool trc_attr_set = false;
  DevBuf beam_rows;             // ts_beam: frontier state rows, double-buffered
  HostBuf h_sel;                // ts_beam: the next frontier's (parent, child) pairs
  unsigned long long greedy_distinct = 0;
  int64_t greedy_visited = 0;
  bool tr_group_attr_set = false;
};

// fused greedy: per layer up to this many children; their row hashes for
// every layer of the largest pipeline plus the per-layer counts and ticket
constexpr int kGreedyMaxChildren = 4096;
static size_t greedy_hash_bytes() {
  return sizeof(unsigned long long) * (size_t)TS_MAX_STAGES * kGreedyMaxChildren +
         sizeof(int) * (size_t)(TS_MAX_STAGES + 1);
}

namespace {
void swap_buf(DevBuf& a, DevBuf& b) {
  std::swap(a.p, b.p);
  std::swap(a.bytes, b.bytes);
}
// Swaps the second lane's stream and scratch into the context for a scope.
struct LaneSwap {
  ts_ctx* c;
  bool on;
  LaneSwap(ts_ctx* ctx, bool alt) : c(ctx), on(alt) { swap_all(); }
  ~LaneSwap() { swap_all(); }
  void swap_all() {
    if (!on) return;
    std::swap(c->stream, c->stream2);
    swap_buf(c->reps, c->reps2);
    swap_buf(c->rows, c->rows2);
    swap_buf(c->tile_ctr, c->tile_ctr2);
    swap_buf(c->scan_tmp, c->scan_tmp2);
    swap_buf(c->resc, c->resc2);
  }
};
}  // namespace

namespace {

int fail(ts_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

int cuda_fail(ts_ctx* c, cudaError_t e, const char* where) {
  return fail(c, TS_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define TS_CUDA(call)                                       \
  do {                                                      \
    cudaError_t _e = (call);                                \
    if (_e != cudaSuccess) return cuda_fail(ctx, _e, #call); \
  } while (0)

#define TS_LAUNCHED()                                          \
  do {                                                         \
    ++ctx->launches;                                           \
    cudaError_t _e = cudaGetLastError();                       \
    if (_e != cudaSuccess) return cuda_fail(ctx, _e, "launch"); \
  } while (0)

#define TS_NEED_DEVICE()                                                        \
  do {                                                                          \
    if (ctx->device < 0) return fail(ctx, TS_ERR_NO_DEVICE, "host-only context"); \
  } while (0)

const char* status_name(int s) {
  switch (s) {
    case TS_ERR_ARG: return "bad argument";
    case TS_ERR_PIPELINE: return "pipeline outside the supported envelope";
    case TS_ERR_ILLEGAL: return "illegal decision record for its state";
    case TS_ERR_OVERFLOW: return "integer exceeded 256 bits";
    default: return "error";
  }
}

cudaEvent_t take_event(ts_ctx* ctx) {
  cudaEvent_t e;
  if (!ctx->event_pool.empty()) {
    e = ctx->event_pool.back();
    ctx->event_pool.pop_back();
  } else {
    cudaEventCreate(&e);
  }
  return e;
}

// RAII timer: records start/stop events around one launch when timing is on.
struct KTimer {
  ts_ctx* ctx;
  int cls;
  cudaEvent_t a = nullptr;
  KTimer(ts_ctx* c, int k) : ctx(c), cls(k) {
    if (ctx->timing) {
      a = take_event(ctx);
      cudaEventRecord(a, ctx->stream);
    }
  }
  ~KTimer() {
    if (a) {
      cudaEvent_t b = take_event(ctx);
      cudaEventRecord(b, ctx->stream);
      ctx->pending.push_back({cls, a, b});
    }
  }
};

void resolve_timers(ts_ctx* ctx) {
  for (auto& p : ctx->pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
      ctx->kms[p.cls] += ms;
      ctx->kcount[p.cls] += 1;
    }
    ctx->event_pool.push_back(p.a);
    ctx->event_pool.push_back(p.b);
  }
  ctx->pending.clear();
}

// Reads back and clears the device status word.
int check_device_status(ts_ctx* ctx) {
  int st = 0;
  TS_CUDA(cudaMemcpyAsync(&st, ctx->status.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  TS_CUDA(cudaStreamSynchronize(ctx->stream));
  resolve_timers(ctx);
  if (st) {
    TS_CUDA(cudaMemsetAsync(ctx->status.p, 0, sizeof(int), ctx->stream));
    return fail(ctx, st, std::string("device: ") + status_name(st));
  }
  return TS_OK;
}

PipelineSlot* get_pipe(ts_ctx* ctx, int id) {
  if (id < 0 || id >= (int)ctx->pipes.size()) return nullptr;
  return ctx->pipes[id].get();
}

LstmW lstm_weights(ts_ctx* ctx) {
  LstmW W;
  W.Wx = ctx->Wx.as<double>();
  W.Wh = ctx->Wh.as<double>();
  W.b = ctx->b.as<double>();
  W.w = ctx->w.as<double>();
  W.H = ctx->hidden;
  return W;
}

// Dynamic shared memory for the featurize kernels' nest slots.
size_t slot_smem(PipelineSlot* P, int block) {
  const int ns = P->h->n_slots > 0 ? P->h->n_slots : 1;
  return (size_t)ns * sizeof(Nest) * block;
}

// Init rows + exact prefix for the current parameters.
int ensure_pipe_ready(ts_ctx* ctx, PipelineSlot* P) {
  if (!ctx->params_version) return fail(ctx, TS_ERR_STATE, "no parameters uploaded");
  if (P->rows_version == ctx->params_version) return TS_OK;
  const int T = P->h->n_stages;
  TS_CUDA(P->init_raw.reserve(sizeof(double) * T * F));
  TS_CUDA(P->init_norm.reserve(sizeof(double) * T * F));
  TS_CUDA(P->pre_exact.reserve(sizeof(double) * (T + 1) * 72));
  k_init_rows<<<(T + 127) / 128, 128, 0, ctx->stream>>>(P->d.as<PipelineDesc>(), ctx->mean.as<double>(),
                                                       ctx->stdv.as<double>(), P->init_raw.as<double>(),
                                                       P->init_norm.as<double>());
  TS_LAUNCHED();
  const size_t pre_smem = prefix_mw_smem(T);
  if (ctx->hidden == 32 && pre_smem <= 200 * 1024) {  // the four-warp step (H = 32)
    if (pre_smem > 40 * 1024)  // with the static 4 KB
      TS_CUDA(cudaFuncSetAttribute(k_prefix_exact_mw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pre_smem));
    k_prefix_exact_mw<<<1, 128, pre_smem, ctx->stream>>>(lstm_weights(ctx), P->init_norm.as<double>(), T,
                                                         ctx->b_out, P->pre_exact.as<double>());
  } else {
    k_prefix_exact<<<1, 32, 0, ctx->stream>>>(lstm_weights(ctx), P->init_norm.as<double>(), T,
                                              ctx->b_out, P->pre_exact.as<double>());
  }
  TS_LAUNCHED();
  P->rows_version = ctx->params_version;
  return TS_OK;
}

int self_test(ts_ctx* ctx) {
  // Values: all ints in [1, 2^16], known non-correctly-rounded ints, and a
  // spread of doubles; compare device glibc_log2 and the host port against
  // the host libm log2 bit for bit.
  std::vector<double> xs;
  for (int i = 1; i <= 65536; ++i) xs.push_back((double)i);
  const double extra[] = {1621.0, 3242.0, 57803.0, 0.999, 1.0001, 1.5, 0.75, 3.0e-3, 1.0e30, 2.0e40};
  for (double e : extra) xs.push_back(e);
  uint64_t st = 0x1234567ull;
  for (int i = 0; i < 16384; ++i) {
    const uint64_t z = splitmix_next(st);
    const double u = (double)(z >> 11) * 1.1102230246251565e-16;
    xs.push_back(std::exp2(u * 120.0 - 20.0));
    xs.push_back(1.0 + (u - 0.5) * 0.1);
  }
  const size_t n = xs.size();
  for (size_t i = 0; i < n; ++i) {
    const double want = std::log2(xs[i]);
    if (as_u64(glibc_log2(xs[i])) != as_u64(want)) {
      char buf[160];
      snprintf(buf, sizeof buf, "host log2 port mismatch at %.17g: libm build differs from glibc 2.39",
               xs[i]);
      return fail(ctx, TS_ERR_SELFTEST, buf);
    }
  }
  DevBuf dx, dy;
  TS_CUDA(dx.reserve(n * 8));
  TS_CUDA(dy.reserve(n * 8));
  TS_CUDA(cudaMemcpy(dx.p, xs.data(), n * 8, cudaMemcpyHostToDevice));
  k_log2_selftest<<<(int)((n + 255) / 256), 256>>>(dx.as<double>(), dy.as<double>(), (int64_t)n);
  TS_LAUNCHED();
  std::vector<double> ys(n);
  TS_CUDA(cudaMemcpy(ys.data(), dy.p, n * 8, cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < n; ++i) {
    if (as_u64(ys[i]) != as_u64(std::log2(xs[i]))) {
      char buf[160];
      snprintf(buf, sizeof buf, "device log2 mismatch at %.17g", xs[i]);
      return fail(ctx, TS_ERR_SELFTEST, buf);
    }
  }
  // glibc exp / tanh ports (the exact leg's transcendentals): the host port
  // and the device against the host libm, bit for bit, over the LSTM's
  // ranges (gate pre-activations, cell states, V exponents), the branch
  // boundaries of both routines and the special values
  {
    std::vector<double> ts;
    uint64_t s2 = 0x9E3779B97F4A7C15ull;
    for (int i = 0; i < 200000; ++i) {
      const uint64_t z = splitmix_next(s2);
      const double u = (double)(z >> 11) * 1.1102230246251565e-16;
      switch (i % 5) {
        case 0: ts.push_back((u - 0.5) * 60.0); break;                        // gates, cells
        case 1: ts.push_back((u - 0.5) * 1500.0); break;                      // |x| up to 750: special cases
        case 2: ts.push_back(std::ldexp(u, -(int)(z % 60)) * ((z >> 7) & 1 ? -1 : 1)); break;  // tiny
        case 3: ts.push_back((u - 0.5) * 4.0); break;                         // |x| < 2: tanh's two forms
        default: ts.push_back(std::ldexp(1.0, (int)(z % 20)) * (1.0 + (u - 0.5) * 1e-6) *
                              ((z >> 9) & 1 ? -1 : 1));                        // near powers of two
      }
    }
    const double special[] = {0.0, -0.0, 1.0, -1.0, 22.0, -22.0, 0.34657359027997264, 1.0397207708399179,
                              38.816242111356935, 512.0, -512.0, 709.78, -745.1, 1e-300, -1e-300,
                              5e-324, 1.0 / 0.0, -1.0 / 0.0, 2.0, 44.0, -44.0, 0.5, -0.25};
    for (double v : special) ts.push_back(v);
    const size_t m = ts.size();
    for (size_t i = 0; i < m; ++i) {
      if (as_u64(glibc_exp(ts[i])) != as_u64(std::exp(ts[i])) || as_u64(glibc_tanh(ts[i])) != as_u64(std::tanh(ts[i]))) {
        char buf[160];
        snprintf(buf, sizeof buf, "host exp/tanh port mismatch at %.17g: libm build differs from glibc 2.39", ts[i]);
        return fail(ctx, TS_ERR_SELFTEST, buf);
      }
    }
    DevBuf tx, ty;
    TS_CUDA(tx.reserve(m * 8));
    TS_CUDA(ty.reserve(m * 24));
    TS_CUDA(cudaMemcpy(tx.p, ts.data(), m * 8, cudaMemcpyHostToDevice));
    k_glibc_selftest<<<(int)((m + 255) / 256), 256>>>(tx.as<double>(), ty.as<double>(), (int64_t)m);
    TS_LAUNCHED();
    std::vector<double> yy(3 * m);
    TS_CUDA(cudaMemcpy(yy.data(), ty.p, m * 24, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < m; ++i) {
      const uint64_t th = as_u64(std::tanh(ts[i]));
      if (as_u64(yy[3 * i]) != as_u64(std::exp(ts[i])) || as_u64(yy[3 * i + 1]) != th ||
          as_u64(yy[3 * i + 2]) != th) {
        char buf[160];
        snprintf(buf, sizeof buf, "device exp/tanh port mismatch at %.17g", ts[i]);
        return fail(ctx, TS_ERR_SELFTEST, buf);
      }
    }
  }
  // tanh_bf (the branch-free restatement the exact LSTM kernels use) must
  // equal the device tanh bit for bit
  DevBuf db;
  TS_CUDA(db.reserve(16));
  TS_CUDA(cudaMemset(db.p, 0, 16));
  k_tanh_selftest<<<296, 256>>>((int64_t)1 << 22, db.as<unsigned long long>());
  TS_LAUNCHED();
  unsigned long long hb[2];
  TS_CUDA(cudaMemcpy(hb, db.p, 16, cudaMemcpyDeviceToHost));
  if (hb[0]) {
    char buf[160];
    double bx;
    memcpy(&bx, &hb[1], 8);
    snprintf(buf, sizeof buf, "device tanh_bf mismatch at %.17g (%llu inputs)", bx, hb[0]);
    return fail(ctx, TS_ERR_SELFTEST, buf);
  }
  return TS_OK;
}

}  // namespace

extern "C" {

int ts_abi_version(void) { return TS_ABI_VERSION; }

const char* ts_last_error(ts_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int ts_ctx_create(int device, ts_ctx** out) {
  if (!out) return TS_ERR_ARG;
  *out = nullptr;
  if (device == -1) {
    // host-only context: descriptor registry + candidate enumeration and
    // legality; every device entry point refuses with TS_ERR_NO_DEVICE
    auto* ctx = new ts_ctx();
    ctx->device = -1;
    *out = ctx;
    return TS_OK;
  }
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count <= device || device < 0)
    return TS_ERR_NO_DEVICE;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major != 10)
    return TS_ERR_NO_DEVICE;
  auto* ctx = new ts_ctx();
  ctx->device = device;
  ctx->sm_count = prop.multiProcessorCount;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->d2h_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess)
    e = cudaMemcpyToSymbol(d_log2_data, ts_log2_data_bits, sizeof(uint64_t) * TS_LOG2_NDATA);
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(d_exp_tab, ts_exp_tab_bits, sizeof(uint64_t) * TS_EXP_NTAB);
  if (e == cudaSuccess) e = ctx->status.reserve(sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(ctx->status.p, 0, sizeof(int));
  // the greedy's scratch (child-row hashes, state rows), sized for the
  // largest pipeline here: allocated inside a first greedy call it cost
  // 7-110 ms of cudaMalloc once the device holds the bench's earlier legs
  if (e == cudaSuccess) e = ctx->ghash.reserve(greedy_hash_bytes());
  if (e == cudaSuccess) e = ctx->tmp.reserve(sizeof(double) * TS_MAX_STAGES * (F + 128));
  if (e != cudaSuccess) {
    delete ctx;
    return TS_ERR_CUDA;
  }
  {
    const int max_slot_smem = MAX_SLOTS * (int)sizeof(Nest) * 128;
    e = cudaFuncSetAttribute(k_featurize_full, cudaFuncAttributeMaxDynamicSharedMemorySize, max_slot_smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_featurize_rows<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               max_slot_smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_featurize_rows<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               max_slot_smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_rescore_exact, cudaFuncAttributeMaxDynamicSharedMemorySize, max_slot_smem);

    if (e != cudaSuccess) {
      delete ctx;
      return TS_ERR_CUDA;
    }
  }
  int rc = self_test(ctx);
  if (!rc) {
    k_fill_log2_table<<<(LOG2_TABLE + 255) / 256, 256>>>();
    if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) rc = TS_ERR_CUDA;
  }
  if (rc) {
    fprintf(stderr, "tensched_b200: %s\n", ctx->err.c_str());
    delete ctx;
    return rc;
  }
  *out = ctx;
  return TS_OK;
}

void ts_ctx_destroy(ts_ctx* ctx) {
  if (!ctx) return;
  if (ctx->device < 0) {
    delete ctx;
    return;
  }
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->copy_stream) cudaStreamSynchronize(ctx->copy_stream);
  if (ctx->d2h_stream) cudaStreamSynchronize(ctx->d2h_stream);
  ctx->pipes.clear();
  for (auto e : ctx->event_pool) cudaEventDestroy(e);
  if (ctx->stream2) cudaStreamSynchronize(ctx->stream2);
  cudaStream_t s = ctx->stream, c = ctx->copy_stream, o = ctx->d2h_stream, s2 = ctx->stream2;
  delete ctx;
  if (s) cudaStreamDestroy(s);
  if (s2) cudaStreamDestroy(s2);
  if (c) cudaStreamDestroy(c);
  if (o) cudaStreamDestroy(o);
}

int ts_set_timing(ts_ctx* ctx, int on) {
  if (!ctx) return TS_ERR_ARG;
  ctx->timing = on != 0;
  return TS_OK;
}

int ts_kernel_times(ts_ctx* ctx, double* ms, int64_t* counts, int reset) {
  if (!ctx || !ms || !counts) return TS_ERR_ARG;
  if (ctx->device >= 0) {
    TS_CUDA(cudaStreamSynchronize(ctx->stream));
    resolve_timers(ctx);
  }
  for (int k = 0; k < TS_KCLASSES; ++k) {
    ms[k] = ctx->kms[k];
    counts[k] = ctx->kcount[k];
    if (reset) {
      ctx->kms[k] = 0.0;
      ctx->kcount[k] = 0;
    }
  }
  return TS_OK;
}

int ts_sync(ts_ctx* ctx) {
  if (!ctx) return TS_ERR_ARG;
  TS_NEED_DEVICE();
  TS_CUDA(cudaStreamSynchronize(ctx->stream));
  return TS_OK;
}

void* ts_stream(ts_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int64_t ts_launch_count(ts_ctx* ctx) { return ctx ? ctx->launches : -1; }

// Clear the device status word after a reported failure: drain the stream
// first (kernels of the failed call may still be running and write it), then
// clear it in stream order.
static void reset_status(ts_ctx* ctx) {
  cudaStreamSynchronize(ctx->stream);
  cudaMemsetAsync(ctx->status.p, 0, sizeof(int), ctx->stream);
  cudaStreamSynchronize(ctx->stream);
}

int ts_pipeline_upload(ts_ctx* ctx, const int64_t* desc, int64_t n_words, int* pipeline_id) {
  if (!ctx || !desc || !pipeline_id) return TS_ERR_ARG;
  if (n_words < DESC_HEADER || desc[0] != 0x54534231 /* "TSB1" */)
    return fail(ctx, TS_ERR_ARG, "bad descriptor header");
  const int64_t T = desc[1], n_slots = desc[2];
  if (T < 1 || T > TS_MAX_STAGES) return fail(ctx, TS_ERR_PIPELINE, "stage count outside 1..512");
  if (n_slots < 0 || n_slots > MAX_SLOTS)
    return fail(ctx, TS_ERR_PIPELINE, "too many simultaneously live nests (max 16)");
  if (n_words != DESC_HEADER + T * DESC_STAGE_WORDS) return fail(ctx, TS_ERR_ARG, "descriptor size");
  auto slot = std::make_unique<PipelineSlot>();
  slot->h = std::make_unique<PipelineDesc>();
  PipelineDesc& P = *slot->h;
  memset(&P, 0, sizeof(P));
  P.n_stages = (int32_t)T;
  P.n_slots = (int32_t)n_slots;
  for (int64_t s = 0; s < T; ++s) {
    const int64_t* w = desc + DESC_HEADER + s * DESC_STAGE_WORDS;
    StageDesc& sd = P.st[s];
    sd.n_pure = (int32_t)w[0];
    sd.n_red = (int32_t)w[1];
    if (sd.n_pure < 1 || sd.n_pure > TS_MAX_PURE || sd.n_red < 0 || sd.n_red > TS_MAX_RED)
      return fail(ctx, TS_ERR_PIPELINE, "stage dims outside 1..4 pure / 0..4 reduction");
    for (int k = 0; k < 8; ++k) sd.ext[k] = w[2 + k];
    sd.pure_points = (uint64_t)w[10];
    sd.red_points = (uint64_t)w[11];
    sd.domain_points = (uint64_t)w[12];
    sd.i_points = (uint64_t)w[13];
    sd.i_flops = (uint64_t)w[14];
    sd.i_in_bytes = (uint64_t)w[15];
    sd.i_out_bytes = (uint64_t)w[16];
    sd.n_inputs = (int32_t)w[17];
    sd.ov_window = (int32_t)w[18];
    sd.ov_stride = (int32_t)w[19];
    sd.consumer = (int32_t)w[20];
    sd.n_cedges = (int32_t)w[21];
    if (sd.n_cedges < 0 || sd.n_cedges > 2)
      return fail(ctx, TS_ERR_PIPELINE, "more than 2 parallel edges from the sole consumer");
    for (int e = 0; e < 2; ++e)
      for (int k = 0; k < 4; ++k) {
        sd.cdim[e][k] = (int32_t)w[22 + e * 4 + k];
        sd.cstride[e][k] = w[30 + e * 4 + k];
        sd.cwindow[e][k] = w[38 + e * 4 + k];
      }
    sd.slot = (int32_t)w[46];
    sd.n_splittable = (int32_t)w[47];
    for (int k = 0; k < 8; ++k)
      if (sd.ext[k] < 0 || sd.ext[k] >= (1ll << 31)) return fail(ctx, TS_ERR_PIPELINE, "extent >= 2^31");
    if (sd.domain_points == 0) return fail(ctx, TS_ERR_PIPELINE, "empty domain");
    sd.dp = make_divisor(sd.domain_points);
    sd.io = make_divisor(1 + sd.i_in_bytes + sd.i_out_bytes);
    // FAST leg's f13 = log2(inv) + log2(region) + log2(red_points / domain_points)
    sd.fast_c13 = std::log2((double)sd.red_points) - std::log2((double)sd.domain_points);
    if (sd.consumer >= T || sd.slot >= n_slots || (sd.consumer >= 0 && sd.consumer <= s))
      return fail(ctx, TS_ERR_PIPELINE, "bad consumer/slot");
  }
  for (int64_t s = 0; s < T; ++s)
    if (P.st[s].consumer >= 0 && P.st[P.st[s].consumer].slot < 0)
      return fail(ctx, TS_ERR_PIPELINE, "sole consumer without a nest slot");
  if (ctx->device >= 0) {
    TS_CUDA(cudaSetDevice(ctx->device));
    TS_CUDA(slot->d.reserve(sizeof(PipelineDesc)));
    TS_CUDA(cudaMemcpyAsync(slot->d.p, &P, sizeof(PipelineDesc), cudaMemcpyHostToDevice, ctx->stream));
    TS_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  ctx->pipes.push_back(std::move(slot));
  *pipeline_id = (int)ctx->pipes.size() - 1;
  return TS_OK;
}

int ts_params_upload(ts_ctx* ctx, int hidden, const double* Wx, const double* Wh, const double* b,
                     const double* w, double b_out, double target_scale, const double* norm_mean,
                     const double* norm_std) {
  if (!ctx || !Wx || !Wh || !b || !w || !norm_mean || !norm_std) return TS_ERR_ARG;
  TS_NEED_DEVICE();
  if (hidden < 1 || hidden > 32) return fail(ctx, TS_ERR_ARG, "hidden size must be in 1..32");
  TS_CUDA(cudaSetDevice(ctx->device));
  TS_CUDA(cudaStreamSynchronize(ctx->stream));
  const size_t G = 4 * (size_t)hidden;
  TS_CUDA(ctx->Wx.reserve(sizeof(double) * F * G));
  TS_CUDA(ctx->Wh.reserve(sizeof(double) * hidden * G));
  TS_CUDA(ctx->b.reserve(sizeof(double) * G));
  TS_CUDA(ctx->w.reserve(sizeof(double) * hidden));
  TS_CUDA(ctx->mean.reserve(sizeof(double) * F));
  TS_CUDA(ctx->stdv.reserve(sizeof(double) * F));
  TS_CUDA(cudaMemcpyAsync(ctx->Wx.p, Wx, sizeof(double) * F * G, cudaMemcpyHostToDevice, ctx->stream));
  TS_CUDA(cudaMemcpyAsync(ctx->Wh.p, Wh, sizeof(double) * hidden * G, cudaMemcpyHostToDevice, ctx->stream));
  TS_CUDA(cudaMemcpyAsync(ctx->b.p, b, sizeof(double) * G, cudaMemcpyHostToDevice, ctx->stream));
  TS_CUDA(cudaMemcpyAsync(ctx->w.p, w, sizeof(double) * hidden, cudaMemcpyHostToDevice, ctx->stream));
  TS_CUDA(cudaMemcpyAsync(ctx->mean.p, norm_mean, sizeof(double) * F, cudaMemcpyHostToDevice, ctx->stream));
  TS_CUDA(cudaMemcpyAsync(ctx->stdv.p, norm_std, sizeof(double) * F, cudaMemcpyHostToDevice, ctx->stream));
  ctx->hidden = hidden;
  ctx->b_out = b_out;
  ctx->target_scale = target_scale;
  ++ctx->params_version;
  if (hidden == 32) {
    // tensor-core weight image: fp16 hi/lo split-concatenated B' + f32 bias/readout
    std::vector<uint8_t> img(tc::TILE_BYTES + 4 * 32);
    tc::pack_weights(Wx, Wh, b, w, img.data());
    TS_CUDA(ctx->fast_w.reserve(img.size()));
    TS_CUDA(cudaMemcpyAsync(ctx->fast_w.p, img.data(), img.size(), cudaMemcpyHostToDevice, ctx->stream));
  }
  TS_CUDA(cudaStreamSynchronize(ctx->stream));
  return TS_OK;
}

int ts_featurize_states(ts_ctx* ctx, int pipeline_id, const ts_decision* records,
                        const int64_t* offsets, int64_t n_states, int normalized, double* out) {
  if (!ctx || !offsets || !out || n_states < 0) return TS_ERR_ARG;
  TS_NEED_DEVICE();
  PipelineSlot* P = get_pipe(ctx, pipeline_id);
  if (!P) return fail(ctx, TS_ERR_ARG, "unknown pipeline id");
  if (n_states == 0) return TS_OK;
  TS_CUDA(cudaSetDevice(ctx->device));
  int rc = ensure_pipe_ready(ctx, P);
  if (rc) return rc;
  const int T = P->h->n_stages;
  const int64_t n_rec = offsets[n_states];
  TS_CUDA(ctx->records.reserve(sizeof(ts_decision) * (n_rec > 0 ? n_rec : 1)));
  TS_CUDA(ctx->offsets.reserve(sizeof(int64_t) * (n_states + 1)));
  TS_CUDA(ctx->out.reserve(sizeof(double) * n_states * T * F));
  if (n_rec)
    TS_CUDA(cudaMemcpyAsync(ctx->records.p, records, sizeof(ts_decision) * n_rec, cudaMemcpyHostToDevice,
                            ctx->stream));
  TS_CUDA(cudaMemcpyAsync(ctx->offsets.p, offsets, sizeof(int64_t) * (n_states + 1),
                          cudaMemcpyHostToDevice, ctx->stream));
  k_featurize_full<<<(unsigned)((n_states + 127) / 128), 128, slot_smem(P, 128), ctx->stream>>>(
      P->d.as<PipelineDesc>(), ctx->records.as<ts_decision>(), ctx->offsets.as<int64_t>(), n_states,
      P->init_raw.as<double>(), ctx->mean.as<double>(), ctx->stdv.as<double>(), normalized,
      ctx->out.as<double>(), ctx->status.as<int>());
  TS_LAUNCHED();
  TS_CUDA(cudaMemcpyAsync(out, ctx->out.p, sizeof(double) * n_states * T * F, cudaMemcpyDeviceToHost,
                          ctx->stream));
  return check_device_status(ctx);
}

static size_t fast_pre_bytes(int T) { return sizeof(float) * (T + 1) * tc::PRE_STRIDE; }

// Fast-path prefix (h, c, raw before every position of the all-unscheduled
// sequence) computed by the tensor-core kernel itself, so replaying prefix
// rows inside a tile is bit-identical to starting from the stored prefix.
static int ensure_fast_prefix(ts_ctx* ctx, PipelineSlot* P) {
  if (P->fast_version == ctx->params_version) return TS_OK;
  const int T = P->h->n_stages;
  {  // the unscheduled rows (and every row's intrinsic half) as operands
    std::vector<double> rows((size_t)T * F);
    TS_CUDA(cudaMemcpyAsync(rows.data(), P->init_norm.p, sizeof(double) * T * F, cudaMemcpyDeviceToHost,
                            ctx->stream));
    TS_CUDA(cudaStreamSynchronize(ctx->stream));
    P->fast_safe = true;
    for (double v : rows)
      if (!(std::fabs((double)(float)v) <= (double)TS_FAST_RANGE)) P->fast_safe = false;
    if (!P->fast_safe) {
      P->fast_version = ctx->params_version;
      return TS_OK;
    }
  }
  TS_CUDA(P->pre_fast.reserve(fast_pre_bytes(T) + sizeof(float) * T * F));
  uint4* initx = reinterpret_cast<uint4*>(P->pre_fast.as<uint8_t>() + fast_pre_bytes(T));
  tc::k_init_split<<<(unsigned)((T + 63) / 64), 64, 0, ctx->stream>>>(P->init_norm.as<double>(), T, initx);
  TS_LAUNCHED();
  if (!ctx->tc_attr_set) {
    TS_CUDA(cudaFuncSetAttribute(tc::k_lstm_tc<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 tc::smem_bytes(4)));
    TS_CUDA(cudaFuncSetAttribute(tc::k_lstm_tc<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 tc::smem_bytes(2)));
    TS_CUDA(cudaFuncSetAttribute(tc::k_lstm_tc<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 tc::smem_bytes(1)));
    ctx->tc_attr_set = true;
  }
  tc::TcArgs ta;
  memset(&ta, 0, sizeof ta);
  ta.wpack = ctx->fast_w.as<uint8_t>();
  ta.initx = initx;
  ta.pre = P->pre_fast.as<float>();
  ta.T = T;
  ta.n_tiles = 1;
  ta.record_prefix = 1;
  ta.b_out = ctx->b_out;
  tc::k_prefix0<<<1, 64, 0, ctx->stream>>>(ta.pre, T, ctx->b_out);
  TS_LAUNCHED();
  tc::k_lstm_tc<4><<<1, 4 * tc::TM, tc::smem_bytes(4), ctx->stream>>>(ta);
  TS_LAUNCHED();
  P->fast_version = ctx->params_version;
  return TS_OK;
}

// FAST scratch of a batch: rowoff[T + 2] (int64), perm[n], hist/cursor[T + 2],
// the range-guard flags (n bytes, 16-byte aligned and padded)
static size_t fast_reps_bytes(int T, int64_t n_states) {
  return sizeof(int64_t) * (T + 2) + sizeof(int) * (n_states + 2 * (T + 2)) + 16 + ((n_states + 15) & ~15ll);
}

// TS_MODE_FAST on a pipeline whose unscheduled rows leave the tensor-core
// operand range runs on the exact leg (TS_FAST_RANGE).
static int resolve_mode(ts_ctx* ctx, PipelineSlot* P, int& mode) {
  if (mode != TS_MODE_FAST || ctx->hidden != 32) return TS_OK;
  int rc = ensure_pipe_ready(ctx, P);
  if (rc) return rc;
  rc = ensure_fast_prefix(ctx, P);
  if (rc) return rc;
  if (!P->fast_safe) mode = TS_MODE_EXACT;
  return TS_OK;
}

// d_codes (optional): 16-bit action codes instead of records, same offsets
// n_records: records of this batch (offsets[n] - offsets[0]); rec_base =
// offsets[0] (callers scoring a chunk of a larger batch keep its absolute
// offsets): the exact leg's rows are indexed from it, so its scratch is the
// chunk's, not the batch's
static int score_device(ts_ctx* ctx, PipelineSlot* P, const ts_decision* d_records,
                        const int64_t* d_offsets, int64_t n_states, int64_t n_records, int mode,
                        double* d_out, const uint16_t* d_codes = nullptr, int64_t rec_base = 0) {
  int rc = ensure_pipe_ready(ctx, P);
  if (rc) return rc;
  const int T = P->h->n_stages;
  if (mode == TS_MODE_EXACT) {
    TS_CUDA(ctx->rows.reserve(sizeof(double) * F * (n_records > 0 ? n_records : 1), ctx->stream));
    {
      KTimer kt(ctx, TS_K_FEATURIZE);
      k_featurize_rows<double><<<(unsigned)((n_states + 127) / 128), 128, slot_smem(P, 128), ctx->stream>>>(
          P->d.as<PipelineDesc>(), d_records, d_offsets, n_states, P->init_norm.as<double>(),
          ctx->mean.as<double>(), ctx->stdv.as<double>(), ctx->rows.as<double>(), ctx->status.as<int>(),
          nullptr, nullptr, d_codes, nullptr, rec_base);
      TS_LAUNCHED();
    }
    {
      const int64_t threads = n_states * 32;
      KTimer kt(ctx, TS_K_LSTM_EXACT);
      if (ctx->hidden == 32) {
        // 16 warps per block share one copy of the weights in shared memory
        if (!ctx->exact_attr_set) {
          TS_CUDA(cudaFuncSetAttribute(k_score_exact32, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sizeof(ExactSmem)));
          TS_CUDA(cudaFuncSetAttribute(k_children_exact32, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sizeof(ExactSmem)));
          ctx->exact_attr_set = true;
        }
        if (n_states >= 4096 && !getenv("TS_EXACT_X1")) {
          // depth-sorted pairs, two states per warp (k_score_exact32x2)
          TS_CUDA(ctx->reps.reserve(fast_reps_bytes(T, n_states), ctx->stream));
          int64_t* rowoff = ctx->reps.as<int64_t>();
          int* perm = reinterpret_cast<int*>(rowoff + (T + 2));
          int* hist = perm + n_states;
          int* cursor = hist + (T + 2);
          const unsigned g = (unsigned)((n_states + 255) / 256);
          TS_CUDA(cudaMemsetAsync(hist, 0, sizeof(int) * (T + 2), ctx->stream));
          tc::k_depth_hist<<<std::min<unsigned>(g, 4u * ctx->sm_count), 256, sizeof(int) * (T + 1),
                             ctx->stream>>>(d_offsets, n_states, T, hist);
          TS_LAUNCHED();
          tc::k_depth_scan<<<1, 32, 0, ctx->stream>>>(hist, T, cursor, rowoff);
          TS_LAUNCHED();
          const int64_t per_block = (int64_t)tc::SCATTER_THREADS * tc::SCATTER_PER;
          tc::k_depth_scatter<<<(unsigned)((n_states + per_block - 1) / per_block), tc::SCATTER_THREADS,
                                sizeof(int) * 2 * (T + 1), ctx->stream>>>(d_offsets, n_states, T, cursor, perm);
          TS_LAUNCHED();
          // states per warp (TS_EXACT_NS: 2, 3 or 4; 2 measured best)
          int ns = 2;
          if (const char* e = getenv("TS_EXACT_NS")) ns = std::min(4, std::max(2, atoi(e)));
          if (!ctx->exact2_attr_set) {
            TS_CUDA(cudaFuncSetAttribute(k_score_exact32xn<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)exact32xn_smem<2>(256)));
            TS_CUDA(cudaFuncSetAttribute(k_score_exact32xn<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)exact32xn_smem<3>(256)));
            TS_CUDA(cudaFuncSetAttribute(k_score_exact32xn<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)exact32xn_smem<4>(256)));
            ctx->exact2_attr_set = true;
          }
          const int64_t warps = (n_states + ns - 1) / ns;
          const unsigned grid = (unsigned)((warps + 7) / 8);
          const LstmW W = lstm_weights(ctx);
          if (ns == 4)
            k_score_exact32xn<4><<<grid, 256, exact32xn_smem<4>(256), ctx->stream>>>(
                W, P->pre_exact.as<double>(), T, d_offsets, ctx->rows.as<double>(), perm, n_states,
                ctx->target_scale, d_out, rec_base);
          else if (ns == 3)
            k_score_exact32xn<3><<<grid, 256, exact32xn_smem<3>(256), ctx->stream>>>(
                W, P->pre_exact.as<double>(), T, d_offsets, ctx->rows.as<double>(), perm, n_states,
                ctx->target_scale, d_out, rec_base);
          else
            k_score_exact32xn<2><<<grid, 256, exact32xn_smem<2>(256), ctx->stream>>>(
                W, P->pre_exact.as<double>(), T, d_offsets, ctx->rows.as<double>(), perm, n_states,
                ctx->target_scale, d_out, rec_base);
        } else {
          k_score_exact32<<<(unsigned)((threads + 511) / 512), 512, sizeof(ExactSmem), ctx->stream>>>(
              lstm_weights(ctx), P->pre_exact.as<double>(), T, d_offsets, ctx->rows.as<double>(), n_states,
              ctx->target_scale, d_out, rec_base);
        }
      } else {
        k_score_exact<<<(unsigned)((threads + 255) / 256), 256, 0, ctx->stream>>>(
            lstm_weights(ctx), P->pre_exact.as<double>(), T, d_offsets, ctx->rows.as<double>(), n_states,
            ctx->target_scale, d_out, rec_base);
      }
      TS_LAUNCHED();
    }
    return TS_OK;
  }
  if (mode == TS_MODE_FAST) {
    if (ctx->hidden != 32) return fail(ctx, TS_ERR_ARG, "the tensor-core path needs hidden = 32");
    rc = ensure_fast_prefix(ctx, P);
    if (rc) return rc;
    // bucket states by depth (descending) so tiles share their depth
    TS_CUDA(ctx->reps.reserve(fast_reps_bytes(T, n_states), ctx->stream));
    int64_t* rowoff = ctx->reps.as<int64_t>();
    int* perm = reinterpret_cast<int*>(rowoff + (T + 2));
    int* hist = perm + n_states;
    int* cursor = hist + (T + 2);
    uint8_t* range_flag = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(cursor + (T + 2)) + 15) & ~(uintptr_t)15);
    const unsigned g = (unsigned)((n_states + 255) / 256);
    {
      KTimer kt(ctx, TS_K_OTHER);
      TS_CUDA(cudaMemsetAsync(hist, 0, sizeof(int) * (T + 2), ctx->stream));
      TS_CUDA(cudaMemsetAsync(range_flag, 0, (n_states + 15) & ~15ll, ctx->stream));
      tc::k_depth_hist<<<std::min<unsigned>(g, 4u * ctx->sm_count), 256, sizeof(int) * (T + 1), ctx->stream>>>(
          d_offsets, n_states, T, hist);
      TS_LAUNCHED();
      tc::k_depth_scan<<<1, 32, 0, ctx->stream>>>(hist, T, cursor, rowoff);
      TS_LAUNCHED();
      const int64_t per_block = (int64_t)tc::SCATTER_THREADS * tc::SCATTER_PER;
      tc::k_depth_scatter<<<(unsigned)((n_states + per_block - 1) / per_block), tc::SCATTER_THREADS,
                            sizeof(int) * 2 * (T + 1), ctx->stream>>>(d_offsets, n_states, T, cursor, perm);
      TS_LAUNCHED();
    }
    TS_CUDA(ctx->rows.reserve(sizeof(float) * 8 * (n_records > 0 ? n_records : 1), ctx->stream));
    {
      KTimer kt(ctx, TS_K_FEATURIZE);
      k_featurize_rows<float><<<(unsigned)((n_states + TS_FEAT_BLOCK - 1) / TS_FEAT_BLOCK), TS_FEAT_BLOCK,
                                slot_smem(P, TS_FEAT_BLOCK), ctx->stream>>>(
          P->d.as<PipelineDesc>(), d_records, d_offsets, n_states, P->init_norm.as<double>(),
          ctx->mean.as<double>(), ctx->stdv.as<double>(), ctx->rows.as<float>(), ctx->status.as<int>(),
          perm, rowoff, d_codes, range_flag);
      TS_LAUNCHED();
    }
    tc::TcArgs ta;
    ta.wpack = ctx->fast_w.as<uint8_t>();
    ta.initx = reinterpret_cast<const uint4*>(P->pre_fast.as<uint8_t>() + fast_pre_bytes(T));
    ta.rowsx = ctx->rows.as<uint4>();
    ta.offsets = d_offsets;
    ta.perm = perm;
    ta.rowoff = rowoff;
    ta.pre = P->pre_fast.as<float>();
    ta.out = d_out;
    ta.n = n_states;
    ta.T = T;
    ta.n_tiles = (int)((n_states + tc::TM - 1) / tc::TM);
    ta.record_prefix = 0;
    ta.target_scale = ctx->target_scale;
    ta.b_out = ctx->b_out;
    TS_CUDA(ctx->tile_ctr.reserve(sizeof(int), ctx->stream));
    TS_CUDA(cudaMemsetAsync(ctx->tile_ctr.p, 0, sizeof(int), ctx->stream));
    ta.tile_counter = ctx->tile_ctr.as<int>();
    {
      KTimer kt(ctx, TS_K_LSTM_FAST);
      // four tiles per SM when there are enough; fewer per CTA (more SMs)
      // for small batches
      const int nwg = ta.n_tiles <= ctx->sm_count ? 1 : ta.n_tiles <= 2 * ctx->sm_count ? 2 : 4;
      const int grid = std::min((ta.n_tiles + nwg - 1) / nwg, ctx->sm_count);
      if (nwg == 4)
        tc::k_lstm_tc<4><<<grid, 4 * tc::TM, tc::smem_bytes(4), ctx->stream>>>(ta);
      else if (nwg == 2)
        tc::k_lstm_tc<2><<<grid, 2 * tc::TM, tc::smem_bytes(2), ctx->stream>>>(ta);
      else
        tc::k_lstm_tc<1><<<grid, tc::TM, tc::smem_bytes(1), ctx->stream>>>(ta);
      TS_LAUNCHED();
    }
    {  // range guard: flagged states rescored on the exact leg
      KTimer kt(ctx, TS_K_OTHER);
      const int rblocks = ctx->sm_count;
      TS_CUDA(ctx->resc.reserve(sizeof(double) * F * T * (size_t)rblocks * 4, ctx->stream));
      k_rescore_exact<<<rblocks, 128, slot_smem(P, 128), ctx->stream>>>(
          P->d.as<PipelineDesc>(), d_records, d_offsets, d_codes, perm, n_states, P->init_norm.as<double>(),
          ctx->mean.as<double>(), ctx->stdv.as<double>(), lstm_weights(ctx), P->pre_exact.as<double>(),
          ctx->target_scale, range_flag, ctx->resc.as<double>(), d_out, ctx->status.as<int>());
      TS_LAUNCHED();
    }
    return TS_OK;
  }
  return fail(ctx, TS_ERR_ARG, "unknown mode");
}

// Host-path chunking: chunks overlap H2D with scoring; measured on B200
// (1M VGG-16 states): 4 chunks beat 1 (no overlap) and 8-16 (per-chunk tile
// tails), so ~n/4 capped at 2^18.
// Sum of n bytes, eight at a time (SWAR, 16-bit lanes flushed every 128
// words): the host-side record count of a depth vector.
static uint64_t sum_bytes(const uint8_t* p, int64_t n) {
  const uint64_t M = 0x00FF00FF00FF00FFull;
  uint64_t total = 0;
  int64_t i = 0;
#ifdef __SSE2__
  {  // psadbw: eight byte sums per instruction
    __m128i acc = _mm_setzero_si128();
    const __m128i z = _mm_setzero_si128();
    for (; i + 16 <= n; i += 16) acc = _mm_add_epi64(acc, _mm_sad_epu8(_mm_loadu_si128((const __m128i*)(p + i)), z));
    total += (uint64_t)_mm_cvtsi128_si64(acc) + (uint64_t)_mm_cvtsi128_si64(_mm_unpackhi_epi64(acc, acc));
  }
#endif
  while (i + 8 <= n) {
    uint64_t lanes = 0;
    for (int w = 0; w < 128 && i + 8 <= n; ++w, i += 8) {
      uint64_t x;
      memcpy(&x, p + i, 8);
      lanes += (x & M) + ((x >> 8) & M);
    }
    lanes = (lanes & 0x0000FFFF0000FFFFull) + ((lanes >> 16) & 0x0000FFFF0000FFFFull);
    total += (lanes & 0xFFFFFFFFull) + (lanes >> 32);
  }
  for (; i < n; ++i) total += p[i];
  return total;
}

static int64_t e2e_chunk(int64_t n) {
  int64_t c = std::max<int64_t>(1 << 16, std::min<int64_t>(1 << 18, (n + 3) / 4));
  if (const char* e = getenv("TS_E2E_CHUNK")) c = std::max<int64_t>(1024, atoll(e));
  return c;
}

int ts_score_states(ts_ctx* ctx, int pipeline_id, const ts_decision* records, const int64_t* offsets,
                    int64_t n_states, int mode, double* out_v) {
  if (!ctx || !offsets || !out_v || n_states < 0) return TS_ERR_ARG;
  TS_NEED_DEVICE();
  PipelineSlot* P = get_pipe(ctx, pipeline_id);
  if (!P) return fail(ctx, TS_ERR_ARG, "unknown pipeline id");
  if (n_states == 0) return TS_OK;
  TS_CUDA(cudaSetDevice(ctx->device));
  {
    const int rc0 = resolve_mode(ctx, P, mode);
    if (rc0) return rc0;
  }
  const int64_t n_rec = offsets[n_states];
  TS_CUDA(ctx->records.reserve(sizeof(ts_decision) * (n_rec > 0 ? n_rec : 1)));
  TS_CUDA(ctx->offsets.reserve(sizeof(int64_t) * (n_states + 1)));
  TS_CUDA(ctx->out.reserve(sizeof(double) * n_states));
  int rc = ensure_pipe_ready(ctx, P);
  if (rc) return rc;
  if (mode == TS_MODE_FAST) {
    rc = ensure_fast_prefix(ctx, P);
    if (rc) return rc;
  }
  // Pipelined host path: every chunk's records are queued H2D on the copy
  // stream up front; the compute stream scores chunk k as soon as its copy
  // event fires (while chunk k+1 is still in flight) and returns its V D2H.
  // Offsets stay absolute, so every chunk indexes the one device records array.
  int64_t chunk = e2e_chunk(n_states);
  if (chunk > n_states) chunk = n_states;
  const int64_t n_chunks = (n_states + chunk - 1) / chunk;
  TS_CUDA(cudaMemcpyAsync(ctx->offsets.p, offsets, sizeof(int64_t) * (n_states + 1), cudaMemcpyHostToDevice,
                          ctx->copy_stream));
  ts_decision* d_rec = ctx->records.as<ts_decision>();
  std::vector<cudaEvent_t> ev;
  for (int64_t k = 0; k < n_chunks; ++k) {
    const int64_t s0 = k * chunk, s1 = std::min(n_states, s0 + chunk);
    const int64_t r0 = offsets[s0], r1 = offsets[s1];
    if (r1 > r0)
      TS_CUDA(cudaMemcpyAsync(d_rec + r0, records + r0, sizeof(ts_decision) * (r1 - r0), cudaMemcpyHostToDevice,
                              ctx->copy_stream));
    cudaEvent_t in = take_event(ctx);
    ev.push_back(in);
    TS_CUDA(cudaEventRecord(in, ctx->copy_stream));
  }
  for (int64_t k = 0; k < n_chunks; ++k) {
    const int64_t s0 = k * chunk, s1 = std::min(n_states, s0 + chunk);
    TS_CUDA(cudaStreamWaitEvent(ctx->stream, ev[k], 0));
    rc = score_device(ctx, P, d_rec, ctx->offsets.as<int64_t>() + s0, s1 - s0, offsets[s1] - offsets[s0], mode,
                      ctx->out.as<double>() + s0, nullptr, offsets[s0]);
    if (rc) return rc;
    TS_CUDA(cudaMemcpyAsync(out_v + s0, ctx->out.as<double>() + s0, sizeof(double) * (s1 - s0),
                            cudaMemcpyDeviceToHost, ctx->stream));
  }
  TS_CUDA(cudaStreamSynchronize(ctx->copy_stream));
  for (auto e : ev) ctx->event_pool.push_back(e);
  return check_device_status(ctx);
}

// ---- packed wire format (8-byte decisions + u8 depths) for host callers
__constant__ uint8_t c_split_table[16] = {0, 2, 3, 4, 5, 6, 7, 8, 12, 16, 24, 32, 48, 64, 128, 255};

// off[0] = base, off[i + 1] = depth[i] (+ base for i = 0): an inclusive scan
// of off[1..n] then gives the offsets of a chunk whose records start at base
__global__ void k_depths_to_counts(const uint8_t* __restrict__ depth, int64_t n, int64_t* __restrict__ off,
                                   int64_t base = 0) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) off[i + 1] = depth[i] + (i == 0 ? base : 0);
  if (i == 0) off[0] = base;
}

__global__ void k_unpack(const uint64_t* __restrict__ packed, int64_t n, ts_decision* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t w = packed[i];
  ts_decision d;
  for (int j = 0; j < TS_MAX_LOOPS; ++j) d.order[j] = (uint8_t)((w >> (4 * j)) & 0xF);
  d.n_loops = (uint8_t)((w >> 32) & 0xF);
  for (int j = d.n_loops; j < TS_MAX_LOOPS; ++j) d.order[j] = 0xFF;
  for (int k = 0; k < TS_MAX_PURE; ++k) d.split[k] = c_split_table[(w >> (36 + 4 * k)) & 0xF];
  const int vc = (int)((w >> 52) & 3);
  d.vec = (uint8_t)(vc == 0 ? 1 : vc == 1 ? 4 : vc == 2 ? 8 : 16);
  d.flags = (uint8_t)((w >> 54) & 3);
  d.anchor = (int8_t)((int)((w >> 56) & 0xF) - 1);
  out[i] = d;
}

int ts_score_states_packed(ts_ctx* ctx, int pipeline_id, const uint64_t* packed, const uint8_t* depths,
                           int64_t n_states, int mode, double* out_v) {
  if (!ctx || !depths || !out_v || n_states < 0) return TS_ERR_ARG;
  TS_NEED_DEVICE();
  PipelineSlot* P = get_pipe(ctx, pipeline_id);
  if (!P) return fail(ctx, TS_ERR_ARG, "unknown pipeline id");
  if (n_states == 0) return TS_OK;
  TS_CUDA(cudaSetDevice(ctx->device));
  {
    const int rc0 = resolve_mode(ctx, P, mode);
    if (rc0) return rc0;
  }
  int rc = ensure_pipe_ready(ctx, P);
  if (rc) return rc;
  if (mode == TS_MODE_FAST) {
    rc = ensure_fast_prefix(ctx, P);
    if (rc) return rc;
  }
  int64_t chunk = e2e_chunk(n_states);
  if (chunk > n_states) chunk = n_states;
  const int64_t n_chunks = (n_states + chunk - 1) / chunk;
  std::vector<int64_t> rec_at(n_chunks + 1);
  {
    int64_t acc = 0;
    for (int64_t k = 0; k < n_chunks; ++k) {
      rec_at[k] = acc;
      const int64_t s1 = std::min(n_states, (k + 1) * chunk);
      acc += (int64_t)sum_bytes(depths + k * chunk, s1 - k * chunk);
    }
    rec_at[n_chunks] = acc;
  }
  const int64_t n_rec = rec_at[n_chunks];
  TS_CUDA(ctx->records.reserve(sizeof(ts_decision) * (n_rec > 0 ? n_rec : 1)));
  TS_CUDA(ctx->offsets.reserve(sizeof(int64_t) * (n_states + 1)));
  TS_CUDA(ctx->out.reserve(sizeof(double) * n_states));
  TS_CUDA(ctx->tmp2.reserve(sizeof(uint64_t) * (n_rec > 0 ? n_rec : 1) + n_states + 64));
  uint64_t* d_packed = ctx->tmp2.as<uint64_t>();
  uint8_t* d_depth = reinterpret_cast<uint8_t*>(d_packed + n_rec);
  int64_t* d_off = ctx->offsets.as<int64_t>();
  TS_CUDA(cudaMemcpyAsync(d_depth, depths, n_states, cudaMemcpyHostToDevice, ctx->copy_stream));
  std::vector<cudaEvent_t> ev;
  cudaEvent_t dep = take_event(ctx);
  TS_CUDA(cudaEventRecord(dep, ctx->copy_stream));
  ev.push_back(dep);
  for (int64_t k = 0; k < n_chunks; ++k) {
    const int64_t r0 = rec_at[k], r1 = rec_at[k + 1];
    if (r1 > r0)
      TS_CUDA(cudaMemcpyAsync(d_packed + r0, packed + r0, sizeof(uint64_t) * (r1 - r0), cudaMemcpyHostToDevice,
                              ctx->copy_stream));
    cudaEvent_t in = take_event(ctx);
    ev.push_back(in);
    TS_CUDA(cudaEventRecord(in, ctx->copy_stream));
  }
  // offsets = exclusive scan of the depths (on the compute stream)
  TS_CUDA(cudaStreamWaitEvent(ctx->stream, dep, 0));
  k_depths_to_counts<<<(unsigned)((n_states + 255) / 256), 256, 0, ctx->stream>>>(d_depth, n_states, d_off);
  TS_LAUNCHED();
  {
    size_t temp = 0;
    TS_CUDA(cub::DeviceScan::InclusiveSum(nullptr, temp, d_off + 1, d_off + 1, n_states, ctx->stream));
    TS_CUDA(ctx->scan_tmp.reserve(temp + 16));
    TS_CUDA(cub::DeviceScan::InclusiveSum(ctx->scan_tmp.p, temp, d_off + 1, d_off + 1, n_states, ctx->stream));
    ++ctx->launches;
  }
  ts_decision* d_rec = ctx->records.as<ts_decision>();
  for (int64_t k = 0; k < n_chunks; ++k) {
    const int64_t s0 = k * chunk, s1 = std::min(n_states, s0 + chunk);
    const int64_t r0 = rec_at[k], r1 = rec_at[k + 1];
    TS_CUDA(cudaStreamWaitEvent(ctx->stream, ev[k + 1], 0));
    if (r1 > r0) {
      KTimer kt(ctx, TS_K_OTHER);
      k_unpack<<<(unsigned)((r1 - r0 + 255) / 256), 256, 0, ctx->stream>>>(d_packed + r0, r1 - r0, d_rec + r0);
      TS_LAUNCHED();
    }
    rc = score_device(ctx, P, d_rec, d_off + s0, s1 - s0, r1 - r0, mode, ctx->out.as<double>() + s0, nullptr, r0);
    if (rc) return rc;
    TS_CUDA(cudaMemcpyAsync(out_v + s0, ctx->out.as<double>() + s0, sizeof(double) * (s1 - s0),
                            cudaMemcpyDeviceToHost, ctx->stream));
  }
  TS_CUDA(cudaStreamSynchronize(ctx->copy_stream));
  for (auto e : ev) ctx->event_pool.push_back(e);
  return check_device_status(ctx);
}

int ts_score_states_coded(ts_ctx* ctx, int pipeline_id, const uint16_t* codes, const uint8_t* depths,
                          int64_t n_states, int mode, double* out_v) {
  if (!ctx || !depths || !out_v || n_states < 0) return TS_ERR_ARG;
  TS_NEED_DEVICE();
  PipelineSlot* P = get_pipe(ctx, pipeline_id);
  if (!P) return fail(ctx, TS_ERR_ARG, "unknown pipeline id");
  if (n_states == 0) return TS_OK;
  TS_CUDA(cudaSetDevice(ctx->device));
  {
    const int rc0 = resolve_mode(ctx, P, mode);
    if (rc0) return rc0;
  }
  int rc = ensure_pipe_ready(ctx, P);
  if (rc) return rc;
  if (mode == TS_MODE_FAST) {
    rc = ensure_fast_prefix(ctx, P);
    if (rc) return rc;
  }
  // Chunks: codes cost ~36 B per state over PCIe against ~2 ns of device
  // work, so transfers run well ahead of the compute.  A short first chunk
  // starts the device early; up to 2^20 states the rest goes as one batch,
  // beyond that in batches of 2^20 (each result block streams back on its
  // own stream while the next batch computes; only the last one is exposed).
  // Beyond 2^20 states the chunks grow geometrically (x2 per chunk up to
  // `step`): each chunk's transfer (~0.65 ns per state) then finishes within
  // the previous chunk's compute (~1.9 ns per state), so the device never
  // waits for bytes, while large chunks keep the per-chunk kernel tails few.
  int64_t first = n_states >= (1 << 18) ? std::min<int64_t>(n_states / 4, 1 << 18) : n_states;
  int64_t step = 1 << 21;
  bool stepped = n_states > (1 << 20);
  bool grow = true;
  if (const char* e = getenv("TS_CODED_CHUNK")) first = std::max<int64_t>(1024, atoll(e));
  if (const char* e = getenv("TS_CODED_STEP")) {
    step = std::max<int64_t>(1024, atoll(e));
    stepped = true;
    grow = false;
  }
  if (const char* e = getenv("TS_CODED_CAP")) step = std::max<int64_t>(1024, atoll(e));  // growth cap
  if (first > n_states) first = n_states;
  std::vector<int64_t> st_at = {0, first};
  if (!stepped) {
    if (first < n_states) st_at.push_back(n_states);
  } else {
    int64_t c = first;
    for (int64_t s0 = first; s0 < n_states;) {
      c = grow ? std::min(step, 2 * c) : step;
      s0 = std::min(n_states, s0 + c);
      st_at.push_back(s0);
    }
  }
  const int64_t n_chunks = (int64_t)st_at.size() - 1;
  // Each chunk's record count is summed on the host just before its copies
  // are queued (the copies of earlier chunks are already in flight), and
  // its offsets are scanned on the device from its own depths with the
  // host-known base, so the first chunk starts after its own bytes only.
  const int T = P->h->n_stages;
  const int64_t rec_cap = n_states * (int64_t)T;  // depths are <= T (checked by the featurizer)
  // chunk k owns offsets d_off[s0 + k .. s1 + k] (its own first entry, so no
  // two chunks - possibly on different lanes - ever touch the same word)
  TS_CUDA(ctx->offsets.reserve(sizeof(int64_t) * (n_states + n_chunks + 1)));
  TS_CUDA(ctx->out.reserve(sizeof(double) * n_states));
  TS_CUDA(ctx->tmp2.reserve(sizeof(uint16_t) * (rec_cap > 0 ? rec_cap : 1) + n_states + 64));
  uint16_t* d_codes = ctx->tmp2.as<uint16_t>();
  uint8_t* d_depth = reinterpret_cast<uint8_t*>(ctx->tmp2.as<uint8_t>() + ((sizeof(uint16_t) * rec_cap + 15) & ~15ull));
  int64_t* d_off = ctx->offsets.as<int64_t>();
  if (!P->code_table.p) {  // every code of every stage, decoded once per pipeline
    TS_CUDA(P->code_table.reserve(sizeof(ts_decision) * (size_t)T * (TS_CODE_SPACE + 1)));
    k_code_table<<<(unsigned)((T * (TS_CODE_SPACE + 1) + 255) / 256), 256, 0, ctx->stream>>>(
        P->d.as<PipelineDesc>(), T, P->code_table.as<ts_decision>());
    TS_LAUNCHED();
  }
  std::vector<cudaEvent_t> ev;
  // every exit (errors included) waits for all four streams before the
  // caller's buffers are released, and returns the events to the pool
  struct Drain {
    ts_ctx* c;
    std::vector<cudaEvent_t>& ev;
    ~Drain() {
      cudaStreamSynchronize(c->copy_stream);
      cudaStreamSynchronize(c->stream);
      if (c->stream2) cudaStreamSynchronize(c->stream2);
      cudaStreamSynchronize(c->d2h_stream);
      for (auto e : ev) c->event_pool.push_back(e);
      ev.clear();
    }
  } drain{ctx, ev};
  // FAST: chunks alternate between two lanes (the exact leg, latency-free
  // and fp64-bound, stays on one)
  const bool two_lanes = mode == TS_MODE_FAST && n_chunks > 1 && !getenv("TS_ONE_LANE");
  {  // per-lane scratch sized for the largest chunk up front, so no buffer a
     // queued kernel reads is reallocated while chunks are in flight
    int64_t max_chunk = 0;
    for (int64_t k = 0; k < n_chunks; ++k) max_chunk = std::max(max_chunk, st_at[k + 1] - st_at[k]);
    size_t temp = 0;
    TS_CUDA(cub::DeviceScan::InclusiveSum(nullptr, temp, d_off + 1, d_off + 1, max_chunk, ctx->stream));
    const size_t rows_bound = sizeof(float) * 8 * (size_t)max_chunk * T;  // depth <= T
    if (two_lanes && !ctx->stream2) TS_CUDA(cudaStreamCreateWithFlags(&ctx->stream2, cudaStreamNonBlocking));
    for (int ln = 0; ln < (two_lanes ? 2 : 1); ++ln) {
      LaneSwap lane(ctx, ln == 1);
      TS_CUDA(ctx->scan_tmp.reserve(temp + 16, ctx->stream));
      // depth bucketing scratch (both legs sort by depth)
      TS_CUDA(ctx->reps.reserve(fast_reps_bytes(T, max_chunk), ctx->stream));
      if (mode == TS_MODE_FAST) {
        if (rows_bound <= ((size_t)4 << 30)) TS_CUDA(ctx->rows.reserve(rows_bound, ctx->stream));
      }
    }
  }
  if (two_lanes) {
    if (!ctx->stream2) TS_CUDA(cudaStreamCreateWithFlags(&ctx->stream2, cudaStreamNonBlocking));
    cudaEvent_t setup = take_event(ctx);  // code table, prefix: issued on lane 0
    ev.push_back(setup);
    TS_CUDA(cudaEventRecord(setup, ctx->stream));
    TS_CUDA(cudaStreamWaitEvent(ctx->stream2, setup, 0));
  }
  int64_t n_rec = 0;
  for (int64_t k = 0; k < n_chunks; ++k) {
    const int64_t s0 = st_at[k], s1 = st_at[k + 1];
    LaneSwap lane(ctx, two_lanes && (k & 1));
    const int64_t r0 = n_rec, r1 = r0 + (int64_t)sum_bytes(depths + s0, s1 - s0);
    if (r1 > rec_cap || (r1 > r0 && !codes))  // (Drain: no copy outlives the caller's buffers)
      return fail(ctx, TS_ERR_ARG, r1 > rec_cap ? "state depth exceeds the pipeline's stage count" : "no codes");
    n_rec = r1;
    TS_CUDA(cudaMemcpyAsync(d_depth + s0, depths + s0, s1 - s0, cudaMemcpyHostToDevice, ctx->copy_stream));
    if (r1 > r0)
      TS_CUDA(cudaMemcpyAsync(d_codes + r0, codes + r0, sizeof(uint16_t) * (r1 - r0), cudaMemcpyHostToDevice,
                              ctx->copy_stream));
    cudaEvent_t in = take_event(ctx);
    ev.push_back(in);
    TS_CUDA(cudaEventRecord(in, ctx->copy_stream));
    TS_CUDA(cudaStreamWaitEvent(ctx->stream, in, 0));
    // offsets of this chunk, chunk-local (off_k[0] = 0, then the scan of its
    // depths); its codes are read from d_codes + r0
    int64_t* off_k = d_off + s0 + k;
    k_depths_to_counts<<<(unsigned)((s1 - s0 + 255) / 256), 256, 0, ctx->stream>>>(d_depth + s0, s1 - s0,
                                                                                     off_k, 0);
    TS_LAUNCHED();
    size_t temp = 0;
    TS_CUDA(cub::DeviceScan::InclusiveSum(nullptr, temp, off_k + 1, off_k + 1, s1 - s0, ctx->stream));
    TS_CUDA(ctx->scan_tmp.reserve(temp + 16, ctx->stream));
    TS_CUDA(cub::DeviceScan::InclusiveSum(ctx->scan_tmp.p, temp, off_k + 1, off_k + 1, s1 - s0, ctx->stream));
    ++ctx->launches;
    // rows are chunk-local in both legs (FAST: decision-major by rowoff;
    // exact: by the chunk-local record offsets), so scratch scales with the
    // largest chunk, not with the batch
    rc = score_device(ctx, P, P->code_table.as<ts_decision>(), off_k, s1 - s0, r1 - r0, mode,
                      ctx->out.as<double>() + s0, d_codes + r0);
    if (rc) return rc;
    cudaEvent_t done = take_event(ctx);
    ev.push_back(done);
    TS_CUDA(cudaEventRecord(done, ctx->stream));
    TS_CUDA(cudaStreamWaitEvent(ctx->d2h_stream, done, 0));
    TS_CUDA(cudaMemcpyAsync(out_v + s0, ctx->out.as<double>() + s0, sizeof(double) * (s1 - s0),
                            cudaMemcpyDeviceToHost, ctx->d2h_stream));
  }
  TS_CUDA(cudaStreamSynchronize(ctx->copy_stream));
  TS_CUDA(cudaStreamSynchronize(ctx->d2h_stream));
  return check_device_status(ctx);
}

int ts_encode_codes_device(ts_ctx* ctx, int pipeline_id, const ts_decision* d_records, const int64_t* d_offsets,
                           int64_t n_states, uint16_t* d_codes) {
  if (!ctx || !d_offsets || n_states < 0) return TS_ERR_ARG;
  TS_NEED_DEVICE();
  PipelineSlot* P = get_pipe(ctx, pipeline_id);
  if (!P) return fail(ctx, TS_ERR_ARG, "unknown pipeline id");
  if (n_states == 0) return TS_OK;
  TS_CUDA(cudaSetDevice(ctx->device));
  k_encode_codes<<<(unsigned)((n_states + 255) / 256), 256, 0, ctx->stream>>>(
      P->d.as<PipelineDesc>(), d_records, d_offsets, n_states, d_codes, ctx->status.as<int>());
  TS_LAUNCHED();
  return check_device_status(ctx);
}

int ts_encode_codes(ts_ctx* ctx, int pipeline_id, const ts_decision* records, const uint8_t* depths,
                    int64_t n_states, uint16_t* out_codes) {
  if (!ctx || !depths || n_states < 0) return TS_ERR_ARG;
  PipelineSlot* P = get_pipe(ctx, pipeline_id);
  if (!P) return fail(ctx, TS_ERR_ARG, "unknown pipeline id");
  const PipelineDesc& D = *P->h;
  const int T = D.n_stages;
  int64_t r = 0;
  for (int64_t i = 0; i < n_states; ++i) {
    if (depths[i] > T) return fail(ctx, TS_ERR_ARG, "depth exceeds the pipeline's stages");
    for (int j = 0; j < depths[i]; ++j, ++r) {
      const uint32_t c = encode_action(D.st[T - 1 - j], records[r]);
      if (c > 0xFFFEu) return fail(ctx, TS_ERR_ILLEGAL, "decision outside the action-code space");
      out_codes[r] = (uint16_t)c;
    }
  }
  return TS_OK;
}

int ts_decode_codes(ts_ctx* ctx, int pipeline_id, const uint16_t* codes, const uint8_t* depths,
                    int64_t n_states, ts_decision* out_records) {
  if (!ctx || !depths || n_states < 0) return TS_ERR_ARG;
  PipelineSlot* P = get_pipe(ctx, pipeline_id);
  if (!P) return fail(ctx, TS_ERR_ARG, "unknown pipeline id");
  const PipelineDesc& D = *P->h;
  const int T = D.n_stages;
  int64_t r = 0;
  for (int64_t i = 0; i < n_states; ++i) {
    if (depths[i] > T) return fail(ctx, TS_ERR_ARG, "depth exceeds the pipeline's stages");
    for (int j = 0; j < depths[i]; ++j, ++r) out_records[r] = decode_action(D.st[T - 1 - j], codes[r]);
  }
  return TS_OK;
}

int ts_score_states_device(ts_ctx* ctx, int pipeline_id, const ts_decision* d_records,
                           const int64_t* d_offsets, int64_t n_states, int64_t n_records, int mode,
                           double* d_out_v) {
  if (!ctx || !d_offsets || !d_out_v || n_states < 0) return TS_ERR_ARG;
  TS_NEED_DEVICE();
  PipelineSlot* P = get_pipe(ctx, pipeline_id);
  if (!P) return fail(ctx, TS_ERR_ARG, "unknown pipeline id");
  if (n_states == 0) return TS_OK;
  TS_CUDA(cudaSetDevice(ctx->device));
  {
    const int rc0 = resolve_mode(ctx, P, mode);
    if (rc0) return rc0;
  }
  int rc = score_device(ctx, P, d_records, d_offsets, n_states, n_records, mode, d_out_v);
  if (rc) return rc;
  return check_device_status(ctx);
}

int ts_score_states_coded_device(ts_ctx* ctx, int pipeline_id, const uint16_t* d_codes, const int64_t* d_offsets,
                                 int64_t n_states, int64_t n_records, int mode, double* d_out_v) {
  if (!ctx || !d_offsets || !d_out_v || n_states < 0 || (n_records > 0 && !d_codes)) return TS_ERR_ARG;
  TS_NEED_DEVICE();
  PipelineSlot* P = get_pipe(ctx, pipeline_id);
  if (!P) return fail(ctx, TS_ERR_ARG, "unknown pipeline id");
  if (n_states == 0) return TS_OK;
  TS_CUDA(cudaSetDevice(ctx->device));
  {
    const int rc0 = resolve_mode(ctx, P, mode);
    if (rc0) return rc0;
  }
  int rc = ensure_pipe_ready(ctx, P);
  if (rc) return rc;
  if (!P->code_table.p) {  // every code of every stage, decoded once per pipeline
    const int T = P->h->n_stages;
    TS_CUDA(P->code_table.reserve(sizeof(ts_decision) * (size_t)T * (TS_CODE_SPACE + 1)));
    k_code_table<<<(unsigned)((T * (TS_CODE_SPACE + 1) + 255) / 256), 256, 0, ctx->stream>>>(
        P->d.as<PipelineDesc>(), T, P->code_table.as<ts_decision>());
    TS_LAUNCHED();
  }
  rc = score_device(ctx, P, P->code_table.as<ts_decision>(), d_offsets, n_states, n_records, mode, d_out_v,
                    d_codes);
  if (rc) return rc;
  return check_device_status(ctx);
}

int ts_lstm_forward(ts_ctx* ctx, const double* X, int64_t B, int64_t T, int64_t Fdim, const double* Wx,
                    const double* Wh, const double* b, const double* w, int64_t H, double b_out, int mode,
                    double* raw_out) {
  if (!ctx || !X || !raw_out || B < 0 || T < 0) return TS_ERR_ARG;
  TS_NEED_DEVICE();
  if (Fdim != F) return fail(ctx, TS_ERR_ARG, "feature width must be 16");
  if (H < 1 || H > 32) return fail(ctx, TS_ERR_ARG, "hidden size must be in 1..32");
  if (mode != TS_MODE_EXACT) return fail(ctx, TS_ERR_ARG, "lstm_forward supports the exact mode");
  if (B == 0) return TS_OK;
  TS_CUDA(cudaSetDevice(ctx->device));
  const size_t G = 4 * (size_t)H;
  // weights travel with the call (backend.py:26 signature); staged in tmp2
  const size_t wbytes = sizeof(double) * (F * G + H * G + G + H);
  TS_CUDA(ctx->tmp2.reserve(wbytes));
  double* dW = ctx->tmp2.as<double>();
  TS_CUDA(cudaMemcpyAsync(dW, Wx, sizeof(double) * F * G, cudaMemcpyHostToDevice, ctx->stream));
  TS_CUDA(cudaMemcpyAsync(dW + F * G, Wh, sizeof(double) * H * G, cudaMemcpyHostToDevice, ctx->stream));
  TS_CUDA(cudaMemcpyAsync(dW + F * G + H * G, b, sizeof(double) * G, cudaMemcpyHostToDevice, ctx->stream));
  TS_CUDA(cudaMemcpyAsync(dW + F * G + H * G + G, w, sizeof(double) * H, cudaMemcpyHostToDevice,
                          ctx->stream));
  TS_CUDA(ctx->tmp.reserve(sizeof(double) * B * T * F + 8));
  TS_CUDA(ctx->out.reserve(sizeof(double) * B));
  if (T) TS_CUDA(cudaMemcpyAsync(ctx->tmp.p, X, sizeof(double) * B * T * F, cudaMemcpyHostToDevice, ctx->stream));
  LstmW W;
  W.Wx = dW;
  W.Wh = dW + F * G;
  W.b = dW + F * G + H * G;
  W.w = dW + F * G + H * G + G;
  W.H = (int)H;
  k_lstm_forward_exact<<<(unsigned)((B * 32 + 255) / 256), 256, 0, ctx->stream>>>(
      W, ctx->tmp.as<double>(), B, (int)T, b_out, ctx->out.as<double>());
  TS_LAUNCHED();
  TS_CUDA(cudaMemcpyAsync(raw_out, ctx->out.p, sizeof(double) * B, cudaMemcpyDeviceToHost, ctx->stream));
  TS_CUDA(cudaStreamSynchronize(ctx->stream));
  return TS_OK;
}

// Host-side state walk: nests of the scheduled prefix.
static int host_nests(ts_ctx* ctx, const PipelineDesc& P, const ts_decision* prefix, int64_t n,
                      std::vector<Nest>& nests) {
  const int T = P.n_stages;
  nests.assign(T, Nest());
  for (int64_t i = 0; i < n; ++i) {
    const int s = T - 1 - (int)i;
    const StageDesc& sd = P.st[s];
    const ts_decision& d = prefix[i];
    const StageDesc* cs = nullptr;
    const Nest* cn = nullptr;
    if (d.anchor >= 0) {
      if (sd.consumer < 0) return fail(ctx, TS_ERR_ILLEGAL, "compute_at without a sole consumer");
      cs = &P.st[sd.consumer];
      cn = &nests[sd.consumer];
    }
    int64_t pe[TS_MAX_PURE];
    const int rc = build_nest(sd, cs, cn, d, nests[s], pe);
    if (rc) return fail(ctx, rc, status_name(rc));
  }
  return TS_OK;
}

int ts_candidates(ts_ctx* ctx, int pipeline_id, const ts_decision* prefix, int64_t n_prefix,
                  ts_decision* out, int64_t capacity, int64_t* n_out) {
  if (!ctx || !n_out || n_prefix < 0) return TS_ERR_ARG;
  PipelineSlot* P = get_pipe(ctx, pipeline_id);
  if (!P) return fail(ctx, TS_ERR_ARG, "unknown pipeline id");
  const PipelineDesc& D = *P->h;
  const int T = D.n_stages;
  if (n_prefix >= T) return fail(ctx, TS_ERR_ILLEGAL, "state is already complete");
  std::vector<Nest> nests;
  int rc = host_nests(ctx, D, prefix, n_prefix, nests);
  if (rc) return rc;
  const int s = T - 1 - (int)n_prefix;
  const StageDesc& sd = D.st[s];
  const StageDesc* cs = sd.consumer >= 0 ? &D.st[sd.consumer] : nullptr;
  const Nest* cn = sd.consumer >= 0 ? &nests[sd.consumer] : nullptr;
  int64_t k = 0;
  const int64_t cnt = enumerate_candidates(sd, cs, cn, [&](const ts_decision& d) {
    if (out && k < capacity) out[k] = d;
    ++k;
  });
  if (cnt < 0) return fail(ctx, (int)-cnt, status_name((int)-cnt));
  *n_out = cnt;
  if (out && cnt > capacity) return fail(ctx, TS_ERR_ARG, "candidate buffer too small");
  return TS_OK;
}

int ts_check_action(ts_ctx* ctx, int pipeline_id, const ts_decision* prefix, int64_t n_prefix,
                    const ts_decision* a) {
  if (!ctx || !a || n_prefix < 0) return TS_ERR_ARG;
  PipelineSlot* P = get_pipe(ctx, pipeline_id);
  if (!P) return fail(ctx, TS_ERR_ARG, "unknown pipeline id");
  const PipelineDesc& D = *P->h;
  const int T = D.n_stages;
  if (n_prefix >= T) return fail(ctx, TS_ERR_ILLEGAL, "state is already complete");
  std::vector<Nest> nests;
  int rc = host_nests(ctx, D, prefix, n_prefix, nests);
  if (rc) return rc;
  const int s = T - 1 - (int)n_prefix;
  const StageDesc& sd = D.st[s];
  const StageDesc* cs = sd.consumer >= 0 ? &D.st[sd.consumer] : nullptr;
  const Nest* cn = sd.consumer >= 0 ? &nests[sd.consumer] : nullptr;
  const char* why = check_decision(sd, cs, cn, *a);
  if (why) return fail(ctx, TS_ERR_ILLEGAL, why);
  return TS_OK;
}

int ts_greedy(ts_ctx* ctx, int pipeline_id, double epsilon, uint64_t* rng_state,
              ts_decision* out_decisions, int64_t* visited, double* out_best_v) {
  if (!ctx || !out_decisions || !visited) return TS_ERR_ARG;
  TS_NEED_DEVICE();
  if (epsilon > 0.0 && !rng_state) return fail(ctx, TS_ERR_ARG, "noisy evaluation needs an rng");
  PipelineSlot* P = get_pipe(ctx, pipeline_id);
  if (!P) return fail(ctx, TS_ERR_ARG, "unknown pipeline id");
  TS_CUDA(cudaSetDevice(ctx->device));
  // TS_GREEDY_TRACE: setup phases (first calls per pipeline) on stderr
  const bool setup_trace = getenv("TS_GREEDY_TRACE") != nullptr;
  double t_mark = 0.0;
  auto mark = [&](const char* what) {
    if (!setup_trace) return;
    const double t = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
    if (what) fprintf(stderr, "ts_greedy setup: %s %.0f us\n", what, t - t_mark);
    t_mark = t;
  };
  mark(nullptr);
  int rc = ensure_pipe_ready(ctx, P);
  mark("pipeline rows and prefix");
  if (rc) return rc;
  TS_CUDA(ctx->gstat.reserve(sizeof(unsigned long long)));
  TS_CUDA(cudaMemsetAsync(ctx->gstat.p, 0, sizeof(unsigned long long), ctx->stream));
  mark("stats");
  const PipelineDesc& D = *P->h;
  const int T = D.n_stages;
  constexpr int kMaxChildren = kGreedyMaxChildren;
  // fused layers (H = 32): children row hashes per layer for the distinct
  // count, and the layer ticket, zeroed once (each layer's last block re-zeroes it)
  const bool fused_layers = ctx->hidden == 32;
  unsigned long long* ghash = nullptr;
  int* gcount = nullptr;
  int* gticket = nullptr;
  if (fused_layers) {
    const size_t hb = sizeof(unsigned long long) * (size_t)T * kMaxChildren;
    TS_CUDA(ctx->ghash.reserve(greedy_hash_bytes(), ctx->stream));  // (sized at context creation)
    ghash = ctx->ghash.as<unsigned long long>();
    gcount = reinterpret_cast<int*>(ctx->ghash.as<char>() + hb);
    gticket = gcount + T;
    TS_CUDA(cudaMemsetAsync(gcount, 0, sizeof(int) * (size_t)(T + 1), ctx->stream));
  }
  mark("child-row hashes");
  std::vector<Nest> nests(T);
  std::vector<ts_decision> cands;
  cands.reserve(1024);
  // device state rows start as the all-unscheduled normalized matrix
  // device state: rows (all-unscheduled normalized matrix to start), then
  // b + x.Wx per scheduled row (H = 32; written as each winner is installed)
  TS_CUDA(ctx->tmp.reserve(sizeof(double) * TS_MAX_STAGES * (F + 128), ctx->stream));  // (sized at context creation)
  mark("state rows");
  double* state_rows = ctx->tmp.as<double>();
  double* zx_state = state_rows + (int64_t)T * F;
  TS_CUDA(cudaMemcpyAsync(state_rows, P->init_norm.p, sizeof(double) * T * F, cudaMemcpyDeviceToDevice,
                          ctx->stream));
  TS_CUDA(ctx->nest.reserve(sizeof(Nest)));
  TS_CUDA(ctx->h_stage.reserve(sizeof(ts_decision) * (4096 + 8)));
  TS_CUDA(ctx->h_out.reserve(sizeof(double) * 4));
  mark("nest, staging");
  uint64_t rng = rng_state ? *rng_state : 0;
  const bool trace = getenv("TS_GREEDY_TRACE") != nullptr;
  double t_enum = 0.0, t_wait = 0.0;
  auto now_us = [] {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
  };
  const double t_call = trace ? now_us() : 0.0;
  int64_t vis = 0;
  double best_v = 0.0;
  for (int i = 0; i < T; ++i) {
    const int s = T - 1 - i;
    const StageDesc& sd = D.st[s];
    const StageDesc* cs = sd.consumer >= 0 ? &D.st[sd.consumer] : nullptr;
    const Nest* cn = sd.consumer >= 0 ? &nests[sd.consumer] : nullptr;
    cands.clear();
    const double te0 = trace ? now_us() : 0.0;
    const int64_t cnt = enumerate_candidates(sd, cs, cn, [&](const ts_decision& d) { cands.push_back(d); });
    if (trace) t_enum += now_us() - te0;
    if (cnt <= 0) return fail(ctx, cnt < 0 ? (int)-cnt : TS_ERR_PIPELINE, "candidate enumeration");
    const int n = (int)cnt;
    if (n > kMaxChildren) return fail(ctx, TS_ERR_PIPELINE, "more than 4096 candidates in one layer");
    TS_CUDA(ctx->records.reserve(sizeof(ts_decision) * (n + 8)));
    TS_CUDA(ctx->rows.reserve(sizeof(double) * F * n));
    TS_CUDA(ctx->reps.reserve(sizeof(int) * (n + 1)));
    TS_CUDA(ctx->raw.reserve(sizeof(double) * n));
    TS_CUDA(ctx->out.reserve(sizeof(double) * 3));
    const bool fused = fused_layers;  // H = 32: the one-kernel layer with the last-block argmin
    // stage host data in pinned memory: candidate records, then the consumer
    // nest right behind them (one H2D per layer)
    ts_decision* hs = ctx->h_stage.as<ts_decision>();
    memcpy(hs, cands.data(), sizeof(ts_decision) * n);
    Nest* hn = reinterpret_cast<Nest*>(hs + n);
    static_assert(sizeof(Nest) <= 8 * sizeof(ts_decision), "nest staging");
    if (cn) *hn = *cn;
    if (fused) {
      // H = 32: ONE kernel per layer - every block computes its child's row
      // from the candidate and the consumer nest in the mapped staging buffer
      // (no copy), runs the exact LSTM over the T - s timesteps it differs
      // in, and the last block to finish runs the argmin, installs the
      // winner's row and writes the layer's result into mapped host memory,
      // which the host polls (no copy, no stream sync)
      ChildRow& cr = ctx->child_row;  // ~3.5 KB: kept in the context, not on the stack per layer
      cr.P = P->d.as<PipelineDesc>();
      cr.cands = hs;
      cr.cnest = cn ? hn : nullptr;
      cr.n_inline = n <= kInlineCands ? n : 0;
      cr.has_nest = cn != nullptr;
      cr.consumer = sd.consumer;
      if (cn) cr.nest = *cn;
      if (cr.n_inline) memcpy(cr.c, cands.data(), sizeof(ts_decision) * n);
      cr.init_raw = P->init_raw.as<double>();
      cr.mean = ctx->mean.as<double>();
      cr.stdv = ctx->stdv.as<double>();
      cr.rows_out = ctx->rows.as<double>();
      cr.hashes = ghash + (size_t)i * kMaxChildren;
      cr.counts = gcount + i;
      cr.status = ctx->status.as<int>();
      GreedyTail tail{};
      tail.ticket = gticket;
      tail.reset_ticket = 1;
      tail.out = ctx->out.as<double>();
      volatile double* ho = ctx->h_out.as<double>();
      const double seq = (double)++ctx->greedy_seq;
      ho[3] = 0.0;
      tail.host_out = ho;
      tail.seq = seq;
      tail.status = ctx->status.as<int>();
      tail.state_row = state_rows + (int64_t)s * F;
      tail.zx_row = zx_state + (int64_t)s * 128;
      tail.target_scale = ctx->target_scale;
      tail.eps = epsilon;
      tail.rng_state0 = rng;
      const size_t xs_bytes = exact_mw_smem(T, s, true);
      if (xs_bytes > 40 * 1024)  // with the kernel's static shared memory
        TS_CUDA(cudaFuncSetAttribute(k_children_exact_mw, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)xs_bytes));
      k_children_exact_mw<<<n, 128, xs_bytes, ctx->stream>>>(
          lstm_weights(ctx), P->pre_exact.as<double>(), T, s, nullptr, nullptr, n, state_rows,
          ctx->raw.as<double>(), zx_state, tail, nullptr, cr);
      TS_LAUNCHED();
      const double tw0 = trace ? now_us() : 0.0;
      // poll the result; every few thousand spins ask the stream whether it
      // failed or finished without writing one
      for (uint32_t spin = 1; ho[3] != seq; ++spin) {
        if ((spin & 4095u) == 0) {
          const cudaError_t q = cudaStreamQuery(ctx->stream);
          if (q != cudaSuccess && q != cudaErrorNotReady) TS_CUDA(q);
          if (q == cudaSuccess && ho[3] != seq) return fail(ctx, TS_ERR_CUDA, "greedy layer wrote no result");
        }
      }
      if (trace) t_wait += now_us() - tw0;
      // the device wrote {v, index, status} before seq (__threadfence_system);
      // order the host's reads of them after its read of seq (not implied on
      // weakly ordered hosts such as aarch64)
      std::atomic_thread_fence(std::memory_order_acquire);
      const int st = (int)ho[2];
      if (st) {
        reset_status(ctx);
        return fail(ctx, st, std::string("device: ") + status_name(st));
      }
      const int best = (int)ho[1];
      best_v = ho[0];
      if (best < 0 || best >= n) return fail(ctx, TS_ERR_CUDA, "argmin produced no index");
      if (epsilon > 0.0) rng += (uint64_t)n * 0x9E3779B97F4A7C15ull;
      vis += n;
      out_decisions[i] = cands[best];
      int64_t pe[TS_MAX_PURE];
      const int brc = build_nest(sd, cands[best].anchor >= 0 ? cs : nullptr,
                                 cands[best].anchor >= 0 ? cn : nullptr, cands[best], nests[s], pe);
      if (brc) return fail(ctx, brc, status_name(brc));
      continue;  // the winner's row is already in the state matrix
    }
    TS_CUDA(cudaMemcpyAsync(ctx->records.p, hs, sizeof(ts_decision) * n, cudaMemcpyHostToDevice, ctx->stream));
    if (cn) TS_CUDA(cudaMemcpyAsync(ctx->nest.p, hn, sizeof(Nest), cudaMemcpyHostToDevice, ctx->stream));
    k_children_rows<<<(n + 127) / 128, 128, 0, ctx->stream>>>(
        P->d.as<PipelineDesc>(), s, ctx->records.as<ts_decision>(), n, ctx->nest.as<Nest>(),
        P->init_raw.as<double>(), ctx->mean.as<double>(), ctx->stdv.as<double>(), ctx->rows.as<double>(),
        ctx->status.as<int>());
    TS_LAUNCHED();
    k_dedup<<<1, 512, 0, ctx->stream>>>(ctx->rows.as<double>(), n, ctx->reps.as<int>(),
                                        ctx->gstat.as<unsigned long long>());
    TS_LAUNCHED();
    if (ctx->hidden == 32) {
      // a few warps per block: the children are few and latency-bound
      if (!ctx->exact_attr_set) {
        TS_CUDA(cudaFuncSetAttribute(k_score_exact32, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(ExactSmem)));
        TS_CUDA(cudaFuncSetAttribute(k_children_exact32, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(ExactSmem)));
        ctx->exact_attr_set = true;
      }
      const size_t xs_bytes = exact_mw_smem(T, s, false);
      if (xs_bytes > 40 * 1024)  // with the kernel's static shared memory
        TS_CUDA(cudaFuncSetAttribute(k_children_exact_mw, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)xs_bytes));
      k_children_exact_mw<<<n, 128, xs_bytes, ctx->stream>>>(
          lstm_weights(ctx), P->pre_exact.as<double>(), T, s,
                                                      ctx->rows.as<double>(), ctx->reps.as<int>(), n, state_rows,
                                                      ctx->raw.as<double>());
    } else {
      k_children_exact<<<(n * 32 + 127) / 128, 128, 0, ctx->stream>>>(
          lstm_weights(ctx), P->pre_exact.as<double>(), T, s, ctx->rows.as<double>(), ctx->reps.as<int>(), n,
          state_rows, ctx->raw.as<double>());
    }
    TS_LAUNCHED();
    k_argmin<<<1, 1024, 0, ctx->stream>>>(ctx->raw.as<double>(), ctx->reps.as<int>(), n,
                                          ctx->target_scale, epsilon, rng, ctx->out.as<double>());
    TS_LAUNCHED();
    double* ho = ctx->h_out.as<double>();
    TS_CUDA(cudaMemcpyAsync(ho, ctx->out.p, sizeof(double) * 2, cudaMemcpyDeviceToHost, ctx->stream));
    int* hst = reinterpret_cast<int*>(ho + 2);
    TS_CUDA(cudaMemcpyAsync(hst, ctx->status.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    const double tw0 = trace ? now_us() : 0.0;
    TS_CUDA(cudaStreamSynchronize(ctx->stream));
    if (trace) t_wait += now_us() - tw0;
    const int st = *hst;
    if (st) {
      reset_status(ctx);
      return fail(ctx, st, std::string("device: ") + status_name(st));
    }
    const int best = (int)ho[1];
    best_v = ho[0];
    if (best < 0 || best >= n) return fail(ctx, TS_ERR_CUDA, "argmin produced no index");
    if (epsilon > 0.0) rng += (uint64_t)n * 0x9E3779B97F4A7C15ull;
    vis += n;
    out_decisions[i] = cands[best];
    int64_t pe[TS_MAX_PURE];
    const int brc = build_nest(sd, cands[best].anchor >= 0 ? cs : nullptr,
                               cands[best].anchor >= 0 ? cn : nullptr, cands[best], nests[s], pe);
    if (brc) return fail(ctx, brc, status_name(brc));
    TS_CUDA(cudaMemcpyAsync(state_rows + (int64_t)s * F, ctx->rows.as<double>() + (int64_t)best * F,
                            sizeof(double) * F, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  if (trace)
    fprintf(stderr, "ts_greedy: T %d, host enumeration %.0f us, waiting on the device %.0f us, layer loop %.0f us\n", T,
            t_enum, t_wait, now_us() - t_call);
  if (rng_state && epsilon > 0.0) *rng_state = rng;
  *visited = vis;
  if (out_best_v) *out_best_v = best_v;
  if (fused_layers) {  // distinct children rows per layer, after the search
    k_greedy_distinct<<<T, 256, 0, ctx->stream>>>(ghash, gcount, kMaxChildren, ctx->gstat.as<unsigned long long>());
    TS_LAUNCHED();
  }
  TS_CUDA(cudaMemcpyAsync(&ctx->greedy_distinct, ctx->gstat.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                          ctx->stream));
  TS_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->greedy_visited = vis;
  return TS_OK;
}

int ts_greedy_stats(ts_ctx* ctx, int64_t* visited, int64_t* distinct) {
  if (!ctx || !visited || !distinct) return TS_ERR_ARG;
  *visited = ctx->greedy_visited;
  *distinct = (int64_t)ctx->greedy_distinct;
  return TS_OK;
}

// One greedy layer for an arbitrary parent: the children's new rows, dedup,
// the exact LSTM from the shared unscheduled prefix over only the T - s
// timesteps a child differs in, then V per child and/or the (noisy) argmin.
int ts_score_children(ts_ctx* ctx, int pipeline_id, const ts_decision* parent, int64_t n_parent,
                      const ts_decision* children, int64_t n_children, double epsilon, uint64_t* rng_state,
                      double* out_v, int64_t* out_best, double* out_best_v) {
  if (!ctx || (n_parent > 0 && !parent) || !children || n_parent < 0 || n_children < 1) return TS_ERR_ARG;
  if (!out_v && !out_best) return TS_ERR_ARG;
  TS_NEED_DEVICE();
  if (epsilon > 0.0 && !rng_state) return fail(ctx, TS_ERR_ARG, "noisy evaluation needs an rng");
  if (n_children > 4096) return fail(ctx, TS_ERR_ARG, "more than 4096 children");
  PipelineSlot* P = get_pipe(ctx, pipeline_id);
  if (!P) return fail(ctx, TS_ERR_ARG, "unknown pipeline id");
  const PipelineDesc& D = *P->h;
  const int T = D.n_stages;
  if (n_parent >= T) return fail(ctx, TS_ERR_ILLEGAL, "state is already complete");
  TS_CUDA(cudaSetDevice(ctx->device));
  int rc = ensure_pipe_ready(ctx, P);
  if (rc) return rc;
  // host: the parent's nests (legality checked on the way) and the children
  std::vector<Nest> nests;
  rc = host_nests(ctx, D, parent, n_parent, nests);
  if (rc) return rc;
  const int s = T - 1 - (int)n_parent;
  const StageDesc& sd = D.st[s];
  const StageDesc* cs = sd.consumer >= 0 ? &D.st[sd.consumer] : nullptr;
  const Nest* cn = sd.consumer >= 0 ? &nests[sd.consumer] : nullptr;
  for (int64_t i = 0; i < n_children; ++i) {
    const char* why = check_decision(sd, cs, cn, children[i]);
    if (why) return fail(ctx, TS_ERR_ILLEGAL, why);
  }
  const int n = (int)n_children, d = (int)n_parent;
  // device: state rows = init rows + the parent's featurized rows
  TS_CUDA(ctx->tmp.reserve(sizeof(double) * (T + std::max(d, 1)) * F));
  double* state_rows = ctx->tmp.as<double>();
  double* prow = state_rows + (int64_t)T * F;
  TS_CUDA(cudaMemcpyAsync(state_rows, P->init_norm.p, sizeof(double) * T * F, cudaMemcpyDeviceToDevice,
                          ctx->stream));
  TS_CUDA(ctx->h_stage.reserve(sizeof(ts_decision) * (4096 + T) + sizeof(Nest) + sizeof(int64_t) * 2));
  ts_decision* hs = ctx->h_stage.as<ts_decision>();
  memcpy(hs, children, sizeof(ts_decision) * n);
  if (d) memcpy(hs + 4096, parent, sizeof(ts_decision) * d);
  Nest* hn = reinterpret_cast<Nest*>(hs + 4096 + T);
  if (cn) *hn = *cn;
  int64_t* hoff = reinterpret_cast<int64_t*>(hn + 1);
  hoff[0] = 0;
  hoff[1] = d;
  TS_CUDA(ctx->records.reserve(sizeof(ts_decision) * (n + T)));
  TS_CUDA(ctx->rows.reserve(sizeof(double) * F * n));
  TS_CUDA(ctx->reps.reserve(sizeof(int) * n));
  TS_CUDA(ctx->raw.reserve(sizeof(double) * 2 * n));
  TS_CUDA(ctx->out.reserve(sizeof(double) * 2 + sizeof(int64_t) * 2));
  TS_CUDA(ctx->nest.reserve(sizeof(Nest)));
  ts_decision* d_children = ctx->records.as<ts_decision>();
  ts_decision* d_parent = d_children + n;
  TS_CUDA(cudaMemcpyAsync(d_children, hs, sizeof(ts_decision) * n, cudaMemcpyHostToDevice, ctx->stream));
  if (cn) TS_CUDA(cudaMemcpyAsync(ctx->nest.p, hn, sizeof(Nest), cudaMemcpyHostToDevice, ctx->stream));
  if (d) {
    int64_t* d_off = reinterpret_cast<int64_t*>(ctx->out.as<double>() + 2);
    TS_CUDA(cudaMemcpyAsync(d_parent, hs + 4096, sizeof(ts_decision) * d, cudaMemcpyHostToDevice, ctx->stream));
    TS_CUDA(cudaMemcpyAsync(d_off, hoff, sizeof(int64_t) * 2, cudaMemcpyHostToDevice, ctx->stream));
    k_featurize_rows<double><<<1, 128, slot_smem(P, 128), ctx->stream>>>(
        P->d.as<PipelineDesc>(), d_parent, d_off, 1, P->init_norm.as<double>(), ctx->mean.as<double>(),
        ctx->stdv.as<double>(), prow, ctx->status.as<int>());
    TS_LAUNCHED();
    k_parent_rows<<<(d * F + 127) / 128, 128, 0, ctx->stream>>>(prow, d, T, state_rows);
    TS_LAUNCHED();
  }
  k_children_rows<<<(n + 127) / 128, 128, 0, ctx->stream>>>(
      P->d.as<PipelineDesc>(), s, d_children, n, ctx->nest.as<Nest>(), P->init_raw.as<double>(),
      ctx->mean.as<double>(), ctx->stdv.as<double>(), ctx->rows.as<double>(), ctx->status.as<int>());
  TS_LAUNCHED();
  k_dedup<<<1, 512, 0, ctx->stream>>>(ctx->rows.as<double>(), n, ctx->reps.as<int>());
  TS_LAUNCHED();
  double* raw = ctx->raw.as<double>();
  if (ctx->hidden == 32) {
    const size_t xs_bytes = exact_mw_smem(T, s, false);
    if (xs_bytes > 40 * 1024)  // with the kernel's static shared memory
      TS_CUDA(cudaFuncSetAttribute(k_children_exact_mw, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)xs_bytes));
    k_children_exact_mw<<<n, 128, xs_bytes, ctx->stream>>>(lstm_weights(ctx), P->pre_exact.as<double>(), T, s,
                                                           ctx->rows.as<double>(), ctx->reps.as<int>(), n,
                                                           state_rows, raw);
  } else {
    k_children_exact<<<(n * 32 + 127) / 128, 128, 0, ctx->stream>>>(
        lstm_weights(ctx), P->pre_exact.as<double>(), T, s, ctx->rows.as<double>(), ctx->reps.as<int>(), n,
        state_rows, raw);
  }
  TS_LAUNCHED();
  TS_CUDA(ctx->h_out.reserve(sizeof(double) * (2 + n) + sizeof(int)));
  double* ho = ctx->h_out.as<double>();
  if (out_v) {
    double* dv = raw + n;
    k_children_v<<<(n + 127) / 128, 128, 0, ctx->stream>>>(raw, ctx->reps.as<int>(), n, ctx->target_scale, dv);
    TS_LAUNCHED();
    TS_CUDA(cudaMemcpyAsync(ho + 2, dv, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  }
  const uint64_t rng = rng_state ? *rng_state : 0;
  if (out_best) {
    k_argmin<<<1, 1024, 0, ctx->stream>>>(raw, ctx->reps.as<int>(), n, ctx->target_scale, epsilon, rng,
                                          ctx->out.as<double>());
    TS_LAUNCHED();
    TS_CUDA(cudaMemcpyAsync(ho, ctx->out.p, sizeof(double) * 2, cudaMemcpyDeviceToHost, ctx->stream));
  }
  int* hst = reinterpret_cast<int*>(ho + 2 + n);
  TS_CUDA(cudaMemcpyAsync(hst, ctx->status.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  TS_CUDA(cudaStreamSynchronize(ctx->stream));
  if (*hst) {
    const int st = *hst;
    reset_status(ctx);
    return fail(ctx, st, std::string("device: ") + status_name(st));
  }
  if (out_v) memcpy(out_v, ho + 2, sizeof(double) * n);
  if (out_best) {
    const int best = (int)ho[1];
    if (best < 0 || best >= n) return fail(ctx, TS_ERR_CUDA, "argmin produced no index");
    *out_best = best;
    if (out_best_v) *out_best_v = ho[0];
    if (rng_state && epsilon > 0.0) *rng_state = rng + (uint64_t)n * 0x9E3779B97F4A7C15ull;
  }
  return TS_OK;
}

// beam_search (search.py:115-133) from a prefix, fused per layer: the
// children of every frontier state are enumerated on the host (native
// candidate_actions, the frontier's nests kept incrementally) and scored in
// ONE device pass - each child's new row (one thread each, its parent's
// consumer nest), dedup of bit-identical rows inside each parent's children,
// the exact fp64 LSTM from the shared unscheduled prefix through the new row
// and the parent's rows (one CTA per distinct child, the parent's rows
// selected per child) - then ranked on the host by (V, index) exactly as
// sorted(range, key=(v, i)) and the `width` best become the next frontier
// (their state rows assembled on the device).  Returns frontier[0] of the
// last layer: the reference's final V(frontier) re-scores the same states
// and its argmin by (v, i) is that entry.
int ts_beam(ts_ctx* ctx, int pipeline_id, const ts_decision* prefix, int64_t n_prefix, int width,
            ts_decision* out_decisions, int64_t* visited, double* out_v) {
  if (!ctx || (n_prefix > 0 && !prefix) || !out_decisions || n_prefix < 0) return TS_ERR_ARG;
  TS_NEED_DEVICE();
  if (width < 1) return fail(ctx, TS_ERR_PIPELINE, "beam width must be >= 1");
  if (width > 1024) return fail(ctx, TS_ERR_ARG, "beam width above 1024");
  PipelineSlot* P = get_pipe(ctx, pipeline_id);
  if (!P) return fail(ctx, TS_ERR_ARG, "unknown pipeline id");
  if (ctx->hidden != 32) return fail(ctx, TS_ERR_ARG, "the fused beam needs hidden size 32");
  const PipelineDesc& D = *P->h;
  const int T = D.n_stages;
  if (n_prefix > T) return fail(ctx, TS_ERR_ILLEGAL, "prefix longer than the pipeline");
  TS_CUDA(cudaSetDevice(ctx->device));
  int rc = ensure_pipe_ready(ctx, P);
  if (rc) return rc;
  struct Entry {
    std::vector<ts_decision> decs;
    std::vector<Nest> nests;
  };
  std::vector<Entry> frontier(1);
  rc = host_nests(ctx, D, prefix, n_prefix, frontier[0].nests);
  if (rc) return rc;
  frontier[0].decs.assign(prefix, prefix + n_prefix);
  if (visited) *visited = 0;
  const int d0 = (int)n_prefix;
  if (d0 == T) {  // complete: the prefix itself (V through the scoring path)
    memcpy(out_decisions, prefix, sizeof(ts_decision) * T);
    if (out_v) {
      const int64_t offs[2] = {0, T};
      return ts_score_states(ctx, pipeline_id, prefix, offs, 1, TS_MODE_EXACT, out_v);
    }
    return TS_OK;
  }
  // device state rows of the frontier, double-buffered: [width][T][F]
  const size_t frow = (size_t)T * F;
  TS_CUDA(ctx->beam_rows.reserve(sizeof(double) * frow * 2 * width, ctx->stream));
  TS_CUDA(ctx->beam_ticket.reserve(sizeof(int), ctx->stream));
  int* bticket = ctx->beam_ticket.as<int>();
  TS_CUDA(cudaMemsetAsync(bticket, 0, sizeof(int), ctx->stream));
  TS_CUDA(ctx->h_sel.reserve(sizeof(int) * 2 * width));
  double* cur = ctx->beam_rows.as<double>();
  double* nxt = cur + frow * width;
  TS_CUDA(cudaMemcpyAsync(cur, P->init_norm.p, sizeof(double) * frow, cudaMemcpyDeviceToDevice, ctx->stream));
  if (d0) {  // the prefix's scheduled rows
    TS_CUDA(ctx->tmp.reserve(sizeof(double) * d0 * F + sizeof(ts_decision) * d0 + 2 * sizeof(int64_t)));
    double* prow = ctx->tmp.as<double>();
    ts_decision* d_pre = reinterpret_cast<ts_decision*>(prow + (size_t)d0 * F);
    int64_t* d_off = reinterpret_cast<int64_t*>(d_pre + d0);
    const int64_t hoff[2] = {0, d0};
    TS_CUDA(cudaMemcpyAsync(d_pre, prefix, sizeof(ts_decision) * d0, cudaMemcpyHostToDevice, ctx->stream));
    TS_CUDA(cudaMemcpyAsync(d_off, hoff, sizeof(hoff), cudaMemcpyHostToDevice, ctx->stream));
    k_featurize_rows<double><<<1, 128, slot_smem(P, 128), ctx->stream>>>(
        P->d.as<PipelineDesc>(), d_pre, d_off, 1, P->init_norm.as<double>(), ctx->mean.as<double>(),
        ctx->stdv.as<double>(), prow, ctx->status.as<int>());
    TS_LAUNCHED();
    k_parent_rows<<<(d0 * F + 127) / 128, 128, 0, ctx->stream>>>(prow, d0, T, cur);
    TS_LAUNCHED();
  }
  std::vector<ts_decision> cands;
  std::vector<int> parent_of, seg;
  std::vector<std::pair<double, int>> ranked;
  int64_t vis = 0;
  const bool trace = getenv("TS_BEAM_TRACE") != nullptr;
  auto now_us = [] {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
  };
  double t_host = 0.0, t_wait = 0.0, t_enum = 0.0;
  const double t_call = trace ? now_us() : 0.0;
  double t_mark = t_call;
  for (int i = d0; i < T; ++i) {
    const int s = T - 1 - i;
    const StageDesc& sd = D.st[s];
    const StageDesc* cs = sd.consumer >= 0 ? &D.st[sd.consumer] : nullptr;
    const int W = (int)frontier.size();
    cands.clear();
    parent_of.clear();
    seg.assign(1, 0);
    for (int w = 0; w < W; ++w) {
      const Nest* cn = cs ? &frontier[w].nests[sd.consumer] : nullptr;
      const int64_t cnt = enumerate_candidates(sd, cs, cn, [&](const ts_decision& d) {
        cands.push_back(d);
        parent_of.push_back(w);
      });
      if (cnt <= 0) return fail(ctx, cnt < 0 ? (int)-cnt : TS_ERR_PIPELINE, "candidate enumeration");
      if (cnt > 4096) return fail(ctx, TS_ERR_PIPELINE, "more than 4096 candidates in one layer");
      seg.push_back((int)cands.size());
    }
    const int n = (int)cands.size();
    vis += n;
    if (trace) {
      const double tn = now_us();
      t_enum += tn - t_mark;
      t_host += tn - t_mark;
      t_mark = tn;
    }
    // pinned staging: records | parent_of | seg | consumer nests (one H2D)
    const size_t b_rec = sizeof(ts_decision) * n, b_par = sizeof(int) * n, b_seg = sizeof(int) * (W + 1);
    const size_t o_par = b_rec, o_seg = o_par + b_par, o_nest = (o_seg + b_seg + 15) & ~(size_t)15;
    const size_t b_all = o_nest + sizeof(Nest) * W;
    TS_CUDA(ctx->h_stage.reserve(b_all));  // its last H2D finished at the previous sync
    TS_CUDA(ctx->records.reserve(b_all, ctx->stream));
    uint8_t* hb = ctx->h_stage.as<uint8_t>();
    memcpy(hb, cands.data(), b_rec);
    memcpy(hb + o_par, parent_of.data(), b_par);
    memcpy(hb + o_seg, seg.data(), b_seg);
    Nest* hn = reinterpret_cast<Nest*>(hb + o_nest);
    if (cs)
      for (int w = 0; w < W; ++w) hn[w] = frontier[w].nests[sd.consumer];
    uint8_t* db = ctx->records.as<uint8_t>();
    TS_CUDA(cudaMemcpyAsync(db, hb, b_all, cudaMemcpyHostToDevice, ctx->stream));
    const ts_decision* d_c = reinterpret_cast<const ts_decision*>(db);
    const int* d_par = reinterpret_cast<const int*>(db + o_par);
    const int* d_seg = reinterpret_cast<const int*>(db + o_seg);
    const Nest* d_nest = cs ? reinterpret_cast<const Nest*>(db + o_nest) : nullptr;
    TS_CUDA(ctx->rows.reserve(sizeof(double) * F * n, ctx->stream));
    TS_CUDA(ctx->reps.reserve(sizeof(int) * n, ctx->stream));
    TS_CUDA(ctx->raw.reserve(sizeof(double) * 2 * n, ctx->stream));
    double* raw = ctx->raw.as<double>();
    k_children_rows<<<(n + 127) / 128, 128, 0, ctx->stream>>>(
        P->d.as<PipelineDesc>(), s, d_c, n, d_nest, P->init_raw.as<double>(), ctx->mean.as<double>(),
        ctx->stdv.as<double>(), ctx->rows.as<double>(), ctx->status.as<int>(), d_par);
    TS_LAUNCHED();
    k_dedup_segments<<<W, 512, 0, ctx->stream>>>(ctx->rows.as<double>(), d_seg, ctx->reps.as<int>());
    TS_LAUNCHED();
    const size_t xs_bytes = exact_mw_smem(T, s, false);
    if (xs_bytes > 40 * 1024)
      TS_CUDA(cudaFuncSetAttribute(k_children_exact_mw, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)xs_bytes));
    // the last CTA writes every child's V and the device status into mapped
    // host memory and then a sequence number, which the host polls (no
    // copies, no stream sync per layer)
    TS_CUDA(ctx->h_out.reserve(sizeof(double) * (n + 4)));
    double* hv = ctx->h_out.as<double>();
    volatile double* ho = hv + n;  // {-, -, status, seq}
    const double seq = (double)++ctx->greedy_seq;
    ho[3] = 0.0;
    GreedyTail tail{};
    tail.ticket = bticket;
    tail.reset_ticket = 1;
    tail.status = ctx->status.as<int>();
    tail.target_scale = ctx->target_scale;
    tail.host_v = hv;
    tail.host_out = ho;
    tail.seq = seq;
    k_children_exact_mw<<<n, 128, xs_bytes, ctx->stream>>>(lstm_weights(ctx), P->pre_exact.as<double>(), T, s,
                                                           ctx->rows.as<double>(), ctx->reps.as<int>(), n, cur,
                                                           raw, nullptr, tail, d_par);
    TS_LAUNCHED();
    if (trace) {
      const double tn = now_us();
      t_host += tn - t_mark;
      t_mark = tn;
    }
    for (uint32_t spin = 1; ho[3] != seq; ++spin) {
      if ((spin & 4095u) == 0) {
        const cudaError_t q = cudaStreamQuery(ctx->stream);
        if (q != cudaSuccess && q != cudaErrorNotReady) TS_CUDA(q);
        if (q == cudaSuccess && ho[3] != seq) return fail(ctx, TS_ERR_CUDA, "beam layer wrote no result");
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);  // V and status were written before seq
    if (trace) {
      const double tn = now_us();
      t_wait += tn - t_mark;
      t_mark = tn;
    }
    if (const int st = (int)ho[2]) {
      reset_status(ctx);
      return fail(ctx, st, std::string("device: ") + status_name(st));
    }
    // sorted(range(len(children)), key=(v, i))[:width]
    ranked.resize(n);
    for (int c = 0; c < n; ++c) ranked[c] = {hv[c], c};
    const int keep = std::min(width, n);
    std::partial_sort(ranked.begin(), ranked.begin() + keep, ranked.end(),
                      [](const std::pair<double, int>& a, const std::pair<double, int>& b) {
                        return a.first < b.first || (a.first == b.first && a.second < b.second);
                      });
    std::vector<Entry> next(keep);
    std::vector<int> sel(2 * keep);
    for (int k = 0; k < keep; ++k) {
      const int c = ranked[k].second, w = parent_of[c];
      sel[2 * k] = w;
      sel[2 * k + 1] = c;
      next[k].decs = frontier[w].decs;
      next[k].decs.push_back(cands[c]);
      next[k].nests = frontier[w].nests;
      int64_t pe[TS_MAX_PURE];
      const int brc = build_nest(sd, cands[c].anchor >= 0 ? cs : nullptr,
                                 cands[c].anchor >= 0 ? &frontier[w].nests[sd.consumer] : nullptr, cands[c],
                                 next[k].nests[s], pe);
      if (brc) return fail(ctx, brc, status_name(brc));
    }
    if (i + 1 < T) {  // the next frontier's state rows
      // (own pinned buffer: its H2D completes before the next layer's sync,
      // the only point after which the host rewrites it)
      int* hsel = ctx->h_sel.as<int>();
      memcpy(hsel, sel.data(), sizeof(int) * 2 * keep);
      TS_CUDA(cudaMemcpyAsync(ctx->records.p, hsel, sizeof(int) * 2 * keep, cudaMemcpyHostToDevice, ctx->stream));
      k_beam_advance<<<keep, 256, 0, ctx->stream>>>(cur, nxt, T, s, ctx->records.as<int>(), ctx->rows.as<double>());
      TS_LAUNCHED();
      std::swap(cur, nxt);
    }
    frontier.swap(next);
    if (i + 1 == T && out_v) *out_v = ranked[0].first;
  }
  memcpy(out_decisions, frontier[0].decs.data(), sizeof(ts_decision) * T);
  if (visited) *visited = vis;
  TS_CUDA(cudaStreamSynchronize(ctx->stream));
  if (trace)
    fprintf(stderr, "ts_beam: T %d, width %d, visited %lld: host %.0f us (of which rank + frontier + enumerate "
            "%.0f us), waiting %.0f us, total %.0f us\n", T, width, (long long)vis, t_host, t_enum, t_wait,
            now_us() - t_call);
  return TS_OK;
}

int ts_featurize_rows_device(ts_ctx* ctx, int pipeline_id, const ts_decision* d_records,
                             const int64_t* d_offsets, int64_t n_states, double* d_rows) {
  if (!ctx || !d_records || !d_offsets || !d_rows || n_states < 0) return TS_ERR_ARG;
  TS_NEED_DEVICE();
  PipelineSlot* P = get_pipe(ctx, pipeline_id);
  if (!P) return fail(ctx, TS_ERR_ARG, "unknown pipeline id");
  if (n_states == 0) return TS_OK;
  TS_CUDA(cudaSetDevice(ctx->device));
  int rc = ensure_pipe_ready(ctx, P);
  if (rc) return rc;
  k_featurize_rows<double><<<(unsigned)((n_states + 127) / 128), 128, slot_smem(P, 128), ctx->stream>>>(
      P->d.as<PipelineDesc>(), d_records, d_offsets, n_states, P->init_norm.as<double>(), ctx->mean.as<double>(),
      ctx->stdv.as<double>(), d_rows, ctx->status.as<int>());
  TS_LAUNCHED();
  return check_device_status(ctx);
}

int ts_init_rows(ts_ctx* ctx, int pipeline_id, int normalized, double* out) {
  if (!ctx || !out) return TS_ERR_ARG;
  TS_NEED_DEVICE();
  PipelineSlot* P = get_pipe(ctx, pipeline_id);
  if (!P) return fail(ctx, TS_ERR_ARG, "unknown pipeline id");
  TS_CUDA(cudaSetDevice(ctx->device));
  int rc = ensure_pipe_ready(ctx, P);
  if (rc) return rc;
  const int T = P->h->n_stages;
  TS_CUDA(cudaMemcpyAsync(out, normalized ? P->init_norm.p : P->init_raw.p, sizeof(double) * T * F,
                          cudaMemcpyDefault, ctx->stream));
  TS_CUDA(cudaStreamSynchronize(ctx->stream));
  return TS_OK;
}

int ts_generate_schedules_device(ts_ctx* ctx, int pipeline_id, uint64_t seed0, uint64_t stride, int64_t n,
                                 ts_decision* d_records) {
  if (!ctx || !d_records || n < 0) return TS_ERR_ARG;
  TS_NEED_DEVICE();
  PipelineSlot* P = get_pipe(ctx, pipeline_id);
  if (!P) return fail(ctx, TS_ERR_ARG, "unknown pipeline id");
  TS_CUDA(cudaSetDevice(ctx->device));
  TS_CUDA(ctx->tmp.reserve(sizeof(int) * (n > 0 ? n : 1)));
  k_generate<<<(unsigned)((n + 127) / 128), 128, 0, ctx->stream>>>(
      P->d.as<PipelineDesc>(), seed0, n, d_records, ctx->tmp.as<int>(), ctx->status.as<int>(), 1, stride);
  TS_LAUNCHED();
  return check_device_status(ctx);
}

int ts_benchmark(ts_ctx* ctx, int pipeline_id, const int64_t* cost_desc, int64_t n_words,
                 const uint64_t* machine, const ts_decision* records, const int64_t* offsets, int64_t n,
                 uint64_t* out_millis) {
  if (!ctx || !cost_desc || !machine || !offsets || !out_millis || n < 0) return TS_ERR_ARG;
  TS_NEED_DEVICE();
  PipelineSlot* P = get_pipe(ctx, pipeline_id);
  if (!P) return fail(ctx, TS_ERR_ARG, "unknown pipeline id");
  if (n == 0) return TS_OK;
  const int T = P->h->n_stages;
  if (n_words != (int64_t)T * cost::WORDS_PER_STAGE) return fail(ctx, TS_ERR_ARG, "cost descriptor size");
  auto C = std::make_unique<cost::CostDesc>();
  for (int s = 0; s < T; ++s) {
    const int64_t* w = cost_desc + (int64_t)s * cost::WORDS_PER_STAGE;
    cost::StageCostDesc& sc = C->st[s];
    sc.flops_per_point = (uint64_t)w[0];
    sc.n_in = (int32_t)w[1];
    if (sc.n_in < 0 || sc.n_in > cost::MAX_IN) return fail(ctx, TS_ERR_PIPELINE, "more than 4 inputs");
    for (int e = 0; e < cost::MAX_IN; ++e) {
      const int64_t* q = w + 2 + e * cost::WORDS_PER_IN;
      cost::Edge& ed = sc.in[e];
      ed.producer = (int32_t)q[0];
      ed.elem = (int32_t)q[1];
      ed.n_maps = (int32_t)q[2];
      if (ed.n_maps < 0 || ed.n_maps > cost::MAX_MAPS) return fail(ctx, TS_ERR_PIPELINE, "more than 6 maps");
      for (int k = 0; k < cost::MAX_MAPS; ++k) {
        ed.cdim[k] = (int32_t)q[3 + 3 * k];
        ed.stride[k] = q[4 + 3 * k];
        ed.window[k] = q[5 + 3 * k];
      }
    }
  }
  cost::Machine m{machine[0], machine[1], machine[2], machine[3], machine[4], machine[5]};
  TS_CUDA(cudaSetDevice(ctx->device));
  const int64_t n_rec = offsets[n];
  TS_CUDA(ctx->tmp2.reserve(sizeof(cost::CostDesc)));
  TS_CUDA(cudaMemcpyAsync(ctx->tmp2.p, C.get(), sizeof(cost::CostDesc), cudaMemcpyHostToDevice, ctx->stream));
  TS_CUDA(ctx->records.reserve(sizeof(ts_decision) * (n_rec > 0 ? n_rec : 1)));
  TS_CUDA(ctx->offsets.reserve(sizeof(int64_t) * (n + 1)));
  TS_CUDA(ctx->out.reserve(sizeof(uint64_t) * 4 * n));
  TS_CUDA(ctx->tmp.reserve(sizeof(cost::StageRec) * n * T));
  if (n_rec)
    TS_CUDA(cudaMemcpyAsync(ctx->records.p, records, sizeof(ts_decision) * n_rec, cudaMemcpyHostToDevice,
                            ctx->stream));
  TS_CUDA(cudaMemcpyAsync(ctx->offsets.p, offsets, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, ctx->stream));
  cost::k_benchmark<<<(unsigned)((n + 127) / 128), 128, 0, ctx->stream>>>(
      P->d.as<PipelineDesc>(), ctx->tmp2.as<cost::CostDesc>(), m, ctx->records.as<ts_decision>(),
      ctx->offsets.as<int64_t>(), n, ctx->tmp.as<cost::StageRec>(), ctx->out.as<uint64_t>(),
      ctx->status.as<int>());
  TS_LAUNCHED();
  TS_CUDA(cudaMemcpyAsync(out_millis, ctx->out.p, sizeof(uint64_t) * 4 * n, cudaMemcpyDeviceToHost, ctx->stream));
  return check_device_status(ctx);
}

int ts_generate_states_device(ts_ctx* ctx, int pipeline_id, uint64_t seed0, int64_t n_states,
                              ts_decision* d_records, int64_t* d_offsets, int64_t* n_records) {
  if (!ctx || !d_records || !d_offsets || !n_records || n_states < 0) return TS_ERR_ARG;
  TS_NEED_DEVICE();
  PipelineSlot* P = get_pipe(ctx, pipeline_id);
  if (!P) return fail(ctx, TS_ERR_ARG, "unknown pipeline id");
  TS_CUDA(cudaSetDevice(ctx->device));
  const int T = P->h->n_stages;
  TS_CUDA(ctx->tmp.reserve(sizeof(ts_decision) * n_states * T + sizeof(int) * n_states + 16));
  ts_decision* fixed = ctx->tmp.as<ts_decision>();
  int* depth = reinterpret_cast<int*>(fixed + n_states * T);
  k_generate<<<(unsigned)((n_states + 127) / 128), 128, 0, ctx->stream>>>(
      P->d.as<PipelineDesc>(), seed0, n_states, fixed, depth, ctx->status.as<int>(), 0);
  // (the generator keeps its nests in registers/local memory: untimed)
  TS_LAUNCHED();
  std::vector<int> hd(n_states);
  std::vector<int64_t> ho(n_states + 1);
  TS_CUDA(cudaMemcpyAsync(hd.data(), depth, sizeof(int) * n_states, cudaMemcpyDeviceToHost, ctx->stream));
  int rc = check_device_status(ctx);
  if (rc) return rc;
  ho[0] = 0;
  for (int64_t i = 0; i < n_states; ++i) ho[i + 1] = ho[i] + hd[i];
  TS_CUDA(cudaMemcpyAsync(d_offsets, ho.data(), sizeof(int64_t) * (n_states + 1), cudaMemcpyHostToDevice,
                          ctx->stream));
  k_compact_records<<<(unsigned)((n_states + 127) / 128), 128, 0, ctx->stream>>>(fixed, depth, d_offsets,
                                                                                 n_states, T, d_records);
  TS_LAUNCHED();
  TS_CUDA(cudaStreamSynchronize(ctx->stream));
  *n_records = ho[n_states];
  return TS_OK;
}

// ------------------------------------------------------------------ training
int ts_train_load(ts_ctx* ctx, const double* rows, int64_t n_rows, const double* init, int64_t n_init,
                  const int64_t* row_base, const int32_t* init_base, const int32_t* Tlen,
                  const int32_t* depth, const double* logt, int64_t N, int hidden, int device_ptrs) {
  if (!ctx || !rows || !row_base || !init_base || !Tlen || !depth || !logt || N < 1 || n_rows < 1)
    return TS_ERR_ARG;
  TS_NEED_DEVICE();
  if (hidden < 1 || hidden > 32) return fail(ctx, TS_ERR_ARG, "hidden size must be in 1..32");
  TS_CUDA(cudaSetDevice(ctx->device));
  TS_CUDA(cudaStreamSynchronize(ctx->stream));
  const cudaMemcpyKind kind = device_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  std::vector<int32_t> hT(N);
  TS_CUDA(cudaMemcpyAsync(hT.data(), Tlen, sizeof(int32_t) * N, device_ptrs ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost, ctx->stream));
  TS_CUDA(cudaStreamSynchronize(ctx->stream));
  int Tmax = 1;
  for (int64_t i = 0; i < N; ++i) Tmax = std::max(Tmax, (int)hT[i]);
  ctx->tr_H = hidden;
  ctx->tr_Tmax = Tmax;
  ctx->tr_N = N;
  TS_CUDA(ctx->tr_X.reserve(sizeof(double) * (n_rows + std::max<int64_t>(n_init, 1)) * F));
  TS_CUDA(ctx->tr_T.reserve((sizeof(int64_t) + 3 * sizeof(int32_t)) * N));
  TS_CUDA(ctx->tr_logt.reserve(sizeof(double) * N));
  double* drows = ctx->tr_X.as<double>();
  double* dinit = drows + n_rows * F;
  int64_t* drb = ctx->tr_T.as<int64_t>();
  int32_t* dib = reinterpret_cast<int32_t*>(drb + N);
  TS_CUDA(cudaMemcpyAsync(drows, rows, sizeof(double) * n_rows * F, kind, ctx->stream));
  if (n_init) TS_CUDA(cudaMemcpyAsync(dinit, init, sizeof(double) * n_init * F, kind, ctx->stream));
  TS_CUDA(cudaMemcpyAsync(drb, row_base, sizeof(int64_t) * N, kind, ctx->stream));
  TS_CUDA(cudaMemcpyAsync(dib, init_base, sizeof(int32_t) * N, kind, ctx->stream));
  TS_CUDA(cudaMemcpyAsync(dib + N, Tlen, sizeof(int32_t) * N, kind, ctx->stream));
  TS_CUDA(cudaMemcpyAsync(dib + 2 * N, depth, sizeof(int32_t) * N, kind, ctx->stream));
  TS_CUDA(cudaMemcpyAsync(ctx->tr_logt.p, logt, sizeof(double) * N, kind, ctx->stream));
  ctx->tr_data.rows = drows;
  ctx->tr_data.init = dinit;
  ctx->tr_data.row_base = drb;
  ctx->tr_data.init_base = dib;
  ctx->tr_data.Tlen = dib + N;
  ctx->tr_data.depth = dib + 2 * N;
  ctx->tr_data.logt = ctx->tr_logt.as<double>();
  const tr::Layout L(hidden);
  TS_CUDA(ctx->tr_P.reserve(sizeof(double) * L.n));
  TS_CUDA(ctx->tr_grad.reserve(sizeof(double) * L.n));
  TS_CUDA(ctx->tr_norm.reserve(sizeof(double)));
  TS_CUDA(cudaStreamSynchronize(ctx->stream));
  return TS_OK;
}

int ts_train_set_params(ts_ctx* ctx, const double* flat, int64_t n) {
  if (!ctx || !flat) return TS_ERR_ARG;
  TS_NEED_DEVICE();
  const tr::Layout L(ctx->tr_H);
  if (!ctx->tr_H || n != L.n) return fail(ctx, TS_ERR_ARG, "parameter vector size");
  TS_CUDA(cudaMemcpyAsync(ctx->tr_P.p, flat, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
  TS_CUDA(cudaStreamSynchronize(ctx->stream));
  return TS_OK;
}

int ts_train_get_params(ts_ctx* ctx, double* flat, int64_t n) {
  if (!ctx || !flat) return TS_ERR_ARG;
  TS_NEED_DEVICE();
  const tr::Layout L(ctx->tr_H);
  if (!ctx->tr_H || n != L.n) return fail(ctx, TS_ERR_ARG, "parameter vector size");
  TS_CUDA(cudaMemcpyAsync(flat, ctx->tr_P.p, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  TS_CUDA(cudaStreamSynchronize(ctx->stream));
  return TS_OK;
}

static int train_args(ts_ctx* ctx, const int32_t* idx, int64_t B, tr::TrainArgs& a) {
  TS_CUDA(ctx->tr_batch.reserve(sizeof(int32_t) * B));
  TS_CUDA(ctx->tr_raw.reserve(sizeof(double) * B));
  TS_CUDA(ctx->tr_draw.reserve(sizeof(double) * B));
  TS_CUDA(cudaMemcpyAsync(ctx->tr_batch.p, idx, sizeof(int32_t) * B, cudaMemcpyHostToDevice, ctx->stream));
  a.D = ctx->tr_data;
  a.batch = ctx->tr_batch.as<int>();
  a.P = ctx->tr_P.as<double>();
  a.cache = nullptr;
  a.dz = nullptr;
  a.pvalid = nullptr;
  a.draw = ctx->tr_draw.as<double>();
  a.raw = ctx->tr_raw.as<double>();
  a.B = (int)B;
  a.Tmax = ctx->tr_Tmax;
  a.H = ctx->tr_H;
  a.target_scale = 0.0;
  a.n_total = 1.0;
  a.partial = nullptr;
  a.draw_in = nullptr;
  return TS_OK;
}

int ts_train_set_mode(ts_ctx* ctx, int mode) {
  if (!ctx || (mode != TS_TRAIN_EXACT && mode != TS_TRAIN_TC && mode != TS_TRAIN_TCF)) return TS_ERR_ARG;
  ctx->tr_mode = mode;
  return TS_OK;
}

// Gradient of the loss over this rank's part of a minibatch whose global size
// is n_total (d_raw divides by it); written to d_grad (device pointer, or the
// context's buffer when null).  Data-parallel callers all-reduce d_grad.
// Forward + BPTT + weight gradients of a filled TrainArgs (batch a.B, longest
// sequence a.Tmax) into grad, in the context's gradient mode.
static int launch_grads(ts_ctx* ctx, tr::TrainArgs& a, int mode, double* grad, double* raw_out) {
  const int64_t B = a.B;
  const int H = a.H, Tmax = a.Tmax;
  const tr::Layout L(H);
  const bool grouped = H == tr::GH && !getenv("TS_TRAIN_WARP");
  const int64_t K = (int64_t)Tmax * B;
  if (mode == TS_TRAIN_TCF) {
    // forward and backward recurrences on the tensor cores (ts_train_tc.cuh)
    if (H != trc::H) return fail(ctx, TS_ERR_ARG, "tensor-core training needs hidden size 32");
    // sequences per tile: 128 when the batch fills the SMs, else fewer (a
    // multiple of 32, every tile's recurrence is latency-bound, so more
    // partly filled tiles finish sooner than fewer full ones)
    int rows = trc::TM;
    if (B < (int64_t)trc::TM * ctx->sm_count)
      rows = std::max<int>(32, (int)(((B + ctx->sm_count - 1) / ctx->sm_count + 31) / 32 * 32));
    if (const char* e = getenv("TS_TRC_ROWS")) rows = std::min(trc::TM, std::max(1, atoi(e)));
    const int n_tiles = (int)((B + rows - 1) / rows);
    const size_t img_bytes = tc::TILE_BYTES + 128 + 2 * trc::WT_BYTES;
    TS_CUDA(ctx->trc_img.reserve(img_bytes, ctx->stream));
    TS_CUDA(ctx->tr_cache.reserve(sizeof(float) * (size_t)n_tiles * Tmax * trc::NF * 4 * trc::TM * 8, ctx->stream));
    TS_CUDA(ctx->tr_partial.reserve(sizeof(double) * (size_t)n_tiles * L.n + 16, ctx->stream));
    if (!ctx->trc_attr_set) {
      TS_CUDA(cudaFuncSetAttribute(trc::k_trc_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, trc::FWD_SMEM));
      TS_CUDA(cudaFuncSetAttribute(trc::k_trc_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, trc::BWD_SMEM));
      ctx->trc_attr_set = true;
    }
    trc::Args ta;
    ta.D = a.D;
    ta.batch = a.batch;
    ta.B = (int)B;
    ta.Tmax = Tmax;
    ta.wimg = ctx->trc_img.as<uint8_t>();
    ta.P = a.P;
    ta.cache = ctx->tr_cache.as<float>();
    ta.raw = a.raw;
    ta.draw = a.draw;
    ta.target_scale = a.target_scale;
    ta.n_total = a.n_total;
    ta.draw_in = a.draw_in;
    ta.partial = ctx->tr_partial.as<double>();
    ta.rows = rows;
    ta.dmax = reinterpret_cast<unsigned*>(ctx->tr_partial.as<double>() + (size_t)n_tiles * L.n);
    TS_CUDA(cudaMemsetAsync(ta.dmax, 0, sizeof(unsigned), ctx->stream));
    trc::k_trc_pack<<<32, 256, 0, ctx->stream>>>(a.P, ctx->trc_img.as<uint8_t>());
    TS_LAUNCHED();
    trc::k_trc_fwd<<<n_tiles, trc::FWD_THREADS, trc::FWD_SMEM, ctx->stream>>>(ta);
    TS_LAUNCHED();
    trc::k_trc_bwd<<<n_tiles, trc::BWD_THREADS, trc::BWD_SMEM, ctx->stream>>>(ta);
    TS_LAUNCHED();
    tr::k_train_reduce<<<(L.n + 63) / 64, 64, 0, ctx->stream>>>(ctx->tr_partial.as<double>(), n_tiles, L.n, grad);
    TS_LAUNCHED();
  } else if (mode == TS_TRAIN_TC) {
    // fp64 recurrences, weight gradients on the tensor cores fused into BPTT
    if (H != tr::GH) return fail(ctx, TS_ERR_ARG, "tensor-core training needs hidden size 32");
    TS_CUDA(ctx->tr_cache.reserve(sizeof(double) * B * Tmax * tr::CACHE_FIELDS * H, ctx->stream));
    a.cache = ctx->tr_cache.as<double>();
    const int nblk = (int)((B + tr::GS - 1) / tr::GS);
    TS_CUDA(ctx->tr_partial.reserve(sizeof(double) * nblk * L.n, ctx->stream));
    a.partial = ctx->tr_partial.as<double>();
    if (!ctx->tr_tc_attr_set) {
      TS_CUDA(cudaFuncSetAttribute(tr::k_train_fb_group<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)sizeof(tr::GroupSmem)));
      ctx->tr_tc_attr_set = true;
    }
    tr::k_train_fb_group<true><<<nblk, tr::GTHREADS, sizeof(tr::GroupSmem), ctx->stream>>>(a);
    TS_LAUNCHED();
    tr::k_train_reduce<<<(L.n + 63) / 64, 64, 0, ctx->stream>>>(ctx->tr_partial.as<double>(), nblk, L.n, grad);
    TS_LAUNCHED();
  } else {
    TS_CUDA(ctx->tr_cache.reserve(sizeof(double) * B * Tmax * tr::CACHE_FIELDS * H, ctx->stream));
    TS_CUDA(ctx->tr_dz.reserve(sizeof(double) * K * (grouped ? tr::PROW : L.G), ctx->stream));
    a.cache = ctx->tr_cache.as<double>();
    a.dz = ctx->tr_dz.as<double>();
    int ksplit;
    if (grouped) {
      TS_CUDA(ctx->tr_pvalid.reserve(K, ctx->stream));
      TS_CUDA(cudaMemsetAsync(ctx->tr_pvalid.p, 0, K, ctx->stream));
      a.pvalid = ctx->tr_pvalid.as<uint8_t>();
      // grouped kernels (bit-identical forward/BPTT; weight gradients in the
      // same pair order within each of ksplit ranges)
      if (!ctx->tr_group_attr_set) {
        TS_CUDA(cudaFuncSetAttribute(tr::k_train_fb_group<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(tr::GroupSmem)));
        ctx->tr_group_attr_set = true;
      }
      tr::k_train_fb_group<false><<<(unsigned)((B + tr::GS - 1) / tr::GS), tr::GTHREADS, sizeof(tr::GroupSmem),
                                    ctx->stream>>>(a);
      TS_LAUNCHED();
      ksplit = (int)std::min<int64_t>(2 * ctx->sm_count, std::max<int64_t>(1, K / 64));
      TS_CUDA(ctx->tr_partial.reserve(sizeof(double) * ksplit * L.n, ctx->stream));
      tr::k_train_wgrad_group<<<ksplit, tr::GTHREADS, sizeof(tr::WgradSmem), ctx->stream>>>(
          a, ksplit, ctx->tr_partial.as<double>());
      TS_LAUNCHED();
    } else {
      tr::k_train_fb<<<(unsigned)((B * 32 + 127) / 128), 128, 0, ctx->stream>>>(a);
      TS_LAUNCHED();
      ksplit = (int)std::min<int64_t>(64, std::max<int64_t>(1, K / 512));
      TS_CUDA(ctx->tr_partial.reserve(sizeof(double) * ksplit * L.n, ctx->stream));
      tr::k_train_wgrad<<<dim3((L.n + 255) / 256, ksplit), 256, 0, ctx->stream>>>(a, ksplit,
                                                                                 ctx->tr_partial.as<double>());
      TS_LAUNCHED();
    }
    tr::k_train_reduce<<<(L.n + 63) / 64, 64, 0, ctx->stream>>>(ctx->tr_partial.as<double>(), ksplit, L.n, grad);
    TS_LAUNCHED();
  }
  if (raw_out) {
    TS_CUDA(cudaMemcpyAsync(raw_out, a.raw, sizeof(double) * B, cudaMemcpyDeviceToHost, ctx->stream));
    TS_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  return TS_OK;
}

// Gradient of the loss over this rank's part of a minibatch whose global size
// is n_total (d_raw divides by it); written to d_grad (device pointer, or the
// context's buffer when null).  Data-parallel callers all-reduce d_grad.
int ts_train_grads(ts_ctx* ctx, const int32_t* idx, int64_t B, int64_t n_total, double target_scale,
                   double* d_grad, double* raw_out) {
  if (!ctx || !idx || B < 0 || n_total < 1) return TS_ERR_ARG;
  TS_NEED_DEVICE();
  if (!ctx->tr_H) return fail(ctx, TS_ERR_STATE, "no training data loaded");
  TS_CUDA(cudaSetDevice(ctx->device));
  const tr::Layout L(ctx->tr_H);
  double* grad = d_grad ? d_grad : ctx->tr_grad.as<double>();
  if (B == 0) {
    TS_CUDA(cudaMemsetAsync(grad, 0, sizeof(double) * L.n, ctx->stream));
    return TS_OK;
  }
  tr::TrainArgs a;
  int rc = train_args(ctx, idx, B, a);
  if (rc) return rc;
  a.target_scale = target_scale;
  a.n_total = (double)n_total;
  return launch_grads(ctx, a, ctx->tr_mode, grad, raw_out);
}

// backend.lstm_backward (_recurrent_np.py:62-96): gradients of
// sum_b d_raw[b] * raw[b] for a dense batch X [B][T][F] under the given
// weights, fp64 throughout (the forward is recomputed on the device; the
// reference's activation cache never crosses the boundary).  Independent of
// the context's training dataset and parameters.
int ts_lstm_backward(ts_ctx* ctx, const double* X, int64_t B, int64_t T, int64_t Fin, const double* Wx,
                     const double* Wh, const double* b, const double* w, int64_t H, double b_out,
                     const double* d_raw, double* grad_out) {
  if (!ctx || !X || !Wx || !Wh || !b || !w || !d_raw || !grad_out || B < 0 || T < 0) return TS_ERR_ARG;
  TS_NEED_DEVICE();
  if (Fin != F) return fail(ctx, TS_ERR_ARG, "feature width must be 16");
  if (H < 1 || H > 32) return fail(ctx, TS_ERR_ARG, "hidden size must be in 1..32");
  if (B > (int64_t)1 << 30 || T > 4096) return fail(ctx, TS_ERR_ARG, "batch or sequence too long");
  TS_CUDA(cudaSetDevice(ctx->device));
  const tr::Layout L((int)H);
  std::vector<double> flat(L.n);
  memcpy(flat.data() + L.oWx, Wx, sizeof(double) * F * L.G);
  memcpy(flat.data() + L.oWh, Wh, sizeof(double) * H * L.G);
  memcpy(flat.data() + L.ob, b, sizeof(double) * L.G);
  memcpy(flat.data() + L.ow, w, sizeof(double) * H);
  flat[L.obout] = b_out;
  if (B == 0 || T == 0) {  // dWx = dWh = db = dw = 0, db_out = T * sum(d_raw)
    double s = 0.0;
    for (int64_t i = 0; i < B; ++i) s += d_raw[i];
    memset(grad_out, 0, sizeof(double) * L.n);
    grad_out[L.obout] = (double)T * s;
    return TS_OK;
  }
  // the batch as a training dataset: sequence i = init rows i*T .. i*T+T-1
  // (no scheduled rows), batch = 0..B-1, d_raw given
  if (B * T > INT32_MAX) return fail(ctx, TS_ERR_ARG, "batch x sequence too large");
  std::vector<int32_t> meta(3 * B + B);
  std::vector<int64_t> rb(B, 0);
  for (int64_t i = 0; i < B; ++i) {
    meta[i] = (int32_t)(i * T);      // init_base
    meta[B + i] = (int32_t)T;        // Tlen
    meta[2 * B + i] = 0;             // depth
    meta[3 * B + i] = (int32_t)i;    // batch
  }
  TS_CUDA(ctx->bk_X.reserve(sizeof(double) * B * T * F, ctx->stream));
  TS_CUDA(ctx->bk_meta.reserve(sizeof(int32_t) * 4 * B + sizeof(int64_t) * B, ctx->stream));
  TS_CUDA(ctx->bk_P.reserve(sizeof(double) * (L.n + L.n + 2 * B), ctx->stream));
  TS_CUDA(ctx->tr_raw.reserve(sizeof(double) * B, ctx->stream));
  TS_CUDA(ctx->tr_draw.reserve(sizeof(double) * B, ctx->stream));
  int32_t* dmeta = ctx->bk_meta.as<int32_t>();
  int64_t* drb = reinterpret_cast<int64_t*>(dmeta + 4 * B);
  double* dP = ctx->bk_P.as<double>();
  double* dgrad = dP + L.n;
  double* ddraw = dgrad + L.n;
  TS_CUDA(cudaMemcpyAsync(ctx->bk_X.p, X, sizeof(double) * B * T * F, cudaMemcpyHostToDevice, ctx->stream));
  TS_CUDA(cudaMemcpyAsync(dmeta, meta.data(), sizeof(int32_t) * 4 * B, cudaMemcpyHostToDevice, ctx->stream));
  TS_CUDA(cudaMemcpyAsync(drb, rb.data(), sizeof(int64_t) * B, cudaMemcpyHostToDevice, ctx->stream));
  TS_CUDA(cudaMemcpyAsync(dP, flat.data(), sizeof(double) * L.n, cudaMemcpyHostToDevice, ctx->stream));
  TS_CUDA(cudaMemcpyAsync(ddraw, d_raw, sizeof(double) * B, cudaMemcpyHostToDevice, ctx->stream));
  tr::TrainArgs a;
  memset(&a, 0, sizeof a);
  a.D.rows = ctx->bk_X.as<double>();
  a.D.init = ctx->bk_X.as<double>();
  a.D.row_base = drb;
  a.D.init_base = dmeta;
  a.D.Tlen = dmeta + B;
  a.D.depth = dmeta + 2 * B;
  a.D.logt = ddraw;  // unused (draw_in)
  a.batch = dmeta + 3 * B;
  a.P = dP;
  a.draw = ctx->tr_draw.as<double>();
  a.raw = ctx->tr_raw.as<double>();
  a.B = (int)B;
  a.Tmax = (int)T;
  a.H = (int)H;
  a.n_total = 1.0;
  a.draw_in = ddraw;
  int rc = launch_grads(ctx, a, TS_TRAIN_EXACT, dgrad, nullptr);
  if (rc) return rc;
  TS_CUDA(cudaMemcpyAsync(grad_out, dgrad, sizeof(double) * L.n, cudaMemcpyDeviceToHost, ctx->stream));
  TS_CUDA(cudaStreamSynchronize(ctx->stream));
  return TS_OK;
}

// _clip + SGD step with the gradient in d_grad (or the context buffer).
int ts_train_apply(ts_ctx* ctx, const double* d_grad, double lr, double clip_norm, double* norm_out) {
  if (!ctx) return TS_ERR_ARG;
  TS_NEED_DEVICE();
  if (!ctx->tr_H) return fail(ctx, TS_ERR_STATE, "no training data loaded");
  const tr::Layout L(ctx->tr_H);
  const double* grad = d_grad ? d_grad : ctx->tr_grad.as<double>();
  tr::k_train_apply<<<1, 1024, 0, ctx->stream>>>(ctx->tr_P.as<double>(), grad, L.n, lr, clip_norm,
                                                 ctx->tr_norm.as<double>());
  TS_LAUNCHED();
  if (norm_out) {
    TS_CUDA(cudaMemcpyAsync(norm_out, ctx->tr_norm.p, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    TS_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  return TS_OK;
}

// raw scores of dataset entries idx[0..n) under the current training params.
int ts_train_forward(ts_ctx* ctx, const int32_t* idx, int64_t n, double* raw_out) {
  if (!ctx || !idx || !raw_out || n < 0) return TS_ERR_ARG;
  TS_NEED_DEVICE();
  if (!ctx->tr_H) return fail(ctx, TS_ERR_STATE, "no training data loaded");
  if (n == 0) return TS_OK;
  tr::TrainArgs a;
  int rc = train_args(ctx, idx, n, a);
  if (rc) return rc;
  tr::k_train_fwd<<<(unsigned)((n * 32 + 127) / 128), 128, 0, ctx->stream>>>(a);
  TS_LAUNCHED();
  TS_CUDA(cudaMemcpyAsync(raw_out, ctx->tr_raw.p, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  TS_CUDA(cudaStreamSynchronize(ctx->stream));
  return TS_OK;
}

}  // extern "C"
