// api.cu -- C ABI (include/rsvd_b200.h) and the host orchestrator of the
// randomized SVD hot path.  Host code only; every numerical step runs in the
// kernels of pass_ozaki.cu / pass_tf32.cu / gemm_pass.cu / omega.cu /
// cholqr.cu / panel.cu / jacobi.cu / qrcp.cu / ialm.cu on ctx->stream.
//
// Pass schedule of one rsvd (Alg. 4 + Alg. 2 + Alg. 5):
//   K1 Omega -> X                                   (Alg. 4 step 2)
//   K2 Y = A X                                      (step 3; pass 1)
//   q x [ orth(Y) -> Q ; K3 Z = A^T Q (+allreduce) ; orth(Z) ; K2 Y = A Z ]   (Alg. 2)
//   orth(Y) -> Q ; K3 B^T = A^T Q (+allreduce)      (steps 9, 10; pass 2q+2)
//   orth(B^T) -> Q_B, R_B ; Jacobi(R_B^T) -> Sigma, U~ (= W), J
//   V = Q_B J ; signs from V (reading R9) ; U = Q (U~ diag(sgn))   (Alg. 5 steps 2-3)
// orth = CholeskyQR (intermediate) / CholeskyQR2 (final) with a breakdown bit
// in the call's status word; the Householder TSQR fallback kernels are
// enqueued behind every CholeskyQR and run only once that bit is set (device
// predicate).  Panels that fit one CTA use Householder QR
// directly.  No call synchronises with the host except rsvd_sync, rsvd_rrpca
// and rsvd_run_host.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvtx3.hpp>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/rsvd_b200.h"
#include "common.cuh"
#include "kernels.h"

using namespace rsvd;

namespace {

// bits of the call's status word flags_dev[0] (flags_dev[8] = Jacobi sweeps)
constexpr int kFlagCholBreak = 1,   // a CholeskyQR broke down: the TSQR fallback runs (not an error)
              kFlagJacobiCap = 2,   // one-sided Jacobi hit the sweep cap (error)
              kFlagNonFinite = 4,   // non-finite input / intermediate (error)
              kFlagRankDef = 8,     // rid / rcur: numerical rank of the pivoted QR < k (error)
              kFlagLuZero = 16,     // informational: an exactly zero LU pivot (multipliers set to 0)
              kFlagNoFallback = 32, // a breakdown with no TSQR fallback possible for the shape (error)
              kFlagWideBreak = 64;  // CholeskyQR breakdown in a wide plan (l > kMaxL; error, reading R34)
constexpr int kMaxL = 120;       // Jacobi + leaf QR shared-memory envelope
constexpr int kMaxWide = 4096;   // wide plans (l > kMaxL, wide.cu): l x l factors in global memory

struct ProfRec { int kind; double bytes; cudaEvent_t a, b; };

}  // namespace

// ----------------------------------------------------------------- collectives
// The row-sharded path needs sum / max allreduces and one allgather; they are
// behind this interface so that the same orchestration runs over NCCL (one
// process per GPU) or over an in-process rank group (rsvd_group).
struct Comm {
  virtual ~Comm() {}
  virtual int nranks() const = 0;
  virtual int rank() const = 0;
  virtual rsvd_status allreduce(rsvd_ctx* ctx, double* buf, size_t n, bool op_max) = 0;
  virtual rsvd_status allgather(rsvd_ctx* ctx, const double* send, double* recv, size_t n) = 0;
  // a member returns an error from a call: peers must not wait for it
  virtual void on_error() {}
};

struct rsvd_group {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool aborted = false;
  struct Slot {
    double* stage = nullptr; size_t cap = 0; int device = 0;
    cudaEvent_t ready = nullptr, done = nullptr; bool done_valid = false;
    bool joined = false;
  };
  std::vector<Slot> slots;
  // host barrier over the n member threads; false if the group was aborted
  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) return false;
    const uint64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    cv.wait(lk, [&] { return gen != g || aborted; });
    return !aborted;
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    aborted = true;
    cv.notify_all();
  }
};

struct rsvd_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  std::string err;
  // workspace (grown on demand; kept between calls)
  char* ws = nullptr;
  size_t ws_bytes = 0;
  char* ws2 = nullptr;            // TSQR stacks, LU / pivoted-QR scratch
  size_t ws2_bytes = 0;
  int* flags_dev = nullptr;       // the call's status word (16 ints); [64, 128): launch_tsqr_fused's words
  int* sticky_dev = nullptr;      // accumulated status for rsvd_sync (4 ints)
  int* flags_host = nullptr;      // pinned
  int* sweeps_dev = nullptr;
  double* hbuf = nullptr;         // pinned host scratch (small D2H/H2D transfers)
  char* ws3 = nullptr;            // rrpca buffers
  size_t ws3_bytes = 0;
  char* ws5 = nullptr;            // rsvd_run_host device staging
  size_t ws5_bytes = 0;
  // comm
  Comm* comm = nullptr;
  int nranks = 1, rank = 0;
  // profiling
  int prof = 0;                   // 0 off, 1 every kind, 2 the pass kernels only (kinds 0, 1, 6)
  int prof_phase = 0;             // level 2: the pass kind (0 / 1) timed in this call, alternating per call
  bool debug = getenv("RSVD_DEBUG") != nullptr;
  std::vector<ProfRec> pending;
  std::vector<cudaEvent_t> pool;
  double prof_ms[7] = {0, 0, 0, 0, 0, 0, 0};
  double prof_bytes[7] = {0, 0, 0, 0, 0, 0, 0};
  int64_t prof_count[7] = {0, 0, 0, 0, 0, 0, 0};
  int last_sweeps = 0;
  bool fp32_tcgen05 = true;       // RSVD_FP32_PATH=dmma selects the FP64-DMMA path for FP32 inputs
  bool fp64_ozaki = true;         // RSVD_FP64_PATH=dmma selects the DMMA path for FP64 inputs
  bool fp32_ozaki = true;         // FP32 A: 3-digit Ozaki slices (RSVD_FP32_PATH=tf32: 3xTF32 passes, =dmma: CUDA cores)
  char* ws4 = nullptr;            // Ozaki slices of A (+ X slice scratch)
  size_t ws4_bytes = 0;
  int64_t ozaki_calls = 0;
  int last_robust = 0;
  unsigned* gemm_flags = nullptr; // stream-K fix-up flags / counters (4096, zeroed at creation)
  unsigned gemm_epoch = 0;
};

namespace {

rsvd_status fail(rsvd_ctx* c, rsvd_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) {
    c->err = buf;
    if (c->comm) c->comm->on_error();   // an in-process rank group is aborted (its peers return RSVD_ENCCL)
  }
  return s;
}

#define CK(expr)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(ctx, RSVD_ECUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                    \
  } while (0)

#define CKS(expr)                         \
  do {                                    \
    rsvd_status s_ = (expr);              \
    if (s_ != RSVD_OK) return s_;         \
  } while (0)

// ----------------------------------------------------------------- NCCL / group communicators
struct NcclComm : Comm {
  ncclComm_t c = nullptr;
  int n = 1, r = 0;
  ~NcclComm() override { if (c) ncclCommDestroy(c); }
  int nranks() const override { return n; }
  int rank() const override { return r; }
  rsvd_status allreduce(rsvd_ctx* ctx, double* buf, size_t cnt, bool op_max) override {
    const rsvd_status s = allreduce_(ctx, buf, cnt, op_max);
    if (s != RSVD_OK) return s;
    CK(launch_stream_fence(ctx->stream));
    return RSVD_OK;
  }
  rsvd_status allreduce_(rsvd_ctx* ctx, double* buf, size_t cnt, bool op_max) {
    ncclResult_t e = ncclAllReduce(buf, buf, cnt, ncclDouble, op_max ? ncclMax : ncclSum, c, ctx->stream);
    ncclResult_t async = ncclSuccess;
    if (e == ncclSuccess && ncclCommGetAsyncError(c, &async) == ncclSuccess && async != ncclSuccess &&
        async != ncclInProgress)
      e = async;
    if (e != ncclSuccess) return fail(ctx, RSVD_ENCCL, "ncclAllReduce: %s", ncclGetErrorString(e));
    return RSVD_OK;
  }
  rsvd_status allgather(rsvd_ctx* ctx, const double* send, double* recv, size_t cnt) override {
    const ncclResult_t e = ncclAllGather(send, recv, cnt, ncclDouble, c, ctx->stream);
    if (e != ncclSuccess) return fail(ctx, RSVD_ENCCL, "ncclAllGather: %s", ncclGetErrorString(e));
    CK(launch_stream_fence(ctx->stream));
    return RSVD_OK;
  }
};

// In-process rank group: rank r stages its buffer, every rank then reduces all
// the stages in rank order into its own buffer (identical bits everywhere).
// Two host barriers per collective; a rank's stage is rewritten only after
// every rank's reduction that read it (the previous `done` events) finished.
struct GroupComm : Comm {
  rsvd_group* g = nullptr;
  int r = 0;
  void on_error() override { g->abort(); }
  int nranks() const override { return g->n; }
  int rank() const override { return r; }
  rsvd_status stage(rsvd_ctx* ctx, const double* src, size_t cnt) {
    rsvd_group::Slot& me = g->slots[r];
    if (me.cap < cnt) {
      // every member's reduction of the previous collective may still read this
      // stage: wait for all of them (their `done` events precede the last barrier)
      for (int s = 0; s < g->n; ++s)
        if (g->slots[s].done_valid) cudaEventSynchronize(g->slots[s].done);
      cudaStreamSynchronize(ctx->stream);
      if (me.stage) cudaFree(me.stage);
      me.stage = nullptr; me.cap = 0;
      const size_t cap = std::max(cnt, (size_t)1 << 16);   // >= 512 KB: few regrowths
      if (cudaMalloc(&me.stage, cap * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        g->abort();
        return fail(ctx, RSVD_ENOMEM, "rank group staging of %zu doubles failed", cap);
      }
      me.cap = cap;
    }
    for (int s = 0; s < g->n; ++s)
      if (g->slots[s].done_valid) CK(cudaStreamWaitEvent(ctx->stream, g->slots[s].done, 0));
    CK(cudaMemcpyAsync(me.stage, src, cnt * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaEventRecord(me.ready, ctx->stream));
    if (!g->barrier()) return fail(ctx, RSVD_ENCCL, "rank group aborted by another member");
    for (int s = 0; s < g->n; ++s) CK(cudaStreamWaitEvent(ctx->stream, g->slots[s].ready, 0));
    return RSVD_OK;
  }
  rsvd_status finish(rsvd_ctx* ctx) {
    rsvd_group::Slot& me = g->slots[r];
    CK(cudaEventRecord(me.done, ctx->stream));
    me.done_valid = true;
    if (!g->barrier()) return fail(ctx, RSVD_ENCCL, "rank group aborted by another member");
    return RSVD_OK;
  }
  rsvd_status allreduce(rsvd_ctx* ctx, double* buf, size_t cnt, bool op_max) override {
    rsvd_status s = stage(ctx, buf, cnt);
    if (s != RSVD_OK) { g->abort(); return s; }
    GroupPtrs in{};
    for (int q = 0; q < g->n; ++q) in.p[q] = g->slots[q].stage;
    const cudaError_t e = launch_group_reduce(in, g->n, (int64_t)cnt, op_max ? 1 : 0, buf, ctx->stream);
    if (e != cudaSuccess) { g->abort(); return fail(ctx, RSVD_ECUDA, "group reduce: %s", cudaGetErrorString(e)); }
    return finish(ctx);
  }
  rsvd_status allgather(rsvd_ctx* ctx, const double* send, double* recv, size_t cnt) override {
    rsvd_status s = stage(ctx, send, cnt);
    if (s != RSVD_OK) { g->abort(); return s; }
    for (int q = 0; q < g->n; ++q) {
      const cudaError_t e = cudaMemcpyAsync(recv + (size_t)q * cnt, g->slots[q].stage, cnt * sizeof(double),
                                            cudaMemcpyDeviceToDevice, ctx->stream);
      if (e != cudaSuccess) { g->abort(); return fail(ctx, RSVD_ECUDA, "group allgather: %s", cudaGetErrorString(e)); }
    }
    CK(launch_stream_fence(ctx->stream));
    return finish(ctx);
  }
};

cudaEvent_t take_event(rsvd_ctx* c) {
  if (!c->pool.empty()) {
    cudaEvent_t e = c->pool.back();
    c->pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// NVTX ranges (header-only nvtx3: no-ops unless a profiler such as nsys is
// attached) around the enqueue of each phase, named as bench.py's per-kind split
static const char* const kKindName[7] = {"rsvd:pass_AX", "rsvd:pass_AtX", "rsvd:panel_orth", "rsvd:jacobi_svd",
                                         "rsvd:omega", "rsvd:ozaki_slice_A", "rsvd:ozaki_slice_X"};
struct Prof {
  rsvd_ctx* c; int kind; double bytes; cudaEvent_t a = nullptr;
  Prof(rsvd_ctx* c_, int k, double b) : c(c_), kind(k), bytes(b) {
    nvtxRangePushA(kind >= 0 && kind < 7 ? kKindName[kind] : "rsvd");
    if (on()) { a = take_event(c); cudaEventRecord(a, c->stream); }
  }
  bool on() const { return c->prof == 1 || (c->prof == 2 && kind == c->prof_phase); }
  ~Prof() {
    nvtxRangePop();
    if (on()) {
      cudaEvent_t b2 = take_event(c);
      cudaEventRecord(b2, c->stream);
      c->pending.push_back({kind, bytes, a, b2});
    }
  }
};

void prof_collect(rsvd_ctx* c) {
  for (auto& r : c->pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) {
      c->prof_ms[r.kind] += ms;
      c->prof_bytes[r.kind] += r.bytes;
      c->prof_count[r.kind] += 1;
    }
    c->pool.push_back(r.a);
    c->pool.push_back(r.b);
  }
  c->pending.clear();
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// ----------------------------------------------------------------- workspace plan
struct Plan {
  int64_t M, n;      // local rows, columns (after the m < n transpose swap: M x n "A")
  int l, Np;         // sketch width, padded width (multiple of 16)
  bool f32;
  bool trans_input;  // single-GPU m < n: work on A^T without copying
  bool scaled = false;  // implicit column scaling active (rpca scale = TRUE)
  const void* A; int64_t lda;
  int64_t m_global;
  // workspace offsets
  size_t oW0 = 0;
  size_t oX, oY, oT, oZ, oPart, oSmall, oColc, oColr, oColp, oColss, oSplit, oJlog, total;
  bool use_tf32 = false;          // FP32 A on tcgen05 (3-term TF32 split)
  bool use_ozaki = false;         // FP64 A on tcgen05 (Ozaki int8 slices)
  bool wide = false;              // l > kMaxL: DMMA column blocks, CholeskyQR2, wide Jacobi (wide.cu)
  OzakiA oz{};
  void* ozx = nullptr;            // X slice scratch
  void* ozx2 = nullptr;           // second 64-column block (Np > 64)
  size_t oz_bytes = 0;            // Ozaki slices + X scratch
  float* split = nullptr;
  void* jlog = nullptr;
  size_t part_bytes;
  // small-buffer offsets (doubles from oSmall)
  double* W0 = nullptr;           // wide plans: the panel saved for the Householder fallback
  double *X, *Y, *T, *Z, *part, *G, *Rinv, *R1, *R2, *RB, *W, *J, *sigma, *sgn, *colc, *colr, *cols, *colp, *colss,
      *Rsm, *tv;
};

bool small_panel(int64_t rows, int l) { return rows <= leaf_rows_cap(l); }

size_t plan_bytes(rsvd_ctx* ctx, Plan& p) {
  const int Np = p.Np;
  size_t part = 0;
  auto upd = [&](int64_t M, int64_t K, int N) {
    part = std::max(part, gemm_partial_bytes(std::min(N, 128), gemm_choose_grid(M, K, ctx->num_sms)));
  };
  upd(p.M, p.n, Np);       // Y = A X
  upd(p.n, p.M, Np);       // Z = A^T Q
  if (p.use_tf32) part = std::max(part, tf32_partial_bytes(Np, ctx->num_sms));
  if (p.use_ozaki) part = std::max(part, ozaki_partial_bytes(Np, ctx->num_sms));
  if (!p.wide) part = std::max(part, gram_partial_bytes(Np, ctx->num_sms));
  else upd(Np, std::max(p.M, p.n), 128);   // the Gram and small-K products of the wide panels
  p.part_bytes = part;
  const int64_t big = std::max(p.M, p.n);
  size_t o = 0;
  p.oX = o; o = align256(o + (size_t)p.n * Np * 8);
  p.oY = o; o = align256(o + (size_t)p.M * Np * 8);
  p.oT = o; o = align256(o + (size_t)big * Np * 8);
  p.oZ = o; o = align256(o + (size_t)p.n * Np * 8);
  p.oPart = o; o = align256(o + part);
  p.oSmall = o; o = align256(o + (size_t)(9 * Np * Np + 4 * Np + 8) * 8);
  p.oColc = o; o = align256(o + (size_t)p.n * 8);
  p.oColr = o; o = align256(o + (size_t)p.n * 16);
  p.oColp = o; o = align256(o + colsum_partial_bytes(p.M, p.n) + 256);
  p.oColss = o; o = align256(o + (size_t)p.n * 8);
  p.oSplit = o; o = align256(o + (p.use_tf32 ? tf32_split_bytes(big, Np) : 0));
  p.oW0 = o; o = align256(o + (p.wide ? (size_t)big * Np * 8 : 0));
  p.oJlog = o;
  o = align256(o + (p.wide ? std::max(jacobi_wide_scratch_bytes(p.l), chol_wide_scratch_bytes(Np))
                            : jacobi_scratch_bytes(p.l)));
  p.total = o;
  return o;
}

rsvd_status ensure_buf(rsvd_ctx* ctx, char** buf, size_t* have, size_t bytes, const char* what) {
  if (bytes <= *have) return RSVD_OK;
  if (*buf) { cudaStreamSynchronize(ctx->stream); cudaFree(*buf); *buf = nullptr; *have = 0; }
  if (cudaMalloc(buf, bytes) != cudaSuccess) {
    cudaGetLastError();
    return fail(ctx, RSVD_ENOMEM, "%s allocation of %zu bytes failed", what, bytes);
  }
  *have = bytes;
  return RSVD_OK;
}
rsvd_status ensure_ws(rsvd_ctx* ctx, size_t bytes) { return ensure_buf(ctx, &ctx->ws, &ctx->ws_bytes, bytes, "workspace"); }
rsvd_status ensure_ws2(rsvd_ctx* ctx, size_t bytes) { return ensure_buf(ctx, &ctx->ws2, &ctx->ws2_bytes, bytes, "TSQR / scratch workspace"); }

void bind(rsvd_ctx* ctx, Plan& p) {
  char* b = ctx->ws;
  const int Np = p.Np;
  p.X = (double*)(b + p.oX); p.Y = (double*)(b + p.oY); p.T = (double*)(b + p.oT);
  p.Z = (double*)(b + p.oZ); p.part = (double*)(b + p.oPart);
  double* s = (double*)(b + p.oSmall);
  p.G = s; s += Np * Np; p.Rinv = s; s += Np * Np; p.R1 = s; s += Np * Np; p.R2 = s; s += Np * Np;
  p.RB = s; s += Np * Np; p.W = s; s += Np * Np; p.J = s; s += Np * Np; p.Rsm = s; s += 2 * Np * Np;
  p.sigma = s; s += Np; p.sgn = s; s += Np; p.tv = s; s += 8;
  p.colc = (double*)(b + p.oColc); p.colr = (double*)(b + p.oColr); p.cols = p.colr + p.n; p.colp = (double*)(b + p.oColp);
  p.colss = (double*)(b + p.oColss);
  p.split = (float*)(b + p.oSplit);
  p.jlog = (void*)(b + p.oJlog);
  if (p.wide) p.W0 = (double*)(b + p.oW0);
}

rsvd_status allreduce_sum(rsvd_ctx* ctx, double* buf, size_t count) {
  if (!ctx->comm || count == 0) return RSVD_OK;   // one rank has no communicator (but see RSVD_NCCL_SINGLE)
  return ctx->comm->allreduce(ctx, buf, count, false);
}
rsvd_status allreduce_max(rsvd_ctx* ctx, double* buf, size_t count) {
  if (!ctx->comm || count == 0) return RSVD_OK;
  return ctx->comm->allreduce(ctx, buf, count, true);
}
rsvd_status allgather(rsvd_ctx* ctx, const double* send, double* recv, size_t count) {
  return ctx->comm->allgather(ctx, send, recv, count);
}

// ----------------------------------------------------------------- passes over A
// Y (M x Np) = f(A) X  (K2).   With trans_input the stored matrix is A^T (n x M
// row-major), so this is the TN form of the stored matrix.
rsvd_status pass_tf32(rsvd_ctx* ctx, Plan& p, bool trans, const double* B, double* C, int64_t M, int64_t K) {
  Tf32Call t{};
  t.A = (const float*)p.A; t.lda = p.lda; t.trans = trans;
  t.B = B; t.ldb = p.Np; t.C = C; t.ldc = p.Np; t.P = p.part; t.split = p.split;
  t.M = M; t.K = K; t.N = p.Np; t.Nout = p.Np; t.grid = ctx->num_sms;
  t.flags = ctx->gemm_flags; t.epoch = ++ctx->gemm_epoch;
  CK(tf32_pass(t, ctx->stream));
  return RSVD_OK;
}

// One Ozaki pass: profile kind 6 = X slicing, `kind` (0 / 1) = the pass kernel(s)
rsvd_status pass_ozaki(rsvd_ctx* ctx, Plan& p, bool trans, const double* B, double* C, int64_t M, int64_t K,
                       int kind) {
  nvtx3::scoped_range_in<nvtx3::domain::global> nv{kind == 0 ? "rsvd:pass_AX (ozaki)" : "rsvd:pass_AtX (ozaki)"};
  OzakiCall o{};
  o.a = &p.oz; o.trans = trans; o.B = B; o.ldb = p.Np; o.C = C; o.ldc = p.Np; o.Nout = p.Np;
  o.P = p.part; o.flags = ctx->gemm_flags; o.epoch = ++ctx->gemm_epoch; o.epoch2 = ++ctx->gemm_epoch;
  o.xscratch = p.ozx; o.xscratch2 = p.ozx2;
  o.M = M; o.K = K; o.N = p.Np; o.grid = ctx->num_sms;
  ++ctx->ozaki_calls;
  if (!ctx->prof || (ctx->prof == 2 && kind != ctx->prof_phase)) {
    CK(ozaki_pass(o, ctx->stream));
    return RSVD_OK;
  }
  // level 2: only the pass kernel(s) (2 events); level 1 also the X slicing
  const bool all = ctx->prof == 1;
  cudaEvent_t e0 = all ? take_event(ctx) : nullptr, e1 = all ? take_event(ctx) : nullptr;
  cudaEvent_t e1b = take_event(ctx), e2 = take_event(ctx);
  if (all) cudaEventRecord(e0, ctx->stream);
  o.mark = e1; o.mark2 = e1b;
  CK(ozaki_pass(o, ctx->stream));
  cudaEventRecord(e2, ctx->stream);
  if (all) ctx->pending.push_back({6, 0.0, e0, e1});
  ctx->pending.push_back({kind, (double)p.M * p.n * (p.f32 ? 4 : 8), e1b, e2});
  return RSVD_OK;
}

// C (M x Nout, ld ldc) = f(Aop) (M x K) * B (K x N, ld ldb) as DMMA gemm_pass
// launches over column blocks of <= 128 (wide plans; N % 16 == 0).  C must not
// alias A or B: every block re-reads the whole of A.
rsvd_status gemm_blocks(rsvd_ctx* ctx, Plan& p, const void* A, int64_t lda, bool a_f32, bool trans,
                        const double* center, const double* rscale, const double* B, int64_t ldb, int N, double* C,
                        int64_t ldc, int Nout, int64_t M, int64_t K) {
  for (int j0 = 0; j0 < N && j0 < Nout; j0 += 128) {
    GemmCall g{};
    g.A = A; g.lda = lda; g.a_f32 = a_f32; g.trans = trans;
    g.B = B + j0; g.ldb = ldb; g.C = C + j0; g.ldc = ldc; g.P = p.part;
    g.center = center; g.rscale = rscale;
    g.M = M; g.K = K; g.N = std::min(128, N - j0); g.Nout = std::min(g.N, Nout - j0);
    g.grid = ctx->num_sms;
    g.flags = ctx->gemm_flags; g.epoch = ++ctx->gemm_epoch;
    CK(gemm_pass(g, ctx->stream));
  }
  return RSVD_OK;
}

rsvd_status pass_ax(rsvd_ctx* ctx, Plan& p, const double* X, double* Y, bool centred) {
  if (p.wide) {
    Prof pr(ctx, 0, (double)p.M * p.n * (p.f32 ? 4 : 8));
    return gemm_blocks(ctx, p, p.A, p.lda, p.f32, p.trans_input, centred ? p.colc : nullptr,
                       p.scaled ? p.colr : nullptr, X, p.Np, p.Np, Y, p.Np, p.Np, p.M, p.n);
  }
  if (p.use_ozaki) return pass_ozaki(ctx, p, p.trans_input, X, Y, p.M, p.n, 0);
  if (p.use_tf32 && !centred) {
    Prof pr(ctx, 0, (double)p.M * p.n * 4);
    return pass_tf32(ctx, p, p.trans_input, X, Y, p.M, p.n);
  }
  GemmCall g{};
  g.A = p.A; g.lda = p.lda; g.a_f32 = p.f32; g.trans = p.trans_input;
  g.B = X; g.ldb = p.Np; g.C = Y; g.ldc = p.Np; g.P = p.part;
  g.center = centred ? p.colc : nullptr;
  g.rscale = p.scaled ? p.colr : nullptr;
  g.M = p.M; g.K = p.n; g.N = p.Np; g.Nout = p.Np;
  g.grid = ctx->num_sms;
  g.flags = ctx->gemm_flags; g.epoch = ++ctx->gemm_epoch;
  const double bytes = (double)p.M * p.n * (p.f32 ? 4 : 8);
  Prof pr(ctx, 0, bytes);
  CK(gemm_pass(g, ctx->stream));
  return RSVD_OK;
}

// Z (n x Np) = f(A)^T Q (K3), then allreduce over ranks.
rsvd_status pass_atx(rsvd_ctx* ctx, Plan& p, const double* Q, double* Z, bool centred) {
  if (p.wide) {
    {
      Prof pr(ctx, 1, (double)p.M * p.n * (p.f32 ? 4 : 8));
      CKS(gemm_blocks(ctx, p, p.A, p.lda, p.f32, !p.trans_input, centred ? p.colc : nullptr,
                      p.scaled ? p.colr : nullptr, Q, p.Np, p.Np, Z, p.Np, p.Np, p.n, p.M));
    }
    return allreduce_sum(ctx, Z, (size_t)p.n * p.Np);
  }
  if (p.use_ozaki) {
    CKS(pass_ozaki(ctx, p, !p.trans_input, Q, Z, p.n, p.M, 1));
    return allreduce_sum(ctx, Z, (size_t)p.n * p.Np);
  }
  if (p.use_tf32 && !centred) {
    {
      Prof pr(ctx, 1, (double)p.M * p.n * 4);
      CKS(pass_tf32(ctx, p, !p.trans_input, Q, Z, p.n, p.M));
    }
    return allreduce_sum(ctx, Z, (size_t)p.n * p.Np);
  }
  GemmCall g{};
  g.A = p.A; g.lda = p.lda; g.a_f32 = p.f32; g.trans = !p.trans_input;
  g.B = Q; g.ldb = p.Np; g.C = Z; g.ldc = p.Np; g.P = p.part;
  g.center = centred ? p.colc : nullptr;
  g.rscale = p.scaled ? p.colr : nullptr;
  g.M = p.n; g.K = p.M; g.N = p.Np; g.Nout = p.Np;
  g.grid = ctx->num_sms;
  g.flags = ctx->gemm_flags; g.epoch = ++ctx->gemm_epoch;
  const double bytes = (double)p.M * p.n * (p.f32 ? 4 : 8);
  {
    Prof pr(ctx, 1, bytes);
    CK(gemm_pass(g, ctx->stream));
  }
  return allreduce_sum(ctx, Z, (size_t)p.n * p.Np);
}

// C (rows x Nout) = S (rows x Np) * Bsm (Np x Np) (small-K product, panel_apply)
rsvd_status small_k(rsvd_ctx* ctx, Plan& p, const double* S, int64_t rows, const double* Bsm, double* C,
                    int64_t ldc, int Nout, bool upper = false, Pred pr = Pred{}) {
  if (p.wide) {
    if (C == S) return fail(ctx, RSVD_EINVAL, "internal: in-place small-K product in a wide plan");
    return gemm_blocks(ctx, p, S, p.Np, false, false, nullptr, nullptr, Bsm, p.Np, p.Np, C, ldc, Nout, rows, p.Np);
  }
  CK(launch_panel_apply(S, p.Np, rows, p.Np, Bsm, p.Np, C, ldc, Nout, upper, ctx->num_sms, ctx->stream, pr));
  return RSVD_OK;
}

// G (Np x Np) = S^T S (gram_partial + fixed-order reduce), allreduce when the
// rows are distributed (always enqueued: every rank takes part in every collective).
rsvd_status gram(rsvd_ctx* ctx, Plan& p, const double* S, int64_t rows, bool dist, Pred pr) {
  CK(launch_gram(S, p.Np, rows, p.Np, p.part, p.G, p.Np, ctx->num_sms, ctx->stream, pr));
  if (dist) return allreduce_sum(ctx, p.G, (size_t)p.Np * p.Np);
  return RSVD_OK;
}

// TSQR level structure of a rows x l panel: leaves of <= leaf_rows_cap(l) rows,
// their R factors stacked, repeated until one leaf remains.  Returns false if
// the panel cannot be reduced (fewer than l rows per leaf).
bool tsqr_levels(int64_t rows, int l, std::vector<int64_t>* leaves, size_t* stack_bytes) {
  const int cap = leaf_rows_cap(l);
  int64_t Mc = rows;
  size_t need = 0;
  while (Mc > cap) {
    int64_t P = ceil_div(Mc, cap);
    if (Mc / P < l) P = Mc / l;
    if (P < 1 || P * l >= Mc) return false;
    need += align256((size_t)P * l * l * 8);
    if (leaves) leaves->push_back(P);
    Mc = P * l;
  }
  if (stack_bytes) *stack_bytes = need + 256;
  return true;
}

// TSQR on the rows x l panel S (ld ld_s) on this device, one predicated
// cooperative launch (launch_tsqr_fused); R (l x l, ld l) to Rout, and also to
// Rout2 (ld ldo2) if non-null.
rsvd_status tsqr_local(rsvd_ctx* ctx, const Plan& p, double* S, int64_t ld_s, int64_t rows, double* Rout, Pred pr,
                       double* Rout2 = nullptr, int64_t ldo2 = 0) {
  const int l = p.l;
  std::vector<int64_t> leaves;
  size_t need = 0;
  if (!tsqr_levels(rows, l, &leaves, &need))
    return fail(ctx, RSVD_EUNSUPPORTED, "TSQR cannot reduce %lld rows at l = %d", (long long)rows, l);
  if ((int)leaves.size() > kTsqrMaxLev)
    return fail(ctx, RSVD_EUNSUPPORTED, "TSQR of %lld rows needs more than %d levels", (long long)rows, kTsqrMaxLev);
  CKS(ensure_ws2(ctx, need + 256));
  TsqrArgs a = {};
  char* wp = ctx->ws2;
  double* cur = S;
  int64_t ld = ld_s, Mc = rows;
  for (const int64_t P : leaves) {
    double* stack = (double*)wp;
    wp += align256((size_t)P * l * l * 8);
    a.lev[a.nlev++] = TsqrLevel{cur, ld, Mc, P};
    cur = stack; ld = l; Mc = P * l;
  }
  a.l = l;
  a.cur = cur; a.ldc = ld; a.Mc = Mc;
  a.R = Rout; a.Rout = Rout2; a.ldro = ldo2;
  a.bar = reinterpret_cast<unsigned*>(ctx->flags_dev + 64);
  CK(launch_tsqr_fused(a, ctx->num_sms, ctx->stream, pr));
  return RSVD_OK;
}

// Householder TSQR of the first l columns of S (rows x Np, ld Np), run only
// when the call's breakdown bit is set (pr).  Distributed: local TSQR, then
// the allgather of the R factors (always enqueued: every rank takes part), the
// redundant QR of the stack and Q_local <- Q_local S_rank.  R to Rout (ld Np).
rsvd_status orth_fallback(rsvd_ctx* ctx, Plan& p, double* S, int64_t rows, bool dist, double* Rout, Pred pr) {
  const int l = p.l, Np = p.Np;
  const size_t rr = (size_t)l * l;
  if (rows < l || !tsqr_levels(rows, l, nullptr, nullptr)) {
    // no Householder fallback for this shape: a breakdown becomes an error
    CK(launch_flag_or(ctx->flags_dev, kFlagNoFallback, ctx->stream, pr));
    if (dist) {   // keep the collective sequence identical on every rank
      double* stack = p.T;
      CKS(allgather(ctx, p.Rsm, stack, rr));
    }
    return RSVD_OK;
  }
  if (!dist) return tsqr_local(ctx, p, S, Np, rows, p.Rsm, pr, Rout, Np);
  CKS(tsqr_local(ctx, p, S, Np, rows, p.Rsm, pr));
  const int64_t srows = (int64_t)ctx->nranks * l;
  if ((size_t)srows * l > (size_t)std::max(p.M, p.n) * Np)
    return fail(ctx, RSVD_EUNSUPPORTED, "too many ranks for the robust panel QR workspace");
  double* stack = p.T;
  CKS(allgather(ctx, p.Rsm, stack, rr));
  double* Rg = p.Rsm + rr;
  if (srows <= leaf_rows_cap(l)) {
    CK(launch_hqr_leaves(stack, l, srows, l, 1, Rg, ctx->stream, pr));
  } else {
    CKS(tsqr_local(ctx, p, stack, l, srows, Rg, pr));
  }
  // Q_local <- Q_local S_rank (the rank's l x l block of the stack's Q), zero padded to Np x Np
  CK(launch_fill(p.Rinv, (int64_t)Np * Np, 0.0, ctx->stream));
  CK(launch_copy_in(stack + (size_t)ctx->rank * rr, false, l, l, l, l, p.Rinv, Np, ctx->stream));
  CKS(small_k(ctx, p, S, rows, p.Rinv, S, Np, Np, false, pr));
  if (Rout) CK(launch_copy_out(Rg, l, l, l, Rout, Np, false, nullptr, ctx->stream, pr));
  return RSVD_OK;
}

// Orthonormalise the first l columns of S (rows x Np, ld Np) in place.
// dist: rows are distributed over ranks.  R (l x l, ld Np) to Rout if non-null.
// exact = false: one CholeskyQR pass (intermediate subspace bases, Alg. 2
// steps 2-3: only span(Y) matters downstream); true: CholeskyQR2.  The
// CholeskyQR kernels run while the breakdown bit is clear, the Householder
// TSQR fallback once it is set (a breakdown in this or an earlier panel of
// the call): decided on the device, no host round trip.
// Wide plans (l > kMaxL): shifted CholeskyQR3 in every position (Fukaya et
// al.: one CholeskyQR of G + s I, s = 11 (m l + l (l + 1)) u ||S||_F^2, then
// CholeskyQR2), S -> T -> S -> T, copied back to S.  The Gram G = S^T S by
// gemm_pass (TN form, column blocks), R and R^-1 by the cooperative
// chol_wide_kernel.  The shift keeps the first factorisation defined for any
// numerically full-rank panel (kappa up to ~1/u, e.g. the deterministic SVD of
// a nearly low-rank IALM iterate); a panel that is rank-deficient to working
// precision breaks the second CholeskyQR: then (decided on the device) the
// cooperative Householder QR of the saved panel replaces Q and R (single GPU;
// row-sharded panels report the breakdown as RSVD_ENUMERIC, reading R34).
rsvd_status orth_wide(rsvd_ctx* ctx, Plan& p, double* S, int64_t rows, bool dist, double* Rout) {
  const int l = p.l, Np = p.Np;
  if (!dist) CK(launch_copy_out(S, Np, rows, Np, p.W0, Np, false, nullptr, ctx->stream));
  double* src = S;
  double* dst = p.T;
  double* Rs[3] = {p.Rsm, p.R1, p.R2};
  const double mrows = dist ? (double)p.m_global : (double)rows;
  const double shift_c = 11.0 * (mrows * l + (double)l * (l + 1)) * 0x1.0p-53;
  for (int it = 0; it < 3; ++it) {
    CKS(gemm_blocks(ctx, p, src, Np, false, true, nullptr, nullptr, src, Np, Np, p.G, Np, Np, Np, rows));
    if (dist) CKS(allreduce_sum(ctx, p.G, (size_t)Np * Np));
    CK(launch_chol_wide(p.G, Np, l, Np, Rs[it], p.Rinv, p.jlog, ctx->flags_dev, kFlagWideBreak,
                        it == 0 ? shift_c : 0.0, ctx->num_sms, ctx->stream));
    CKS(gemm_blocks(ctx, p, src, Np, false, false, nullptr, nullptr, p.Rinv, Np, Np, dst, Np, Np, rows, Np));
    std::swap(src, dst);
  }
  CK(launch_copy_out(src, Np, rows, Np, S, Np, false, nullptr, ctx->stream));
  // R = R3 R2 R1 (G is free again)
  if (Rout) {
    CKS(gemm_blocks(ctx, p, Rs[1], Np, false, false, nullptr, nullptr, Rs[0], Np, Np, p.G, Np, Np, Np, Np));
    CKS(gemm_blocks(ctx, p, Rs[2], Np, false, false, nullptr, nullptr, p.G, Np, Np, Rout, Np, Np, Np, Np));
  }
  if (!dist)   // a no-op launch unless a CholeskyQR above broke down
    CK(launch_hqr_wide(p.W0, rows, l, Np, S, Rout, p.part, p.jlog, ctx->flags_dev, kFlagWideBreak, kFlagCholBreak,
                       ctx->num_sms, ctx->stream));
  return RSVD_OK;
}

rsvd_status orth(rsvd_ctx* ctx, Plan& p, double* S, int64_t rows, bool dist, double* Rout, bool exact = true) {
  const int l = p.l, Np = p.Np;
  Prof pr_(ctx, 2, (double)rows * Np * 8 * 4);
  if (p.wide) return orth_wide(ctx, p, S, rows, dist, Rout);
  if (!dist && small_panel(rows, l)) {
    // register-column Householder when the panel fits (l <= 32, rows <= 1024), else in shared memory
    static const bool small_regs = [] { const char* v = getenv("RSVD_HQR_REGS"); return !v || atoi(v) != 0; }();
    const cudaError_t eh = small_regs ? launch_hqr_small(S, Np, rows, l, p.Rsm, ctx->stream) : cudaErrorNotSupported;
    if (eh == cudaErrorNotSupported) CK(launch_hqr_leaves(S, Np, rows, l, 1, p.Rsm, ctx->stream));
    else CK(eh);
    if (Rout) CK(launch_copy_out(p.Rsm, l, l, l, Rout, Np, false, nullptr, ctx->stream));
    return RSVD_OK;
  }
  const Pred ok{ctx->flags_dev, kFlagCholBreak, 0}, bad{ctx->flags_dev, kFlagCholBreak, 1};
  if (!exact) {
    CKS(gram(ctx, p, S, rows, dist, ok));
    CK(launch_chol_aug(p.G, Np, l, Np, p.R1, p.Rinv, ctx->flags_dev, kFlagCholBreak, ctx->stream, ok));
    // in place: each output row of S R^-1 depends only on the same input row
    CKS(small_k(ctx, p, S, rows, p.Rinv, S, Np, Np, true, ok));
  } else {
    // CholeskyQR2: S -> T = S R1^-1 -> S = T R2^-1 (S intact until the last step)
    CKS(gram(ctx, p, S, rows, dist, ok));
    CK(launch_chol_aug(p.G, Np, l, Np, p.R1, p.Rinv, ctx->flags_dev, kFlagCholBreak, ctx->stream, ok));
    CKS(small_k(ctx, p, S, rows, p.Rinv, p.T, Np, Np, true, ok));
    CKS(gram(ctx, p, p.T, rows, dist, ok));
    CK(launch_chol_aug(p.G, Np, l, Np, p.R2, p.Rinv, ctx->flags_dev, kFlagCholBreak, ctx->stream, ok));
    CKS(small_k(ctx, p, p.T, rows, p.Rinv, S, Np, Np, true, ok));
    if (Rout) CK(launch_panel_apply(p.R2, Np, Np, Np, p.R1, Np, Rout, Np, Np, true, ctx->num_sms, ctx->stream, ok));
  }
  return orth_fallback(ctx, p, S, rows, dist, Rout, bad);
}

rsvd_status validate(rsvd_ctx* ctx, const rsvd_matrix* A, const rsvd_params* prm, int64_t* m_out,
                     int64_t* n_out) {
  if (!ctx) return RSVD_EINVAL;
  if (!A || !prm) return fail(ctx, RSVD_EINVAL, "null argument");
  if (A->dtype != RSVD_F64 && A->dtype != RSVD_F32) return fail(ctx, RSVD_EINVAL, "dtype must be F64 or F32");
  if (!A->A) return fail(ctx, RSVD_EINVAL, "A is null");
  if (A->m_local < 1 || A->n < 1 || A->lda < A->n) return fail(ctx, RSVD_EINVAL, "bad shape or lda < n");
  const int64_t mg = ctx->nranks > 1 ? A->m_global : A->m_local;
  if (ctx->nranks > 1) {
    if (A->m_global < A->m_local || A->row_offset < 0 || A->row_offset + A->m_local > A->m_global)
      return fail(ctx, RSVD_EINVAL, "bad distributed row range");
    if (mg < A->n) return fail(ctx, RSVD_EUNSUPPORTED, "distributed mode needs m_global >= n");
  }
  const int64_t mn = std::min(mg, A->n);
  if (prm->k < 1 || prm->k > mn) return fail(ctx, RSVD_EINVAL, "k must satisfy 1 <= k <= min(m, n)");
  if (prm->p < 0 || prm->q < 0) return fail(ctx, RSVD_EINVAL, "p and q must be >= 0");
  if (prm->sdist < 0 || prm->sdist > 2) return fail(ctx, RSVD_EINVAL, "sdist must be normal, unif or rademacher");
  if (prm->nu < 0 || prm->nv < 0) return fail(ctx, RSVD_EINVAL, "nu, nv must be >= 0");
  if (prm->power < 0 || prm->power > 2) return fail(ctx, RSVD_EINVAL, "power must be 0 (Alg. 2), 1 (Alg. 1) or 2 (Alg. 3)");
  if (prm->power == 2 && ctx->nranks > 1) return fail(ctx, RSVD_EUNSUPPORTED, "Alg. 3 (pivoted LU) is single-GPU");
  *m_out = mg;
  *n_out = A->n;
  return RSVD_OK;
}

// Column statistics of rpca (Alg. 6): c (means), ss (sums of squares of
// the centred columns, when scaling or the total variance is needed), rs = 1/s.d.
rsvd_status column_stats(rsvd_ctx* ctx, Plan& p, bool centred, bool want_ss) {
  if (centred) {
    CK(launch_colsum(p.A, p.lda, p.f32, p.M, p.n, 0, nullptr, p.colp, p.colc, ctx->stream, nullptr));
    CKS(allreduce_sum(ctx, p.colc, (size_t)p.n));
    CK(launch_colstat_finish(p.colc, p.n, (double)p.m_global, 0, nullptr, ctx->stream));
  } else {
    CK(launch_fill(p.colc, p.n, 0.0, ctx->stream));
  }
  if (p.scaled || want_ss) {
    CK(launch_colsum(p.A, p.lda, p.f32, p.M, p.n, 1, p.colc, p.colp, p.colss, ctx->stream, nullptr));
    CKS(allreduce_sum(ctx, p.colss, (size_t)p.n));
  }
  if (p.scaled) CK(launch_colstat_scale(p.colss, p.n, (double)p.m_global, p.colr, p.cols, ctx->stream));
  return RSVD_OK;
}

// Core of rsvd: fills p.Y (= Q, M x Np), p.X (= V, n x Np, sign-fixed),
// p.W (= U~ diag(sgn), Np x Np), p.sigma.  Status bits in ctx->flags_dev.
rsvd_status rsvd_core(rsvd_ctx* ctx, Plan& p, const rsvd_params* prm, bool want_svd, bool want_ss = false) {
  const int l = p.l, Np = p.Np;
  ctx->prof_phase ^= 1;           // level-2 profiling samples A.X and A^T.X passes on alternate calls
  const bool dist = ctx->nranks > 1;
  const bool centred = prm->center != 0 || prm->scale != 0;
  CK(launch_zero_words(ctx->flags_dev, 16, ctx->stream));
  p.scaled = prm->scale != 0;
  if (centred || p.scaled || want_ss) CKS(column_stats(ctx, p, prm->center != 0, want_ss));
  if (p.use_ozaki) {
    // slices of f(A) once per call; every pass below reads them (pass_ozaki.cu)
    Prof pr(ctx, 5, (double)p.M * p.n * (p.f32 ? 4 : 8));
    CK(ozaki_slice_a(p.oz, p.A, p.f32, p.lda, centred ? p.colc : nullptr, p.scaled ? p.colr : nullptr,
                     ctx->flags_dev, ctx->stream));
  }
  {
    Prof pr(ctx, 4, 0);
    CK(launch_omega(p.n, l, Np, Np, prm->sdist, prm->seed, prm->stream, p.f32, false, p.X, ctx->stream));
  }
  CKS(pass_ax(ctx, p, p.X, p.Y, centred));                          // Y = A Omega
  for (int j = 0; j < prm->q; ++j) {
    if (prm->power == 1) {                                           // Alg. 1 (direct)
      CKS(pass_atx(ctx, p, p.Y, p.Z, centred));                      //   (2) Y = A^T Y
      CKS(pass_ax(ctx, p, p.Z, p.Y, centred));                       //   (3) Y = A Y
      continue;
    }
    if (prm->power == 2) {                                           // Alg. 3 (normalized, pivoted LU)
      CKS(ensure_ws2(ctx, lu_scratch_bytes(std::max(p.M, p.n), ctx->num_sms)));
      {
        Prof pr(ctx, 2, (double)p.M * Np * 8 * 2);
        CK(launch_lu_rows(p.Y, Np, p.M, l, ctx->ws2, ctx->flags_dev, kFlagLuZero, ctx->num_sms, ctx->stream));
      }                                                              //   (2) [L,~] = lu(Y)
      CKS(pass_atx(ctx, p, p.Y, p.Z, centred));                      //   A^T L
      {
        Prof pr(ctx, 2, (double)p.n * Np * 8 * 2);
        CK(launch_lu_rows(p.Z, Np, p.n, l, ctx->ws2, ctx->flags_dev, kFlagLuZero, ctx->num_sms, ctx->stream));
      }                                                              //   (3) [L,~] = lu(A^T L)
      CKS(pass_ax(ctx, p, p.Z, p.Y, centred));                       //   (4) Y = A L
      continue;
    }
    CKS(orth(ctx, p, p.Y, p.M, dist, nullptr, false));              // Alg. 2 (2) [Q,~] = qr(Y)
    CKS(pass_atx(ctx, p, p.Y, p.Z, centred));                        //   A^T Q
    CKS(orth(ctx, p, p.Z, p.n, false, nullptr, false));             //   (3) [Q,~] = qr(A^T Q)
    CKS(pass_ax(ctx, p, p.Z, p.Y, centred));                         //   (4) Y = A Q
  }
  CKS(orth(ctx, p, p.Y, p.M, dist, nullptr));                       // Alg. 4 step 9
  CKS(pass_atx(ctx, p, p.Y, p.Z, centred));                          // step 10: B^T = A^T Q
  if (!want_svd) return RSVD_OK;
  // economic SVD of B via B^T = Q_B R_B and Jacobi on R_B^T (Alg. 5 step 2)
  CKS(orth(ctx, p, p.Z, p.n, false, p.RB));
  {
    Prof pr(ctx, 3, 0);
    if (p.wide)
      CK(launch_jacobi_wide(p.RB, Np, l, p.sigma, p.W, p.J, Np, ctx->flags_dev, ctx->sweeps_dev, p.jlog,
                            ctx->num_sms, ctx->stream));
    else
      CK(launch_jacobi(p.RB, Np, l, p.sigma, p.W, p.J, Np, ctx->flags_dev, ctx->sweeps_dev, p.jlog, ctx->stream));
  }
  // (launch_jacobi leaves the padding of W and J exact zeros)
  // V = Q_B J  (n x Np) into X
  CKS(small_k(ctx, p, p.Z, p.n, p.J, p.X, Np, Np));
  if (!p.trans_input) {
    // reading R9: signs from V; U = Q (U~ diag(sgn)) is formed by the caller-facing step
    CK(launch_sign_from_v(p.X, Np, p.n, l, p.sgn, ctx->stream));
    CK(launch_scale_cols(p.X, Np, p.n, l, p.sgn, ctx->stream));
    CK(launch_scale_cols(p.W, Np, l, l, p.sgn, ctx->stream));
  } else {
    // worked on A^T: the V of A is U' = Q U~ (M x Np, into T); signs from it
    CKS(small_k(ctx, p, p.Y, p.M, p.W, p.T, Np, Np));
    CK(launch_sign_from_v(p.T, Np, p.M, l, p.sgn, ctx->stream));
    CK(launch_scale_cols(p.T, Np, p.M, l, p.sgn, ctx->stream));
    CK(launch_scale_cols(p.X, Np, p.n, l, p.sgn, ctx->stream));
  }
  CK(launch_check_finite(p.sigma, l, ctx->flags_dev, ctx->stream));
  return RSVD_OK;
}

// Ozaki slices of A (and X slice scratch) for the plan
rsvd_status plan_ozaki(rsvd_ctx* ctx, Plan& p, int64_t m_local, int64_t n_stored, bool alloc) {
  const int s = p.f32 ? OZ_S32 : OZ_S;
  const size_t sa = align256(ozaki_a_bytes(m_local, n_stored, s));
  const int xc = ozaki_x_cols(s, p.Np);
  const size_t sx = align256(ozaki_x_bytes(std::max(p.M, p.n), xc, s));
  const size_t nx = p.Np > xc ? 2 : 1;
  p.oz_bytes = sa + nx * sx;
  if (!alloc) return RSVD_OK;
  CKS(ensure_buf(ctx, &ctx->ws4, &ctx->ws4_bytes, p.oz_bytes, "Ozaki slice workspace"));
  p.oz = ozaki_layout_a(ctx->ws4, m_local, n_stored, s);
  p.ozx = ctx->ws4 + sa;
  p.ozx2 = nx > 1 ? ctx->ws4 + sa + sx : nullptr;
  return RSVD_OK;
}

// Build the plan for A (handles the single-GPU m < n case by working on A^T).
// alloc = false: sizes only (rsvd_workspace_bytes).
rsvd_status make_plan(rsvd_ctx* ctx, const rsvd_matrix* A, int k, int p_over, bool center_or_scale, Plan& p,
                      bool alloc = true) {
  const int64_t mg = ctx->nranks > 1 ? A->m_global : A->m_local;
  p.f32 = A->dtype == RSVD_F32;
  p.A = A->A; p.lda = A->lda;
  p.trans_input = (ctx->nranks <= 1) && (A->m_local < A->n);
  if (p.trans_input && center_or_scale)
    return fail(ctx, RSVD_EUNSUPPORTED, "centring/scaling needs m >= n");
  if (p.trans_input) { p.M = A->n; p.n = A->m_local; p.m_global = A->n; }
  else { p.M = A->m_local; p.n = A->n; p.m_global = mg; }
  const int64_t mn = std::min(mg, A->n);
  p.l = (int)std::min<int64_t>((int64_t)k + p_over, mn);
  p.Np = (int)round_up(p.l, 16);      // GEMM N granularity: two warps x n8 tiles
  p.wide = p.l > kMaxL;
  p.use_ozaki = !p.wide && (p.f32 ? ctx->fp32_ozaki : ctx->fp64_ozaki) && ozaki_supported(p.Np);
  p.use_tf32 = !p.wide && !p.use_ozaki && p.f32 && !center_or_scale && ctx->fp32_tcgen05 &&
               tf32_pass_supported(p.A, p.lda);
  if (p.l > kMaxWide) return fail(ctx, RSVD_EUNSUPPORTED, "l = k + p = %d exceeds this build's limit %d", p.l, kMaxWide);
  if (ctx->nranks > 1 && p.M < p.l)
    return fail(ctx, RSVD_EUNSUPPORTED, "each rank needs at least l = %d rows", p.l);
  const size_t bytes = plan_bytes(ctx, p);
  if (alloc) {
    CKS(ensure_ws(ctx, bytes));
    bind(ctx, p);
  }
  if (p.use_ozaki) CKS(plan_ozaki(ctx, p, A->m_local, A->n, alloc));
  return RSVD_OK;
}

// TSQR fallback scratch for the panels of a plan (rows M and n)
size_t plan_tsqr_bytes(const Plan& p, int nranks) {
  size_t a = 0, b = 0, c = 0;
  tsqr_levels(p.M, p.l, nullptr, &a);
  tsqr_levels(p.n, p.l, nullptr, &b);
  tsqr_levels((int64_t)nranks * p.l, p.l, nullptr, &c);
  return std::max(std::max(a, b), c) + 512;
}

// One call: the core, then the caller's output kernels (`emit`), then the
// end-of-call status kernel (flags OR-ed into the sticky word for rsvd_sync).
rsvd_status run_call(rsvd_ctx* ctx, Plan& p, const rsvd_params* prm, bool want_svd,
                     const std::function<rsvd_status()>& emit = nullptr, bool want_ss = false) {
  ctx->err.clear();
  if (prm->power == 2 && p.l > 128)   // the cooperative GEPP holds a row of the panel per lane group
    return fail(ctx, RSVD_EUNSUPPORTED, "Alg. 3 (pivoted LU power scheme) needs l = k + p <= 128");
  CKS(ensure_ws2(ctx, plan_tsqr_bytes(p, ctx->nranks)));   // before any launch: no reallocation mid-call
  CKS(rsvd_core(ctx, p, prm, want_svd, want_ss));
  if (emit) CKS(emit());
  CK(launch_status_finish(ctx->flags_dev, ctx->sticky_dev, kFlagCholBreak, ctx->stream));
  return RSVD_OK;
}

// Wait for the stream and turn the sticky status into a return code.
rsvd_status sync_status(rsvd_ctx* ctx) {
  CK(cudaMemcpyAsync(ctx->flags_host, ctx->sticky_dev, sizeof(int) * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemsetAsync(ctx->sticky_dev, 0, sizeof(int) * 4, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (ctx->prof) prof_collect(ctx);
  const int f = ctx->flags_host[0];
  ctx->last_sweeps = ctx->flags_host[1];
  ctx->last_robust = ctx->flags_host[2];
  if (f & kFlagNonFinite) return fail(ctx, RSVD_ENUMERIC, "non-finite intermediate (input contains Inf/NaN?)");
  if (f & kFlagJacobiCap) return fail(ctx, RSVD_ENUMERIC, "one-sided Jacobi hit the 30-sweep cap");
  if (f & kFlagRankDef) return fail(ctx, RSVD_ENUMERIC, "pivoted QR: numerical rank < k");
  if (f & kFlagWideBreak)
    return fail(ctx, RSVD_ENUMERIC, "CholeskyQR breakdown at l > %d (numerically rank-deficient sketch; no Householder "
                "fallback at this width)", kMaxL);
  if (f & kFlagNoFallback)
    return fail(ctx, RSVD_ENUMERIC, "CholeskyQR breakdown on a panel with fewer rows than l (no TSQR fallback)");
  return RSVD_OK;
}

}  // namespace

// =================================================================== C ABI
extern "C" {

const char* rsvd_version(void) { return "rsvd_b200 0.2 (sm_100a)"; }

rsvd_status rsvd_create(rsvd_ctx** out, int device, void* stream) {
  if (!out) return RSVD_EINVAL;
  *out = nullptr;
  rsvd_ctx* ctx = new rsvd_ctx();
  ctx->device = device;
  ctx->stream = (cudaStream_t)stream;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->flags_dev, 128 * sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(ctx->flags_dev, 0, 128 * sizeof(int));
  if (e == cudaSuccess) e = cudaMallocHost(&ctx->flags_host, 16 * sizeof(int));
  if (e == cudaSuccess) e = cudaMallocHost(&ctx->hbuf, 1024 * sizeof(double));
  if (e == cudaSuccess) { ctx->sweeps_dev = ctx->flags_dev + 8; ctx->sticky_dev = ctx->flags_dev + 16; }
  if (e == cudaSuccess) e = cudaMalloc(&ctx->gemm_flags, 4096 * sizeof(unsigned));
  if (e == cudaSuccess) e = cudaMemset(ctx->gemm_flags, 0, 4096 * sizeof(unsigned));
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  {
    const char* fp = getenv("RSVD_FP32_PATH");
    if (fp && strcmp(fp, "dmma") == 0) ctx->fp32_tcgen05 = ctx->fp32_ozaki = false;
    if (fp && strcmp(fp, "tf32") == 0) ctx->fp32_ozaki = false;
    const char* f64 = getenv("RSVD_FP64_PATH");
    if (f64 && strcmp(f64, "dmma") == 0) ctx->fp64_ozaki = false;
  }
  if (e != cudaSuccess) {
    delete ctx;
    return RSVD_ECUDA;
  }
  *out = ctx;
  return RSVD_OK;
}

rsvd_status rsvd_destroy(rsvd_ctx* ctx) {
  if (!ctx) return RSVD_EINVAL;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  delete ctx->comm;
  for (auto& r : ctx->pending) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (auto e : ctx->pool) cudaEventDestroy(e);
  cudaFree(ctx->ws);
  cudaFree(ctx->ws2);
  cudaFree(ctx->flags_dev);
  cudaFreeHost(ctx->flags_host);
  cudaFreeHost(ctx->hbuf);
  cudaFree(ctx->ws3);
  cudaFree(ctx->ws5);
  cudaFree(ctx->gemm_flags);
  cudaFree(ctx->ws4);
  delete ctx;
  return RSVD_OK;
}

const char* rsvd_last_error(const rsvd_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

rsvd_status rsvd_sync(rsvd_ctx* ctx) {
  if (!ctx) return RSVD_EINVAL;
  CK(cudaSetDevice(ctx->device));
  return sync_status(ctx);
}

rsvd_status rsvd_nccl_unique_id(void* out128) {
  if (!out128) return RSVD_EINVAL;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return RSVD_ENCCL;
  memcpy(out128, &id, sizeof id);
  return RSVD_OK;
}

rsvd_status rsvd_comm_init(rsvd_ctx* ctx, const void* id128, int nranks, int rank) {
  if (!ctx || nranks < 1 || rank < 0 || rank >= nranks) return fail(ctx, RSVD_EINVAL, "bad comm args");
  if (ctx->comm) return fail(ctx, RSVD_EINVAL, "context already has a communicator");
  // One rank needs no communicator.  RSVD_NCCL_SINGLE=1 (tests) still builds a
  // one-rank NCCL communicator, so that every allreduce of the call goes through
  // ncclAllReduce on the context's stream (an identity) on a single GPU.
  const char* single = getenv("RSVD_NCCL_SINGLE");
  if (nranks == 1 && !(single && single[0] == '1')) { ctx->nranks = 1; ctx->rank = 0; return RSVD_OK; }
  ncclUniqueId id;
  if (id128) memcpy(&id, id128, sizeof id);
  else if (nranks == 1) {
    if (ncclGetUniqueId(&id) != ncclSuccess) return fail(ctx, RSVD_ENCCL, "ncclGetUniqueId failed");
  } else return fail(ctx, RSVD_EINVAL, "null unique id");
  cudaSetDevice(ctx->device);
  NcclComm* c = new NcclComm();
  ncclResult_t r = ncclCommInitRank(&c->c, nranks, id, rank);
  if (r != ncclSuccess) { delete c; return fail(ctx, RSVD_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r)); }
  c->n = nranks; c->r = rank;
  ctx->comm = c;
  ctx->nranks = nranks;
  ctx->rank = rank;
  return RSVD_OK;
}

rsvd_status rsvd_group_create(rsvd_group** out, int nranks) {
  if (!out || nranks < 2 || nranks > kMaxGroup) return RSVD_EINVAL;
  rsvd_group* g = new rsvd_group();
  g->n = nranks;
  g->slots.resize(nranks);
  *out = g;
  return RSVD_OK;
}

rsvd_status rsvd_group_destroy(rsvd_group* g) {
  if (!g) return RSVD_EINVAL;
  for (auto& s : g->slots) {
    if (!s.joined) continue;
    cudaSetDevice(s.device);
    if (s.stage) cudaFree(s.stage);
    if (s.ready) cudaEventDestroy(s.ready);
    if (s.done) cudaEventDestroy(s.done);
  }
  delete g;
  return RSVD_OK;
}

rsvd_status rsvd_comm_init_group(rsvd_ctx* ctx, rsvd_group* g, int rank) {
  if (!ctx) return RSVD_EINVAL;
  if (!g || rank < 0 || rank >= g->n) return fail(ctx, RSVD_EINVAL, "bad group or rank");
  if (ctx->comm) return fail(ctx, RSVD_EINVAL, "context already has a communicator");
  CK(cudaSetDevice(ctx->device));
  rsvd_group::Slot& s = g->slots[rank];
  if (s.joined) return fail(ctx, RSVD_EINVAL, "rank %d of the group is already taken", rank);
  CK(cudaEventCreateWithFlags(&s.ready, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
  s.device = ctx->device;
  s.joined = true;
  GroupComm* c = new GroupComm();
  c->g = g; c->r = rank;
  ctx->comm = c;
  ctx->nranks = g->n;
  ctx->rank = rank;
  return RSVD_OK;
}

void rsvd_params_default(rsvd_params* prm, int32_t k) {
  if (!prm) return;
  memset(prm, 0, sizeof *prm);
  prm->k = k; prm->nu = k; prm->nv = k; prm->p = 10; prm->q = 2;
  prm->sdist = RSVD_NORMAL;
}

void rsvd_rpca_params_default(rsvd_params* prm, int32_t k) {
  rsvd_params_default(prm, k);
  if (!prm) return;
  prm->center = 1;
  prm->scale = 1;                 // rpca(..., center = TRUE, scale = TRUE, ...)
}

void rsvd_rrpca_params_default(rsvd_rrpca_params* prm) {
  if (!prm) return;
  memset(prm, 0, sizeof *prm);
  prm->lambda = 0.0; prm->tol = 1e-5; prm->maxiter = 50; prm->k = 20; prm->p = 10; prm->q = 2;
  prm->sdist = RSVD_NORMAL;
  prm->rand = 1;
}

rsvd_status rsvd_workspace_bytes(rsvd_ctx* ctx, const rsvd_matrix* A, const rsvd_params* prm, size_t* bytes) {
  int64_t mg, n;
  CKS(validate(ctx, A, prm, &mg, &n));
  if (!bytes) return fail(ctx, RSVD_EINVAL, "bytes is null");
  Plan p{};
  CKS(make_plan(ctx, A, prm->k, prm->p, prm->center || prm->scale, p, false));
  size_t tot = p.total + p.oz_bytes + plan_tsqr_bytes(p, ctx->nranks);
  if (prm->power == 2) tot += lu_scratch_bytes(std::max(p.M, p.n), ctx->num_sms);
  *bytes = tot;
  return RSVD_OK;
}

rsvd_status rsvd_run(rsvd_ctx* ctx, const rsvd_matrix* A, const rsvd_params* prm_in, void* u, int64_t ldu,
                     void* d, void* v, int64_t ldv) {
  int64_t mg, n;
  CKS(validate(ctx, A, prm_in, &mg, &n));
  rsvd_params prm = *prm_in;
  ctx->err.clear();
  std::string warn;
  if (prm.nu > prm.k || prm.nv > prm.k) {
    prm.nu = std::min(prm.nu, prm.k);
    prm.nv = std::min(prm.nv, prm.k);
    warn = "warning: nu/nv > k clamped to k";
  }
  if (!d) return fail(ctx, RSVD_EINVAL, "d is null");
  if (prm.nu > 0 && (!u || ldu < prm.nu)) return fail(ctx, RSVD_EINVAL, "u null or ldu < nu");
  if (prm.nv > 0 && (!v || ldv < prm.nv)) return fail(ctx, RSVD_EINVAL, "v null or ldv < nv");
  CK(cudaSetDevice(ctx->device));
  Plan p{};
  CKS(make_plan(ctx, A, prm.k, prm.p, prm.center || prm.scale, p));
  const bool f32 = p.f32;
  const int Np = p.Np;
  const int nu = prm.nu, nv = prm.nv;
  // outputs: U = Q (U~ diag sgn), V (sign-fixed), d = sigma(1:k)
  auto emit = [&]() -> rsvd_status {
    double* Uo = p.T;      // M x Np scratch
    if (!p.trans_input) {
      if (nu > 0) {
        if (!f32) { CKS(small_k(ctx, p, p.Y, p.M, p.W, (double*)u, ldu, nu)); }
        else {
          CKS(small_k(ctx, p, p.Y, p.M, p.W, Uo, Np, nu));
          CK(launch_copy_out(Uo, Np, p.M, nu, u, ldu, true, nullptr, ctx->stream));
        }
      }
      if (nv > 0) CK(launch_copy_out(p.X, Np, p.n, nv, v, ldv, f32, nullptr, ctx->stream));
    } else {
      // worked on A^T = U' S V'^T  =>  A = V' S U'^T: u <- V' (n_eff rows), v <- U'
      if (nu > 0) CK(launch_copy_out(p.X, Np, p.n, nu, u, ldu, f32, nullptr, ctx->stream));
      if (nv > 0) CK(launch_copy_out(p.T, Np, p.M, nv, v, ldv, f32, nullptr, ctx->stream));
    }
    CK(launch_copy_out(p.sigma, 1, prm.k, 1, d, 1, f32, nullptr, ctx->stream));
    return RSVD_OK;
  };
  CKS(run_call(ctx, p, &prm, true, emit));
  if (!warn.empty()) ctx->err = warn;
  return RSVD_OK;
}

rsvd_status rsvd_run_host(rsvd_ctx* ctx, const rsvd_matrix* A, const rsvd_params* prm, void* u, int64_t ldu,
                          void* d, void* v, int64_t ldv) {
  int64_t mg, n;
  CKS(validate(ctx, A, prm, &mg, &n));
  if (!d) return fail(ctx, RSVD_EINVAL, "d is null");
  const int k = prm->k, nu = std::min(prm->nu, k), nv = std::min(prm->nv, k);
  if (nu > 0 && (!u || ldu < nu)) return fail(ctx, RSVD_EINVAL, "u null or ldu < nu");
  if (nv > 0 && (!v || ldv < nv)) return fail(ctx, RSVD_EINVAL, "v null or ldv < nv");
  CK(cudaSetDevice(ctx->device));
  const size_t es = A->dtype == RSVD_F32 ? 4 : 8;
  const int64_t m = A->m_local;
  const size_t bA = align256((size_t)m * n * es), bU = align256((size_t)m * std::max(nu, 1) * es),
               bD = align256((size_t)k * es), bV = align256((size_t)n * std::max(nv, 1) * es);
  CKS(ensure_buf(ctx, &ctx->ws5, &ctx->ws5_bytes, bA + bU + bD + bV, "host-call staging"));
  char* dA = ctx->ws5;
  char* dU = dA + bA;
  char* dD = dU + bU;
  char* dV = dD + bD;
  // A: host (lda) -> device (ld n)
  CK(cudaMemcpy2DAsync(dA, n * es, A->A, A->lda * es, n * es, m, cudaMemcpyHostToDevice, ctx->stream));
  rsvd_matrix Ad = *A;
  Ad.A = dA; Ad.lda = n;                  // this rank's row block keeps its place in the sharded matrix
  if (ctx->nranks <= 1) { Ad.m_global = m; Ad.row_offset = 0; }
  rsvd_params pr = *prm;
  pr.nu = nu; pr.nv = nv;
  CKS(rsvd_run(ctx, &Ad, &pr, nu ? dU : nullptr, std::max(nu, 1), dD, nv ? dV : nullptr, std::max(nv, 1)));
  if (nu > 0) CK(cudaMemcpy2DAsync(u, ldu * es, dU, nu * es, nu * es, m, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(d, dD, k * es, cudaMemcpyDeviceToHost, ctx->stream));
  if (nv > 0) CK(cudaMemcpy2DAsync(v, ldv * es, dV, nv * es, nv * es, n, cudaMemcpyDeviceToHost, ctx->stream));
  return sync_status(ctx);
}

rsvd_status rsvd_rqb(rsvd_ctx* ctx, const rsvd_matrix* A, const rsvd_params* prm, void* Q, int64_t ldq, void* Bt,
                     int64_t ldb) {
  int64_t mg, n;
  CKS(validate(ctx, A, prm, &mg, &n));
  if (prm->center) return fail(ctx, RSVD_EUNSUPPORTED, "rqb with centring: use rsvd_rpca");
  CK(cudaSetDevice(ctx->device));
  Plan p{};
  CKS(make_plan(ctx, A, prm->k, prm->p, prm->center || prm->scale, p));
  if (p.trans_input) return fail(ctx, RSVD_EUNSUPPORTED, "rqb needs m >= n");
  if (!Q || !Bt || ldq < p.l || ldb < p.l) return fail(ctx, RSVD_EINVAL, "Q/Bt null or ld < l");
  auto emit = [&]() -> rsvd_status {
    CK(launch_copy_out(p.Y, p.Np, p.M, p.l, Q, ldq, p.f32, nullptr, ctx->stream));
    CK(launch_copy_out(p.Z, p.Np, p.n, p.l, Bt, ldb, p.f32, nullptr, ctx->stream));
    return RSVD_OK;
  };
  return run_call(ctx, p, prm, false, emit);
}

// Alg. rid: [~, B] = rqb(A, k, p, q); [~, Z, J] = id(B, k) (Alg. id,
// P:2059-2095) by the pivoted QR of B (qrcp.cu, on B^T = A^T Q as computed);
// C = A(:, J).  Reading R31.
rsvd_status rsvd_rid(rsvd_ctx* ctx, const rsvd_matrix* A, const rsvd_params* prm, void* C, int64_t ldc, void* Z,
                     int64_t ldz, int64_t* J) {
  int64_t mg, n;
  CKS(validate(ctx, A, prm, &mg, &n));
  if (A->dtype != RSVD_F64) return fail(ctx, RSVD_EUNSUPPORTED, "rid is FP64 only");
  if (prm->center || prm->scale) return fail(ctx, RSVD_EUNSUPPORTED, "rid has no centring / scaling");
  const int k = prm->k;
  if (!C || !Z || !J || ldc < k || ldz < n) return fail(ctx, RSVD_EINVAL, "C/Z/J null or ldc < k or ldz < n");
  CK(cudaSetDevice(ctx->device));
  Plan p{};
  CKS(make_plan(ctx, A, k, prm->p, false, p));
  if (p.trans_input) return fail(ctx, RSVD_EUNSUPPORTED, "rid needs m >= n");
  if (p.l > 128) return fail(ctx, RSVD_EUNSUPPORTED, "rid needs l <= 128");
  CKS(ensure_ws2(ctx, std::max(plan_tsqr_bytes(p, ctx->nranks), qrcp_scratch_bytes(p.n, k, ctx->num_sms))));
  auto emit = [&]() -> rsvd_status {
    CK(launch_qrcp(p.Z, p.Np, p.l, p.n, k, J, (double*)Z, ldz, ctx->ws2, ctx->flags_dev, kFlagRankDef,
                   ctx->num_sms, ctx->stream));
    CK(launch_gather_cols((const double*)A->A, A->lda, A->m_local, J, k, (double*)C, ldc, ctx->stream));
    return RSVD_OK;
  };
  return run_call(ctx, p, prm, false, emit);
}

// Alg. rcur: [C, Z, J] = rid(A, k, p, q); [~, S, P] = qr(C^T)
// pivoted (k pivots over the m columns of C^T = rows of C); I = P(1:k);
// R = A(I, :); U = Z pinv(R) with pinv(R) = Q_R S_R^-T from the Householder
// TSQR of R^T (reading R31).
rsvd_status rsvd_rcur(rsvd_ctx* ctx, const rsvd_matrix* A, const rsvd_params* prm, void* C, int64_t ldc, void* U,
                      int64_t ldu, void* R, int64_t ldr, int64_t* J, int64_t* I) {
  int64_t mg, n;
  CKS(validate(ctx, A, prm, &mg, &n));
  if (A->dtype != RSVD_F64) return fail(ctx, RSVD_EUNSUPPORTED, "rcur is FP64 only");
  if (ctx->nranks > 1) return fail(ctx, RSVD_EUNSUPPORTED, "rcur is single-GPU (pivoted QR over distributed rows)");
  if (prm->center || prm->scale) return fail(ctx, RSVD_EUNSUPPORTED, "rcur has no centring / scaling");
  const int k = prm->k;
  if (!C || !U || !R || !J || !I || ldc < k || ldu < k || ldr < n)
    return fail(ctx, RSVD_EINVAL, "C/U/R/J/I null or ldc < k, ldu < k, ldr < n");
  CK(cudaSetDevice(ctx->device));
  Plan p{};
  CKS(make_plan(ctx, A, k, prm->p, false, p));
  if (p.trans_input) return fail(ctx, RSVD_EUNSUPPORTED, "rcur needs m >= n");
  if (p.l > 128) return fail(ctx, RSVD_EUNSUPPORTED, "rcur needs l <= 128");
  const int64_t m = A->m_local;
  const double* Ad = (const double*)A->A;
  const int Np2 = (int)round_up(k, 16);
  double* Zs = p.X;                        // k x n, ld n (p.X is n x Np >= k x n)
  double* Ct = p.T;                        // m x k copy of C for the pivoted QR of C^T
  double* Rt = p.Y;                        // n x Np2 panel R^T -> Q_R
  double* Sr = p.RB;                       // S_R (k x k, ld Np2)
  Plan q = p;
  q.l = k; q.Np = Np2;
  CKS(ensure_ws2(ctx, std::max({plan_tsqr_bytes(p, 1), plan_tsqr_bytes(q, 1), qrcp_scratch_bytes(p.n, k, ctx->num_sms),
                                qrcp_scratch_bytes(m, k, ctx->num_sms)})));
  auto emit = [&]() -> rsvd_status {
    CK(launch_qrcp(p.Z, p.Np, p.l, p.n, k, J, Zs, p.n, ctx->ws2, ctx->flags_dev, kFlagRankDef, ctx->num_sms,
                   ctx->stream));                                        // rid: Z, J
    CK(launch_gather_cols(Ad, A->lda, m, J, k, (double*)C, ldc, ctx->stream));   // C = A(:, J)
    CK(launch_gather_cols(Ad, A->lda, m, J, k, Ct, k, ctx->stream));
    CK(launch_qrcp(Ct, k, k, m, k, I, nullptr, 0, ctx->ws2, ctx->flags_dev, kFlagRankDef, ctx->num_sms,
                   ctx->stream));                                        // I = P(1:k) of qr(C^T)
    CK(launch_fill(Rt, p.n * Np2, 0.0, ctx->stream));
    CK(launch_gather_rows(Ad, A->lda, p.n, I, k, (double*)R, ldr, Rt, Np2, ctx->stream));   // R = A(I, :), R^T
    // R^T = Q_R S_R by Householder TSQR (always: R^T may be rank deficient)
    CKS(tsqr_local(ctx, q, Rt, Np2, p.n, p.Rsm, Pred{}));
    CK(launch_copy_out(p.Rsm, k, k, k, Sr, Np2, false, nullptr, ctx->stream));
    CK(launch_zq(Zs, p.n, Rt, Np2, p.n, k, p.part, p.G, k, ctx->num_sms, ctx->stream));   // W = Z Q_R
    CK(launch_rtsolve(p.G, k, Sr, Np2, k, (double*)U, ldu, ctx->stream));              // U = W S_R^-T
    return RSVD_OK;
  };
  return run_call(ctx, p, prm, false, emit);
}

rsvd_status rsvd_rpca(rsvd_ctx* ctx, const rsvd_matrix* A, const rsvd_params* prm_in, const rsvd_pca_out* o) {
  int64_t mg, n;
  CKS(validate(ctx, A, prm_in, &mg, &n));
  if (!o) return fail(ctx, RSVD_EINVAL, "null output descriptor");
  rsvd_params prm = *prm_in;
  const int k = prm.k;
  if (o->rotation && o->ldr < k) return fail(ctx, RSVD_EINVAL, "ldr < k");
  if (o->x && o->ldx < k) return fail(ctx, RSVD_EINVAL, "ldx < k");
  if (o->loadings && o->ldl < k) return fail(ctx, RSVD_EINVAL, "ldl < k");
  if (o->x_white && o->ldw < k) return fail(ctx, RSVD_EINVAL, "ldw < k");
  CK(cudaSetDevice(ctx->device));
  Plan p{};
  CKS(make_plan(ctx, A, k, prm.p, prm.center || prm.scale, p));
  if (p.trans_input) return fail(ctx, RSVD_EUNSUPPORTED, "rpca needs m >= n");
  const bool want_total = o->var_ratio || o->var_cum || o->total_var;
  auto emit = [&]() -> rsvd_status {
    const int Np = p.Np;
    const bool f32 = p.f32;
    const double mgd = (double)p.m_global;
    if (want_total) CK(launch_total_var(p.colss, p.scaled ? p.colr : nullptr, p.n, mgd, p.tv, ctx->stream));
    CK(launch_pca_stats(p.sigma, k, mgd, want_total ? p.tv : nullptr, o->eigvals, o->sdev, o->var_ratio,
                        o->var_cum, f32, ctx->stream));
    if (o->total_var) CK(launch_copy_out(p.tv, 1, 1, 1, o->total_var, 1, f32, nullptr, ctx->stream));
    if (o->rotation) CK(launch_copy_out(p.X, Np, p.n, k, o->rotation, o->ldr, f32, nullptr, ctx->stream));
    if (o->loadings) {                     // L = W Lambda^{1/2}: rotation columns times sdev
      CK(launch_vec_map(p.sigma, false, k, 2, mgd, p.sgn, ctx->stream));
      CK(launch_copy_out(p.X, Np, p.n, k, o->loadings, o->ldl, f32, p.sgn, ctx->stream));
    }
    if (o->x || o->x_white) {
      CKS(small_k(ctx, p, p.Y, p.M, p.W, p.T, Np, k));                   // U (this rank's rows)
      if (o->x) CK(launch_copy_out(p.T, Np, p.M, k, o->x, o->ldx, f32, p.sigma, ctx->stream));   // Z = U diag(d)
      if (o->x_white) {                    // z_i / sqrt(lambda_i) = u_i sqrt(m - 1)
        CK(launch_vec_map(nullptr, false, k, 3, sqrt(mgd - 1.0), p.sgn, ctx->stream));
        CK(launch_copy_out(p.T, Np, p.M, k, o->x_white, o->ldw, f32, p.sgn, ctx->stream));
      }
    }
    if (o->center && prm.center) CK(launch_copy_out(p.colc, 1, p.n, 1, o->center, 1, f32, nullptr, ctx->stream));
    if (o->scale && prm.scale) CK(launch_copy_out(p.cols, 1, p.n, 1, o->scale, 1, f32, nullptr, ctx->stream));
    return RSVD_OK;
  };
  return run_call(ctx, p, &prm, true, emit, want_total && !p.scaled);
}

rsvd_status rsvd_rpca_host(rsvd_ctx* ctx, const rsvd_matrix* A, const rsvd_params* prm, const rsvd_pca_out* o) {
  int64_t mg, n;
  CKS(validate(ctx, A, prm, &mg, &n));
  if (!o) return fail(ctx, RSVD_EINVAL, "null output descriptor");
  CK(cudaSetDevice(ctx->device));
  const size_t es = A->dtype == RSVD_F32 ? 4 : 8;
  const int64_t m = A->m_local, k = prm->k;
  // device staging: A, then every requested output (dense, ld = its column count)
  struct Out { void* host; int64_t ldh, rows, cols; size_t off; } outs[12];
  int no = 0;
  size_t off = align256((size_t)m * n * es);
  auto add = [&](void* h, int64_t ldh, int64_t rows, int64_t cols) {
    if (!h) return;
    outs[no++] = {h, ldh, rows, cols, off};
    off += align256((size_t)rows * cols * es);
  };
  add(o->rotation, o->ldr, n, k); add(o->eigvals, 1, k, 1); add(o->sdev, 1, k, 1); add(o->x, o->ldx, m, k);
  add(o->center, 1, n, 1); add(o->scale, 1, n, 1); add(o->loadings, o->ldl, n, k); add(o->x_white, o->ldw, m, k);
  add(o->var_ratio, 1, k, 1); add(o->var_cum, 1, k, 1); add(o->total_var, 1, 1, 1);
  CKS(ensure_buf(ctx, &ctx->ws5, &ctx->ws5_bytes, off, "host-call staging"));
  char* dA = ctx->ws5;
  CK(cudaMemcpy2DAsync(dA, n * es, A->A, A->lda * es, n * es, m, cudaMemcpyHostToDevice, ctx->stream));
  rsvd_matrix Ad = *A;
  Ad.A = dA; Ad.lda = n;                  // this rank's row block keeps its place in the sharded matrix
  if (ctx->nranks <= 1) { Ad.m_global = m; Ad.row_offset = 0; }
  rsvd_pca_out od = *o;
  auto dptr = [&](void* h) -> void* {
    for (int i = 0; i < no; ++i) if (outs[i].host == h) return ctx->ws5 + outs[i].off;
    return nullptr;
  };
  od.rotation = dptr(o->rotation); od.ldr = k; od.eigvals = dptr(o->eigvals); od.sdev = dptr(o->sdev);
  od.x = dptr(o->x); od.ldx = k; od.center = dptr(o->center); od.scale = dptr(o->scale);
  od.loadings = dptr(o->loadings); od.ldl = k; od.x_white = dptr(o->x_white); od.ldw = k;
  od.var_ratio = dptr(o->var_ratio); od.var_cum = dptr(o->var_cum); od.total_var = dptr(o->total_var);
  CKS(rsvd_rpca(ctx, &Ad, prm, &od));
  for (int i = 0; i < no; ++i) {
    const Out& q = outs[i];
    CK(cudaMemcpy2DAsync(q.host, q.ldh * es, ctx->ws5 + q.off, q.cols * es, q.cols * es, q.rows,
                         cudaMemcpyDeviceToHost, ctx->stream));
  }
  return sync_status(ctx);
}

rsvd_status rsvd_rpca_predict(rsvd_ctx* ctx, const rsvd_matrix* Anew, int32_t k, const void* rotation, int64_t ldr,
                              const void* center, const void* scale, void* out, int64_t ldo) {
  if (!ctx) return RSVD_EINVAL;
  if (!Anew || !Anew->A || !rotation || !out) return fail(ctx, RSVD_EINVAL, "null argument");
  if (Anew->dtype != RSVD_F64 && Anew->dtype != RSVD_F32) return fail(ctx, RSVD_EINVAL, "dtype must be F64 or F32");
  if (Anew->m_local < 1 || Anew->n < 1 || Anew->lda < Anew->n) return fail(ctx, RSVD_EINVAL, "bad shape or lda < n");
  if (k < 1 || k > 128 || ldr < k || ldo < k) return fail(ctx, RSVD_EINVAL, "need 1 <= k <= 128, ldr >= k, ldo >= k");
  CK(cudaSetDevice(ctx->device));
  ctx->err.clear();
  rsvd_matrix Am = *Anew;
  Am.m_global = Am.m_local; Am.row_offset = 0;
  // a plan with l = k over the new rows, never transposed (the projection is row-wise)
  Plan p{};
  const bool cs = center || scale;
  p.f32 = Am.dtype == RSVD_F32;
  p.A = Am.A; p.lda = Am.lda;
  p.trans_input = false;
  p.M = Am.m_local; p.n = Am.n; p.m_global = Am.m_local;
  p.l = k; p.Np = (int)round_up(k, 16);
  p.use_ozaki = (p.f32 ? ctx->fp32_ozaki : ctx->fp64_ozaki) && ozaki_supported(p.Np);
  p.use_tf32 = !p.use_ozaki && p.f32 && !cs && ctx->fp32_tcgen05 && tf32_pass_supported(p.A, p.lda);
  CKS(ensure_ws(ctx, plan_bytes(ctx, p)));
  bind(ctx, p);
  if (p.use_ozaki) CKS(plan_ozaki(ctx, p, Am.m_local, Am.n, true));
  const bool f32 = p.f32;
  CK(launch_zero_words(ctx->flags_dev, 16, ctx->stream));
  CK(launch_copy_in(rotation, f32, ldr, p.n, k, p.Np, p.X, p.Np, ctx->stream));       // W, zero padded
  if (center) CK(launch_vec_map(center, f32, p.n, 0, 0.0, p.colc, ctx->stream));
  else CK(launch_fill(p.colc, p.n, 0.0, ctx->stream));
  p.scaled = scale != nullptr;
  if (scale) CK(launch_vec_map(scale, f32, p.n, 1, 0.0, p.colr, ctx->stream));          // 1 / s
  if (p.use_ozaki)
    CK(ozaki_slice_a(p.oz, p.A, p.f32, p.lda, center ? p.colc : nullptr, scale ? p.colr : nullptr,
                     ctx->flags_dev, ctx->stream));
  CKS(pass_ax(ctx, p, p.X, p.Y, cs));                                                   // f(Anew) W
  CK(launch_copy_out(p.Y, p.Np, p.M, k, out, ldo, f32, nullptr, ctx->stream));
  CK(launch_status_finish(ctx->flags_dev, ctx->sticky_dev, kFlagCholBreak, ctx->stream));
  return RSVD_OK;
}

rsvd_status rsvd_omega(rsvd_ctx* ctx, int64_t n, int64_t l, int32_t sdist, uint64_t seed, uint64_t stream,
                       int32_t dtype, void* out, int64_t ldo) {
  if (!ctx) return RSVD_EINVAL;
  if (n < 1 || l < 1 || ldo < l || !out || sdist < 0 || sdist > 2) return fail(ctx, RSVD_EINVAL, "bad omega args");
  CK(cudaSetDevice(ctx->device));
  const bool f32 = dtype == RSVD_F32;
  CK(launch_omega(n, l, ldo, l, sdist, seed, stream, f32, f32, out, ctx->stream));
  return RSVD_OK;
}

rsvd_status rsvd_set_profiling(rsvd_ctx* ctx, int enable) {
  if (!ctx) return RSVD_EINVAL;
  ctx->prof = enable == 2 ? 2 : (enable != 0 ? 1 : 0);
  return RSVD_OK;
}

rsvd_status rsvd_profile(rsvd_ctx* ctx, int kind, double* total_ms, int64_t* count, double* bytes) {
  if (!ctx || kind < 0 || kind > 6) return RSVD_EINVAL;
  if (!ctx->pending.empty()) {
    cudaStreamSynchronize(ctx->stream);
    prof_collect(ctx);
  }
  if (total_ms) *total_ms = ctx->prof_ms[kind];
  if (count) *count = ctx->prof_count[kind];
  if (bytes) *bytes = ctx->prof_bytes[kind];
  return RSVD_OK;
}

rsvd_status rsvd_profile_reset(rsvd_ctx* ctx) {
  if (!ctx) return RSVD_EINVAL;
  if (!ctx->pending.empty()) { cudaStreamSynchronize(ctx->stream); prof_collect(ctx); }
  for (int i = 0; i < 7; ++i) { ctx->prof_ms[i] = 0; ctx->prof_bytes[i] = 0; ctx->prof_count[i] = 0; }
  rsvd::g_kernel_launches = 0;
  return RSVD_OK;
}

int64_t rsvd_launch_count(const rsvd_ctx* ctx) { return ctx ? rsvd::g_kernel_launches.load() : 0; }

rsvd_status rsvd_stats(const rsvd_ctx* ctx, int64_t* out, int n) {
  if (!ctx || !out || n < 0) return RSVD_EINVAL;
  const int64_t v[4] = {ctx->last_sweeps, ctx->last_robust, rsvd::g_kernel_launches.load(), ctx->ozaki_calls};
  for (int i = 0; i < n && i < 4; ++i) out[i] = v[i];
  return RSVD_OK;
}

}  // extern "C"

// =================================================================== rrpca (Alg. 7)
namespace {

// rsvd into device buffers (enqueued; step (6) of Alg. 7)
rsvd_status rsvd_device(rsvd_ctx* ctx, const rsvd_matrix* A, const rsvd_params* prm, double* U, int64_t ldu,
                        double* d, double* V, int64_t ldv) {
  int64_t mg, n;
  CKS(validate(ctx, A, prm, &mg, &n));
  Plan p{};
  CKS(make_plan(ctx, A, prm->k, prm->p, false, p));
  if (p.trans_input) return fail(ctx, RSVD_EUNSUPPORTED, "rrpca needs m >= n");
  auto emit = [&]() -> rsvd_status {
    if (U) CKS(small_k(ctx, p, p.Y, p.M, p.W, U, ldu, prm->k));
    if (V) CK(launch_copy_out(p.X, p.Np, p.n, prm->k, V, ldv, false, nullptr, ctx->stream));
    CK(launch_copy_out(p.sigma, 1, prm->k, 1, d, 1, false, nullptr, ctx->stream));
    return RSVD_OK;
  };
  return run_call(ctx, p, prm, true, emit);
}

}  // namespace

extern "C" rsvd_status rsvd_rrpca_host(rsvd_ctx* ctx, const rsvd_matrix* A, const rsvd_rrpca_params* prm, void* L,
                                       void* S, int64_t ld, int32_t* iters_out, double* res_out, double* trace) {
  if (!ctx) return RSVD_EINVAL;
  if (!A || !A->A || !prm || !L || !S) return fail(ctx, RSVD_EINVAL, "null argument");
  if (A->dtype != RSVD_F64) return fail(ctx, RSVD_EUNSUPPORTED, "rrpca is FP64 only");
  if (A->m_local < 1 || A->n < 1 || A->lda != A->n || ld != A->n)
    return fail(ctx, RSVD_EUNSUPPORTED, "rrpca needs contiguous A, L, S (lda == ld == n)");
  CK(cudaSetDevice(ctx->device));
  const size_t bytes = (size_t)A->m_local * A->n * 8, b = align256(bytes);
  CKS(ensure_buf(ctx, &ctx->ws5, &ctx->ws5_bytes, 3 * b, "host-call staging"));
  char* dA = ctx->ws5;
  char* dL = dA + b;
  char* dS = dL + b;
  CK(cudaMemcpyAsync(dA, A->A, bytes, cudaMemcpyHostToDevice, ctx->stream));
  rsvd_matrix Ad = *A;
  Ad.A = dA;
  if (ctx->nranks <= 1) { Ad.m_global = A->m_local; Ad.row_offset = 0; }
  CKS(rsvd_rrpca(ctx, &Ad, prm, dL, dS, ld, iters_out, res_out, trace));
  CK(cudaMemcpyAsync(L, dL, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(S, dS, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  return sync_status(ctx);
}

extern "C" rsvd_status rsvd_rrpca(rsvd_ctx* ctx, const rsvd_matrix* A, const rsvd_rrpca_params* prm, void* Lout,
                                  void* Sout, int64_t ld, int32_t* iters_out, double* res_out, double* trace) {
  if (!ctx) return RSVD_EINVAL;
  if (!A || !prm || !Lout || !Sout) return fail(ctx, RSVD_EINVAL, "null argument");
  if (A->dtype != RSVD_F64) return fail(ctx, RSVD_EUNSUPPORTED, "rrpca is FP64 only");
  if (ld < A->n) return fail(ctx, RSVD_EINVAL, "ld < n");
  if (A->lda != A->n || ld != A->n)
    return fail(ctx, RSVD_EUNSUPPORTED, "rrpca needs contiguous A, L, S (lda == ld == n)");
  if (prm->maxiter < 1 || prm->k < 0 || !(prm->tol > 0))
    return fail(ctx, RSVD_EINVAL, "bad rrpca params (k >= 0, maxiter >= 1, tol > 0)");
  const bool adaptive = prm->k == 0;   // Alg. 7 steps (1), (7): k = 2, predict_rank (reading R30)
  rsvd_params rp;
  rsvd_params_default(&rp, adaptive ? 1 : prm->k);
  rp.p = prm->p; rp.q = prm->q; rp.sdist = prm->sdist; rp.seed = prm->seed;
  int64_t mg, n;
  CKS(validate(ctx, A, &rp, &mg, &n));
  CK(cudaSetDevice(ctx->device));
  const int64_t m = A->m_local;
  const int64_t minmn = std::min(mg, n);
  // library envelope: l = k + p <= kMaxWide (l > kMaxL runs as a wide plan,
  // wide.cu).  The deterministic SVD of Remark 2 and rand = FALSE is
  // rsvd with l = min(m, n), q = 0 (reading R30), available while
  // min(m, n) <= kMaxWide; above that the randomized SVD is kept (warning in
  // rsvd_last_error) and the adaptive k is capped at kMaxWide - p.
  const int kcap = (int)(minmn <= kMaxWide ? minmn : std::min<int64_t>(minmn, kMaxWide - rp.p));
  if (kcap < 1) return fail(ctx, RSVD_EUNSUPPORTED, "p = %d leaves no room for k under l <= %d", rp.p, kMaxWide);
  if (!adaptive && prm->k > kcap)
    return fail(ctx, RSVD_EUNSUPPORTED, "k = %d exceeds min(m, n) or l = k + p <= %d", prm->k, kMaxWide);
  int k = adaptive ? std::min(2, kcap) : prm->k;
  const int kbuf = adaptive ? kcap : prm->k;
  const double lam = prm->lambda > 0 ? prm->lambda : 1.0 / sqrt((double)std::max(mg, n));
  const double* Ad = (const double*)A->A;
  double* S = (double*)Sout;
  double* Lm = (double*)Lout;
  // rrpca buffers: Z, M (m x n, ld n), U (m x kbuf), V (n x kbuf), d, dl, partials
  const int nb = ialm_blocks();
  const int npart = ialm_partials(n, nb);
  size_t o = 0;
  const size_t oZ = o; o = align256(o + (size_t)m * n * 8);
  const size_t oM = o; o = align256(o + (size_t)m * n * 8);
  const size_t oU = o; o = align256(o + (size_t)m * kbuf * 8);
  const size_t oV = o; o = align256(o + (size_t)n * kbuf * 8);
  const size_t od = o; o = align256(o + (size_t)std::max(128, kbuf) * 8);
  const size_t odl = o; o = align256(o + (size_t)std::max(128, kbuf) * 8);
  const size_t oP = o; o = align256(o + (size_t)2 * nb * 8 + 64);
  // ranks above 128 (wide): L materialised by gemm_pass from U and diag(dl) V^T (kbuf x npad)
  const int64_t npad = round_up(n, 16);
  const bool maybe_wide = kbuf > 128;
  const size_t oVt = o; o = align256(o + (maybe_wide ? (size_t)kbuf * npad * 8 : 0));
  const size_t oGP = o; o = align256(o + (maybe_wide ? gemm_partial_bytes(128, ctx->num_sms) : 0));
  if (o > ctx->ws3_bytes) {
    if (ctx->ws3) { cudaStreamSynchronize(ctx->stream); cudaFree(ctx->ws3); ctx->ws3 = nullptr; ctx->ws3_bytes = 0; }
    if (cudaMalloc(&ctx->ws3, o) != cudaSuccess) { cudaGetLastError(); return fail(ctx, RSVD_ENOMEM, "rrpca workspace"); }
    ctx->ws3_bytes = o;
  }
  double* Z = (double*)(ctx->ws3 + oZ);
  double* M = (double*)(ctx->ws3 + oM);
  double* U = (double*)(ctx->ws3 + oU);
  double* V = (double*)(ctx->ws3 + oV);
  double* dd = (double*)(ctx->ws3 + od);
  double* dl = (double*)(ctx->ws3 + odl);
  double* part = (double*)(ctx->ws3 + oP);
  double* scal = part + 2 * nb;   // [0] = sum, [1] = max, [2] = l
  double* Vt = (double*)(ctx->ws3 + oVt);
  double* gpart = (double*)(ctx->ws3 + oGP);
  double* h = ctx->hbuf;

  // ||A||_2 = sigma_1 of rsvd(A, 1, p, q) with Omega stream 0 (reading R18)
  rsvd_params r1 = rp;
  r1.k = 1; r1.nu = 0; r1.nv = 0; r1.stream = 0;
  CKS(rsvd_device(ctx, A, &r1, nullptr, 0, dd, nullptr, 0));
  // ||A||_F^2 and max|A|
  CK(launch_ialm_init(Ad, A->lda, m, n, part, part + nb, nb, ctx->stream));
  CK(launch_reduce_blocks(part, nb, 0, scal, ctx->stream));
  CK(launch_reduce_blocks(part + nb, nb, 1, scal + 1, ctx->stream));
  CKS(allreduce_sum(ctx, scal, 1));
  CKS(allreduce_max(ctx, scal + 1, 1));
  CK(cudaMemcpyAsync(h, dd, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(h + 1, scal, 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  const double norm2 = h[0], normF = sqrt(h[1]), maxabs = h[2];
  if (!(norm2 > 0) || !std::isfinite(norm2)) return fail(ctx, RSVD_ENUMERIC, "||A||_2 is zero or non-finite");
  const double mu0 = 1.25 / norm2;                         // reading R17
  double mu = mu0;
  const double dual = std::max(norm2, maxabs / lam);       // reading R19
  CK(launch_scale_copy(Ad, A->lda, m, n, dual, Z, ctx->stream));   // Z = A / J(A)
  CK(cudaMemset2DAsync(S, ld * 8, 0, n * 8, m, ctx->stream));       // S = 0
  CK(launch_ialm_form_m(Ad, S, Z, n, m, n, 1.0 / mu, M, ctx->stream));
  rsvd_matrix Mdesc = *A;
  Mdesc.A = M;
  Mdesc.lda = n;
  int it = 0;
  double res = INFINITY;
  int kused = k;
  std::string warn;
  for (it = 1; it <= prm->maxiter; ++it) {
    rsvd_params ri = rp;
    ri.k = ri.nu = ri.nv = k;
    ri.stream = (uint64_t)it;                               // fresh Omega per iteration (R23)
    // deterministic SVD (rand = FALSE, or Remark 2's switch for k > min(m, n)/4):
    // l = min(m, n), q = 0 -> Q Q^T M = M, the SVD of B is the exact SVD
    const bool want_det = !prm->rand || (adaptive && 4 * (int64_t)k > minmn);
    const bool det = want_det && minmn <= kMaxWide;
    if (want_det && !det) {
      char b[200];
      snprintf(b, sizeof b, "warning: deterministic SVD needs min(m, n) <= %d; the randomized SVD is kept (iteration %d, k = %d)",
               kMaxWide, it, k);
      warn = b;
    }
    if (det) {
      ri.p = (int)(minmn - k);
      ri.q = 0;
    }
    CKS(rsvd_device(ctx, &Mdesc, &ri, U, k, dd, V, k));      // step (6)
    CK(launch_ialm_threshold(dd, k, 1.0 / mu, dl, scal + 2, ctx->stream));   // steps (7)-(8)
    const double mu_next = std::min(1.5 * mu, 1e7 * mu0);  // step (12), R20
    if (k <= 128) {
      CK(launch_ialm_update(Ad, S, Z, M, n, m, n, U, k, V, k, dl, k, 1.0 / mu, mu, lam, 1.0 / mu_next, part, nb,
                            ctx->stream));                 // steps (9)-(11) fused
      CK(launch_reduce_blocks(part, npart, 0, scal, ctx->stream));
    } else {
      // step (9) materialised into the L output: L = U (diag(dl) V^T), column blocks of 128
      CK(launch_scale_transpose(V, k, n, k, dl, Vt, npad, ctx->stream));
      for (int64_t j0 = 0; j0 < n; j0 += 128) {
        GemmCall g{};
        g.A = U; g.lda = k; g.a_f32 = false; g.trans = false;
        g.B = Vt + j0; g.ldb = npad; g.C = Lm + j0; g.ldc = ld; g.P = gpart;
        g.M = m; g.K = k; g.N = (int)std::min<int64_t>(128, npad - j0); g.Nout = (int)std::min<int64_t>(g.N, n - j0);
        g.grid = ctx->num_sms;
        g.flags = ctx->gemm_flags; g.epoch = ++ctx->gemm_epoch;
        CK(gemm_pass(g, ctx->stream));
      }
      CK(launch_ialm_update_dense(Ad, S, Z, M, Lm, m * n, 1.0 / mu, mu, lam, 1.0 / mu_next, part, nb,
                                  ctx->stream));           // steps (10)-(11)
      CK(launch_reduce_blocks(part, nb, 0, scal, ctx->stream));
    }
    CKS(allreduce_sum(ctx, scal, 1));
    CK(cudaMemcpyAsync(h + 128, scal, 3 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    res = sqrt(h[128]) / normF;
    const int nl = (int)h[130];
    kused = k;
    if (ctx->debug)
      fprintf(stderr, "rrpca it %d k %d l %d det %d res %.3e mu %.3e t %.3f ms\n", it, k, nl, (int)det, res, mu,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count());
    if (trace) {
      double* tr = trace + 4 * (it - 1);
      tr[0] = res; tr[1] = nl; tr[2] = mu; tr[3] = k;
    }
    if (adaptive) {                                         // step (7) predict_rank (R30)
      const int l1 = std::max(nl, 1);
      int64_t kn = l1 < k ? l1 + 1 : std::min<int64_t>(l1 + (int64_t)ceil(0.05 * (double)minmn), minmn);
      if (kn > kcap) {
        char b[200];
        snprintf(b, sizeof b, "warning: predicted rank %lld capped at %d (l = k + p <= %d)", (long long)kn, kcap, kMaxWide);
        warn = b;
      }
      k = (int)std::min<int64_t>(kn, kcap);
    }
    mu = mu_next;
    if (res < prm->tol) break;
  }
  if (it > prm->maxiter) it = prm->maxiter;
  if (kused <= 128)   // above, the last iteration left L materialised in Lm
    CK(launch_lowrank_materialise(U, kused, V, kused, dl, kused, m, n, Lm, ld, ctx->stream));
  if (iters_out) *iters_out = it;
  if (res_out) *res_out = res;
  CKS(sync_status(ctx));
  if (!warn.empty()) ctx->err = warn;
  return RSVD_OK;
}
