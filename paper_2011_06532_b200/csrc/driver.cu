#include <atomic>
#include <chrono>
// Native drivers behind the C ABI (include/ttb.h): TT construction, Gram
// sweeps, orthonormalization and the four rounding variants.  These replace
// the reference's Python sweep loops (parallel.py:164-209, 293-438;
// ops.py:71-155) with a host loop that only enqueues kernels on the context
// stream; the single host sync per truncation step reads back the kept rank.
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <mutex>
#include <thread>
#include <vector>

#include "ops.cuh"
#include "prof.cuh"
#include "svd.cuh"

struct ttb_tsqr {
  ttb::Tsqr f;
};

namespace ttb {

__global__ void eye_kernel(double* e, int b) {
  for (int idx = threadIdx.x + blockIdx.x * blockDim.x; idx < b * b; idx += blockDim.x * gridDim.x)
    e[idx] = (idx % b == idx / b) ? 1.0 : 0.0;
}

static double* make_eye(Ctx& ctx, int b) {
  double* e = (double*)ctx.alloc((size_t)b * b * sizeof(double));
  eye_kernel<<<1, 256, 0, ctx.stream>>>(e, b);
  TTB_LAUNCHED();
  return e;
}

static void copy_d2d(Ctx& ctx, double* dst, const double* src, int64_t n) {
  if (n > 0) TTB_CUDA(cudaMemcpyAsync(dst, src, (size_t)n * sizeof(double), cudaMemcpyDeviceToDevice, ctx.stream));
}

static Panel panel_of(const double* p, int64_t rl, int64_t I, int64_t rr, int trans) {
  Panel q;
  q.base = const_cast<double*>(p);
  q.rl = rl;
  q.I = I;
  q.rr = rr;
  q.trans = trans;
  q.kron = Kron();
  return q;
}

static void check_chain(int ndim, const int64_t* dims, const int64_t* ranks) {
  TTB_CHECK(ndim >= 1, TTB_ERR_SHAPE, "a TT tensor needs at least one core");
  TTB_CHECK(ranks[0] == 1 && ranks[ndim] == 1, TTB_ERR_SHAPE, "end ranks must be 1");
  for (int n = 0; n < ndim; ++n) {
    TTB_CHECK(dims[n] >= 0, TTB_ERR_SHAPE, "local mode sizes must be >= 0");
    TTB_CHECK(ranks[n + 1] >= 1, TTB_ERR_SHAPE, "ranks must be positive");
  }
}

static double host_scalar(Ctx& ctx, const double* d) {
  double h = 0.0;
  ctx.read_small(d, sizeof(double), &h);
  return h;
}

// sum of squares of a device vector, allreduced over ranks; returns host value
static double global_sumsq(Ctx& ctx, int64_t n, const double* x) {
  double* d = (double*)ctx.alloc(2 * sizeof(double));
  if (n > 0) sumsq_dev(ctx, n, x, d);
  else fill_zero(ctx, d, 1);
  if (ctx.nranks > 1) ctx.allreduce_sum(d, d + 1, 1);
  double v = host_scalar(ctx, ctx.nranks > 1 ? d + 1 : d);
  ctx.free(d);
  return v;
}

// side-stream helpers: the side stream starts after everything enqueued on
// the main stream so far; its allocations are released after the main
// stream's next uses (event ordering, never blocking the main stream).
static void side_begin(Ctx& ctx, Ctx& sctx) {
  cudaEvent_t e;
  TTB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  TTB_CUDA(cudaEventRecord(e, ctx.stream));
  TTB_CUDA(cudaStreamWaitEvent(sctx.stream, e, 0));
  TTB_CUDA(cudaEventDestroy(e));
}

static void side_join(Ctx& ctx, Ctx& sctx) {
  cudaEvent_t e;
  TTB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  TTB_CUDA(cudaEventRecord(e, sctx.stream));
  TTB_CUDA(cudaStreamWaitEvent(ctx.stream, e, 0));
  TTB_CUDA(cudaEventDestroy(e));
}

// diagnostics (TTB_DEBUG_NAN=1): count non-finite entries of a device array, synchronously
static void dbg_nan(Ctx& ctx, cudaStream_t st, const char* what, int n, const double* p, int64_t count) {
  static const bool on = getenv("TTB_DEBUG_NAN") != nullptr;
  if (!on || !p || count <= 0) return;
  std::vector<double> h((size_t)count);
  cudaStreamSynchronize(st);
  cudaMemcpy(h.data(), p, (size_t)count * sizeof(double), cudaMemcpyDeviceToHost);
  int64_t bad = 0;
  double amax = 0.0;
  for (double v : h) {
    if (!std::isfinite(v)) ++bad;
    else amax = std::max(amax, std::fabs(v));
  }
  fprintf(stderr, "[nan] %-28s n=%d count=%lld nonfinite=%lld max|x|=%.3e\n", what, n, (long long)count, (long long)bad, amax);
  (void)ctx;
}

struct SvdOut {
  double* C = nullptr;
  double* Vk = nullptr;
  double* s = nullptr;
  int* info = nullptr;
  double* dinfo = nullptr;
  void* mem = nullptr;
  int keep = 0, capped = 0;
  double tail = 0.0;
};

// SVD of A = R^T (R the b x b TSQR factor), truncated; host learns keep
static void svd_of_rt(Ctx& ctx, const double* R, int b, double eps, int max_rank, SvdOut& o) {
  const size_t bb = (size_t)b * b;
  o.mem = ctx.alloc((2 * bb + b + 1) * sizeof(double) + 4 * sizeof(int) + 64);
  o.C = (double*)o.mem;
  o.Vk = o.C + bb;
  o.s = o.Vk + bb;
  o.dinfo = o.s + b;
  o.info = (int*)(o.dinfo + 1);
  jacobi_svd(ctx, R, b, b, b, true, eps, max_rank, o.C, o.Vk, o.s, o.info, o.dinfo);
  int hinfo[4] = {0, 0, 0, 0};
  ctx.read_small(o.info, 4 * sizeof(int), hinfo);
  prof_note("svd_sweeps", hinfo[3]);
  if (hinfo[2] != 0) {
    ctx.free(o.mem);
    o.mem = nullptr;
    TTB_THROW(TTB_ERR_NUMERIC, "non-finite entries in SVD input");
  }
  o.keep = hinfo[0];
  o.capped = hinfo[1];
}

}  // namespace ttb

using namespace ttb;

extern "C" {

int ttb_scale(ttb_ctx* h, int64_t n, const double* x, double s, double* out) {
  TTB_TRY_BEGIN
  scale_vec(h->c, n, x, s, out);
  TTB_TRY_END
}

int ttb_add(ttb_ctx* h, int nterms, int ndim, const int64_t* dims, const int64_t* ranks, const double* const* cores,
            const double* scales, double* const* out) {
  TTB_TRY_BEGIN
  Ctx& ctx = h->c;
  TTB_CHECK(nterms >= 1 && nterms <= kMaxAddTerms, TTB_ERR_CAPABILITY, "add: 1..16 terms");
  for (int p = 0; p < nterms; ++p) check_chain(ndim, dims, ranks + (int64_t)p * (ndim + 1));
  for (int n = 0; n < ndim; ++n) {
    AddTerm t[kMaxAddTerms];
    int64_t offa = 0, offc = 0;
    for (int p = 0; p < nterms; ++p) {
      const int64_t* rk = ranks + (int64_t)p * (ndim + 1);
      t[p].x = cores[(int64_t)p * ndim + n];
      t[p].rl = rk[n];
      t[p].rr = rk[n + 1];
      t[p].offa = offa;
      t[p].offc = offc;
      t[p].s = scales ? scales[p] : 1.0;
      offa += rk[n];
      offc += rk[n + 1];
    }
    int mode;
    int64_t RL, RR;
    if (ndim == 1) { mode = 3; RL = 1; RR = 1; }
    else if (n == 0) { mode = 1; RL = 1; RR = offc; }
    else if (n == ndim - 1) { mode = 2; RL = offa; RR = 1; }
    else { mode = 0; RL = offa; RR = offc; }
    add_core(ctx, mode, nterms, t, RL, dims[n], RR, out[n]);
  }
  TTB_TRY_END
}

int ttb_hadamard(ttb_ctx* h, int ndim, const int64_t* dims, const int64_t* rx, const int64_t* ry,
                 const double* const* x, const double* const* y, double* const* out) {
  TTB_TRY_BEGIN
  check_chain(ndim, dims, rx);
  check_chain(ndim, dims, ry);
  for (int n = 0; n < ndim; ++n) hadamard_core(h->c, x[n], rx[n], rx[n + 1], y[n], ry[n], ry[n + 1], dims[n], out[n]);
  TTB_TRY_END
}

int ttb_inner(ttb_ctx* h, int ndim, const int64_t* dims, const int64_t* rx, const int64_t* ry,
              const double* const* x, const double* const* y, double* result) {
  TTB_TRY_BEGIN
  Ctx& ctx = h->c;
  check_chain(ndim, dims, rx);
  check_chain(ndim, dims, ry);
  int64_t wmax = 64 * 64;  // largest carry (ranks above 64 take the general path, wide.cu)
  for (int n = 0; n <= ndim; ++n) wmax = std::max<int64_t>(wmax, rx[n] * ry[n]);
  wmax = (wmax + 1) & ~1LL;
  double* buf = (double*)ctx.alloc((size_t)(3 * wmax) * sizeof(double) + 8 * sizeof(int));
  double* W = buf;
  double* Wn = buf + wmax;
  double* Wr = buf + 2 * wmax;
  int* ticket = (int*)(buf + 3 * wmax);  // the 16 x 16 kernel's last-CTA reduction
  static const double one = 1.0;
  TTB_CUDA(cudaMemcpyAsync(W, &one, sizeof(double), cudaMemcpyHostToDevice, ctx.stream));
  TTB_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int), ctx.stream));
  for (int n = 0; n < ndim; ++n) {
    gram_step(ctx, W, x[n], rx[n], rx[n + 1], y[n], ry[n], ry[n + 1], dims[n], Wn, ticket);
    if (ctx.nranks > 1) {
      ctx.allreduce_sum(Wn, Wr, (size_t)(rx[n + 1] * ry[n + 1]));
      std::swap(Wn, Wr);
    }
    std::swap(W, Wn);
  }
  *result = host_scalar(ctx, W);
  ctx.free(buf);
  TTB_TRY_END
}

// ||x||^2 by the symmetric Gram route (norm(method="innerprod_sym"),
// ops.py:179-205): per mode a pivoted Cholesky of the carry, Z = (P L)^T
// H(x_n), W = Z^T Z, allreduced.  An indefinite carry (reconstruction
// residual above 1e-6 ||W||_F at any mode) sets *indefinite and leaves
// *result unspecified: the caller falls back to ttb_inner (ops.py:226-230).
int ttb_norm_sym(ttb_ctx* h, int ndim, const int64_t* dims, const int64_t* ranks, const double* const* in,
                 double* result, int* indefinite) {
  TTB_TRY_BEGIN
  Ctx& ctx = h->c;
  check_chain(ndim, dims, ranks);
  TTB_CHECK(result && indefinite, TTB_ERR_CONTRACT, "null result");
  for (int n = 0; n <= ndim; ++n)
    if (ranks[n] > 64) {
      // ranks above 64: the symmetric route's pivoted Cholesky of the carry
      // is a 64 x 64 kernel; the general Gram sweep computes the same <x, x>
      *indefinite = 0;
      return ttb_inner(h, ndim, dims, ranks, ranks, in, in, result);
    }
  double* buf = (double*)ctx.alloc(5 * 64 * 64 * sizeof(double) + 72 * sizeof(int));
  double* W = buf;
  double* Wn = buf + 4096;
  double* Wr = buf + 8192;
  double* PL = buf + 12288;
  double* Wrec = buf + 16384;
  int* perm = (int*)(buf + 20480);
  int* ticket = perm + 64;
  static const double one = 1.0;
  TTB_CUDA(cudaMemcpyAsync(W, &one, sizeof(double), cudaMemcpyHostToDevice, ctx.stream));
  TTB_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int), ctx.stream));
  ctx.flag_reset();
  pivoted_cholesky(ctx, W, 1, PL, Wrec, perm, nullptr);
  for (int n = 0; n < ndim; ++n) {
    const bool last = n == ndim - 1;
    // one rank: the 16 x 16 step factors the next carry in its own tail
    if (!last && ctx.nranks == 1 && sym16_fusable(ranks[n], ranks[n + 1], dims[n], in[n])) {
      gram_sym_step(ctx, PL, perm, Wrec, in[n], ranks[n], ranks[n + 1], dims[n], nullptr, ticket);
      continue;
    }
    gram_sym_step(ctx, PL, perm, Wrec, in[n], ranks[n], ranks[n + 1], dims[n], Wn, nullptr);
    if (ctx.nranks > 1) {
      ctx.allreduce_sum(Wn, Wr, (size_t)(ranks[n + 1] * ranks[n + 1]));
      std::swap(Wn, Wr);
    }
    std::swap(W, Wn);
    if (!last) pivoted_cholesky(ctx, W, (int)ranks[n + 1], PL, Wrec, perm, nullptr);
  }
  *result = host_scalar(ctx, W);
  *indefinite = ctx.flag_read() ? 1 : 0;
  ctx.free(buf);
  TTB_TRY_END
}

// the reference's _pivoted_cholesky (ops.py:162-176) on one device carry:
// w and pl are device n x n (col-major); pl = P L in w's row order with zero
// columns past the numeric rank; perm (host, n ints) lists the pivots first.
int ttb_pivoted_cholesky(ttb_ctx* h, int n, const double* w, double* pl, int* perm, int* rank, int* indefinite) {
  TTB_TRY_BEGIN
  Ctx& ctx = h->c;
  TTB_CHECK(w && pl && perm && rank && indefinite, TTB_ERR_CONTRACT, "null argument");
  int* ints = (int*)ctx.alloc(72 * sizeof(int));
  ctx.flag_reset();
  pivoted_cholesky(ctx, w, n, pl, nullptr, ints, ints + 64);
  int hbuf[65];
  TTB_CUDA(cudaMemcpyAsync(hbuf, ints, 65 * sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
  TTB_CUDA(cudaStreamSynchronize(ctx.stream));
  for (int i = 0; i < n; ++i) perm[i] = hbuf[i];
  *rank = hbuf[64];
  *indefinite = ctx.flag_read() ? 1 : 0;
  ctx.free(ints);
  TTB_TRY_END
}

int ttb_sumsq(ttb_ctx* h, int64_t n, const double* x, double* result) {
  TTB_TRY_BEGIN
  *result = global_sumsq(h->c, n, x);
  TTB_TRY_END
}

int ttb_orthonormalize(ttb_ctx* h, int direction, int ndim, const int64_t* dims, const int64_t* ranks,
                       const double* const* in, double* const* out) {
  TTB_TRY_BEGIN
  Ctx& ctx = h->c;
  check_chain(ndim, dims, ranks);
  TTB_CHECK(direction == 0 || direction == 1, TTB_ERR_CONTRACT, "direction must be 'left' or 'right'");
  const int N = ndim;
  if (N == 1) {
    copy_d2d(ctx, out[0], in[0], ranks[0] * dims[0] * ranks[1]);
    return TTB_OK;
  }
  ctx.flag_reset();
  if (direction == 0) {
    const double* work = in[0];
    for (int n = 0; n < N - 1; ++n) {
      const int b = (int)ranks[n + 1];
      Tsqr f;
      tsqr_factor(ctx, panel_of(work, ranks[n], dims[n], ranks[n + 1], 0), f);
      double* eye = make_eye(ctx, b);
      tsqr_apply(ctx, f, eye, b, panel_of(out[n], ranks[n], dims[n], b, 0));
      gemm_small_left(ctx, b, b, dims[n + 1] * ranks[n + 2], f.R, b, false, in[n + 1], out[n + 1], true);
      ctx.free(eye);
      tsqr_release(ctx, f);
      work = out[n + 1];
    }
  } else {
    const double* work = in[N - 1];
    for (int n = N - 1; n >= 1; --n) {
      const int b = (int)ranks[n];
      Tsqr f;
      tsqr_factor(ctx, panel_of(work, ranks[n], dims[n], ranks[n + 1], 1), f);
      double* eye = make_eye(ctx, b);
      tsqr_apply(ctx, f, eye, b, panel_of(out[n], b, dims[n], ranks[n + 1], 1));
      gemm_small_right(ctx, ranks[n - 1] * dims[n - 1], b, b, in[n - 1], f.R, b, true, out[n - 1], true);
      ctx.free(eye);
      tsqr_release(ctx, f);
      work = out[n - 1];
    }
  }
  TTB_CHECK(!ctx.flag_read(), TTB_ERR_NUMERIC, "non-finite entries in the tensor (orthonormalization)");
  TTB_TRY_END
}

// ||x||^2 by the orthonormalization route (ops.py:208-235, method "ortho"):
// a right-to-left sweep of R factors only -- TSQR of H(work_n)^T, fold R
// into core n-1 -- without forming the orthonormal cores (no implicit-Q
// apply, no output writes); ||x|| = ||work_0||_F.
int ttb_norm_ortho(ttb_ctx* h, int ndim, const int64_t* dims, const int64_t* ranks, const double* const* in,
                   double* result) {
  TTB_TRY_BEGIN
  Ctx& ctx = h->c;
  check_chain(ndim, dims, ranks);
  TTB_CHECK(result, TTB_ERR_CONTRACT, "null result");
  const int N = ndim;
  if (N == 1) {
    *result = global_sumsq(ctx, ranks[0] * dims[0] * ranks[1], in[0]);
    return TTB_OK;
  }
  int64_t maxc = 1;
  for (int n = 0; n < N - 1; ++n) maxc = std::max<int64_t>(maxc, ranks[n] * dims[n] * ranks[n + 1]);
  double* buf[2] = {(double*)ctx.alloc((size_t)maxc * sizeof(double)),
                    (double*)ctx.alloc((size_t)maxc * sizeof(double))};
  ctx.flag_reset();
  const double* work = in[N - 1];
  int which = 0;
  for (int n = N - 1; n >= 1; --n) {
    const int b = (int)ranks[n];
    Tsqr f;
    f.r_only = true;  // no implicit Q is ever applied: the leaf skips Y and T
    tsqr_factor(ctx, panel_of(work, ranks[n], dims[n], ranks[n + 1], 1), f);
    gemm_small_right(ctx, ranks[n - 1] * dims[n - 1], b, b, in[n - 1], f.R, b, true, buf[which], true);
    tsqr_release(ctx, f);
    work = buf[which];
    which ^= 1;
  }
  TTB_CHECK(!ctx.flag_read(), TTB_ERR_NUMERIC, "non-finite entries in the tensor (orthonormalization)");
  *result = global_sumsq(ctx, ranks[0] * dims[0] * ranks[1], work);
  ctx.free(buf[0]);
  ctx.free(buf[1]);
  TTB_TRY_END
}

// Host-resident cores for ttb_round_host: the H2D copy of every input core
// is queued up front on the context's copy stream (one event per core) and
// the compute stream waits for core n only where the sweep first reads it;
// every output core is copied back as soon as it is final (event on the
// stream that finished it), so both transfers overlap the sweeps.  Host
// pageable buffers go through the context's page-locked staging ring: a
// worker thread copies 32 MB chunks user -> ring with several host threads
// while the copy engine drains the previous chunks (and the mirror image for
// outputs), so the call neither page-locks user memory (cudaHostRegister
// costs ~0.25 ms per MB: 570 ms on cfg3) nor falls back to the driver's
// synchronous pageable copies (290 ms).
struct HostIO {
  Ctx& ctx;
  int N;
  const double* const* hin;
  double* const* hout;
  std::vector<cudaEvent_t> in_ev;
  std::vector<char> waited;
  std::vector<cudaEvent_t> evs;
  // staging worker
  struct Job {
    int kind;  // 0: host -> device, 1: device -> host
    int n;
    const char* src;
    char* dst;
    size_t bytes;
    cudaEvent_t after;  // D2H: the producer's completion
  };
  std::deque<Job> jobs;
  std::mutex mu;
  std::condition_variable cv_job, cv_rec;
  std::vector<char> recorded;  // in_ev[n] has been recorded (staged uploads: by the worker)
  bool closing = false;
  std::atomic<bool> failed{false};
  std::thread worker;
  int slot = 0;
  bool staged_ok = false;

  HostIO(Ctx& c, int n, const double* const* in, double* const* out)
      : ctx(c), N(n), hin(in), hout(out), in_ev(n, nullptr), waited(n, 0), recorded(n, 0) {}
  cudaStream_t cs() { return ctx.copy_stream(); }
  static bool device_visible(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) == cudaSuccess &&
        (a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged))
      return true;
    cudaGetLastError();
    return false;
  }
  static void par_memcpy(char* dst, const char* src, size_t bytes) {
    constexpr int kThreads = 6;
    const size_t part = ((bytes / kThreads) + 4095) & ~size_t(4095);
    if (bytes < (size_t(4) << 20) || part == 0) {
      memcpy(dst, src, bytes);
      return;
    }
    std::thread th[kThreads - 1];
    int nth = 0;
    size_t off = part;
    for (; nth < kThreads - 1 && off < bytes; ++nth, off += part) {
      const size_t len = std::min(part, bytes - off);
      th[nth] = std::thread([=] { memcpy(dst + off, src + off, len); });
    }
    memcpy(dst, src, std::min(part, bytes));
    for (int i = 0; i < nth; ++i) th[i].join();
  }
  void run_job(const Job& j) {
    const size_t CH = Ctx::kStageBytes;
    if (j.kind == 0) {
      for (size_t off = 0; off < j.bytes; off += CH) {
        const size_t len = std::min(CH, j.bytes - off);
        const int s = slot++ % Ctx::kStageSlots;
        TTB_CUDA(cudaEventSynchronize(ctx.stage_ev[s]));  // the slot's previous transfer has drained
        par_memcpy((char*)ctx.stage_buf[s], j.src + off, len);
        TTB_CUDA(cudaMemcpyAsync(j.dst + off, ctx.stage_buf[s], len, cudaMemcpyHostToDevice, cs()));
        TTB_CUDA(cudaEventRecord(ctx.stage_ev[s], cs()));
      }
      TTB_CUDA(cudaEventRecord(in_ev[j.n], cs()));
      {
        std::lock_guard<std::mutex> lk(mu);
        recorded[j.n] = 1;
      }
      cv_rec.notify_all();
    } else {
      TTB_CUDA(cudaStreamWaitEvent(cs(), j.after, 0));
      int prev = -1;
      size_t poff = 0, plen = 0;
      for (size_t off = 0; off < j.bytes; off += CH) {
        const size_t len = std::min(CH, j.bytes - off);
        const int s = slot++ % Ctx::kStageSlots;
        TTB_CUDA(cudaEventSynchronize(ctx.stage_ev[s]));
        TTB_CUDA(cudaMemcpyAsync(ctx.stage_buf[s], j.src + off, len, cudaMemcpyDeviceToHost, cs()));
        TTB_CUDA(cudaEventRecord(ctx.stage_ev[s], cs()));
        if (prev >= 0) {  // the previous chunk leaves the ring while this one arrives
          TTB_CUDA(cudaEventSynchronize(ctx.stage_ev[prev]));
          par_memcpy(j.dst + poff, (const char*)ctx.stage_buf[prev], plen);
        }
        prev = s;
        poff = off;
        plen = len;
      }
      if (prev >= 0) {
        TTB_CUDA(cudaEventSynchronize(ctx.stage_ev[prev]));
        par_memcpy(j.dst + poff, (const char*)ctx.stage_buf[prev], plen);
      }
    }
  }
  void worker_main() {
    cudaSetDevice(ctx.device);
    for (;;) {
      Job j;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv_job.wait(lk, [&] { return closing || !jobs.empty(); });
        if (jobs.empty()) return;
        j = jobs.front();
        jobs.pop_front();
      }
      try {
        if (!failed) run_job(j);
      } catch (...) {
        failed = true;
      }
      if (failed && j.kind == 0) {  // never leave the compute thread waiting
        {
          std::lock_guard<std::mutex> lk(mu);
          recorded[j.n] = 1;
        }
        cv_rec.notify_all();
      }
    }
  }
  void submit(const Job& j) {
    if (!worker.joinable()) worker = std::thread([this] { worker_main(); });
    {
      std::lock_guard<std::mutex> lk(mu);
      jobs.push_back(j);
    }
    cv_job.notify_one();
  }
  bool staged(const void* p, size_t bytes) {
    static const bool off = getenv("TTB_HOSTIO_NOSTAGE") != nullptr;  // diagnostics: plain pageable copies
    if (off || !p || bytes == 0 || device_visible(p)) return false;
    if (!staged_ok) staged_ok = ctx.stage_init();
    return staged_ok;
  }
  void upload(int n, double* dst, int64_t count) {
    const size_t bytes = (size_t)count * sizeof(double);
    TTB_CUDA(cudaEventCreateWithFlags(&in_ev[n], cudaEventDisableTiming));
    if (staged(hin[n], bytes)) {
      submit(Job{0, n, (const char*)hin[n], (char*)dst, bytes, nullptr});
      return;
    }
    TTB_CUDA(cudaMemcpyAsync(dst, hin[n], bytes, cudaMemcpyHostToDevice, cs()));
    TTB_CUDA(cudaEventRecord(in_ev[n], cs()));
    recorded[n] = 1;
  }
  void need(int n, cudaStream_t st) {
    if (n < 0 || n >= N || waited[n]) return;
    if (!recorded[n]) {  // a staged upload: wait until the worker has enqueued its last chunk
      std::unique_lock<std::mutex> lk(mu);
      cv_rec.wait(lk, [&] { return recorded[n] != 0; });
    }
    TTB_CHECK(!failed, TTB_ERR_CUDA, "host staging copy failed");
    TTB_CUDA(cudaStreamWaitEvent(st, in_ev[n], 0));
    waited[n] = 1;
  }
  void ready(int n, const double* src, int64_t count, cudaStream_t st) {
    cudaEvent_t e;
    TTB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    TTB_CUDA(cudaEventRecord(e, st));
    evs.push_back(e);
    const size_t bytes = (size_t)count * sizeof(double);
    if (staged(hout[n], bytes)) {
      submit(Job{1, n, (const char*)src, (char*)hout[n], bytes, e});
      return;
    }
    if (worker.joinable()) drain();  // keep the copy stream's order: staged jobs first
    TTB_CUDA(cudaStreamWaitEvent(cs(), e, 0));
    TTB_CUDA(cudaMemcpyAsync(hout[n], src, bytes, cudaMemcpyDeviceToHost, cs()));
  }
  void drain() {
    if (!worker.joinable()) return;
    {
      std::lock_guard<std::mutex> lk(mu);
      closing = true;
    }
    cv_job.notify_all();
    worker.join();
    closing = false;
  }
  void finish() {
    drain();
    // the compute stream must not run past the copies (device buffers are
    // freed stream-ordered on it), and the caller reads host memory
    cudaEvent_t e;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess) {
      cudaEventRecord(e, cs());
      cudaStreamWaitEvent(ctx.stream, e, 0);
      cudaEventDestroy(e);
    }
    cudaStreamSynchronize(cs());
    for (auto e2 : in_ev)
      if (e2) cudaEventDestroy(e2);
    for (auto e2 : evs) cudaEventDestroy(e2);
    in_ev.clear();
    evs.clear();
  }
  ~HostIO() {
    if (worker.joinable()) {
      {
        std::lock_guard<std::mutex> lk(mu);
        closing = true;
      }
      cv_job.notify_all();
      worker.join();
    }
  }
};


struct HostTimer {  // diagnostics: TTB_DEBUG_HOSTTIME prints host-side phase times per round
  const char* name;
  double* acc;
  std::chrono::steady_clock::time_point t0;
  HostTimer(const char* n, double* a) : name(n), acc(a), t0(std::chrono::steady_clock::now()) {}
  ~HostTimer() { *acc += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); }
};

// kin (optional, ndim entries): the input cores are implicit Hadamard cores
// (ttb_round_hadamard); they are only ever read by the first sweep's first
// TSQR panel and its R-folds, which form the Kronecker slices on the fly.
static void round_impl(Ctx& ctx, int variant, double eps0, int64_t max_rank, int ndim, const int64_t* dims,
                       const int64_t* ranks, const double* const* in, double* const* out, int64_t* out_ranks,
                       double* meta, HostIO* io, const Kron* kin = nullptr) {
  check_chain(ndim, dims, ranks);
  static const bool htime = getenv("TTB_DEBUG_HOSTTIME") != nullptr;
  double t_all = 0, t_fac = 0, t_svd = 0, t_app = 0, t_flush = 0, t_norm = 0;
  const double alloc0 = g_host_alloc_ms;
  struct Report {
    bool on; double *a, *f, *s, *p, *fl, *nm; double alloc0;
    ~Report() {
      if (on)
        fprintf(stderr, "[hosttime] factor %.2f svd %.2f apply %.2f flush %.2f norm %.2f alloc %.2f ms\n", *f, *s, *p, *fl,
                *nm, g_host_alloc_ms - alloc0);
    }
  } rep{htime, &t_all, &t_fac, &t_svd, &t_app, &t_flush, &t_norm, alloc0};
  TTB_CHECK(variant >= 0 && variant <= 3, TTB_ERR_CONTRACT, "unknown rounding variant");
  TTB_CHECK(eps0 >= 0.0, TTB_ERR_CONTRACT, "eps0 must be nonnegative");
  const int N = ndim;
  const bool implicit = (variant == 0 || variant == 2);
  const bool left_first = (variant == 0 || variant == 1);
  std::vector<int64_t> r(ranks, ranks + N + 1);
  std::vector<int64_t> d(dims, dims + N);
  meta[0] = NAN;  // norm
  meta[1] = NAN;  // eps_bond
  meta[2] = 0.0;  // error_bound_violated
  meta[3] = 0.0;  // zero
  if (N == 1) {
    if (io) io->need(0, ctx.stream);
    if (kin) hadamard_core(ctx, kin[0].x, kin[0].rxl, kin[0].rxr, kin[0].w, kin[0].rwl, kin[0].rwr, d[0], out[0]);
    else copy_d2d(ctx, out[0], in[0], r[0] * d[0] * r[1]);
    for (int n = 0; n <= N; ++n) out_ranks[n] = r[n];
    if (io) io->ready(0, out[0], r[0] * d[0] * r[1], ctx.stream);
    return;
  }
  const int mr = max_rank > 0 ? (int)std::min<int64_t>(max_rank, 1 << 30) : 0;
  std::vector<Tsqr> facs(N);
  int64_t maxcore = 0;
  for (int n = 0; n < N; ++n) maxcore = std::max(maxcore, r[n] * d[n] * r[n + 1]);
  double* scratch = implicit ? nullptr : (double*)ctx.alloc((size_t)std::max<int64_t>(maxcore, 1) * sizeof(double));
  // unwind (a NumericError from the SVD of non-finite data, a CUDA error):
  // hand every live workspace block back to the pool, after the side stream
  // drained into the main stream, so the context stays usable
  Ctx sctx = ctx;
  bool side_used = false;
  Tsqr f2cur;
  SvdOut socur;
  struct PendingOut {
    bool on = false;
    Tsqr f2;
    SvdOut so;
    Panel out;
    int n = 0;
    int64_t count = 0;
  } pend;
  struct Unwind {
    Ctx& ctx;
    Ctx& sctx;
    bool& side_used;
    std::vector<Tsqr>& facs;
    double*& scratch;
    Tsqr& f2cur;
    SvdOut& socur;
    PendingOut& pend;
    bool armed = true;
    ~Unwind() {
      if (!armed) return;
      try {
        if (side_used) side_join(ctx, sctx);
        for (auto& f : facs)
          if (f.mem) tsqr_release(ctx, f);
        if (f2cur.mem) tsqr_release(ctx, f2cur);
        if (socur.mem) ctx.free(socur.mem);
        if (pend.on) {
          if (pend.f2.mem) tsqr_release(ctx, pend.f2);
          if (pend.so.mem) ctx.free(pend.so.mem);
        }
        if (scratch) ctx.free(scratch);
        ctx.collect(true);
      } catch (...) {
      }
    }
  } unwind{ctx, sctx, side_used, facs, scratch, f2cur, socur, pend};

  // ---- orthonormalization sweep (implicit Q kept for *I variants) ----
  const double* last = nullptr;
  int64_t last_n = 0;
  if (left_first) {
    for (int n = 0; n < N - 1; ++n) {
      const double* src = (n == 0) ? in[0] : out[n];
      const int b = (int)r[n + 1];
      if (io && n == 0) io->need(0, ctx.stream);
      Panel pn = panel_of(src, r[n], d[n], r[n + 1], 0);
      if (kin && n == 0) pn.kron = kin[0];
      { HostTimer ht("fac", &t_fac); tsqr_factor(ctx, pn, facs[n]); }
      if (io) io->need(n + 1, ctx.stream);
      if (!implicit) {
        double* eye = make_eye(ctx, b);
        tsqr_apply(ctx, facs[n], eye, b, panel_of(out[n], r[n], d[n], b, 0));
        ctx.free(eye);
      }
      gemm_small_left(ctx, b, b, d[n + 1] * r[n + 2], facs[n].R, b, false, kin ? nullptr : in[n + 1], out[n + 1],
                      true, kin ? &kin[n + 1] : nullptr, d[n + 1]);
      if (!implicit) tsqr_release(ctx, facs[n]);
    }
    last = out[N - 1];
    last_n = r[N - 1] * d[N - 1] * r[N];
  } else {
    for (int n = N - 1; n >= 1; --n) {
      const double* src = (n == N - 1) ? in[N - 1] : out[n];
      const int b = (int)r[n];
      if (io && n == N - 1) io->need(N - 1, ctx.stream);
      Panel pn = panel_of(src, r[n], d[n], r[n + 1], 1);
      if (kin && n == N - 1) pn.kron = kin[N - 1];
      tsqr_factor(ctx, pn, facs[n]);
      if (io) io->need(n - 1, ctx.stream);
      if (!implicit) {
        double* eye = make_eye(ctx, b);
        tsqr_apply(ctx, facs[n], eye, b, panel_of(out[n], b, d[n], r[n + 1], 1));
        ctx.free(eye);
      }
      gemm_small_right(ctx, r[n - 1] * d[n - 1], b, b, kin ? nullptr : in[n - 1], facs[n].R, b, true, out[n - 1], true,
                       kin ? &kin[n - 1] : nullptr, d[n - 1]);
      if (!implicit) tsqr_release(ctx, facs[n]);
    }
    last = out[0];
    last_n = r[0] * d[0] * r[1];
  }

  // ---- norm and per-bond threshold ----
  double nx;
  { HostTimer ht("norm", &t_norm); nx = std::sqrt(std::max(global_sumsq(ctx, last_n, last), 0.0)); }
  meta[0] = nx;
  if (nx < 1e-300) {
    for (int n = 0; n < N; ++n) {
      if (implicit && facs[n].mem) tsqr_release(ctx, facs[n]);
      fill_zero(ctx, out[n], d[n]);
    }
    for (int n = 0; n <= N; ++n) out_ranks[n] = 1;
    meta[3] = 1.0;
    unwind.armed = false;
    if (scratch) ctx.free(scratch);
    if (io)
      for (int n = 0; n < N; ++n) io->ready(n, out[n], d[n], ctx.stream);
    return;
  }
  const double eps = eps0 * nx / std::sqrt((double)(N - 1));
  meta[1] = eps;

  // ---- truncation sweep ----
  // The output core of step n (Q2 V, from this step's TSQR factor and SVD)
  // is off the critical path: it is computed on the side stream, deferred
  // until the next step's TSQR has been enqueued, so that it runs while the
  // main stream sits in the one-CTA SVD instead of competing with the
  // critical carry apply.
  bool violated = false;
  sctx.stream = ctx.side_stream();
  sctx.deferred.clear();  // deferred frees belong to the main context only
  auto flush = [&]() {
    if (!pend.on) return;
    side_begin(ctx, sctx);  // after everything enqueued on main so far
    side_used = true;
    dbg_nan(ctx, sctx.stream, "flush: Vk", pend.n, pend.so.Vk, (int64_t)pend.f2.b * pend.so.keep);
    dbg_nan(ctx, sctx.stream, "flush: f2.T (tile 0)", pend.n, pend.f2.T, (int64_t)pend.f2.b * pend.f2.b);
    dbg_nan(ctx, sctx.stream, "flush: f2.D", pend.n, pend.f2.D, pend.f2.b);
    tsqr_apply(sctx, pend.f2, pend.so.Vk, pend.so.keep, pend.out);
    dbg_nan(ctx, sctx.stream, "flush: output core", pend.n, pend.out.base, pend.count);
    if (io) io->ready(pend.n, pend.out.base, pend.count, sctx.stream);
    ctx.free_after(pend.f2.mem, sctx.stream);  // returned to the pool on the main stream
    pend.f2.mem = nullptr;
    if (pend.f2.t_ready) {  // the apply above waited on it
      cudaEventDestroy(pend.f2.t_ready);
      pend.f2.t_ready = nullptr;
    }
    ctx.free_after(pend.so.mem, sctx.stream);
    pend.on = false;
  };
  if (left_first) {
    for (int n = N - 1; n >= 1; --n) {
      const int b = (int)r[n];
      Tsqr& f2 = f2cur;
      dbg_nan(ctx, ctx.stream, "sweep2: panel in", n, out[n], r[n] * d[n] * r[n + 1]);
      { HostTimer ht("fac", &t_fac); tsqr_factor(ctx, panel_of(out[n], r[n], d[n], r[n + 1], 1), f2); }
      dbg_nan(ctx, ctx.stream, "sweep2: R", n, f2.R, (int64_t)r[n] * r[n]);
      { HostTimer ht("flush", &t_flush); flush(); }  // previous step's output core overlaps this step's SVD
      SvdOut& so = socur;
      { HostTimer ht("svd", &t_svd); svd_of_rt(ctx, f2.R, b, eps, mr, so); }
      const int keep = so.keep;
      violated |= so.capped != 0;
      if (implicit) {
        HostTimer ht("app", &t_app);
        tsqr_apply(ctx, facs[n - 1], so.C, keep, panel_of(out[n - 1], r[n - 1], d[n - 1], keep, 0));
        tsqr_release(ctx, facs[n - 1]);
      } else {
        const int64_t Mb = r[n - 1] * d[n - 1];
        gemm_small_right(ctx, Mb, b, keep, out[n - 1], so.C, b, false, scratch);
        copy_d2d(ctx, out[n - 1], scratch, Mb * keep);
      }
      pend.on = true;
      pend.f2 = f2;
      pend.so = so;
      f2cur = Tsqr();
      socur = SvdOut();
      pend.out = panel_of(out[n], keep, d[n], r[n + 1], 1);
      pend.n = n;
      pend.count = (int64_t)keep * d[n] * r[n + 1];
      r[n] = keep;
    }
    flush();
    if (io) io->ready(0, out[0], r[0] * d[0] * r[1], ctx.stream);
  } else {
    for (int n = 0; n < N - 1; ++n) {
      const int b = (int)r[n + 1];
      Tsqr& f2 = f2cur;
      tsqr_factor(ctx, panel_of(out[n], r[n], d[n], r[n + 1], 0), f2);
      flush();
      SvdOut& so = socur;
      svd_of_rt(ctx, f2.R, b, eps, mr, so);
      const int keep = so.keep;
      violated |= so.capped != 0;
      if (implicit) {
        tsqr_apply(ctx, facs[n + 1], so.C, keep, panel_of(out[n + 1], keep, d[n + 1], r[n + 2], 1));
        tsqr_release(ctx, facs[n + 1]);
      } else {
        const int64_t Nb = d[n + 1] * r[n + 2];
        gemm_small_left(ctx, keep, b, Nb, so.C, b, true, out[n + 1], scratch);
        copy_d2d(ctx, out[n + 1], scratch, keep * Nb);
      }
      pend.on = true;
      pend.f2 = f2;
      pend.so = so;
      f2cur = Tsqr();
      socur = SvdOut();
      pend.out = panel_of(out[n], r[n], d[n], keep, 0);
      pend.n = n;
      pend.count = r[n] * d[n] * (int64_t)keep;
      r[n + 1] = keep;
    }
    flush();
    if (io) io->ready(N - 1, out[N - 1], r[N - 1] * d[N - 1] * r[N], ctx.stream);
  }
  side_join(ctx, sctx);
  unwind.armed = false;
  ctx.collect(true);
  if (scratch) ctx.free(scratch);
  meta[2] = violated ? 1.0 : 0.0;
  for (int n = 0; n <= N; ++n) out_ranks[n] = r[n];
}

int ttb_round(ttb_ctx* h, int variant, double eps0, int64_t max_rank, int ndim, const int64_t* dims,
              const int64_t* ranks, const double* const* in, double* const* out, int64_t* out_ranks, double* meta) {
  TTB_TRY_BEGIN
  round_impl(h->c, variant, eps0, max_rank, ndim, dims, ranks, in, out, out_ranks, meta, nullptr);
  TTB_TRY_END
}

int ttb_round_hadamard(ttb_ctx* h, int variant, double eps0, int64_t max_rank, int ndim, const int64_t* dims,
                       const int64_t* rx, const int64_t* rw, const double* const* x, const double* const* w,
                       double* const* out, int64_t* out_ranks, double* meta) {
  TTB_TRY_BEGIN
  check_chain(ndim, dims, rx);
  check_chain(ndim, dims, rw);
  TTB_CHECK(x && w && out, TTB_ERR_CONTRACT, "null core pointer array");
  std::vector<int64_t> r(ndim + 1);
  std::vector<Kron> kz(ndim);
  for (int n = 0; n <= ndim; ++n) r[n] = rx[n] * rw[n];
  for (int n = 0; n < ndim; ++n) {
    kz[n].x = x[n];
    kz[n].w = w[n];
    kz[n].rxl = rx[n];
    kz[n].rxr = rx[n + 1];
    kz[n].rwl = rw[n];
    kz[n].rwr = rw[n + 1];
  }
  bool wide = false;
  for (int n = 0; n <= ndim; ++n) wide |= r[n] > 64;
  if (wide) {
    // product ranks above 64 take the general path (wide.cu), which reads
    // materialised cores: form the Hadamard product once, then round it
    Ctx& ctx = h->c;
    std::vector<double*> z(ndim, nullptr);
    std::vector<const double*> zc(ndim, nullptr);
    try {
      for (int n = 0; n < ndim; ++n) {
        z[n] = (double*)ctx.alloc((size_t)std::max<int64_t>(r[n] * dims[n] * r[n + 1], 1) * sizeof(double));
        zc[n] = z[n];
        hadamard_core(ctx, x[n], rx[n], rx[n + 1], w[n], rw[n], rw[n + 1], dims[n], z[n]);
      }
      round_impl(ctx, variant, eps0, max_rank, ndim, dims, r.data(), zc.data(), out, out_ranks, meta, nullptr);
    } catch (...) {
      for (double* p : z)
        if (p) ctx.free(p);
      throw;
    }
    for (double* p : z) ctx.free(p);
    return TTB_OK;
  }
  std::vector<const double*> none(ndim, nullptr);
  round_impl(h->c, variant, eps0, max_rank, ndim, dims, r.data(), none.data(), out, out_ranks, meta, nullptr,
             kz.data());
  TTB_TRY_END
}

int ttb_round_host(ttb_ctx* h, int variant, double eps0, int64_t max_rank, int ndim, const int64_t* dims,
                   const int64_t* ranks, const double* const* in, double* const* out, int64_t* out_ranks,
                   double* meta) {
  TTB_TRY_BEGIN
  Ctx& ctx = h->c;
  check_chain(ndim, dims, ranks);
  TTB_CHECK(in && out, TTB_ERR_CONTRACT, "null core pointer array");
  static const bool dbg = getenv("TTB_DEBUG_HOSTIO") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!dbg) return;
    cudaStreamSynchronize(ctx.stream);
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    fprintf(stderr, "[hostio] %-28s %8.2f ms\n", what, ms);
  };
  std::vector<int64_t> sz(ndim);
  int64_t total = 0;
  for (int n = 0; n < ndim; ++n) {
    sz[n] = ranks[n] * dims[n] * ranks[n + 1];
    total += (sz[n] + 31) / 32 * 32;
  }
  // device images of the input and output cores (output cores sized by the
  // input ranks, as ttb_round)
  double* dmem = (double*)ctx.alloc((size_t)std::max<int64_t>(2 * total, 1) * sizeof(double));
  std::vector<const double*> din(ndim);
  std::vector<double*> dout(ndim);
  int64_t off = 0;
  for (int n = 0; n < ndim; ++n) {
    din[n] = dmem + off;
    dout[n] = dmem + total + off;
    off += (sz[n] + 31) / 32 * 32;
  }
  HostIO io(ctx, ndim, in, out);
  {  // the copy stream may only touch dmem after its stream-ordered allocation
    cudaEvent_t e;
    TTB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    TTB_CUDA(cudaEventRecord(e, ctx.stream));
    TTB_CUDA(cudaStreamWaitEvent(io.cs(), e, 0));
    TTB_CUDA(cudaEventDestroy(e));
  }
  mark("alloc");
  for (int n = 0; n < ndim; ++n) io.upload(n, const_cast<double*>(din[n]), sz[n]);
  mark("uploads queued");
  try {
    round_impl(ctx, variant, eps0, max_rank, ndim, dims, ranks, din.data(), dout.data(), out_ranks, meta, &io);
  } catch (...) {
    io.finish();
    ctx.free(dmem);
    throw;
  }
  mark("round done (compute stream)");
  io.finish();
  mark("copies done");
  ctx.free(dmem);
  TTB_CHECK(!io.failed, TTB_ERR_CUDA, "host staging copy failed");
  TTB_TRY_END
}



int ttb_tsqr_factor(ttb_ctx* h, int64_t rl, int64_t I, int64_t rr, int trans, const double* slab, ttb_tsqr** out,
                    double* r_out) {
  TTB_TRY_BEGIN
  Ctx& ctx = h->c;
  TTB_CHECK(out, TTB_ERR_CONTRACT, "null factor handle");
  ttb_tsqr* f = new ttb_tsqr();
  try {
    ctx.flag_reset();
    tsqr_factor(ctx, panel_of(slab, rl, I, rr, trans ? 1 : 0), f->f);
    if (ctx.flag_read()) {
      tsqr_release(ctx, f->f);
      TTB_THROW(TTB_ERR_NUMERIC, "non-finite entries in the TSQR panel");
    }
  } catch (...) {
    delete f;
    throw;
  }
  if (r_out) copy_d2d(ctx, r_out, f->f.R, (int64_t)f->f.b * f->f.b);
  *out = f;
  TTB_TRY_END
}

int ttb_tsqr_apply(ttb_ctx* h, const ttb_tsqr* f, int64_t k, const double* c, double* out) {
  TTB_TRY_BEGIN
  const Tsqr& F = f->f;
  Panel o = F.panel;
  o.base = out;
  if (o.trans) o.rl = k;
  else o.rr = k;
  tsqr_apply(h->c, F, c, (int)k, o);
  TTB_TRY_END
}

int ttb_tsqr_free(ttb_ctx* h, ttb_tsqr* f) {
  TTB_TRY_BEGIN
  if (f) {
    tsqr_release(h->c, f->f);
    delete f;
  }
  TTB_TRY_END
}

int ttb_truncated_svd(ttb_ctx* h, int64_t m, int64_t n, const double* a, double eps, int64_t max_rank, double* u,
                      double* s, double* v, int64_t* keep, double* tail, int* capped) {
  TTB_TRY_BEGIN
  Ctx& ctx = h->c;
  TTB_CHECK(m >= 1 && n >= 1 && m <= 4096 && n <= 4096, TTB_ERR_CAPABILITY, "truncated_svd: 1 <= m, n <= 4096");
  TTB_CHECK(eps >= 0.0, TTB_ERR_CONTRACT, "eps must be nonnegative");
  const bool tall = m >= n;
  const int M = (int)(tall ? m : n), Nn = (int)(tall ? n : m);
  const size_t need = (size_t)(M * Nn + Nn * Nn + Nn + 1) * sizeof(double) + 4 * sizeof(int);
  char* mem = (char*)ctx.alloc(need + 64);
  double* C = (double*)mem;
  double* Vk = C + (size_t)M * Nn;
  double* sd = Vk + (size_t)Nn * Nn;
  double* dinfo = sd + Nn;
  int* info = (int*)(dinfo + 1);
  jacobi_svd(ctx, a, (int)m, M, Nn, !tall, eps, max_rank > 0 ? (int)max_rank : 0, C, Vk, sd, info, dinfo);
  int hinfo[3];
  TTB_CUDA(cudaMemcpyAsync(hinfo, info, 3 * sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
  TTB_CUDA(cudaMemcpyAsync(tail, dinfo, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
  ctx.sync();
  TTB_CHECK(hinfo[2] == 0, TTB_ERR_NUMERIC, "non-finite entries in SVD input");
  const int kp = hinfo[0];
  *keep = kp;
  *capped = hinfo[1];
  copy_d2d(ctx, s, sd, kp);
  if (tall) {  // A = (C/s) V^T
    svd_normalize_u(ctx, C, sd, M, kp, u);
    copy_d2d(ctx, v, Vk, (int64_t)Nn * kp);
  } else {     // A^T = (C/s) Vk^T  =>  A = Vk s (C/s)^T
    copy_d2d(ctx, u, Vk, (int64_t)Nn * kp);
    svd_normalize_u(ctx, C, sd, M, kp, v);
  }
  ctx.sync();
  ctx.free(mem);
  TTB_TRY_END
}

}  // extern "C"
