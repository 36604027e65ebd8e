// Context, error plumbing, NCCL (dlopen) and the context C-ABI entry points.
#include <dlfcn.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "ctx.cuh"

namespace ttb {

static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};
// collective traffic of this process (Trace words / messages): [0] TSQR
// allgathers, [1] their doubles, [2] allreduces + point-to-point exchanges,
// [3] their doubles
static std::atomic<long long> g_comm[4] = {{0}, {0}, {0}, {0}};

void set_last_error(const std::string& msg) { g_last_error = msg; }
void count_launch(int n) { g_launches += n; }

void smem_attr(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;  // (kernel, device) -> bytes set
  int dev = 0;
  TTB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto it = done.find({fn, dev});
  if (it != done.end() && it->second >= bytes) return;
  TTB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  done[{fn, dev}] = bytes;
}

// ---- in-process group ------------------------------------------------------
// P contexts of one process (each driven by its own host thread) exchange
// device buffers at the very call sites NCCL serves in a multi-process run.
// Every collective is two host rendezvous: (1) every rank posts its send
// buffers and records a "ready" event on its stream; (2) after copying what
// it needs (stream-ordered behind the owners' ready events) every rank
// records "done"; its stream then waits for every peer's done event, so no
// rank reuses or frees a buffer a peer still reads.  The GPU never waits on
// an event that was not recorded yet (the rendezvous orders the host calls).
// Reductions are rank-ascending sums (bitwise deterministic, as the
// reference's _SimGroup._combine, comm.py:213-227).
struct LocalGroup {
  int P;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long gen = 0;
  bool broken = false;
  int joined = 0;
  std::vector<const void*> post;                  // allgather / allreduce: per rank
  std::vector<std::pair<const double*, int64_t>> p2p;  // [src * P + dst]
  std::vector<cudaEvent_t> ready, done;
  explicit LocalGroup(int p) : P(p), post(p, nullptr), p2p((size_t)p * p, {nullptr, 0}), ready(p, nullptr), done(p, nullptr) {}
  void barrier() {
    static const int timeout_s = getenv("TTB_GROUP_TIMEOUT_S") ? atoi(getenv("TTB_GROUP_TIMEOUT_S")) : 300;
    std::unique_lock<std::mutex> lk(mu);
    TTB_CHECK(!broken, TTB_ERR_DEADLOCK, "in-process group: a peer failed or timed out");
    const unsigned long long g = gen;
    if (++arrived == P) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    if (!cv.wait_for(lk, std::chrono::seconds(timeout_s), [&] { return gen != g || broken; })) {
      broken = true;
      cv.notify_all();
      TTB_THROW(TTB_ERR_DEADLOCK, "in-process group: collective timed out waiting for a peer");
    }
    TTB_CHECK(gen != g, TTB_ERR_DEADLOCK, "in-process group: a peer failed or timed out");
  }
  void fail() {
    std::lock_guard<std::mutex> lk(mu);
    broken = true;
    cv.notify_all();
  }
};

namespace {
// a failing rank must release its peers from the rendezvous
struct GroupGuard {
  LocalGroup* g;
  bool ok = false;
  ~GroupGuard() {
    if (!ok && g) g->fail();
  }
};
}  // namespace

__global__ void rank_sum_kernel(const double* __restrict__ stage, int P, size_t count, double* __restrict__ out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    double acc = stage[i];
    for (int p = 1; p < P; ++p) acc += stage[(size_t)p * count + i];
    out[i] = acc;
  }
}

static void group_allgather(Ctx& c, const double* send, double* recv, size_t count) {
  LocalGroup& g = *c.group;
  GroupGuard guard{&g};
  g.post[c.rank] = send;
  TTB_CUDA(cudaEventRecord(g.ready[c.rank], c.stream));
  g.barrier();
  for (int q = 0; q < g.P; ++q) {
    if (count == 0) break;
    if (q != c.rank) TTB_CUDA(cudaStreamWaitEvent(c.stream, g.ready[q], 0));
    TTB_CUDA(cudaMemcpyAsync(recv + (size_t)q * count, g.post[q], count * sizeof(double), cudaMemcpyDefault, c.stream));
  }
  TTB_CUDA(cudaEventRecord(g.done[c.rank], c.stream));
  g.barrier();
  for (int q = 0; q < g.P; ++q)
    if (q != c.rank) TTB_CUDA(cudaStreamWaitEvent(c.stream, g.done[q], 0));
  guard.ok = true;
}

// ---- NCCL through dlopen -------------------------------------------------
struct NcclApi {
  void* h = nullptr;
  int (*getUniqueId)(void* id) = nullptr;
  int (*allGather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  int (*allReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*commDestroy)(void*) = nullptr;
  const char* (*getErrorString)(int) = nullptr;
  int (*send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*groupStart)() = nullptr;
  int (*groupEnd)() = nullptr;
};

struct UniqueId { char internal[128]; };
typedef int (*commInitRank_byval_t)(void** comm, int nranks, UniqueId id, int rank);

static NcclApi g_nccl;
static commInitRank_byval_t g_commInitRank = nullptr;
static std::mutex g_nccl_mu;

static void load_nccl() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.h) return;
  const char* env = getenv("TTB_NCCL_LIB");
  const char* cands[] = {env, "libnccl.so.2", "libnccl.so"};
  for (const char* c : cands) {
    if (!c) continue;
    g_nccl.h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
    if (g_nccl.h) break;
  }
  TTB_CHECK(g_nccl.h, TTB_ERR_NCCL, "could not dlopen libnccl.so.2 (set TTB_NCCL_LIB)");
  g_nccl.getUniqueId = (int (*)(void*))dlsym(g_nccl.h, "ncclGetUniqueId");
  g_commInitRank = (commInitRank_byval_t)dlsym(g_nccl.h, "ncclCommInitRank");
  g_nccl.allGather = (int (*)(const void*, void*, size_t, int, void*, cudaStream_t))dlsym(g_nccl.h, "ncclAllGather");
  g_nccl.allReduce = (int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t))dlsym(g_nccl.h, "ncclAllReduce");
  g_nccl.commDestroy = (int (*)(void*))dlsym(g_nccl.h, "ncclCommDestroy");
  g_nccl.getErrorString = (const char* (*)(int))dlsym(g_nccl.h, "ncclGetErrorString");
  g_nccl.send = (int (*)(const void*, size_t, int, int, void*, cudaStream_t))dlsym(g_nccl.h, "ncclSend");
  g_nccl.recv = (int (*)(void*, size_t, int, int, void*, cudaStream_t))dlsym(g_nccl.h, "ncclRecv");
  g_nccl.groupStart = (int (*)())dlsym(g_nccl.h, "ncclGroupStart");
  g_nccl.groupEnd = (int (*)())dlsym(g_nccl.h, "ncclGroupEnd");
  TTB_CHECK(g_nccl.getUniqueId && g_commInitRank && g_nccl.allGather && g_nccl.allReduce, TTB_ERR_NCCL,
            "libnccl is missing required symbols");
}

static void nccl_check(int rc, const char* what) {
  if (rc != 0) {
    std::string msg = std::string(what) + " failed";
    if (g_nccl.getErrorString) msg += std::string(": ") + g_nccl.getErrorString(rc);
    TTB_THROW(TTB_ERR_NCCL, msg);
  }
}

static constexpr int kNcclDouble = 8;  // ncclFloat64
static constexpr int kNcclSum = 0;     // ncclSum

double g_host_alloc_ms = 0.0;  // diagnostics (TTB_DEBUG_HOSTTIME)

void* Ctx::alloc(size_t bytes) {
  void* p = nullptr;
  if (bytes == 0) bytes = 256;
  if (!deferred.empty()) collect(false);
  const auto t0 = std::chrono::steady_clock::now();
  cudaError_t e = cudaMallocAsync(&p, bytes, stream);
  g_host_alloc_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (e != cudaSuccess) {
    cudaGetLastError();
    TTB_THROW(TTB_ERR_CAPACITY, std::string("device allocation of ") + std::to_string(bytes) +
                                    " bytes failed: " + cudaGetErrorString(e));
  }
  return p;
}

void Ctx::free(void* p) {
  if (p) TTB_CUDA(cudaFreeAsync(p, stream));
}

void Ctx::free_after(void* p, cudaStream_t used_on) {
  if (!p) return;
  cudaEvent_t e;
  TTB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  TTB_CUDA(cudaEventRecord(e, used_on));
  deferred.push_back({p, e});
}

void Ctx::collect(bool all) {
  size_t keep = 0;
  for (size_t i = 0; i < deferred.size(); ++i) {
    Deferred d = deferred[i];
    const cudaError_t q = all ? cudaSuccess : cudaEventQuery(d.ev);
    if (q == cudaSuccess) {
      TTB_CUDA(cudaStreamWaitEvent(stream, d.ev, 0));
      TTB_CUDA(cudaFreeAsync(d.p, stream));
      cudaEventDestroy(d.ev);
    } else {
      if (q != cudaErrorNotReady) TTB_CUDA(q);
      deferred[keep++] = d;
    }
  }
  deferred.resize(keep);
}

void Ctx::allgather(const double* send, double* recv, size_t count) {
  if (group) {
    g_comm[0] += 1;
    g_comm[1] += (long long)count * (nranks - 1);
    group_allgather(*this, send, recv, count);
    return;
  }
  TTB_CHECK(nccl_comm, TTB_ERR_CONTRACT, "multi-rank call without an initialised communicator");
  g_comm[0] += 1;
  g_comm[1] += (long long)count * (nranks - 1);
  nccl_check(g_nccl.allGather(send, recv, count, kNcclDouble, nccl_comm, stream), "ncclAllGather");
}

void Ctx::allreduce_sum(const double* send, double* recv, size_t count) {
  if (group) {
    TTB_CHECK(send != recv, TTB_ERR_CONTRACT, "allreduce: in-place reduction is not supported");
    g_comm[2] += 1;
    g_comm[3] += (long long)count;
    double* stage = (double*)alloc(std::max<size_t>(1, count * nranks) * sizeof(double));
    group_allgather(*this, send, stage, count);
    if (count > 0) {
      const int grid = (int)std::min<size_t>(1024, (count + 255) / 256);
      rank_sum_kernel<<<grid, 256, 0, stream>>>(stage, nranks, count, recv);
      TTB_LAUNCHED();
    }
    free(stage);
    return;
  }
  TTB_CHECK(nccl_comm, TTB_ERR_CONTRACT, "multi-rank call without an initialised communicator");
  g_comm[2] += 1;
  g_comm[3] += (long long)count;
  nccl_check(g_nccl.allReduce(send, recv, count, kNcclDouble, kNcclSum, nccl_comm, stream), "ncclAllReduce");
}

void Ctx::sendrecv(int npeers, const int* peers, const double* const* send, const int64_t* send_n,
                   double* const* recv, const int64_t* recv_n) {
  if (group) {
    // every rank takes part in the rendezvous (its peer list may be empty)
    LocalGroup& g = *group;
    GroupGuard guard{&g};
    const int P = g.P;
    for (int k = 0; k < npeers; ++k) {
      TTB_CHECK(peers[k] >= 0 && peers[k] < P && peers[k] != rank, TTB_ERR_CONTRACT, "sendrecv: bad peer");
      g.p2p[(size_t)rank * P + peers[k]] = {send[k], send_n[k]};
      g_comm[2] += (send_n[k] > 0) + (recv_n[k] > 0);
      g_comm[3] += send_n[k];
    }
    TTB_CUDA(cudaEventRecord(g.ready[rank], stream));
    g.barrier();
    for (int k = 0; k < npeers; ++k) {
      if (recv_n[k] <= 0) continue;
      const auto& src = g.p2p[(size_t)peers[k] * P + rank];
      TTB_CHECK(src.second == recv_n[k] && src.first, TTB_ERR_CONTRACT,
                "sendrecv: peer " + std::to_string(peers[k]) + " sends " + std::to_string(src.second) +
                    " values, " + std::to_string(recv_n[k]) + " expected");
      TTB_CUDA(cudaStreamWaitEvent(stream, g.ready[peers[k]], 0));
      TTB_CUDA(cudaMemcpyAsync(recv[k], src.first, (size_t)recv_n[k] * sizeof(double), cudaMemcpyDefault, stream));
    }
    TTB_CUDA(cudaEventRecord(g.done[rank], stream));
    g.barrier();
    for (int k = 0; k < npeers; ++k) {
      TTB_CUDA(cudaStreamWaitEvent(stream, g.done[peers[k]], 0));
      g.p2p[(size_t)rank * P + peers[k]] = {nullptr, 0};
    }
    guard.ok = true;
    return;
  }
  if (npeers == 0) return;
  TTB_CHECK(nccl_comm, TTB_ERR_CONTRACT, "multi-rank call without an initialised communicator");
  TTB_CHECK(g_nccl.send && g_nccl.recv && g_nccl.groupStart && g_nccl.groupEnd, TTB_ERR_NCCL,
            "libnccl lacks ncclSend/ncclRecv");
  nccl_check(g_nccl.groupStart(), "ncclGroupStart");
  for (int k = 0; k < npeers; ++k) {
    g_comm[2] += (send_n[k] > 0) + (recv_n[k] > 0);
    g_comm[3] += send_n[k];
    if (send_n[k] > 0) nccl_check(g_nccl.send(send[k], (size_t)send_n[k], kNcclDouble, peers[k], nccl_comm, stream),
                                  "ncclSend");
    if (recv_n[k] > 0) nccl_check(g_nccl.recv(recv[k], (size_t)recv_n[k], kNcclDouble, peers[k], nccl_comm, stream),
                                  "ncclRecv");
  }
  nccl_check(g_nccl.groupEnd(), "ncclGroupEnd");
}

void Ctx::sync() { TTB_CUDA(cudaStreamSynchronize(stream)); }

bool Ctx::stage_init() {
  if (stage_buf[0]) return true;
  for (int i = 0; i < kStageSlots; ++i) {
    if (cudaHostAlloc(&stage_buf[i], kStageBytes, cudaHostAllocDefault) != cudaSuccess ||
        cudaEventCreateWithFlags(&stage_ev[i], cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      for (int k = 0; k <= i; ++k) {
        if (stage_buf[k]) cudaFreeHost(stage_buf[k]);
        if (stage_ev[k]) cudaEventDestroy(stage_ev[k]);
        stage_buf[k] = nullptr;
        stage_ev[k] = nullptr;
      }
      return false;
    }
  }
  return true;
}

cudaStream_t Ctx::aux_stream() {
  if (!aux) TTB_CUDA(cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking));
  return aux;
}

cudaStream_t Ctx::side_stream() {
  if (!side) TTB_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
  return side;
}

__global__ void read_small_kernel(const unsigned char* __restrict__ src, volatile unsigned char* dst, int bytes,
                                  volatile unsigned* flag, unsigned seq) {
  for (int i = threadIdx.x; i < bytes; i += blockDim.x) dst[i] = src[i];
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    *flag = seq;
  }
}

// The host spins on the flag word instead of blocking in
// cudaStreamSynchronize: blocking waits can take milliseconds to wake in a
// virtualised host, and the rounding sweep reads a rank back after every
// truncated SVD.  cudaStreamQuery is polled now and then so launch or
// kernel errors surface instead of spinning forever.
void Ctx::read_small(const void* dev, size_t bytes, void* host) {
  TTB_CHECK(bytes <= 256, TTB_ERR_CONTRACT, "read_small: at most 256 bytes");
  if (!mapped_host) {
    TTB_CUDA(cudaHostAlloc(&mapped_host, 512, cudaHostAllocMapped));
    TTB_CUDA(cudaHostGetDevicePointer(&mapped_dev, mapped_host, 0));
    memset(mapped_host, 0, 512);
  }
  volatile unsigned* hflag = reinterpret_cast<volatile unsigned*>((char*)mapped_host + 256);
  unsigned* dflag = reinterpret_cast<unsigned*>((char*)mapped_dev + 256);
  const unsigned seq = ++read_seq;
  read_small_kernel<<<1, 32, 0, stream>>>((const unsigned char*)dev, (volatile unsigned char*)mapped_dev, (int)bytes,
                                          dflag, seq);
  TTB_LAUNCHED();
  for (long spin = 0; *hflag != seq; ++spin) {
    if ((spin & 0xFFFF) == 0xFFFF) {
      const cudaError_t q = cudaStreamQuery(stream);
      if (q == cudaSuccess) break;  // completed (flag visibility lagging)
      if (q != cudaErrorNotReady) TTB_CUDA(q);
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  memcpy(host, mapped_host, bytes);
}

int* Ctx::flag() {
  if (!dflag) {
    TTB_CUDA(cudaMalloc(&dflag, 256));
    TTB_CUDA(cudaMemsetAsync(dflag, 0, 256, stream));
  }
  return dflag;
}

void Ctx::flag_reset() { TTB_CUDA(cudaMemsetAsync(flag(), 0, sizeof(int), stream)); }

bool Ctx::flag_read() {
  int h = 0;
  read_small(flag(), sizeof(int), &h);
  return h != 0;
}

cudaStream_t Ctx::copy_stream() {
  if (!copy) TTB_CUDA(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking));
  return copy;
}

}  // namespace ttb

using namespace ttb;

extern "C" {

const char* ttb_last_error(void) { return g_last_error.c_str(); }

int ttb_abi_version(void) { return TTB_ABI_VERSION; }

long long ttb_launch_counter(void) { return g_launches.load(); }

int ttb_comm_stats(long long* out4) {
  TTB_TRY_BEGIN
  TTB_CHECK(out4, TTB_ERR_CONTRACT, "null output");
  for (int k = 0; k < 4; ++k) out4[k] = g_comm[k].load();
  TTB_TRY_END
}

int ttb_ctx_create(int device, void* stream, ttb_ctx** out) {
  TTB_TRY_BEGIN
  TTB_CHECK(out, TTB_ERR_CONTRACT, "null output pointer");
  TTB_CUDA(cudaSetDevice(device));
  ttb_ctx* c = new ttb_ctx();
  c->c.device = device;
  c->c.stream = (cudaStream_t)stream;
  TTB_CUDA(cudaDeviceGetAttribute(&c->c.num_sms, cudaDevAttrMultiProcessorCount, device));
  int cc_major = 0, cc_minor = 0;
  TTB_CUDA(cudaDeviceGetAttribute(&cc_major, cudaDevAttrComputeCapabilityMajor, device));
  TTB_CUDA(cudaDeviceGetAttribute(&cc_minor, cudaDevAttrComputeCapabilityMinor, device));
  if (cc_major != 10 || cc_minor != 0) {
    delete c;
    TTB_THROW(TTB_ERR_CAPABILITY, "this build targets sm_100a (B200); device is sm_" +
                                      std::to_string(cc_major) + std::to_string(cc_minor));
  }
  // keep freed workspace mapped in the stream-ordered pool: the default
  // release threshold (0) unmaps it at every stream sync, which costs more
  // than the kernels (GB-sized TSQR factors are re-allocated every call)
  cudaMemPool_t pool;
  TTB_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t thr = UINT64_MAX;
  TTB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  *out = c;
  TTB_TRY_END
}

int ttb_ctx_destroy(ttb_ctx* ctx) {
  TTB_TRY_BEGIN
  if (ctx) {
    if (ctx->c.nccl_comm && g_nccl.commDestroy) g_nccl.commDestroy(ctx->c.nccl_comm);
    if (ctx->c.side) cudaStreamDestroy(ctx->c.side);
    if (ctx->c.aux) cudaStreamDestroy(ctx->c.aux);
    if (ctx->c.copy) cudaStreamDestroy(ctx->c.copy);
    if (ctx->c.mapped_host) cudaFreeHost(ctx->c.mapped_host);
    for (int i = 0; i < Ctx::kStageSlots; ++i) {
      if (ctx->c.stage_buf[i]) cudaFreeHost(ctx->c.stage_buf[i]);
      if (ctx->c.stage_ev[i]) cudaEventDestroy(ctx->c.stage_ev[i]);
    }
    if (ctx->c.dflag) cudaFree(ctx->c.dflag);
    delete ctx;
  }
  TTB_TRY_END
}

int ttb_ctx_set_stream(ttb_ctx* ctx, void* stream) {
  TTB_TRY_BEGIN
  ctx->c.stream = (cudaStream_t)stream;
  TTB_TRY_END
}

int ttb_ctx_trim(ttb_ctx* ctx) {
  TTB_TRY_BEGIN
  TTB_CHECK(ctx, TTB_ERR_CONTRACT, "null context");
  TTB_CUDA(cudaSetDevice(ctx->c.device));
  ctx->c.collect(true);
  TTB_CUDA(cudaStreamSynchronize(ctx->c.stream));
  if (ctx->c.side) TTB_CUDA(cudaStreamSynchronize(ctx->c.side));
  if (ctx->c.aux) TTB_CUDA(cudaStreamSynchronize(ctx->c.aux));
  cudaMemPool_t pool;
  TTB_CUDA(cudaDeviceGetDefaultMemPool(&pool, ctx->c.device));
  TTB_CUDA(cudaMemPoolTrimTo(pool, 0));
  TTB_TRY_END
}

int ttb_group_create(int nranks, ttb_group** out) {
  TTB_TRY_BEGIN
  TTB_CHECK(out, TTB_ERR_CONTRACT, "null output pointer");
  TTB_CHECK(nranks >= 1 && nranks <= 1024, TTB_ERR_CONTRACT, "group size must be in [1, 1024]");
  *out = reinterpret_cast<ttb_group*>(new LocalGroup(nranks));
  TTB_TRY_END
}

int ttb_group_destroy(ttb_group* grp) {
  TTB_TRY_BEGIN
  if (grp) {
    LocalGroup* g = reinterpret_cast<LocalGroup*>(grp);
    for (auto e : g->ready)
      if (e) cudaEventDestroy(e);
    for (auto e : g->done)
      if (e) cudaEventDestroy(e);
    delete g;
  }
  TTB_TRY_END
}

int ttb_group_abort(ttb_group* grp) {
  TTB_TRY_BEGIN
  if (grp) reinterpret_cast<LocalGroup*>(grp)->fail();
  TTB_TRY_END
}

int ttb_ctx_join_group(ttb_ctx* ctx, ttb_group* grp, int rank) {
  TTB_TRY_BEGIN
  TTB_CHECK(ctx && grp, TTB_ERR_CONTRACT, "null context or group");
  LocalGroup* g = reinterpret_cast<LocalGroup*>(grp);
  TTB_CHECK(rank >= 0 && rank < g->P, TTB_ERR_CONTRACT, "bad rank");
  TTB_CHECK(!ctx->c.nccl_comm && !ctx->c.group, TTB_ERR_CONTRACT, "context already has a communicator");
  TTB_CUDA(cudaSetDevice(ctx->c.device));
  {
    std::lock_guard<std::mutex> lk(g->mu);
    TTB_CHECK(!g->ready[rank], TTB_ERR_CONTRACT, "rank " + std::to_string(rank) + " already joined");
    TTB_CUDA(cudaEventCreateWithFlags(&g->ready[rank], cudaEventDisableTiming));
    TTB_CUDA(cudaEventCreateWithFlags(&g->done[rank], cudaEventDisableTiming));
  }
  ctx->c.group = g;
  ctx->c.nranks = g->P;
  ctx->c.rank = rank;
  TTB_TRY_END
}

int ttb_comm_unique_id(void* out128) {
  TTB_TRY_BEGIN
  load_nccl();
  nccl_check(g_nccl.getUniqueId(out128), "ncclGetUniqueId");
  TTB_TRY_END
}

int ttb_ctx_init_comm(ttb_ctx* ctx, int nranks, int rank, const void* id128) {
  TTB_TRY_BEGIN
  TTB_CHECK(nranks >= 1 && rank >= 0 && rank < nranks, TTB_ERR_CONTRACT, "bad rank/size");
  ctx->c.nranks = nranks;
  ctx->c.rank = rank;
  if (nranks > 1) {
    load_nccl();
    TTB_CUDA(cudaSetDevice(ctx->c.device));
    UniqueId id;
    memcpy(id.internal, id128, 128);
    void* comm = nullptr;
    nccl_check(g_commInitRank(&comm, nranks, id, rank), "ncclCommInitRank");
    ctx->c.nccl_comm = comm;
  }
  TTB_TRY_END
}

}  // extern "C"
