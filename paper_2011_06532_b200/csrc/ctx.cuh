// Per-device execution context: stream, SM count, stream-ordered workspace
// allocation, and the (optional) NCCL communicator used by the multi-GPU
// paths.  NCCL is resolved at run time with dlopen so the library does not
// pin a second libnccl next to the one torch loads.
#pragma once

#include <vector>

#include "common.cuh"
#include "tsqr.cuh"

namespace ttb {

struct NcclApi;     // defined in ctx.cu
struct LocalGroup;  // defined in ctx.cu: in-process emulated collectives
extern double g_host_alloc_ms;  // diagnostics: host time in cudaMallocAsync

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  int nranks = 1;
  int rank = 0;
  void* nccl_comm = nullptr;
  // in-process group (ttb_group_create / ttb_ctx_join_group): P contexts in
  // one process, one host thread each, exchanging device buffers by
  // stream-ordered copies with host rendezvous -- the same call sites as
  // NCCL, for running the multi-rank path on one device
  LocalGroup* group = nullptr;
  cudaEvent_t ev = nullptr;
  cudaStream_t side = nullptr;  // second stream for off-critical-path work (lazily created)

  cudaStream_t side_stream();
  cudaStream_t aux = nullptr;   // third stream: per-tile T factors of a TSQR, formed beside the tree (lazily created)
  cudaStream_t aux_stream();
  cudaStream_t copy = nullptr;  // host<->device transfers of the host API (lazily created)
  cudaStream_t copy_stream();
  // page-locked staging ring of the host API (pageable user buffers are
  // copied through it by a worker thread; lazily allocated, kept)
  static constexpr int kStageSlots = 4;
  static constexpr size_t kStageBytes = size_t(32) << 20;
  void* stage_buf[kStageSlots] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t stage_ev[kStageSlots] = {nullptr, nullptr, nullptr, nullptr};
  bool stage_init();  // false: no page-locked memory to be had (callers fall back to plain pageable copies)
  // small device -> host reads (ranks, norms) go through mapped pinned
  // memory written by a kernel: they never queue behind bulk DMA copies
  // (e.g. the host API's output downloads on the copy engine)
  void* mapped_host = nullptr;
  void* mapped_dev = nullptr;
  unsigned read_seq = 0;
  void read_small(const void* dev, size_t bytes, void* host);
  // sticky device flag: set by kernels that meet non-finite data (TSQR R
  // factors); reset / read once per API call
  int* dflag = nullptr;
  int* flag();
  void flag_reset();
  bool flag_read();
  void* alloc(size_t bytes);
  void free(void* p);
  // free memory last used on another stream: the block goes back to the
  // pool on THIS stream once that use has completed (checked at later
  // allocations), so the stream-ordered pool never has to pick between
  // cross-stream reuse and growth
  void free_after(void* p, cudaStream_t used_on);
  void collect(bool all);
  struct Deferred {
    void* p;
    cudaEvent_t ev;
  };
  std::vector<Deferred> deferred;
  // collectives on this->stream (nranks > 1 only)
  void allgather(const double* send, double* recv, size_t count);
  void allreduce_sum(const double* send, double* recv, size_t count);
  // grouped point-to-point exchange with a set of peers (zero counts skip)
  void sendrecv(int npeers, const int* peers, const double* const* send, const int64_t* send_n,
                double* const* recv, const int64_t* recv_n);
  void sync();
};

constexpr int kMaxWideBlk = 64;  // column blocks of the general TSQR path (b <= 4096)

// host-side TSQR factor object (see tsqr.cu)
struct Tsqr {
  int b = 0, cls = 0;
  Panel panel;
  LeafPlan plan;
  bool r_only = false;  // set by the caller before tsqr_factor: only R is wanted (no Y / T written, no apply)
  int wl = 0;    // 1: team-pipelined leaf (wleaf.cu): wplan, Y in 64-row tiles, T holds U = T^{-1}
  WPlan wplan;
  int ldy = 0, ldy_tree = 0, ftree = 0;
  double *Y = nullptr, *T = nullptr, *Rleaf = nullptr;
  int nloc = 0, nglob = 0;
  double *locY[kMaxLevels], *locT[kMaxLevels], *locR[kMaxLevels];
  double *gloY[kMaxLevels], *gloT[kMaxLevels], *gloR[kMaxLevels];
  double* Rstack = nullptr;
  const double* Rlocal = nullptr;
  const double* Rraw = nullptr;
  double* D = nullptr;  // sign fix (b)
  double* R = nullptr;  // final sign-fixed R (b x b, col-major), replicated
  // leaf T factors formed by tile_T_kernel on the aux stream: consumers of T
  // (the chain apply) and the release of mem wait on this event
  cudaEvent_t t_ready = nullptr;
  unsigned* prog = nullptr;  // tree progress counters (one per node)
  double* Rrow = nullptr;    // tree row streams (one b x ldr block per node)
  int ldr = 0;
  void* mem = nullptr;
  // general path (wide.cu: more than 64 columns, or slices taller than a leaf
  // tile): explicit orthonormal column blocks wQ (wm x b, col-major, rows in
  // view memory order), block p = columns [wc0[p], wc0[p+1])
  int wide = 0, wnblk = 0;
  int64_t wm = 0;
  int wc0[kMaxWideBlk + 1];
  double* wQ = nullptr;
};

int tsqr_class(int b);
// blocked (panel warp + fp64 MMA) leaf for 32 < b <= 64 (leaf2.cu)
void launch_leaf2(Ctx& ctx, const Panel& panel, const LeafPlan& plan, double* Y, double* T, double* Rleaf);
// row-distributed blocked leaf for 32 < b <= 64 (leaf3.cu)
void launch_leaf3(Ctx& ctx, const Panel& panel, const LeafPlan& plan, double* Y, double* T, double* Rleaf);
// team-pipelined leaf and its chain + product apply (wleaf.cu)
int wleaf_teams(int b);
size_t wleaf_y_doubles(const WPlan& p);
size_t wleaf_u_doubles(const WPlan& p);
void launch_wleaf(Ctx& ctx, const Panel& panel, const WPlan& plan, double* Y, double* U, double* Rleaf);
void wleaf_apply_tail(Ctx& ctx, const WPlan& plan, const double* Y, const double* U, const double* zin,
                      const double* D, int k, const Panel& out, double* ubuf, double* z0buf);
void tsqr_factor(Ctx& ctx, const Panel& panel, Tsqr& f);
// out (view with k columns, same slicing as the factored panel) = Q [D z; 0]
void tsqr_apply(Ctx& ctx, const Tsqr& f, const double* z, int k, const Panel& out);
void tsqr_release(Ctx& ctx, Tsqr& f);

}  // namespace ttb

struct ttb_ctx {
  ttb::Ctx c;
};
