// TSQR kernels (leaf chain, tree nodes, apply) and the host-side factor object.
// See tsqr.cuh for the decomposition.  Reference: ttpar tsqr.py:103-327.
#include <string>
#include <vector>

#include "tsqr.cuh"
#include "ctx.cuh"
#include "prof.cuh"
#include "dmma.cuh"
#include "wide.cuh"

namespace ttb {

// bulk-copy (TMA engine) helpers
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// ------------------------------------------------------------------------
// leaf kernel: one CTA = one chain of tiles over a contiguous slice run
// ------------------------------------------------------------------------
template <class C>
__global__ void __launch_bounds__(C::NT, C::MINB)
tsqr_leaf_kernel(Panel P, LeafPlan plan, double* __restrict__ Yg, double* __restrict__ Tg,
                 double* __restrict__ Rleaf, int defer_T, int r_only) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TileSmem<C>& sm = *reinterpret_cast<TileSmem<C>*>(smem_raw);
  const int g = blockIdx.x;
  const int b = plan.b, rs = plan.rs, ni = plan.ni;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lc = lane / C::LR, lr = lane % C::LR;
  const int64_t n_g = plan.count(g), s0 = plan.start(g);
  const int ntiles = plan.tiles_of(n_g);
  const int64_t tb = plan.tile_base(g);

  double A[C::RPL][C::CPL];
  init_ring<C>(sm);
  if (ntiles == 0) {  // no rows (an idle rank): R = 0
    for (int idx = threadIdx.x; idx < C::BMAX * C::BMAX; idx += C::NT) sm.Rs[idx] = 0.0;
    __syncthreads();
  }
  // load tile t (zero padded): one row offset per register row, all loads of
  // the tile issued back to back (implicit Hadamard panels form elements on load)
  auto load_tile = [&](int t) {
    const int64_t ia = s0 + (int64_t)t * ni;
    const int nsl = (int)min64(ni, n_g - (int64_t)t * ni);
    const int rows = nsl * rs;
    if (P.kron.x) {
#pragma unroll
      for (int s = 0; s < C::RPL; ++s) {
        const int r = C::row(s, lr);
        int si, w;
        tile_row(P.trans, r, nsl, rs, si, w);
#pragma unroll
        for (int u = 0; u < C::CPL; ++u) {
          const int k = col_of<C>(u, warp, lc);
          A[s][u] = (r < rows && k < b) ? P.load(w, ia + si, k) : 0.0;
        }
      }
    } else {
      // rows come in pairs (r, r + 1) every 2 LR rows: (slice, row-in-slice)
      // advances by a constant step, no division per row
      const int64_t cst = P.trans ? 1 : P.rl * P.I;
      const int per = P.trans ? nsl : rs;  // the fast index wraps at `per`
      const int step = 2 * C::LR, dq = step / per, dr = step - dq * per;
      int q0 = (2 * lr) / per, r0 = 2 * lr - q0 * per;  // fast index r0 < per, slow index q0
#pragma unroll
      for (int s = 0; s < C::RPL; s += 2) {
        const int r = C::row(s, lr);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          int fq = q0, fr = r0 + h;
          if (fr == per) {
            fr = 0;
            ++fq;
          }
          // V: slice = fq, row-in-slice = fr; H^T: row-in-slice (w) = fq, slice = fr
          const int si = P.trans ? fr : fq, w = P.trans ? fq : fr;
          const double* rp = P.base + P.addr(w, ia + si, 0);
          const bool rok = r + h < rows;
#pragma unroll
          for (int u = 0; u < C::CPL; ++u) {
            const int k = col_of<C>(u, warp, lc);
            A[s + h][u] = (rok && k < b) ? __ldg(rp + cst * k) : 0.0;
          }
        }
        r0 += dr;
        q0 += dq;
        if (r0 >= per) {
          r0 -= per;
          ++q0;
        }
      }
    }
  };
  if (ntiles > 0) load_tile(0);
  for (int t = 0; t < ntiles; ++t) {
    TTB_TILE_CLK(t, 0);
    const int64_t ia = s0 + (int64_t)t * ni;
    // pull the next-but-one tile's rows into L2 (the next tile's loads are
    // issued at the end of this one): its load then waits on L2, not HBM
    // (the runs of a tile are contiguous: V views one run of rl*nsl doubles
    // per column, H^T views one per row-in-slice)
    if (t + 2 < ntiles && P.kron.x == nullptr) {
      const int64_t ia2 = ia + 2 * ni;
      const int nsl2 = (int)min64(ni, n_g - (int64_t)(t + 2) * ni);
      const int64_t runlen = P.rl * (int64_t)nsl2;  // doubles per run
      const int nruns = P.trans ? rs : b;
      const int lines = (int)((runlen * 8 + 127) / 128) + 1;
      for (int idx = threadIdx.x; idx < nruns * lines; idx += C::NT) {
        const int q = idx / lines, ln = idx - q * lines;
        const double* p0 = P.base + P.rl * (ia2 + P.I * (int64_t)q);
        const char* pl = reinterpret_cast<const char*>(p0) + (int64_t)ln * 128;
        if (pl < reinterpret_cast<const char*>(p0 + runlen))
          asm volatile("prefetch.global.L2 [%0];\n" ::"l"(pl));
      }
    }
    zero_G<C>(sm);
    __syncthreads();
    TTB_TILE_CLK(t, 1);
    const bool head = (t == 0);
    tile_qr<C>(A, b, head, sm, t * b);
    TTB_TILE_CLK(t, 2);
    const int64_t tile = tb + t;
    if (!r_only) store_Y_units<C>(A, b, head, Yg + tile * y_tile_stride(C::MC, b));  // R-only: no Q to apply later
    if (head) extract_R<C>(A, b, sm);
    // the next tile's loads are in flight while T is formed
    if (t + 1 < ntiles) load_tile(t + 1);
    if (r_only) {
      TTB_TILE_CLK(t, 5);
    } else if (defer_T) {
      // T is formed outside the chain (tile_T_kernel, beside the tree): hand
      // over striu(V^T V) with tau on the diagonal
      TTB_TILE_CLK(t, 5);
      double* Tt = Tg + tile * (((int64_t)b * b + 1) & ~1LL);
      for (int idx = threadIdx.x; idx < b * b; idx += C::NT) {
        const int k = idx % b, j = idx / b;
        Tt[idx] = k < j ? sm.Gs[k + C::BMAX * j] : (k == j ? sm.taus[j] : 0.0);
      }
    } else {
      build_T<C>(sm, b);
      TTB_TILE_CLK(t, 5);
      store_T<C>(sm, b, Tg + tile * (((int64_t)b * b + 1) & ~1LL));
    }
    __syncthreads();
    TTB_TILE_CLK(t, 3);
  }
  for (int idx = threadIdx.x; idx < b * b; idx += C::NT) {
    const int r = idx % b, k = idx / b;
    Rleaf[(int64_t)g * b * b + idx] = sm.Rs[r + C::BMAX * k];
  }
}

// ------------------------------------------------------------------------
// Per-tile T = (diag(1/tau) + striu(V^T V))^{-1} outside the leaf chain: the
// leaf hands over striu(V^T V) with tau on the diagonal (defer_T); one CTA
// per tile inverts it in place.  Launched on the aux stream, it runs beside
// the tree (a latency chain on a third of the SMs) instead of inside every
// chain's critical path.
// ------------------------------------------------------------------------
struct TCfg256 {
  static constexpr int NT = 256, BMAX = 64;
  __device__ __forceinline__ static void sync() { __syncthreads(); }
};
struct TSmem {
  double Gs[64 * 64];
  double Xs[64 * 64 / 2];
  double taus[64];
};
__global__ void __launch_bounds__(256) tile_T_kernel(double* __restrict__ Tg, int b, int64_t tsz) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TSmem& sm = *reinterpret_cast<TSmem*>(smem_raw);
  double* Tt = Tg + (int64_t)blockIdx.x * tsz;
  for (int idx = threadIdx.x; idx < 64 * 64; idx += 256) {
    const int k = idx & 63, j = idx >> 6;
    sm.Gs[idx] = (k < j && j < b) ? Tt[k + b * j] : 0.0;
  }
  if (threadIdx.x < b) sm.taus[threadIdx.x] = Tt[threadIdx.x + b * threadIdx.x];
  __syncthreads();
  build_T<TCfg256>(sm, b);
  for (int idx = threadIdx.x; idx < b * b; idx += 256) {
    const int k = idx % b, j = idx / b;
    Tt[idx] = sm.Gs[k + 64 * j];
  }
}

// ------------------------------------------------------------------------
// tree kernel: every level of the reduction tree in ONE launch.  Node q of
// level L factors the stacked triangles of its children.  Level-0 inputs
// (the leaf triangles) are complete at launch; a node of level L >= 1 reads
// its children's R rows as they become final: a child publishes row j of R
// once it applied reflector j, and counts finished chunks of kTreeChunk rows
// in a per-node progress counter.  The parent's column j only needs rows
// <= j of every child (the support of reflector j of a stacked-triangle QR
// is block 0's row j and rows 0..j of the other blocks), so levels run as a
// wavefront a few columns apart instead of one after another.  All nodes
// are co-resident (one CTA per SM, nodes < SMs); children have lower block
// indices than their parents and never wait on them.
// ------------------------------------------------------------------------
struct TreePlan {
  int nlev, b, f, ldy;  // ldy: rows of a node's stored V (= the stack: f * b)
  int first[kMaxLevels + 1];  // global node index of each level's first node
  int n_in[kMaxLevels];       // inputs (children) of each level
  const double* Rin[kMaxLevels];
  double* Y[kMaxLevels];
  double* T[kMaxLevels];
  double* R[kMaxLevels];
  double* Rrow;               // per node: R rows as they finalise, row-major, ld ldr
  int ldr;
  unsigned* prog;             // per node: NW x finished chunks (zeroed per launch)
  unsigned* ticket;           // node-id dispenser (zeroed per launch)
};

constexpr int kMaxChunks = 64;

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// polling load without acquire ordering (later memory operations of the
// warp do not wait for it); a fence.acq_rel follows a successful poll
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p));
  return v;
}

#if defined(TTB_TCLK2) && !defined(TTB_TCLK)
#define TTB_TCLK
#define TTB_TCLK_NOCHUNK
#endif
#ifdef TTB_TCLK
static __device__ unsigned long long g_tclk[160 * 64];
extern "C" int ttb_dbg_tclk(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_tclk, sizeof(unsigned long long) * 160 * 64) == cudaSuccess ? 0 : 5;
}
#define TTB_TSTAMP(nd, idx)                                    \
  do {                                                         \
    unsigned long long tnow;                                   \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));   \
    g_tclk[(nd) * 64 + (idx)] = tnow;                          \
  } while (0)
#else
#define TTB_TSTAMP(nd, idx) \
  do {                      \
  } while (0)
#endif

// Column-loop hooks of a tree node.
//  inputs: complete (level 0: loaded whole at the start) or streamed: a
//    data-mover warp (its own warpgroup, registers handed to the compute
//    warps with setmaxnreg) polls the children's progress counters and, as
//    soon as a chunk of rows is final in every child, lane c bulk-copies
//    child c's rows into the shared staging area (one mbarrier per chunk);
//    the compute warps wait on that barrier only when they reach the chunk.
//  outputs: after step j every warp writes row j of R (its columns) into
//    the node's row-major stream and, per finished chunk, bumps the node's
//    progress counter.
template <class C>
struct TreeHooks {
  const double* Rin;        // complete inputs: children's triangles (col-major)
  const double* Rrow_in;    // streamed inputs: children's row streams (ld ldr)
  const unsigned* prog_in;  // streamed: children's counters (null: complete)
  double* Rrow_out;         // this node's row stream (null: root)
  unsigned* prog_out;
  double* stage;            // shared: MC x ldr
  unsigned long long* sbar; // shared: one per chunk
  int c0, cnt, b, ldr, nchunks;
  int node;  // debug stamps only
  double* Rs;  // shared: the node is factored as a body tile [R_child0; children 1..]: child 0 -> Rs
  // no mover warp (XW == 0): warp 0 issues the children's chunks itself -- a
  // relaxed poll of the children's counters is loaded at the start of each
  // column step and tested at its end (off the step's critical path); a
  // chunk that is still missing when a step needs it is polled for blocking
  int issued = 0;
  unsigned pv = 0;

  __device__ __forceinline__ unsigned need(int ci) const { return (unsigned)C::NW * (unsigned)(ci + 1); }
  __device__ __forceinline__ void issue(int ci) {
    const int lane = threadIdx.x & 31;
    const int j0 = ci * kTreeChunk, rows = min(kTreeChunk, b - j0);
    const unsigned bytes = (unsigned)(rows * ldr * 8);
    asm volatile("fence.proxy.async.global;\n" ::: "memory");
    if (lane == 0) mbar_expect_tx(&sbar[ci], bytes * (unsigned)cnt);
    __syncwarp();
    for (int c = lane; c < cnt; c += 32)
      bulk_g2s(stage + ((int64_t)c * b + j0) * ldr, Rrow_in + ((int64_t)(c0 + c) * b + j0) * ldr, bytes, &sbar[ci]);
  }
  // the data-mover warp (C::XW) issues every chunk as soon as it is final
  // in every child; the compute warps never poll or fence for inputs
  __device__ __forceinline__ void mover() {
    if (!prog_in) return;
    const int lane = threadIdx.x & 31;
    for (int ci = 0; ci < nchunks; ++ci) {
      for (int c = lane; c < cnt; c += 32)
        while (ld_acquire(prog_in + c) < need(ci)) {
        }
      __syncwarp();
      issue(ci);
    }
  }
  __device__ __forceinline__ void pre(int) {
    if (C::XW != 0 || !prog_in || issued >= nchunks || (threadIdx.x >> 5) != 0) return;
    const int lane = threadIdx.x & 31;
    pv = lane < cnt ? ld_relaxed(prog_in + lane) : 0xffffffffu;
  }
  // warp 0: issue chunk `issued` if every child has published it (pv loaded in pre)
  __device__ __forceinline__ void try_issue() {
    if (C::XW != 0 || !prog_in || issued >= nchunks || (threadIdx.x >> 5) != 0) return;
    if (__all_sync(0xffffffffu, pv >= need(issued))) {
      asm volatile("fence.acq_rel.gpu;\n" ::: "memory");  // acquire the children's rows
      issue(issued++);
    }
  }
  template <class T>
  __device__ __forceinline__ void feed(T& A, int j0) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int lc = lane / C::LR, lr = lane % C::LR;
    // child 0 goes to Rs, written only by the warp that owns column j0: it
    // publishes column j0 (and reads its pivot) next, and every other warp
    // reads Rs rows >= j0 only after that publication's full barrier
    if (!prog_in) {  // complete inputs: everything at the start (every compute warp is here)
      if (j0 > 0) return;
      for (int idx = threadIdx.x; idx < b * b; idx += C::NT) {
        const int r = idx % b, k = idx / b;
        Rs[r + C::BMAX * k] = r <= k ? Rin[(int64_t)c0 * b * b + idx] : 0.0;
      }
#pragma unroll
      for (int s = 0; s < C::RPL; ++s) {
        const int r = C::row(s, lr);
        const int ch = r / b + 1, i = r % b;
#pragma unroll
        for (int t = 0; t < C::CPL; ++t) {
          const int k = col_of<C>(t, warp, lc);
          A[s][t] = (ch < cnt && k < b) ? Rin[(int64_t)(c0 + ch) * b * b + i + (int64_t)b * k] : 0.0;
        }
      }
      C::sync();
      return;
    }
    const int ci = j0 / kTreeChunk;
    if (C::XW == 0 && warp == 0) {  // no mover warp: warp 0 issues what is still missing, blocking
      while (issued <= ci) {
        for (int c = lane; c < cnt; c += 32)
          while (ld_acquire(prog_in + c) < need(issued)) {
          }
        __syncwarp();
        issue(issued++);
      }
    }
    mbar_wait(&sbar[ci], 0);
    const int j1 = min(j0 + kTreeChunk, b);
    if (warp == C::owner_warp(j0)) {
      for (int idx = lane; idx < (j1 - j0) * b; idx += 32) {
        const int i = j0 + idx / b, k = idx % b;
        Rs[i + C::BMAX * k] = k >= i ? stage[(int64_t)i * ldr + k] : 0.0;
      }
    }
#pragma unroll
    for (int s = 0; s < C::RPL; ++s) {
      const int r = C::row(s, lr);
      const int ch = r / b + 1, i = r % b;
      if (ch >= cnt || i < j0 || i >= j1) continue;
#pragma unroll
      for (int t = 0; t < C::CPL; ++t) {
        const int k = col_of<C>(t, warp, lc);
        if (k < b) A[s][t] = k >= i ? stage[(int64_t)(ch * b + i) * ldr + k] : 0.0;
      }
    }
  }
  template <class T>
  __device__ __forceinline__ void post(T& A, int j) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    try_issue();
#ifdef TTB_TCLK2
    if (lane == 0 && warp == 0) TTB_TSTAMP(node, j);
#endif
    if (!prog_out) return;
    const int lc = lane / C::LR, lr = lane % C::LR;
    // row j of R is final in Rs once this warp applied reflector j: the
    // lr == 0 lane of each column group wrote its columns' entries itself
    // (update_slot), the diagonal came from the owner group's publish
    if (lr == 0) {
#pragma unroll
      for (int t = 0; t < C::CPL; ++t) {
        const int k = col_of<C>(t, warp, lc);
        if (k >= b) continue;
        Rrow_out[(int64_t)j * ldr + k] = k >= j ? Rs[j + C::BMAX * k] : 0.0;
      }
    }
    if ((j + 1) % kTreeChunk == 0 || j + 1 == b) {
      // release this warp's rows: the warp barrier orders every lane's row
      // stores before lane 0's release-increment (cumulative), which the
      // parent's acquire-poll pairs with -- no GPU-scope fence per thread
      __syncwarp();
      if (lane == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(prog_out) : "memory");
#if defined(TTB_TCLK) && !defined(TTB_TCLK_NOCHUNK)
      if (lane == 0 && warp == 0) TTB_TSTAMP(node, j / kTreeChunk);
#endif
    }
  }
};

template <class C>
__global__ void __launch_bounds__(C::NTT, 1) tsqr_tree_kernel(TreePlan tp) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  TileSmem<C>& sm = *reinterpret_cast<TileSmem<C>*>(smem_raw);
  unsigned long long* sbar = reinterpret_cast<unsigned long long*>(smem_raw + ((sizeof(TileSmem<C>) + 127) & ~size_t(127)));
  double* stage = reinterpret_cast<double*>(sbar + kMaxChunks);
  // node ids come from an atomic ticket in CTA start order, not from
  // blockIdx: a node only ever waits on children with lower ids, i.e. on
  // CTAs that already started (and are resident), whatever order the
  // hardware dispatches the grid in and whatever else shares the SMs
  __shared__ int node_s;
  if (threadIdx.x == 0) node_s = (int)atomicAdd(tp.ticket, 1u);
  __syncthreads();
  const int node = node_s;
  int L = 0;
  while (L + 1 < tp.nlev && node >= tp.first[L + 1]) ++L;
  const int q = node - tp.first[L];
  const int b = tp.b, f = tp.f;
  const int c0 = q * f, cnt = min(f, tp.n_in[L] - c0);
  const int nchunks = (b + kTreeChunk - 1) / kTreeChunk;
  double A[C::RPL][C::CPL];
#pragma unroll
  for (int s = 0; s < C::RPL; ++s)
#pragma unroll
    for (int t = 0; t < C::CPL; ++t) A[s][t] = 0.0;
  zero_G<C>(sm);
  init_ring<C>(sm);
  if (threadIdx.x < nchunks) mbar_init(&sbar[threadIdx.x], 1);
  if (threadIdx.x == 0) asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
#ifdef TTB_TCLK
  if (threadIdx.x == 0) TTB_TSTAMP(node, 63);
#endif
  const bool has_parent = L + 1 < tp.nlev;
  TreeHooks<C> h;
  h.Rin = tp.Rin[L];
  h.Rrow_in = L > 0 ? tp.Rrow + (int64_t)tp.first[L - 1] * b * tp.ldr : nullptr;
  h.prog_in = L > 0 ? tp.prog + tp.first[L - 1] + c0 : nullptr;
  h.Rrow_out = has_parent ? tp.Rrow + (int64_t)node * b * tp.ldr : nullptr;
  h.prog_out = has_parent ? tp.prog + node : nullptr;
  h.stage = stage;
  h.sbar = sbar;
  h.c0 = c0;
  h.cnt = cnt;
  h.b = b;
  h.ldr = tp.ldr;
  h.nchunks = nchunks;
  h.node = node;
  h.Rs = sm.Rs;
  // warp specialisation: the extra warp(s) move the children's rows; the
  // compute warps hold the register tile
  if constexpr (C::XW == 4) {  // a mover warpgroup hands its registers to the compute warps
    if (threadIdx.x >= C::NT) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
      if (threadIdx.x < C::NT + 32) h.mover();
      return;
    }
    asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
  } else {
    if (threadIdx.x >= C::NT) {
      if (threadIdx.x < C::NT + 32) h.mover();
      return;
    }
  }
  // the stacked triangles as a body tile: [R_child0; R_child1; ...] with
  // R_child0 in Rs -- reflector j has the support a plain QR of the stack
  // gives it (row j of child 0, rows <= j of the others), so Y / T are the
  // same, but the column loop runs the cheaper body path
  tile_qr_t<C, false>(A, b, sm, 0, h);
  {
    const int ldy = tp.ldy;
    double* Yn = tp.Y[L] + (int64_t)q * ldy * b;
    for (int idx = threadIdx.x; idx < b * b; idx += C::NT) {
      const int i = idx % b, k = idx / b;
      Yn[i + (int64_t)ldy * k] = i == k ? 1.0 : 0.0;  // child 0's block of V: the identity
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int lc = lane / C::LR, lr = lane % C::LR;
#pragma unroll
    for (int t = 0; t < C::CPL; ++t) {
      const int k = col_of<C>(t, warp, lc);
      if (k >= b) continue;
#pragma unroll
      for (int s = 0; s < C::RPL; ++s) {
        const int r = b + C::row(s, lr);
        if (r < ldy) Yn[r + (int64_t)ldy * k] = A[s][t];
      }
    }
  }
  build_T<C>(sm, b);
  store_T<C>(sm, b, tp.T[L] + (int64_t)q * (((int64_t)b * b + 1) & ~1LL));
  C::sync();
  double* Rout = tp.R[L] + (int64_t)q * b * b;
  for (int idx = threadIdx.x; idx < b * b; idx += C::NT) {
    const int r = idx % b, k = idx / b;
    Rout[idx] = sm.Rs[r + C::BMAX * k];
  }
}

// sign fix: D = sign(diag R) (0 -> +1), Rout = D R (upper), both device
// (non-finite entries anywhere in the panel reach R: *bad is set, as
// local_qr raises NumericError for them, tsqr.py:116-117)
__global__ void sign_fix_kernel(const double* __restrict__ R, int b, double* __restrict__ D,
                                double* __restrict__ Rout, int* __restrict__ bad) {
  bool finite = true;
  for (int idx = threadIdx.x; idx < b * b; idx += blockDim.x) {
    const int r = idx % b, k = idx / b;
    const double dr = R[r + b * r] < 0.0 ? -1.0 : 1.0;
    Rout[idx] = (r <= k) ? dr * R[idx] : 0.0;
    if (r <= k && !isfinite(R[idx])) finite = false;
    if (k == 0) D[r] = dr;
  }
  if (!finite) *bad = 1;
}

// ------------------------------------------------------------------------
// apply: out = Q [D z0; 0], in three launches
//   1. tree levels, top-down: one CTA per node computes every child's
//      b x k block  z_c = [z;0]_c - V_c T V_top^T z   (written once, not
//      recomputed by every leaf CTA)
//   2. chains: one CTA per leaf chain walks its tiles in reverse with the
//      compact-WY T factors only: u_t = T_t z_t (head: T_0 V_top^T z_0),
//      z_{t-1} = z_t - u_t; writes every u_t (and z_0) to scratch
//   3. products: one CTA per tile, fully parallel: out_t = -Y_t u_t
//      (+ z_0 on the head tile's top rows); Y_t streamed into shared memory
//      by the bulk-copy (TMA) engine, 4x4 register blocks
// ------------------------------------------------------------------------
constexpr int kApplyNT = 256;
constexpr int kApplyKM = 64;   // max k

// one thread: copy `bytes` (multiple of 16) from global to shared, signalling bar
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  mbar_expect_tx(bar, bytes);
  constexpr unsigned kChunk = 32768;
  for (unsigned off = 0; off < bytes; off += kChunk) {
    const unsigned n = bytes - off < kChunk ? bytes - off : kChunk;
    bulk_g2s((char*)dst + off, (const char*)src + off, n, bar);
  }
}

__host__ __device__ __forceinline__ int64_t tstride_of(int b) { return ((int64_t)b * b + 1) & ~1LL; }
__host__ __device__ __forceinline__ int kpad(int k) { return (k + 3) & ~3; }

// shared-memory leading dimension for DMMA operand staging: >= n and
// congruent to 4 mod 16 (in doubles), so the 4x4 lane pattern of an m8n8k4
// fragment load (fr + ld*fc, fr, fc < 4) hits 16 distinct 8-byte banks
__host__ __device__ __forceinline__ int ldpad(int n) { return ((n + 11) & ~15) + 4; }

// ---- 1. tree levels -------------------------------------------------------
// One (node q, child c) pair: U = T_q Z, z_c = [Z;0]_c - V_c U, with Z the
// node's input block (D, optional, multiplies its rows: the root's sign
// fix).  Every node is factored as a body tile [R_child0; ...] (tsqr_tree_
// kernel), so child 0's block of V is the identity: V_top^T Z = Z and
// z_0 = Z - U.  Both products run on the fp64 MMA path (cta_dmma).
__device__ __forceinline__ void tree_apply_pair(const Level& L, int q, int c, int b, int k,
                                                const double* __restrict__ zq, const double* __restrict__ D,
                                                double* __restrict__ zc, double* tsm) {
  constexpr int NW = kApplyNT / 32;
  const int ld = ldpad(b);
  double* Z = tsm;            // b x k (ld)
  double* U = Z + ld * k;     // b x k
  double* Tm = U + ld * k;    // b x b
  double* Vc = Tm + ld * b;   // b x b  this child's block (c > 0)
  const double* Yg = L.Y + (int64_t)q * L.ldy * b;
  const double* Tg = L.T + (int64_t)q * tstride_of(b);
#pragma unroll 4
  for (int idx = threadIdx.x; idx < b * k; idx += kApplyNT) {
    const int i = idx % b, cc = idx / b;
    const double d = D ? D[i] : 1.0;
    Z[i + ld * cc] = d * zq[idx];
  }
#pragma unroll 4
  for (int idx = threadIdx.x; idx < b * b; idx += kApplyNT) {
    const int i = idx % b, j = idx / b;
    Tm[i + ld * j] = Tg[idx];
    if (c > 0) Vc[i + ld * j] = Yg[(int64_t)c * b + i + (int64_t)L.ldy * j];
  }
  __syncthreads();
  // U = T Z  (T upper)
  cta_dmma(
      b, k, b, NW, [&](int m, int l) { return (l >= m && l < b && m < b) ? Tm[m + ld * l] : 0.0; },
      [&](int l, int n) { return (l < b && n < k) ? Z[l + ld * n] : 0.0; },
      [&](int m, int n, double v) { U[m + ld * n] = v; });
  __syncthreads();
  if (c == 0) {
    for (int idx = threadIdx.x; idx < b * k; idx += kApplyNT) {
      const int m = idx % b, n = idx / b;
      zc[idx] = Z[m + ld * n] - U[m + ld * n];
    }
  } else {
    cta_dmma(
        b, k, b, NW, [&](int m, int l) { return (m < b && l < b) ? Vc[m + ld * l] : 0.0; },
        [&](int l, int n) { return (l < b && n < k) ? U[l + ld * n] : 0.0; },
        [&](int m, int n, double v) { zc[m + b * n] = -v; });
  }
}

// one level, one CTA per (node, child): zin (nodes) blocks of b x k (ld b),
// zout (nodes * f) child blocks
__global__ void __launch_bounds__(kApplyNT) tsqr_tree_apply_kernel(Level L, int nnodes_below, int b, int k,
                                                                   const double* __restrict__ zin,
                                                                   const double* __restrict__ D,
                                                                   double* __restrict__ zout) {
  extern __shared__ __align__(16) double tsm[];
  const int q = blockIdx.x / L.f, c = blockIdx.x - q * L.f;
  if (q * L.f + c >= nnodes_below) return;
  tree_apply_pair(L, q, c, b, k, zin + (int64_t)q * b * k, D, zout + ((int64_t)q * L.f + c) * b * k, tsm);
}

// Every level of a rank's local tree in ONE launch, top-down.  CTAs take
// pair ids from an atomic ticket in level order (root first), so a pair
// only waits (on its input block's ready flag) for a pair of the level
// above, which started earlier; per-level launches cost ~4 launch
// latencies per apply on the truncation sweep's critical path.
struct TreeApplyAll {
  int nlev, b, k;
  Level lev[kMaxLevels];
  int below[kMaxLevels];  // child blocks of each level
  int npair[kMaxLevels];  // nodes * f
  double* out[kMaxLevels];  // per level: npair blocks of b x k
  const double* zin;        // the root's input block
  const double* D;
  unsigned* flags;          // one per output block of every level (zeroed per launch)
  int flag_off[kMaxLevels];
  unsigned* ticket;
};

__global__ void __launch_bounds__(kApplyNT) tsqr_tree_apply_all_kernel(TreeApplyAll a) {
  extern __shared__ __align__(16) double tsm[];
  __shared__ int id_s;
  if (threadIdx.x == 0) id_s = (int)atomicAdd(a.ticket, 1u);
  __syncthreads();
  int id = id_s, L = a.nlev - 1;
  while (L > 0 && id >= a.npair[L]) id -= a.npair[L--];
  const Level& lv = a.lev[L];
  const int q = id / lv.f, c = id - q * lv.f;
  if (q * lv.f + c >= a.below[L]) return;
  const double* zq;
  if (L == a.nlev - 1) {
    zq = a.zin;
  } else {
    const unsigned* fl = a.flags + a.flag_off[L + 1] + q;
    if (threadIdx.x == 0)
      while (ld_acquire(fl) == 0u) {
      }
    __syncthreads();
    zq = a.out[L + 1] + (int64_t)q * a.b * a.k;
  }
  double* zc = a.out[L] + ((int64_t)q * lv.f + c) * a.b * a.k;
  tree_apply_pair(lv, q, c, a.b, a.k, zq, L == a.nlev - 1 ? a.D : nullptr, zc, tsm);
  __syncthreads();  // the block is written
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
    atomicExch(a.flags + a.flag_off[L] + q * lv.f + c, 1u);
  }
}

// ---- 2. chains ------------------------------------------------------------
struct ChainArgs {
  LeafPlan plan;
  int ldy;
  const double* Y;
  const double* T;
  const double* zin;     // per CTA b x k (ld b)
  const double* D;       // sign fix when there is no tree above (else null)
  int k;
  double* u;             // per tile b x ldpad(k), row-major (l*ldu + c); columns >= k unused
  double* z0;            // per CTA b x k: the head tile's input z_0
};

// One CTA per leaf chain, tiles in reverse.  z ping-pongs between two
// shared buffers so that u_t = T_t z_t, z_{t-1} = z_t - u_t is one MMA pass
// and one barrier per tile; T_t arrives by bulk copy two tiles ahead.
__global__ void __launch_bounds__(kApplyNT) tsqr_chain_kernel(ChainArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int NW = kApplyNT / 32;
  const int g = blockIdx.x;
  const LeafPlan& pl = a.plan;
  const int b = pl.b, k = a.k, KP = ldpad(k), ld = ldpad(b);  // KP: row stride of u
  const int64_t tsz = tstride_of(b);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem_raw);  // T double buffer
  double* const Zb0 = reinterpret_cast<double*>(smem_raw + 64);
  double* const Zb1 = Zb0 + ld * k;
  double* W = Zb1 + ld * k;
  double* Tb0 = W + ld * k;
  double* Tb1 = Tb0 + tsz;
  const int64_t n_g = pl.count(g);
  const int ntiles = pl.tiles_of(n_g);
  const int64_t tb = pl.tile_base(g);
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int idx = threadIdx.x; idx < b * k; idx += kApplyNT) {
    const int i = idx % b, c = idx / b;
    const double d = a.D ? a.D[i] : 1.0;
    Zb0[i + ld * c] = d * a.zin[(int64_t)g * b * k + idx];
  }
  __syncthreads();
  const unsigned tbytes = (unsigned)(tsz * 8);
  if (threadIdx.x == 0) {
    bulk_load(Tb0, a.T + (tb + ntiles - 1) * tsz, tbytes, &bars[0]);
    if (ntiles > 1) bulk_load(Tb1, a.T + (tb + ntiles - 2) * tsz, tbytes, &bars[1]);
  }
  int zc = 0;
  for (int t = ntiles - 1, it = 0; t >= 0; --t, ++it) {
    const int cur = it & 1;
    const double* Tc = cur ? Tb1 : Tb0;
    const double* Z = zc ? Zb1 : Zb0;
    double* Zn = zc ? Zb0 : Zb1;
    mbar_wait(&bars[cur], (it >> 1) & 1);
    double* ut = a.u + (tb + t) * (int64_t)b * KP;
    auto Ta = [&](int m, int l) { return (l >= m && l < b && m < b) ? Tc[m + b * l] : 0.0; };
    if (t == 0) {
      // head: u_0 = T_0 (V_top^T z_0), V_top = rows 0..b-1 of Y_0 (global)
      const double* Y0 = a.Y + tb * y_tile_stride(a.ldy, b);  // rows < b: unit 0
      cta_dmma(
          b, k, b, NW, [&](int m, int l) { return (l >= m && l < b) ? Y0[l + (int64_t)kYLd * m] : 0.0; },
          [&](int l, int n) { return (l < b && n < k) ? Z[l + ld * n] : 0.0; },
          [&](int m, int n, double v) { W[m + ld * n] = v; });
      __syncthreads();
      cta_dmma(
          b, k, b, NW, Ta, [&](int l, int n) { return (l < b && n < k) ? W[l + ld * n] : 0.0; },
          [&](int m, int n, double v) { ut[m * KP + n] = v; });
      for (int idx = threadIdx.x; idx < b * k; idx += kApplyNT) {
        const int i = idx % b, c = idx / b;
        a.z0[(int64_t)g * b * k + idx] = Z[i + ld * c];
      }
    } else {
      cta_dmma(
          b, k, b, NW, Ta, [&](int l, int n) { return (l < b && n < k) ? Z[l + ld * n] : 0.0; },
          [&](int m, int n, double v) {
            ut[m * KP + n] = v;
            Zn[m + ld * n] = Z[m + ld * n] - v;
          });
    }
    __syncthreads();
    zc ^= 1;
    if (threadIdx.x == 0 && t >= 2) {
      fence_proxy_async();
      bulk_load(const_cast<double*>(Tc), a.T + (tb + t - 2) * tsz, tbytes, &bars[cur]);
    }
  }
}

// ---- 3. products ----------------------------------------------------------
struct ProductArgs {
  LeafPlan plan;
  int ldy;
  int unit_rows;
  int stages;
  int upw;
  const double* Y;
  const double* u;
  const double* z0;
  int k;
  Panel out;
};

// One CTA per tile: out_t = -Y_t u_t (+ z_0 on the head tile's top rows).
// Y_t is bulk-copied column by column into a bank-padded shared layout.
// Persistent: one CTA per SM walks work units blockIdx.x, +gridDim.x, ...
// (a unit = 128 rows of one tile) with a two-stage bulk-copy pipeline: unit
// i+1's rows of Y_t and its u_t stream into shared memory while unit i is
// multiplied.
constexpr int kProdMaxStages = 8;  // stage count: as many units as fit ~200 KB (>= 2)

struct ProductUnit {
  int rows;  // rows per work unit (kYUnit)
  __host__ __device__ static size_t smem(int ur, int b, int k) {
    return ((size_t)(ur + 4) * b + (size_t)b * ldpad(k)) * sizeof(double);  // one stage
  }
};

__device__ __forceinline__ void product_tile_of(const LeafPlan& pl, int64_t tile, int& g, int64_t& t) {
  const int rem = pl.rem();
  const int64_t t1 = pl.tiles_of(pl.base() + 1), t0 = pl.tiles_of(pl.base());
  if (tile < (int64_t)rem * t1) {
    g = (int)(tile / t1);
    t = tile - (int64_t)g * t1;
  } else {
    const int64_t x = tile - (int64_t)rem * t1;
    g = rem + (int)(x / t0);
    t = x - (int64_t)(g - rem) * t0;
  }
}

constexpr int kProdNT = 512;  // 16 warps: one 16x16 output block each per unit at k <= 32

__global__ void __launch_bounds__(kProdNT, 1) tsqr_product_kernel(ProductArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int NW = kProdNT / 32;
  const LeafPlan& pl = a.plan;
  const int b = pl.b, k = a.k, ldy = a.ldy, rs = pl.rs, ni = pl.ni;
  const int upw = a.upw;     // Y units per work item (consecutive, contiguous in global)
  const int UR = kYUnit * upw;
  const int lys = kYLd;
  const int64_t ustride = (int64_t)b * kYLd;  // one unit of Y
  const int ldu = ldpad(k);
  const int halves = ldy / UR;
  const int64_t nunits = pl.total_tiles() * halves;
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem_raw);  // stage full (tx bytes)
  unsigned* cnt = reinterpret_cast<unsigned*>(smem_raw + 64);                  // warps done with a stage
  double* Ysb = reinterpret_cast<double*>(smem_raw + 128);
  const int64_t ystage = ustride * upw, ustage = (int64_t)b * ldu;
  const int S = a.stages;
  double* Usb = Ysb + S * ystage;
  const unsigned ubytes = (unsigned)(ustage * 8);
  if (threadIdx.x == 0) {
    for (int s2 = 0; s2 < S; ++s2) {
      mbar_init(&bar[s2], 1);
      cnt[s2] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // one thread issues the copies of a work unit into a stage (the unit is one
  // contiguous block: unit-major Y layout)
  auto issue = [&](int64_t unit, int st) {
    const int64_t tile = unit / halves;
    const int r0 = (int)(unit - tile * halves) * UR;
    const double* Yg = a.Y + tile * y_tile_stride(ldy, b) + (int64_t)(r0 / kYUnit) * b * kYLd;
    mbar_expect_tx(&bar[st], (unsigned)(ystage * 8) + ubytes);
    bulk_g2s(Ysb + st * ystage, Yg, (unsigned)(ystage * 8), &bar[st]);
    bulk_g2s(Usb + st * ustage, a.u + tile * ustage, ubytes, &bar[st]);
  };
  int64_t unit = blockIdx.x;
  if (threadIdx.x == 0)
    for (int s2 = 0; s2 < S; ++s2)
      if (unit + (int64_t)s2 * gridDim.x < nunits) issue(unit + (int64_t)s2 * gridDim.x, s2);
  // No CTA-wide barrier per unit: every warp waits for the stage, computes its
  // output tiles with row offsets it derives itself, and counts itself out of
  // the stage; the LAST warp out refills the stage with the unit S ahead.
  // Warps drift apart by up to a unit, so the output stores of one overlap the
  // MMAs of the others (in lockstep every warp reached its MMA phase together:
  // math_pipe_throttle was the first stall reason with the pipe 49 % busy).
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, t4 = lane & 3;
  const int64_t cstride = a.out.trans ? 1 : a.out.rl * a.out.I;
  double* ob = a.out.base;
  for (int it = 0; unit < nunits; ++it, unit += gridDim.x) {
    const int st = it % S;
    const int64_t tile = unit / halves;
    const int r0 = (int)(unit - tile * halves) * UR;
    int g;
    int64_t t;
    product_tile_of(pl, tile, g, t);
    const int64_t n_g = pl.count(g);
    const int64_t ia = pl.start(g) + t * ni;
    const int nsl = (int)min64(ni, n_g - t * ni);
    const int rows = min(nsl * rs - r0, UR);
    const bool head = (t == 0) && r0 == 0;
    const double* z0 = a.z0 + (int64_t)g * b * k;
    const double* Ys = Ysb + st * ystage;
    const double* Us = Usb + st * ustage;
    mbar_wait(&bar[st], (it / S) & 1);
    if (rows > 0) {
      // 16 x 8 output tiles on the m16n8k8 fp64 MMA; Y rows beyond `rows`
      // are exact zeros (zero-padded leaf tiles), so only the reflector index
      // needs a bound (columns of u beyond k only feed outputs never stored)
      const int mt = (rows + 15) >> 4, ntl = (k + 7) >> 3, kst = (b + 7) >> 3;
      // two output tiles per warp pass share a row tile (the A fragments) and
      // run as two independent MMA chains
      const int ntiles2 = mt * ((ntl + 1) >> 1);
      for (int tt = warp; tt < ntiles2; tt += NW) {
        const int m0 = (tt % mt) * 16, n0 = (tt / mt) * 16;
        const bool two = n0 + 8 < k;
        // output addresses of this lane's two rows (one division pair per row)
        int64_t ro[2];
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int m = m0 + gq + 8 * h2;
          int si, w;
          tile_row(a.out.trans, r0 + (m < rows ? m : 0), nsl, rs, si, w);
          ro[h2] = a.out.addr(w, ia + si, 0);
        }
        const double* ya = Ys + (m0 >> 7) * ustride + (m0 & (kYUnit - 1)) + gq;
        const double* ub = Us + n0 + gq;
        double d[4] = {0.0, 0.0, 0.0, 0.0}, e[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 4
        for (int ks = 0; ks < kst; ++ks) {
          const int l0 = ks * 8 + t4, l1 = l0 + 4;
          const bool ok0 = l0 < b, ok1 = l1 < b;
          const double a0 = ok0 ? ya[lys * l0] : 0.0, a1 = ok0 ? ya[8 + lys * l0] : 0.0;
          const double a2 = ok1 ? ya[lys * l1] : 0.0, a3 = ok1 ? ya[8 + lys * l1] : 0.0;
          const double b0 = ok0 ? ub[l0 * ldu] : 0.0, b1 = ok1 ? ub[l1 * ldu] : 0.0;
          dmma_1688(d, a0, a1, a2, a3, b0, b1);
          if (two) {
            const double c0 = ok0 ? ub[l0 * ldu + 8] : 0.0, c1 = ok1 ? ub[l1 * ldu + 8] : 0.0;
            dmma_1688(e, a0, a1, a2, a3, c0, c1);
          }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int h2 = (i >> 1) & 1;
          const int m = m0 + gq + 8 * h2, n = n0 + 8 * (i >> 2) + 2 * t4 + (i & 1);
          if (m < rows && n < k) {
            const double base = (head && m < b) ? z0[m + b * n] : 0.0;
            ob[ro[h2] + cstride * n] = base - (i < 4 ? d[i & 3] : e[i & 3]);
          }
        }
      }
    }
    // this warp is done with the stage (its fragment loads have been consumed)
    __syncwarp();
    if (lane == 0) {
      unsigned old;
      asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;\n" : "=r"(old) : "r"(smem_u32(&cnt[st])) : "memory");
      if (old == NW - 1) {  // last warp out: refill
        cnt[st] = 0;
        const int64_t nxt = unit + (int64_t)S * gridDim.x;
        if (nxt < nunits) {
          fence_proxy_async();
          issue(nxt, st);
        }
      }
    }
  }
}
// ------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------
namespace {

template <class C>
size_t tile_smem() { return sizeof(TileSmem<C>); }
template <class C>
size_t tree_smem() {
  // staging of the children's streamed rows: up to MC / b + 1 children of b rows
  return ((sizeof(TileSmem<C>) + 127) & ~size_t(127)) + kMaxChunks * 8 + (size_t)(C::MC + C::BMAX) * C::BMAX * 8;
}

template <class C>
void set_smem_attr(const void* fn) {
  smem_attr(fn, sizeof(TileSmem<C>));
}

template <class LC_, class TC_>
void run_factor(Ctx& ctx, Tsqr& f) {
  cudaStream_t st = ctx.stream;
  auto leaf = tsqr_leaf_kernel<LC_>;
  set_smem_attr<LC_>((const void*)leaf);
  bool deferred_T = false;
  cudaEvent_t leaf_done = nullptr;
  {
    // TTB_LEAF2=1 selects the blocked panel-warp leaf (leaf2.cu): correct, but
    // measured slower than the column pipeline on B200, so opt-in
    static const bool v2 = getenv("TTB_LEAF2") != nullptr;
    static const bool v3 = getenv("TTB_LEAF3") != nullptr;
    ProfScope ps("tsqr_leaf", st);
    if (f.wl) {
      launch_wleaf(ctx, f.panel, f.wplan, f.Y, f.T, f.Rleaf);
    } else if (f.cls == 64 && v3) {
      launch_leaf3(ctx, f.panel, f.plan, f.Y, f.T, f.Rleaf);
    } else if (f.cls == 64 && v2) {
      launch_leaf2(ctx, f.panel, f.plan, f.Y, f.T, f.Rleaf);
    } else {
      // TTB_LEAF_T=defer moves build_T out of the chain into tile_T_kernel on the
      // aux stream (measured: leaf 12.55 -> 11.93 ms per cfg3 round, but the
      // ~1.0 ms of T blocks slow whatever they run beside by as much -- the
      // tree when enqueued before it, the R-fold and the SVD when after --
      // so the step stays at 20.5 ms: opt-in)
      static const bool dfr = getenv("TTB_LEAF_T") && std::string(getenv("TTB_LEAF_T")) == "defer";
      const int defer = dfr ? 1 : 0;
      leaf<<<f.plan.G, LC_::NT, tile_smem<LC_>(), st>>>(f.panel, f.plan, f.Y, f.T, f.Rleaf, f.r_only ? 0 : defer,
                                                         f.r_only ? 1 : 0);
      TTB_LAUNCHED();
      deferred_T = defer != 0 && !f.r_only;
    }
  }
  auto tree = tsqr_tree_kernel<TC_>;
  smem_attr((const void*)tree, tree_smem<TC_>());
  // levels [0, n) of a tree over n_in complete inputs, one launch
  auto run_tree = [&](const double* rin, int n_in, int nlev, double* const* Ys, double* const* Ts,
                      double* const* Rs) {
    TreePlan tp;
    tp.nlev = nlev;
    tp.b = f.b;
    tp.f = f.ftree;
    tp.ldy = f.ldy_tree;
    int total = 0;
    for (int L = 0; L < nlev; ++L) {
      const int nodes = (n_in + f.ftree - 1) / f.ftree;
      tp.first[L] = total;
      tp.n_in[L] = n_in;
      tp.Rin[L] = rin;
      tp.Y[L] = Ys[L];
      tp.T[L] = Ts[L];
      tp.R[L] = Rs[L];
      total += nodes;
      rin = Rs[L];
      n_in = nodes;
    }
    tp.first[nlev] = total;
    TTB_CHECK(total <= ctx.num_sms, TTB_ERR_CAPABILITY, "TSQR tree: more nodes than SMs");
    tp.prog = f.prog;
    tp.ticket = f.prog + ctx.num_sms;
    tp.Rrow = f.Rrow;
    tp.ldr = f.ldr;
    TTB_CHECK((f.b + kTreeChunk - 1) / kTreeChunk <= kMaxChunks, TTB_ERR_CAPABILITY, "TSQR tree: too many chunks");
    TTB_CUDA(cudaMemsetAsync(f.prog, 0, sizeof(unsigned) * total, st));
    TTB_CUDA(cudaMemsetAsync(tp.ticket, 0, sizeof(unsigned), st));
    ProfScope ps("tsqr_tree", st);
    tree<<<total, TC_::NTT, tree_smem<TC_>(), st>>>(tp);
    TTB_LAUNCHED();
    return rin;
  };
  const int G = f.wl ? f.wplan.G : f.plan.G;
  f.Rlocal = f.nloc > 0 ? run_tree(f.Rleaf, G, f.nloc, f.locY, f.locT, f.locR) : f.Rleaf;
  if (deferred_T && f.plan.total_tiles() > 0) {
    // per-tile T factors on the aux stream, after the local tree: they run
    // beside what follows it -- the one-CTA SVD of the truncation sweep, the
    // R-fold of the orthonormalization sweep -- not beside the tree, whose
    // nodes need a whole SM's shared memory each and were placed late when
    // the T blocks got there first (tree 150 -> 176 us)
    TTB_CUDA(cudaEventCreateWithFlags(&leaf_done, cudaEventDisableTiming));
    TTB_CUDA(cudaEventRecord(leaf_done, st));
    cudaStream_t ax = ctx.aux_stream();
    TTB_CUDA(cudaStreamWaitEvent(ax, leaf_done, 0));
    TTB_CUDA(cudaEventDestroy(leaf_done));
    {
      ProfScope pt("tile_T", ax);
      smem_attr((const void*)tile_T_kernel, sizeof(TSmem));
      tile_T_kernel<<<(unsigned)f.plan.total_tiles(), 256, sizeof(TSmem), ax>>>(f.T, f.b,
                                                                                ((int64_t)f.b * f.b + 1) & ~1LL);
      TTB_LAUNCHED();
    }
    TTB_CUDA(cudaEventCreateWithFlags(&f.t_ready, cudaEventDisableTiming));
    TTB_CUDA(cudaEventRecord(f.t_ready, ax));
  }
  if (ctx.nranks > 1) {
    // allgather the rank roots, then a redundant (bitwise identical) tree
    ctx.allgather(f.Rlocal, f.Rstack, (size_t)f.b * f.b);
    f.Rraw = f.nglob > 0 ? run_tree(f.Rstack, ctx.nranks, f.nglob, f.gloY, f.gloT, f.gloR) : f.Rstack;
  } else {
    f.Rraw = f.Rlocal;
  }
  sign_fix_kernel<<<1, 256, 0, st>>>(f.Rraw, f.b, f.D, f.R, ctx.flag());
  TTB_LAUNCHED();
}

}  // namespace

int tsqr_class(int b) {
  if (b <= 16) return 16;
  if (b <= 32) return 32;
  if (b <= 64) return 64;
  return 0;
}

static int leaf_mc(int cls) { return cls == 16 ? Leaf16::MC : cls == 32 ? Leaf32::MC : Leaf64::MC; }
static int tree_mc(int cls) { return cls == 16 ? Tree16::MC : cls == 32 ? Tree32::MC : Tree64::MC; }

void tsqr_factor(Ctx& ctx, const Panel& panel, Tsqr& f) {
  if (tsqr_needs_wide(panel)) {  // more than 64 columns or slices taller than a tile: the general path
    wide_tsqr_factor(ctx, panel, f);
    return;
  }
  const int b = (int)panel.ncols();
  const int64_t rs = panel.rs();
  f.b = b;
  f.panel = panel;
  f.cls = tsqr_class(b);
  TTB_CHECK(b >= 1, TTB_ERR_SHAPE, "TSQR needs at least one column");
  TTB_CHECK(f.cls != 0, TTB_ERR_CAPABILITY, "TSQR: column count " + std::to_string(b) + " exceeds 64");
  const int MC = leaf_mc(f.cls), MT = tree_mc(f.cls);
  const int64_t ns = panel.I;
  // TTB_WLEAF=1 selects the team-pipelined leaf (wleaf.cu): correct on every
  // GPU test, but measured no faster than the CTA-wide column pipeline on
  // the BASELINE panels, so opt-in
  static const bool wl_on = getenv("TTB_WLEAF") != nullptr;
  f.wl = wl_on ? 1 : 0;
  TTB_CHECK(rs >= 1 && (f.wl || rs <= MC - b + 1), TTB_ERR_CAPABILITY,
            "TSQR: rows per slice " + std::to_string(rs) + " too large for the tile (" + std::to_string(MC) + ")");
  f.plan.nslices = ns;
  f.plan.rs = (int)rs;
  f.plan.b = b;
  f.plan.ni = (int)std::max<int64_t>(1, MC / rs);
  // CTAs: at most 2 per SM; every CTA gets >= 2 tiles of rows, so small
  // panels are one chain (one head tile = the reference's single dgeqrf
  // pivot order) and the head tile always reaches b rows.
  const int64_t min_sl = std::max<int64_t>((b + rs - 1) / rs, 2 * (int64_t)f.plan.ni);
  int64_t gmax = ns >= min_sl ? ns / min_sl : 1;
  // resident CTAs per SM of the leaf configuration (TCfg::MINB)
  const int minb = f.cls == 16 ? Leaf16::MINB : f.cls == 32 ? Leaf32::MINB : Leaf64::MINB;
  static const int cps_env = getenv("TTB_LEAF_CPS") ? atoi(getenv("TTB_LEAF_CPS")) : 0;
  const int cps = cps_env > 0 ? cps_env : minb;
  int G = (int)std::min<int64_t>((int64_t)cps * ctx.num_sms, std::max<int64_t>(1, gmax));
  if (ns == 0) G = 1;
  f.plan.G = G;
  if (f.wl) {
    // chains: one per SM at most, every team of a chain gets a tile, and
    // every chain has at least b rows (its head tile is a full QR)
    const int teams = wleaf_teams(b);
    const int64_t tiles = (ns * rs + kWH - 1) / kWH;
    const int64_t per = (b + rs - 1) / rs;  // slices that reach b rows
    int64_t gw = std::min<int64_t>((int64_t)ctx.num_sms, (tiles + teams - 1) / teams);
    gw = std::min<int64_t>(gw, ns / per);
    G = (int)std::max<int64_t>(1, gw);
    f.wplan.nslices = ns;
    f.wplan.G = G;
    f.wplan.rs = (int)rs;
    f.wplan.b = b;
  }
  f.ftree = MT / b + 1;  // child 0 is the node's shared-memory R, the others fill the register tile
  f.ldy = MC;
  f.ldy_tree = f.ftree * b;
  // tree sizes
  f.nloc = 0;
  int n = G;
  int nodes_loc[kMaxLevels];
  while (n > 1) {
    TTB_CHECK(f.nloc < kMaxLevels, TTB_ERR_CAPABILITY, "TSQR tree too deep");
    n = (n + f.ftree - 1) / f.ftree;
    nodes_loc[f.nloc++] = n;
  }
  f.nglob = 0;
  int nodes_glo[kMaxLevels];
  n = ctx.nranks;
  while (n > 1) {
    TTB_CHECK(f.nglob < kMaxLevels, TTB_ERR_CAPABILITY, "TSQR global tree too deep");
    n = (n + f.ftree - 1) / f.ftree;
    nodes_glo[f.nglob++] = n;
  }
  const int64_t ntiles = f.plan.total_tiles();
  const int64_t bb = (int64_t)b * b;
  size_t total = 0;
  auto add = [&](int64_t cnt) { size_t off = total; total += ((size_t)cnt * 8 + 255) / 256 * 256; return off; };
  const int64_t tsz = (bb + 1) & ~1LL;
  const int64_t nyd = f.wl ? (int64_t)wleaf_y_doubles(f.wplan) : ntiles * y_tile_stride(MC, b);
  const int64_t ntd = f.wl ? (int64_t)wleaf_u_doubles(f.wplan) : ntiles * tsz;
  size_t oY = add(nyd), oT = add(ntd), oRl = add((int64_t)G * bb);
  size_t oLY[kMaxLevels], oLT[kMaxLevels], oLR[kMaxLevels];
  for (int L = 0; L < f.nloc; ++L) {
    oLY[L] = add((int64_t)nodes_loc[L] * f.ldy_tree * b);
    oLT[L] = add((int64_t)nodes_loc[L] * tsz);
    oLR[L] = add((int64_t)nodes_loc[L] * bb);
  }
  size_t oGS = add((int64_t)ctx.nranks * bb);
  size_t oGY[kMaxLevels], oGT[kMaxLevels], oGR[kMaxLevels];
  for (int L = 0; L < f.nglob; ++L) {
    oGY[L] = add((int64_t)nodes_glo[L] * f.ldy_tree * b);
    oGT[L] = add((int64_t)nodes_glo[L] * tsz);
    oGR[L] = add((int64_t)nodes_glo[L] * bb);
  }
  size_t oD = add(b), oR = add(bb), oP = add(ctx.num_sms + 1);
  f.ldr = (b + 1) & ~1;
  size_t oRr = add((int64_t)ctx.num_sms * b * f.ldr);
  f.mem = ctx.alloc(total);
  char* base = (char*)f.mem;
  f.Y = (double*)(base + oY);
  f.T = (double*)(base + oT);
  f.Rleaf = (double*)(base + oRl);
  for (int L = 0; L < f.nloc; ++L) {
    f.locY[L] = (double*)(base + oLY[L]);
    f.locT[L] = (double*)(base + oLT[L]);
    f.locR[L] = (double*)(base + oLR[L]);
  }
  f.Rstack = (double*)(base + oGS);
  for (int L = 0; L < f.nglob; ++L) {
    f.gloY[L] = (double*)(base + oGY[L]);
    f.gloT[L] = (double*)(base + oGT[L]);
    f.gloR[L] = (double*)(base + oGR[L]);
  }
  f.D = (double*)(base + oD);
  f.R = (double*)(base + oR);
  f.prog = (unsigned*)(base + oP);
  f.Rrow = (double*)(base + oRr);
  if (f.cls == 16) run_factor<Leaf16, Tree16>(ctx, f);
  else if (f.cls == 32) run_factor<Leaf32, Tree32>(ctx, f);
  else run_factor<Leaf64, Tree64>(ctx, f);
}

void tsqr_apply(Ctx& ctx, const Tsqr& f, const double* z, int k, const Panel& out) {
  if (f.wide) {
    wide_tsqr_apply(ctx, f, z, k, out);
    return;
  }
  TTB_CHECK(!f.r_only, TTB_ERR_CONTRACT, "TSQR apply: the factor was computed for R only");
  TTB_CHECK(k >= 1 && k <= kApplyKM, TTB_ERR_CAPABILITY, "TSQR apply: k must be in [1, 64]");
  TTB_CHECK(out.rs() == f.panel.rs() && out.I == f.panel.I && out.ncols() == k, TTB_ERR_SHAPE,
            "TSQR apply: output view does not match the factored panel");
  const int b = f.b, KP = kpad(k), G = f.wl ? f.wplan.G : f.plan.G;
  const int64_t bk = (int64_t)b * k, ntiles = f.wl ? f.wplan.total_tiles() : f.plan.total_tiles();
  // node counts per level
  std::vector<int> lnodes(f.nloc), gnodes(ctx.nranks > 1 ? f.nglob : 0);
  for (int L = 0, n = G; L < f.nloc; ++L) lnodes[L] = n = (n + f.ftree - 1) / f.ftree;
  for (int L = 0, n = ctx.nranks; L < (int)gnodes.size(); ++L) gnodes[L] = n = (n + f.ftree - 1) / f.ftree;
  int64_t maxlev = 1;
  for (int L = 0; L < f.nloc; ++L) maxlev = std::max<int64_t>(maxlev, (int64_t)lnodes[L] * f.ftree);
  for (size_t L = 0; L < gnodes.size(); ++L) maxlev = std::max<int64_t>(maxlev, (int64_t)gnodes[L] * f.ftree);
  int64_t treeblocks = 0;  // every local level's output blocks (one launch holds them all)
  for (int L = 0; L < f.nloc; ++L) treeblocks += (int64_t)lnodes[L] * f.ftree;
  const int64_t nscr = 2 * maxlev * bk + ntiles * b * ldpad(k) + (int64_t)G * bk + treeblocks * bk +
                       (treeblocks + 2) / 2 + 1;
  double* scr = (double*)ctx.alloc((size_t)nscr * sizeof(double));
  double* lev[2] = {scr, scr + maxlev * bk};
  double* ubuf = scr + 2 * maxlev * bk;
  double* z0buf = ubuf + ntiles * b * ldpad(k);
  double* treebuf = z0buf + (int64_t)G * bk;
  unsigned* treeflags = reinterpret_cast<unsigned*>(treebuf + treeblocks * bk);
  smem_attr((const void*)tsqr_tree_apply_kernel, 227 * 1024);
  smem_attr((const void*)tsqr_chain_kernel, 227 * 1024);
  smem_attr((const void*)tsqr_product_kernel, 227 * 1024);
  const double* cur = z;
  const double* Dp = f.D;
  int which = 0;
  const int ldb = ldpad(b);
  const size_t tsmem = (size_t)(2 * (int64_t)ldb * k + 2 * (int64_t)ldb * b) * sizeof(double);
  // global levels (redundant on every rank), then this rank's block
  for (int L = (int)gnodes.size() - 1; L >= 0; --L) {
    const int below = L == 0 ? ctx.nranks : gnodes[L - 1];
    Level lv{f.gloY[L], f.gloT[L], f.ldy_tree, f.ftree, -1};
    ProfScope ps("apply_tree", ctx.stream);
    tsqr_tree_apply_kernel<<<gnodes[L] * f.ftree, kApplyNT, tsmem, ctx.stream>>>(lv, below, b, k, cur, Dp, lev[which]);
    TTB_LAUNCHED();
    Dp = nullptr;
    cur = lev[which] + (L == 0 ? (int64_t)ctx.rank * bk : 0);
    which ^= 1;
  }
  if (f.nloc > 0) {
    TreeApplyAll ta;
    ta.nlev = f.nloc;
    ta.b = b;
    ta.k = k;
    int nflags = 0, npairs = 0;
    for (int L = 0; L < f.nloc; ++L) {
      ta.lev[L] = Level{f.locY[L], f.locT[L], f.ldy_tree, f.ftree, -1};
      ta.below[L] = L == 0 ? G : lnodes[L - 1];
      ta.npair[L] = lnodes[L] * f.ftree;
      ta.flag_off[L] = nflags;
      nflags += ta.npair[L];
      npairs += ta.npair[L];
    }
    int64_t off = 0;
    for (int L = 0; L < f.nloc; ++L) {
      ta.out[L] = treebuf + off;
      off += (int64_t)ta.npair[L] * bk;
    }
    ta.zin = cur;
    ta.D = Dp;
    ta.flags = treeflags;
    ta.ticket = treeflags + nflags;
    TTB_CUDA(cudaMemsetAsync(treeflags, 0, sizeof(unsigned) * (nflags + 1), ctx.stream));
    smem_attr((const void*)tsqr_tree_apply_all_kernel, tsmem);
    ProfScope ps("apply_tree", ctx.stream);
    tsqr_tree_apply_all_kernel<<<npairs, kApplyNT, tsmem, ctx.stream>>>(ta);
    TTB_LAUNCHED();
    Dp = nullptr;
    cur = ta.out[0];
  }
  if (f.wl) {
    wleaf_apply_tail(ctx, f.wplan, f.Y, f.T, cur, Dp, k, out, ubuf, z0buf);
    ctx.free(scr);
    return;
  }
  if (f.t_ready) TTB_CUDA(cudaStreamWaitEvent(ctx.stream, f.t_ready, 0));
  ChainArgs ca;
  ca.plan = f.plan;
  ca.ldy = f.ldy;
  ca.Y = f.Y;
  ca.T = f.T;
  ca.zin = cur;
  ca.D = Dp;
  ca.k = k;
  ca.u = ubuf;
  ca.z0 = z0buf;
  const size_t csmem = 64 + (size_t)(3 * (int64_t)ldb * k + 2 * tstride_of(b)) * sizeof(double);
  {
  ProfScope ps("apply_chain", ctx.stream);
  tsqr_chain_kernel<<<G, kApplyNT, csmem, ctx.stream>>>(ca);
  TTB_LAUNCHED();
  }
  ProductArgs pa;
  pa.plan = f.plan;
  pa.ldy = f.ldy;
  pa.Y = f.Y;
  pa.u = ubuf;
  pa.z0 = z0buf;
  pa.k = k;
  pa.out = out;
  TTB_CHECK(f.ldy % kYUnit == 0, TTB_ERR_CAPABILITY, "TSQR apply: tile rows not a multiple of 128");
  // small panels: several units per work item (more rows per CTA pass)
  pa.upw = 1;
  const size_t ubytes1 = (size_t)b * kYLd * sizeof(double);
  while (pa.upw * 2 <= f.ldy / kYUnit && (size_t)(pa.upw * 2) * ubytes1 <= 72 * 1024) pa.upw *= 2;
  pa.unit_rows = kYUnit * pa.upw;
  const size_t pstage = (size_t)pa.upw * ubytes1 + (size_t)b * ldpad(k) * sizeof(double);
  pa.stages = (int)std::max<size_t>(2, std::min<size_t>(kProdMaxStages, (200 * 1024) / pstage));
  // + 256: the B fragments of the last n-tile read up to 7 columns past k in
  // the last row of u (they only feed outputs that are never stored)
  const size_t psmem = 128 + (size_t)pa.stages * pstage + 256;
  ProfScope ps("apply_product", ctx.stream);
  const int64_t nunits = ntiles * (f.ldy / pa.unit_rows);
  const unsigned pgrid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nunits, ctx.num_sms));
  tsqr_product_kernel<<<pgrid, kProdNT, psmem, ctx.stream>>>(pa);
  TTB_LAUNCHED();
  ctx.free(scr);
}

void tsqr_release(Ctx& ctx, Tsqr& f) {
  if (f.t_ready) {  // the aux stream may still be writing T into mem
    TTB_CUDA(cudaStreamWaitEvent(ctx.stream, f.t_ready, 0));
    TTB_CUDA(cudaEventDestroy(f.t_ready));
    f.t_ready = nullptr;
  }
  if (f.mem) ctx.free(f.mem);
  f.mem = nullptr;
}

}  // namespace ttb

#ifdef TTB_DEBUG_TILE
extern "C" int ttb_dbg_tile(long long* out) {
  return cudaMemcpyFromSymbol(out, ttb::g_tile_clk, sizeof(long long) * 64 * 8) == cudaSuccess ? 0 : 5;
}
#endif
#ifdef TTB_DEBUG_CLK
extern "C" int ttb_dbg_clk(long long* out) {
  return cudaMemcpyFromSymbol(out, ttb::g_dclk, sizeof(long long) * 16 * 64 * 16) == cudaSuccess ? 0 : 5;
}
#endif
