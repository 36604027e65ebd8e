// TSQR kernels (leaf chain, tree nodes, apply) and the host-side factor object.
// See tsqr.cuh for the decomposition.  Reference: ttpar tsqr.py:103-327.
#include "tsqr.cuh"
#include "ctx.cuh"

namespace ttb {

// ------------------------------------------------------------------------
// leaf kernel: one CTA = one chain of tiles over a contiguous slice run
// ------------------------------------------------------------------------
template <class C>
__global__ void __launch_bounds__(C::NT, (C::NT <= 256 ? 2 : 1))
tsqr_leaf_kernel(Panel P, LeafPlan plan, double* __restrict__ Yg, double* __restrict__ Tg,
                 double* __restrict__ Rleaf) {
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
  for (int t = 0; t < ntiles; ++t) {
    const int64_t ia = s0 + (int64_t)t * ni;
    const int nsl = (int)min64(ni, n_g - (int64_t)t * ni);
    const int rows = nsl * rs;
    // load (zero padded)
#pragma unroll
    for (int s = 0; s < C::RPL; ++s) {
      const int r = s * C::LR + lr;
      int si, w;
      tile_row(P.trans, r, nsl, rs, si, w);
#pragma unroll
      for (int u = 0; u < C::CPL; ++u) {
        const int k = col_of<C>(u, warp, lc);
        A[s][u] = (r < rows && k < b) ? P.base[P.addr(w, ia + si, k)] : 0.0;
      }
    }
    zero_G<C>(sm);
    __syncthreads();
    const bool head = (t == 0);
    tile_qr<C>(A, b, head, sm);
    const int64_t tile = tb + t;
    store_Y<C>(A, b, head, Yg + tile * (int64_t)C::MC * b, C::MC);
    store_T<C>(sm, b, Tg + tile * (int64_t)b * b);
    if (head) extract_R<C>(A, b, sm);
    __syncthreads();
  }
  for (int idx = threadIdx.x; idx < b * b; idx += C::NT) {
    const int r = idx % b, k = idx / b;
    Rleaf[(int64_t)g * b * b + idx] = sm.Rs[r + C::BMAX * k];
  }
}

// ------------------------------------------------------------------------
// tree kernel: node q factors the stacked triangles Rin[q*f .. q*f+cnt)
// ------------------------------------------------------------------------
template <class C>
__global__ void __launch_bounds__(C::NT, 1)
tsqr_tree_kernel(const double* __restrict__ Rin, int n_in, int b, int f, double* __restrict__ Yn,
                 double* __restrict__ Tn, double* __restrict__ Rout) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TileSmem<C>& sm = *reinterpret_cast<TileSmem<C>*>(smem_raw);
  const int q = blockIdx.x;
  const int c0 = q * f, cnt = min(f, n_in - c0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lc = lane / C::LR, lr = lane % C::LR;
  double A[C::RPL][C::CPL];
#pragma unroll
  for (int s = 0; s < C::RPL; ++s) {
    const int r = s * C::LR + lr;
    const int ch = r / b, rr = r - ch * b;
#pragma unroll
    for (int u = 0; u < C::CPL; ++u) {
      const int k = col_of<C>(u, warp, lc);
      A[s][u] = (ch < cnt && k < b) ? Rin[(int64_t)(c0 + ch) * b * b + rr + (int64_t)b * k] : 0.0;
    }
  }
  zero_G<C>(sm);
  __syncthreads();
  tile_qr<C>(A, b, true, sm);
  store_Y<C>(A, b, true, Yn + (int64_t)q * C::MC * b, C::MC);
  store_T<C>(sm, b, Tn + (int64_t)q * b * b);
  extract_R<C>(A, b, sm);
  __syncthreads();
  for (int idx = threadIdx.x; idx < b * b; idx += C::NT) {
    const int r = idx % b, k = idx / b;
    Rout[(int64_t)q * b * b + idx] = sm.Rs[r + C::BMAX * k];
  }
}

// sign fix: D = sign(diag R) (0 -> +1), Rout = D R (upper), both device
__global__ void sign_fix_kernel(const double* __restrict__ R, int b, double* __restrict__ D,
                                double* __restrict__ Rout) {
  for (int idx = threadIdx.x; idx < b * b; idx += blockDim.x) {
    const int r = idx % b, k = idx / b;
    const double dr = R[r + b * r] < 0.0 ? -1.0 : 1.0;
    Rout[idx] = (r <= k) ? dr * R[idx] : 0.0;
    if (k == 0) D[r] = dr;
  }
}

// ------------------------------------------------------------------------
// apply kernel: out(rows of this CTA) = Q [D z0; 0]
// ------------------------------------------------------------------------
constexpr int kApplyNT = 256;
constexpr int kApplyBM = 64;   // max b
constexpr int kApplyKM = 64;   // max k
constexpr int kApplyCW = 16;   // output columns per thread pass

struct ApplyArgs {
  LeafPlan plan;
  int ldy;                     // leaf tile rows (MC of the leaf config)
  const double* Y;
  const double* T;
  TreeDesc local;              // levels above the CTA leaves, lev[0] lowest
  TreeDesc global;             // levels above the rank roots (multi-GPU), lev[0] lowest
  int rank;
  const double* z0;            // b x k, col-major, ld b
  int k;
  const double* D;             // b signs or nullptr
  Panel out;                   // output view with k columns
};

struct ApplySmem {
  double Z[kApplyBM * kApplyKM];
  double W[kApplyBM * kApplyKM];
  double U[kApplyBM * kApplyKM];
};

// S_out[i, c] = sum_l M(i, l) * S_in[l, c],  M(i,l) = trans ? Mg[l + ld*i] : Mg[i + ld*l]
// lo_tri != 0: M(i, l) vanishes for l < i (T upper, V_top^T upper)
__device__ __forceinline__ void small_gemm(const double* __restrict__ Mg, int ld, bool trans, int lo_tri,
                                           const double* Sin, double* Sout, int b, int k) {
  for (int idx = threadIdx.x; idx < b * k; idx += kApplyNT) {
    const int i = idx % b, c = idx / b;
    double acc = 0.0;
    const int l0 = lo_tri ? i : 0, l1 = b;  // triangular operands: l >= i
    for (int l = l0; l < l1; ++l) {
      const double m = trans ? Mg[l + (int64_t)ld * i] : Mg[i + (int64_t)ld * l];
      acc = fma(m, Sin[l + kApplyBM * c], acc);
    }
    Sout[i + kApplyBM * c] = acc;
  }
}

// One tree level: z <- rows of child c of Q_node [z; 0]
__device__ void apply_node(ApplySmem& sm, const Level& L, int q, int c, int b, int k) {
  const double* Y = L.Y + (int64_t)q * L.ldy * b;
  const double* T = L.T + (int64_t)q * b * b;
  // W = V_top^T Z   (V_top unit lower triangular: V_top^T upper)
  small_gemm(Y, L.ldy, true, 2, sm.Z, sm.W, b, k);
  __syncthreads();
  small_gemm(T, b, false, 1, sm.W, sm.U, b, k);   // U = T W
  __syncthreads();
  // Z <- [Z;0]_child - V_child U
  const double* Vc = Y + (int64_t)c * b;
  for (int idx = threadIdx.x; idx < b * k; idx += kApplyNT) {
    const int i = idx % b, cc = idx / b;
    double acc = (c == 0) ? sm.Z[i + kApplyBM * cc] : 0.0;
    for (int l = 0; l < b; ++l) acc = fma(-Vc[i + (int64_t)L.ldy * l], sm.U[l + kApplyBM * cc], acc);
    sm.W[i + kApplyBM * cc] = acc;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < b * k; idx += kApplyNT) {
    const int i = idx % b, cc = idx / b;
    sm.Z[i + kApplyBM * cc] = sm.W[i + kApplyBM * cc];
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kApplyNT, 2) tsqr_apply_kernel(ApplyArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ApplySmem& sm = *reinterpret_cast<ApplySmem*>(smem_raw);
  const int g = blockIdx.x;
  const LeafPlan& pl = a.plan;
  const int b = pl.b, k = a.k, rs = pl.rs, ni = pl.ni, ldy = a.ldy;
  for (int idx = threadIdx.x; idx < b * k; idx += kApplyNT) {
    const int i = idx % b, c = idx / b;
    const double d = a.D ? a.D[i] : 1.0;
    sm.Z[i + kApplyBM * c] = d * a.z0[i + (int64_t)b * c];
  }
  __syncthreads();
  // global levels (identical on every rank), top-down, leaf index = rank
  for (int L = a.global.nlev - 1; L >= 0; --L) {
    const Level& lv = a.global.lev[L];
    int x = a.rank;
    for (int u = 0; u < L; ++u) x /= lv.f;
    apply_node(sm, lv, x / lv.f, x % lv.f, b, k);
  }
  // local levels, leaf index = CTA
  for (int L = a.local.nlev - 1; L >= 0; --L) {
    const Level& lv = a.local.lev[L];
    int x = g;
    for (int u = 0; u < L; ++u) x /= lv.f;
    apply_node(sm, lv, x / lv.f, x % lv.f, b, k);
  }
  // chain, last tile first
  const int64_t n_g = pl.count(g), s0 = pl.start(g);
  const int ntiles = pl.tiles_of(n_g);
  const int64_t tb = pl.tile_base(g);
  for (int t = ntiles - 1; t >= 0; --t) {
    const int64_t tile = tb + t;
    const double* Y = a.Y + tile * (int64_t)ldy * b;
    const double* T = a.T + tile * (int64_t)b * b;
    const bool head = (t == 0);
    if (head) {
      small_gemm(Y, ldy, true, 2, sm.Z, sm.W, b, k);  // W = V_top^T Z
      __syncthreads();
      small_gemm(T, b, false, 1, sm.W, sm.U, b, k);   // U = T W
    } else {
      small_gemm(T, b, false, 1, sm.Z, sm.U, b, k);   // U = T Z
    }
    __syncthreads();
    const int64_t ia = s0 + (int64_t)t * ni;
    const int nsl = (int)min64(ni, n_g - (int64_t)t * ni);
    const int rows = nsl * rs;
    const int ncg = (k + kApplyCW - 1) / kApplyCW;
    for (int idx = threadIdx.x; idx < ldy * ncg; idx += kApplyNT) {
      const int r = idx % ldy, cg = idx / ldy;
      if (r >= rows) continue;
      const int c0 = cg * kApplyCW;
      const int nc = min(kApplyCW, k - c0);
      double acc[kApplyCW];
#pragma unroll
      for (int cc = 0; cc < kApplyCW; ++cc)
        acc[cc] = (head && r < b && cc < nc) ? sm.Z[r + kApplyBM * (c0 + cc)] : 0.0;
      for (int l = 0; l < b; ++l) {
        const double y = Y[r + (int64_t)ldy * l];
#pragma unroll
        for (int cc = 0; cc < kApplyCW; ++cc)
          if (cc < nc) acc[cc] = fma(-y, sm.U[l + kApplyBM * (c0 + cc)], acc[cc]);
      }
      int si, w;
      tile_row(a.out.trans, r, nsl, rs, si, w);
#pragma unroll
      for (int cc = 0; cc < kApplyCW; ++cc)
        if (cc < nc) a.out.base[a.out.addr(w, ia + si, c0 + cc)] = acc[cc];
    }
    if (!head) {
      for (int idx = threadIdx.x; idx < b * k; idx += kApplyNT) {
        const int i = idx % b, c = idx / b;
        sm.Z[i + kApplyBM * c] -= sm.U[i + kApplyBM * c];
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------
namespace {

template <class C>
size_t tile_smem() { return sizeof(TileSmem<C>); }

template <class C>
void set_smem_attr(const void* fn) {
  static bool done = false;  // per instantiation
  if (!done) {
    TTB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(TileSmem<C>)));
    done = true;
  }
}

template <class LC_, class TC_>
void run_factor(Ctx& ctx, Tsqr& f) {
  cudaStream_t st = ctx.stream;
  auto leaf = tsqr_leaf_kernel<LC_>;
  set_smem_attr<LC_>((const void*)leaf);
  leaf<<<f.plan.G, LC_::NT, tile_smem<LC_>(), st>>>(f.panel, f.plan, f.Y, f.T, f.Rleaf);
  TTB_LAUNCHED();
  auto tree = tsqr_tree_kernel<TC_>;
  set_smem_attr<TC_>((const void*)tree);
  const double* rin = f.Rleaf;
  int n_in = f.plan.G;
  for (int L = 0; L < f.nloc; ++L) {
    int nodes = (n_in + f.ftree - 1) / f.ftree;
    tree<<<nodes, TC_::NT, tile_smem<TC_>(), st>>>(rin, n_in, f.b, f.ftree, f.locY[L], f.locT[L], f.locR[L]);
    TTB_LAUNCHED();
    rin = f.locR[L];
    n_in = nodes;
  }
  f.Rlocal = (f.nloc > 0) ? f.locR[f.nloc - 1] : f.Rleaf;
  if (ctx.nranks > 1) {
    // allgather the rank roots, then a redundant (bitwise identical) tree
    ctx.allgather(f.Rlocal, f.Rstack, (size_t)f.b * f.b);
    rin = f.Rstack;
    n_in = ctx.nranks;
    for (int L = 0; L < f.nglob; ++L) {
      int nodes = (n_in + f.ftree - 1) / f.ftree;
      tree<<<nodes, TC_::NT, tile_smem<TC_>(), st>>>(rin, n_in, f.b, f.ftree, f.gloY[L], f.gloT[L], f.gloR[L]);
      TTB_LAUNCHED();
      rin = f.gloR[L];
      n_in = nodes;
    }
    f.Rraw = rin;
  } else {
    f.Rraw = f.Rlocal;
  }
  sign_fix_kernel<<<1, 256, 0, st>>>(f.Rraw, f.b, f.D, f.R);
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
  const int b = (int)panel.ncols();
  const int64_t rs = panel.rs();
  f.b = b;
  f.panel = panel;
  f.cls = tsqr_class(b);
  TTB_CHECK(b >= 1, TTB_ERR_SHAPE, "TSQR needs at least one column");
  TTB_CHECK(f.cls != 0, TTB_ERR_CAPABILITY, "TSQR: column count " + std::to_string(b) + " exceeds 64");
  const int MC = leaf_mc(f.cls), MT = tree_mc(f.cls);
  TTB_CHECK(rs >= 1 && rs <= MC - b + 1, TTB_ERR_CAPABILITY,
            "TSQR: rows per slice " + std::to_string(rs) + " too large for the tile (" + std::to_string(MC) + ")");
  const int64_t ns = panel.I;
  f.plan.nslices = ns;
  f.plan.rs = (int)rs;
  f.plan.b = b;
  f.plan.ni = (int)(MC / rs);
  // CTAs: at most 2 per SM; every CTA gets >= 2 tiles of rows, so small
  // panels are one chain (one head tile = the reference's single dgeqrf
  // pivot order) and the head tile always reaches b rows.
  const int64_t min_sl = std::max<int64_t>((b + rs - 1) / rs, 2 * (int64_t)f.plan.ni);
  int64_t gmax = ns >= min_sl ? ns / min_sl : 1;
  int G = (int)std::min<int64_t>((int64_t)2 * ctx.num_sms, std::max<int64_t>(1, gmax));
  if (ns == 0) G = 1;
  f.plan.G = G;
  f.ftree = MT / b;
  f.ldy = MC;
  f.ldy_tree = MT;
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
  size_t oY = add(ntiles * MC * b), oT = add(ntiles * bb), oRl = add((int64_t)G * bb);
  size_t oLY[kMaxLevels], oLT[kMaxLevels], oLR[kMaxLevels];
  for (int L = 0; L < f.nloc; ++L) {
    oLY[L] = add((int64_t)nodes_loc[L] * MT * b);
    oLT[L] = add((int64_t)nodes_loc[L] * bb);
    oLR[L] = add((int64_t)nodes_loc[L] * bb);
  }
  size_t oGS = add((int64_t)ctx.nranks * bb);
  size_t oGY[kMaxLevels], oGT[kMaxLevels], oGR[kMaxLevels];
  for (int L = 0; L < f.nglob; ++L) {
    oGY[L] = add((int64_t)nodes_glo[L] * MT * b);
    oGT[L] = add((int64_t)nodes_glo[L] * bb);
    oGR[L] = add((int64_t)nodes_glo[L] * bb);
  }
  size_t oD = add(b), oR = add(bb);
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
  if (f.cls == 16) run_factor<Leaf16, Tree16>(ctx, f);
  else if (f.cls == 32) run_factor<Leaf32, Tree32>(ctx, f);
  else run_factor<Leaf64, Tree64>(ctx, f);
}

void tsqr_apply(Ctx& ctx, const Tsqr& f, const double* z, int k, const Panel& out) {
  TTB_CHECK(k >= 1 && k <= kApplyKM, TTB_ERR_CAPABILITY, "TSQR apply: k must be in [1, 64]");
  TTB_CHECK(out.rs() == f.plan.rs && out.I == f.plan.nslices && out.ncols() == k, TTB_ERR_SHAPE,
            "TSQR apply: output view does not match the factored panel");
  ApplyArgs a;
  a.plan = f.plan;
  a.ldy = f.ldy;
  a.Y = f.Y;
  a.T = f.T;
  a.local.nlev = f.nloc;
  for (int L = 0; L < f.nloc; ++L) a.local.lev[L] = Level{f.locY[L], f.locT[L], f.ldy_tree, f.ftree, -1};
  a.global.nlev = ctx.nranks > 1 ? f.nglob : 0;
  for (int L = 0; L < a.global.nlev; ++L) a.global.lev[L] = Level{f.gloY[L], f.gloT[L], f.ldy_tree, f.ftree, -1};
  a.rank = ctx.rank;
  a.z0 = z;
  a.k = k;
  a.D = f.D;
  a.out = out;
  static bool attr = false;
  if (!attr) {
    TTB_CUDA(cudaFuncSetAttribute(tsqr_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(ApplySmem)));
    attr = true;
  }
  tsqr_apply_kernel<<<f.plan.G, kApplyNT, sizeof(ApplySmem), ctx.stream>>>(a);
  TTB_LAUNCHED();
}

void tsqr_release(Ctx& ctx, Tsqr& f) {
  if (f.mem) ctx.free(f.mem);
  f.mem = nullptr;
}

}  // namespace ttb
