// Blocked Householder TSQR leaf for bond ranks 33..64 (the tsqr_leaf kernel
// class of the rounding's orthonormalization and truncation sweeps).
//
// Same contract as tsqr_leaf_kernel (tsqr.cu): one CTA walks its slice run
// as a chain of 256-row tiles -- tile 0 a plain Householder QR (pivot rows
// 0..b-1 of the tile), tile t > 0 the QR of [R_{t-1}; A_t] -- and writes
// per tile the Householder vectors Y (unit-major layout, y_index) and the
// compact-WY factor T (Q_t = I - V T V^T), plus the CTA's final triangle R.
// The apply kernels and the tree consume exactly the same data.
// Reference: ttpar tsqr.py:103-130 (local_qr: dgeqrf of each block) and the
// stacked-triangle QR of the tree (tsqr.py:166-221).
//
// What changes is how a tile is factored.  The unblocked column pipeline
// (tile_qr_t) pays a ~2k-cycle dependency chain per column for only
// 256 x b x 4 flops of work.  Here the columns are factored in panels of 8:
//
//  * one PANEL WARP holds the 8 current columns of all 256 tile rows (8 rows
//    x 8 columns per lane) plus the 8 x 8 pivot block ([R; A]: R's rows of
//    the panel for chain tiles, the tile's own pivot rows for the head tile)
//    and factors them with warp shuffles only: per column one butterfly of
//    8 sums (the squared norm below the pivot, the 7 other columns' dots --
//    the trailing ones for the update, the finished ones for V^T V) and one
//    reflector-scalar chain.  It also forms the panel's 8 x 8 T by the
//    dlarft recurrence and writes Y_p (256 x 8) to shared memory.
//  * seven COMPUTE WARPS hold the tile (40 or 32 rows x 64 columns each) in
//    registers, TRANSPOSED, in the D-fragment layout of the fp64 MMA
//    m16n8k8 (m = column, n = row).  A D fragment of that product is, with
//    the contraction index permuted inside each 8-block (k = t <-> row 2t,
//    k = t+4 <-> row 2t+1), an A fragment of the next one, so
//      W^T = A^T Y_p        (m = column, n = reflector, k = row)
//      A^T -= W'^T Y_p^T     (m = column, n = row, k = reflector)
//    both run on the tensor pipe straight from the register tile, no
//    shuffles; per-warp W partials are summed in shared memory, and
//    W' = T_p^T W takes eight shuffles per column.  The R rows of a chain
//    tile (the E part of V = [E; Y]) are updated in shared memory.
//  * look-ahead: the update of the NEXT panel's columns runs first and
//    hands them to the panel warp, which factors panel p+1 while the compute
//    warps finish panel p's trailing update and extend the tile's T:
//      T[0:c0, p] = -T[0:c0, 0:c0] (V_{0:c0}^T V_p) T_pp,
//    the cross Gram V_{0:c0}^T V_p coming out of the same W product (the
//    register tile holds the finished V columns).
//
// Shared-memory panels use a swizzle (bsw) under which the panel warp's
// (row, column) pattern and all four MMA fragment patterns are bank-
// conflict free.
#include "ctx.cuh"
#include "prof.cuh"
#include "tsqr.cuh"

namespace ttb {

namespace lf2 {

#ifdef TTB_LF2_CLK
// debug: cycle stamps of CTA 0's first 64 panels, 8 per panel
__device__ long long g_lf2clk[64 * 8];
__device__ long long g_lf2col[64 * 12];  // panel warp: load done, after each column, after writes
#define LF2_COL(gp, slot)                                                              \
  do {                                                                                 \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && (gp) < 64) g_lf2col[(gp) * 12 + (slot)] = clock64(); \
  } while (0)
#define LF2_CLK(gp, slot)                                                               \
  do {                                                                                  \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && (gp) < 64) g_lf2clk[(gp) * 8 + (slot)] = clock64(); \
  } while (0)
#else
#define LF2_CLK(gp, slot) \
  do {                    \
  } while (0)
#define LF2_COL(gp, slot) \
  do {                    \
  } while (0)
#endif

// 8 warps in all, two per SM sub-partition, so every warp may use up to 255
// registers: seven compute warps share the 256 tile rows (warps 0-3 hold 40
// rows = 5 n8 tiles, warps 4-6 hold 32) and one panel warp
constexpr int NCW = 7;               // compute warps
constexpr int NTC = NCW * 32;        // compute threads
constexpr int NT = NTC + 32;         // + the panel warp
constexpr int MC = 256;              // tile rows
constexpr int BM = 64;               // max columns
constexpr int NMT = 4;               // m16 column tiles
constexpr int NNT_MAX = 5;           // n8 row tiles per compute warp (40 or 32 rows)
__device__ __forceinline__ int warp_rbase(int w) { return w < 4 ? 40 * w : 160 + 32 * (w - 4); }
constexpr int NB = 8;                // panel width
constexpr int WNLD = 12;             // row stride of Wneg (conflict-free A fragments)

struct Smem {
  double Rs[BM * BM];                // chain triangle R (col-major, ld 64)
  double Ts[BM * BM];                // the tile's T (col-major, ld 64; upper part valid)
  double B[2][MC * NB];              // panel in / Householder vectors out (swizzled)
  double Wpart[NCW][BM * NB];        // per-warp partials of W^T, [col][refl]
  double Wneg[BM * WNLD];            // -W'^T, [col][refl]
  double Xc[BM * NB];                // cross Gram V_k . V_{c0+i}, [k][i]
  double Xs[BM * NB];                // X = Xc T_pp, [k][j]
  double Tpp[2][NB * NB];            // panel T, row-major [i][j]
  unsigned long long ready;          // compute warps -> panel warp (a panel is in B)
  unsigned long long done;           // panel warp -> compute warps (Y_p, T_pp, R block written)
};

// swizzled (row, column) -> offset of a 256 x 8 panel in shared memory:
// slot bits (c0^r3, c1^r4, r1, r0^r2), then (c2, r2), then the 8-row block
__device__ __forceinline__ int bsw(int r, int c) {
  const int slot = ((c ^ (r >> 3)) & 3) | (((r >> 1) & 1) << 2) | (((r ^ (r >> 2)) & 1) << 3);
  const int q = ((c >> 2) & 1) | (((r >> 2) & 1) << 1);
  return (r >> 3) * 64 + q * 16 + slot;
}
// panel warp: lane l owns tile rows prow(l, s), s = 0..7
__device__ __forceinline__ int prow(int lane, int s) { return (lane >> 4) + 2 * (lane & 15) + 32 * s; }

__device__ __forceinline__ void csync() { asm volatile("bar.sync 1, %0;\n" ::"n"(NTC) : "memory"); }

__device__ __forceinline__ void mma1688(double (&d)[4], double a0, double a1, double a2, double a3, double b0,
                                        double b1) {
  asm("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
}

// ------------------------------------------------------------------------
// panel warp: QR of [P (8 x 8); A (256 x 8)] with pivots in P
// ------------------------------------------------------------------------
__device__ __forceinline__ void panel_factor(Smem& sm, double* Bp, double* Tpp, int c0, int nbp, int b, bool head,
                                             unsigned gp) {
  const int lane = threadIdx.x & 31;
  double a[8][8], pr[8], tr[8];
  // A part: head tiles exclude rows < c0 + 8 (R above, the pivot block itself)
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int r = prow(lane, s);
    const bool use = !head || r >= c0 + NB;
#pragma unroll
    for (int c = 0; c < 8; ++c) a[s][c] = use ? Bp[bsw(r, c)] : 0.0;
  }
  // pivot block rows (lanes 0..7): chain tiles R[c0+l, c0..c0+7]; head tile rows c0+l
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    double v = 0.0;
    if (lane < NB) v = head ? Bp[bsw(c0 + lane, c)] : sm.Rs[(c0 + lane) + BM * (c0 + c)];
    pr[c] = v;
    tr[c] = 0.0;
  }
  const bool plane = lane < NB;
  LF2_COL(gp, 0);
  // every lane runs all 8 column steps (no data-dependent exit around the
  // shuffles); columns past the panel width are zero and get tau = 0
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const bool act = j < nbp;
    const bool below = plane && lane > j;  // pivot-block rows below the pivot
    // partial sums: acc[j] = |x|^2 below the pivot, acc[k] = x . col k (raw x)
    double acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = 0.0;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const double x = a[s][j];
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = fma(x, a[s][k], acc[k]);
    }
    if (below) {
      const double x = pr[j];
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = fma(x, pr[k], acc[k]);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], off);
    // the pivot row (row j of the block) from lane j
    double prj[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) prj[k] = __shfl_sync(0xffffffffu, pr[k], j);
    double beta, tau, scal, bv;
    reflector_scalars<false>(prj[j], acc[j], beta, tau, scal, bv);
    if (!act) {
      tau = 0.0;
      scal = 0.0;
      beta = prj[j];
    }
    // d_k = v . a_k (k > j) and G[k][j] = v_k . v_j (k < j): the same formula
    double dd[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) dd[k] = fma(scal, acc[k], prj[k]);
    // trailing update: a_k -= tau d_k v, v = [e_j; scal x]
#pragma unroll
    for (int k = j + 1; k < 8; ++k) {
      const double cc = tau * dd[k] * scal;
#pragma unroll
      for (int s = 0; s < 8; ++s) a[s][k] = fma(-cc, a[s][j], a[s][k]);
      if (below) pr[k] = fma(-cc, pr[j], pr[k]);
      if (plane && lane == j) pr[k] = fma(-tau, dd[k], pr[k]);
    }
    // column j becomes v (R's diagonal entry beta at the pivot)
#pragma unroll
    for (int s = 0; s < 8; ++s) a[s][j] *= scal;
    if (below) pr[j] *= scal;
    if (plane && lane == j) pr[j] = beta;
    // dlarft: T[0:j, j] = -tau_j T[0:j, 0:j] G[0:j, j]; T[j][j] = tau_j (lane i holds row i)
    double sum = 0.0;
#pragma unroll
    for (int m = 0; m < j; ++m) sum = fma(tr[m], dd[m], sum);
    tr[j] = lane < j ? -tau * sum : (lane == j ? tau : 0.0);
    LF2_COL(gp, 1 + j);
  }
  // Y_p -> B (head: rows < c0 zero, pivot rows unit lower from the block)
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int r = prow(lane, s);
#pragma unroll
    for (int c = 0; c < 8; ++c) Bp[bsw(r, c)] = c < nbp ? a[s][c] : 0.0;
  }
  __syncwarp();
  if (plane) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (head) Bp[bsw(c0 + lane, c)] = (c < nbp && c <= lane) ? (c == lane ? 1.0 : pr[c]) : 0.0;
      if (c >= lane && c0 + c < b) sm.Rs[(c0 + lane) + BM * (c0 + c)] = pr[c];  // R block (upper)
      Tpp[lane * NB + c] = tr[c];
    }
  }
  LF2_COL(gp, 9);
}

// ------------------------------------------------------------------------
// compute warps
// ------------------------------------------------------------------------
struct TileIO {
  Panel P;
  int rs;
  int64_t ia;
  int nsl;
};


// registers: A[mt][nt][z], z = {(col g, row 2t), (g, 2t+1), (g+8, 2t), (g+8, 2t+1)} of the
// m16 column tile mt and the warp's n8 row tile nt
template <int NN>
__device__ __forceinline__ void load_tile(double (&A)[NMT][NN][4], const TileIO& io, int b, int rbase) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  const int rows = io.nsl * io.rs;
  const int64_t cstride = io.P.trans ? 1 : io.P.rl * io.P.I;  // column step of the view
  const double* base = io.P.base;
#pragma unroll
  for (int nt = 0; nt < NN; ++nt) {
    int64_t off[2];
    bool ok[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // one division pair per row, not per element
      const int r = rbase + nt * 8 + 2 * t4 + h;
      int si, w;
      tile_row(io.P.trans, r, io.nsl, io.rs, si, w);
      ok[h] = r < rows;
      off[h] = ok[h] ? io.P.addr(w, io.ia + si, 0) : 0;
    }
    if (io.P.kron.x) {  // implicit Hadamard core: elements formed on load
      int si0, w0, si1, w1;
      tile_row(io.P.trans, rbase + nt * 8 + 2 * t4, io.nsl, io.rs, si0, w0);
      tile_row(io.P.trans, rbase + nt * 8 + 2 * t4 + 1, io.nsl, io.rs, si1, w1);
#pragma unroll
      for (int mt = 0; mt < NMT; ++mt) {
        const int c = mt * 16 + g;
        A[mt][nt][0] = ok[0] && c < b ? io.P.load(w0, io.ia + si0, c) : 0.0;
        A[mt][nt][1] = ok[1] && c < b ? io.P.load(w1, io.ia + si1, c) : 0.0;
        A[mt][nt][2] = ok[0] && c + 8 < b ? io.P.load(w0, io.ia + si0, c + 8) : 0.0;
        A[mt][nt][3] = ok[1] && c + 8 < b ? io.P.load(w1, io.ia + si1, c + 8) : 0.0;
      }
      continue;
    }
#pragma unroll
    for (int mt = 0; mt < NMT; ++mt) {
      const int c = mt * 16 + g;
      A[mt][nt][0] = ok[0] && c < b ? __ldg(base + off[0] + cstride * c) : 0.0;
      A[mt][nt][1] = ok[1] && c < b ? __ldg(base + off[1] + cstride * c) : 0.0;
      A[mt][nt][2] = ok[0] && c + 8 < b ? __ldg(base + off[0] + cstride * (c + 8)) : 0.0;
      A[mt][nt][3] = ok[1] && c + 8 < b ? __ldg(base + off[1] + cstride * (c + 8)) : 0.0;
    }
  }
}

// panel p's columns of the register tile -> B (all 256 rows); head tiles also
// publish the finished R entries above the panel's pivot block
template <int MT, int NN>
__device__ __forceinline__ void handoff_mt(const double (&A)[NMT][NN][4], int h, double* Bn, Smem& sm, bool head,
                                           int c0, int rbase) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
#pragma unroll
  for (int nt = 0; nt < NN; ++nt) {
    const int r = rbase + nt * 8 + 2 * t4;
    const double v0 = h ? A[MT][nt][2] : A[MT][nt][0];
    const double v1 = h ? A[MT][nt][3] : A[MT][nt][1];
    Bn[bsw(r, g)] = v0;
    Bn[bsw(r + 1, g)] = v1;
    if (head) {
      if (r < c0) sm.Rs[r + BM * (c0 + g)] = v0;
      if (r + 1 < c0) sm.Rs[r + 1 + BM * (c0 + g)] = v1;
    }
  }
}

template <int NN>
__device__ __forceinline__ void handoff(const double (&A)[NMT][NN][4], int p, double* Bn, Smem& sm, bool head,
                                        int rbase) {
  const int c0 = p * NB, h = p & 1;
  switch (p >> 1) {
    case 0: handoff_mt<0, NN>(A, h, Bn, sm, head, c0, rbase); break;
    case 1: handoff_mt<1, NN>(A, h, Bn, sm, head, c0, rbase); break;
    case 2: handoff_mt<2, NN>(A, h, Bn, sm, head, c0, rbase); break;
    default: handoff_mt<3, NN>(A, h, Bn, sm, head, c0, rbase); break;
  }
}

// the factored panel (V form) back into the register tile
template <int MT, int NN>
__device__ __forceinline__ void reload_mt(double (&A)[NMT][NN][4], int h, const double* Yb, int rbase) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
#pragma unroll
  for (int nt = 0; nt < NN; ++nt) {
    const int r = rbase + nt * 8 + 2 * t4;
    const double v0 = Yb[bsw(r, g)], v1 = Yb[bsw(r + 1, g)];
    if (h) {
      A[MT][nt][2] = v0;
      A[MT][nt][3] = v1;
    } else {
      A[MT][nt][0] = v0;
      A[MT][nt][1] = v1;
    }
  }
}

template <int NN>
__device__ __forceinline__ void reload(double (&A)[NMT][NN][4], int p, const double* Yb, int rbase) {
  const int h = p & 1;
  switch (p >> 1) {
    case 0: reload_mt<0, NN>(A, h, Yb, rbase); break;
    case 1: reload_mt<1, NN>(A, h, Yb, rbase); break;
    case 2: reload_mt<2, NN>(A, h, Yb, rbase); break;
    default: reload_mt<3, NN>(A, h, Yb, rbase); break;
  }
}

// W^T partial of m-tile MT over this warp's rows -> sm.Wpart[warp]
template <int MT, int NN>
__device__ __forceinline__ void wpart_mt(const double (&A)[NMT][NN][4], const double (&yw)[NN][2], Smem& sm) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, g = lane >> 2, t4 = lane & 3;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int nt = 0; nt < NN; ++nt)
    mma1688(acc, A[MT][nt][0], A[MT][nt][2], A[MT][nt][1], A[MT][nt][3], yw[nt][0], yw[nt][1]);
  double* wp = sm.Wpart[w];
  *reinterpret_cast<double2*>(&wp[(MT * 16 + g) * NB + 2 * t4]) = make_double2(acc[0], acc[1]);
  *reinterpret_cast<double2*>(&wp[(MT * 16 + g + 8) * NB + 2 * t4]) = make_double2(acc[2], acc[3]);
}

// A^T[m-tile MT] += Wneg^T-fragment x Y_p^T
template <int MT, int NN>
__device__ __forceinline__ void update_mt(double (&A)[NMT][NN][4], const double (&yu)[NN][2], const Smem& sm) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  const double* wn = sm.Wneg;
  const double a0 = wn[(MT * 16 + g) * WNLD + t4], a1 = wn[(MT * 16 + g + 8) * WNLD + t4];
  const double a2 = wn[(MT * 16 + g) * WNLD + t4 + 4], a3 = wn[(MT * 16 + g + 8) * WNLD + t4 + 4];
#pragma unroll
  for (int nt = 0; nt < NN; ++nt) mma1688(A[MT][nt], a0, a1, a2, a3, yu[nt][0], yu[nt][1]);
}

// dispatch a per-m-tile routine over a mask of m-tiles
#define LF2_FOR_MT(mask, CALL)    \
  do {                            \
    if ((mask) & 1) CALL(0);      \
    if ((mask) & 2) CALL(1);      \
    if ((mask) & 4) CALL(2);      \
    if ((mask) & 8) CALL(3);      \
  } while (0)

// Reduce the W partials of column k (one 8-lane group per column, lane j =
// reflector j), then W' = T_pp^T W by shuffles.  Returns raw (tile rows only)
// in *raw and W' (R rows included for chain tiles) as the result.
__device__ __forceinline__ double reduce_col(const Smem& sm, const double* Tp, int k, int j, int c0, bool head,
                                             double& raw) {
  double wsum = 0.0;
#pragma unroll
  for (int w = 0; w < NCW; ++w) wsum += sm.Wpart[w][k * NB + j];
  raw = wsum;
  double wv = wsum;
  if (!head && k >= c0 + NB) wv += sm.Rs[(c0 + j) + BM * k];
  const int lane = threadIdx.x & 31, base = lane & ~7;
  double out = 0.0;
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const double wi = __shfl_sync(0xffffffffu, wv, base + i);
    out = fma(Tp[i * NB + j], wi, out);  // Tp upper: zero for i > j
  }
  return out;
}

}  // namespace lf2

using namespace lf2;

template <int NN>
__device__ __forceinline__ void compute_role(Smem& sm, const Panel& P, const LeafPlan& plan, double* __restrict__ Yg,
                                             double* __restrict__ Tg, int rbase) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int gcta = blockIdx.x;
  const int b = plan.b, rs = plan.rs, ni = plan.ni;
  const int np = (b + NB - 1) / NB;
  const int64_t n_g = plan.count(gcta), s0 = plan.start(gcta);
  const int ntiles = plan.tiles_of(n_g);
  const int64_t tb = plan.tile_base(gcta);
    const int g = lane >> 2, t4 = lane & 3;
    double A[NMT][NN][4];
    unsigned gp = 0;
    for (int t = 0; t < ntiles; ++t) {
      const bool head = t == 0;
      TileIO io;
      io.P = P;
      io.rs = rs;
      io.ia = s0 + (int64_t)t * ni;
      io.nsl = (int)min64(ni, n_g - (int64_t)t * ni);
      load_tile<NN>(A, io, b, rbase);
      handoff<NN>(A, 0, sm.B[gp & 1], sm, head, rbase);
      csync();
      if (tid == 0) mbar_arrive(&sm.ready);
      for (int p = 0; p < np; ++p, ++gp) {
        const int c0 = p * NB;
        const bool has_next = p + 1 < np;
        const int mt1 = has_next ? (p + 1) >> 1 : -1;
        if (threadIdx.x == 0) LF2_CLK(gp, 3);
        mbar_wait(&sm.done, gp & 1);
        if (threadIdx.x == 0) LF2_CLK(gp, 4);
        const double* Yb = sm.B[gp & 1];
        const double* Tp = sm.Tpp[gp & 1];
        reload<NN>(A, p, Yb, rbase);
        double yw[NN][2], yu[NN][2];
#pragma unroll
        for (int nt = 0; nt < NN; ++nt) {
          const int r = rbase + nt * 8;
          yw[nt][0] = Yb[bsw(r + 2 * t4, g)];
          yw[nt][1] = Yb[bsw(r + 2 * t4 + 1, g)];
          yu[nt][0] = Yb[bsw(r + g, t4)];
          yu[nt][1] = Yb[bsw(r + g, t4 + 4)];
        }
        // ---- critical path: the next panel's columns ----
        if (has_next) {
#define LF2_W(MT) wpart_mt<MT, NN>(A, yw, sm)
          LF2_FOR_MT(1 << mt1, LF2_W);
          csync();
          {  // 128 (column, reflector) items; threads >= 128 recompute 0..95 and store nothing
            const int item = tid & 127;
            const int k = mt1 * 16 + (item >> 3), j = item & 7;
            double raw;
            const double wv = reduce_col(sm, Tp, k, j, c0, head, raw);
            const bool upd = k >= c0 + NB && k < b;  // panel p+1 (and p+2 when they share the m-tile)
            if (tid < 128) {
              sm.Wneg[k * WNLD + j] = upd ? -wv : 0.0;
              if (!head && upd) sm.Rs[(c0 + j) + BM * k] -= wv;
            }
          }
          csync();
#define LF2_U(MT) update_mt<MT, NN>(A, yu, sm)
          LF2_FOR_MT(1 << mt1, LF2_U);
          handoff<NN>(A, p + 1, sm.B[(gp + 1) & 1], sm, head, rbase);
          csync();
          if (tid == 0) LF2_CLK(gp, 5);
          if (tid == 0) mbar_arrive(&sm.ready);
        }
        // ---- the rest: trailing columns, cross Gram ----
        const unsigned all = (1u << NMT) - 1;
        const unsigned rest = has_next ? (all & ~(1u << mt1)) : all;
#ifndef LF2_DBG_NOREST
        LF2_FOR_MT(rest, LF2_W);
#endif
        csync();
#pragma unroll
        for (int rnd = 0; rnd < (BM * NB + NTC - 1) / NTC; ++rnd) {  // uniform trip count (shuffles inside)
          const int it0 = tid + rnd * NTC;
          const int it = it0 & (BM * NB - 1);
          const int k = it >> 3, j = it & 7;
          double raw;
          const double wv = reduce_col(sm, Tp, k, j, c0, head, raw);
          if (it0 < BM * NB && !(has_next && (k >> 4) == mt1)) {
            const bool upd = k >= c0 + NB && k < b;
            if (k < c0) sm.Xc[k * NB + j] = raw;
            sm.Wneg[k * WNLD + j] = upd ? -wv : 0.0;
            if (!head && upd) sm.Rs[(c0 + j) + BM * k] -= wv;
          }
        }
        csync();
        // m-tiles holding trailing columns (>= c0 + 8), except the critical one
        const int first_tr = (c0 + NB) >> 4;
        unsigned trail = 0;
        for (int mt = first_tr; mt < NMT; ++mt)
          if (mt * 16 < b) trail |= 1u << mt;
        trail &= rest;
#ifndef LF2_DBG_NOREST
        LF2_FOR_MT(trail, LF2_U);
#endif
#undef LF2_W
#undef LF2_U
        // ---- T: diagonal block, then T[0:c0, p] = -T[0:c0, 0:c0] (Xc T_pp) ----
#ifndef LF2_DBG_NOT
        for (int it = tid; it < NB * NB; it += NTC) {
          const int i = it >> 3, j = it & 7;
          sm.Ts[(c0 + i) + BM * (c0 + j)] = Tp[i * NB + j];
        }
        for (int it = tid; it < c0 * NB; it += NTC) {
          const int k = it >> 3, j = it & 7;
          double x = 0.0;
#pragma unroll
          for (int i = 0; i < NB; ++i) x = fma(sm.Xc[k * NB + i], Tp[i * NB + j], x);
          sm.Xs[k * NB + j] = x;
        }
        csync();
        for (int it = tid; it < c0 * NB; it += NTC) {
          const int m = it >> 3, j = it & 7;
          double x = 0.0;
          for (int k = m; k < c0; ++k) x = fma(sm.Ts[m + BM * k], sm.Xs[k * NB + j], x);
          sm.Ts[m + BM * (c0 + j)] = -x;
        }
#endif
        if (tid == 0) LF2_CLK(gp, 6);
      }
      csync();
      // ---- tile outputs: Y (unit-major), T ----
      const int64_t tile = tb + t;
      double* Yt = Yg + tile * y_tile_stride(MC, b);
#pragma unroll
      for (int mt = 0; mt < NMT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NN; ++nt) {
          const int r = rbase + nt * 8 + 2 * t4;
          const int c = mt * 16 + g;
          if (c < b) *reinterpret_cast<double2*>(&Yt[y_index(r, c, b)]) = make_double2(A[mt][nt][0], A[mt][nt][1]);
          if (c + 8 < b)
            *reinterpret_cast<double2*>(&Yt[y_index(r, c + 8, b)]) = make_double2(A[mt][nt][2], A[mt][nt][3]);
        }
      double* Tt = Tg + tile * (((int64_t)b * b + 1) & ~1LL);
      for (int idx = tid; idx < b * b; idx += NTC) {
        const int k = idx % b, j = idx / b;
        Tt[idx] = k <= j ? sm.Ts[k + BM * j] : 0.0;
      }
    }
}

__global__ void __launch_bounds__(lf2::NT, 1)
tsqr_leaf2_kernel(Panel P, LeafPlan plan, double* __restrict__ Yg, double* __restrict__ Tg,
                  double* __restrict__ Rleaf) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gcta = blockIdx.x;
  const int b = plan.b, rs = plan.rs, ni = plan.ni;
  const int np = (b + NB - 1) / NB;
  const int64_t n_g = plan.count(gcta), s0 = plan.start(gcta);
  const int ntiles = plan.tiles_of(n_g);
  const int64_t tb = plan.tile_base(gcta);
  for (int idx = tid; idx < BM * BM; idx += NT) sm.Rs[idx] = 0.0;
  if (tid == 0) {
    mbar_init(&sm.ready, 1);
    mbar_init(&sm.done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == NCW) {
    // ---------------- panel warp ----------------
    unsigned gp = 0;
    for (int t = 0; t < ntiles; ++t) {
      const bool head = t == 0;
      for (int p = 0; p < np; ++p, ++gp) {
        const int c0 = p * NB, nbp = min(NB, b - c0);
        LF2_CLK(gp, 0);
        mbar_wait(&sm.ready, gp & 1);
        LF2_CLK(gp, 1);
        panel_factor(sm, sm.B[gp & 1], sm.Tpp[gp & 1], c0, nbp, b, head, gp);
        __syncwarp();
        LF2_CLK(gp, 2);
        if (lane == 0) mbar_arrive(&sm.done);
      }
    }
  } else if (warp < 4) {
    compute_role<5>(sm, P, plan, Yg, Tg, warp_rbase(warp));
  } else {
    compute_role<4>(sm, P, plan, Yg, Tg, warp_rbase(warp));
  }
  __syncthreads();
  for (int idx = tid; idx < b * b; idx += NT) {
    const int r = idx % b, k = idx / b;
    Rleaf[(int64_t)gcta * b * b + idx] = r <= k ? sm.Rs[r + BM * k] : 0.0;
  }
}

size_t leaf2_smem() { return sizeof(lf2::Smem); }

#ifdef TTB_LF2_CLK
extern "C" int ttb_dbg_lf2clk(long long* out) {
  return cudaMemcpyFromSymbol(out, lf2::g_lf2clk, sizeof(long long) * 64 * 8) == cudaSuccess ? 0 : 5;
}
extern "C" int ttb_dbg_lf2col(long long* out) {
  return cudaMemcpyFromSymbol(out, lf2::g_lf2col, sizeof(long long) * 64 * 12) == cudaSuccess ? 0 : 5;
}
#endif

void launch_leaf2(Ctx& ctx, const Panel& panel, const LeafPlan& plan, double* Y, double* T, double* Rleaf) {
  smem_attr((const void*)tsqr_leaf2_kernel, sizeof(lf2::Smem));
  tsqr_leaf2_kernel<<<plan.G, lf2::NT, sizeof(lf2::Smem), ctx.stream>>>(panel, plan, Y, T, Rleaf);
  TTB_LAUNCHED();
}

}  // namespace ttb
