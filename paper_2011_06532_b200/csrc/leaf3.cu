// Row-distributed blocked Householder TSQR leaf for bond ranks 33..64.
//
// Same contract as tsqr_leaf_kernel (tsqr.cu): one CTA walks its slice run
// as a chain of 256-row tiles -- tile 0 a plain Householder QR (pivot rows
// 0..b-1 of the tile), tile t > 0 the QR of [R_{t-1}; A_t] -- and writes per
// tile the Householder vectors Y (unit-major layout, y_index) and the
// compact-WY factor T (Q_t = I - V T V^T), plus the CTA's final triangle R.
// The tree and the apply kernels consume exactly the same data.
// Reference: ttpar tsqr.py:103-130 (local_qr: dgeqrf of each block) and the
// stacked-triangle QR of the tree (tsqr.py:166-221).
//
// The column pipeline of tile_qr_t hands every column from warp to warp
// through shared-memory rings (two mbarrier hand-offs, a sigma reduction and
// a reciprocal chain per column: ~1.7k cycles per column step, DESIGN 3.5).
// Here the tile is distributed by ROWS: eight warps hold 32 rows x 64 columns
// each, transposed, in the accumulator-fragment layout of the fp64 MMA
// m16n8k8 (m = column, n = row).  Columns are factored in panels of 8:
//
//  * a column step is ONE CTA-wide reduction: every lane multiplies its rows
//    of the pivot column x_j (fetched from the owning lanes by shuffles) with
//    its own panel column, two shuffle rounds sum the warp's rows, the eight
//    per-warp partials of the eight panel columns meet in shared memory at one
//    barrier, and every thread derives the same reflector scalars from the
//    same sums (sig = x_j . x_j; d_k = R[j,k] + scal x_j . a_k serves the
//    update for k > j and is the Gram entry v_k . v_j for k < j);
//  * the trailing update runs on the tensor pipe straight from the register
//    tile (an accumulator fragment of one product is, with the contraction
//    index permuted inside each 8-block, an A fragment of the next):
//      W^T = A^T V_p (m = column, n = reflector, k = row), summed over warps
//      in shared memory, W' = T_pp^T W by shuffles, A^T -= W'^T V_p^T;
//    the same W product over the finished columns yields the cross Gram
//    V_k . V_p that the tile's T needs, so T = (diag(1/tau) + striu(V^T V))^-1
//    is formed once per tile by build_T (tsqr.cuh).
#include "ctx.cuh"
#include "prof.cuh"
#include "tsqr.cuh"

namespace ttb {

namespace lf3 {

#ifdef TTB_LF3_CLK
// debug: cycle stamps of CTA 0, thread 0: per tile 8 phase slots
__device__ long long g_lf3clk[64 * 16];
#define LF3_CLK(t, slot)                                                                    \
  do {                                                                                      \
    if (blockIdx.x == 0 && threadIdx.x == 0 && (t) < 64) g_lf3clk[(t) * 16 + (slot)] = clock64(); \
  } while (0)
// phase accumulators over the panels of a tile (slots 10..13)
#define LF3_ACC_BEGIN() long long lf3_t0 = clock64()
#define LF3_ACC(t, slot)                                                                    \
  do {                                                                                      \
    const long long lf3_t1 = clock64();                                                     \
    if (blockIdx.x == 0 && threadIdx.x == 0 && (t) < 64) g_lf3clk[(t) * 16 + (slot)] += lf3_t1 - lf3_t0; \
    lf3_t0 = lf3_t1;                                                                        \
  } while (0)
// fine stamps of one column step (body tiles, panel 2, step 3): slots of row 60
#define LF3_STEP(slot)                                                                                  \
  do {                                                                                                  \
    if (!HEAD && blockIdx.x == 0 && threadIdx.x == 0 && c0 == 16 && j == 3) g_lf3clk[60 * 16 + (slot)] = clock64(); \
  } while (0)
#else
#define LF3_STEP(slot) \
  do {                 \
  } while (0)
#define LF3_ACC_BEGIN() \
  do {                  \
  } while (0)
#define LF3_ACC(t, slot) \
  do {                   \
  } while (0)
#define LF3_CLK(t, slot) \
  do {                   \
  } while (0)
#endif

constexpr int NW = 8;          // warps, 32 tile rows each
constexpr int NT = NW * 32;
constexpr int MC = 256;        // tile rows
constexpr int BM = 64;         // max columns
constexpr int NMT = 4;         // m16 column tiles
constexpr int NN = 4;          // n8 row tiles per warp
constexpr int NB = 8;          // panel width
constexpr int WNLD = 12;       // row stride of Wneg (conflict-free A fragments)
// T formed inside the leaf (cross Gram from the W product + build_T); off: the
// tile's T is formed from the stored Y by tile_T_kernel, outside the chain
#ifdef TTB_LF3_NOT
constexpr bool kInT = false;
#else
constexpr bool kInT = true;
#endif

struct Cfg {
  static constexpr int NT = lf3::NT, BMAX = BM;
  __device__ __forceinline__ static void sync() { __syncthreads(); }
};

struct Smem {
  double Rs[BM * BM];          // chain triangle R (col-major, ld 64)
  double Gs[BM * BM];          // striu(V^T V) -> T (build_T)
  double Xs[BM * BM / 2];      // build_T scratch
  double taus[BM];
  double Yb[MC * NB];          // the factored panel V_p (swizzled, bsw)
  double Wpart[NW][BM * NB];   // per-warp partials of W^T, [col][refl]
  double Wneg[BM * WNLD];      // -W'^T, [col][refl]
  double part[2][NW][NB];  // per-warp column sums of a step, [buf][warp][col]
  double pvs[2][NB];           // head tiles: the pivot row of the step
  double Tpp[NB * NB];         // panel T, row-major [i][j]
};

// swizzled (row, column) -> offset of a 256 x 8 panel in shared memory (as
// leaf2.cu): the lane pattern of the register tile and all MMA fragment
// patterns are bank-conflict free
__device__ __forceinline__ int bsw(int r, int c) {
  const int slot = ((c ^ (r >> 3)) & 3) | (((r >> 1) & 1) << 2) | (((r ^ (r >> 2)) & 1) << 3);
  const int q = ((c >> 2) & 1) | (((r >> 2) & 1) << 1);
  return (r >> 3) * 64 + q * 16 + slot;
}

__device__ __forceinline__ void mma1688(double (&d)[4], double a0, double a1, double a2, double a3, double b0,
                                        double b1) {
  asm("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
}

struct TileIO {
  Panel P;
  int rs;
  int64_t ia;
  int nsl;
};

// registers: A[mt][nt][z], z = {(col g, row 2t), (g, 2t+1), (g+8, 2t), (g+8, 2t+1)} of the
// m16 column tile mt and the warp's n8 row tile nt (g = lane / 4, t = lane % 4)
__device__ __forceinline__ void load_tile(double (&A)[NMT][NN][4], const TileIO& io, int b, int rbase) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  const int rows = io.nsl * io.rs;
  const int64_t cstride = io.P.trans ? 1 : io.P.rl * io.P.I;  // column step of the view
  const double* base = io.P.base;
#pragma unroll
  for (int nt = 0; nt < NN; ++nt) {
    int64_t off[2];
    bool ok[2];
    int si[2], w[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // one division pair per row, not per element
      const int r = rbase + nt * 8 + 2 * t4 + h;
      tile_row(io.P.trans, r, io.nsl, io.rs, si[h], w[h]);
      ok[h] = r < rows;
      off[h] = ok[h] ? io.P.addr(w[h], io.ia + si[h], 0) : 0;
    }
    if (io.P.kron.x) {  // implicit Hadamard core: elements formed on load
#pragma unroll
      for (int mt = 0; mt < NMT; ++mt) {
        const int c = mt * 16 + g;
        A[mt][nt][0] = ok[0] && c < b ? io.P.load(w[0], io.ia + si[0], c) : 0.0;
        A[mt][nt][1] = ok[1] && c < b ? io.P.load(w[1], io.ia + si[1], c) : 0.0;
        A[mt][nt][2] = ok[0] && c + 8 < b ? io.P.load(w[0], io.ia + si[0], c + 8) : 0.0;
        A[mt][nt][3] = ok[1] && c + 8 < b ? io.P.load(w[1], io.ia + si[1], c + 8) : 0.0;
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

// panel p's columns of the register tile <-> x[nt][h] (lane (g, t): column g of the panel)
template <int MT, int H>
__device__ __forceinline__ void get_panel(const double (&A)[NMT][NN][4], double (&x)[NN][2]) {
#pragma unroll
  for (int nt = 0; nt < NN; ++nt) {
    x[nt][0] = A[MT][nt][2 * H];
    x[nt][1] = A[MT][nt][2 * H + 1];
  }
}
template <int MT, int H>
__device__ __forceinline__ void put_panel(double (&A)[NMT][NN][4], const double (&x)[NN][2]) {
#pragma unroll
  for (int nt = 0; nt < NN; ++nt) {
    A[MT][nt][2 * H] = x[nt][0];
    A[MT][nt][2 * H + 1] = x[nt][1];
  }
}

// sum over the warps of column c's partials (p = part[buf][0] + c, warp stride NB)
__device__ __forceinline__ double sum8(const double* p) {
  const double a = p[0], b = p[NB], c = p[2 * NB], d = p[3 * NB];
  const double e = p[4 * NB], f = p[5 * NB], g = p[6 * NB], h = p[7 * NB];
  return ((a + b) + (c + d)) + ((e + f) + (g + h));
}

// Householder QR of the panel's 8 columns over [pivot rows; tile rows]:
// HEAD: pivots are tile rows c0 + j (rows above stay R entries); otherwise
// pivots are rows c0 + j of sm.Rs.  Finished columns stay RAW in registers
// during the panel (v_g = scal_g x_g is formed once at the end: no per-step
// scaling on the column chain).  On exit x holds V_p (head: R entries on and
// above the pivots), sm.Yb its swizzled copy, sm.taus / sm.Gs the panel's
// tau and Gram entries v_g . v_J and, for chain tiles, the panel block of
// sm.Rs is updated.
template <bool HEAD>
__device__ __forceinline__ void factor_panel(double (&x)[NN][2], Smem& sm, int c0, int nbp, int rbase) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t4 = lane & 3;
  const bool writer = warp == 0 && t4 == 0;
  // a chain tile's new R entry of the previous step, written one barrier later
  // (other warps read the old row until then)
  double pend = 0.0;
  int pend_at = -1;
  double myscal = 0.0, mybeta = 0.0;  // of this lane's own column, once it is factored
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    if (j < nbp) {
      const int J = c0 + j;
      LF3_STEP(0);
      // chain tiles: row J of R is final input until this step (prefetched off the critical path)
      const double pvg_r = HEAD ? 0.0 : sm.Rs[J + BM * (c0 + g)];
      const double alpha_r = HEAD ? 0.0 : sm.Rs[J + BM * J];
      double xj[NN][2];
#pragma unroll
      for (int nt = 0; nt < NN; ++nt) {
        xj[nt][0] = __shfl_sync(0xffffffffu, x[nt][0], j * 4 + t4);
        xj[nt][1] = __shfl_sync(0xffffffffu, x[nt][1], j * 4 + t4);
        if (HEAD) {  // rows <= J take no part in reflector J
          const int r = rbase + nt * 8 + 2 * t4;
          xj[nt][0] = r > J ? xj[nt][0] : 0.0;
          xj[nt][1] = r + 1 > J ? xj[nt][1] : 0.0;
        }
      }
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int nt = 0; nt < NN; ++nt) {
        a0 = fma(xj[nt][0], x[nt][0], a0);
        a1 = fma(xj[nt][1], x[nt][1], a1);
      }
      double acc = a0 + a1;
      LF3_STEP(1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      const int buf = j & 1;
      LF3_STEP(2);
      if (t4 == 0) sm.part[buf][warp][g] = acc;
      if (HEAD) {
#pragma unroll
        for (int nt = 0; nt < NN; ++nt) {
          const int r = rbase + nt * 8 + 2 * t4;
          if (r == J) sm.pvs[buf][g] = x[nt][0];
          if (r + 1 == J) sm.pvs[buf][g] = x[nt][1];
        }
      }
      LF3_STEP(3);
      __syncthreads();
      LF3_STEP(4);
      if (!HEAD && writer && pend_at >= 0) sm.Rs[pend_at] = pend;
      const double sig = sum8(&sm.part[buf][0][j]);
      const double sg = sum8(&sm.part[buf][0][g]);
      // pivot-row entry of this lane's column: R[J, g] (chain), tile row J (head; a
      // finished column g < j holds raw x_g there: v_g[J] = scal_g x_g[J])
      const double pvg = HEAD ? (g < j ? myscal * sm.pvs[buf][g] : sm.pvs[buf][g]) : pvg_r;
      const double alpha = HEAD ? sm.pvs[buf][j] : alpha_r;
      double beta, tau, scal, bv;
      LF3_STEP(5);
      reflector_scalars<false>(alpha, sig, beta, tau, scal, bv);
      LF3_STEP(6);
      // d = v_J . a_g (g > j: the update; g < j with v_g = scal_g x_g: the Gram entry)
      const double d = fma(scal * (g < j ? myscal : 1.0), sg, pvg);
      const double td = tau * d;
      const double coef = g > j ? -(td * scal) : 0.0;
#pragma unroll
      for (int nt = 0; nt < NN; ++nt) {
        x[nt][0] = fma(coef, xj[nt][0], x[nt][0]);
        x[nt][1] = fma(coef, xj[nt][1], x[nt][1]);
      }
      if (HEAD && g > j) {  // the pivot row: v_J = 1
#pragma unroll
        for (int nt = 0; nt < NN; ++nt) {
          const int r = rbase + nt * 8 + 2 * t4;
          if (r == J) x[nt][0] -= td;
          if (r + 1 == J) x[nt][1] -= td;
        }
      }
      if (g == j) {
        myscal = scal;
        mybeta = beta;
      }
      if (!HEAD) {
        pend = g > j ? pvg - td : beta;
        pend_at = g >= j ? J + BM * (c0 + g) : -1;
      }
      if (writer) {
        if (g == j) sm.taus[J] = tau;
        if (g < j) sm.Gs[(c0 + g) + BM * J] = d;  // v_g . v_J
      }
      LF3_STEP(7);
    }
  }
  // v = scal x (head: rows below the pivot; the pivot row takes R's beta), then V_p -> Yb
  // (head: zeros above the pivot, unit pivot)
#pragma unroll
  for (int nt = 0; nt < NN; ++nt) {
    const int r = rbase + nt * 8 + 2 * t4;
    double v0, v1;
    if (HEAD) {
      const int Jg = c0 + g;
      x[nt][0] = r > Jg ? x[nt][0] * myscal : (r == Jg ? mybeta : x[nt][0]);
      x[nt][1] = r + 1 > Jg ? x[nt][1] * myscal : (r + 1 == Jg ? mybeta : x[nt][1]);
      v0 = r < Jg ? 0.0 : (r == Jg ? 1.0 : x[nt][0]);
      v1 = r + 1 < Jg ? 0.0 : (r + 1 == Jg ? 1.0 : x[nt][1]);
    } else {
      x[nt][0] *= myscal;
      x[nt][1] *= myscal;
      v0 = x[nt][0];
      v1 = x[nt][1];
    }
    if (g >= nbp) {
      v0 = 0.0;
      v1 = 0.0;
    }
    sm.Yb[bsw(r, g)] = v0;
    sm.Yb[bsw(r + 1, g)] = v1;
  }
  __syncthreads();
  if (!HEAD && writer && pend_at >= 0) sm.Rs[pend_at] = pend;
}

// W^T partial of m-tile MT over this warp's rows -> sm.Wpart[warp]
template <int MT>
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

// A^T[m-tile MT] += Wneg-fragment x V_p^T
template <int MT>
__device__ __forceinline__ void update_mt(double (&A)[NMT][NN][4], const double (&yu)[NN][2], const Smem& sm) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  const double* wn = sm.Wneg;
  const double a0 = wn[(MT * 16 + g) * WNLD + t4], a1 = wn[(MT * 16 + g + 8) * WNLD + t4];
  const double a2 = wn[(MT * 16 + g) * WNLD + t4 + 4], a3 = wn[(MT * 16 + g + 8) * WNLD + t4 + 4];
#pragma unroll
  for (int nt = 0; nt < NN; ++nt) mma1688(A[MT][nt], a0, a1, a2, a3, yu[nt][0], yu[nt][1]);
}

#define LF3_FOR_MT(mask, CALL) \
  do {                         \
    if ((mask) & 1) CALL(0);   \
    if ((mask) & 2) CALL(1);   \
    if ((mask) & 4) CALL(2);   \
    if ((mask) & 8) CALL(3);   \
  } while (0)

template <bool HEAD>
__device__ __forceinline__ void factor_tile(double (&A)[NMT][NN][4], Smem& sm, int b, int rbase, int t) {
  const int tid = threadIdx.x, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  const int np = (b + NB - 1) / NB;
  unsigned mt_all = 0;
  for (int mt = 0; mt < NMT; ++mt)
    if (mt * 16 < b) mt_all |= 1u << mt;
  for (int p = 0; p < np; ++p) {
    const int c0 = p * NB, nbp = min(NB, b - c0);
    double x[NN][2];
    switch (p) {
      case 0: get_panel<0, 0>(A, x); break;
      case 1: get_panel<0, 1>(A, x); break;
      case 2: get_panel<1, 0>(A, x); break;
      case 3: get_panel<1, 1>(A, x); break;
      case 4: get_panel<2, 0>(A, x); break;
      case 5: get_panel<2, 1>(A, x); break;
      case 6: get_panel<3, 0>(A, x); break;
      default: get_panel<3, 1>(A, x); break;
    }
    LF3_ACC_BEGIN();
    factor_panel<HEAD>(x, sm, c0, nbp, rbase);
    LF3_ACC(t, 10);
    switch (p) {
      case 0: put_panel<0, 0>(A, x); break;
      case 1: put_panel<0, 1>(A, x); break;
      case 2: put_panel<1, 0>(A, x); break;
      case 3: put_panel<1, 1>(A, x); break;
      case 4: put_panel<2, 0>(A, x); break;
      case 5: put_panel<2, 1>(A, x); break;
      case 6: put_panel<3, 0>(A, x); break;
      default: put_panel<3, 1>(A, x); break;
    }
    // panel T by back substitution of (diag(1/tau) + striu(G_pp)) X = I (one column per lane)
    if (tid < NB) {
      const int c = tid;
      double xc[NB];
#pragma unroll
      for (int i = NB - 1; i >= 0; --i) {
        const double tau = i < nbp ? sm.taus[c0 + i] : 0.0;
        double acc = (i == c) ? 1.0 : 0.0;
#pragma unroll
        for (int m = i + 1; m < NB; ++m) acc = fma(-sm.Gs[(c0 + i) + BM * (c0 + m)], xc[m], acc);
        xc[i] = (i <= c) ? tau * acc : 0.0;
      }
#pragma unroll
      for (int i = 0; i < NB; ++i) sm.Tpp[i * NB + c] = xc[i];
    }
    {
      // V_p as the B fragment of W^T = A^T V_p (k = row, n = reflector)
      double yw[NN][2];
#pragma unroll
      for (int nt = 0; nt < NN; ++nt) {
        const int r = rbase + nt * 8;
        yw[nt][0] = sm.Yb[bsw(r + 2 * t4, g)];
        yw[nt][1] = sm.Yb[bsw(r + 2 * t4 + 1, g)];
      }
#define LF3_W(MT) wpart_mt<MT>(A, yw, sm)
      unsigned wmask = mt_all;
      if (!kInT) wmask &= ~((1u << ((c0 + NB) >> 4)) - 1);  // trailing m-tiles only
      LF3_FOR_MT(wmask, LF3_W);
#undef LF3_W
    }
    __syncthreads();
    LF3_ACC(t, 11);
    // sum the partials; cross Gram for finished columns, W' = T_pp^T W for trailing ones
#pragma unroll
    for (int rnd = 0; rnd < (BM * NB) / NT; ++rnd) {
      const int it = tid + rnd * NT;
      const int k = it >> 3, j = it & 7;
      double raw = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) raw += sm.Wpart[w][k * NB + j];
      const bool upd = k >= c0 + NB && k < b;
      double wv = raw;
      if (!HEAD && upd) wv += sm.Rs[(c0 + j) + BM * k];
      const int base = lane & ~7;
      double out = 0.0;
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        const double wi = __shfl_sync(0xffffffffu, wv, base + i);
        out = fma(sm.Tpp[i * NB + j], wi, out);  // T_pp upper: zero for i > j
      }
      if (kInT && k < c0 && c0 + j < b) sm.Gs[k + BM * (c0 + j)] = raw;
      sm.Wneg[k * WNLD + j] = upd ? -out : 0.0;
      if (!HEAD && upd) sm.Rs[(c0 + j) + BM * k] -= out;
    }
    __syncthreads();
    LF3_ACC(t, 12);
    unsigned trail = 0;
    for (int mt = (c0 + NB) >> 4; mt < NMT; ++mt)
      if (mt * 16 < b) trail |= 1u << mt;
    // V_p^T as the B fragment of the update (k = reflector, n = row)
    double yu[NN][2];
#pragma unroll
    for (int nt = 0; nt < NN; ++nt) {
      const int r = rbase + nt * 8;
      yu[nt][0] = sm.Yb[bsw(r + g, t4)];
      yu[nt][1] = sm.Yb[bsw(r + g, t4 + 4)];
    }
#define LF3_U(MT) update_mt<MT>(A, yu, sm)
    LF3_FOR_MT(trail, LF3_U);
#undef LF3_U
    LF3_ACC(t, 13);
  }
}

}  // namespace lf3

using namespace lf3;

__global__ void __launch_bounds__(lf3::NT, 1)
tsqr_leaf3_kernel(Panel P, LeafPlan plan, double* __restrict__ Yg, double* __restrict__ Tg,
                  double* __restrict__ Rleaf) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  lf3::Smem& sm = *reinterpret_cast<lf3::Smem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t4 = lane & 3;
  const int gcta = blockIdx.x;
  const int b = plan.b, rs = plan.rs, ni = plan.ni;
  const int64_t n_g = plan.count(gcta), s0 = plan.start(gcta);
  const int ntiles = plan.tiles_of(n_g);
  const int64_t tb = plan.tile_base(gcta);
  const int rbase = 32 * warp;
  for (int idx = tid; idx < BM * BM; idx += lf3::NT) sm.Rs[idx] = 0.0;

  double A[NMT][NN][4];
  auto tile_io = [&](int t) {
    lf3::TileIO io;
    io.P = P;
    io.rs = rs;
    io.ia = s0 + (int64_t)t * ni;
    io.nsl = (int)min64(ni, n_g - (int64_t)t * ni);
    return io;
  };
  if (ntiles > 0) lf3::load_tile(A, tile_io(0), b, rbase);
  for (int t = 0; t < ntiles; ++t) {
    LF3_CLK(t, 0);
    const bool head = t == 0;
    // pull the next-but-one tile's rows into L2 (as tsqr_leaf_kernel)
    if (t + 2 < ntiles && P.kron.x == nullptr) {
      const int64_t ia2 = s0 + (int64_t)(t + 2) * ni;
      const int nsl2 = (int)min64(ni, n_g - (int64_t)(t + 2) * ni);
      const int64_t runlen = P.rl * (int64_t)nsl2;
      const int nruns = P.trans ? rs : b;
      const int lines = (int)((runlen * 8 + 127) / 128) + 1;
      for (int idx = tid; idx < nruns * lines; idx += lf3::NT) {
        const int q = idx / lines, ln = idx - q * lines;
        const double* p0 = P.base + P.rl * (ia2 + P.I * (int64_t)q);
        const char* pl = reinterpret_cast<const char*>(p0) + (int64_t)ln * 128;
        if (pl < reinterpret_cast<const char*>(p0 + runlen)) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(pl));
      }
    }
    if (lf3::kInT)
      for (int k = tid; k < BM * BM; k += lf3::NT) sm.Gs[k] = 0.0;
    __syncthreads();
    LF3_CLK(t, 1);
    if (head) lf3::factor_tile<true>(A, sm, b, rbase, t);
    else lf3::factor_tile<false>(A, sm, b, rbase, t);
    __syncthreads();
    LF3_CLK(t, 7);
    // ---- tile outputs: Y (unit-major), head: R out of the register tile ----
    const int64_t tile = tb + t;
    double* Yt = Yg + tile * y_tile_stride(MC, b);
#pragma unroll
    for (int mt = 0; mt < NMT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NN; ++nt) {
        const int r = rbase + nt * 8 + 2 * t4;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int c = mt * 16 + g + 8 * hh;
          if (c >= b) continue;
          double v0 = A[mt][nt][2 * hh], v1 = A[mt][nt][2 * hh + 1];
          if (head) {
            if (r < b) sm.Rs[r + BM * c] = r <= c ? v0 : 0.0;
            if (r + 1 < b) sm.Rs[r + 1 + BM * c] = r + 1 <= c ? v1 : 0.0;
            v0 = r < c ? 0.0 : (r == c ? 1.0 : v0);
            v1 = r + 1 < c ? 0.0 : (r + 1 == c ? 1.0 : v1);
          }
          *reinterpret_cast<double2*>(&Yt[y_index(r, c, b)]) = make_double2(v0, v1);
        }
      }
    // the next tile's loads are in flight while T is formed
    if (t + 1 < ntiles) lf3::load_tile(A, tile_io(t + 1), b, rbase);
    if (lf3::kInT) {
      build_T<lf3::Cfg>(sm, b);
      LF3_CLK(t, 8);
      double* Tt = Tg + tile * (((int64_t)b * b + 1) & ~1LL);
      for (int idx = tid; idx < b * b; idx += lf3::NT) {
        const int k = idx % b, j = idx / b;
        Tt[idx] = sm.Gs[k + BM * j];
      }
    } else {
      LF3_CLK(t, 8);
      // the tile's tau for tile_T_kernel: the diagonal of the T block
      double* Tt = Tg + tile * (((int64_t)b * b + 1) & ~1LL);
      for (int idx = tid; idx < b; idx += lf3::NT) Tt[idx + b * idx] = sm.taus[idx];
    }
    __syncthreads();
    LF3_CLK(t, 9);
  }
  __syncthreads();
  for (int idx = tid; idx < b * b; idx += lf3::NT) {
    const int r = idx % b, k = idx / b;
    Rleaf[(int64_t)gcta * b * b + idx] = r <= k ? sm.Rs[r + BM * k] : 0.0;
  }
}

#ifdef TTB_LF3_CLK
extern "C" int ttb_dbg_lf3clk(long long* out) {
  return cudaMemcpyFromSymbol(out, lf3::g_lf3clk, sizeof(long long) * 64 * 16) == cudaSuccess ? 0 : 5;
}
#endif

void launch_leaf3(Ctx& ctx, const Panel& panel, const LeafPlan& plan, double* Y, double* T, double* Rleaf) {
  smem_attr((const void*)tsqr_leaf3_kernel, sizeof(lf3::Smem));
  tsqr_leaf3_kernel<<<plan.G, lf3::NT, sizeof(lf3::Smem), ctx.stream>>>(panel, plan, Y, T, Rleaf);
  TTB_LAUNCHED();
}

}  // namespace ttb
