// Tall-skinny Householder QR (TSQR) for B200, fp64.
//
// Replaces the reference's leaf dgeqrf + butterfly tree + dormqr/dorgqr apply
// (ttpar tsqr.py:103-130 local_qr, 166-221 tsqr_factor, 248-327 tsqr_apply_q).
//
// Decomposition:
//  * A panel is a row-sliced view of a TT slab (V(X) or H(X)^T), split into
//    whole mode slices.  Each CTA owns a contiguous run of slices and walks
//    it as a *chain of register tiles*: tile 0 is a plain Householder QR of
//    its rows (pivots inside the tile, LAPACK layout); tile t>0 factors the
//    stacked [R_{t-1}; A_t] with R kept in shared memory, so every CTA ends
//    with one b x b triangle.  Per tile we keep the Householder vectors Y and
//    the compact-WY factor T (Q_t = I - V_t T_t V_t^T, T^{-1} = diag(1/tau)
//    + striu(V^T V), accumulated inside the column loop).
//  * The per-CTA triangles are reduced by a tree of stacked-triangle QRs
//    (fan-in MC/b), one launch per level.
//  * Apply Q to a b x k block: every CTA walks its own root-to-leaf path
//    (only its child's b rows of each node), then its chain in reverse;
//    each tile costs one (rows x b)(b x k) product -- no row reductions.
//
// Register tile layout (per CTA, NW warps): lane = lc*LR + lr.  Column
// k = t*(NW*LC) + w*LC + lc (t < CPL) lives in warp w, lane group lc; row
// r = s*LR + lr (s < RPL).  Column dot products reduce over the LR lanes of
// a group with shuffles; the Householder vector of the current column is
// broadcast through shared memory (double buffered, one barrier per column).
#pragma once

#include "common.cuh"

namespace ttb {

template <int NW_, int LC_, int CPL_, int RPL_>
struct TCfg {
  static constexpr int NW = NW_, LC = LC_, LR = 32 / LC_, CPL = CPL_, RPL = RPL_;
  static constexpr int NT = NW * 32;
  static constexpr int BMAX = NW * LC * CPL;
  static constexpr int MC = LR * RPL;
};

// leaf (2 CTAs / SM) and tree-node (one big CTA) configurations per BMAX
using Leaf64 = TCfg<8, 2, 4, 8>;    // b <= 64, 128-row tiles
using Leaf32 = TCfg<8, 1, 4, 8>;    // b <= 32, 256-row tiles
using Leaf16 = TCfg<8, 1, 2, 16>;   // b <= 16, 512-row tiles
using Tree64 = TCfg<32, 2, 1, 16>;  // 1024 thr, 256 rows: fan-in 4 at b=64
using Tree32 = TCfg<16, 1, 2, 16>;  // 512 thr, 512 rows: fan-in 16 at b=32
using Tree16 = TCfg<16, 1, 1, 32>;  // 512 thr, 1024 rows: fan-in 64 at b=16

// A row-sliced view of an F-order slab (rl, I, rr):
//   trans == 0: V(X)    rows per slice rs = rl, columns = rr
//   trans == 1: H(X)^T  rows per slice rs = rr, columns = rl
// element (w, i, col) at  V: w + rl*(i + I*col);  H^T: col + rl*(i + I*w)
struct Panel {
  double* base;
  int64_t rl, I, rr;
  int trans;
  __host__ __device__ int64_t rs() const { return trans ? rr : rl; }
  __host__ __device__ int64_t ncols() const { return trans ? rl : rr; }
  __host__ __device__ int64_t addr(int64_t w, int64_t i, int64_t col) const {
    return trans ? col + rl * (i + I * w) : w + rl * (i + I * col);
  }
};

// Row order inside a tile of nsl whole slices (rows = nsl*rs).  V views are
// slice-major (left rank fastest, as V(X) itself); H^T views are mode-index
// fastest (as H(X)^T itself, parallel.py:144-161).  This keeps the head
// tile's pivot rows where the reference's dgeqrf puts them, so structurally
// zero rows (from rank-deficient R folds) never become pivots and exact
// zeros survive -- which eps0 = 0 rounding relies on.
__device__ __forceinline__ void tile_row(int trans, int r, int nsl, int rs, int& si, int& w) {
  if (trans) {
    w = r / nsl;
    si = r - w * nsl;
  } else {
    si = r / rs;
    w = r - si * rs;
  }
}

// Balanced split of nslices over G CTAs; per-CTA tile counts in closed form.
struct LeafPlan {
  int64_t nslices;
  int G;       // CTAs
  int ni;      // slices per tile
  int rs;      // rows per slice
  int b;       // columns
  __host__ __device__ int64_t base() const { return nslices / G; }
  __host__ __device__ int rem() const { return (int)(nslices % G); }
  __host__ __device__ int64_t count(int g) const { return base() + (g < rem() ? 1 : 0); }
  __host__ __device__ int64_t start(int g) const { return (int64_t)g * base() + (g < rem() ? g : rem()); }
  __host__ __device__ int tiles_of(int64_t n) const { return (int)((n + ni - 1) / ni); }
  __host__ __device__ int64_t tile_base(int g) const {
    int64_t t1 = tiles_of(base() + 1), t0 = tiles_of(base());
    int64_t a = g < rem() ? g : rem();
    int64_t c = g > rem() ? g - rem() : 0;
    return a * t1 + c * t0;
  }
  __host__ __device__ int64_t total_tiles() const { return tile_base(G); }
};

constexpr int kMaxLevels = 12;

// One level of the reduction tree as seen by the apply kernel.
struct Level {
  const double* Y;  // node Householder vectors, ld = ldy, node stride ldy*b
  const double* T;  // node T factors, b*b per node
  int ldy;          // rows per node tile (MC of the tree config)
  int f;            // fan-in of this level
  int fixed_child;  // >= 0: child index is this value (global root: rank); -1: derive
};

struct TreeDesc {
  int nlev;
  Level lev[kMaxLevels];  // lev[0] = first level above the leaves ... lev[nlev-1] = root
};

// ------------------------------------------------------------------------
// tile QR (device)
// ------------------------------------------------------------------------

template <class C>
struct TileSmem {
  double Rs[C::BMAX * C::BMAX];    // chain triangle R (col-major, ld BMAX)
  double Gs[C::BMAX * C::BMAX];    // V^T V strict upper -> T after inversion
  double Xs[C::BMAX * C::BMAX / 2];  // inversion scratch
  double vbuf[2][C::MC];
  double taus[C::BMAX];
};

template <class C>
__device__ __forceinline__ int col_of(int t, int warp, int lc) {
  return t * (C::NW * C::LC) + warp * C::LC + lc;
}

// In-place T = (diag(1/tau) + striu(G))^{-1}, blocked recursive inversion.
// On entry Gs holds striu(V^T V) (zeros elsewhere) and taus; on exit Gs = T.
template <class C>
__device__ void build_T(TileSmem<C>& sm, int b) {
  const int tid = threadIdx.x;
  constexpr int BM = C::BMAX;
  int BP = 1;
  while (BP < b) BP <<= 1;
  for (int k = tid; k < BP; k += C::NT) sm.Gs[k + BM * k] = (k < b) ? sm.taus[k] : 1.0;
  __syncthreads();
  for (int s = 1; s < BP; s <<= 1) {
    const int nblk = BP / (2 * s);
    const int items = nblk * s * s;
    // X = U[A,C] * T[C,C]
    for (int idx = tid; idx < items; idx += C::NT) {
      int q = idx / (s * s), rem = idx - q * s * s;
      int r = rem % s, c = rem / s;
      int a0 = q * 2 * s, c0 = a0 + s;
      double acc = 0.0;
      for (int l = 0; l <= c; ++l) acc += sm.Gs[(a0 + r) + BM * (c0 + l)] * sm.Gs[(c0 + l) + BM * (c0 + c)];
      sm.Xs[idx] = acc;
    }
    __syncthreads();
    // T[A,C] = -T[A,A] * X
    for (int idx = tid; idx < items; idx += C::NT) {
      int q = idx / (s * s), rem = idx - q * s * s;
      int r = rem % s, c = rem / s;
      int a0 = q * 2 * s, c0 = a0 + s;
      double acc = 0.0;
      for (int l = r; l < s; ++l) acc += sm.Gs[(a0 + r) + BM * (a0 + l)] * sm.Xs[q * s * s + l + s * c];
      sm.Gs[(a0 + r) + BM * (c0 + c)] = -acc;
    }
    __syncthreads();
  }
}

// Householder QR of one register tile.  head: pivots are tile rows 0..b-1
// (plain QR); otherwise pivots are rows of the chain triangle sm.Rs (the
// stacked [R; A] factorization).  On exit: A holds the Householder vectors
// (head: R in the upper triangle of rows < b, beta on the diagonal), sm.Gs
// holds T, sm.Rs holds R (body) -- the caller extracts R for head tiles.
template <class C>
__device__ void tile_qr(double (&A)[C::RPL][C::CPL], int b, bool head, TileSmem<C>& sm) {
  constexpr int LR = C::LR, LC = C::LC, RPL = C::RPL, CPL = C::CPL, BM = C::BMAX;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lc = lane / LR, lr = lane % LR;

  for (int j = 0; j < b; ++j) {
    const int ow = (j / LC) % C::NW, olc = j % LC, ot = j / (C::NW * LC);
    double* vb = sm.vbuf[j & 1];
    if (warp == ow) {
      // every lane group computes "its" column at slot ot; only olc is used
      double colv[RPL];
#pragma unroll
      for (int s = 0; s < RPL; ++s) {
        double x = 0.0;
#pragma unroll
        for (int t = 0; t < CPL; ++t) x = (t == ot) ? A[s][t] : x;
        colv[s] = x;
      }
      double sig = 0.0, aj = 0.0;
#pragma unroll
      for (int s = 0; s < RPL; ++s) {
        const int r = s * LR + lr;
        if (!head || r > j) sig = fma(colv[s], colv[s], sig);
        if (head && r == j) aj = colv[s];
      }
#pragma unroll
      for (int off = LR / 2; off > 0; off >>= 1) {
        sig += __shfl_xor_sync(0xffffffffu, sig, off);
        aj += __shfl_xor_sync(0xffffffffu, aj, off);
      }
      const double alpha = head ? aj : sm.Rs[j + BM * j];
      double beta, tau, scal;
      if (sig == 0.0) {  // reflect e_j onto -e_j: keeps tau in [1, 2] always
        beta = -alpha; tau = 2.0; scal = 0.0;
      } else {
        const double nrm = sqrt(fma(alpha, alpha, sig));
        beta = alpha >= 0.0 ? -nrm : nrm;
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      if (lc == olc) {
#pragma unroll
        for (int s = 0; s < RPL; ++s) {
          const int r = s * LR + lr;
          double v, keepv;
          if (head) {
            v = r < j ? 0.0 : (r == j ? 1.0 : colv[s] * scal);
            keepv = r > j ? v : (r == j ? beta : colv[s]);
          } else {
            v = colv[s] * scal;
            keepv = v;
          }
#pragma unroll
          for (int t = 0; t < CPL; ++t)
            if (t == ot) A[s][t] = keepv;
          vb[r] = v;
        }
        if (lr == 0) {
          sm.taus[j] = tau;
          if (!head) sm.Rs[j + BM * j] = beta;
        }
      }
    }
    __syncthreads();
    double vr[RPL];
#pragma unroll
    for (int s = 0; s < RPL; ++s) vr[s] = vb[s * LR + lr];
    const double tau = sm.taus[j];
    double d[CPL];
#pragma unroll
    for (int t = 0; t < CPL; ++t) {
      const int k = col_of<C>(t, warp, lc);
      double acc = 0.0;
      if (k < b && k != j) {
#pragma unroll
        for (int s = 0; s < RPL; ++s) acc = fma(vr[s], A[s][t], acc);
        if (!head && k > j && lr == 0) acc += sm.Rs[j + BM * k];
      }
      d[t] = acc;
    }
#pragma unroll
    for (int off = LR / 2; off > 0; off >>= 1) {
#pragma unroll
      for (int t = 0; t < CPL; ++t) d[t] += __shfl_xor_sync(0xffffffffu, d[t], off);
    }
#pragma unroll
    for (int t = 0; t < CPL; ++t) {
      const int k = col_of<C>(t, warp, lc);
      if (k > j && k < b) {
        const double coef = tau * d[t];
#pragma unroll
        for (int s = 0; s < RPL; ++s) A[s][t] = fma(-coef, vr[s], A[s][t]);
        if (!head && lr == 0) sm.Rs[j + BM * k] -= coef;
      } else if (k < j && lr == 0) {
        sm.Gs[k + BM * j] = d[t];
      }
    }
  }
  __syncthreads();
  build_T<C>(sm, b);
}

template <class C>
__device__ __forceinline__ void zero_G(TileSmem<C>& sm) {
  for (int k = threadIdx.x; k < C::BMAX * C::BMAX; k += C::NT) sm.Gs[k] = 0.0;
}

// write Householder vectors of a tile: Y[r + ldy*k], head => unit lower trapezoid
template <class C>
__device__ void store_Y(const double (&A)[C::RPL][C::CPL], int b, bool head, double* Y, int ldy) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lc = lane / C::LR, lr = lane % C::LR;
#pragma unroll
  for (int t = 0; t < C::CPL; ++t) {
    const int k = col_of<C>(t, warp, lc);
    if (k >= b) continue;
#pragma unroll
    for (int s = 0; s < C::RPL; ++s) {
      const int r = s * C::LR + lr;
      double v = A[s][t];
      if (head) v = r < k ? 0.0 : (r == k ? 1.0 : v);
      Y[r + (int64_t)ldy * k] = v;
    }
  }
}

template <class C>
__device__ void store_T(const TileSmem<C>& sm, int b, double* T) {
  for (int idx = threadIdx.x; idx < b * b; idx += C::NT) {
    int k = idx % b, j = idx / b;
    T[idx] = sm.Gs[k + C::BMAX * j];
  }
}

// head tile: R = upper triangle of tile rows < b  ->  sm.Rs
template <class C>
__device__ void extract_R(const double (&A)[C::RPL][C::CPL], int b, TileSmem<C>& sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lc = lane / C::LR, lr = lane % C::LR;
#pragma unroll
  for (int t = 0; t < C::CPL; ++t) {
    const int k = col_of<C>(t, warp, lc);
    if (k >= b) continue;
#pragma unroll
    for (int s = 0; s < C::RPL; ++s) {
      const int r = s * C::LR + lr;
      if (r < b) sm.Rs[r + C::BMAX * k] = (r <= k) ? A[s][t] : 0.0;
    }
  }
}

}  // namespace ttb
