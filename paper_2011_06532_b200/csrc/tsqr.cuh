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

// XW_: extra warps of the CTA beyond the NW compute warps (the tree's data
// mover); the tile routines then synchronise the compute warps only.
template <int NW_, int LC_, int CPL_, int RPL_, int XW_ = 0>
struct TCfg {
  static constexpr int NW = NW_, LC = LC_, LR = 32 / LC_, CPL = CPL_, RPL = RPL_, XW = XW_;
  static constexpr int NT = NW * 32;        // compute threads (the first NT of the CTA)
  static constexpr int NTT = NT + 32 * XW;  // all threads of the CTA
  __device__ __forceinline__ static void sync() {
    if (XW == 0) {
      __syncthreads();
    } else {
      asm volatile("bar.sync 1, %0;\n" ::"n"(NT) : "memory");
    }
  }
  static constexpr int BMAX = NW * LC * CPL;
  static constexpr int MC = LR * RPL;
  // resident CTAs per SM: two only when the register tile leaves room
  static constexpr int MINB = (NT <= 256 && 2 * RPL * CPL + 64 <= 128) ? 2 : 1;
  static_assert(RPL % 2 == 0, "rows come in pairs (128-bit vector loads)");
  // tile row of register slot s in lane-row lr: consecutive pairs per lane
  __device__ __forceinline__ static int row(int s, int lr) { return (s >> 1) * (2 * LR) + 2 * lr + (s & 1); }
  // head tiles: pivot rows are < BMAX; register slot s only holds rows >= (s/2)*2LR,
  // so for slots with (s/2)*2LR >= BMAX every row-vs-pivot test is known at compile time
  __host__ __device__ static constexpr bool pivot_slot(int s) { return (s >> 1) * 2 * LR < BMAX; }
  // owner of column j: warp j % NW, lane group (j / NW) % LC, slot j / (NW*LC)
  __device__ __forceinline__ static int owner_warp(int j) { return j % NW; }
  __device__ __forceinline__ static int owner_lc(int j) { return (j / NW) % LC; }
  __device__ __forceinline__ static int owner_slot(int j) { return j / (NW * LC); }
};

// Leaf (2 CTAs / SM) and tree-node configurations per BMAX.  Column groups
// of LR = 8 lanes keep the per-column reductions at 3 shuffle rounds; each
// lane holds RPL rows x CPL columns of the register tile.
// (TTB_LEAF64 etc. override a configuration at compile time for tuning runs)
#ifndef TTB_LEAF64
#define TTB_LEAF64 8, 2, 4, 16
#endif
#ifndef TTB_LEAF32
#define TTB_LEAF32 8, 1, 4, 16
#endif
#ifndef TTB_LEAF16
#define TTB_LEAF16 8, 1, 2, 32
#endif
#ifndef TTB_TREE64
#define TTB_TREE64 8, 2, 4, 12
#endif
#ifndef TTB_TREE32
#define TTB_TREE32 8, 4, 1, 32
#endif
#ifndef TTB_TREE16
#define TTB_TREE16 8, 2, 1, 32
#endif
using Leaf64 = TCfg<TTB_LEAF64>;   // b <= 64: 256-row tiles, 256 threads (4 columns each), 1 CTA / SM
using Leaf32 = TCfg<TTB_LEAF32>;   // b <= 32: 512-row tiles, 32 lanes per column
using Leaf16 = TCfg<TTB_LEAF16>;   // b <= 16: 1024-row tiles, 32 lanes per column
// Tree nodes: NW compute warps (+ an optional data-mover warpgroup,
// TTB_TREE_XW=4).  The node's register tile holds the children other than
// child 0 (which sits in shared memory as the body tile's R): 192 rows at
// b <= 64, fan-in MC / b + 1.  Default: no mover -- warp 0 polls the
// children's counters off the column step's critical path and issues the
// bulk copies itself -- so the CTA has 8 warps and the column loop gets the
// leaf's register budget (a mover warpgroup makes 12 warps, and the register
// file, 16K registers per sub-partition, caps the whole kernel at 168 per
// thread at compile time: setmaxnreg only moves registers at run time).
// Measured per tree (cfg3 panel): 148 us with the mover, 143 us without.
#ifndef TTB_TREE_XW
#define TTB_TREE_XW 0
#endif
using Tree64 = TCfg<TTB_TREE64, TTB_TREE_XW>;   // 192 rows: fan-in 4 at b = 60..64
using Tree32 = TCfg<TTB_TREE32, TTB_TREE_XW>;   // 256 rows: fan-in 9 at b = 32
using Tree16 = TCfg<TTB_TREE16, TTB_TREE_XW>;   // 512 rows: fan-in 33 at b = 16

// A row-sliced view of an F-order slab (rl, I, rr):
//   trans == 0: V(X)    rows per slice rs = rl, columns = rr
//   trans == 1: H(X)^T  rows per slice rs = rr, columns = rl
// element (w, i, col) at  V: w + rl*(i + I*col);  H^T: col + rl*(i + I*w)
// An implicit Hadamard core (ops.py:109-132 layout, never materialised):
//   Z[a rwl + c, i, b rwr + d] = X[a, i, b] * W[c, i, d]
// (x == nullptr: no Kronecker source).
struct Kron {
  const double* x = nullptr;
  const double* w = nullptr;
  int64_t rxl = 0, rxr = 0, rwl = 0, rwr = 0;
  __device__ __forceinline__ double at(int64_t l, int64_t i, int64_t m, int64_t I) const {
    const int64_t a = l / rwl, c = l - a * rwl, b = m / rwr, d = m - b * rwr;
    return __dmul_rn(x[a + rxl * (i + I * b)], w[c + rwl * (i + I * d)]);
  }
};

struct Panel {
  double* base;
  int64_t rl, I, rr;
  int trans;
  Kron kron;  // kron.x set: the panel is a view of an implicit Hadamard core (base unused)
  __host__ __device__ int64_t rs() const { return trans ? rr : rl; }
  __host__ __device__ int64_t ncols() const { return trans ? rl : rr; }
  __host__ __device__ int64_t addr(int64_t w, int64_t i, int64_t col) const {
    return trans ? col + rl * (i + I * w) : w + rl * (i + I * col);
  }
  // element (w, i, col) of the view, whatever the source
  __device__ __forceinline__ double load(int64_t w, int64_t i, int64_t col) const {
    if (kron.x) return trans ? kron.at(col, i, w, I) : kron.at(w, i, col, I);
    return base[addr(w, i, col)];
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

// Team-pipelined leaf (wleaf.cu): each CTA owns a contiguous run of slices;
// its rows, in the reference's row order for that run (V: slice-major, as
// V(X); H^T: mode index fastest over the whole run, as H(X)^T), are cut into
// tiles of kWH rows regardless of slice boundaries.
constexpr int kWH = 64;        // tile rows
constexpr int kWLDY = kWH + 4; // Y column stride inside a tile (= 4 mod 16: conflict-free MMA fragments)

struct WPlan {
  int64_t nslices;
  int G;   // CTAs (chains)
  int rs;  // rows per slice
  int b;   // columns
  __host__ __device__ int64_t base() const { return nslices / G; }
  __host__ __device__ int rem() const { return (int)(nslices % G); }
  __host__ __device__ int64_t count(int g) const { return base() + (g < rem() ? 1 : 0); }
  __host__ __device__ int64_t start(int g) const { return (int64_t)g * base() + (g < rem() ? g : rem()); }
  __host__ __device__ int tiles_of(int64_t cnt) const { return (int)((cnt * rs + kWH - 1) / kWH); }
  __host__ __device__ int64_t tile_base(int g) const {
    int64_t t1 = tiles_of(base() + 1), t0 = tiles_of(base());
    int64_t a = g < rem() ? g : rem();
    int64_t c = g > rem() ? g - rem() : 0;
    return a * t1 + c * t0;
  }
  __host__ __device__ int64_t total_tiles() const { return tile_base(G); }
  // chain and tile index of a global tile number
  __host__ __device__ void tile_of(int64_t tile, int& g, int64_t& t) const {
    const int64_t t1 = tiles_of(base() + 1), t0 = tiles_of(base());
    if (tile < (int64_t)rem() * t1) {
      g = (int)(tile / t1);
      t = tile - (int64_t)g * t1;
    } else {
      const int64_t x = tile - (int64_t)rem() * t1;
      g = rem() + (int)(x / t0);
      t = x - (int64_t)(g - rem()) * t0;
    }
  }
};
// row r of a chain of cnt slices -> (slice offset si, row-in-slice w)
__host__ __device__ __forceinline__ void wrow(int trans, int64_t r, int64_t cnt, int rs, int64_t& si, int64_t& w) {
  if (trans) {
    w = r / cnt;
    si = r - w * cnt;
  } else {
    si = r / rs;
    w = r - si * rs;
  }
}
// advance (si, w) to the next row of the chain
__host__ __device__ __forceinline__ void wrow_next(int trans, int64_t cnt, int rs, int64_t& si, int64_t& w) {
  if (trans) {
    if (++si == cnt) {
      si = 0;
      ++w;
    }
  } else {
    if (++w == rs) {
      w = 0;
      ++si;
    }
  }
}

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

constexpr int kRing = 4;  // Householder vectors in flight between warps

// Debug-only cycle stamps of the column pipeline (CTA 0, second tile):
// build with NVCC_EXTRA=-DTTB_DEBUG_CLK, read back with ttb_dbg_clk.
#ifdef TTB_DEBUG_CLK
static __device__ long long g_dclk[16 * 64 * 16];
#define TTB_DCLK(ph)                                                                     \
  do {                                                                                   \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && gbase == b && j < 64 && threadIdx.x < 512) \
      g_dclk[((threadIdx.x >> 5) * 64 + j) * 16 + (ph)] = clock64();                     \
  } while (0)
#define TTB_DCLK2(ph)                                                                        \
  do {                                                                                       \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && (gj - j) > 0 && (gj - j) <= 64 && j < 64 && threadIdx.x < 512) \
      g_dclk[((threadIdx.x >> 5) * 64 + j) * 16 + (ph)] = clock64();                         \
  } while (0)
#else
#define TTB_DCLK(ph) \
  do {               \
  } while (0)
#define TTB_DCLK2(ph) \
  do {                \
  } while (0)
#endif

template <class C>
struct TileSmem {
  double Rs[C::BMAX * C::BMAX];      // chain triangle R (col-major, ld BMAX)
  double Gs[C::BMAX * C::BMAX];      // V^T V strict upper -> T after inversion
  double Xs[C::BMAX * C::BMAX / 2];  // inversion scratch
  double vring[kRing][C::MC];        // published raw columns
  alignas(16) double sc[kRing][4];   // published tau, scal, bv, beta
  double taus[C::BMAX];
  unsigned long long full[kRing];    // raw column ready (count 1)
  unsigned long long fulls[kRing];   // scalars ready (count 1)
  unsigned long long empty[kRing];   // consumers -> producer (count NW)
};

template <class C>
__device__ __forceinline__ int col_of(int t, int warp, int lc) {
  return (t * C::LC + lc) * C::NW + warp;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  unsigned long long st;
  asm volatile("mbarrier.arrive.shared::cta.b64 %0, [%1];\n" : "=l"(st) : "r"(smem_u32(bar)) : "memory");
  (void)st;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned done = 0;
  do {
    asm volatile(
#ifdef TTB_MBAR_HINT
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity), "r"(TTB_MBAR_HINT)
        : "memory");
#else
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
#endif
  } while (!done);
}

// once per CTA, before the first tile (count: full 1, empty NW)
template <class C>
__device__ void init_ring(TileSmem<C>& sm) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < kRing; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.fulls[s], 1);
      mbar_init(&sm.empty[s], C::NW);
    }
  }
}

// In-place T = (diag(1/tau) + striu(G))^{-1}.  On entry Gs holds striu(V^T V)
// (zeros elsewhere) and taus; on exit Gs = T.  The 8 x 8 diagonal blocks are
// inverted by back substitution (one thread per block column), then the
// off-diagonal blocks of growing size s = 8, 16, 32 by two fp64 MMA products
// per block pair, T_AC = -T_AA (U_AC T_CC), skipping the zero halves of the
// triangular factors.  Seven CTA barriers in all (the previous scalar
// recursion took twelve plus ~b^3/3 shared-memory FMAs on the SIMT pipe).
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <class C, class SM = TileSmem<C>>
__device__ void build_T(SM& sm, int b) {
  constexpr int BM = C::BMAX;
  constexpr int NWARP = C::NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int BP = 8;
  while (BP < b) BP <<= 1;
  const int nbl = BP / 8;
  // 1. diagonal 8 x 8 blocks: column c of block q (U's diagonal is 1/tau; padded columns: tau = 1)
  double xcol[8];
  const bool dthr = tid < nbl * 8;
  const int q0 = tid >> 3, cq = tid & 7, i0 = q0 * 8;
  if (dthr) {
#pragma unroll
    for (int i = 7; i >= 0; --i) {
      const int gi = i0 + i;
      const double tau = gi < b ? sm.taus[gi] : 1.0;
      double acc = (i == cq) ? 1.0 : 0.0;
#pragma unroll
      for (int m = i + 1; m < 8; ++m) acc = fma(-sm.Gs[gi + BM * (i0 + m)], xcol[m], acc);
      xcol[i] = (i <= cq) ? tau * acc : 0.0;
    }
  }
  C::sync();
  if (dthr) {
#pragma unroll
    for (int i = 0; i < 8; ++i) sm.Gs[(i0 + i) + BM * (i0 + cq)] = xcol[i];
  }
  C::sync();
  // 2. off-diagonal blocks, level by level
  const int fr = lane >> 2, fc = lane & 3;
  for (int s = 8; s < BP; s <<= 1) {
    const int tps = s / 8, ntile = (BP / (2 * s)) * tps * tps;
    // X_q = U_AC T_CC  (T_CC upper: rows k < (tj + 1) 8 of column tile tj)
    for (int t = warp; t < ntile; t += NWARP) {
      const int q = t / (tps * tps), rem = t - q * tps * tps, ti = rem % tps, tj = rem / tps;
      const int a0 = q * 2 * s, c0 = a0 + s;
      double d0 = 0.0, d1 = 0.0;
      for (int k0 = 0; k0 < (tj + 1) * 8; k0 += 4) {
        const double av = sm.Gs[(a0 + ti * 8 + fr) + BM * (c0 + k0 + fc)];
        const double bv = sm.Gs[(c0 + k0 + fc) + BM * (c0 + tj * 8 + fr)];
        dmma884(d0, d1, av, bv);
      }
      double* X = sm.Xs + q * s * s;
      const int r = ti * 8 + fr, cc = tj * 8 + 2 * fc;
      X[r + s * cc] = d0;
      X[r + s * (cc + 1)] = d1;
    }
    C::sync();
    // T_AC = -T_AA X_q  (T_AA upper: columns k >= ti 8 of row tile ti)
    for (int t = warp; t < ntile; t += NWARP) {
      const int q = t / (tps * tps), rem = t - q * tps * tps, ti = rem % tps, tj = rem / tps;
      const int a0 = q * 2 * s, c0 = a0 + s;
      const double* X = sm.Xs + q * s * s;
      double d0 = 0.0, d1 = 0.0;
      for (int k0 = ti * 8; k0 < s; k0 += 4) {
        const double av = sm.Gs[(a0 + ti * 8 + fr) + BM * (a0 + k0 + fc)];
        const double bv = X[(k0 + fc) + s * (tj * 8 + fr)];
        dmma884(d0, d1, av, bv);
      }
      const int r = ti * 8 + fr, cc = tj * 8 + 2 * fc;
      sm.Gs[(a0 + r) + BM * (c0 + cc)] = -d0;
      sm.Gs[(a0 + r) + BM * (c0 + cc + 1)] = -d1;
    }
    C::sync();
  }
}

// ---- column pipeline with delayed scaling --------------------------------
//
// The owner of column j publishes the RAW updated column x (rows < j zeroed
// for head tiles) as soon as it has applied reflector j-1, then computes the
// reflector scalars (sigma reduction, sqrt, reciprocal) and publishes those
// separately.  With v = scal * (x - beta e_j) (head) or v = [e_j; scal x]
// (body), consumers compute p = x . a (and q = a_j for head tiles) while the
// scalars are still in flight, and only then finish d = v . a and the update
// a -= tau d v.  sqrt/div leave the column-to-column critical path.
// Reflector scalars from alpha (pivot) and sig (squared norm below it):
// beta = -sign(alpha) |(alpha, x)|, tau = 1 + |alpha| / |(alpha, x)|,
// scal = 1 / (alpha - beta) (v = scal (x - bv e_j) for head tiles, [e_j; scal x]
// for body tiles).  sig == 0 reflects e_j onto -e_j (tau = 2, keeps tau in
// [1, 2]); bv differs from beta only for an all-zero head column (v = e_j).
// One rsqrt and one reciprocal, no divides.  Bitwise identical wherever it
// is evaluated from the same (alpha, sig).
// A column whose norm (pivot included) is below kTinyCol is treated as a zero
// column: its squares sit in the underflow range, sig loses its bits (or is
// flushed to an exact 0 while the entries are not), and 1 / (alpha - beta)
// overflows -- a Householder vector of size 1e130 once put infinities into T
// (LAPACK's dlarfg rescales such columns; here they only arise as roundoff of
// roundoff on structurally rank-deficient bonds, 1e-140 of anything that
// matters, so they are dropped: the reflector degenerates to a sign flip of
// row j and the stored vector stays bounded).
constexpr double kTinyCol = 1e-140;

template <bool HEAD>
__device__ __forceinline__ void reflector_scalars(double alpha, double sig, double& beta, double& tau, double& scal,
                                                  double& bv) {
  const double n2 = fma(alpha, alpha, sig);
  if (sig == 0.0 || n2 < kTinyCol * kTinyCol) {
    beta = -alpha;
    tau = 2.0;
    if (HEAD && fabs(alpha) < kTinyCol) {
      scal = 1.0;
      bv = -1.0;
    } else {
      scal = HEAD ? 0.5 / alpha : 0.0;
      bv = beta;
    }
  } else {
    const double rn = rsqrt(n2);
    const double nrm = n2 * rn;
    const double den = fabs(alpha) + nrm;
    const double rden = __drcp_rn(den);
    beta = alpha >= 0.0 ? -nrm : nrm;
    tau = den * rn;
    scal = alpha >= 0.0 ? rden : -rden;
    bv = beta;
  }
}

template <class C, bool HEAD, int OT>
__device__ __forceinline__ void publish_slot(double (&A)[C::RPL][C::CPL], int j, int gj, TileSmem<C>& sm) {
  constexpr int LR = C::LR, RPL = C::RPL, BM = C::BMAX;
  const int lane = threadIdx.x & 31;
  const int lc = lane / LR, lr = lane % LR;
  const bool mine = (lc == C::owner_lc(j));
  const int slot = gj % kRing;
  const double alpha_r = HEAD ? 0.0 : sm.Rs[j + BM * j];  // prefetched: it heads the scalar chain
  // 1. raw column
  if (mine) {
    double* xb = sm.vring[slot];
#pragma unroll
    for (int s = 0; s < RPL; s += 2) {
      double x0 = A[s][OT], x1 = A[s + 1][OT];
      if (HEAD && C::pivot_slot(s)) {
        x0 = C::row(s, lr) < j ? 0.0 : x0;
        x1 = C::row(s + 1, lr) < j ? 0.0 : x1;
      }
      *reinterpret_cast<double2*>(&xb[C::row(s, lr)]) = make_double2(x0, x1);
    }
  }
  TTB_DCLK2(10);
  __syncwarp();
  TTB_DCLK2(11);
  if (lane == 0) mbar_arrive(&sm.full[slot]);
  TTB_DCLK2(4);
  // 2. scalars
  double sg[4] = {0.0, 0.0, 0.0, 0.0}, aj = 0.0;
#pragma unroll
  for (int s = 0; s < RPL; ++s) {
    double x = A[s][OT];
    if (HEAD && C::pivot_slot(s)) {
      const int r = C::row(s, lr);
      if (r == j) aj = x;
      x = r > j ? x : 0.0;
    }
    sg[s & 3] = fma(x, x, sg[s & 3]);
  }
  double sig = (sg[0] + sg[1]) + (sg[2] + sg[3]);
#pragma unroll
  for (int off = LR / 2; off > 0; off >>= 1) {
    sig += __shfl_xor_sync(0xffffffffu, sig, off);
    if (HEAD) aj += __shfl_xor_sync(0xffffffffu, aj, off);
  }
  TTB_DCLK2(5);
  const double alpha = HEAD ? aj : alpha_r;
  double beta, tau, scal, bv;
  reflector_scalars<HEAD>(alpha, sig, beta, tau, scal, bv);
  TTB_DCLK2(6);
  if (mine && lr == 0) {  // the owner group holds this column's sigma / alpha
    double2* scp = reinterpret_cast<double2*>(sm.sc[slot]);
    scp[0] = make_double2(tau, scal);
    scp[1] = make_double2(bv, beta);
    TTB_DCLK2(12);
    mbar_arrive(&sm.fulls[slot]);
    TTB_DCLK2(13);
    sm.taus[j] = tau;  // off the chain: read at the end of the tile
    if (!HEAD) sm.Rs[j + BM * j] = beta;
  }
  TTB_DCLK2(7);
  // 3. own column becomes the stored Householder vector (R on top for head)
  if (mine) {
#pragma unroll
    for (int s = 0; s < RPL; ++s) {
      const double x = A[s][OT];
      if (HEAD && C::pivot_slot(s)) {  // rows > j: v = scal x (x_r for r > j); row j keeps R's beta
        const int r = C::row(s, lr);
        A[s][OT] = r > j ? x * scal : (r == j ? beta : x);
      } else {
        A[s][OT] = x * scal;
      }
    }
  }
}

// register-slot index clamped to the configuration (dispatch helpers)
template <class C, int T>
constexpr int kSlot = T < C::CPL ? T : C::CPL - 1;

template <class C, bool HEAD>
__device__ __forceinline__ void publish(double (&A)[C::RPL][C::CPL], int j, int gj, TileSmem<C>& sm) {
  static_assert(C::CPL <= 8, "slot dispatch handles CPL <= 8");
  switch (C::owner_slot(j)) {
    case 0: publish_slot<C, HEAD, 0>(A, j, gj, sm); break;
    case 1: publish_slot<C, HEAD, kSlot<C, 1>>(A, j, gj, sm); break;
    case 2: publish_slot<C, HEAD, kSlot<C, 2>>(A, j, gj, sm); break;
    case 3: publish_slot<C, HEAD, kSlot<C, 3>>(A, j, gj, sm); break;
    case 4: publish_slot<C, HEAD, kSlot<C, 4>>(A, j, gj, sm); break;
    case 5: publish_slot<C, HEAD, kSlot<C, 5>>(A, j, gj, sm); break;
    case 6: publish_slot<C, HEAD, kSlot<C, 6>>(A, j, gj, sm); break;
    default: publish_slot<C, HEAD, kSlot<C, 7>>(A, j, gj, sm); break;
  }
}

// finish column slot T for reflector j: a -= c x (+ head pivot-row fix)
// RW: also update the chain triangle's entry R[j, k] (the producer's slot does
// that after the next column is published: it is off the column chain)
template <class C, bool HEAD, int T, bool RW = true>
__device__ __forceinline__ void update_slot(double (&A)[C::RPL][C::CPL], const double (&xr)[C::RPL], double c,
                                            double beta, double rcoef, int k, int j, int b, int lr, TileSmem<C>& sm) {
  if (k > j && k < b) {
#pragma unroll
    for (int s = 0; s < C::RPL; ++s) {
      double a = fma(-c, xr[s], A[s][T]);
      if (HEAD && C::pivot_slot(s) && C::row(s, lr) == j) a = fma(c, beta, a);
      A[s][T] = a;
    }
    if (RW && !HEAD && lr == 0) sm.Rs[j + C::BMAX * k] -= rcoef;
  }
}

// Householder QR of one register tile.  HEAD: pivots are tile rows 0..b-1
// (plain QR); otherwise pivots are rows of the chain triangle sm.Rs (the
// stacked [R; A] factorization).  gbase: number of columns this CTA has
// already pushed through the ring (phase bookkeeping across tiles).
// No CTA-wide barrier per column: consumers wait on the ring's full /
// fulls barriers, the next producer on the empty barrier (slot reuse).
// On exit: A holds the Householder vectors (head: R in the upper triangle
// of rows < b, beta on the diagonal), sm.Gs holds T, sm.Rs holds R (body).
// Hooks of the column loop (all no-ops for leaf tiles):
//  h.feed(A, j0): called by every warp before any use of rows >= j0 (at the
//    start and before each chunk of kTreeChunk columns): loads rows j0.. of
//    late-arriving inputs into the register tile;
//  h.pre(j) / h.post(A, j): start / end of column step j in every warp;
//    post runs after the warp applied reflector j to all its columns, so
//    row j of R is final in this warp's columns.
struct NoHooks {
  template <class T>
  __device__ __forceinline__ void feed(T&, int) {}
  __device__ __forceinline__ void pre(int) {}
  template <class T>
  __device__ __forceinline__ void post(T&, int) {}
};
#ifndef TTB_TREE_CHUNK
#define TTB_TREE_CHUNK 4
#endif
constexpr int kTreeChunk = TTB_TREE_CHUNK;

// Debug-only tile-phase stamps of the leaf (CTA 0, thread 0): build with
// NVCC_EXTRA=-DTTB_DEBUG_TILE, read back with ttb_dbg_tile.
#ifdef TTB_DEBUG_TILE
static __device__ long long g_tile_clk[64 * 8];
#define TTB_TILE_CLK(t, ph)                                                                  \
  do {                                                                                       \
    if (blockIdx.x == 0 && threadIdx.x == 0 && (t) < 64) g_tile_clk[(t) * 8 + (ph)] = clock64(); \
  } while (0)
#else
#define TTB_TILE_CLK(t, ph) \
  do {                      \
  } while (0)
#endif

template <class C, bool HEAD, class H = NoHooks>
__device__ void tile_qr_t(double (&A)[C::RPL][C::CPL], int b, TileSmem<C>& sm, int gbase, H&& h = H()) {
  constexpr int LR = C::LR, RPL = C::RPL, CPL = C::CPL, BM = C::BMAX;
  constexpr int T1 = CPL > 1 ? 1 : 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lc = lane / LR, lr = lane % LR;
  int kk[CPL];
#pragma unroll
  for (int t = 0; t < CPL; ++t) kk[t] = col_of<C>(t, warp, lc);

  h.feed(A, 0);
  if (warp == C::owner_warp(0)) {
    if (gbase >= kRing) mbar_wait(&sm.empty[gbase % kRing], ((gbase / kRing) - 1) & 1);
    publish<C, HEAD>(A, 0, gbase, sm);
  }
  for (int j = 0; j < b; ++j) {
    TTB_DCLK(0);
    h.pre(j);
    if ((j + 1) % kTreeChunk == 0 && j + 1 < b) h.feed(A, j + 1);  // before column j+1 is published
    const int gj = gbase + j;
    const int slot = gj % kRing;
    const int nx = j + 1;
    const bool producer = (nx < b) && (warp == C::owner_warp(nx));
    mbar_wait(&sm.full[slot], (gj / kRing) & 1);
    TTB_DCLK(1);
    double xr[RPL];
#pragma unroll
    for (int s = 0; s < RPL; s += 2) {
      const double2 p = *reinterpret_cast<const double2*>(&sm.vring[slot][C::row(s, lr)]);
      xr[s] = p.x;
      xr[s + 1] = p.y;
    }
    double p[CPL], q[CPL];
#pragma unroll
    for (int t = 0; t < CPL; ++t) {
#ifdef TTB_EXPT_NODOT  // timing experiment only
      if (!producer) { p[t] = 0.0; q[t] = 0.0; continue; }
#endif
      double a0 = 0.0, a1 = 0.0, qa = 0.0;
#pragma unroll
      for (int s = 0; s < RPL; ++s) {
        if (s & 1) a1 = fma(xr[s], A[s][t], a1); else a0 = fma(xr[s], A[s][t], a0);
        if (HEAD && C::pivot_slot(s) && C::row(s, lr) == j) qa = A[s][t];
      }
      p[t] = a0 + a1;
      q[t] = qa;
    }
#pragma unroll
    for (int off = LR / 2; off > 0; off >>= 1) {
#pragma unroll
      for (int t = 0; t < CPL; ++t) {
        p[t] += __shfl_xor_sync(0xffffffffu, p[t], off);
        if (HEAD) q[t] += __shfl_xor_sync(0xffffffffu, q[t], off);
      }
    }
    if (producer && gj + 1 >= kRing) mbar_wait(&sm.empty[(gj + 1) % kRing], (((gj + 1) / kRing) - 1) & 1);
    mbar_wait(&sm.fulls[slot], (gj / kRing) & 1);
    const double2 sc01 = *reinterpret_cast<const double2*>(&sm.sc[slot][0]);
    const double2 sc23 = *reinterpret_cast<const double2*>(&sm.sc[slot][2]);
    const double tau = sc01.x, scal = sc01.y, beta = sc23.x;
    TTB_DCLK(2);
    double rjk[CPL];
#pragma unroll
    for (int t = 0; t < CPL; ++t) rjk[t] = (!HEAD && kk[t] > j && kk[t] < b) ? sm.Rs[j + BM * kk[t]] : 0.0;
    double d[CPL], c[CPL];
#pragma unroll
    for (int t = 0; t < CPL; ++t) {
      // d = v . a  (head: scal (x.a - beta a_j); body: R[j,k] + scal x.a)
      d[t] = HEAD ? scal * fma(-beta, q[t], p[t]) : fma(scal, p[t], rjk[t]);
      c[t] = tau * d[t] * scal;
    }
    const int tn = producer ? C::owner_slot(nx) : -1;
    TTB_DCLK(8);
#define TTB_UPD(T) update_slot<C, HEAD, T>(A, xr, c[T], beta, tau * d[T], kk[T], j, b, lr, sm)
    // the next column first (it is on the critical path): its update and its
    // publication in ONE dispatch on the owner slot (column nx > j always
    // needs the update), the R entry afterwards
#define TTB_UPDPUB(T)                                                                                    \
  do {                                                                                                   \
    update_slot<C, HEAD, T, false>(A, xr, c[T], beta, tau * d[T], kk[T], j, b, lr, sm);                  \
    TTB_DCLK(9);                                                                                         \
    publish_slot<C, HEAD, T>(A, nx, gj + 1, sm);                                                         \
    if (!HEAD && lr == 0 && kk[T] > j && kk[T] < b) sm.Rs[j + BM * kk[T]] -= tau * d[T];                 \
  } while (0)
    if (producer) {
      switch (tn) {
        case 0: TTB_UPDPUB(0); break;
        case 1: TTB_UPDPUB(T1); break;
        case 2: TTB_UPDPUB((kSlot<C, 2>)); break;
        case 3: TTB_UPDPUB((kSlot<C, 3>)); break;
        case 4: TTB_UPDPUB((kSlot<C, 4>)); break;
        case 5: TTB_UPDPUB((kSlot<C, 5>)); break;
        case 6: TTB_UPDPUB((kSlot<C, 6>)); break;
        default: TTB_UPDPUB((kSlot<C, 7>)); break;
      }
      TTB_DCLK(3);
    }
#undef TTB_UPDPUB
    __syncwarp();  // slot gj consumed by every lane of this warp (x and scalars are in registers)
    if (lane == 0) mbar_arrive(&sm.empty[slot]);
#ifndef TTB_EXPT_NOUPD  // timing experiment only: skip the off-critical-path updates
    if (tn != 0) TTB_UPD(0);
    if (CPL > 1 && tn != 1) TTB_UPD(T1);
    if (CPL > 2 && tn != 2) TTB_UPD((kSlot<C, 2>));
    if (CPL > 3 && tn != 3) TTB_UPD((kSlot<C, 3>));
    if (CPL > 4 && tn != 4) TTB_UPD((kSlot<C, 4>));
    if (CPL > 5 && tn != 5) TTB_UPD((kSlot<C, 5>));
    if (CPL > 6 && tn != 6) TTB_UPD((kSlot<C, 6>));
    if (CPL > 7 && tn != 7) TTB_UPD((kSlot<C, 7>));
#endif
#undef TTB_UPD
#pragma unroll
    for (int t = 0; t < CPL; ++t)
      if (kk[t] < j && lr == 0) sm.Gs[kk[t] + BM * j] = d[t];
    h.post(A, j);
  }
  TTB_TILE_CLK(gbase / (b > 0 ? b : 1), 4);
  C::sync();
  // T = (diag(1/tau) + striu(V^T V))^{-1} is formed by the caller (build_T)
  // after the register tile was stored: the tile's registers are then free
  // for the MMA fragments (keeping them live across build_T cost the column
  // loop ~10 % through register pressure)
}

template <class C>
__device__ __forceinline__ void tile_qr(double (&A)[C::RPL][C::CPL], int b, bool head, TileSmem<C>& sm, int gbase) {
  if (head) tile_qr_t<C, true>(A, b, sm, gbase);
  else tile_qr_t<C, false>(A, b, sm, gbase);
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
      const int r = C::row(s, lr);
      double v = A[s][t];
      if (head) v = r < k ? 0.0 : (r == k ? 1.0 : v);
      Y[r + (int64_t)ldy * k] = v;
    }
  }
}

// Leaf Householder vectors in global memory, unit-major: a tile of MC rows is
// MC / kYUnit units of kYUnit rows, each unit column-major with the padded
// leading dimension kYLd, so one unit is ONE contiguous block (a single bulk
// copy for the apply product) whose shared-memory image has conflict-free
// MMA fragment loads (kYLd = 4 mod 16).
constexpr int kYUnit = 128;
constexpr int kYLd = kYUnit + 4;
__host__ __device__ __forceinline__ int64_t y_tile_stride(int mc, int b) { return (int64_t)(mc / kYUnit) * b * kYLd; }
__host__ __device__ __forceinline__ int64_t y_index(int r, int k, int b) {
  return ((int64_t)(r / kYUnit) * b + k) * kYLd + (r % kYUnit);
}

template <class C>
__device__ void store_Y_units(const double (&A)[C::RPL][C::CPL], int b, bool head, double* Y) {
  static_assert(C::MC % kYUnit == 0, "leaf tiles are whole units");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lc = lane / C::LR, lr = lane % C::LR;
#pragma unroll
  for (int t = 0; t < C::CPL; ++t) {
    const int k = col_of<C>(t, warp, lc);
    if (k >= b) continue;
    // rows come in pairs (2 lr, 2 lr + 1): one 16-byte store per pair
#pragma unroll
    for (int s = 0; s < C::RPL; s += 2) {
      const int r = C::row(s, lr);
      double v0 = A[s][t], v1 = A[s + 1][t];
      if (head) {
        v0 = r < k ? 0.0 : (r == k ? 1.0 : v0);
        v1 = r + 1 < k ? 0.0 : (r + 1 == k ? 1.0 : v1);
      }
      *reinterpret_cast<double2*>(&Y[y_index(r, k, b)]) = make_double2(v0, v1);
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
      const int r = C::row(s, lr);
      if (r < b) sm.Rs[r + C::BMAX * k] = (r <= k) ? A[s][t] : 0.0;
    }
  }
}

}  // namespace ttb
