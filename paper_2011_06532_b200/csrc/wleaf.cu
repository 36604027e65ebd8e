// Team-pipelined TSQR leaf (the tsqr_leaf kernel class) and its apply
// kernels.  Reference: ttpar tsqr.py:103-130 (local_qr: dgeqrf of the local
// block) and tsqr.py:248-327 (apply of the implicit Q).
//
// Why: the column loop of a Householder QR is a dependency chain (pivot
// column -> norm -> sqrt / reciprocal -> dot products -> update -> next pivot
// column).  The CTA-wide column pipeline (tsqr.cuh tile_qr_t) pays ~1.8k
// cycles per column for 256 rows x b columns of work per SM.  Here the chain
// is short and there are several of them per SM:
//
//  * a TEAM (two warps for 32 < b <= 64, one for b <= 32) factors a 64-row
//    tile held in registers, TRANSPOSED: lane = column, 64 rows per lane.
//    Per column j the owner lane publishes its raw column x through shared
//    memory; every lane forms p = x . a for its own column with plain FMAs
//    (no shuffle reductions: the owner's p IS |x|^2), the reflector scalars
//    follow from (alpha, |x|^2), and every lane updates its own column.  The
//    only cross-warp traffic is x and (sigma, alpha), guarded by mbarriers.
//  * the CTA's chain of tiles [R_{t-1}; A_t] is dealt round-robin to NTEAM
//    teams that run as a SYSTOLIC pipeline: team p needs row j of R_{t-1}
//    only at its column step j, and row j of R_{t-1} is final as soon as
//    team p-1 finished ITS step j.  Rows of R flow team to team through a
//    shared-memory ring (full / empty mbarriers), so NTEAM tiles are in
//    flight per SM, a few column steps apart, and the CTA still ends with
//    ONE triangle (the tree above is unchanged).
//  * the head tile (first 64 rows of the chain, the reference's dgeqrf pivot
//    rows) is a plain Householder QR in the same layout.
//
// Per tile the leaf writes Y (64 x b, unit-major with ld kWLDY; head tile
// unit lower trapezoidal) and U = T^{-1} = diag(1/tau) + striu(V^T V), with
// tau stored on U's diagonal.  The strictly upper entries v_m . v_j come out
// of the column loop for free: lanes whose column is already finished compute
// the same dot product against x.  No triangular inversion happens in the
// leaf; the apply's chain kernel solves with U instead of multiplying by T.
#include "ctx.cuh"
#include "dmma.cuh"
#include "prof.cuh"
#include "tsqr.cuh"

namespace ttb {

namespace wl {

constexpr int kXR = 4;  // pivot columns in flight inside a team
// R rows in flight between consecutive teams.  The ring into team 0 is only
// drained when team 0 starts its next tile, so with depth D the last team can
// run D rows ahead, the one before it 2D, ... and team 0 finishes its tile
// only if NTEAM * D >= b: D = ceil(64 / NTEAM) (no deadlock for any b <= 64,
// and no stall in steady state, where consecutive tiles start b / NTEAM
// column steps apart).
#ifndef TTB_WL_RING
#define TTB_WL_RING 2
#endif
template <int NTEAM>
constexpr int ring_depth() { return TTB_WL_RING * ((64 + NTEAM - 1) / NTEAM); }

#ifdef TTB_WL_CLK
// debug: per-phase clock stamps of CTA 0, local tile 1 of every team, every warp
__device__ long long g_wlclk[8][2][64][8];
#define WL_CLK(ph)                                                                              \
  do {                                                                                          \
    if (blockIdx.x == 0 && li == 1 && lane == 0 && j < 64) g_wlclk[team][wt][j][ph] = clock64(); \
  } while (0)
#else
#define WL_CLK(ph) \
  do {             \
  } while (0)
#endif

__host__ __device__ __forceinline__ int64_t ustride(int b) { return ((int64_t)b * b + 1) & ~1LL; }
__host__ __device__ __forceinline__ int64_t ystride(int b) { return (int64_t)b * kWLDY; }

// Register tile of a warp: 64 rows x 32 columns, lane = (rg, cg) with row
// group rg = lane / 8 (rows 16 rg .. 16 rg + 15) and column group cg =
// lane % 8 (columns 32 w + cg + 8 i, slot i = 0..3).  Column dot products
// are partial over a lane's 16 rows and reduced over the 4 row groups with
// two butterfly shuffles; the pivot column x reaches every lane through
// shared memory, but each lane loads only its own 16 rows (a quarter of the
// column) and keeps them in registers for the update.
constexpr int kRG = 4;         // row groups
constexpr int kRR = 16;        // rows per lane
constexpr int kSL = 4;         // column slots per lane
constexpr int kXLD = kRR + 2;  // row-group stride of a published column (bank-conflict free)

template <int NTEAM>
struct Sm {
  double x[NTEAM][kXR][kRG * kXLD];
  double sg[NTEAM][kXR][2];
  double rin[NTEAM][ring_depth<NTEAM>()][64];
  unsigned long long xfull[NTEAM][kXR], sfull[NTEAM][kXR], xempty[NTEAM][kXR];
  unsigned long long rfull[NTEAM][ring_depth<NTEAM>()], rempty[NTEAM][ring_depth<NTEAM>()];
};

// v[s] for a warp-uniform runtime s
__device__ __forceinline__ double pick16(const double (&v)[kRR], int s) {
  double r = 0.0;
#pragma unroll
  for (int u = 0; u < kRR; ++u) r = (u == s) ? v[u] : r;
  return r;
}
__device__ __forceinline__ double pick4(const double (&v)[kSL], int i) {
  return i == 0 ? v[0] : i == 1 ? v[1] : i == 2 ? v[2] : v[3];
}

__device__ __forceinline__ double2 lds2(const double* p) { return *reinterpret_cast<const double2*>(p); }

// the owner lanes (column group cgo) write slot I of their rows to x (head: rows <= j zeroed)
template <int I, bool HEAD>
__device__ __forceinline__ void publish_slot(const double (&A)[kSL][kRR], double* xb, int rg, int j) {
#pragma unroll
  for (int s = 0; s < kRR; s += 2) {
    double x0 = A[I][s], x1 = A[I][s + 1];
    if (HEAD) {
      x0 = rg * kRR + s > j ? x0 : 0.0;
      x1 = rg * kRR + s + 1 > j ? x1 : 0.0;
    }
    *reinterpret_cast<double2*>(xb + rg * kXLD + s) = make_double2(x0, x1);
  }
}

// One tile of a team.  HEAD: plain QR, pivots are rows 0..b-1 of the tile.
// Otherwise the stacked [R_{t-1}; A_t]: row j of R_{t-1} arrives through
// this team's ring at step j.  Row j of the new R leaves through the next
// team's ring (or to global memory for the chain's last tile).
template <int NWT, int NTEAM, bool HEAD>
__device__ __forceinline__ void tile(Sm<NTEAM>& sm, const Panel& P, int b, int rs, int64_t cnt, int64_t s0,
                                     int64_t r0, int nr, int li, int team, bool last, double* __restrict__ Yt,
                                     double* __restrict__ Ut, double* __restrict__ Rout) {
  constexpr int kRD = ring_depth<NTEAM>();
  const int lane = threadIdx.x & 31, wt = (threadIdx.x >> 5) % NWT;
  const int rg = lane >> 3, cg = lane & 7;
  const int nt = team + 1 == NTEAM ? 0 : team + 1;
  int colv[kSL];
#pragma unroll
  for (int i = 0; i < kSL; ++i) colv[i] = wt * 32 + cg + 8 * i;
  double A[kSL][kRR];
  {
    int64_t si, w;
    wrow(P.trans, r0 + rg * kRR, cnt, rs, si, w);
#pragma unroll
    for (int s = 0; s < kRR; ++s) {
      const bool rok = rg * kRR + s < nr;
      if (P.kron.x) {
#pragma unroll
        for (int i = 0; i < kSL; ++i) A[i][s] = (rok && colv[i] < b) ? P.load(w, s0 + si, colv[i]) : 0.0;
      } else {
        const int64_t ra = P.addr(w, s0 + si, 0);
        const int64_t cst = P.trans ? 1 : P.rl * P.I;
#pragma unroll
        for (int i = 0; i < kSL; ++i) A[i][s] = (rok && colv[i] < b) ? __ldg(P.base + ra + cst * colv[i]) : 0.0;
      }
      wrow_next(P.trans, cnt, rs, si, w);
    }
  }
  const int cs = team == 0 ? li - 1 : li;  // ring sequence consumed by a body tile
  double myscal[kSL] = {0.0, 0.0, 0.0, 0.0};
  for (int j = 0; j < b; ++j) {
    const int ow = NWT == 2 ? (j >> 5) : 0;
    const bool own = wt == ow;
    const int jc = j & 31, cgo = jc & 7, io = jc >> 3;
    const int xs = li * b + j;
    const int xsl = xs % kXR;
    const unsigned xph = (unsigned)(xs / kXR) & 1u;
    double* xb = sm.x[team][xsl];
    WL_CLK(0);
    // 1. the owner column group publishes its raw column (head: rows <= j zeroed)
    if (own) {
      if (NWT == 2 && xs >= kXR) mbar_wait(&sm.xempty[team][xsl], (unsigned)((xs / kXR) - 1) & 1u);
      if (cg == cgo) {
        switch (io) {
          case 0: publish_slot<0, HEAD>(A, xb, rg, j); break;
          case 1: publish_slot<1, HEAD>(A, xb, rg, j); break;
          case 2: publish_slot<2, HEAD>(A, xb, rg, j); break;
          default: publish_slot<3, HEAD>(A, xb, rg, j); break;
        }
      }
      __syncwarp();
      if (NWT == 2 && lane == 0) mbar_arrive(&sm.xfull[team][xsl]);
    } else {
      mbar_wait(&sm.xfull[team][xsl], xph);
    }
    WL_CLK(1);
    // 2. partial dots over this lane's rows, reduced over the row groups
    double xr[kRR];
#pragma unroll
    for (int s = 0; s < kRR; s += 2) {
      const double2 u = lds2(xb + rg * kXLD + s);
      xr[s] = u.x;
      xr[s + 1] = u.y;
    }
    double pp[kSL];
#pragma unroll
    for (int i = 0; i < kSL; ++i) {
      double a0 = 0.0, a1 = 0.0;
      if (wt * 32 + 8 * i < b) {
#pragma unroll
        for (int s = 0; s < kRR; s += 2) {
          a0 = fma(xr[s], A[i][s], a0);
          a1 = fma(xr[s + 1], A[i][s + 1], a1);
        }
      }
      pp[i] = a0 + a1;
    }
#pragma unroll
    for (int i = 0; i < kSL; ++i) pp[i] += __shfl_xor_sync(0xffffffffu, pp[i], 8);
#pragma unroll
    for (int i = 0; i < kSL; ++i) pp[i] += __shfl_xor_sync(0xffffffffu, pp[i], 16);
    WL_CLK(2);
    // 3. pivot-row entries q of this lane's columns and the pivot alpha
    double q[kSL], alpha = 0.0;
    if (HEAD) {
      const int rgj = j / kRR, sj = j % kRR;
#pragma unroll
      for (int i = 0; i < kSL; ++i) {
        const double v = pick16(A[i], sj);
        q[i] = __shfl_sync(0xffffffffu, v, rgj * 8 + cg);
      }
    } else {
      const int gs = cs * b + j, rsl = gs % kRD;
      mbar_wait(&sm.rfull[team][rsl], (unsigned)(gs / kRD) & 1u);
      const double* rr = sm.rin[team][rsl];
#pragma unroll
      for (int i = 0; i < kSL; ++i) q[i] = rr[colv[i]];
      alpha = rr[j];
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.rempty[team][rsl]);
    }
    WL_CLK(3);
    double sigma;
    if (own) {
      sigma = __shfl_sync(0xffffffffu, pick4(pp, io), cgo);
      if (HEAD) alpha = __shfl_sync(0xffffffffu, pick4(q, io), cgo);
      if (NWT == 2) {
        if (lane == 0) {
          sm.sg[team][xsl][0] = sigma;
          sm.sg[team][xsl][1] = alpha;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.sfull[team][xsl]);
      }
    } else {
      mbar_wait(&sm.sfull[team][xsl], xph);
      sigma = sm.sg[team][xsl][0];
      if (HEAD) alpha = sm.sg[team][xsl][1];
    }
    WL_CLK(4);
    // 4. reflector v = e_j + scal x (identical in every lane of the team)
    double beta, tau, scal, bv;
    reflector_scalars<false>(alpha, sigma, beta, tau, scal, bv);
    double d[kSL], rv[kSL];
#pragma unroll
    for (int i = 0; i < kSL; ++i) {
      const int col = colv[i];
      d[i] = fma(scal, pp[i], q[i]);  // v . a  (finished columns: v_col . v_j / scal_col)
      if (col == j) myscal[i] = scal;
      rv[i] = col > j ? fma(-tau, d[i], q[i]) : (col == j ? beta : 0.0);
      if (rg == 0 && col < b) {
        if (col < j) Ut[col + (int64_t)b * j] = myscal[i] * d[i];
        else if (col == j) Ut[col + (int64_t)b * j] = tau;
      }
    }
    WL_CLK(5);
    // 5. row j of the new R
    if (last) {
      if (rg == 0) {
#pragma unroll
        for (int i = 0; i < kSL; ++i)
          if (colv[i] < b) Rout[j + (int64_t)b * colv[i]] = rv[i];
      }
    } else {
      const int ps = li * b + j, psl = ps % kRD;
      if (ps >= kRD) mbar_wait(&sm.rempty[nt][psl], (unsigned)((ps / kRD) - 1) & 1u);
      if (rg == 0) {
#pragma unroll
        for (int i = 0; i < kSL; ++i) sm.rin[nt][psl][colv[i]] = rv[i];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.rfull[nt][psl]);
    }
    WL_CLK(6);
    // 6. trailing update of the slots that still hold columns > j
#pragma unroll
    for (int i = 0; i < kSL; ++i) {
      if (wt * 32 + 8 * i + 7 > j && wt * 32 + 8 * i < b) {
        const double c = (colv[i] > j && colv[i] < b) ? tau * d[i] * scal : 0.0;
#pragma unroll
        for (int s = 0; s < kRR; ++s) A[i][s] = fma(-c, xr[s], A[i][s]);
      }
    }
    if (NWT == 2 && !own) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.xempty[team][xsl]);
    }
    WL_CLK(7);
  }
  // Householder vectors: raw columns scaled (head: unit lower trapezoid)
#pragma unroll
  for (int i = 0; i < kSL; ++i) {
    const int col = colv[i];
    if (col >= b) continue;
    double* yc = Yt + (int64_t)col * kWLDY + rg * kRR;
#pragma unroll
    for (int s = 0; s < kRR; s += 2) {
      const int r = rg * kRR + s;
      double y0 = myscal[i] * A[i][s], y1 = myscal[i] * A[i][s + 1];
      if (HEAD) {
        y0 = r < col ? 0.0 : (r == col ? 1.0 : y0);
        y1 = r + 1 < col ? 0.0 : (r + 1 == col ? 1.0 : y1);
      }
      *reinterpret_cast<double2*>(yc + s) = make_double2(y0, y1);
    }
  }
}

template <int NWT, int NTEAM>
__global__ void __launch_bounds__(NWT* NTEAM * 32, 1)
    wleaf_kernel(Panel P, WPlan plan, double* __restrict__ Yg, double* __restrict__ Ug, double* __restrict__ Rleaf) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Sm<NTEAM>& sm = *reinterpret_cast<Sm<NTEAM>*>(smem_raw);
  const int g = blockIdx.x;
  const int b = plan.b, rs = plan.rs;
  const int64_t cnt = plan.count(g), s0 = plan.start(g);
  const int ntiles = plan.tiles_of(cnt);
  const int64_t tb = plan.tile_base(g);
  const int team = (threadIdx.x >> 5) / NWT;
  if (threadIdx.x == 0) {
    for (int q = 0; q < NTEAM; ++q) {
      for (int s = 0; s < kXR; ++s) {
        mbar_init(&sm.xfull[q][s], 1);
        mbar_init(&sm.sfull[q][s], 1);
        mbar_init(&sm.xempty[q][s], 1);
      }
      for (int s = 0; s < ring_depth<NTEAM>(); ++s) {
        mbar_init(&sm.rfull[q][s], NWT);
        mbar_init(&sm.rempty[q][s], NWT);
      }
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  double* Rout = Rleaf + (int64_t)g * b * b;
  if (ntiles == 0) {  // an idle chain (a rank without slices): R = 0
    for (int idx = threadIdx.x; idx < b * b; idx += blockDim.x) Rout[idx] = 0.0;
    return;
  }
  const int64_t rows = cnt * rs;
  int li = 0;
  for (int t = team; t < ntiles; t += NTEAM, ++li) {
    const int64_t r0 = (int64_t)t * kWH;
    const int nr = (int)min64(kWH, rows - r0);
    double* Yt = Yg + (tb + t) * ystride(b);
    double* Ut = Ug + (tb + t) * ustride(b);
    const bool last = t == ntiles - 1;
    if (t == 0)
      tile<NWT, NTEAM, true>(sm, P, b, rs, cnt, s0, r0, nr, li, team, last, Yt, Ut, Rout);
    else
      tile<NWT, NTEAM, false>(sm, P, b, rs, cnt, s0, r0, nr, li, team, last, Yt, Ut, Rout);
  }
}

// ---------------------------------------------------------------------------
// apply, chains: one CTA per leaf chain walks its tiles in reverse,
//   u_t = U_t^{-1} z_t,  z_{t-1} = z_t - u_t   (head: u_0 = U_0^{-1} V_top^T z_0)
// by a blocked back substitution: the 8 x 8 diagonal blocks of U are
// inverted first (independent of z), then per block (bottom up)
//   u_B = inv(U_BB) r_B,  r_A -= U_AB u_B  (rows above)
// U_t arrives by bulk copy two tiles ahead.
// ---------------------------------------------------------------------------
constexpr int kChainNT = 256;
constexpr int kSB = 8;  // solve block rows

struct ChainArgs {
  WPlan plan;
  const double* Y;
  const double* U;
  const double* zin;  // per chain b x k (ld b)
  const double* D;    // sign fix (no tree above) or null
  int k;
  int ldu;            // row stride of u (>= k)
  double* u;          // per tile b x ldu, row-major
  double* z0;         // per chain b x k: the head tile's input
};

__device__ __forceinline__ void bulk_g2s_w(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_load_w(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  constexpr unsigned kChunk = 32768;
  for (unsigned off = 0; off < bytes; off += kChunk) {
    const unsigned n = bytes - off < kChunk ? bytes - off : kChunk;
    bulk_g2s_w((char*)dst + off, (const char*)src + off, n, bar);
  }
}

__global__ void __launch_bounds__(kChainNT) wchain_kernel(ChainArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int g = blockIdx.x;
  const WPlan& pl = a.plan;
  const int b = pl.b, k = a.k, ldz = k | 1;
  const int64_t ust = ustride(b);
  const int nbk = (b + kSB - 1) / kSB;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem_raw);
  double* const Ub0 = reinterpret_cast<double*>(smem_raw + 64);
  double* const Ub1 = Ub0 + ust;
  double* Z = Ub1 + ust;            // b x ldz: z of the current tile
  double* Rr = Z + (int64_t)b * ldz;  // residual / right-hand side
  double* Us = Rr + (int64_t)b * ldz;  // u of the current tile
  double* Di = Us + (int64_t)b * ldz;  // nbk blocks of kSB x kSB: inverses of the diagonal blocks
  const int64_t cnt = pl.count(g);
  const int ntiles = pl.tiles_of(cnt);
  const int64_t tb = pl.tile_base(g);
  if (ntiles == 0) return;
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int idx = threadIdx.x; idx < b * k; idx += kChainNT) {
    const int i = idx % b, c = idx / b;
    const double dd = a.D ? a.D[i] : 1.0;
    Z[i * ldz + c] = dd * a.zin[(int64_t)g * b * k + idx];
  }
  __syncthreads();
  const unsigned ubytes = (unsigned)(ust * 8);
  if (threadIdx.x == 0) {
    bulk_load_w(Ub0, a.U + (tb + ntiles - 1) * ust, ubytes, &bars[0]);
    if (ntiles > 1) bulk_load_w(Ub1, a.U + (tb + ntiles - 2) * ust, ubytes, &bars[1]);
  }
  for (int t = ntiles - 1, it = 0; t >= 0; --t, ++it) {
    const int cur = it & 1;
    const double* Uc = cur ? Ub1 : Ub0;
    // right-hand side: z_t (body) or V_top^T z_0 (head)
    if (t == 0) {
      const double* Y0 = a.Y + tb * ystride(b);
      for (int idx = threadIdx.x; idx < b * k; idx += kChainNT) {
        const int m = idx / k, c = idx - m * k;
        const double* ym = Y0 + (int64_t)m * kWLDY;  // column m of V_top: unit at row m
        double s = Z[m * ldz + c];
        for (int l = m + 1; l < b; ++l) s = fma(ym[l], Z[l * ldz + c], s);
        Rr[m * ldz + c] = s;
      }
    } else {
      for (int idx = threadIdx.x; idx < b * k; idx += kChainNT) {
        const int i = idx / k, c = idx - i * k;
        Rr[i * ldz + c] = Z[i * ldz + c];
      }
    }
    mbar_wait(&bars[cur], (unsigned)(it >> 1) & 1u);
    // inverses of the diagonal blocks: column c of block q by back substitution
    // (U's diagonal holds tau: the diagonal of U is 1/tau)
    for (int idx = threadIdx.x; idx < nbk * kSB; idx += kChainNT) {
      const int q = idx / kSB, c = idx % kSB;
      const int i0 = q * kSB, n = min(kSB, b - i0);
      double x[kSB];
#pragma unroll
      for (int i = kSB - 1; i >= 0; --i) {
        double s = (i == c) ? 1.0 : 0.0;
#pragma unroll
        for (int m = i + 1; m < kSB; ++m)
          if (m < n && i < n) s = fma(-Uc[(i0 + i) + (int64_t)b * (i0 + m)], x[m], s);
        x[i] = (i < n && i <= c) ? Uc[(i0 + i) + (int64_t)b * (i0 + i)] * s : 0.0;
      }
#pragma unroll
      for (int i = 0; i < kSB; ++i) Di[(q * kSB + i) * kSB + c] = x[i];
    }
    __syncthreads();
    for (int q = nbk - 1; q >= 0; --q) {
      const int i0 = q * kSB, n = min(kSB, b - i0);
      // u_B = inv(U_BB) r_B
      for (int idx = threadIdx.x; idx < n * k; idx += kChainNT) {
        const int i = idx / k, c = idx - i * k;
        const double* di = Di + (q * kSB + i) * kSB;
        double s = 0.0;
        for (int m = i; m < n; ++m) s = fma(di[m], Rr[(i0 + m) * ldz + c], s);
        Us[(i0 + i) * ldz + c] = s;
      }
      __syncthreads();
      // r_A -= U_AB u_B for the rows above
      for (int idx = threadIdx.x; idx < i0 * k; idx += kChainNT) {
        const int i = idx / k, c = idx - i * k;
        double s = Rr[i * ldz + c];
        for (int m = 0; m < n; ++m) s = fma(-Uc[i + (int64_t)b * (i0 + m)], Us[(i0 + m) * ldz + c], s);
        Rr[i * ldz + c] = s;
      }
      __syncthreads();
    }
    double* ut = a.u + (tb + t) * (int64_t)b * a.ldu;
    if (t == 0) {
      for (int idx = threadIdx.x; idx < b * k; idx += kChainNT) {
        const int i = idx / k, c = idx - i * k;
        ut[(int64_t)i * a.ldu + c] = Us[i * ldz + c];
        a.z0[(int64_t)g * b * k + i + (int64_t)b * c] = Z[i * ldz + c];
      }
    } else {
      for (int idx = threadIdx.x; idx < b * k; idx += kChainNT) {
        const int i = idx / k, c = idx - i * k;
        const double uv = Us[i * ldz + c];
        ut[(int64_t)i * a.ldu + c] = uv;
        Z[i * ldz + c] -= uv;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0 && t >= 2) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      bulk_load_w(const_cast<double*>(Uc), a.U + (tb + t - 2) * ust, ubytes, &bars[cur]);
    }
  }
}

// ---------------------------------------------------------------------------
// apply, products: out_t = -Y_t u_t (+ z_0 on the head tile's rows < b).
// Persistent (one CTA per SM); a work unit is one 64-row tile, Y_t and u_t
// stream into shared memory through an S-stage bulk-copy pipeline.
// ---------------------------------------------------------------------------
constexpr int kProdNT = 256;

struct ProductArgs {
  WPlan plan;
  const double* Y;
  const double* u;
  const double* z0;
  int k, ldu, stages;
  Panel out;
};

__global__ void __launch_bounds__(kProdNT, 1) wproduct_kernel(ProductArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int NW = kProdNT / 32;
  const WPlan& pl = a.plan;
  const int b = pl.b, k = a.k, rs = pl.rs, ldu = a.ldu;
  const int64_t ys = ystride(b), us = (int64_t)b * ldu;
  const int S = a.stages;
  const int64_t ntiles = pl.total_tiles();
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem_raw);
  double* Ysb = reinterpret_cast<double*>(smem_raw + 128);
  double* Usb = Ysb + S * ys;
  int64_t* rowoff = reinterpret_cast<int64_t*>(Usb + S * us);  // kWH entries
  const unsigned ybytes = (unsigned)(ys * 8), ubytes = (unsigned)(us * 8);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int64_t tile, int st) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&bar[st])),
                   "r"(ybytes + ubytes)
                   : "memory");
      bulk_g2s_w(Ysb + st * ys, a.Y + tile * ys, ybytes, &bar[st]);
      bulk_g2s_w(Usb + st * us, a.u + tile * us, ubytes, &bar[st]);
    }
  };
  int64_t tile = blockIdx.x;
  for (int s = 0; s < S - 1; ++s)
    if (tile + (int64_t)s * gridDim.x < ntiles) issue(tile + (int64_t)s * gridDim.x, s);
  const int64_t cstride = a.out.trans ? 1 : a.out.rl * a.out.I;
  for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
    const int st = it % S;
    const int64_t nxt = tile + (int64_t)(S - 1) * gridDim.x;
    if (nxt < ntiles) {  // its stage was released by the barrier that ended the previous tile
      if (threadIdx.x == 0) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      issue(nxt, (it + S - 1) % S);
    }
    int g;
    int64_t t;
    pl.tile_of(tile, g, t);
    const int64_t cnt = pl.count(g), s0 = pl.start(g);
    const int64_t r0 = t * kWH;
    const int rows = (int)min64(kWH, cnt * rs - r0);
    const bool head = t == 0;
    const double* z0 = a.z0 + (int64_t)g * b * k;
    for (int m = threadIdx.x; m < rows; m += kProdNT) {
      int64_t si, w;
      wrow(a.out.trans, r0 + m, cnt, rs, si, w);
      rowoff[m] = a.out.addr(w, s0 + si, 0);
    }
    mbar_wait(&bar[st], (unsigned)(it / S) & 1u);
    __syncthreads();
    const double* Ys = Ysb + st * ys;
    const double* Us = Usb + st * us;
    double* ob = a.out.base;
    cta_dmma(
        rows, k, b, NW, [&](int m, int l) { return l < b ? Ys[l * kWLDY + m] : 0.0; },
        [&](int l, int n) { return (l < b && n < k) ? Us[l * ldu + n] : 0.0; },
        [&](int m, int n, double v) {
          const double base = (head && m < b) ? z0[m + (int64_t)b * n] : 0.0;
          ob[rowoff[m] + cstride * n] = base - v;
        });
    __syncthreads();
  }
}

}  // namespace wl

#ifdef TTB_WL_CLK
extern "C" int ttb_dbg_wlclk(long long* out) {
  return cudaMemcpyFromSymbol(out, wl::g_wlclk, sizeof(wl::g_wlclk)) == cudaSuccess ? 0 : 5;
}
#endif

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
int wleaf_teams(int b) { return b <= 32 ? 8 : 4; }

size_t wleaf_y_doubles(const WPlan& p) { return (size_t)(p.total_tiles() * wl::ystride(p.b)); }
size_t wleaf_u_doubles(const WPlan& p) { return (size_t)(p.total_tiles() * wl::ustride(p.b)); }

void launch_wleaf(Ctx& ctx, const Panel& panel, const WPlan& plan, double* Y, double* U, double* Rleaf) {
  if (plan.b <= 32) {
    constexpr int NWT = 1, NTEAM = 8;
    auto kern = wl::wleaf_kernel<NWT, NTEAM>;
    const size_t sm = sizeof(wl::Sm<NTEAM>);
    smem_attr((const void*)kern, sm);
    kern<<<plan.G, NWT * NTEAM * 32, sm, ctx.stream>>>(panel, plan, Y, U, Rleaf);
  } else {
    constexpr int NWT = 2, NTEAM = 4;
    auto kern = wl::wleaf_kernel<NWT, NTEAM>;
    const size_t sm = sizeof(wl::Sm<NTEAM>);
    smem_attr((const void*)kern, sm);
    kern<<<plan.G, NWT * NTEAM * 32, sm, ctx.stream>>>(panel, plan, Y, U, Rleaf);
  }
  TTB_LAUNCHED();
}

// u / z0 scratch: tiles * b * ldu + G * b * k doubles
void wleaf_apply_tail(Ctx& ctx, const WPlan& plan, const double* Y, const double* U, const double* zin,
                      const double* D, int k, const Panel& out, double* ubuf, double* z0buf) {
  const int b = plan.b;
  const int ldu = (k + 1) & ~1;
  wl::ChainArgs ca;
  ca.plan = plan;
  ca.Y = Y;
  ca.U = U;
  ca.zin = zin;
  ca.D = D;
  ca.k = k;
  ca.ldu = ldu;
  ca.u = ubuf;
  ca.z0 = z0buf;
  const int ldz = k | 1, nbk = (b + wl::kSB - 1) / wl::kSB;
  const size_t csm = 64 + (size_t)(2 * wl::ustride(b) + 3 * (int64_t)b * ldz + (int64_t)nbk * wl::kSB * wl::kSB) *
                              sizeof(double);
  smem_attr((const void*)wl::wchain_kernel, csm);
  {
    ProfScope ps("apply_chain", ctx.stream);
    wl::wchain_kernel<<<plan.G, wl::kChainNT, csm, ctx.stream>>>(ca);
    TTB_LAUNCHED();
  }
  wl::ProductArgs pa;
  pa.plan = plan;
  pa.Y = Y;
  pa.u = ubuf;
  pa.z0 = z0buf;
  pa.k = k;
  pa.ldu = ldu;
  pa.out = out;
  const size_t stage = (size_t)(wl::ystride(b) + (int64_t)b * ldu) * sizeof(double);
  pa.stages = (int)std::max<size_t>(2, std::min<size_t>(8, (200 * 1024) / stage));
  const size_t psm = 128 + (size_t)pa.stages * stage + kWH * sizeof(int64_t);
  smem_attr((const void*)wl::wproduct_kernel, psm);
  const int64_t ntiles = plan.total_tiles();
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ntiles, ctx.num_sms));
  ProfScope ps("apply_product", ctx.stream);
  wl::wproduct_kernel<<<grid, wl::kProdNT, psm, ctx.stream>>>(pa);
  TTB_LAUNCHED();
}

}  // namespace ttb
