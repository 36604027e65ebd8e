// Gram-sweep step of the TT inner product (ops.py:135-155):
//     W_n = sum_i  Y_n(i)^T  W_{n-1}  X_n(i)
// as one fused batched r x r x n contraction: the intermediate
// Z(i) = W X(i) lives only in shared memory (never in HBM).  Each CTA
// streams a run of slices in chunks (coalesced: for every right-rank index
// the (a, i) block of a chunk is contiguous in the F-order core), computes
// Z for the chunk, accumulates Y(i)^T Z(i) in per-thread register tiles,
// and writes one partial W; a second kernel sums the CTA partials in a
// fixed order (bitwise deterministic, no atomics).
#include "ops.cuh"
#include "wide.cuh"
#include "prof.cuh"

namespace ttb {

constexpr int kGrNT = 256;
constexpr int kGrSmemDoubles = 12 * 1024;  // 96 KB of chunk buffers per CTA
constexpr int kGrTM = 4, kGrTN = 4;

struct GramArgs {
  const double* W;  // rbl x ral
  const double* X;  // (ral, I, rar)
  const double* Y;  // (rbl, I, rbr)
  int ral, rar, rbl, rbr;
  int64_t I;
  int ns;           // slices per chunk
  int64_t per_cta;  // slices per CTA
  double* part;     // gridDim.x partials of rbr x rar
};

__global__ void __launch_bounds__(kGrNT, 2) gram_kernel(GramArgs a) {
  extern __shared__ __align__(16) double gsm[];
  const int ral = a.ral, rar = a.rar, rbl = a.rbl, rbr = a.rbr, ns = a.ns;
  double* Ws = gsm;                          // rbl x ral
  double* Xc = Ws + rbl * ral;               // ral x ns x rar
  double* Yc = Xc + (int64_t)ral * ns * rar; // rbl x ns x rbr
  double* Zc = Yc + (int64_t)rbl * ns * rbr; // rbl x ns x rar
  const int tid = threadIdx.x;
  for (int e = tid; e < rbl * ral; e += kGrNT) Ws[e] = a.W[e];

  // step-B tiling: output (rbr x rar) in TM x TN tiles, K split across groups
  const int tb_m = (rbr + kGrTM - 1) / kGrTM, tb_n = (rar + kGrTN - 1) / kGrTN;
  const int ntile = tb_m * tb_n;
  const int kgroups = max(1, kGrNT / ntile);
  const int my_tile = tid % ntile, my_kg = tid / ntile;
  const bool active_b = tid < ntile * kgroups;
  const int d0 = (my_tile % tb_m) * kGrTM, b0 = (my_tile / tb_m) * kGrTN;
  double acc[kGrTM][kGrTN];
#pragma unroll
  for (int u = 0; u < kGrTM; ++u)
#pragma unroll
    for (int v = 0; v < kGrTN; ++v) acc[u][v] = 0.0;

  const int64_t s_begin = (int64_t)blockIdx.x * a.per_cta;
  const int64_t s_end = min64(a.I, s_begin + a.per_cta);
  for (int64_t i0 = s_begin; i0 < s_end; i0 += ns) {
    const int nn = (int)min64(ns, s_end - i0);
    __syncthreads();
    // load X chunk: for each b, ral*nn contiguous doubles
    for (int64_t e = tid; e < (int64_t)ral * nn * rar; e += kGrNT) {
      const int64_t bq = e / (ral * nn), rem = e - bq * ral * nn;
      Xc[rem + (int64_t)ral * ns * bq] = a.X[rem + ral * (i0 + a.I * bq)];
    }
    for (int64_t e = tid; e < (int64_t)rbl * nn * rbr; e += kGrNT) {
      const int64_t dq = e / (rbl * nn), rem = e - dq * rbl * nn;
      Yc[rem + (int64_t)rbl * ns * dq] = a.Y[rem + rbl * (i0 + a.I * dq)];
    }
    __syncthreads();
    // step A: Z[c, (ii, b)] = sum_a W[c, a] X[a, (ii, b)]   (columns j = ii + ns*b)
    {
      const int tm = (rbl + kGrTM - 1) / kGrTM;
      const int ncols = ns * rar;
      const int tn = (ncols + kGrTN - 1) / kGrTN;
      for (int t = tid; t < tm * tn; t += kGrNT) {
        const int c0 = (t % tm) * kGrTM, j0 = (t / tm) * kGrTN;
        double z[kGrTM][kGrTN];
#pragma unroll
        for (int u = 0; u < kGrTM; ++u)
#pragma unroll
          for (int v = 0; v < kGrTN; ++v) z[u][v] = 0.0;
        for (int al = 0; al < ral; ++al) {
          double w[kGrTM], x[kGrTN];
#pragma unroll
          for (int u = 0; u < kGrTM; ++u) w[u] = (c0 + u < rbl) ? Ws[(c0 + u) + rbl * al] : 0.0;
#pragma unroll
          for (int v = 0; v < kGrTN; ++v) x[v] = (j0 + v < ncols) ? Xc[al + ral * (j0 + v)] : 0.0;
#pragma unroll
          for (int u = 0; u < kGrTM; ++u)
#pragma unroll
            for (int v = 0; v < kGrTN; ++v) z[u][v] = fma(w[u], x[v], z[u][v]);
        }
#pragma unroll
        for (int u = 0; u < kGrTM; ++u)
#pragma unroll
          for (int v = 0; v < kGrTN; ++v)
            if (c0 + u < rbl && j0 + v < ncols) Zc[(c0 + u) + rbl * (j0 + v)] = z[u][v];
      }
    }
    __syncthreads();
    // step B: acc[d, b] += sum_{kappa = c + rbl*ii} Y[kappa, d] Z[kappa, b]
    if (active_b) {
      const int K = rbl * nn;
      const int64_t ldk = (int64_t)rbl * ns;
      for (int kk = my_kg; kk < K; kk += kgroups) {
        double y[kGrTM], z[kGrTN];
#pragma unroll
        for (int u = 0; u < kGrTM; ++u) y[u] = (d0 + u < rbr) ? Yc[kk + ldk * (d0 + u)] : 0.0;
#pragma unroll
        for (int v = 0; v < kGrTN; ++v) z[v] = (b0 + v < rar) ? Zc[kk + ldk * (b0 + v)] : 0.0;
#pragma unroll
        for (int u = 0; u < kGrTM; ++u)
#pragma unroll
          for (int v = 0; v < kGrTN; ++v) acc[u][v] = fma(y[u], z[v], acc[u][v]);
      }
    }
  }
  // reduce the k-groups in shared memory (fixed order), write the CTA partial
  __syncthreads();
  double* red = gsm;  // kgroups x ntile x TM*TN
  if (active_b) {
#pragma unroll
    for (int u = 0; u < kGrTM; ++u)
#pragma unroll
      for (int v = 0; v < kGrTN; ++v) red[((int64_t)my_kg * ntile + my_tile) * (kGrTM * kGrTN) + u * kGrTN + v] = acc[u][v];
  }
  __syncthreads();
  for (int e = tid; e < rbr * rar; e += kGrNT) {
    const int d = e % rbr, bq = e / rbr;
    const int tile = (d / kGrTM) + tb_m * (bq / kGrTN);
    const int slot = (d % kGrTM) * kGrTN + (bq % kGrTN);
    double s = 0.0;
    for (int g = 0; g < kgroups; ++g) s += red[((int64_t)g * ntile + tile) * (kGrTM * kGrTN) + slot];
    a.part[(int64_t)blockIdx.x * rbr * rar + e] = s;
  }
}

// ---------------------------------------------------------------------------
// fp64-MMA version with an S-stage bulk-copy pipeline (even ranks).
//
// For every right index the (left, slice) block of a chunk of NS slices is
// contiguous in the F-order core, so a chunk of X and Y arrives as
// rar + rbr bulk copies (TMA engine, mbarrier completion), S - 1 chunks
// ahead.  Each warp owns one 8-wide tile of right indices b of X and a
// share of the chunk's slices; per slice ii it computes
//   Z^T(b, c) = sum_a X(a, ii, b) W(c, a)       (m8n8k4: A = X^T, B = W^T)
// and feeds the D fragments of Z^T straight back as B fragments of
//   acc(d, b) += sum_c Y(c, ii, d) Z(c, ii, b)
// (a D fragment holds k = c = 2 fc + h for n = b = fr, i.e. two k4 steps
// with the k order {0,2,4,6}, {1,3,5,7}; the A fragments of Y are loaded in
// the same order, one 16-byte load for both steps).  Z never leaves the
// registers, and the CTA synchronises once per chunk.  Leading dimensions:
// X 4 mod 16, Y 8 mod 16, W 4 mod 16 (conflict-free fragment loads).
// ---------------------------------------------------------------------------

struct Gram2Args {
  const double* W;  // rbl x ral (col-major)
  const double* X;  // (ral, I, rar)
  const double* Y;  // (rbl, I, rbr)
  int ral, rar, rbl, rbr;
  int64_t I;
  int lns;          // log2(slices per chunk)
  int stages;       // chunk buffers
  int64_t per_cta;  // slices per CTA (multiple of the chunk)
  int ldw, ldx, ldy;
  double* part;     // gridDim.x partials of rbr x rar
};

__host__ __device__ __forceinline__ int g2_ld4(int n) { return ((n + 11) & ~15) + 4; }  // >= n, 4 mod 16
__host__ __device__ __forceinline__ int g2_ld8(int n) { return ((n + 7) & ~15) + 8; }   // >= n, 8 mod 16

__device__ __forceinline__ unsigned g2_smem(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void g2_bulk(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   g2_smem(dst)),
               "l"(src), "r"(bytes), "r"(g2_smem(bar))
               : "memory");
}
__device__ __forceinline__ void g2_expect(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(g2_smem(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void g2_wait(unsigned long long* bar, unsigned parity) {
  unsigned done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(g2_smem(bar)), "r"(parity)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ void dmma884g(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// MAXD: d tiles of 8 this instantiation handles (rbr <= 8 MAXD); NT threads
template <int MAXD, int NT>
__global__ void __launch_bounds__(NT, 1) gram2_kernel(Gram2Args a) {
  constexpr int kG2NT = NT, kG2NW = NT / 32, kG2MaxD = MAXD;
  extern __shared__ __align__(128) double g2[];
  const int ral = a.ral, rar = a.rar, rbl = a.rbl, rbr = a.rbr;
  const int lns = a.lns, NS = 1 << lns, S = a.stages;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int fr = lane >> 2, fc = lane & 3;
  const int64_t xstage = (int64_t)rar * a.ldx, ystage = (int64_t)rbr * a.ldy;
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(g2);  // S <= 16 barriers
  double* Ws = g2 + 16;                            // Ws[c + ldw a]
  double* Xs = Ws + (int64_t)a.ldw * ral;          // S stages: Xs[b * ldx + a + ral * ii]
  Xs += (16 - ((Xs - g2) & 15)) & 15;              // 128-byte aligned stages
  double* Ys = Xs + S * xstage;                    // S stages: Ys[d * ldy + c + rbl * ii]
  if (tid < S) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(g2_smem(&bar[tid])) : "memory");
  if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  for (int e = tid; e < rbl * ral; e += kG2NT) Ws[(e % rbl) + a.ldw * (e / rbl)] = a.W[e];

  const int64_t s_begin = (int64_t)blockIdx.x * a.per_cta;
  const int64_t s_end = min64(a.I, s_begin + a.per_cta);
  const int nch = s_end > s_begin ? (int)((s_end - s_begin + NS - 1) >> lns) : 0;
  __syncthreads();

  auto issue = [&](int c, int st) {  // warp 0: one bulk copy per right index
    if (warp != 0) return;
    const int64_t i0 = s_begin + ((int64_t)c << lns);
    const int nn = (int)min64(NS, s_end - i0);
    const unsigned bx = (unsigned)(ral * nn * 8), by = (unsigned)(rbl * nn * 8);
    if (lane == 0) g2_expect(&bar[st], bx * rar + by * rbr);
    __syncwarp();
    for (int b = lane; b < rar; b += 32)
      g2_bulk(Xs + st * xstage + (int64_t)b * a.ldx, a.X + ral * (i0 + a.I * b), bx, &bar[st]);
    for (int d = lane; d < rbr; d += 32)
      g2_bulk(Ys + st * ystage + (int64_t)d * a.ldy, a.Y + rbl * (i0 + a.I * d), by, &bar[st]);
  };

  // warp -> (b tile, slice share)
  const int nbt = (rar + 7) / 8;
  const int wpb = kG2NW / nbt;              // warps per b tile (>= 1 for rar <= 64)
  const int bt = warp / wpb, wsl = warp % wpb;
  const bool bactive = bt < nbt;
  const int b = bt * 8 + fr;                // this lane's b in A fragments of X^T
  const int nct = (rbl + 7) / 8, ndt = (rbr + 7) / 8;
#ifndef TTB_GRAM_U
#define TTB_GRAM_U 2
#endif
  constexpr int U = TTB_GRAM_U;  // slices in flight per warp (independent accumulator chains)
  double acc[U][kG2MaxD][2];
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int q = 0; q < kG2MaxD; ++q) acc[u][q][0] = acc[u][q][1] = 0.0;

  for (int c = 0; c < S && c < nch; ++c) issue(c, c);
  for (int c = 0, st = 0, ph = 0; c < nch; ++c) {
    const int64_t i0 = s_begin + ((int64_t)c << lns);
    const int nn = (int)min64(NS, s_end - i0);
    g2_wait(&bar[st], ph);
    if (bactive) {
      const double* xs = Xs + st * xstage + (int64_t)b * a.ldx;
      const double* ys = Ys + st * ystage;
      for (int ii0 = wsl; ii0 < nn; ii0 += U * wpb) {
        bool val[U];
#pragma unroll
        for (int u = 0; u < U; ++u) val[u] = ii0 + u * wpb < nn;
#pragma unroll 1
        for (int ct = 0; ct < nct; ++ct) {
          // Z^T(b, c) tiles for c in [8 ct, 8 ct + 8): K = ral
          double z[U][2];
#pragma unroll
          for (int u = 0; u < U; ++u) z[u][0] = z[u][1] = 0.0;
          const int cw = ct * 8 + fr;
          for (int k0 = 0; k0 < ral; k0 += 4) {
            const int k = k0 + fc;
            const double wb = (cw < rbl && k < ral) ? Ws[cw + a.ldw * k] : 0.0;
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const double xa = (val[u] && b < rar && k < ral) ? xs[ral * (ii0 + u * wpb) + k] : 0.0;
              dmma884g(z[u][0], z[u][1], xa, wb);
            }
          }
          // acc(d, b) += Y(c, ii, d) Z(c, ii, b): k = c = 8 ct + 2 fc + h
          const int c2 = ct * 8 + 2 * fc;
#pragma unroll
          for (int dt = 0; dt < kG2MaxD; ++dt) {
            if (dt >= ndt) break;
            const int d = dt * 8 + fr;
#pragma unroll
            for (int u = 0; u < U; ++u) {
              double2 yv = make_double2(0.0, 0.0);
              if (val[u] && d < rbr && c2 < rbl)
                yv = *reinterpret_cast<const double2*>(ys + (int64_t)d * a.ldy + c2 + rbl * (ii0 + u * wpb));
              dmma884g(acc[u][dt][0], acc[u][dt][1], yv.x, z[u][0]);
              dmma884g(acc[u][dt][0], acc[u][dt][1], yv.y, z[u][1]);
            }
          }
        }
      }
    }
    __syncthreads();  // stage st is free
    if (c + S < nch) {
      if (warp == 0) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      issue(c + S, st);
    }
    if (++st == S) {
      st = 0;
      ph ^= 1;
    }
  }
  // reduce the slice shares in a fixed order, write this CTA's partial
  double* red = Xs;  // wpb x rbr x rar
  for (int e = tid; e < wpb * rbr * rar; e += kG2NT) red[e] = 0.0;
  __syncthreads();
  if (bactive) {
#pragma unroll
    for (int dt = 0; dt < kG2MaxD; ++dt) {
      if (dt >= ndt) break;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int d = dt * 8 + fr, bb = bt * 8 + 2 * fc + h;
        double v = 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u) v += acc[u][dt][h];
        if (d < rbr && bb < rar) red[(int64_t)wsl * rbr * rar + d + rbr * bb] = v;
      }
    }
  }
  __syncthreads();
  for (int e = tid; e < rbr * rar; e += kG2NT) {
    double sum = 0.0;
    for (int g = 0; g < wpb; ++g) sum += red[(int64_t)g * rbr * rar + e];
    a.part[(int64_t)blockIdx.x * rbr * rar + e] = sum;
  }
}

// ---------------------------------------------------------------------------
// innerprod_sym (ops.py:158-205): the Gram carry is factored W = (P L)(P L)^T
// by a rank-revealing pivoted Cholesky (dpstrf's greedy largest-remaining-
// diagonal pivoting, stop when the pivot is not above 1e-14 * max diag W) and
// the recurrence carries Z = (P L)^T H(x_n), W' = Z^T Z.  The (n <= 64)
// carry is read from its lower triangle, as dpstrf(lower=1) does, one
// element per thread (registers), with no row swaps: column j of P L is
// written in the carry's own row order, and (P L)(P L)^T accumulates
// alongside for the reconstruction check -- a residual above 1e-6 ||W||_F
// (ops.py:173-175) sets the context flag and the caller falls back to the
// plain inner product.
// ---------------------------------------------------------------------------
constexpr double kPstrfRtol = 1e-14;
constexpr double kGramResidRtol = 1e-6;

struct PcholSmem {
  double diag[64], colp[64], red[2][16];
  int chosen[64], order[64];
  int p, rank;
  double piv, tol;
};

// W: n x n (col-major, generic pointer, lower triangle read).  Outputs (any
// may be null): PL (n x n), Wrec = (P L)(P L)^T, perm (pivots then the rest),
// rank; *flag = 1 on an indefinite carry.
template <int NT, int NMAX>
__device__ void pchol_dev(const double* W, int n, double* PL, double* Wrec, int* perm, int* rank_out, int* flag,
                          PcholSmem& S) {
  constexpr int Q = (NMAX * NMAX + NT - 1) / NT;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nn = n * n;
  double a[Q], rec[Q], w0[Q];
  int ii[Q], kk[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int e = tid + NT * q;
    ii[q] = e < nn ? e % n : -1;
    kk[q] = e < nn ? e / n : -1;
    a[q] = e < nn ? W[max(ii[q], kk[q]) + n * min(ii[q], kk[q])] : 0.0;
    w0[q] = a[q];
    rec[q] = 0.0;
    if (e < nn && ii[q] == kk[q]) S.diag[ii[q]] = a[q];
  }
  for (int i = tid; i < 64; i += NT) S.chosen[i] = 0;
  __syncthreads();
  if (warp == 0) {
    double m = -INFINITY;
    for (int i = lane; i < n; i += 32) m = fmax(m, S.diag[i]);
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) {
      S.tol = kPstrfRtol * fmax(m, 0.0);
      S.rank = n;
    }
  }
  for (int j = 0; j < n; ++j) {
    if (j > 0) {
#pragma unroll
      for (int q = 0; q < Q; ++q)
        if (ii[q] >= 0 && ii[q] == kk[q]) S.diag[ii[q]] = S.chosen[ii[q]] ? -INFINITY : a[q];
    }
    __syncthreads();
    if (warp == 0) {  // the largest remaining diagonal, lowest index on ties
      double v = -INFINITY;
      int p = n;
      for (int i = lane; i < n; i += 32) {
        const double d = S.diag[i];
        if (d > v) {
          v = d;
          p = i;
        }
      }
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int op = __shfl_xor_sync(0xffffffffu, p, o);
        if (ov > v || (ov == v && op < p)) {
          v = ov;
          p = op;
        }
      }
      if (lane == 0) {
        S.p = p;
        S.piv = v;
      }
    }
    __syncthreads();
    const double piv = S.piv;
    if (!(piv > S.tol)) {  // numeric rank reached (NaN pivots stop too)
      if (tid == 0) S.rank = j;
      break;
    }
    const int p = S.p;
    const double d = sqrt(piv), rd = 1.0 / d;  // dpstrf scales by the reciprocal
#pragma unroll
    for (int q = 0; q < Q; ++q)
      if (kk[q] == p) {
        const int i = ii[q];
        const double v = i == p ? d : (S.chosen[i] ? 0.0 : a[q] * rd);
        S.colp[i] = v;
        if (PL) PL[i + n * j] = v;
      }
    if (tid == 0) {
      S.chosen[p] = 1;
      S.order[j] = p;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < Q; ++q)
      if (ii[q] >= 0) {
        const double ci = S.colp[ii[q]], ck = S.colp[kk[q]];
        rec[q] = fma(ci, ck, rec[q]);
        if (!S.chosen[ii[q]] && !S.chosen[kk[q]]) a[q] = fma(-ci, ck, a[q]);
      }
  }
  __syncthreads();
  const int rank = S.rank;
  double r2 = 0.0, w2 = 0.0;
#pragma unroll
  for (int q = 0; q < Q; ++q)
    if (ii[q] >= 0) {
      r2 += (rec[q] - w0[q]) * (rec[q] - w0[q]);
      w2 += w0[q] * w0[q];
      if (Wrec) Wrec[ii[q] + n * kk[q]] = rec[q];
      if (PL && kk[q] >= rank) PL[ii[q] + n * kk[q]] = 0.0;
    }
  for (int o = 16; o; o >>= 1) {
    r2 += __shfl_xor_sync(0xffffffffu, r2, o);
    w2 += __shfl_xor_sync(0xffffffffu, w2, o);
  }
  if (lane == 0) {
    S.red[0][warp] = r2;
    S.red[1][warp] = w2;
  }
  __syncthreads();
  if (tid == 0) {
    double R2 = 0.0, W2 = 0.0;
    for (int w = 0; w < NT / 32; ++w) {
      R2 += S.red[0][w];
      W2 += S.red[1][w];
    }
    if (!(sqrt(R2) <= kGramResidRtol * fmax(sqrt(W2), 1e-300))) *flag = 1;
    if (rank_out) *rank_out = rank;
    if (perm) {
      int q = rank;
      for (int i = 0; i < rank; ++i) perm[i] = S.order[i];
      for (int i = 0; i < n; ++i)
        if (!S.chosen[i]) perm[q++] = i;
    }
  }
}

template <int NMAX>
__global__ void __launch_bounds__(256) pchol_kernel(const double* __restrict__ W, int n, double* __restrict__ PL,
                                                    double* __restrict__ Wrec, int* __restrict__ perm,
                                                    int* __restrict__ rank_out, int* __restrict__ flag) {
  __shared__ PcholSmem S;
  pchol_dev<256, NMAX>(W, n, PL, Wrec, perm, rank_out, flag, S);
}

// ---------------------------------------------------------------------------
// Rank-16 specialisation (every rank 16: the interior cores of BASELINE
// cfg2) on the m16n8k8 fp64 MMA: a whole 16 x 16 Z^T and accumulator per
// warp, W^T fragments held in registers for the whole launch, 8 MMAs and 12
// shared loads per slice (the generic kernel issues 32 m8n8k4 and ~50
// loads).  Z^T(b, c) = sum_a X(a, ii, b) W(c, a) as (M = b, N = c, K = a);
// acc(d, b) += sum_c Y(c, ii, d) Z(c, ii, b) as (M = d, N = b, K = c) with
// the contraction index permuted inside each 8-block (k = t <-> c = 2t,
// k = t + 4 <-> c = 2t + 1) so the D fragments of Z^T are directly the B
// fragments of the second product.  Slices stream through a 3-stage
// bulk-copy pipeline (one copy per right index, 16-slice chunks).
// ---------------------------------------------------------------------------
#ifndef TTB_G16_NS
#define TTB_G16_NS 16
#endif
#ifndef TTB_G16_STAGES
#define TTB_G16_STAGES 3
#endif
#ifndef TTB_G16_NT
#define TTB_G16_NT 512
#endif
constexpr int kG16NS = TTB_G16_NS;           // slices per chunk
constexpr int kG16Stages = TTB_G16_STAGES;
constexpr int kG16NT = TTB_G16_NT;           // warps take the chunk's slices round-robin
#ifndef TTB_G16S_NT
#define TTB_G16S_NT 512
#endif
#ifndef TTB_G16S_NS
#define TTB_G16S_NS 32
#endif
#ifndef TTB_G16S_CPS
#define TTB_G16S_CPS 1
#endif
constexpr int kG16sNT = TTB_G16S_NT;   // SYM: threads, slices per chunk, CTAs per SM
constexpr int kG16sNS = TTB_G16S_NS;
constexpr int kG16sCPS = TTB_G16S_CPS;
constexpr int kG16Ldx = 16 * kG16NS + 4;     // 4 mod 16: conflict-free scalar A loads
constexpr int kG16Ldy = 16 * kG16NS + 8;     // 8 mod 16: conflict-free 16-byte A loads
constexpr int kG16Stage = 16 * kG16Ldx + 16 * kG16Ldy;

__device__ __forceinline__ void dmma1688(double (&d)[4], double a0, double a1, double a2, double a3, double b0,
                                         double b1) {
  asm(  // not volatile: the compiler may interleave independent products
      "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
}

// SYM (the innerprod_sym route, ops.py:179-205): W holds P L, the carry's
// pivoted Cholesky factor in the carry's row order (16 x 16, zero columns
// past the numeric rank) and Y is unused; Z^T = H(X)^T M^T as
// above, then acc = Z^T Z with the same D fragments serving as the A operand
// (M = d, K = c: a = {z0, z2, z1, z3}) -- one operand stream instead of two.
// The contraction index a runs in pivot order (perm), where P L is lower
// triangular: the zero (a < 8, c >= 8) block of Z^T's first product is
// skipped, and of the symmetric Z^T Z only the (d, b < 8) m16n8 tile and the
// (d, b >= 8) m8n8 block are formed (the rest is their mirror): 6 instead of
// 8 m16n8k8-equivalents per slice.
__device__ __forceinline__ void dmma884(double (&d)[4], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

template <bool SYM>
__global__ void __launch_bounds__(SYM ? kG16sNT : kG16NT, SYM ? kG16sCPS : 1) gram16_kernel(const double* __restrict__ W, const double* __restrict__ X,
                                                           const double* __restrict__ Y, const int* __restrict__ perm,
                                                           int64_t I, int64_t per_cta, double* __restrict__ part,
                                                           int* __restrict__ ticket, double* __restrict__ Wrec,
                                                           int* __restrict__ flag) {
  // SYM streams one operand: twice the slices per chunk in the same stage
  // bytes, so every warp has a pair of slices per chunk (overlapped chains)
  constexpr int NS = SYM ? kG16sNS : kG16NS;
  constexpr int LDX = 16 * NS + 4;
  constexpr int STAGE = SYM ? 16 * LDX : kG16Stage;
  extern __shared__ __align__(128) double g16[];
  constexpr int NTK = SYM ? kG16sNT : kG16NT;
  constexpr int NW = NTK / 32;
  static_assert(NW * 256 <= kG16Stages * STAGE, "reduction scratch fits the stages");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(g16);
  double* St = g16 + 16;  // stages: X block (16 x LDX), then Y block (16 x kG16Ldy)
  if (tid < kG16Stages) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(g2_smem(&bar[tid])) : "memory");
  if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  // W^T B fragments: (k = a, n = c) -> W(c, a) = W[c + 16 a]
  double wf[2][2][2];
  int pa[2][2] = {{0, 4}, {8, 12}};
  if constexpr (SYM) {
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      pa[ks][0] = perm[8 * ks + t];
      pa[ks][1] = perm[8 * ks + t + 4];
    }
  }
#pragma unroll
  for (int ks = 0; ks < 2; ++ks)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      if constexpr (SYM) {  // W = P L (carry rows, col-major); a in pivot order
        wf[ks][nt][0] = W[pa[ks][0] + 16 * (8 * nt + g)];
        wf[ks][nt][1] = W[pa[ks][1] + 16 * (8 * nt + g)];
      } else {
        wf[ks][nt][0] = W[(8 * nt + g) + 16 * (8 * ks + t)];
        wf[ks][nt][1] = W[(8 * nt + g) + 16 * (8 * ks + t + 4)];
      }
    }
  const int64_t s_begin = (int64_t)blockIdx.x * per_cta;
  const int64_t s_end = min64(I, s_begin + per_cta);
  const int nch = s_end > s_begin ? (int)((s_end - s_begin + NS - 1) / NS) : 0;
  __syncthreads();
  auto issue = [&](int c, int st) {  // warp 0: one bulk copy per right index of X and of Y
    if (warp != 0) return;
    const int64_t i0 = s_begin + (int64_t)c * NS;
    const int nn = (int)min64(NS, s_end - i0);
    const unsigned bytes = (unsigned)(16 * nn * 8);
    if (lane == 0) g2_expect(&bar[st], (SYM ? 16 : 32) * bytes);
    __syncwarp();
    double* xs = St + (int64_t)st * STAGE;
    double* ys = xs + 16 * LDX;
    if (SYM && lane >= 16) return;
    if (lane < 16) g2_bulk(xs + (int64_t)lane * LDX, X + 16 * (i0 + I * lane), bytes, &bar[st]);
    else g2_bulk(ys + (int64_t)(lane - 16) * kG16Ldy, Y + 16 * (i0 + I * (lane - 16)), bytes, &bar[st]);
  };
  for (int c = 0; c < kG16Stages && c < nch; ++c) issue(c, c);
  double acc[2][2][4];
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int bt = 0; bt < 2; ++bt)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[u][bt][q] = 0.0;
  for (int c = 0, st = 0, ph = 0; c < nch; ++c) {
    const int64_t i0 = s_begin + (int64_t)c * NS;
    const int nn = (int)min64(NS, s_end - i0);
    g2_wait(&bar[st], ph);
    const double* xs = St + (int64_t)st * STAGE;
    const double* ys = xs + 16 * LDX;
    // slices in pairs: both Z^T first, then both accumulations (two
    // accumulator sets: independent MMA chains the scheduler can overlap)
    auto zt = [&](int ii, double (&z)[2][4]) {  // Z^T (16 x 16): M = b, N = c, K = a
      const double* xp = xs + 16 * ii;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int q = 0; q < 4; ++q) z[nt][q] = 0.0;
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const int a = SYM ? pa[ks][0] : 8 * ks + t, a4 = SYM ? pa[ks][1] : 8 * ks + t + 4;
        const double a0 = xp[(int64_t)g * LDX + a], a1 = xp[(int64_t)(g + 8) * LDX + a];
        const double a2 = xp[(int64_t)g * LDX + a4], a3 = xp[(int64_t)(g + 8) * LDX + a4];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
          if (!SYM || nt <= ks) dmma1688(z[nt], a0, a1, a2, a3, wf[ks][nt][0], wf[ks][nt][1]);
      }
    };
    auto accum = [&](int ii, const double (&z)[2][4], double (&ac)[2][4]) {  // acc(d, b) += Y(c, d) Z(c, b)
      if constexpr (SYM) {
#pragma unroll
        for (int kc = 0; kc < 2; ++kc) {
          dmma1688(ac[0], z[kc][0], z[kc][2], z[kc][1], z[kc][3], z[kc][0], z[kc][1]);
          dmma884(ac[1], z[kc][2], z[kc][2]);  // (d, b >= 8) block, k = c = 8 kc + 2 t
          dmma884(ac[1], z[kc][3], z[kc][3]);  //                     k = c = 8 kc + 2 t + 1
        }
        return;
      }
      const double* yp = ys + 16 * ii;
#pragma unroll
      for (int kc = 0; kc < 2; ++kc) {
        const double2 y0 = *reinterpret_cast<const double2*>(yp + (int64_t)g * kG16Ldy + 8 * kc + 2 * t);
        const double2 y1 = *reinterpret_cast<const double2*>(yp + (int64_t)(g + 8) * kG16Ldy + 8 * kc + 2 * t);
        dmma1688(ac[0], y0.x, y1.x, y0.y, y1.y, z[kc][0], z[kc][1]);
        dmma1688(ac[1], y0.x, y1.x, y0.y, y1.y, z[kc][2], z[kc][3]);
      }
    };
    for (int ii = warp; ii < nn; ii += 2 * NW) {
      double z0[2][4], z1[2][4];
      const bool two = ii + NW < nn;
      zt(ii, z0);
      if (two) zt(ii + NW, z1);
      accum(ii, z0, acc[0]);
      if (two) accum(ii + NW, z1, acc[1]);
    }
    __syncthreads();  // stage st is free
    if (c + kG16Stages < nch) {
      if (warp == 0) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      issue(c + kG16Stages, st);
    }
    if (++st == kG16Stages) {
      st = 0;
      ph ^= 1;
    }
  }
  // per-warp 16 x 16 partials, summed over warps in a fixed order
  double* red = St;  // NW x 256
  if constexpr (SYM) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int d = g + 8 * (q >> 1), b = 2 * t + (q & 1);
      const double v = acc[0][0][q] + acc[1][0][q];
      red[warp * 256 + d + 16 * b] = v;
      if (q >= 2) red[warp * 256 + b + 16 * d] = v;  // mirror
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) red[warp * 256 + (8 + g) + 16 * (8 + 2 * t + h)] = acc[0][1][h] + acc[1][1][h];
  } else
#pragma unroll
  for (int bt = 0; bt < 2; ++bt)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int d = g + 8 * (q >> 1), b = 8 * bt + 2 * t + (q & 1);
      red[warp * 256 + d + 16 * b] = acc[0][bt][q] + acc[1][bt][q];
    }
  __syncthreads();
  for (int e = tid; e < 256; e += NTK) {
    double sum = 0.0;
    for (int w = 0; w < NW; ++w) sum += red[w * 256 + e];
    part[(int64_t)blockIdx.x * 256 + e] = sum;
  }
  {
    // with a ticket, the last CTA to finish sums the partials (fixed order)
    // and writes W' to Wrec -- or, SYM, factors it in place: P L and perm
    // for the next mode (every CTA read them before its main loop) -- so no
    // second launch sits between two modes
    if (ticket == nullptr) return;
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(ticket, 1) == (int)gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    constexpr int NH = NTK / 256;  // threads per carry entry
    static_assert(NTK % 256 == 0, "one or more threads per carry entry");
    double* Wsm = St;  // (1 + NH) x 256 (the reduction scratch is free again)
    {
      const int e = tid & 255, h = tid >> 8;
      double s0 = 0.0;
#pragma unroll 16
      for (int p = h; p < (int)gridDim.x; p += NH) s0 += __ldcg(part + (int64_t)p * 256 + e);
      Wsm[256 + tid] = s0;
    }
    __syncthreads();
    if (tid < 256) {
      double w = 0.0;
      for (int h = 0; h < NH; ++h) w += Wsm[256 * (h + 1) + tid];
      Wsm[tid] = w;
    }
    __syncthreads();
    if constexpr (SYM) {
      __shared__ PcholSmem S;
      pchol_dev<NTK, 16>(Wsm, 16, const_cast<double*>(W), Wrec, const_cast<int*>(perm), nullptr, flag, S);
    } else {
      if (tid < 256) Wrec[tid] = Wsm[tid];
    }
    if (tid == 0) *ticket = 0;
  }
}

__global__ void gram_final_kernel(const double* __restrict__ part, int nparts, int cnt, double* __restrict__ out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < cnt; e += blockDim.x * gridDim.x) {
    double s = 0.0;
#pragma unroll 16
    for (int p = 0; p < nparts; ++p) s += part[(int64_t)p * cnt + e];
    out[e] = s;
  }
}

void gram_step(Ctx& ctx, const double* W, const double* X, int64_t ral, int64_t rar, const double* Y, int64_t rbl,
               int64_t rbr, int64_t I, double* Wn, int* ticket) {
  if (ral > 64 || rar > 64 || rbl > 64 || rbr > 64) {  // the general path (wide.cu)
    gram_step_wide(ctx, W, X, ral, rar, Y, rbl, rbr, I, Wn);
    return;
  }
  const int64_t cnt = rbr * rar;
  if (I == 0) {
    fill_zero(ctx, Wn, cnt);
    return;
  }
  const bool even = (ral % 2 == 0) && (rbl % 2 == 0) && ((uintptr_t)X % 16 == 0) && ((uintptr_t)Y % 16 == 0);
  static const bool no16 = getenv("TTB_GRAM_NO16") != nullptr;
  if (even && !no16 && ral == 16 && rar == 16 && rbl == 16 && rbr == 16 && getenv("TTB_GRAM_V1") == nullptr) {
    const size_t smem = (16 + (size_t)kG16Stages * kG16Stage) * sizeof(double);
    int grid = (int)std::min<int64_t>((int64_t)ctx.num_sms, (I + kG16NS - 1) / kG16NS);
    int64_t per_cta = (I + grid - 1) / grid;
    per_cta = (per_cta + kG16NS - 1) / kG16NS * kG16NS;
    grid = (int)((I + per_cta - 1) / per_cta);
    double* part = (double*)ctx.alloc((size_t)grid * cnt * sizeof(double));
    smem_attr((const void*)gram16_kernel<false>, smem);
    ProfScope ps("gram", ctx.stream);
    gram16_kernel<false><<<grid, kG16NT, smem, ctx.stream>>>(W, X, Y, nullptr, I, per_cta, part, ticket, Wn,
                                                             nullptr);
    TTB_LAUNCHED();
    if (!ticket) {
      gram_final_kernel<<<1, 256, 0, ctx.stream>>>(part, grid, (int)cnt, Wn);
      TTB_LAUNCHED();
    }
    ctx.free(part);
    return;
  }
  if (even && getenv("TTB_GRAM_V1") == nullptr) {
    Gram2Args g;
    g.W = W;
    g.X = X;
    g.Y = Y;
    g.ral = (int)ral;
    g.rar = (int)rar;
    g.rbl = (int)rbl;
    g.rbr = (int)rbr;
    g.I = I;
    g.ldw = g2_ld4((int)rbl);
    // slices per chunk (a power of two) and stage count: maximise the bytes in
    // flight ((stages - 1) chunks) within ~220 KB, preferring larger chunks
    auto stage_bytes = [&](int n) {
      return ((size_t)rar * g2_ld4((int)ral * n) + (size_t)rbr * g2_ld8((int)rbl * n)) * 8;
    };
    auto fixed_bytes = [&](int n) { return ((size_t)48 + (size_t)g.ldw * ral) * 8; };
    const size_t cap = 220 * 1024;
    int lns = 0, stages = 2;
    for (int need = 3; need >= 2; --need) {  // the largest chunk with >= need stages
      bool found = false;
      for (int l = 7; l >= 0; --l) {
        if (l > 0 && (1 << l) > 2 * I) continue;
        const size_t fb = fixed_bytes(1 << l), sb = stage_bytes(1 << l);
        if (fb + need * sb > cap) continue;
        lns = l;
        stages = (int)std::min<size_t>(8, (cap - fb) / sb);
        found = true;
        break;
      }
      if (found) break;
    }
    if (const char* e = getenv("TTB_GRAM_LNS")) {  // tuning override
      lns = atoi(e);
      stages = (int)std::max<size_t>(2, std::min<size_t>(8, (cap - fixed_bytes(1 << lns)) / stage_bytes(1 << lns)));
    }
    const int ns = 1 << lns;
    const int wpb_h = (rbr <= 16 ? 16 : 8) / (int)((rar + 7) / 8);
    auto bytes = [&](int n) {
      return std::max(fixed_bytes(n) + (size_t)stages * stage_bytes(n),
                      fixed_bytes(n) + (size_t)wpb_h * rbr * rar * 8 + 256);
    };
    g.lns = lns;
    g.stages = stages;
    g.ldx = g2_ld4((int)ral * ns);
    g.ldy = g2_ld8((int)rbl * ns);
    const size_t smem = bytes(ns);
    int grid = (int)std::min<int64_t>((int64_t)ctx.num_sms, (I + ns - 1) / ns);
    int64_t per_cta = (I + grid - 1) / grid;
    per_cta = (per_cta + ns - 1) / ns * ns;
    grid = (int)((I + per_cta - 1) / per_cta);
    g.per_cta = per_cta;
    double* part = (double*)ctx.alloc((size_t)grid * cnt * sizeof(double));
    g.part = part;
    ProfScope ps("gram", ctx.stream);
    auto launch = [&](auto kern, int nt) {
      smem_attr((const void*)kern, smem);
      kern<<<grid, nt, smem, ctx.stream>>>(g);
    };
    if (rbr <= 16) launch(gram2_kernel<2, 512>, 512);
    else if (rbr <= 32) launch(gram2_kernel<4, 256>, 256);
    else launch(gram2_kernel<8, 256>, 256);
    TTB_LAUNCHED();
    gram_final_kernel<<<(int)std::max<int64_t>(1, (cnt + 255) / 256), 256, 0, ctx.stream>>>(part, grid, (int)cnt, Wn);
    TTB_LAUNCHED();
    ctx.free(part);
    return;
  }
  const int64_t per_slice = ral * rar + rbl * rbr + rbl * rar;
  const int64_t budget = kGrSmemDoubles - rbl * ral;
  int ns = (int)std::max<int64_t>(1, std::min<int64_t>(budget / per_slice, 64));
  ns = (int)std::min<int64_t>(ns, I);
  // reduction scratch must fit too
  const int ntile = (int)(((rbr + kGrTM - 1) / kGrTM) * ((rar + kGrTN - 1) / kGrTN));
  const int kgroups = std::max(1, kGrNT / ntile);
  const int64_t need = std::max<int64_t>(rbl * ral + per_slice * ns, (int64_t)kgroups * ntile * kGrTM * kGrTN);
  const size_t smem = (size_t)need * sizeof(double);
  TTB_CHECK(smem <= 200 * 1024, TTB_ERR_CAPABILITY, "inner product: ranks too large for the chunk buffer");
  int grid = (int)std::min<int64_t>((int64_t)ctx.num_sms * 2, (I + ns - 1) / ns);
  int64_t per_cta = (I + grid - 1) / grid;
  per_cta = (per_cta + ns - 1) / ns * ns;
  grid = (int)((I + per_cta - 1) / per_cta);
  double* part = (double*)ctx.alloc((size_t)grid * cnt * sizeof(double));
  GramArgs a{W, X, Y, (int)ral, (int)rar, (int)rbl, (int)rbr, I, ns, per_cta, part};
  smem_attr((const void*)gram_kernel, smem);
  ProfScope ps("gram", ctx.stream);
  gram_kernel<<<grid, kGrNT, smem, ctx.stream>>>(a);
  TTB_LAUNCHED();
  gram_final_kernel<<<(int)std::max<int64_t>(1, (cnt + 255) / 256), 256, 0, ctx.stream>>>(part, grid, (int)cnt, Wn);
  TTB_LAUNCHED();
  ctx.free(part);
}


void pivoted_cholesky(Ctx& ctx, const double* W, int n, double* PL, double* Wrec, int* perm, int* rank) {
  TTB_CHECK(n >= 1 && n <= 64, TTB_ERR_CAPABILITY, "pivoted Cholesky: carry above 64 x 64");
  ProfScope ps("pchol", ctx.stream);
  auto kern = n <= 16 ? pchol_kernel<16> : n <= 32 ? pchol_kernel<32> : pchol_kernel<64>;
  kern<<<1, 256, 0, ctx.stream>>>(W, n, PL, Wrec, perm, rank, ctx.flag());
  TTB_LAUNCHED();
}

// W' = Z^T Z, Z = (P L)^T H(X); X is (ral, I, rar).  Bond ranks 16 run the
// fused single-stream kernel; other shapes contract the reconstructed carry
// (P L)(P L)^T with the two-operand Gram kernels (same value, the flops of
// innerprod).  With a ticket (16 x 16 only; see sym16_fusable) the step
// also factors W' in place -- PL, perm, Wrec, the flag -- and Wn is not
// written.
bool sym16_fusable(int64_t ral, int64_t rar, int64_t I, const double* X) {
  static const bool no16 = getenv("TTB_GRAM_NO16") != nullptr;
  return I > 0 && ral == 16 && rar == 16 && (uintptr_t)X % 16 == 0 && !no16;
}

void gram_sym_step(Ctx& ctx, double* PL, int* perm, double* Wrec, const double* X, int64_t ral, int64_t rar,
                   int64_t I, double* Wn, int* ticket) {
  if (sym16_fusable(ral, rar, I, X)) {
    const size_t smem = (16 + (size_t)kG16Stages * 16 * (16 * kG16sNS + 4)) * sizeof(double);
    constexpr int ns = kG16sNS;
    int grid = (int)std::min<int64_t>((int64_t)ctx.num_sms * kG16sCPS, (I + ns - 1) / ns);
    int64_t per_cta = (I + grid - 1) / grid;
    per_cta = (per_cta + ns - 1) / ns * ns;
    grid = (int)((I + per_cta - 1) / per_cta);
    double* part = (double*)ctx.alloc((size_t)grid * 256 * sizeof(double));
    smem_attr((const void*)gram16_kernel<true>, smem);
    ProfScope ps("gram", ctx.stream);
    gram16_kernel<true><<<grid, kG16sNT, smem, ctx.stream>>>(PL, X, nullptr, perm, I, per_cta, part, ticket, Wrec,
                                                            ctx.flag());
    TTB_LAUNCHED();
    if (!ticket) {
      gram_final_kernel<<<1, 256, 0, ctx.stream>>>(part, grid, 256, Wn);
      TTB_LAUNCHED();
    }
    ctx.free(part);
    return;
  }
  TTB_CHECK(!ticket, TTB_ERR_CONTRACT, "fused carry factorization needs 16 x 16 bonds");
  gram_step(ctx, Wrec, X, ral, rar, X, ral, rar, I, Wn);
}

}  // namespace ttb
