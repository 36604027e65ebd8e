// Bond ranks above 64 (and slices too tall for a leaf tile): the general path.
//
// The reference has no rank limit (tsqr.py:103-130 takes any b, the SVD of
// parallel.py:224-258 any size, the Gram sweep of ops.py:135-155 any ranks);
// the register-tile kernels of tsqr.cu / svd.cu / gram.cu / gemm.cu are sized
// for b <= 64.  Everything wider runs here, built from four pieces:
//
//  * dgemm_strided: a shared-memory tiled fp64 GEMM on arbitrarily strided
//    operands (64 x 64 tiles, 4 x 4 outputs per thread), with a split of the
//    contraction range over grid.y for the tall reductions Q^T C.
//  * wide TSQR: the panel is copied to a dense column-major work matrix and
//    factored in column blocks of <= 64 by the register-tile TSQR.  Block p's
//    orthonormal factor Q_p is formed explicitly (the implicit-Q apply on the
//    identity) in place of its columns; the trailing columns get
//    R_pq = Q_p^T C, C -= Q_p R_pq.  This is block Householder QR of the
//    augmented matrix [0; A] with reflectors H_p = I - Y_p Y_p^T,
//    Y_p = [I; -Q_p] (H_p is orthogonal because Q_p^T Q_p = I to roundoff, the
//    property the Householder TSQR guarantees for any panel), so A = Q R holds
//    to roundoff for any A, rank-deficient included.
//  * wide apply: Q [z; 0] is evaluated as the reflector product
//    H_1 ... H_P [z; 0], i.e. M = Q_P z_P, then for p = P-1 .. 1
//    M += Q_p (z_p - Q_p^T M): each block is re-projected at apply time, so the
//    loss of orthogonality between blocks enters squared.
//  * wide Jacobi SVD: one CTA, the matrix and V in global memory (L1/L2
//    resident), one warp per column pair, the tail rule of svd.cu.
//
// This path is about capability, not speed-of-light: its passes are plain
// HBM-bound GEMMs and a latency-bound one-CTA SVD.
#include <algorithm>
#include <vector>

#include "ops.cuh"
#include "prof.cuh"
#include "svd.cuh"
#include "wide.cuh"

namespace ttb {

// ------------------------------------------------------------------------
// strided GEMM
// ------------------------------------------------------------------------
constexpr int kGT = 64, kGK = 16, kGNT = 256;

struct GemmArgs {
  int64_t M, N, K;
  const double* A;
  int64_t sam, sak;
  const double* B;
  int64_t sbk, sbn;
  double* C;
  int64_t scm, scn;
  double alpha, beta;
  int64_t kchunk;  // contraction range per grid.y slice
  int64_t csplit;  // C advances by this per grid.y slice
  int64_t tiles_m;
};

__global__ void __launch_bounds__(kGNT) dgemm_kernel(GemmArgs a) {
  __shared__ __align__(16) double As[kGK][kGT + 4];
  __shared__ __align__(16) double Bs[kGK][kGT + 4];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t tile = blockIdx.x;
  const int64_t m0 = (tile % a.tiles_m) * kGT, n0 = (tile / a.tiles_m) * kGT;
  const int64_t kb = (int64_t)blockIdx.y * a.kchunk, ke = min64(a.K, kb + a.kchunk);
  const bool a_mfast = a.sam <= a.sak, b_nfast = a.sbn <= a.sbk;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int64_t k0 = kb; k0 < ke; k0 += kGK) {
#pragma unroll
    for (int l = 0; l < (kGT * kGK) / kGNT; ++l) {
      const int idx = tid + kGNT * l;
      {
        const int m = a_mfast ? (idx & (kGT - 1)) : (idx >> 4), k = a_mfast ? (idx >> 6) : (idx & (kGK - 1));
        const int64_t gm = m0 + m, gk = k0 + k;
        As[k][m] = (gm < a.M && gk < ke) ? __ldg(a.A + gm * a.sam + gk * a.sak) : 0.0;
      }
      {
        const int n = b_nfast ? (idx & (kGT - 1)) : (idx >> 4), k = b_nfast ? (idx >> 6) : (idx & (kGK - 1));
        const int64_t gn = n0 + n, gk = k0 + k;
        Bs[k][n] = (gn < a.N && gk < ke) ? __ldg(a.B + gk * a.sbk + gn * a.sbn) : 0.0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kGK; ++kk) {
      const double2 a01 = *reinterpret_cast<const double2*>(&As[kk][tx * 4]);
      const double2 a23 = *reinterpret_cast<const double2*>(&As[kk][tx * 4 + 2]);
      const double2 b01 = *reinterpret_cast<const double2*>(&Bs[kk][ty * 4]);
      const double2 b23 = *reinterpret_cast<const double2*>(&Bs[kk][ty * 4 + 2]);
      const double av[4] = {a01.x, a01.y, a23.x, a23.y}, bv[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  double* Cb = a.C + (int64_t)blockIdx.y * a.csplit;
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t gm = m0 + tx * 4 + i, gn = n0 + ty * 4 + j;
      if (gm < a.M && gn < a.N) {
        double* p = Cb + gm * a.scm + gn * a.scn;
        double v = a.alpha * acc[i][j];
        if (a.beta != 0.0) v = fma(a.beta, *p, v);
        *p = v;
      }
    }
}

__global__ void scale_strided_kernel(int64_t M, int64_t N, double* C, int64_t scm, int64_t scn, double beta) {
  for (int64_t idx = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; idx < M * N; idx += (int64_t)blockDim.x * gridDim.x) {
    const int64_t m = idx % M, n = idx / M;
    double* p = C + m * scm + n * scn;
    *p = beta == 0.0 ? 0.0 : beta * *p;
  }
}

void dgemm_strided(Ctx& ctx, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t sam, int64_t sak,
                   const double* B, int64_t sbk, int64_t sbn, double beta, double* C, int64_t scm, int64_t scn) {
  if (M <= 0 || N <= 0) return;
  if (K <= 0) {
    if (beta != 1.0) {
      const int grid = (int)std::min<int64_t>(4096, (M * N + 255) / 256);
      scale_strided_kernel<<<grid, 256, 0, ctx.stream>>>(M, N, C, scm, scn, beta);
      TTB_LAUNCHED();
    }
    return;
  }
  GemmArgs a{M, N, K, A, sam, sak, B, sbk, sbn, C, scm, scn, alpha, beta, K, 0, (M + kGT - 1) / kGT};
  const int64_t tiles = a.tiles_m * ((N + kGT - 1) / kGT);
  TTB_CHECK(tiles < (1LL << 31), TTB_ERR_CAPABILITY, "dgemm: too many output tiles");
  ProfScope ps("wide_gemm", ctx.stream);
  dgemm_kernel<<<dim3((unsigned)tiles, 1), kGNT, 0, ctx.stream>>>(a);
  TTB_LAUNCHED();
}

// out[e] = base[e] * sbase + sign * sum_s part[s * cnt + e]   (fixed order)
__global__ void split_sum_kernel(const double* __restrict__ part, int nsplit, int64_t cnt, double* __restrict__ out) {
  for (int64_t e = threadIdx.x + (int64_t)blockIdx.x * blockDim.x; e < cnt; e += (int64_t)blockDim.x * gridDim.x) {
    double s = 0.0;
    for (int q = 0; q < nsplit; ++q) s += part[(int64_t)q * cnt + e];
    out[e] = s;
  }
}

// W (na x nb, col-major ld na) = sum over `rows` rows r of A(r, :)^T B(r, :),
// A(r, i) = A[r * sar + i * sac], B(r, j) = B[r * sbr + j * sbc]; the row
// range is split over CTAs and the partial products are summed in a fixed
// order (deterministic); allreduce: summed over ranks as well.
void tall_gram(Ctx& ctx, int64_t rows, int na, int nb, const double* A, int64_t sar, int64_t sac, const double* B,
               int64_t sbr, int64_t sbc, double* W, bool allreduce) {
  const int64_t cnt = (int64_t)na * nb;
  if (cnt == 0) return;
  double* dst = W;
  double* tmp = nullptr;
  if (allreduce && ctx.nranks > 1) {
    tmp = (double*)ctx.alloc((size_t)cnt * sizeof(double));
    dst = tmp;
  }
  if (rows <= 0) {
    fill_zero(ctx, dst, cnt);
  } else {
    const int64_t tiles = (int64_t)((na + kGT - 1) / kGT) * ((nb + kGT - 1) / kGT);
    int64_t nsplit = std::max<int64_t>(1, (4LL * ctx.num_sms) / tiles);
    nsplit = std::min<int64_t>(nsplit, (rows + 255) / 256);
    nsplit = std::min<int64_t>(nsplit, 65535);
    int64_t kchunk = (rows + nsplit - 1) / nsplit;
    kchunk = (kchunk + kGK - 1) / kGK * kGK;
    nsplit = (rows + kchunk - 1) / kchunk;
    double* part = (double*)ctx.alloc((size_t)(nsplit * cnt) * sizeof(double));
    GemmArgs a{na, nb, rows, A, sac, sar, B, sbr, sbc, part, 1, na, 1.0, 0.0, kchunk, cnt, (na + kGT - 1) / kGT};
    {
      ProfScope ps("wide_gram", ctx.stream);
      dgemm_kernel<<<dim3((unsigned)tiles, (unsigned)nsplit), kGNT, 0, ctx.stream>>>(a);
      TTB_LAUNCHED();
      const int grid = (int)std::min<int64_t>(1024, (cnt + 255) / 256);
      split_sum_kernel<<<grid, 256, 0, ctx.stream>>>(part, (int)nsplit, cnt, dst);
      TTB_LAUNCHED();
    }
    ctx.free(part);
  }
  if (tmp) {
    ctx.allreduce_sum(tmp, W, (size_t)cnt);
    ctx.free(tmp);
  }
}

// ------------------------------------------------------------------------
// panel -> dense column-major work matrix (rows in view memory order)
// ------------------------------------------------------------------------
// dst[r + m c] = src(r, c): trans == 0: r = w + rl i (the slab itself);
// trans == 1: r = i + I w, src = slab[c + rl r] (a transpose)
__global__ void __launch_bounds__(256) gather_dense_kernel(Panel P, int64_t m, int b, double* __restrict__ dst) {
  __shared__ double tile[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const int64_t rt = (m + 31) / 32;
  const int ct = (b + 31) / 32;
  for (int64_t t = blockIdx.x; t < rt * ct; t += gridDim.x) {
    const int64_t r0 = (t % rt) * 32;
    const int c0 = (int)(t / rt) * 32;
    if (P.kron.x || !P.trans) {
      // element-wise, rows fastest (V views are the slab; Kronecker slices are formed on load)
      for (int j = ty; j < 32; j += 8) {
        const int64_t r = r0 + tx;
        const int c = c0 + j;
        if (r < m && c < b) {
          double v;
          if (P.kron.x) {
            int64_t w, i;
            if (P.trans) { i = r % P.I; w = r / P.I; }
            else { w = r % P.rl; i = r / P.rl; }
            v = P.load(w, i, c);
          } else {
            v = P.base[r + m * c];
          }
          dst[r + m * c] = v;
        }
      }
    } else {
      for (int j = ty; j < 32; j += 8) {  // read columns fastest
        const int64_t r = r0 + j;
        const int c = c0 + tx;
        tile[j][tx] = (r < m && c < b) ? P.base[c + P.rl * r] : 0.0;
      }
      __syncthreads();
      for (int j = ty; j < 32; j += 8) {  // write rows fastest
        const int64_t r = r0 + tx;
        const int c = c0 + j;
        if (r < m && c < b) dst[r + m * c] = tile[tx][j];
      }
      __syncthreads();
    }
  }
}

__global__ void wide_eye_kernel(double* e, int b) {
  for (int idx = threadIdx.x + blockIdx.x * blockDim.x; idx < b * b; idx += blockDim.x * gridDim.x)
    e[idx] = (idx % b == idx / b) ? 1.0 : 0.0;
}

// dst (ldd) <- src (lds), rows x cols, col-major
__global__ void copy_block_kernel(const double* __restrict__ src, int lds, double* __restrict__ dst, int ldd, int rows,
                                  int cols) {
  for (int idx = threadIdx.x + blockIdx.x * blockDim.x; idx < rows * cols; idx += blockDim.x * gridDim.x) {
    const int r = idx % rows, c = idx / rows;
    dst[r + (int64_t)ldd * c] = src[r + (int64_t)lds * c];
  }
}

// w = z_p - S  (z_p: rows c0.. of z with ld ldz; S, w: nb x k, ld nb)
__global__ void zsub_kernel(const double* __restrict__ z, int ldz, int c0, const double* __restrict__ S, int nb, int k,
                            double* __restrict__ w) {
  for (int idx = threadIdx.x + blockIdx.x * blockDim.x; idx < nb * k; idx += blockDim.x * gridDim.x) {
    const int r = idx % nb, c = idx / nb;
    w[idx] = z[c0 + r + (int64_t)ldz * c] - S[idx];
  }
}

static Panel dense_panel(double* base, int64_t m, int nb) {
  Panel p;
  p.base = base;
  p.rl = 1;
  p.I = m;
  p.rr = nb;
  p.trans = 0;
  p.kron = Kron();
  return p;
}

bool tsqr_needs_wide(const Panel& panel) {
  const int b = (int)panel.ncols();
  const int cls = tsqr_class(b);
  if (cls == 0) return true;
  const int mc = cls == 16 ? Leaf16::MC : cls == 32 ? Leaf32::MC : Leaf64::MC;
  return panel.rs() > mc - b + 1;  // a slice taller than the leaf tile allows
}

void wide_tsqr_factor(Ctx& ctx, const Panel& panel, Tsqr& f) {
  const int b = (int)panel.ncols();
  const int64_t m = panel.rs() * panel.I;
  TTB_CHECK(b >= 1, TTB_ERR_SHAPE, "TSQR needs at least one column");
  const int nblk = (b + 63) / 64;
  TTB_CHECK(nblk <= kMaxWideBlk, TTB_ERR_CAPABILITY, "TSQR: column count " + std::to_string(b) + " exceeds 4096");
  f = Tsqr();
  f.b = b;
  f.cls = 0;
  f.panel = panel;
  f.wide = 1;
  f.wm = m;
  f.wnblk = nblk;
  for (int p = 0; p <= nblk; ++p) f.wc0[p] = (int)(((int64_t)b * p) / nblk);
  const size_t bb = (size_t)b * b;
  const size_t qd = ((size_t)std::max<int64_t>(m, 1) * b + 31) / 32 * 32;
  f.mem = ctx.alloc((qd + bb + 64 * 64) * sizeof(double));
  f.wQ = (double*)f.mem;
  f.R = f.wQ + qd;
  double* eye = f.R + bb;
  fill_zero(ctx, f.R, (int64_t)bb);
  if (m > 0) {
    const int64_t tiles = ((m + 31) / 32) * ((b + 31) / 32);
    const int grid = (int)std::min<int64_t>(tiles, 32LL * ctx.num_sms);
    ProfScope ps("wide_gather", ctx.stream);
    gather_dense_kernel<<<grid, 256, 0, ctx.stream>>>(panel, m, b, f.wQ);
    TTB_LAUNCHED();
  }
  for (int p = 0; p < nblk; ++p) {
    const int c0 = f.wc0[p], nb = f.wc0[p + 1] - c0, rest = b - c0 - nb;
    double* Qp = f.wQ + m * c0;
    Tsqr fp;
    tsqr_factor(ctx, dense_panel(Qp, m, nb), fp);
    try {
      copy_block_kernel<<<8, 256, 0, ctx.stream>>>(fp.R, nb, f.R + c0 + (size_t)b * c0, b, nb, nb);
      TTB_LAUNCHED();
      wide_eye_kernel<<<4, 256, 0, ctx.stream>>>(eye, nb);
      TTB_LAUNCHED();
      // explicit Q_p over its own columns (the implicit factor holds copies of the data)
      tsqr_apply(ctx, fp, eye, nb, dense_panel(Qp, m, nb));
    } catch (...) {
      tsqr_release(ctx, fp);
      throw;
    }
    tsqr_release(ctx, fp);
    if (rest > 0) {
      double* Cn = Qp + m * nb;
      double* S = (double*)ctx.alloc((size_t)nb * rest * sizeof(double));
      tall_gram(ctx, m, nb, rest, Qp, 1, m, Cn, 1, m, S, true);
      copy_block_kernel<<<16, 256, 0, ctx.stream>>>(S, nb, f.R + c0 + (size_t)b * (c0 + nb), b, nb, rest);
      TTB_LAUNCHED();
      dgemm_strided(ctx, m, rest, nb, -1.0, Qp, 1, m, S, 1, nb, 1.0, Cn, 1, m);
      ctx.free(S);
    }
  }
}

void wide_tsqr_apply(Ctx& ctx, const Tsqr& f, const double* z, int k, const Panel& out) {
  TTB_CHECK(k >= 1, TTB_ERR_SHAPE, "TSQR apply: k must be positive");
  TTB_CHECK(out.rs() == f.panel.rs() && out.I == f.panel.I && out.ncols() == k && out.trans == f.panel.trans,
            TTB_ERR_SHAPE, "TSQR apply: output view does not match the factored panel");
  const int64_t m = f.wm;
  const int b = f.b;
  if (m == 0) return;
  // the output view as a strided m x k matrix (rows in view memory order)
  const int64_t scm = out.trans ? k : 1, scn = out.trans ? 1 : m;
  double* S = (double*)ctx.alloc((size_t)2 * 64 * k * sizeof(double));
  double* w = S + (size_t)64 * k;
  for (int p = f.wnblk - 1; p >= 0; --p) {
    const int c0 = f.wc0[p], nb = f.wc0[p + 1] - c0;
    const double* Qp = f.wQ + m * c0;
    if (p == f.wnblk - 1) {
      dgemm_strided(ctx, m, k, nb, 1.0, Qp, 1, m, z + c0, 1, b, 0.0, out.base, scm, scn);
    } else {
      tall_gram(ctx, m, nb, k, Qp, 1, m, out.base, scm, scn, S, true);
      zsub_kernel<<<16, 256, 0, ctx.stream>>>(z, b, c0, S, nb, k, w);
      TTB_LAUNCHED();
      dgemm_strided(ctx, m, k, nb, 1.0, Qp, 1, m, w, 1, nb, 1.0, out.base, scm, scn);
    }
  }
  ctx.free(S);
}

// ------------------------------------------------------------------------
// Gram step for ranks above 64: Z = W H(X), Wn = V(Y)^T V(Z)
// ------------------------------------------------------------------------
void gram_step_wide(Ctx& ctx, const double* W, const double* X, int64_t ral, int64_t rar, const double* Y,
                    int64_t rbl, int64_t rbr, int64_t I, double* Wn) {
  const int64_t cnt = rbr * rar;
  if (I == 0) {
    fill_zero(ctx, Wn, cnt);
    return;
  }
  double* Z = (double*)ctx.alloc((size_t)(rbl * I * rar) * sizeof(double));
  dgemm_strided(ctx, rbl, I * rar, ral, 1.0, W, 1, rbl, X, 1, ral, 0.0, Z, 1, rbl);
  tall_gram(ctx, rbl * I, (int)rbr, (int)rar, Y, 1, rbl * I, Z, 1, rbl * I, Wn, false);
  ctx.free(Z);
}

// ------------------------------------------------------------------------
// one-sided Jacobi SVD of any size (one CTA, data in global memory)
// ------------------------------------------------------------------------
constexpr int kWsNT = 1024;

__device__ __forceinline__ void wide_pair_of(int pr, int round, int np, int& p, int& q) {
  const int M1 = np - 1;
  if (pr == 0) {
    p = M1;
    q = round;
  } else {
    p = round + pr;
    p -= p >= M1 ? M1 : 0;
    q = round - pr;
    q += q < 0 ? M1 : 0;
  }
  if (p > q) {
    const int t = p;
    p = q;
    q = t;
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

__global__ void __launch_bounds__(kWsNT, 1)
jacobi_svd_wide_kernel(const double* __restrict__ Ain, int lda, int m, int n, int transA, double eps, int max_rank,
                       double* Aw, double* Vw, double* nrm, double* sig, int* order, double* tails,
                       double* __restrict__ C, double* __restrict__ Vk, double* __restrict__ s_out,
                       int* __restrict__ info, double* __restrict__ dinfo) {
  __shared__ int s_bad, s_rot, s_big, s_keep;
  __shared__ double s_red[kWsNT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NWARP = kWsNT / 32;
  const int np = (n + 1) & ~1;
  if (tid == 0) s_bad = 0;
  __syncthreads();
  for (int64_t idx = tid; idx < (int64_t)m * n; idx += kWsNT) {
    const int r = (int)(idx % m), c = (int)(idx / m);
    double v = transA ? Ain[c + (int64_t)lda * r] : Ain[r + (int64_t)lda * c];
    if (!isfinite(v)) { s_bad = 1; v = 0.0; }
    Aw[idx] = v;
  }
  for (int64_t idx = tid; idx < (int64_t)n * n; idx += kWsNT) Vw[idx] = (idx % n == idx / n) ? 1.0 : 0.0;
  __syncthreads();
  const double tol = 4.0 * 2.220446049250313e-16 * sqrt((double)m);
  const double tol2 = tol * tol;
  const double noise2 = 2.220446049250313e-16 * 2.220446049250313e-16;
  int sweeps = 0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    // exact squared column norms
    for (int c = warp; c < n; c += NWARP) {
      double acc = 0.0;
      const double* a = Aw + (int64_t)m * c;
      for (int r = lane; r < m; r += 32) acc = fma(a[r], a[r], acc);
      acc = warp_sum(acc);
      if (lane == 0) nrm[c] = acc;
    }
    if (tid == 0) { s_rot = 0; s_big = 0; }
    __syncthreads();
    double nmax = 0.0;
    for (int c = tid; c < n; c += kWsNT) nmax = fmax(nmax, nrm[c]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) nmax = fmax(nmax, __shfl_xor_sync(0xffffffffu, nmax, off));
    if (lane == 0) s_red[warp] = nmax;
    __syncthreads();
    nmax = 0.0;
    for (int q = 0; q < NWARP; ++q) nmax = fmax(nmax, s_red[q]);
    const double floor2 = fmax(noise2 * nmax, eps * eps * 1e-4 / (double)np);
    bool myrot = false, mybig = false;
    for (int round = 0; round < np - 1; ++round) {
      for (int pr = warp; pr < np / 2; pr += NWARP) {
        int p, q;
        wide_pair_of(pr, round, np, p, q);
        if (q >= n) continue;  // the padding slot
        double* ap = Aw + (int64_t)m * p;
        double* aq = Aw + (int64_t)m * q;
        double g = 0.0;
        for (int r = lane; r < m; r += 32) g = fma(ap[r], aq[r], g);
        const double ga = warp_sum(g);
        const double al = nrm[p], be = nrm[q];
        if (ga != 0.0 && ga * ga > tol2 * al * be && fmax(al, be) > floor2) {
          const double dif = be - al;
          const double h = sqrt(fma(dif, dif, 4.0 * ga * ga));
          const double den = fabs(dif) + h;
          const double w = rsqrt(2.0 * h * den);
          const double cs = den * w;
          const double sabs = 2.0 * fabs(ga) * w;
          const double sn = ((dif >= 0.0) == (ga >= 0.0)) ? sabs : -sabs;
          const double tg0 = 4.0 * ga * ga * h * (w * w);
          const double tg = dif >= 0.0 ? tg0 : -tg0;
          for (int r = lane; r < m; r += 32) {
            const double x = ap[r], y = aq[r];
            ap[r] = cs * x - sn * y;
            aq[r] = sn * x + cs * y;
          }
          double* vp = Vw + (int64_t)n * p;
          double* vq = Vw + (int64_t)n * q;
          for (int r = lane; r < n; r += 32) {
            const double x = vp[r], y = vq[r];
            vp[r] = cs * x - sn * y;
            vq[r] = sn * x + cs * y;
          }
          __syncwarp();
          if (lane == 0) {
            nrm[p] = al - tg;
            nrm[q] = be + tg;
          }
          myrot = true;
          mybig |= ga * ga >= 1e-18 * (al * be);
        }
      }
      __syncthreads();
    }
    if (myrot) s_rot = 1;
    if (mybig) s_big = 1;
    __syncthreads();
    const bool stop = !s_rot || !s_big || sweep == 59;
    ++sweeps;
    __syncthreads();
    if (stop) break;
  }
  // singular values, ranking, tail rule (svd.cu)
  for (int c = warp; c < n; c += NWARP) {
    double acc = 0.0;
    const double* a = Aw + (int64_t)m * c;
    for (int r = lane; r < m; r += 32) acc = fma(a[r], a[r], acc);
    acc = warp_sum(acc);
    if (lane == 0) sig[c] = sqrt(acc);
  }
  __syncthreads();
  for (int c = tid; c < n; c += kWsNT) {
    const double v = sig[c];
    int pos = 0;
    for (int o = 0; o < n; ++o) {
      const double w = sig[o];
      pos += (w > v) || (w == v && o < c);
    }
    order[pos] = c;
  }
  __syncthreads();
  if (tid == 0) {
    double tail = 0.0;
    int keep = n;
    tails[n] = 0.0;
    for (int k = n - 1; k >= 0; --k) {
      const double sv = sig[order[k]];
      tail += sv * sv;
      tails[k] = tail;
    }
    const double e2 = eps * eps;
    for (int k = 0; k <= n; ++k) {
      if (tails[k] <= e2) { keep = k; break; }
    }
    if (keep < 1) keep = 1;
    int capped = 0;
    if (max_rank > 0 && keep > max_rank) { keep = max_rank; capped = 1; }
    info[0] = keep;
    info[1] = capped;
    info[2] = s_bad;
    info[3] = sweeps;
    dinfo[0] = sqrt(tails[keep]);
    s_keep = keep;
  }
  for (int k = tid; k < n; k += kWsNT) s_out[k] = sig[order[k]];
  __syncthreads();
  const int keep = s_keep;
  for (int64_t idx = tid; idx < (int64_t)m * keep; idx += kWsNT) {
    const int r = (int)(idx % m), k = (int)(idx / m);
    C[idx] = Aw[r + (int64_t)m * order[k]];
  }
  for (int64_t idx = tid; idx < (int64_t)n * keep; idx += kWsNT) {
    const int r = (int)(idx % n), k = (int)(idx / n);
    Vk[idx] = Vw[r + (int64_t)n * order[k]];
  }
}

void jacobi_svd_wide(Ctx& ctx, const double* A, int lda, int m, int n, bool transA, double eps, int max_rank,
                     double* C, double* Vk, double* s, int* info, double* dinfo) {
  TTB_CHECK(m >= n && n >= 1, TTB_ERR_CAPABILITY, "Jacobi SVD: need 1 <= n <= m");
  const size_t nd = (size_t)m * n + (size_t)n * n + 3 * (size_t)n + 8;
  double* scr = (double*)ctx.alloc(nd * sizeof(double) + (size_t)(n + 2) * sizeof(int));
  double* Aw = scr;
  double* Vw = Aw + (size_t)m * n;
  double* nrm = Vw + (size_t)n * n;
  double* sig = nrm + n;
  double* tails = sig + n;
  int* order = (int*)(tails + n + 2);
  {
    ProfScope ps("jacobi_svd_wide", ctx.stream);
    jacobi_svd_wide_kernel<<<1, kWsNT, 0, ctx.stream>>>(A, lda, m, n, transA ? 1 : 0, eps, max_rank, Aw, Vw, nrm, sig,
                                                        order, tails, C, Vk, s, info, dinfo);
    TTB_LAUNCHED();
  }
  ctx.free(scr);
}

}  // namespace ttb
