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

__global__ void gram_final_kernel(const double* __restrict__ part, int nparts, int cnt, double* __restrict__ out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < cnt; e += blockDim.x * gridDim.x) {
    double s = 0.0;
    for (int p = 0; p < nparts; ++p) s += part[(int64_t)p * cnt + e];
    out[e] = s;
  }
}

void gram_step(Ctx& ctx, const double* W, const double* X, int64_t ral, int64_t rar, const double* Y, int64_t rbl,
               int64_t rbr, int64_t I, double* Wn) {
  TTB_CHECK(ral <= 64 && rar <= 64 && rbl <= 64 && rbr <= 64, TTB_ERR_CAPABILITY, "inner product: ranks above 64");
  const int64_t cnt = rbr * rar;
  if (I == 0) {
    fill_zero(ctx, Wn, cnt);
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
  TTB_CUDA(cudaFuncSetAttribute(gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ProfScope ps("gram", ctx.stream);
  gram_kernel<<<grid, kGrNT, smem, ctx.stream>>>(a);
  TTB_LAUNCHED();
  gram_final_kernel<<<(int)std::max<int64_t>(1, (cnt + 255) / 256), 256, 0, ctx.stream>>>(part, grid, (int)cnt, Wn);
  TTB_LAUNCHED();
  ctx.free(part);
}

}  // namespace ttb
