// Skinny fp64 products on TT unfoldings: the R-fold of the orthonormalization
// sweeps (dtrmm, parallel.py:192, 206, 334, 356) and the explicit variants'
// carry fold (dgemm, parallel.py:401, 432).
//
//  gemm_small_left : out_H = F * H(X)     (F is M x K, K = r_left <= 64, N = I*r_right huge)
//  gemm_small_right: out_V = V(X) * G     (G is K x Nn, K = r_right <= 64, Mb = r_left*I huge)
//
// The small matrix sits in shared memory; the big operand streams through
// once, coalesced, and every output element is written once.
#include "ops.cuh"
#include "prof.cuh"

namespace ttb {

constexpr int kGlNT = 256, kGlNB = 64, kGlTM = 4, kGlTN = 4;

__global__ void __launch_bounds__(kGlNT) gemm_small_left_kernel(int M, int K, int64_t N, const double* __restrict__ F,
                                                                int ldf, int transF, const double* __restrict__ H,
                                                                double* __restrict__ out) {
  extern __shared__ __align__(16) double gl_sm[];
  double* Fs = gl_sm;             // M x K, ld M
  double* Hs = Fs + M * K;        // K x NB, ld K
  const int tid = threadIdx.x;
  for (int e = tid; e < M * K; e += kGlNT) {
    const int i = e % M, l = e / M;
    Fs[e] = transF ? F[l + (int64_t)ldf * i] : F[i + (int64_t)ldf * l];
  }
  const int tm = (M + kGlTM - 1) / kGlTM;
  for (int64_t j0 = (int64_t)blockIdx.x * kGlNB; j0 < N; j0 += (int64_t)gridDim.x * kGlNB) {
    const int nb = (int)min64(kGlNB, N - j0);
    __syncthreads();
    for (int e = tid; e < K * nb; e += kGlNT) Hs[e] = H[(int64_t)K * j0 + e];
    __syncthreads();
    const int tn = (nb + kGlTN - 1) / kGlTN;
    for (int t = tid; t < tm * tn; t += kGlNT) {
      const int i0 = (t % tm) * kGlTM, c0 = (t / tm) * kGlTN;
      double acc[kGlTM][kGlTN];
#pragma unroll
      for (int u = 0; u < kGlTM; ++u)
#pragma unroll
        for (int v = 0; v < kGlTN; ++v) acc[u][v] = 0.0;
      for (int l = 0; l < K; ++l) {
        double f[kGlTM], h[kGlTN];
#pragma unroll
        for (int u = 0; u < kGlTM; ++u) f[u] = (i0 + u < M) ? Fs[(i0 + u) + M * l] : 0.0;
#pragma unroll
        for (int v = 0; v < kGlTN; ++v) h[v] = (c0 + v < nb) ? Hs[l + K * (c0 + v)] : 0.0;
#pragma unroll
        for (int u = 0; u < kGlTM; ++u)
#pragma unroll
          for (int v = 0; v < kGlTN; ++v) acc[u][v] = fma(f[u], h[v], acc[u][v]);
      }
#pragma unroll
      for (int v = 0; v < kGlTN; ++v)
#pragma unroll
        for (int u = 0; u < kGlTM; ++u)
          if (i0 + u < M && c0 + v < nb) out[(i0 + u) + (int64_t)M * (j0 + c0 + v)] = acc[u][v];
    }
  }
}

void gemm_small_left(Ctx& ctx, int M, int K, int64_t N, const double* F, int ldf, bool transF, const double* H,
                     double* out) {
  TTB_CHECK(M <= 64 && K <= 64, TTB_ERR_CAPABILITY, "fold: small dimension above 64");
  if (N == 0 || M == 0) return;
  const size_t smem = (size_t)(M * K + K * kGlNB) * sizeof(double);
  TTB_CUDA(cudaFuncSetAttribute(gemm_small_left_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t blocks = std::min<int64_t>((N + kGlNB - 1) / kGlNB, (int64_t)ctx.num_sms * 4);
  ProfScope ps("fold_left", ctx.stream);
  gemm_small_left_kernel<<<(int)blocks, kGlNT, smem, ctx.stream>>>(M, K, N, F, ldf, transF ? 1 : 0, H, out);
  TTB_LAUNCHED();
}

template <int NC>
__global__ void __launch_bounds__(256) gemm_small_right_kernel(int64_t Mb, int K, int Nn, const double* __restrict__ V,
                                                               const double* __restrict__ G, int ldg, int transG,
                                                               double* __restrict__ out) {
  __shared__ __align__(16) double Gs[64 * NC];  // K x NC, ld NC (row k contiguous)
  for (int e = threadIdx.x; e < K * NC; e += 256) {
    const int l = e / NC, c = e % NC;
    Gs[e] = (c < Nn) ? (transG ? G[c + (int64_t)ldg * l] : G[l + (int64_t)ldg * c]) : 0.0;
  }
  __syncthreads();
  for (int64_t r = blockIdx.x * 256LL + threadIdx.x; r < Mb; r += 256LL * gridDim.x) {
    double acc[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = 0.0;
    for (int l = 0; l < K; ++l) {
      const double v = V[r + Mb * l];
#pragma unroll
      for (int c = 0; c < NC; ++c) acc[c] = fma(v, Gs[l * NC + c], acc[c]);
    }
#pragma unroll
    for (int c = 0; c < NC; ++c)
      if (c < Nn) out[r + Mb * c] = acc[c];
  }
}

void gemm_small_right(Ctx& ctx, int64_t Mb, int K, int Nn, const double* V, const double* G, int ldg, bool transG,
                      double* out) {
  TTB_CHECK(K <= 64 && Nn <= 64, TTB_ERR_CAPABILITY, "fold: small dimension above 64");
  if (Mb == 0 || Nn == 0) return;
  const int blocks = (int)std::min<int64_t>((Mb + 255) / 256, (int64_t)ctx.num_sms * 8);
  ProfScope ps("fold_right", ctx.stream);
  if (Nn <= 16)
    gemm_small_right_kernel<16><<<blocks, 256, 0, ctx.stream>>>(Mb, K, Nn, V, G, ldg, transG ? 1 : 0, out);
  else if (Nn <= 32)
    gemm_small_right_kernel<32><<<blocks, 256, 0, ctx.stream>>>(Mb, K, Nn, V, G, ldg, transG ? 1 : 0, out);
  else
    gemm_small_right_kernel<64><<<blocks, 256, 0, ctx.stream>>>(Mb, K, Nn, V, G, ldg, transG ? 1 : 0, out);
  TTB_LAUNCHED();
}

}  // namespace ttb
