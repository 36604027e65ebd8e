// Skinny fp64 products on TT unfoldings: the R-fold of the orthonormalization
// sweeps (dtrmm, parallel.py:192, 206, 334, 356) and the explicit variants'
// carry fold (dgemm, parallel.py:401, 432).
//
//  gemm_small_left : out_H = F * H(X)     (F is M x K, K = r_left <= 64, N = I*r_right huge)
//  gemm_small_right: out_V = V(X) * G     (G is K x Nn, K = r_right <= 64, Mb = r_left*I huge)
//
// Both are one kernel: out(m, j) = sum_k S(m, k) B(k, j) with a small S
// (<= 64 x 64, staged zero-padded in shared memory) and a long j range,
// computed with warp-level fp64 MMA (mma.sync m8n8k4 f64 -- on sm_100a the
// only fp64 tensor path; it matches the DFMA peak at ~1/16 of the issued
// instructions).  Each warp owns 8 consecutive j and all M rows: per k-step
// of 4 it loads one B fragment (streamed from HBM, 32-byte segments) and
// M/8 A fragments from shared memory.  Every output element is written once.
#include "ops.cuh"
#include "wide.cuh"
#include "prof.cuh"
#include "dmma.cuh"

namespace ttb {

constexpr int kSkNT = 256;  // 8 warps
constexpr int kSkMaxM = 64, kSkMaxK = 64;

struct SkinnyArgs {
  int M, K;           // small operand S: M x K
  int64_t N;          // long dimension
  const double* S;    // S(m, k) = S[m * ssm + k * ssk]
  int64_t ssm, ssk;
  const double* B;    // B(k, j) = B[k * bsk + j * bsj]
  int64_t bsk, bsj;
  double* O;          // out(m, j) = O[m * osm + j * osj]
  int64_t osm, osj;
  int upper;          // S is upper triangular (S(m, k) = 0 for k < m): the R-folds (dtrmm)
  // B from an implicit Hadamard core Z (kron.x set, B unused): kmode 1 = H(Z)
  // (B(k, j) = Z[k, j % I, j / I]), kmode 2 = V(Z)^T (B(k, r) = Z[r % zl, r / zl, k])
  Kron kron;
  int kmode = 0;
  int64_t kI = 0, kzl = 0;
};

__device__ __forceinline__ double skinny_b(const SkinnyArgs& a, int k, int64_t j) {
  if (a.kmode == 1) {
    const int64_t m = j / a.kI;
    return a.kron.at(k, j - m * a.kI, m, a.kI);
  }
  if (a.kmode == 2) {
    const int64_t i = j / a.kzl;
    return a.kron.at(j - i * a.kzl, i, k, a.kI);
  }
  return __ldg(&a.B[k * a.bsk + j * a.bsj]);
}

template <int MB>  // M rounded up to MB*8
__global__ void __launch_bounds__(kSkNT) skinny_dmma_kernel(SkinnyArgs a) {
  constexpr int LDS = kSkMaxK + 1;  // padded row stride of the staged S
  __shared__ double Ss[MB * 8 * LDS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int KP = (a.K + 3) & ~3;
  for (int idx = threadIdx.x; idx < MB * 8 * KP; idx += kSkNT) {
    const int m = idx / KP, k = idx % KP;
    Ss[m * LDS + k] = (m < a.M && k < a.K) ? a.S[m * a.ssm + k * a.ssk] : 0.0;
  }
  __syncthreads();
  const int ar = lane >> 2, ac = lane & 3;  // A fragment: row, k
  const int bk = lane & 3, bj = lane >> 2;  // B fragment: k, column
  const int64_t nwarps = (int64_t)gridDim.x * (kSkNT / 32);
  for (int64_t j0 = ((int64_t)blockIdx.x * (kSkNT / 32) + warp) * 8; j0 < a.N; j0 += nwarps * 8) {
    double acc[MB][2];
#pragma unroll
    for (int mb = 0; mb < MB; ++mb) acc[mb][0] = acc[mb][1] = 0.0;
    const int64_t jb = j0 + bj;
    const bool jin = jb < a.N;
    // all B fragments of this 8-column group first: 16 independent loads in flight
    double bf[kSkMaxK / 4];
#pragma unroll
    for (int q = 0; q < kSkMaxK / 4; ++q) {
      const int kb = 4 * q + bk;
      bf[q] = (jin && kb < a.K) ? skinny_b(a, kb, jb) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < kSkMaxK / 4; ++q) {
      if (4 * q >= KP) break;
#pragma unroll
      for (int mb = 0; mb < MB; ++mb) {
        if (a.upper && 4 * q + 4 <= mb * 8) continue;  // all-zero block of a triangular S
        dmma_884(acc[mb][0], acc[mb][1], Ss[(mb * 8 + ar) * LDS + 4 * q + ac], bf[q]);
      }
    }
    // D fragment: row mb*8 + lane/4, columns j0 + 2*(lane%4) + {0, 1}
    const int orow = lane >> 2, ocol = 2 * (lane & 3);
#pragma unroll
    for (int mb = 0; mb < MB; ++mb) {
      const int m = mb * 8 + orow;
      if (m >= a.M) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t j = j0 + ocol + h;
        if (j < a.N) a.O[m * a.osm + j * a.osj] = acc[mb][h];
      }
    }
  }
}

static void launch_skinny(Ctx& ctx, const SkinnyArgs& a) {
  TTB_CHECK(a.M <= kSkMaxM && a.K <= kSkMaxK, TTB_ERR_CAPABILITY, "fold: small dimension above 64");
  if (a.N == 0 || a.M == 0) return;
  const int64_t groups = (a.N + 7) / 8;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((groups + 7) / 8, (int64_t)ctx.num_sms * 8));
  const int MB = (a.M + 7) / 8;
  switch (MB) {
#define TTB_SK(X) \
  case X: skinny_dmma_kernel<X><<<blocks, kSkNT, 0, ctx.stream>>>(a); break;
    TTB_SK(1) TTB_SK(2) TTB_SK(3) TTB_SK(4) TTB_SK(5) TTB_SK(6) TTB_SK(7) TTB_SK(8)
#undef TTB_SK
    default: TTB_THROW(TTB_ERR_CAPABILITY, "fold: M above 64");
  }
  TTB_LAUNCHED();
}

// ---------------------------------------------------------------------------
// Left fold on a persistent, bulk-copy pipelined kernel: B = H (K x N,
// column-major, ld K) is streamed in chunks of kFoldJ columns -- one
// contiguous block, one bulk copy (TMA engine) each, kFoldStages - 1 chunks
// in flight -- and multiplied by the small operand held in shared memory.
// ---------------------------------------------------------------------------
#ifndef TTB_FOLD_J
#define TTB_FOLD_J 64
#endif
#ifndef TTB_FOLD_STAGES
#define TTB_FOLD_STAGES 2
#endif
#ifndef TTB_FOLD_MINB
#define TTB_FOLD_MINB 2
#endif
constexpr int kFoldJ = TTB_FOLD_J;
constexpr int kFoldStages = TTB_FOLD_STAGES;
constexpr int kFoldNT = 256;
constexpr int kFoldMinB = TTB_FOLD_MINB;  // resident CTAs per SM

__device__ __forceinline__ unsigned fd_smem(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// RIGHT = false: B = H, one contiguous K x J block per chunk (ld K).
// RIGHT = true:  B(k, j) = V[j + Mb k] (the right fold V R^T): a chunk is K
//                runs of J doubles, one bulk copy each, staged k-major with a
//                padded row (ldB = 4 mod 16: conflict-free B fragments).
template <bool RIGHT, int J>
__global__ void __launch_bounds__(kFoldNT, kFoldMinB) fold_kernel(SkinnyArgs a) {
  constexpr int kFoldJ = J;  // columns per chunk
  extern __shared__ __align__(128) double fsm[];
  constexpr int NW = kFoldNT / 32;
  const int M = a.M, K = a.K;
  const int64_t N = a.N;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int fr = lane >> 2, fc = lane & 3;
  const int ldS = ((K + 11) & ~15) + 4;  // >= K, 4 mod 16
  const int MP = (M + 15) & ~15, KP = (K + 3) & ~3;
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(fsm);
  unsigned* cnt = reinterpret_cast<unsigned*>(fsm + 8);  // warps done with a stage
  double* Ss = fsm + 16;                          // MP x ldS (row m)
  double* Bs = Ss + (int64_t)MP * ldS;            // stages of K x kFoldJ
  Bs += (16 - ((Bs - fsm) & 15)) & 15;
  constexpr int ldB = kFoldJ + 4;                 // RIGHT: row stride of a stage
  const int64_t bstage = RIGHT ? (int64_t)K * ldB : (int64_t)K * kFoldJ;
  if (tid < kFoldStages) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(fd_smem(&bar[tid])) : "memory");
    cnt[tid] = 0;
  }
  if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  for (int idx = tid; idx < MP * ldS; idx += kFoldNT) {
    const int m = idx / ldS, k = idx % ldS;
    Ss[idx] = (m < M && k < K) ? a.S[m * a.ssm + k * a.ssk] : 0.0;
  }
  const int64_t nch = (N + kFoldJ - 1) / kFoldJ;
  __syncthreads();
  auto issue = [&](int64_t c, int st) {
    const int64_t j0 = c * kFoldJ;
    const int nj = (int)min64(kFoldJ, N - j0);
    const unsigned bytes = (unsigned)(K * nj * 8);
    if constexpr (!RIGHT) {
      if (lane != 0) return;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(fd_smem(&bar[st])), "r"(bytes)
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                       fd_smem(Bs + st * bstage)),
                   "l"(a.B + K * j0), "r"(bytes), "r"(fd_smem(&bar[st]))
                   : "memory");
    } else {
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(fd_smem(&bar[st])), "r"(bytes)
                     : "memory");
      __syncwarp();
      for (int k = lane; k < K; k += 32)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                         fd_smem(Bs + st * bstage + (int64_t)k * ldB)),
                     "l"(a.B + j0 + a.bsk * k), "r"((unsigned)(nj * 8)), "r"(fd_smem(&bar[st]))
                     : "memory");
    }
  };
  int st = 0, ph = 0, fill = 0;
  if (warp == 0)  // issue() is run by one whole warp
    for (int64_t c = blockIdx.x; c < nch && fill < kFoldStages; c += gridDim.x, ++fill) issue(c, fill);
  const int mt = MP / 16, ntl = kFoldJ / 16;
  for (int64_t c = blockIdx.x; c < nch; c += gridDim.x) {
    const int64_t j0 = c * kFoldJ;
    const int nj = (int)min64(kFoldJ, N - j0);
    unsigned done = 0;
    do {
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(fd_smem(&bar[st])), "r"(ph)
          : "memory");
    } while (!done);
    const double* bs = Bs + st * bstage;
    for (int blk = warp; blk < mt * ntl; blk += NW) {
      const int m0 = (blk % mt) * 16, n0 = (blk / mt) * 16;
      double acc[2][2][2];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      const bool c0 = n0 + fr < nj, c1 = n0 + 8 + fr < nj;
      // B(k, n): left Bs[k + K n], right Bs[n + ldB k]
      const double* b0p = RIGHT ? bs + (n0 + fr) : bs + (int64_t)K * (n0 + fr);
      const double* b1p = RIGHT ? bs + (n0 + 8 + fr) : bs + (int64_t)K * (n0 + 8 + fr);
      constexpr int bks = RIGHT ? ldB : 1;
      const double* a0p = Ss + (int64_t)(m0 + fr) * ldS;
      const double* a1p = Ss + (int64_t)(m0 + 8 + fr) * ldS;
      // upper-triangular S (the R-fold, dtrmm): rows m0.. have no entries left of column m0
#pragma unroll 4
      for (int k0 = a.upper ? m0 : 0; k0 < KP; k0 += 4) {
        const int k = k0 + fc;
        const bool kin = k < K;
        const double a0 = a0p[k], a1 = a1p[k];  // zero padded
        const double b0 = (c0 && kin) ? b0p[k * bks] : 0.0;
        const double b1 = (c1 && kin) ? b1p[k * bks] : 0.0;
        dmma_884(acc[0][0][0], acc[0][0][1], a0, b0);
        dmma_884(acc[0][1][0], acc[0][1][1], a0, b1);
        dmma_884(acc[1][0][0], acc[1][0][1], a1, b0);
        dmma_884(acc[1][1][0], acc[1][1][1], a1, b1);
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int m = m0 + 8 * i + fr, n = n0 + 8 * jj + 2 * fc + h;
            if (m < M && n < nj) {
              if constexpr (RIGHT) a.O[m * a.osm + (j0 + n)] = acc[i][jj][h];
              else a.O[m + (int64_t)M * (j0 + n)] = acc[i][jj][h];
            }
          }
    }
    // no CTA-wide barrier per chunk: every warp counts itself out of the stage
    // and the last one out refills it, so the stores of one warp overlap the
    // MMAs of the others
    __syncwarp();
    unsigned old = 0;
    if (lane == 0)
      asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;\n" : "=r"(old) : "r"(fd_smem(&cnt[st])) : "memory");
    old = __shfl_sync(0xffffffffu, old, 0);
    if (old == NW - 1) {
      if (lane == 0) cnt[st] = 0;
      const int64_t nxt = c + (int64_t)kFoldStages * gridDim.x;
      if (nxt < nch) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        issue(nxt, st);
      }
    }
    if (++st == kFoldStages) {
      st = 0;
      ph ^= 1;
    }
  }
}

template <bool RIGHT, int J>
static bool fold_tma(Ctx& ctx, const SkinnyArgs& a) {
  constexpr int kFoldJ = J;
  // bulk copies need 16-byte sizes / addresses: K * columns (left) or the
  // row count and leading dimension (right) even, aligned base
  if (((uintptr_t)a.B & 15) || a.N < (int64_t)kFoldJ * ctx.num_sms) return false;  // (enough chunks for every SM)
  if (!RIGHT && a.K % 2 != 0) return false;
  if (RIGHT && ((a.N % 2) || (a.bsk % 2) || a.bsj != 1)) return false;
  const int ldS = ((a.K + 11) & ~15) + 4, MP = (a.M + 15) & ~15;
  const size_t bst = RIGHT ? (size_t)a.K * (kFoldJ + 4) : (size_t)a.K * kFoldJ;
  const size_t smem = (16 + (size_t)MP * ldS + 16 + (size_t)kFoldStages * bst) * sizeof(double);
  smem_attr((const void*)fold_kernel<RIGHT, J>, 227 * 1024);
  if (smem * kFoldMinB > 227 * 1024) return false;
  const int64_t nch = (a.N + kFoldJ - 1) / kFoldJ;
  const int grid = (int)std::min<int64_t>(nch, (int64_t)kFoldMinB * ctx.num_sms);
  fold_kernel<RIGHT, J><<<grid, kFoldNT, smem, ctx.stream>>>(a);
  TTB_LAUNCHED();
  return true;
}

// out_H (M x N) = F (M x K) * H (K x N); H col-major ld K, out col-major ld M
// (kz: H = H(Z) of an implicit Hadamard core with I slices instead of a buffer)
void gemm_small_left(Ctx& ctx, int M, int K, int64_t N, const double* F, int ldf, bool transF, const double* H,
                     double* out, bool upper, const Kron* kz, int64_t kI) {
  if (M > kSkMaxM || K > kSkMaxK) {  // the general path (wide.cu)
    TTB_CHECK(!(kz && kz->x), TTB_ERR_CAPABILITY, "fold: implicit Hadamard cores need ranks <= 64");
    dgemm_strided(ctx, M, N, K, 1.0, F, transF ? ldf : 1, transF ? 1 : ldf, H, 1, K, 0.0, out, 1, M);
    return;
  }
  ProfScope ps("fold_left", ctx.stream);
  SkinnyArgs a;
  a.M = M;
  a.K = K;
  a.N = N;
  a.S = F;
  a.ssm = transF ? ldf : 1;  // F(i, l) = transF ? F[l + ldf*i] : F[i + ldf*l]
  a.ssk = transF ? 1 : ldf;
  a.B = H;
  a.bsk = 1;
  a.bsj = K;
  a.O = out;
  a.osm = 1;
  a.osj = M;
  a.upper = upper ? 1 : 0;
  if (kz && kz->x) {  // Z formed on the fly: the generic fragment-loading kernel
    a.kron = *kz;
    a.kmode = 1;
    a.kI = kI;
    launch_skinny(ctx, a);
    return;
  }
  if (getenv("TTB_FOLD_V1") == nullptr && fold_tma<false, 64>(ctx, a)) return;
  launch_skinny(ctx, a);
}

// out_V (Mb x Nn) = V (Mb x K) * G (K x Nn): computed as out^T = G^T V^T
void gemm_small_right(Ctx& ctx, int64_t Mb, int K, int Nn, const double* V, const double* G, int ldg, bool transG,
                      double* out, bool upper, const Kron* kz, int64_t kI) {
  if (Nn > kSkMaxM || K > kSkMaxK) {  // the general path (wide.cu)
    TTB_CHECK(!(kz && kz->x), TTB_ERR_CAPABILITY, "fold: implicit Hadamard cores need ranks <= 64");
    dgemm_strided(ctx, Mb, Nn, K, 1.0, V, 1, Mb, G, transG ? ldg : 1, transG ? 1 : ldg, 0.0, out, 1, Mb);
    return;
  }
  ProfScope ps("fold_right", ctx.stream);
  SkinnyArgs a;
  a.M = Nn;
  a.K = K;
  a.N = Mb;
  a.S = G;  // S(c, k) = G(k, c) = transG ? G[c + ldg*k] : G[k + ldg*c]
  a.ssm = transG ? 1 : ldg;
  a.ssk = transG ? ldg : 1;
  a.B = V;  // B(k, r) = V(r, k) = V[r + Mb*k]
  a.bsk = Mb;
  a.bsj = 1;
  a.O = out;  // out(c, r) = out_V(r, c) = out[r + Mb*c]
  a.osm = Mb;
  a.osj = 1;
  a.upper = upper ? 1 : 0;  // S = G^T: upper triangular when G is lower (V R^T)
  if (kz && kz->x) {
    a.kron = *kz;
    a.kmode = 2;
    a.kI = kI;
    a.kzl = kz->rxl * kz->rwl;
    launch_skinny(ctx, a);
    return;
  }
  // right fold: K runs per chunk -- wider chunks for small K keep each copy >= 2 KB
  if (getenv("TTB_FOLD_V1") == nullptr && (K <= 16 ? fold_tma<true, 256>(ctx, a) : fold_tma<true, 64>(ctx, a))) return;
  launch_skinny(ctx, a);
}

}  // namespace ttb
