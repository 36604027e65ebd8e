// On-device truncated SVD of a small matrix (one-sided Hestenes-Jacobi),
// replacing scipy gesdd + the tail rule of truncated_svd (parallel.py:224-258).
//
// One CTA.  A (m x n, m >= n, n <= 64; or its transpose) and V (n x n) live in
// shared memory.  A round-robin tournament pairs all columns each round;
// a group of 8 threads owns one pair: three dot products (reduced with
// shuffles over the 8 lanes), one Rutishauser rotation, column updates.
// Sweeps repeat until no pair exceeds the orthogonality threshold.
// Afterwards sigma_j = ||a_j||, columns are ranked by sigma (descending,
// ties by index, deterministic), and the reference's tail rule picks keep.
//
// Outputs (all device):
//   C (m x keep, ld m)  = sorted columns of A V        (= U_k diag(s_k))
//   Vk (n x keep, ld n) = sorted columns of V          (right vectors)
//   s (n)               = sorted singular values (all n)
//   info[0] = keep, info[1] = capped ; dinfo[0] = discarded tail
#include "ctx.cuh"
#include "prof.cuh"
#include "svd.cuh"
#include "wide.cuh"

namespace ttb {

#ifndef TTB_SVD_GRP
#define TTB_SVD_GRP 16
#endif
constexpr int kGrp = TTB_SVD_GRP;  // threads per column pair
constexpr int kSvdNT = 2 * 32 * kGrp;  // half on the A columns (one pair slot per group), half trailing on V
constexpr int kSvdMax = 64;
constexpr int kLd = kSvdMax + 1;  // padded column stride: distinct columns start on distinct banks
constexpr int kHalf = kSvdNT / 2;
#ifndef TTB_SVD_DEFLATE
#define TTB_SVD_DEFLATE 1
#endif
constexpr bool kSvdDeflate = TTB_SVD_DEFLATE != 0;
#ifndef TTB_SVD_STOP
#define TTB_SVD_STOP 1e-18  // max cos^2 of a sweep below which the next sweep is skipped
#endif

#ifdef TTB_DEBUG_CLK
static __device__ long long g_sclk[64 * 4];
#define SVD_CLK(ph) do { if (threadIdx.x == 0 && sweep == 0 && round < 64) g_sclk[round * 4 + (ph)] = clock64(); } while (0)
#else
#define SVD_CLK(ph) do {} while (0)
#endif

struct SvdSmem {
  double A[kLd * kSvdMax];   // ld = kLd
  double V[kLd * kSvdMax];
  double nrm[kSvdMax];           // squared column norms, updated with each rotation
  // rotation log of a whole sweep, double buffered by sweep parity: the V
  // side replays sweep s while the A side runs sweep s + 1
  double rotlog[2][kSvdMax][kSvdMax / 2][2];  // [slot][round][pair] (cs, sn); (0, 0): none
  int lcmap[2][kSvdMax];                      // the sweep's tournament slot -> column map
  int lnact[2];
  int lfinal[2];
  unsigned long long logfull[2], logempty[2];  // A -> V (count 1), V -> A (count 1)
  double sig[kSvdMax];
  int order[kSvdMax];
  int cmap[kSvdMax];  // tournament slot -> column (>= n: the empty slot)
  int nact;           // tournament size of the sweep (even)
  int rotated;
  int bad;
  unsigned long long maxoff;  // 1: some rotation of the sweep had ga^2 >= TTB_SVD_STOP al be
};

// reduction over the 8 lanes of one pair group (every lane of the warp
// takes part: each group owns exactly one pair slot, padding slots reduce
// zeros, so the full mask is uniform and the shuffles never serialize)
__device__ __forceinline__ double grp_sum(double v) {
#pragma unroll
  for (int off = kGrp / 2; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// the A-side and V-side thread halves synchronise separately (named barriers)
__device__ __forceinline__ void bar_half(int id) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "n"(kHalf) : "memory"); }
__device__ __forceinline__ unsigned svd_smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void svd_mbar_init(unsigned long long* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(svd_smem_u32(b)) : "memory");
}
__device__ __forceinline__ void svd_mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(svd_smem_u32(b)) : "memory");
}
__device__ __forceinline__ void svd_mbar_wait(unsigned long long* b, unsigned parity) {
  unsigned done = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done)
                 : "r"(svd_smem_u32(b)), "r"(parity)
                 : "memory");
  } while (!done);
}

// columns (p, q) of pair pr in round `round` of the circle-method tournament
// (pr < np/2, round < np-1; no integer division)
__device__ __forceinline__ void pair_of(int pr, int round, int np, int& p, int& q) {
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

// Threads [0, kHalf) run the rotations on A (the serial chain of the
// algorithm); threads [kHalf, kSvdNT) apply each round's rotations to V one
// round later, off that chain.  Column norms are carried along (updated by
// each rotation, recomputed exactly at every sweep start), so a pair needs
// one dot product, not three.
__global__ void __launch_bounds__(kSvdNT, 1)
jacobi_svd_kernel(const double* __restrict__ Ain, int lda, int m, int n, int transA, double eps,
                  int max_rank, double* __restrict__ C, double* __restrict__ Vk, double* __restrict__ s_out,
                  int* __restrict__ info, double* __restrict__ dinfo) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SvdSmem& sm = *reinterpret_cast<SvdSmem*>(smem_raw);
  const int tid = threadIdx.x;
  const int np = (n + 1) & ~1;  // even number of tournament slots (pad column is zero)
  if (tid == 0) {
    sm.bad = 0;
    for (int s2 = 0; s2 < 2; ++s2) {
      svd_mbar_init(&sm.logfull[s2]);
      svd_mbar_init(&sm.logempty[s2]);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  for (int idx = tid; idx < kSvdMax * np; idx += kSvdNT) {
    const int r = idx % kSvdMax, c = idx / kSvdMax;  // rows beyond m stay zero
    double v = 0.0;
    if (r < m && c < n) v = transA ? Ain[c + (int64_t)lda * r] : Ain[r + (int64_t)lda * c];
    if (!isfinite(v)) { sm.bad = 1; v = 0.0; }
    sm.A[r + kLd * c] = v;
    sm.V[r + kLd * c] = (r == c && c < n) ? 1.0 : 0.0;
  }
  __syncthreads();

  const bool vside = tid >= kHalf;
  const int ltid = vside ? tid - kHalf : tid;
  const int grp = ltid / kGrp, gl = ltid % kGrp;
  const double tol = 4.0 * 2.220446049250313e-16 * sqrt((double)m);
  const double tol2 = tol * tol;
  const double noise2 = 2.220446049250313e-16 * 2.220446049250313e-16;
  int sweeps = 0;
  if (!vside) {
    // ---- A side: the rotation chain, barrier over this half only ----
    for (int sweep = 0; sweep < 60; ++sweep) {
      const int slot = sweep & 1;
      // exact squared column norms (one warp per column)
      for (int c = ltid / 32; c < np; c += kHalf / 32) {
        double acc = 0.0;
        for (int r = ltid % 32; r < m; r += 32) acc = fma(sm.A[r + kLd * c], sm.A[r + kLd * c], acc);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if ((ltid % 32) == 0) sm.nrm[c] = acc;
      }
      if (ltid == 0) {
        sm.rotated = 0;
        sm.maxoff = 0ull;
      }
      // the log slot this sweep writes: replayed by the V side two sweeps ago
      if (sweep >= 2) svd_mbar_wait(&sm.logempty[slot], (unsigned)((sweep >> 1) - 1) & 1u);
      bar_half(1);
      double nmax = 0.0;
      for (int c = 0; c < n; ++c) nmax = fmax(nmax, sm.nrm[c]);
      // pairs of columns that are both negligible are left alone: below
      // roundoff of the largest column, or so small that all of them together
      // (<= np * eps^2 * 1e-4 / np) sit inside the discarded tail of the
      // truncation rule -- their mutual rotations cannot change the kept
      // factors, the kept rank or the discarded-tail sum (rotations that
      // involve one non-negligible column are still applied)
      const double floor2 = fmax(noise2 * nmax, eps * eps * 1e-4 / (double)np);
      // deflation: at every sweep start, a column whose norm is at or
      // below the rotation threshold times the largest (4 eps sqrt(m) ||a||max,
      // e.g. the roundoff columns of a rank-deficient R) leaves the tournament:
      // by Weyl, skipping its rotations moves every singular value and factor
      // by at most its norm, the normwise accuracy LAPACK's gesdd itself has.
      // The live columns keep their index order; an odd count is padded with
      // an empty slot
      if (!kSvdDeflate) {
        for (int c = ltid; c < np; c += kHalf) sm.lcmap[slot][c] = c;
        if (ltid == 0) sm.lnact[slot] = np;
      } else if (ltid < 32) {
        int base = 0;
        for (int c0 = 0; c0 < n; c0 += 32) {
          const int c = c0 + ltid;
          const bool act = c < n && sm.nrm[c] > tol2 * nmax;
          const unsigned msk = __ballot_sync(0xffffffffu, act);
          if (act) sm.lcmap[slot][base + __popc(msk & ((1u << ltid) - 1u))] = c;
          base += __popc(msk);
        }
        if (ltid == 0) {
          if (base & 1) sm.lcmap[slot][base] = kSvdMax;
          sm.lnact[slot] = base + (base & 1);
        }
      }
      bar_half(1);
      const int nt = sm.lnact[slot], npairs = nt / 2;
      const int* cmap = sm.lcmap[slot];
      // per-lane sweep flags (published once per sweep, not per rotation:
      // shared atomics of every pair serialised each round)
      bool myrot = false, mybig = false;
      for (int round = 0; round < nt - 1; ++round) {
        SVD_CLK(0);
        // one pair slot per group (npairs <= kHalf / kGrp): the whole
        // warp reaches the shuffles together
        const int pr = grp;
        int p = 0, q = 0;
        const bool live = pr < npairs;
        if (live) {
          pair_of(pr, round, nt, p, q);
          p = cmap[p];
          q = cmap[q];
        }
        const bool valid = live && p < n && q < n;
        double* ap = sm.A + kLd * p;
        double* aq = sm.A + kLd * q;
        double xa[kSvdMax / kGrp], ya[kSvdMax / kGrp];
#pragma unroll
        for (int u = 0; u < kSvdMax / kGrp; ++u) {
          xa[u] = valid ? ap[gl + kGrp * u] : 0.0;
          ya[u] = valid ? aq[gl + kGrp * u] : 0.0;
        }
        double g0 = 0.0, g1 = 0.0;
#pragma unroll
        for (int u = 0; u < kSvdMax / kGrp; u += 2) {
          g0 = fma(xa[u], ya[u], g0);
          g1 = fma(xa[u + 1], ya[u + 1], g1);
        }
        const double al = valid ? sm.nrm[p] : 0.0, be = valid ? sm.nrm[q] : 0.0;
        SVD_CLK(1);
        const double ga = grp_sum(g0 + g1);
        SVD_CLK(2);
        double cs = 0.0, sn = 0.0;
        if (valid && ga != 0.0 && ga * ga > tol2 * al * be && fmax(al, be) > floor2) {
          // with h = sqrt(dif^2 + 4 ga^2) and den = |dif| + h:
          // 1 + t^2 = (den^2 + 4 ga^2) / den^2 = 2 h den / den^2, so
          // cs = den / sqrt(2 h den), sn = sign 2|ga| / sqrt(2 h den):
          // one sqrt and one rsqrt on the chain instead of sqrt, rcp, rsqrt
          // (all terms positive: no cancellation)
          const double dif = be - al;
          const double h = sqrt(fma(dif, dif, 4.0 * ga * ga));
          const double den = fabs(dif) + h;
          const double w = rsqrt(2.0 * h * den);
          cs = den * w;
          const double sabs = 2.0 * fabs(ga) * w;
          sn = ((dif >= 0.0) == (ga >= 0.0)) ? sabs : -sabs;
          // t ga = sign(dif) 2 ga^2 / den and 1 / den = 2 h w^2: no division
          const double tg0 = 4.0 * ga * ga * h * (w * w);
          const double tg = dif >= 0.0 ? tg0 : -tg0;
          SVD_CLK(3);
#pragma unroll
          for (int u = 0; u < kSvdMax / kGrp; ++u) {
            ap[gl + kGrp * u] = cs * xa[u] - sn * ya[u];
            aq[gl + kGrp * u] = sn * xa[u] + cs * ya[u];
          }
          if (gl == 0) {
            sm.nrm[p] = al - tg;
            sm.nrm[q] = be + tg;
          }
          myrot = true;
          mybig |= ga * ga >= TTB_SVD_STOP * (al * be);
        }
        if (live && gl == 0) {
          sm.rotlog[slot][round][pr][0] = cs;
          sm.rotlog[slot][round][pr][1] = sn;
        }
        bar_half(1);
      }
      // quadratic convergence: once every rotation of a sweep had
      // |cos angle(a_p, a_q)| < 1e-9, the next sweep's rotations are of order
      // 1e-18 -- below the rotation threshold tol ~ 1e-14 -- so that sweep
      // would only confirm convergence; skip it
      if (gl == 0 && myrot) sm.rotated = 1;
      if (gl == 0 && mybig) sm.maxoff = 1ull;
      bar_half(1);
      const int any = sm.rotated;
      bool stop = !any || sweep == 59;
#ifndef TTB_SVD_NO_EARLY_STOP
      stop = stop || sm.maxoff == 0ull;  // no rotation with cos^2 >= TTB_SVD_STOP
#endif
      ++sweeps;
      if (ltid == 0) {
        sm.lfinal[slot] = stop ? 1 : 0;
        svd_mbar_arrive(&sm.logfull[slot]);  // release: the log and map of this sweep
      }
      bar_half(1);  // every A thread read rotated / maxoff before the next sweep resets them
      if (stop) break;
    }
  } else {
    // ---- V side: replays each logged sweep one sweep behind, its own barrier ----
    for (int sweep = 0;; ++sweep) {
      const int slot = sweep & 1;
      svd_mbar_wait(&sm.logfull[slot], (unsigned)(sweep >> 1) & 1u);
      const int nt = sm.lnact[slot], npairs = nt / 2;
      const int* cmap = sm.lcmap[slot];
      const bool last = sm.lfinal[slot] != 0;
      for (int rr = 0; rr < nt - 1; ++rr) {
        for (int pr = grp; pr < npairs; pr += kHalf / kGrp) {
          const double cs = sm.rotlog[slot][rr][pr][0], sn = sm.rotlog[slot][rr][pr][1];
          if (cs == 0.0) continue;
          int p, q;
          pair_of(pr, rr, nt, p, q);
          p = cmap[p];
          q = cmap[q];
          double* vp = sm.V + kLd * p;
          double* vq = sm.V + kLd * q;
          double xv[kSvdMax / kGrp], yv[kSvdMax / kGrp];
#pragma unroll
          for (int u = 0; u < kSvdMax / kGrp; ++u) {
            xv[u] = vp[gl + kGrp * u];
            yv[u] = vq[gl + kGrp * u];
          }
#pragma unroll
          for (int u = 0; u < kSvdMax / kGrp; ++u) {
            vp[gl + kGrp * u] = cs * xv[u] - sn * yv[u];
            vq[gl + kGrp * u] = sn * xv[u] + cs * yv[u];
          }
        }
        bar_half(2);
      }
      if (ltid == 0) svd_mbar_arrive(&sm.logempty[slot]);
      if (last) break;
    }
  }
  __syncthreads();
  // singular values
  for (int c = tid / 32; c < n; c += kSvdNT / 32) {
    double acc = 0.0;
    for (int r = tid % 32; r < m; r += 32) acc = fma(sm.A[r + kLd * c], sm.A[r + kLd * c], acc);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if ((tid % 32) == 0) sm.sig[c] = sqrt(acc);
  }
  __syncthreads();
  // deterministic ranking: position = #(larger) + #(equal with lower index)
  for (int c = tid; c < n; c += kSvdNT) {
    const double v = sm.sig[c];
    int pos = 0;
    for (int o = 0; o < n; ++o) {
      const double w = sm.sig[o];
      pos += (w > v) || (w == v && o < c);
    }
    sm.order[pos] = c;
  }
  __syncthreads();
  if (tid == 0) {
    // tail_sq[k] = sum_{j >= k} s_j^2, accumulated from the smallest up
    double tail = 0.0;
    int keep = n;  // tail_sq[n] = 0 <= eps^2 always
    double tails[kSvdMax + 1];
    tails[n] = 0.0;
    for (int k = n - 1; k >= 0; --k) {
      const double sv = sm.sig[sm.order[k]];
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
    info[2] = sm.bad;
    info[3] = sweeps;
    dinfo[0] = sqrt(tails[keep]);
  }
  for (int k = tid; k < n; k += kSvdNT) s_out[k] = sm.sig[sm.order[k]];
  __syncthreads();
  const int keep = info[0];
  for (int idx = tid; idx < m * keep; idx += kSvdNT) {
    const int r = idx % m, k = idx / m;
    C[r + (int64_t)m * k] = sm.A[r + kLd * sm.order[k]];
  }
  for (int idx = tid; idx < n * keep; idx += kSvdNT) {
    const int r = idx % n, k = idx / n;
    Vk[r + (int64_t)n * k] = sm.V[r + kLd * sm.order[k]];
  }
}

// normalize C columns into U (sigma == 0 -> unit vector e_k)
__global__ void svd_u_kernel(const double* C, const double* s, int m, int keep, double* U) {
  for (int idx = threadIdx.x + blockIdx.x * blockDim.x; idx < m * keep; idx += blockDim.x * gridDim.x) {
    const int r = idx % m, k = idx / m;
    const double sv = s[k];
    U[idx] = sv > 0.0 ? C[idx] / sv : (r == k ? 1.0 : 0.0);
  }
}

void jacobi_svd(Ctx& ctx, const double* A, int lda, int m, int n, bool transA, double eps, int max_rank,
                double* C, double* Vk, double* s, int* info, double* dinfo) {
  if (m > kSvdMax) {  // the general path (wide.cu)
    jacobi_svd_wide(ctx, A, lda, m, n, transA, eps, max_rank, C, Vk, s, info, dinfo);
    return;
  }
  TTB_CHECK(m >= n && n >= 1 && m <= kSvdMax, TTB_ERR_CAPABILITY, "Jacobi SVD: need 1 <= n <= m <= 64");
  smem_attr((const void*)jacobi_svd_kernel, sizeof(SvdSmem));
  ProfScope ps("jacobi_svd", ctx.stream);
  static_assert(kSvdMax / 2 <= kHalf / kGrp, "one pair slot per thread group");
  jacobi_svd_kernel<<<1, kSvdNT, sizeof(SvdSmem), ctx.stream>>>(A, lda, m, n, transA ? 1 : 0, eps, max_rank, C, Vk,
                                                               s, info, dinfo);
  TTB_LAUNCHED();
}

void svd_normalize_u(Ctx& ctx, const double* C, const double* s, int m, int keep, double* U) {
  svd_u_kernel<<<1, 256, 0, ctx.stream>>>(C, s, m, keep, U);
  TTB_LAUNCHED();
}

}  // namespace ttb

#ifdef TTB_DEBUG_CLK
extern "C" int ttb_dbg_sclk(long long* out) {
  return cudaMemcpyFromSymbol(out, ttb::g_sclk, sizeof(long long) * 64 * 4) == cudaSuccess ? 0 : 5;
}
#endif
