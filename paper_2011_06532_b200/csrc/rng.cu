// Seeded construction on the device, bitwise equal to the reference's host
// generator (core.py:250-266; DistTTTensor.random parallel.py:88-102):
// every global slice i of core n draws rl*rr standard normals from its own
// stream Generator(Philox(SeedSequence(seed, spawn_key=(n, i)))) and lays
// them down left rank fastest, so slabs are P-invariant by construction.
//
// Pieces, each the published algorithm numpy implements:
//  - SeedSequence (O'Neill's seed_seq mixing, numpy.random.bit_generator):
//    entropy = seed words (padded to the 4-word pool) ++ words(n) ++ words(i)
//    hashed into a 4-word pool, then generate_state(2, uint64) -> Philox key.
//    The (seed, n) prefix is mixed once on the host; each thread mixes only
//    its slice index.
//  - Philox4x64-10 (Salmon et al., SC'11), counter starting at 1 (numpy
//    increments before the first block), four outputs per block.
//  - The 256-strip ziggurat of Generator.standard_normal (tables in
//    zig_tables.cuh, see gen_zig_tables.py), with numpy's exact IEEE order
//    of operations (no FMA contraction).
//
// One thread owns one slice; a warp generates 32 consecutive slices one
// right-rank column b at a time and stages them in shared memory so the
// store of out[:, i0:i0+32, b] (contiguous in the F-order core) is
// coalesced.  Work is Philox integer arithmetic (~50 integer ops per
// normal), comparable to the 8-byte HBM write.
//
// The libm-dependent steps.  The wedge test compares against exp(); a
// single-precision screen settles all but the draws within 1e-5 of the
// curve, and those use the device exp (a different decision than glibc's
// would need an exact one-ulp tie).  The exponential tail beyond r (strip 0,
// ~2.5e-4 of draws) evaluates log1p, which numpy takes from the host libm
// and which is not correctly rounded there.  The device decides the tail
// draw and its value whenever every libm-admissible log1p gives the same
// answer; the remaining few attempts are recorded and the host finishes
// them with the same libm log1p numpy calls (values) or confirms them
// (decisions; a disagreement is reported, never silently accepted).
#include <cmath>
#include <vector>

#include "ctx.cuh"
#include "ops.cuh"
#include "prof.cuh"
#include "zig_tables.cuh"

namespace ttb {

namespace {

// SeedSequence constants (numpy.random.bit_generator)
constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;
// Philox4x64 multipliers and Weyl key increments (Random123)
constexpr uint64_t kPhM0 = 0xD2E7470EE14C6C93ull, kPhM1 = 0xCA5A826395121157ull;
constexpr uint64_t kPhW0 = 0x9E3779B97F4A7C15ull, kPhW1 = 0xBB67AE8584CAA73Bull;

constexpr int kRngNT = 128;  // 4 warps, 32 slices each
constexpr int kRngChunk = 16;  // rows of a column staged per pass

__host__ __device__ __forceinline__ uint32_t hashmix(uint32_t v, uint32_t& hc) {
  v ^= hc;
  hc *= kMultA;
  v *= hc;
  return v ^ (v >> 16);
}

__host__ __device__ __forceinline__ uint32_t mixw(uint32_t x, uint32_t y) {
  const uint32_t r = kMixL * x - kMixR * y;
  return r ^ (r >> 16);
}

struct SeedPrefix {
  uint32_t pool[4];
  uint32_t hc;
};

// pool after the run entropy and words(n); the slice index words follow
SeedPrefix seed_prefix(const uint32_t* seed, int nseed, uint64_t n) {
  std::vector<uint32_t> e(seed, seed + nseed);
  if (e.size() < 4) e.resize(4, 0u);  // spawn key present: pad run entropy to the pool
  uint64_t v = n;
  do {
    e.push_back((uint32_t)(v & 0xffffffffu));
    v >>= 32;
  } while (v);
  SeedPrefix p;
  p.hc = kInitA;
  for (int i = 0; i < 4; ++i) p.pool[i] = hashmix(e[i], p.hc);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) p.pool[d] = mixw(p.pool[d], hashmix(p.pool[s], p.hc));
  for (size_t s = 4; s < e.size(); ++s)
    for (int d = 0; d < 4; ++d) p.pool[d] = mixw(p.pool[d], hashmix(e[s], p.hc));
  return p;
}

struct TailRec {
  unsigned long long index;  // element offset in the slab
  double u1, u2;
  unsigned flags;  // 1: accepted on the device, 2: negative, 4: value needs libm, 8: decision needs libm
  unsigned slab;
};

struct SlabDesc {
  SeedPrefix pre;
  int64_t lo, rl, dl, rr;
  double* out;
  int64_t cta0;  // first CTA of this slab in the launch
  unsigned slab;
};

constexpr int kRngMaxSlabs = 64;  // per launch (kernel parameter space)

struct RngBatch {
  SlabDesc d[kRngMaxSlabs];
  int n;
  TailRec* tail;
  unsigned long long* tail_count;
  unsigned long long tail_cap;
};

constexpr int kRing = 16;  // raw draws buffered per thread (shared memory)

// Each thread's Philox output goes through a small ring in shared memory.
// Refills are warp-synchronous (prefetch()): lanes drift apart by the
// variable number of draws a normal consumes (1 on the fast path, 2 in a
// wedge, more in the tail), and a per-lane "refill when empty" would make
// the warp execute the 10-round block for a different lane subset on almost
// every draw.  Topping up every lane with room for a block whenever any lane
// runs low keeps the block computation converged.
struct Stream {
  uint64_t k0, k1, ctr;
  unsigned long long* ring;  // ring[j * kRngNT], j < kRing
  int head, avail;

  __device__ __forceinline__ void push_block() {
    uint64_t x0 = ++ctr, x1 = 0, x2 = 0, x3 = 0;
    uint64_t a = k0, b = k1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      const uint64_t lo0 = kPhM0 * x0, hi0 = __umul64hi(kPhM0, x0);
      const uint64_t lo1 = kPhM1 * x2, hi1 = __umul64hi(kPhM1, x2);
      x0 = hi1 ^ x1 ^ a;
      x1 = lo1;
      x2 = hi0 ^ x3 ^ b;
      x3 = lo0;
      a += kPhW0;
      b += kPhW1;
    }
    const int t = head + avail;
    ring[((t + 0) & (kRing - 1)) * kRngNT] = x0;
    ring[((t + 1) & (kRing - 1)) * kRngNT] = x1;
    ring[((t + 2) & (kRing - 1)) * kRngNT] = x2;
    ring[((t + 3) & (kRing - 1)) * kRngNT] = x3;
    avail += 4;
  }
  // converged top-up before a normal: afterwards every lane holds >= 4 draws
  __device__ __forceinline__ void prefetch(bool live) {
    while (__any_sync(0xffffffffu, live && avail < 4))
      if (live && avail <= kRing - 4) push_block();
  }
  __device__ __forceinline__ uint64_t next() {
    if (avail == 0) push_block();  // only inside long tail loops
    const uint64_t v = ring[head * kRngNT];
    head = (head + 1) & (kRing - 1);
    --avail;
    return v;
  }
  __device__ __forceinline__ double next_double() {
    return __dmul_rn((double)(next() >> 11), 1.0 / 9007199254740992.0);
  }
};

__device__ __forceinline__ void slice_stream(const SeedPrefix& pre, uint64_t i, Stream& st) {
  uint32_t pool[4] = {pre.pool[0], pre.pool[1], pre.pool[2], pre.pool[3]};
  uint32_t hc = pre.hc;
  uint64_t v = i;
  do {
    const uint32_t w = (uint32_t)(v & 0xffffffffu);
#pragma unroll
    for (int d = 0; d < 4; ++d) pool[d] = mixw(pool[d], hashmix(w, hc));
    v >>= 32;
  } while (v);
  uint32_t s[4];
  uint32_t hb = kInitB;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint32_t x = pool[k] ^ hb;
    hb *= kMultB;
    x *= hb;
    s[k] = x ^ (x >> 16);
  }
  st.k0 = (uint64_t)s[0] | ((uint64_t)s[1] << 32);
  st.k1 = (uint64_t)s[2] | ((uint64_t)s[3] << 32);
  st.ctr = 0;
  st.head = 0;
  st.avail = 0;
}

// Interval of values the host libm's log1p can return when the device's
// log1p(-u) is l: both are within one ulp of the exact value (CUDA math
// library and glibc ulp tables), so a +-|l| 2^-50 (>= 4 ulp) box holds it.
__device__ __forceinline__ double libm_slack(double l) { return fabs(l) * 0x1p-50; }

// Strip 0 beyond r: numpy's exponential tail loop.  The device decides
// accept/reject and the value when every libm-admissible log1p gives the
// same result (the operations are monotone, so checking the ends of the
// slack box suffices); otherwise it records the attempt for the host to
// finish with libm (value) or to confirm (decision).
__device__ __forceinline__ double zig_tail(Stream& st, const RngBatch& a, unsigned slab, uint64_t gidx, bool tneg) {
  for (;;) {
    const double u1 = st.next_double();
    const double u2 = st.next_double();
    const double l1 = log1p(-u1), l2 = log1p(-u2);  // <= 0
    const double d1 = libm_slack(l1), d2 = libm_slack(l2);
    const double xx = __dmul_rn(-kZigRinv, l1);
    const double yy = -l2;
    const bool acc = __dadd_rn(yy, yy) > __dmul_rn(xx, xx);
    const double xx_lo = __dmul_rn(-kZigRinv, __dadd_rn(l1, d1)), xx_hi = __dmul_rn(-kZigRinv, __dsub_rn(l1, d1));
    const double yy_lo = -__dadd_rn(l2, d2), yy_hi = -__dsub_rn(l2, d2);
    const bool sure_acc = __dadd_rn(yy_lo, yy_lo) > __dmul_rn(xx_hi, xx_hi);
    const bool sure_rej = !(__dadd_rn(yy_hi, yy_hi) > __dmul_rn(xx_lo, xx_lo));
    const double v_lo = __dadd_rn(kZigR, xx_lo), v_hi = __dadd_rn(kZigR, xx_hi);
    const bool need_value = acc && v_lo != v_hi;
    const bool need_check = !(sure_acc || sure_rej);
    if (need_value || need_check) {
      const unsigned long long slot = atomicAdd(a.tail_count, 1ull);
      if (slot < a.tail_cap) {
        TailRec t;
        t.index = gidx;
        t.u1 = u1;
        t.u2 = u2;
        t.flags = (acc ? 1u : 0u) | (tneg ? 2u : 0u) | (need_value ? 4u : 0u) | (need_check ? 8u : 0u);
        t.slab = slab;
        a.tail[slot] = t;
      }
    }
    if (acc) {
      const double v = __dadd_rn(kZigR, xx);  // == v_lo == v_hi unless need_value
      return tneg ? -v : v;
    }
  }
}

__device__ __forceinline__ double zig_normal(Stream& st, const double* __restrict__ w,
                                             const unsigned long long* __restrict__ k, const double* __restrict__ f,
                                             const RngBatch& a, unsigned slab, uint64_t gidx) {
  for (;;) {
    uint64_t r = st.next();
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const bool neg = r & 1;
    const uint64_t m = (r >> 1) & 0x000fffffffffffffull;
    double x = __dmul_rn((double)m, w[idx]);
    if (neg) x = -x;
    if (m < k[idx]) return x;
    if (idx == 0) return zig_tail(st, a, slab, gidx, (m >> 8) & 1);
    const double u = st.next_double();
    const double y = __dadd_rn(__dmul_rn(__dsub_rn(f[idx - 1], f[idx]), u), f[idx]);
    const double e = __dmul_rn(__dmul_rn(-0.5, x), x);
    // single-precision screen (relative error < 1e-6); the double exp only
    // decides the rare draws within 1e-5 of the curve
    const double ef = (double)__expf((float)e);
    if (y < ef * (1.0 - 1e-5)) return x;
    if (y > ef * (1.0 + 1e-5)) continue;
    if (y < exp(e)) return x;
  }
}

__global__ void __launch_bounds__(kRngNT, 6) random_slab_kernel(const __grid_constant__ RngBatch a) {
  __shared__ double sw[256], sf[256];
  __shared__ unsigned long long sk[256];
  __shared__ unsigned long long ring[kRing * kRngNT];
  __shared__ double stage[kRngNT / 32][kRngChunk * 33];
  for (int t = threadIdx.x; t < 256; t += kRngNT) {
    sw[t] = kZigW[t];
    sk[t] = kZigK[t];
    sf[t] = kZigF[t];
  }
  __syncthreads();
  int si = 0;
  while (si + 1 < a.n && (int64_t)blockIdx.x >= a.d[si + 1].cta0) ++si;
  const SlabDesc& D = a.d[si];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int64_t s0 = (((int64_t)blockIdx.x - D.cta0) * (kRngNT / 32) + wp) * 32;  // first local slice of this warp
  if (s0 >= D.dl) return;
  const int nv = (int)min64(32, D.dl - s0);
  const bool live = lane < nv;
  Stream st;
  st.ring = ring + threadIdx.x;
  slice_stream(D.pre, (uint64_t)(D.lo + s0 + lane), st);
  double* sg = stage[wp];
  const int64_t rl = D.rl, dl = D.dl;
  for (int64_t b = 0; b < D.rr; ++b) {
    double* col = D.out + (b * dl + s0) * rl;  // out[0, s0, b]
    for (int64_t a0 = 0; a0 < rl; a0 += kRngChunk) {
      const int cnt = (int)min64(kRngChunk, rl - a0);
      const uint64_t g0 = (uint64_t)((b * dl + s0 + lane) * rl + a0);
      for (int j = 0; j < cnt; ++j) {
        st.prefetch(live);
        if (live) sg[j * 33 + lane] = zig_normal(st, sw, sk, sf, a, D.slab, g0 + j);
      }
      __syncwarp();
      // out[a0 + j, s0 + q, b] for q < nv, j < cnt
      const int tot = cnt * nv;
      const int dq = 32 / cnt, dj = 32 - dq * cnt;
      int q = lane / cnt, j = lane - q * cnt;
      if (cnt == rl) {
#pragma unroll 4
        for (int e = lane; e < tot; e += 32) {
          col[e] = sg[j * 33 + q];
          q += dq;
          j += dj;
          if (j >= cnt) { j -= cnt; ++q; }
        }
      } else {
        for (int e = lane; e < tot; e += 32) {
          col[(int64_t)q * rl + a0 + j] = sg[j * 33 + q];
          q += dq;
          j += dj;
          if (j >= cnt) { j -= cnt; ++q; }
        }
      }
      __syncwarp();
    }
  }
}

struct TailPatch {
  double* dst;
  double v;
};

__global__ void tail_patch_kernel(const TailPatch* __restrict__ p, int64_t n) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) *p[t].dst = p[t].v;
}

}  // namespace

}  // namespace ttb

using namespace ttb;

extern "C" int ttb_fill_random(ttb_ctx* h, const uint32_t* seed, int nseed, int nslabs, const int64_t* core,
                               const int64_t* lo, const int64_t* rl, const int64_t* dl, const int64_t* rr,
                               double* const* out) {
  TTB_TRY_BEGIN
  Ctx& ctx = h->c;
  TTB_CHECK(seed && nseed >= 1, TTB_ERR_CONTRACT, "fill_random: seed needs at least one 32-bit word");
  TTB_CHECK(nslabs >= 0, TTB_ERR_CONTRACT, "fill_random: negative slab count");
  int64_t total = 0;
  for (int s = 0; s < nslabs; ++s) {
    TTB_CHECK(core[s] >= 0 && lo[s] >= 0 && rl[s] >= 0 && dl[s] >= 0 && rr[s] >= 0, TTB_ERR_SHAPE,
              "fill_random: negative core index, offset or extent");
    total += rl[s] * dl[s] * rr[s];
  }
  if (total == 0) return TTB_OK;
  unsigned long long cap = (unsigned long long)(total / 1024 + 1024);
  for (int attempt = 0; attempt < 2; ++attempt) {
    unsigned long long* count = (unsigned long long*)ctx.alloc(sizeof(unsigned long long) + cap * sizeof(TailRec));
    TailRec* recs = (TailRec*)(count + 1);
    TTB_CUDA(cudaMemsetAsync(count, 0, sizeof(unsigned long long), ctx.stream));
    {
      ProfScope ps("random_slab", ctx.stream);
      RngBatch bt;
      bt.tail = recs;
      bt.tail_count = count;
      bt.tail_cap = cap;
      bt.n = 0;
      int64_t ctas = 0;
      auto flush = [&]() {
        if (bt.n == 0) return;
        TTB_CHECK(ctas < (1ll << 31), TTB_ERR_CAPACITY, "fill_random: too many slices for one launch");
        random_slab_kernel<<<(unsigned)ctas, kRngNT, 0, ctx.stream>>>(bt);
        TTB_LAUNCHED();
        bt.n = 0;
        ctas = 0;
      };
      for (int s = 0; s < nslabs; ++s) {
        if (rl[s] * dl[s] * rr[s] == 0) continue;
        SlabDesc& d = bt.d[bt.n++];
        d.pre = seed_prefix(seed, nseed, (uint64_t)core[s]);
        d.lo = lo[s];
        d.rl = rl[s];
        d.dl = dl[s];
        d.rr = rr[s];
        d.out = out[s];
        d.cta0 = ctas;
        d.slab = (unsigned)s;
        ctas += (dl[s] + kRngNT - 1) / kRngNT;
        if (bt.n == kRngMaxSlabs) flush();
      }
      flush();
    }
    unsigned long long n = 0;
    ctx.read_small(count, sizeof(n), &n);
    if (n > cap) {  // more tail attempts than budgeted: regenerate with room for all
      ctx.free(count);
      cap = n + 1024;
      continue;
    }
    if (n) {
      std::vector<TailRec> hrec(n);
      TTB_CUDA(cudaMemcpyAsync(hrec.data(), recs, n * sizeof(TailRec), cudaMemcpyDeviceToHost, ctx.stream));
      TTB_CUDA(cudaStreamSynchronize(ctx.stream));
      std::vector<TailPatch> patch;
      patch.reserve(n);
      for (const TailRec& t : hrec) {
        // numpy's tail step with the host libm (the reference's own log1p)
        volatile double l1 = std::log1p(-t.u1);
        volatile double l2 = std::log1p(-t.u2);
        volatile double xx = -kZigRinv * l1;
        volatile double yy = -l2;
        volatile double yy2 = yy + yy;
        volatile double xsq = xx * xx;
        const bool acc = yy2 > xsq;
        TTB_CHECK(acc == ((t.flags & 1u) != 0), TTB_ERR_NUMERIC,
                  "fill_random: device and libm disagree on a ziggurat tail decision (an exact tie); "
                  "the stream cannot be reproduced bitwise");
        if (acc && (t.flags & 4u)) {
          volatile double v = kZigR + xx;
          patch.push_back({out[t.slab] + t.index, (t.flags & 2u) ? -v : (double)v});
        }
      }
      if (!patch.empty()) {
        TailPatch* dp = (TailPatch*)ctx.alloc(patch.size() * sizeof(TailPatch));
        TTB_CUDA(cudaMemcpyAsync(dp, patch.data(), patch.size() * sizeof(TailPatch), cudaMemcpyHostToDevice,
                                 ctx.stream));
        tail_patch_kernel<<<(unsigned)((patch.size() + 255) / 256), 256, 0, ctx.stream>>>(dp, (int64_t)patch.size());
        TTB_LAUNCHED();
        TTB_CUDA(cudaStreamSynchronize(ctx.stream));  // the host patch vector goes out of scope
        ctx.free(dp);
      }
    }
    ctx.free(count);
    return TTB_OK;
  }
  TTB_THROW(TTB_ERR_CAPACITY, "fill_random: tail record buffer overflowed twice");
  TTB_TRY_END
}
