// Construction kernels: fused N-ary block-diagonal add with scales
// (ops.py:71-106), slice-wise Kronecker Hadamard (ops.py:109-132), scale,
// and a deterministic sum of squares (parallel.py:362-365).
//
// All are HBM-streaming kernels: each output element is written exactly once
// with coalesced stores (a CTA owns one output column c and a run of slices,
// i.e. a contiguous (a, i) range of the F-order core); inputs are read once
// (add) or from L1/L2-resident slices (Hadamard).  Arithmetic is the exact
// IEEE sequence of the reference (one multiply, left-to-right sums, no FMA
// contraction) so results are bitwise identical to numpy.
#include "ops.cuh"
#include "prof.cuh"

namespace ttb {

constexpr int kEwNT = 256;
constexpr int kEwElems = 4096;  // target output elements per CTA
#ifndef TTB_EW_ELEMS_VEC
#define TTB_EW_ELEMS_VEC 8192
#endif
constexpr int kEwElemsVec = TTB_EW_ELEMS_VEC;  // the paired-row Hadamard path

// Visit the cells (row r, slice ii) of an RL x nn block of an F-order core
// column, rows fastest so stores coalesce.  mk(r) returns the per-row
// functor g(ii); row-dependent index arithmetic (divisions) runs once per
// thread when RL <= the CTA size instead of once per element.
template <class MK>
__device__ __forceinline__ void for_cells(int RL, int nn, MK&& mk) {
  if (RL <= kEwNT) {
    const int per = kEwNT / RL;
    const int r = threadIdx.x % RL, i0 = threadIdx.x / RL;
    if (i0 >= per) return;
    auto g = mk(r);
    for (int ii = i0; ii < nn; ii += per) g(ii);
  } else {
    for (int ii = 0; ii < nn; ++ii)
      for (int r = threadIdx.x; r < RL; r += kEwNT) mk(r)(ii);
  }
}

struct AddArgs {
  int mode;  // 0 interior (block diagonal), 1 first core (concat along c), 2 last core (stack along a), 3 single core (sum)
  int nterms;
  AddTerm t[kMaxAddTerms];
  int64_t RL, I, RR;
  int ni;  // slices per CTA
  int vec;  // interior mode with even blocks and aligned cores: paired rows
  double* out;
};

__global__ void __launch_bounds__(kEwNT) add_kernel(AddArgs a) {
  const int64_t c = blockIdx.y;
  const int64_t i0 = (int64_t)blockIdx.x * a.ni;
  const int64_t ni = min64(a.ni, a.I - i0);
  const int64_t RL = a.RL;
  const int64_t cnt = RL * ni;
  double* out = a.out + RL * (i0 + a.I * c);
  if (a.mode == 3) {
    for (int64_t e = threadIdx.x; e < cnt; e += kEwNT) {
      double acc = __dmul_rn(a.t[0].s, a.t[0].x[i0 + e]);
      for (int p = 1; p < a.nterms; ++p) acc = __dadd_rn(acc, __dmul_rn(a.t[p].s, a.t[p].x[i0 + e]));
      out[e] = acc;
    }
    return;
  }
  // term owning column c (modes 0, 1); for mode 2 the term is chosen per row
  int pc = 0;
  if (a.mode != 2) {
    for (int p = 0; p < a.nterms; ++p)
      if (c >= a.t[p].offc && c < a.t[p].offc + a.t[p].rr) pc = p;
  }
  const AddTerm T = a.t[pc];
  if (a.mode == 1) {  // RL == 1: out(0, i, c) = s_p X_p(0, i, c - offc)
    const double* x = T.x + (i0 + a.I * (c - T.offc));
    for (int64_t e = threadIdx.x; e < cnt; e += kEwNT) out[e] = __dmul_rn(T.s, x[e]);
    return;
  }
  if (a.mode == 2) {  // RR == 1: out(a, i, 0) = X_p(a - offa, i, 0)
    for_cells((int)RL, (int)ni, [&](int ai) {
      int p = 0;
      for (int q = 0; q < a.nterms; ++q)
        if (ai >= a.t[q].offa) p = q;
      const double* x = a.t[p].x + (ai - a.t[p].offa) + a.t[p].rl * i0;
      const int64_t rl = a.t[p].rl;
      return [=](int ii) { out[ai + RL * ii] = x[rl * ii]; };
    });
    return;
  }
  // interior: block diagonal
  const double* x = T.x + T.rl * (i0 + a.I * (c - T.offc));
  if (a.vec) {  // even blocks: row pairs never straddle one; 16-byte loads, streaming stores
    const int RL2 = (int)(RL >> 1), per = kEwNT / RL2;
    const int r2 = threadIdx.x % RL2, it = threadIdx.x / RL2;
    if (it >= per) return;
    const int64_t ai = 2 * r2, al = ai - T.offa;
    const bool in = al >= 0 && al < T.rl;
    const double* xr = x + al;
    const int64_t rl = T.rl;
    for (int ii = it; ii < ni; ii += per) {
      const double2 v = in ? *reinterpret_cast<const double2*>(xr + rl * ii) : make_double2(0.0, 0.0);
      __stcs(reinterpret_cast<double2*>(out + ai + RL * ii), v);
    }
    return;
  }
  for_cells((int)RL, (int)ni, [&](int ai) {
    const int64_t al = ai - T.offa;
    const bool in = al >= 0 && al < T.rl;
    const double* xr = x + al;
    const int64_t rl = T.rl;
    return [=](int ii) { out[ai + RL * ii] = in ? xr[rl * ii] : 0.0; };
  });
}

void add_core(Ctx& ctx, int mode, int nterms, const AddTerm* terms, int64_t RL, int64_t I, int64_t RR, double* out) {
  TTB_CHECK(nterms >= 1 && nterms <= kMaxAddTerms, TTB_ERR_CAPABILITY, "add: 1..16 terms supported");
  if (I == 0 || RL == 0 || RR == 0) return;
  AddArgs a;
  a.mode = mode;
  a.nterms = nterms;
  for (int p = 0; p < nterms; ++p) a.t[p] = terms[p];
  a.RL = RL;
  a.I = I;
  a.RR = RR;
  bool vec = mode == 0 && RL % 2 == 0 && RL / 2 <= kEwNT && (uintptr_t)out % 16 == 0;
  for (int p = 0; p < nterms; ++p)
    vec = vec && terms[p].rl % 2 == 0 && terms[p].offa % 2 == 0 && (uintptr_t)terms[p].x % 16 == 0;
  a.vec = vec ? 1 : 0;
  a.ni = (int)std::max<int64_t>(1, std::min<int64_t>(I, (vec ? kEwElemsVec : kEwElems) / std::max<int64_t>(1, RL)));
  a.out = out;
  TTB_CHECK(RR <= 65535, TTB_ERR_CAPABILITY, "add: output right rank too large");
  dim3 grid((unsigned)((I + a.ni - 1) / a.ni), (unsigned)RR);
  ProfScope ps("add", ctx.stream);
  add_kernel<<<grid, kEwNT, 0, ctx.stream>>>(a);
  TTB_LAUNCHED();
}

// Z(a*rbl + c, i, b*rbr + d) = X(a, i, b) * Y(c, i, d)
__global__ void __launch_bounds__(kEwNT)
hadamard_kernel(const double* __restrict__ x, int64_t ral, int64_t rar, const double* __restrict__ y, int64_t rbl,
                int64_t rbr, int64_t I, int ni, int col_fast, int vec, double* __restrict__ out) {
  // col_fast: the output column is blockIdx.x, so the CTAs of all columns of
  // a slice run are dispatched together and re-read its input slices from L2
  const int64_t col = col_fast ? blockIdx.x : blockIdx.y;
  const int64_t run = col_fast ? blockIdx.y : blockIdx.x;
  const int64_t bx = col / rbr, dy = col - bx * rbr;
  const int64_t RL = ral * rbl;
  const int64_t i0 = run * ni;
  const int64_t nn = min64(ni, I - i0);
  double* o = out + RL * (i0 + I * col);
  const double* xs = x + ral * (i0 + I * bx);
  const double* ys = y + rbl * (i0 + I * dy);
  if (vec) {  // row pairs: one 16-byte Y load and one 16-byte streaming store per pair
    const int RL2 = (int)(RL >> 1), per = kEwNT / RL2;
    const int r2 = threadIdx.x % RL2, it = threadIdx.x / RL2;
    if (it >= per) return;
    const int row = 2 * r2, ax = row / (int)rbl, cy = row - ax * (int)rbl;
    const double* xp = xs + ax;
    const double* yp = ys + cy;
    double* op = o + row;
    for (int ii = it; ii < nn; ii += per) {
      const double xv = xp[ral * ii];
      const double2 yv = *reinterpret_cast<const double2*>(yp + rbl * ii);
      __stcs(reinterpret_cast<double2*>(op + RL * ii), make_double2(__dmul_rn(xv, yv.x), __dmul_rn(xv, yv.y)));
    }
    return;
  }
  for_cells((int)RL, (int)nn, [&](int row) {
    const int ax = row / (int)rbl, cy = row - ax * (int)rbl;
    const double* xp = xs + ax;
    const double* yp = ys + cy;
    double* op = o + row;
    return [=](int ii) { op[RL * ii] = __dmul_rn(xp[ral * ii], yp[rbl * ii]); };
  });
}

void hadamard_core(Ctx& ctx, const double* x, int64_t ral, int64_t rar, const double* y, int64_t rbl, int64_t rbr,
                   int64_t I, double* out) {
  const int64_t RL = ral * rbl, RR = rar * rbr;
  if (I == 0) return;
  TTB_CHECK(RR <= 65535 && RL <= (1 << 24), TTB_ERR_CAPABILITY, "hadamard: output rank too large");
  // rows in pairs when the pair never straddles a Y column and every pair is
  // 16-byte aligned (even rbl; aligned bases)
  const bool vec = rbl % 2 == 0 && RL / 2 <= kEwNT && (uintptr_t)y % 16 == 0 && (uintptr_t)out % 16 == 0;
  const int64_t elems = vec ? kEwElemsVec : kEwElems;
  int ni = (int)std::max<int64_t>(1, std::min<int64_t>(I, elems / std::max<int64_t>(1, RL)));
  const int64_t runs = (I + ni - 1) / ni;
  const bool col_fast = runs <= 65535;
  dim3 grid = col_fast ? dim3((unsigned)RR, (unsigned)runs) : dim3((unsigned)runs, (unsigned)RR);
  ProfScope ps("hadamard", ctx.stream);
  hadamard_kernel<<<grid, kEwNT, 0, ctx.stream>>>(x, ral, rar, y, rbl, rbr, I, ni, col_fast ? 1 : 0, vec ? 1 : 0,
                                                  out);
  TTB_LAUNCHED();
}

__global__ void scale_kernel(int64_t n, const double* __restrict__ x, double s, double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = __dmul_rn(s, x[e]);
}

void scale_vec(Ctx& ctx, int64_t n, const double* x, double s, double* out) {
  if (n == 0) return;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)ctx.num_sms * 8);
  scale_kernel<<<blocks, 256, 0, ctx.stream>>>(n, x, s, out);
  TTB_LAUNCHED();
}

__global__ void fill_zero_kernel(double* p, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    p[e] = 0.0;
}

void fill_zero(Ctx& ctx, double* p, int64_t n) {
  if (n == 0) return;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)ctx.num_sms * 8);
  fill_zero_kernel<<<blocks, 256, 0, ctx.stream>>>(p, n);
  TTB_LAUNCHED();
}

// two-pass deterministic reduction: fixed grid, fixed per-thread order,
// fixed-shape block trees, then one block sums the partials in order.
constexpr int kRedBlocks = 512;

__global__ void __launch_bounds__(256) sumsq_partial_kernel(int64_t n, const double* __restrict__ x,
                                                            double* __restrict__ part) {
  __shared__ double red[256];
  double acc = 0.0;
  for (int64_t e = blockIdx.x * 256LL + threadIdx.x; e < n; e += 256LL * kRedBlocks) acc = fma(x[e], x[e], acc);
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void __launch_bounds__(256) sum_final_kernel(int n, const double* __restrict__ part, double* res) {
  __shared__ double red[256];
  double acc = 0.0;
  for (int e = threadIdx.x; e < n; e += 256) acc += part[e];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *res = red[0];
}

void sumsq_dev(Ctx& ctx, int64_t n, const double* x, double* dres) {
  double* part = (double*)ctx.alloc(kRedBlocks * sizeof(double));
  ProfScope ps("sumsq", ctx.stream);
  sumsq_partial_kernel<<<kRedBlocks, 256, 0, ctx.stream>>>(n, x, part);
  TTB_LAUNCHED();
  sum_final_kernel<<<1, 256, 0, ctx.stream>>>(kRedBlocks, part, dres);
  TTB_LAUNCHED();
  ctx.free(part);
}

}  // namespace ttb
