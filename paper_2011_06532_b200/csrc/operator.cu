// Kronecker-operator apply (ops.py:238-342): mode-2 sparse products of TT
// cores (core.py:285-297) with the distributed halo exchange of
// _apply_term_dist (ops.py:270-311).
//
//   out(a0 + a, i, c0 + c) = sum_{jj in row i} vals[jj] * src(a, cols[jj], c)
//
// src is this rank's slab (columns < nloc) or the halo buffer of slices
// fetched from peers (columns >= nloc, slice-major: each slice an F-order
// rl x rr block, the reference's exchange payload layout, ops.py:284-287).
// The product of term t is written straight into its diagonal block of the
// summed operator core, so the block-diagonal TT sum of the terms
// (ops.py:330-333 -> add, ops.py:79-106) costs no extra pass.
//
// Arithmetic is scipy's csr_matvecs sequence (y = 0; y += a_jj * x_j in
// stored order, separately rounded multiply and add), so results are bitwise
// those of the reference's sparse products.  HBM-bound: each output element
// is written once; source slices are re-read from L1/L2 by neighbouring rows
// (banded factors) -- the cost is one read of the slab and one write.
#include "ops.cuh"
#include "prof.cuh"

namespace ttb {

constexpr int kSpNT = 256;
constexpr int kSpElems = 4096;

__global__ void __launch_bounds__(kSpNT)
mode2_spmm_kernel(int64_t rl, int64_t rr, int64_t nrows, const int64_t* __restrict__ indptr,
                  const int64_t* __restrict__ cols, const double* __restrict__ vals, int64_t nloc,
                  const double* __restrict__ local, const double* __restrict__ halo, double* __restrict__ out,
                  int64_t out_rl, int64_t out_d, int64_t a0, int64_t c0, int ni) {
  const int64_t c = blockIdx.y;
  const int64_t i0 = (int64_t)blockIdx.x * ni;
  const int nn = (int)min64(ni, nrows - i0);
  const double* loc = local + rl * nloc * c;
  const double* hal = halo + rl * c;
  const int64_t hstride = rl * rr;
  double* o = out + a0 + out_rl * (i0 + out_d * (c0 + c));
  const int64_t* ip = indptr + i0;
  // rows a fastest (coalesced stores); per-thread row fixed when rl <= CTA size
  auto cell = [&](int a, int ii) {
    const int64_t beg = ip[ii], end = ip[ii + 1];
    double acc = 0.0;
    for (int64_t jj = beg; jj < end; ++jj) {
      const int64_t j = cols[jj];
      const double x = j < nloc ? loc[a + rl * j] : hal[a + hstride * (j - nloc)];
      acc = __dadd_rn(acc, __dmul_rn(vals[jj], x));
    }
    o[a + out_rl * ii] = acc;
  };
  if (rl <= kSpNT) {
    const int per = kSpNT / (int)rl;
    const int a = threadIdx.x % (int)rl, g = threadIdx.x / (int)rl;
    if (g < per)
      for (int ii = g; ii < nn; ii += per) cell(a, ii);
  } else {
    for (int ii = 0; ii < nn; ++ii)
      for (int a = threadIdx.x; a < rl; a += kSpNT) cell(a, ii);
  }
}

// One pass over a whole summed operator core: every output cell is written
// once -- term t's product in its diagonal block, exact zeros elsewhere --
// so the block-diagonal TT sum of the terms costs no separate zero fill.
// mode 0: interior core (T rl, I, T rr), block diagonal; mode 1: first core
// (1, I, T rr), blocks side by side; mode 2: last core (T rl, I, 1), stacked.
constexpr int kSpMaxTerms = 16;
struct SpmmTerms {
  int nterms;
  const int64_t* indptr[kSpMaxTerms];
  const int64_t* cols[kSpMaxTerms];
  const double* vals[kSpMaxTerms];
  const double* halo[kSpMaxTerms];
};

__global__ void __launch_bounds__(kSpNT)
mode2_spmm_sum_kernel(SpmmTerms st, int mode, int64_t rl, int64_t rr, int64_t nrows, int64_t nloc,
                      const double* __restrict__ local, double* __restrict__ out, int64_t ORL, int ni) {
  const int64_t C = blockIdx.y;
  const int64_t i0 = (int64_t)blockIdx.x * ni;
  const int nn = (int)min64(ni, nrows - i0);
  const int tC = mode == 2 ? -1 : (int)(C / rr);
  const int64_t c = mode == 2 ? 0 : C - (int64_t)tC * rr;
  double* o = out + ORL * (i0 + nrows * C);
  const int64_t hstride = rl * rr;
  auto cell = [&](int A, int ii) {
    int t;
    int64_t a;
    if (mode == 1) {
      t = tC;
      a = A;
    } else {
      t = (int)(A / rl);
      a = A - (int64_t)t * rl;
    }
    double acc = 0.0;
    if (mode == 2 || t == tC) {
      const int64_t* ip = st.indptr[t] + i0;
      const int64_t* cl = st.cols[t];
      const double* vl = st.vals[t];
      const double* loc = local + rl * nloc * c;
      const double* hal = st.halo[t] + rl * c;
      const int64_t beg = ip[ii], end = ip[ii + 1];
      for (int64_t jj = beg; jj < end; ++jj) {
        const int64_t j = cl[jj];
        const double x = j < nloc ? loc[a + rl * j] : hal[a + hstride * (j - nloc)];
        acc = __dadd_rn(acc, __dmul_rn(vl[jj], x));
      }
    }
    o[A + ORL * ii] = acc;
  };
  if (ORL <= kSpNT) {
    const int per = kSpNT / (int)ORL;
    const int A = threadIdx.x % (int)ORL, g = threadIdx.x / (int)ORL;
    if (g < per)
      for (int ii = g; ii < nn; ii += per) cell(A, ii);
  } else {
    for (int ii = 0; ii < nn; ++ii)
      for (int A = threadIdx.x; A < ORL; A += kSpNT) cell(A, ii);
  }
}

__global__ void gather_slices_kernel(int64_t rl, int64_t I, int64_t rr, const double* __restrict__ slab, int64_t n,
                                     const int64_t* __restrict__ idx, double* __restrict__ out) {
  const int64_t per = rl * rr;
  const int64_t total = per * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / per, r = e % per;
    const int64_t a = r % rl, c = r / rl;
    out[e] = slab[a + rl * (idx[k] + I * c)];
  }
}

}  // namespace ttb

using namespace ttb;

extern "C" {

int ttb_mode2_spmm(ttb_ctx* ctx, int64_t rl, int64_t rr, int64_t nrows, const int64_t* indptr, const int64_t* cols,
                   const double* vals, int64_t nloc, const double* local, const double* halo, double* out,
                   int64_t out_rl, int64_t out_d, int64_t a0, int64_t c0) {
  TTB_TRY_BEGIN
  TTB_CHECK(ctx, TTB_ERR_CONTRACT, "null context");
  TTB_CHECK(rl >= 1 && rr >= 1 && nrows >= 0 && nloc >= 0, TTB_ERR_SHAPE, "mode2_spmm: bad slab shape");
  TTB_CHECK(out_rl >= a0 + rl && out_d >= nrows && a0 >= 0 && c0 >= 0, TTB_ERR_SHAPE,
            "mode2_spmm: output block out of range");
  TTB_CHECK(rr <= 65535, TTB_ERR_CAPABILITY, "mode2_spmm: right rank above 65535");
  if (nrows == 0) return TTB_OK;
  Ctx& c = ctx->c;
  int ni = (int)max64(1, kSpElems / rl);
  if (ni > nrows) ni = (int)nrows;
  dim3 grid(ceil_div(nrows, ni), (unsigned)rr);
  ProfScope ps("mode2_spmm", c.stream);
  mode2_spmm_kernel<<<grid, kSpNT, 0, c.stream>>>(rl, rr, nrows, indptr, cols, vals, nloc, local, halo, out, out_rl,
                                                  out_d, a0, c0, ni);
  TTB_LAUNCHED();
  TTB_TRY_END
}

int ttb_mode2_spmm_sum(ttb_ctx* ctx, int nterms, int mode, int64_t rl, int64_t rr, int64_t nrows,
                       const int64_t* const* indptr, const int64_t* const* cols, const double* const* vals,
                       int64_t nloc, const double* local, const double* const* halo, double* out) {
  TTB_TRY_BEGIN
  TTB_CHECK(ctx, TTB_ERR_CONTRACT, "null context");
  TTB_CHECK(nterms >= 1 && nterms <= kSpMaxTerms, TTB_ERR_CAPABILITY, "mode2_spmm_sum: 1..16 terms");
  TTB_CHECK(mode >= 0 && mode <= 2, TTB_ERR_CONTRACT, "mode2_spmm_sum: bad mode");
  TTB_CHECK(rl >= 1 && rr >= 1 && nrows >= 0 && nloc >= 0, TTB_ERR_SHAPE, "mode2_spmm_sum: bad slab shape");
  TTB_CHECK(mode != 1 || rl == 1, TTB_ERR_SHAPE, "mode2_spmm_sum: first core needs r_left 1");
  TTB_CHECK(mode != 2 || rr == 1, TTB_ERR_SHAPE, "mode2_spmm_sum: last core needs r_right 1");
  if (nrows == 0) return TTB_OK;
  SpmmTerms st;
  st.nterms = nterms;
  for (int t = 0; t < nterms; ++t) {
    st.indptr[t] = indptr[t];
    st.cols[t] = cols[t];
    st.vals[t] = vals[t];
    st.halo[t] = halo[t];
  }
  const int64_t ORL = mode == 1 ? 1 : (int64_t)nterms * rl;
  const int64_t ORR = mode == 2 ? 1 : (int64_t)nterms * rr;
  TTB_CHECK(ORR <= 65535, TTB_ERR_CAPABILITY, "mode2_spmm_sum: output right rank above 65535");
  Ctx& c = ctx->c;
  int ni = (int)max64(1, kSpElems / ORL);
  if (ni > nrows) ni = (int)nrows;
  dim3 grid(ceil_div(nrows, ni), (unsigned)ORR);
  ProfScope ps("mode2_spmm", c.stream);
  mode2_spmm_sum_kernel<<<grid, kSpNT, 0, c.stream>>>(st, mode, rl, rr, nrows, nloc, local, out, ORL, ni);
  TTB_LAUNCHED();
  TTB_TRY_END
}

int ttb_gather_slices(ttb_ctx* ctx, int64_t rl, int64_t I, int64_t rr, const double* slab, int64_t n,
                      const int64_t* idx, double* out) {
  TTB_TRY_BEGIN
  TTB_CHECK(ctx, TTB_ERR_CONTRACT, "null context");
  TTB_CHECK(rl >= 1 && rr >= 1 && I >= 0 && n >= 0, TTB_ERR_SHAPE, "gather_slices: bad shape");
  if (n == 0) return TTB_OK;
  Ctx& c = ctx->c;
  const int64_t total = rl * rr * n;
  const int blocks = (int)min64((total + 255) / 256, (int64_t)c.num_sms * 8);
  gather_slices_kernel<<<blocks, 256, 0, c.stream>>>(rl, I, rr, slab, n, idx, out);
  TTB_LAUNCHED();
  TTB_TRY_END
}

int ttb_exchange(ttb_ctx* ctx, int npeers, const int* peers, const double* const* send, const int64_t* send_n,
                 double* const* recv, const int64_t* recv_n) {
  TTB_TRY_BEGIN
  TTB_CHECK(ctx, TTB_ERR_CONTRACT, "null context");
  TTB_CHECK(npeers >= 0, TTB_ERR_CONTRACT, "exchange: negative peer count");
  Ctx& c = ctx->c;
  for (int k = 0; k < npeers; ++k)
    TTB_CHECK(peers[k] >= 0 && peers[k] < c.nranks && peers[k] != c.rank, TTB_ERR_CONTRACT,
              "exchange: bad peer rank " + std::to_string(peers[k]));
  c.sendrecv(npeers, peers, send, send_n, recv, recv_n);
  TTB_TRY_END
}

}  // extern "C"
