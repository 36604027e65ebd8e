/*
 * ttb.h -- C ABI of the B200-native TT-rounding library (libttb, built as
 * paper_2011_06532_b200/_ttb.so).
 *
 * This is the drop-in boundary for the hot path named in BASELINE.json:
 * TT-rounding with its Gram-sweep (inner product / norm), orthonormalization,
 * and the add / Hadamard constructors.  Every entry point replaces one call
 * of the reference package `ttpar` (pure Python + scipy LAPACK); the
 * reference interface each one stands in for is cited beside it
 * (paths relative to /root/reference/pkg/src/ttpar/).
 *
 * Conventions
 *  - Plain C types only: device pointers as `double*`, sizes as int64_t,
 *    CUDA streams as `void*` (a cudaStream_t).  No torch types.
 *  - A TT "slab set" is ndim device arrays; core n is the LOCAL block of
 *    mode-n slices owned by this rank, Fortran-ordered with shape
 *    (ranks[n], dims[n], ranks[n+1]) -- the reference's natural descending
 *    layout (core.py:1-23) restricted to block_bounds rows (parallel.py:42-46).
 *  - Inputs are never modified (value semantics, parallel.py:315, ops.py:74).
 *    Outputs are caller-allocated; for rank-reducing calls they are sized by
 *    the INPUT ranks and the kernels write the (smaller) result packed at
 *    the front of each buffer, reporting the actual ranks.
 *  - Every function returns TTB_OK (0) or an error code; the message is in
 *    ttb_last_error().  Codes map 1:1 onto the reference's exception classes
 *    (errors.py:4-33).  Calls are asynchronous on the context stream unless
 *    they return a host value (then they synchronize that stream).
 *  - Multi-GPU: one process per GPU.  Call ttb_ctx_init_comm on every rank
 *    with the same 128-byte NCCL unique id; all collective calls must then
 *    be made by every rank in the same order (the reference's SPMD contract,
 *    comm.py:134-160).  Not thread-safe per context.
 */
#ifndef TTB_H_
#define TTB_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TTB_ABI_VERSION 1

enum {
  TTB_OK = 0,
  TTB_ERR_SHAPE = 1,      /* ttpar.errors.ShapeError      */
  TTB_ERR_CONTRACT = 2,   /* ttpar.errors.ContractError   */
  TTB_ERR_NUMERIC = 3,    /* ttpar.errors.NumericError    */
  TTB_ERR_CAPACITY = 4,   /* ttpar.errors.CapacityError   */
  TTB_ERR_CUDA = 5,       /* CUDA runtime failure          */
  TTB_ERR_NCCL = 6,       /* NCCL failure                  */
  TTB_ERR_CAPABILITY = 7, /* ttpar.errors.CapabilityError */
  TTB_ERR_DEADLOCK = 8    /* ttpar.errors.DeadlockError: a collective
                             timed out waiting for a peer (comm.py:20-33) */
};

typedef struct ttb_ctx ttb_ctx;
typedef struct ttb_tsqr ttb_tsqr;
typedef struct ttb_group ttb_group;

/* ---- library / context ------------------------------------------------ */
const char* ttb_last_error(void);
int ttb_abi_version(void);
/* number of kernels this library has launched in the process (evidence) */
long long ttb_launch_counter(void);

/* collective traffic issued by this process since load (the reference's
 * Trace words / messages, comm.py:57-124): out4 = {TSQR allgathers, their
 * doubles sent, allreduces + point-to-point transfers, their doubles} */
int ttb_comm_stats(long long* out4);

/* One context per (process, device).  Replaces the Communicator endpoint
 * (comm.py:134-160; SerialComm comm.py:163-181). */
int ttb_ctx_create(int device, void* stream, ttb_ctx** out);
int ttb_ctx_destroy(ttb_ctx* ctx);
int ttb_ctx_set_stream(ttb_ctx* ctx, void* stream);
/* Return the device memory the library's stream-ordered pool keeps cached
 * (workspace is kept mapped between calls for speed) to the driver, after
 * the context's streams drained.  The analogue of torch.cuda.empty_cache(). */
int ttb_ctx_trim(ttb_ctx* ctx);
/* NCCL bootstrap: rank 0 creates the id, the host broadcasts it
 * (replaces MPICommunicator, comm.py:359-401). */
int ttb_comm_unique_id(void* out128);
int ttb_ctx_init_comm(ttb_ctx* ctx, int nranks, int rank, const void* id128);

/* In-process group: nranks contexts of ONE process (one host thread per
 * rank, possibly all on one device) joined into a P-rank group whose
 * collectives -- the TSQR triangle allgather, the Gram / norm allreduces and
 * the operator halo exchange -- are stream-ordered device copies with a host
 * rendezvous instead of NCCL calls, at the same call sites.  The stand-in
 * for the reference's thread simulator SimComm / run_spmd (comm.py:184-356):
 * it runs the native multi-rank path (P > 1 R stacks, redundant global
 * trees, rank-offset applies, allreduced Gram partials) on one GPU.
 * Reductions are rank-ascending sums.  A rank that fails or waits longer
 * than TTB_GROUP_TIMEOUT_S (default 300) seconds breaks the group: every
 * later collective returns TTB_ERR_DEADLOCK. */
int ttb_group_create(int nranks, ttb_group** out);
int ttb_group_destroy(ttb_group* grp);
/* break the group: peers blocked in (or later entering) a collective get
 * TTB_ERR_DEADLOCK (a rank that failed outside the library calls this) */
int ttb_group_abort(ttb_group* grp);
int ttb_ctx_join_group(ttb_ctx* ctx, ttb_group* grp, int rank);

/* ---- construction (no communication) ---------------------------------- */
/* out = s * x elementwise over n doubles (scale folds into core 0,
 * ops.py:71-76). */
int ttb_scale(ttb_ctx* ctx, int64_t n, const double* x, double s, double* out);

/* N-ary block-diagonal sum  sum_p scales[p] * X_p  (ops.py:79-106, with
 * scale ops.py:71-76 fused: the scale multiplies core 0 only).
 * ranks: nterms rows of (ndim+1); cores: nterms rows of ndim pointers;
 * out[n] has shape (sum_p ranks[p][n] (1 at n=0), dims[n],
 * sum_p ranks[p][n+1] (1 at n=ndim-1)).  ndim == 1 sums elementwise. */
int ttb_add(ttb_ctx* ctx, int nterms, int ndim, const int64_t* dims, const int64_t* ranks,
            const double* const* cores, const double* scales, double* const* out);

/* Slice-wise Kronecker product (ops.py:109-132): out[n] has shape
 * (rx[n]*ry[n], dims[n], rx[n+1]*ry[n+1]), x's rank index slow. */
int ttb_hadamard(ttb_ctx* ctx, int ndim, const int64_t* dims, const int64_t* rx, const int64_t* ry,
                 const double* const* x, const double* const* y, double* const* out);

/* Seeded N(0,1) slabs, bitwise equal to the reference generator
 * (fill_random_slab core.py:256-266, slice_rng core.py:250-253, used by
 * random_tt core.py:269-282 and DistTTTensor.random parallel.py:88-102):
 * slab s is core core[s]'s block of global slices [lo[s], lo[s] + dl[s]),
 * shape (rl[s], dl[s], rr[s]) F-order, slice i drawn from
 * Generator(Philox(SeedSequence(seed, spawn_key=(core[s], i)))).standard_normal.
 * seed is the non-negative Python int as little-endian 32-bit words (0 -> one
 * word 0; numpy's uint32 coercion).  Synchronizes the context stream (the
 * rare ziggurat tail draws are finished with the host libm's log1p, as numpy
 * does). */
int ttb_fill_random(ttb_ctx* ctx, const uint32_t* seed, int nseed, int nslabs, const int64_t* core,
                    const int64_t* lo, const int64_t* rl, const int64_t* dl, const int64_t* rr,
                    double* const* out);

/* ---- Gram sweeps ------------------------------------------------------ */
/* <x, y> (ops.py:135-155): W_n = sum_i Y_n(i)^T W_{n-1} X_n(i), allreduced
 * per mode.  *result is written on the host. */
int ttb_inner(ttb_ctx* ctx, int ndim, const int64_t* dims, const int64_t* rx, const int64_t* ry,
              const double* const* x, const double* const* y, double* result);

/* ||x||^2 by the symmetric Gram route (norm(method="innerprod_sym"),
 * ops.py:179-205): per mode a rank-revealing pivoted Cholesky of the carry
 * W = (P L)(P L)^T, then W' = Z^T Z with Z = (P L)^T H(x_n), allreduced.
 * *indefinite = 1 when a carry fails the reconstruction check (ops.py:173-
 * 175); *result is then unspecified and the caller falls back to
 * ttb_inner, as ops.py:226-230 does. */
int ttb_norm_sym(ttb_ctx* ctx, int ndim, const int64_t* dims, const int64_t* ranks, const double* const* in,
                 double* result, int* indefinite);

/* _pivoted_cholesky (ops.py:162-176) of a device n x n SPSD matrix w
 * (n <= 64, lower triangle read): pl (device n x n) = P L in w's row order,
 * zero columns past the numeric rank (pivot <= 1e-14 max diag); perm (host,
 * n ints) = the pivots in order, then the remaining rows; *indefinite = 1
 * when ||pl pl^T - w||_F > 1e-6 ||w||_F. */
int ttb_pivoted_cholesky(ttb_ctx* ctx, int n, const double* w, double* pl, int* perm, int* rank, int* indefinite);

/* sum of squares of n doubles, allreduced (parallel.py:362-365, ops.py:232-234) */
int ttb_sumsq(ttb_ctx* ctx, int64_t n, const double* x, double* result);

/* ---- orthonormalization / rounding ------------------------------------ */
/* Alg. 3 sweep (parallel.py:164-209). direction 0 = left, 1 = right.
 * out[n] has the input shapes. */
int ttb_orthonormalize(ttb_ctx* ctx, int direction, int ndim, const int64_t* dims,
                       const int64_t* ranks, const double* const* in, double* const* out);

/* ||x||^2 by the orthonormalization route (norm(method="ortho"),
 * ops.py:208-235): a right-to-left sweep of TSQR R factors folded into the
 * next core, without forming the orthonormal cores; *result on the host. */
int ttb_norm_ortho(ttb_ctx* ctx, int ndim, const int64_t* dims, const int64_t* ranks, const double* const* in,
                   double* result);

/* round_tt (parallel.py:293-438) with RoundingOptions (parallel.py:261-284).
 * variant: 0 LRLI, 1 LRL, 2 RLRI, 3 RLR.  max_rank <= 0 means no cap.
 * out[n] sized by the input ranks; results packed at the front with shape
 * (out_ranks[n], dims[n], out_ranks[n+1]).  meta[0..3] = norm, eps_bond,
 * error_bound_violated (0/1), zero (0/1) -- the reference's meta dict. */
int ttb_round(ttb_ctx* ctx, int variant, double eps0, int64_t max_rank, int ndim,
              const int64_t* dims, const int64_t* ranks, const double* const* in,
              double* const* out, int64_t* out_ranks, double* meta);

/* Implicit Hadamard-then-round: round_tt(hadamard(x, w)) (ops.py:109-132
 * then parallel.py:293-438) WITHOUT materialising the Hadamard product --
 * the rank rx*rw Kronecker slices are formed on the fly where the rounding
 * reads its input (the first sweep's first TSQR panel and its R-folds; the
 * paper's suggestion, survey 8(f) row 4).  x[n] / w[n] are
 * this rank's slabs of the two factors; out[n] is sized by the PRODUCT
 * ranks rx[n]*rw[n] (the first sweep's folded cores live there), results
 * packed at the front as in ttb_round. */
int ttb_round_hadamard(ttb_ctx* ctx, int variant, double eps0, int64_t max_rank, int ndim,
                       const int64_t* dims, const int64_t* rx, const int64_t* rw, const double* const* x,
                       const double* const* w, double* const* out, int64_t* out_ranks, double* meta);

/* ttb_round on HOST-resident cores (the drop-in form of the reference's
 * numpy-level call): in[n] / out[n] are host pointers (out[n] sized by the
 * input ranks, results packed at the front as in ttb_round).  The upload of
 * core n overlaps the orthonormalization sweep up to core n, and each
 * output core is downloaded as soon as it is final.  Page-locked buffers
 * (cudaHostAlloc / torch pin_memory) are copied directly at full PCIe
 * bandwidth; pageable ones pass through the context's page-locked staging
 * ring (a worker thread, 32 MB chunks), never registered.  Returns when
 * out[] is filled. */
int ttb_round_host(ttb_ctx* ctx, int variant, double eps0, int64_t max_rank, int ndim,
                   const int64_t* dims, const int64_t* ranks, const double* const* in,
                   double* const* out, int64_t* out_ranks, double* meta);

/* ---- building blocks (the reference's lower-level public API) --------- */
/* TSQR of the panel view of one slab (rl, I, rr): trans 0 -> V(X) (rows
 * r_left*I, cols rr), trans 1 -> H(X)^T (rows I*rr, cols rl).  A plain
 * column-major m x b matrix is the slab (1, m, b) with trans 0.
 * Replaces tsqr_factor (tsqr.py:166-221); r_out (device, b x b col-major)
 * receives the replicated, sign-fixed R (tsqr.py:127-129). */
int ttb_tsqr_factor(ttb_ctx* ctx, int64_t rl, int64_t I, int64_t rr, int trans, const double* slab,
                    ttb_tsqr** out, double* r_out);
/* out = rows of Q @ [c; 0] on this rank (tsqr_apply_q, tsqr.py:248-327):
 * c is b x k (device, col-major), out is the slab (rl, I, k) for trans 0 or
 * (k, I, rr) for trans 1. */
int ttb_tsqr_apply(ttb_ctx* ctx, const ttb_tsqr* f, int64_t k, const double* c, double* out);
int ttb_tsqr_free(ttb_ctx* ctx, ttb_tsqr* f);

/* truncated_svd (parallel.py:224-258) of an m x n device matrix (col-major,
 * m, n <= 64): one-sided Jacobi on the device.  u (m x min), s (min),
 * v (n x min) are written for the first *keep columns. */
int ttb_truncated_svd(ttb_ctx* ctx, int64_t m, int64_t n, const double* a, double eps,
                      int64_t max_rank, double* u, double* s, double* v, int64_t* keep,
                      double* tail, int* capped);

/* ---- Kronecker-operator apply (ops.py:238-342) ----------------------- */
/* Mode-2 sparse product of one slab (mode2_multiply, core.py:285-297; the
 * local product of _apply_term_dist, ops.py:309-311), written into the
 * block (a0.., :, c0..) of an F-order output slab (out_rl, out_d, *):
 *   out(a0+a, i, c0+c) = sum_{jj = indptr[i]}^{indptr[i+1]-1} vals[jj] * src(a, cols[jj], c)
 * src(:, j, :) is local(:, j, :) for j < nloc (local: (rl, nloc, rr)
 * F-order) and halo slice j - nloc otherwise (halo: slice-major, each slice
 * an F-order rl x rr block -- the exchange payload layout, ops.py:284-287).
 * indptr (nrows+1), cols, vals are DEVICE arrays (CSR, int64 indices).
 * Accumulation is scipy's csr_matvecs sequence (bitwise). */
int ttb_mode2_spmm(ttb_ctx* ctx, int64_t rl, int64_t rr, int64_t nrows, const int64_t* indptr,
                   const int64_t* cols, const double* vals, int64_t nloc, const double* local,
                   const double* halo, double* out, int64_t out_rl, int64_t out_d, int64_t a0,
                   int64_t c0);
/* A whole core of the summed operator (the TT sum of apply_operator's
 * terms, ops.py:330-333) in one pass, every output cell written once:
 * mode 0 interior core (nterms rl, nrows, nterms rr) block diagonal, term t
 * in block (t, t); mode 1 first core (1, nrows, nterms rr), blocks side by
 * side; mode 2 last core (nterms rl, nrows, 1), stacked.  Term t uses the
 * CSR arrays indptr[t] / cols[t] / vals[t] and the halo buffer halo[t]
 * (device pointers, as ttb_mode2_spmm); nterms <= 16. */
int ttb_mode2_spmm_sum(ttb_ctx* ctx, int nterms, int mode, int64_t rl, int64_t rr, int64_t nrows,
                       const int64_t* const* indptr, const int64_t* const* cols, const double* const* vals,
                       int64_t nloc, const double* local, const double* const* halo, double* out);
/* out (slice-major, n slices of rl x rr F-order) = slab(:, idx[k], :) for
 * the F-order slab (rl, I, rr); idx is a DEVICE int64 array.  Packs the
 * payload of the operator exchange (ops.py:284-287). */
int ttb_gather_slices(ttb_ctx* ctx, int64_t rl, int64_t I, int64_t rr, const double* slab, int64_t n,
                      const int64_t* idx, double* out);
/* Pairwise exchange with npeers peers in one NCCL group (replaces the
 * round-robin comm.sendrecv rounds of ops.py:286-307): send[k] (send_n[k]
 * doubles) goes to peers[k], recv[k] (recv_n[k] doubles) comes from it.
 * Zero counts skip; both sides derive them from the replicated operator. */
int ttb_exchange(ttb_ctx* ctx, int npeers, const int* peers, const double* const* send,
                 const int64_t* send_n, double* const* recv, const int64_t* recv_n);

/* ---- TT files (TTPAR1: save_tt / load_tt, core.py:364-398) ------------- */
/* Read this rank's slice blocks [lo[n], hi[n]) of every core of a TTPAR1
 * file into F-order device slabs out[n] (ranks[n], hi-lo, ranks[n+1]);
 * data_offset = byte offset of core 0 (6 + 8 (2 ndim + 2)).  Staged through
 * page-locked double buffers (host pread overlapped with H2D).  A short
 * file raises TTB_ERR_SHAPE ("truncated"), as load_tt does.  Synchronous. */
int ttb_read_slabs(ttb_ctx* ctx, const char* path, int64_t data_offset, int ndim, const int64_t* dims,
                   const int64_t* ranks, const int64_t* lo, const int64_t* hi, double* const* out);
/* Write this rank's slabs into an existing TTPAR1 file whose header is
 * written and whose size is set (every rank writes only its own runs).
 * Synchronous. */
int ttb_write_slabs(ttb_ctx* ctx, const char* path, int64_t data_offset, int ndim, const int64_t* dims,
                    const int64_t* ranks, const int64_t* lo, const int64_t* hi, const double* const* in);

/* opt-in per-kernel-class timing with CUDA events (benchmark roofline);
 * dump writes "name launches total_ms\n" lines and clears the record. */
int ttb_prof_enable(int on);
int ttb_prof_dump(char* buf, long long cap);

/* measured fp64 throughput of this device (TFLOP/s): scalar DFMA and
 * warp-level DMMA (mma.sync m8n8k4 f64).  Roofline denominators. */
int ttb_fp64_peak(void* stream, double* dfma_tflops, double* dmma_tflops);

#ifdef __cplusplus
}
#endif

#endif /* TTB_H_ */
