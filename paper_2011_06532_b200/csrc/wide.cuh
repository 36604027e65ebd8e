// The general path for bond ranks above 64 (wide.cu).
#pragma once
#include "ctx.cuh"

namespace ttb {

// C(m, n) = alpha sum_k A(m, k) B(k, n) + beta C(m, n) on strided operands:
// A(m, k) = A[m sam + k sak], B(k, n) = B[k sbk + n sbn], C(m, n) = C[m scm + n scn]
void dgemm_strided(Ctx& ctx, int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t sam, int64_t sak,
                   const double* B, int64_t sbk, int64_t sbn, double beta, double* C, int64_t scm, int64_t scn);
// W (na x nb, ld na) = A^T B over `rows` rows (deterministic split reduction; allreduce: summed over ranks)
void tall_gram(Ctx& ctx, int64_t rows, int na, int nb, const double* A, int64_t sar, int64_t sac, const double* B,
               int64_t sbr, int64_t sbc, double* W, bool allreduce);
// true when the register-tile TSQR cannot take the panel (more than 64 columns, or slices taller than a tile)
bool tsqr_needs_wide(const Panel& panel);
void wide_tsqr_factor(Ctx& ctx, const Panel& panel, Tsqr& f);
void wide_tsqr_apply(Ctx& ctx, const Tsqr& f, const double* z, int k, const Panel& out);
void gram_step_wide(Ctx& ctx, const double* W, const double* X, int64_t ral, int64_t rar, const double* Y,
                    int64_t rbl, int64_t rbr, int64_t I, double* Wn);
void jacobi_svd_wide(Ctx& ctx, const double* A, int lda, int m, int n, bool transA, double eps, int max_rank,
                     double* C, double* Vk, double* s, int* info, double* dinfo);

}  // namespace ttb
