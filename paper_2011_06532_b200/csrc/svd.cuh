#pragma once
#include "ctx.cuh"
namespace ttb {
// one-sided Jacobi truncated SVD, see svd.cu
void jacobi_svd(Ctx& ctx, const double* A, int lda, int m, int n, bool transA, double eps, int max_rank,
                double* C, double* Vk, double* s, int* info, double* dinfo);
void svd_normalize_u(Ctx& ctx, const double* C, const double* s, int m, int keep, double* U);
}  // namespace ttb
