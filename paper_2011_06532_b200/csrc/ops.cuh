// Internal kernel entry points shared by the drivers (driver.cu).
#pragma once
#include "ctx.cuh"

namespace ttb {

// elementwise.cu
struct AddTerm {
  const double* x;
  int64_t rl, rr;     // term core shape (rl, I, rr)
  int64_t offa, offc; // block offsets in the output core
  double s;           // scale (applied on core 0 only)
};
constexpr int kMaxAddTerms = 16;
void add_core(Ctx& ctx, int mode, int nterms, const AddTerm* terms, int64_t RL, int64_t I, int64_t RR, double* out);
void hadamard_core(Ctx& ctx, const double* x, int64_t ral, int64_t rar, const double* y, int64_t rbl, int64_t rbr,
                   int64_t I, double* out);
void scale_vec(Ctx& ctx, int64_t n, const double* x, double s, double* out);
// deterministic sum of squares -> *dres (device scalar)
void sumsq_dev(Ctx& ctx, int64_t n, const double* x, double* dres);
void fill_zero(Ctx& ctx, double* p, int64_t n);

// gram.cu: Wn (rbr x rar) = sum_i Y(i)^T W X(i); W (rbl x ral) device
void gram_step(Ctx& ctx, const double* W, const double* X, int64_t ral, int64_t rar, const double* Y, int64_t rbl,
               int64_t rbr, int64_t I, double* Wn, int* ticket = nullptr);
void pivoted_cholesky(Ctx& ctx, const double* W, int n, double* PL, double* Wrec, int* perm, int* rank);
bool sym16_fusable(int64_t ral, int64_t rar, int64_t I, const double* X);
void gram_sym_step(Ctx& ctx, double* PL, int* perm, double* Wrec, const double* X, int64_t ral, int64_t rar,
                   int64_t I, double* Wn, int* ticket);

// gemm.cu: skinny products on unfoldings
// out_H (M x N) = F (M x K) * H (K x N); col-major, ldH = K, ldOut = M, F ld = ldf (F^T if transF)
// upper: F is upper triangular (the R-fold, dtrmm) -- zero blocks are skipped
// kz (optional): H is H(Z) of an implicit Hadamard core with kI slices (H unused)
void gemm_small_left(Ctx& ctx, int M, int K, int64_t N, const double* F, int ldf, bool transF, const double* H,
                     double* out, bool upper = false, const Kron* kz = nullptr, int64_t kI = 0);
// out_V (Mb x Nn) = V (Mb x K) * G (K x Nn); col-major, ldV = Mb, ldOut = Mb, G ld = ldg (G^T if transG)
// upper: the effective small operand S(c, k) = G(k, c) is upper triangular (V R^T: transG, G = R)
// kz (optional): V is V(Z) of an implicit Hadamard core with kI slices (V unused)
void gemm_small_right(Ctx& ctx, int64_t Mb, int K, int Nn, const double* V, const double* G, int ldg, bool transG,
                      double* out, bool upper = false, const Kron* kz = nullptr, int64_t kI = 0);

}  // namespace ttb
