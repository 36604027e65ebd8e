// Warp-level fp64 tile GEMM on mma.sync.m8n8k4.f64 (the fp64 tensor path of
// sm_100a; tcgen05 has no f64 kind).  Operands are accessed through
// functors so shared-memory layouts, transposes and zero padding stay at the
// call site.  Fragment layouts (PTX ISA, m8n8k4 .row.col f64):
//   A (8x4, row): lane l holds A[l/4][l%4]
//   B (4x8, col): lane l holds B[l%4][l/4]
//   D (8x8):      lane l holds D[l/4][2*(l%4)] and D[l/4][2*(l%4)+1]
#pragma once

namespace ttb {

__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// D (16x8) += A (16x8) B (8x8), mma.sync m16n8k8 f64 (4x the work of m8n8k4
// per instruction).  Fragments (g = lane / 4, t = lane % 4):
//   A: a0 = A[g][t], a1 = A[g+8][t], a2 = A[g][t+4], a3 = A[g+8][t+4]
//   B: b0 = B[t][g], b1 = B[t+4][g]
//   D: d0 = D[g][2t], d1 = D[g][2t+1], d2 = D[g+8][2t], d3 = D[g+8][2t+1]
__device__ __forceinline__ void dmma_1688(double (&d)[4], double a0, double a1, double a2, double a3, double b0,
                                          double b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
}

// C(m, n) = sum_{k < K} A(m, k) B(k, n) for m < M, n < N, split in 16x16
// blocks (2x2 MMA tiles, operand fragments reused twice) over the warps of
// the CTA.  a(m, k), b(k, n) must return 0 outside [0, M) x [0, K) etc.
// store(m, n, value) is called for m < M, n < N only.  Collective over the
// CTA's warps (no barrier inside).
template <class AF, class BF, class SF>
__device__ __forceinline__ void cta_dmma(int M, int N, int K, int nwarps, AF a, BF b, SF store) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int fr = lane >> 2, fc = lane & 3;
  const int mt = (M + 15) / 16, nt = (N + 15) / 16;
  for (int blk = warp; blk < mt * nt; blk += nwarps) {
    const int m0 = (blk % mt) * 16, n0 = (blk / mt) * 16;
    double acc[2][2][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll 4
    for (int k0 = 0; k0 < K; k0 += 4) {
      const double a0 = a(m0 + fr, k0 + fc), a1 = a(m0 + 8 + fr, k0 + fc);
      const double b0 = b(k0 + fc, n0 + fr), b1 = b(k0 + fc, n0 + 8 + fr);
      dmma_884(acc[0][0][0], acc[0][0][1], a0, b0);
      dmma_884(acc[0][1][0], acc[0][1][1], a0, b1);
      dmma_884(acc[1][0][0], acc[1][0][1], a1, b0);
      dmma_884(acc[1][1][0], acc[1][1][1], a1, b1);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int m = m0 + 8 * i + fr, n = n0 + 8 * j + 2 * fc + h;
          if (m < M && n < N) store(m, n, acc[i][j][h]);
        }
  }
}

}  // namespace ttb
