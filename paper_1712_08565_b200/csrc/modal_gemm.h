// Modal GEMM interface (see modal_gemm.cu).
#pragma once
#include "common.cuh"

namespace mfwq {

// element (k, j) of a mode view sits at k*sk + (j/jdiv)*jhi + (j%jdiv)*jlo
struct ModeView {
  long long sk;
  long long jdiv, jhi, jlo;
};

// epilogue scale 1/(lam1[j % n1] + lam2[j / n1] + lam3[m] + sigma); lam1 == nullptr: none
struct Scale {
  const double* lam1;
  const double* lam2;
  const double* lam3;
  long long n1;
  double sigma;
};

// C(m, j) = sum_k A[m][k] X(k, j), A row-major M x K with even pitch lda >= K (zero padded);
// kcontig: X/C contiguous along k/m
void modal_gemm(const double* A, int lda, int M, int K, const double* X, ModeView xv, double* C, ModeView cv,
                long long N, Scale sc, bool kcontig, cudaStream_t s);

}  // namespace mfwq
