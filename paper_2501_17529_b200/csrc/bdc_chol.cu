// bdc_chol.cu -- GPU base-PTDF setup: the one SPD solve of
// compute_ptdf (factors.py:161-216), P[:, keep] = (L_kk^-1 A^T)^T with L_kk the
// slack-reduced susceptance Laplacian and A the weighted incidence of the retained
// rows -- the reference's scipy.linalg.solve(..., assume_a="pos"), i.e. LAPACK
// potrf + potrs, restated as blocked FP64 kernels:
//   potrf  for each 64-column panel: the diagonal block in shared memory (k_potrf_diag),
//          the panel below it (k_trsm_panel, X L11^T = A21), the trailing lower
//          triangle (k_gemm<false, true, true>: A22 -= L21 L21^T, lower tiles only);
//   potrs  forward (C Y = B: k_trsm_left<false> + k_gemm<false, false>) and backward
//          (C^T X = Y: k_trsm_left<true> + k_gemm<true, false>) over the n x m RHS.
// Row-major, leading dimension ld.  The GEMM tile is 64 x 64 x 16 with a 4 x 4 FP64
// register tile per thread (256 threads): CUDA-core DFMA, the B200's FP64 rate (its
// FP64 tensor path has the same peak).
#include "bdc_device.cuh"

#include <algorithm>

namespace bdc {

namespace {

constexpr int CB = 64;  // panel / tile size

// Cholesky of the diagonal block A[k0:k0+nb, k0:k0+nb] (lower, in place), one CTA.
// info = first failing global column + 1 when the block is not positive definite.
__global__ void k_potrf_diag(double* A, int ld, int k0, int nb, int* info) {
  __shared__ double a[CB][CB + 1];
  const int tid = threadIdx.x;
  for (int e = tid; e < nb * nb; e += blockDim.x) {
    const int i = e / nb, j = e % nb;
    a[i][j] = j <= i ? A[(size_t)(k0 + i) * ld + k0 + j] : 0.0;
  }
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    if (tid == 0) {
      const double d = a[j][j];
      if (!(d > 0.0)) {
        if (*info == 0) *info = k0 + j + 1;
        a[j][j] = 1.0;
      } else {
        a[j][j] = sqrt(d);
      }
    }
    __syncthreads();
    const double djj = a[j][j];
    for (int i = j + 1 + tid; i < nb; i += blockDim.x) a[i][j] /= djj;
    __syncthreads();
    // rank-1 update of the remaining lower triangle of the block
    const int m = nb - j - 1;
    for (int e = tid; e < m * m; e += blockDim.x) {
      const int i = j + 1 + e / m, l = j + 1 + e % m;
      if (l <= i) a[i][l] = fma(-a[i][j], a[l][j], a[i][l]);
    }
    __syncthreads();
  }
  for (int e = tid; e < nb * nb; e += blockDim.x) {
    const int i = e / nb, j = e % nb;
    if (j <= i) A[(size_t)(k0 + i) * ld + k0 + j] = a[i][j];
  }
}

// Panel below the diagonal block: rows r0.. of columns [k0, k0+nb) solve X L11^T = A21
// (forward substitution along each row); a thread per row, L11 in shared memory.
__global__ void k_trsm_panel(double* A, int ld, int k0, int nb, int r0, int n) {
  __shared__ double L[CB][CB + 1];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int i = e / nb, j = e % nb;
    L[i][j] = j <= i ? A[(size_t)(k0 + i) * ld + k0 + j] : 0.0;
  }
  __syncthreads();
  const int r = r0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double x[CB];
  double* row = A + (size_t)r * ld + k0;
  for (int j = 0; j < nb; ++j) {
    double v = row[j];
    for (int l = 0; l < j; ++l) v = fma(-x[l], L[j][l], v);
    x[j] = v / L[j][j];
  }
  for (int j = 0; j < nb; ++j) row[j] = x[j];
}

// Triangular solve of the RHS block rows [k0, k0+nb) against the diagonal block:
// TRANS = false: C11 Y = B (forward), TRANS = true: C11^T X = Y (backward); a thread per
// RHS column.
template <bool TRANS>
__global__ void k_trsm_left(const double* A, int lda, double* B, int ldb, int k0, int nb, int m) {
  __shared__ double L[CB][CB + 1];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int i = e / nb, j = e % nb;
    L[i][j] = j <= i ? A[(size_t)(k0 + i) * lda + k0 + j] : 0.0;
  }
  __syncthreads();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= m) return;
  double x[CB];
  for (int i = 0; i < nb; ++i) x[i] = B[(size_t)(k0 + i) * ldb + c];
  if (!TRANS) {
    for (int i = 0; i < nb; ++i) {
      double v = x[i];
      for (int l = 0; l < i; ++l) v = fma(-L[i][l], x[l], v);
      x[i] = v / L[i][i];
    }
  } else {
    for (int i = nb - 1; i >= 0; --i) {
      double v = x[i];
      for (int l = i + 1; l < nb; ++l) v = fma(-L[l][i], x[l], v);
      x[i] = v / L[i][i];
    }
  }
  for (int i = 0; i < nb; ++i) B[(size_t)(k0 + i) * ldb + c] = x[i];
}

// C[M x N] -= op(A)[M x K] op(B)[K x N]; op(A)(i, l) = TA ? A[l][i] : A[i][l],
// op(B)(l, j) = TB ? B[j][l] : B[l][j].  LOWER: only tiles on or below the diagonal
// (and only elements j <= i inside diagonal tiles) -- the SYRK of the Cholesky update.
template <bool TA, bool TB, bool LOWER>
__global__ void __launch_bounds__(256) k_gemm(double* C, int ldc, const double* A, int lda, const double* B,
                                              int ldb, int M, int N, int K) {
  constexpr int KT = 16;
  __shared__ double sA[KT][CB + 1];  // sA[l][i]
  __shared__ double sB[KT][CB + 1];  // sB[l][j]
  const int bi = blockIdx.y, bj = blockIdx.x;
  if (LOWER && bj > bi) return;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int i0 = bi * CB, j0 = bj * CB;
  double acc[4][4] = {};
  for (int l0 = 0; l0 < K; l0 += KT) {
    // coalesced tile loads: consecutive threads walk the contiguous index of each operand
    for (int e = tid; e < KT * CB; e += 256) {
      const int l = TA ? e / CB : e % KT, i = TA ? e % CB : e / KT;
      const int gi = i0 + i, gl = l0 + l;
      double va = 0.0;
      if (gi < M && gl < K) va = TA ? A[(size_t)gl * lda + gi] : A[(size_t)gi * lda + gl];
      sA[l][i] = va;
    }
    for (int e = tid; e < KT * CB; e += 256) {
      const int l = TB ? e % KT : e / CB, j = TB ? e / KT : e % CB;
      const int gj = j0 + j, gl = l0 + l;
      double vb = 0.0;
      if (gj < N && gl < K) vb = TB ? B[(size_t)gj * ldb + gl] : B[(size_t)gl * ldb + gj];
      sB[l][j] = vb;
    }
    __syncthreads();
#pragma unroll
    for (int l = 0; l < KT; ++l) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = sA[l][ty + 16 * u];
        b[u] = sB[l][tx + 16 * u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int gi = i0 + ty + 16 * u, gj = j0 + tx + 16 * v;
      if (gi < M && gj < N && (!LOWER || gj <= gi)) C[(size_t)gi * ldc + gj] -= acc[u][v];
    }
}

}  // namespace

cudaError_t launch_spd_solve(double* A, int n, double* B, int m, int* info, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(info, 0, sizeof(int), s);
  if (e != cudaSuccess) return e;
  // potrf (lower)
  for (int k0 = 0; k0 < n; k0 += CB) {
    const int nb = std::min(CB, n - k0), k1 = k0 + nb, rest = n - k1;
    k_potrf_diag<<<1, 256, 0, s>>>(A, n, k0, nb, info);
    if (rest > 0) {
      k_trsm_panel<<<(rest + 63) / 64, 64, 0, s>>>(A, n, k0, nb, k1, n);
      const int tiles = (rest + CB - 1) / CB;
      double* A22 = A + (size_t)k1 * n + k1;
      const double* P = A + (size_t)k1 * n + k0;
      k_gemm<false, true, true><<<dim3(tiles, tiles), 256, 0, s>>>(A22, n, P, n, P, n, rest, rest, nb);
    }
  }
  // potrs: forward C Y = B, backward C^T X = Y (B is n x m, overwritten by X)
  for (int k0 = 0; k0 < n; k0 += CB) {
    const int nb = std::min(CB, n - k0), k1 = k0 + nb, rest = n - k1;
    k_trsm_left<false><<<(m + 63) / 64, 64, 0, s>>>(A, n, B, m, k0, nb, m);
    if (rest > 0)
      k_gemm<false, false, false><<<dim3((m + CB - 1) / CB, (rest + CB - 1) / CB), 256, 0, s>>>(
          B + (size_t)k1 * m, m, A + (size_t)k1 * n + k0, n, B + (size_t)k0 * m, m, rest, m, nb);
  }
  for (int k0 = ((n - 1) / CB) * CB; k0 >= 0; k0 -= CB) {
    const int nb = std::min(CB, n - k0);
    k_trsm_left<true><<<(m + 63) / 64, 64, 0, s>>>(A, n, B, m, k0, nb, m);
    if (k0 > 0)
      // Y[0:k0] -= C[k0:k1, 0:k0]^T X[k0:k1]
      k_gemm<true, false, false><<<dim3((m + CB - 1) / CB, (k0 + CB - 1) / CB), 256, 0, s>>>(
          B, m, A + (size_t)k0 * n, n, B + (size_t)k0 * m, m, k0, m, nb);
  }
  return cudaGetLastError();
}

}  // namespace bdc
