// ptap_gen.cu -- device generators of the BASELINE.json inputs.
//
// Bit-identical to the host generators in paper_1905_08423_b200/problems.py
// (same ascending-column entry order, same counter-based edge hash, same
// left-to-right diagonal fold), so the CPU oracle and the GPU consume the
// same CSR; tests/test_gpu_parity.py checks the equality on the device.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/ptap_b200.h"
#include "ptap_kernels.cuh"

namespace {

__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
  unsigned long long z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double edge_uniform(long long i, long long j, unsigned long long nglobal,
                                               unsigned long long seed) {
  unsigned long long lo = (unsigned long long)(i < j ? i : j), hi = (unsigned long long)(i < j ? j : i);
  unsigned long long key = lo * nglobal + hi + seed * 0x94D049BB133111EBull;
  unsigned long long bits = splitmix64(key) >> 11;
  return __dmul_rn((double)bits, 1.1102230246251565e-16);  // 2^-53
}

__device__ __forceinline__ int dim_count(long long x, long long n) { return 1 + (x > 0) + (x < n - 1); }

__global__ void k_stencil_count(int points, long long n, long long lo, long long hi, int64_t *cnt) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= hi - lo) return;
  long long i = lo + r;
  long long x = i % n, y = (i / n) % n, z = i / (n * n);
  int cx = dim_count(x, n), cy = dim_count(y, n), cz = dim_count(z, n);
  cnt[r] = points == 27 ? (int64_t)cx * cy * cz : (int64_t)(1 + (cx - 1) + (cy - 1) + (cz - 1));
}

// kind 0: 7-pt Poisson (6 / -1); kind 1: config-3 random 27-pt
__global__ void k_stencil_fill(int points, int kind, unsigned long long seed, long long n, long long lo, long long hi,
                               const int64_t *rp, int32_t *col, double *val) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= hi - lo) return;
  long long i = lo + r;
  long long x = i % n, y = (i / n) % n, z = i / (n * n);
  unsigned long long N = (unsigned long long)(n * n * n);
  int64_t e = rp[r];
  int64_t diag_pos = -1;
  double acc = 0.0;
  if (points == 7) {
    const int off[7][3] = {{0, 0, -1}, {0, -1, 0}, {-1, 0, 0}, {0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
    for (int q = 0; q < 7; ++q) {
      long long jx = x + off[q][0], jy = y + off[q][1], jz = z + off[q][2];
      if (jx < 0 || jx >= n || jy < 0 || jy >= n || jz < 0 || jz >= n) continue;
      col[e] = (int32_t)(jx + n * (jy + n * jz));
      val[e] = q == 3 ? 6.0 : -1.0;
      ++e;
    }
    return;
  }
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        long long jx = x + dx, jy = y + dy, jz = z + dz;
        if (jx < 0 || jx >= n || jy < 0 || jy >= n || jz < 0 || jz >= n) continue;
        long long j = jx + n * (jy + n * jz);
        col[e] = (int32_t)j;
        if (dx == 0 && dy == 0 && dz == 0) {
          diag_pos = e;
          val[e] = 0.0;
          acc = __dadd_rn(acc, 0.0);
        } else {
          double v = kind == 1 ? -__dadd_rn(0.5, edge_uniform(i, j, N, seed)) : -1.0;
          val[e] = v;
          acc = __dadd_rn(acc, fabs(v));
        }
        ++e;
      }
  if (diag_pos >= 0) val[diag_pos] = kind == 1 ? __dadd_rn(acc, 1e-2) : acc;
}

__device__ __forceinline__ int tri_count(long long f, long long nc) {
  long long b = f / 2;
  if ((f & 1) == 0) return 1;
  return b + 1 < nc ? 2 : 1;
}

__global__ void k_trilinear_count(long long nc, long long lo, long long hi, int64_t *cnt) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= hi - lo) return;
  long long nf = 2 * nc, i = lo + r;
  long long x = i % nf, y = (i / nf) % nf, z = i / (nf * nf);
  cnt[r] = (int64_t)tri_count(x, nc) * tri_count(y, nc) * tri_count(z, nc);
}

__global__ void k_trilinear_fill(long long nc, long long lo, long long hi, const int64_t *rp, int32_t *col,
                                 double *val) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= hi - lo) return;
  long long nf = 2 * nc, i = lo + r;
  long long f[3] = {i % nf, (i / nf) % nf, i / (nf * nf)};
  long long c[3][2];
  double w[3][2];
  int cn[3];
  for (int d = 0; d < 3; ++d) {
    long long b = f[d] / 2;
    if ((f[d] & 1) == 0) { cn[d] = 1; c[d][0] = b; w[d][0] = 1.0; }
    else {
      cn[d] = 1; c[d][0] = b; w[d][0] = 0.5;
      if (b + 1 < nc) { cn[d] = 2; c[d][1] = b + 1; w[d][1] = 0.5; }
    }
  }
  int64_t e = rp[r];
  for (int kz = 0; kz < cn[2]; ++kz)
    for (int ky = 0; ky < cn[1]; ++ky)
      for (int kx = 0; kx < cn[0]; ++kx) {
        col[e] = (int32_t)(c[0][kx] + nc * (c[1][ky] + nc * c[2][kz]));
        val[e] = __dmul_rn(__dmul_rn(w[0][kx], w[1][ky]), w[2][kz]);
        ++e;
      }
}

thread_local std::string g_gen_err;

ptap_status finish_rowptr(int64_t *cnt_then_rp, int64_t nrows, int64_t *nnz_out, cudaStream_t st) {
  // in-place: cnt lives in rp[1..nrows]; scan into a temporary
  int64_t *scratch = nullptr, *tmp = nullptr;
  if (cudaMallocAsync(&scratch, sizeof(int64_t) * ptapdev::scan_scratch_elems(nrows), st) != cudaSuccess ||
      cudaMallocAsync(&tmp, sizeof(int64_t) * (nrows + 1), st) != cudaSuccess)
    return PTAP_ERR_OOM;
  ptapdev::scan_exclusive(cnt_then_rp + 1, tmp, nrows, scratch, st);
  cudaMemcpyAsync(cnt_then_rp, tmp, sizeof(int64_t) * (nrows + 1), cudaMemcpyDeviceToDevice, st);
  cudaMemcpyAsync(nnz_out, tmp + nrows, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(scratch, st);
  cudaFreeAsync(tmp, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return PTAP_ERR_CUDA;
  return PTAP_OK;
}

inline int nb(long long n) { return (int)((n + 255) / 256 > 0 ? (n + 255) / 256 : 1); }

}  // namespace

extern "C" {

ptap_status ptap_gen_stencil_rowptr(int points, int64_t n, int64_t row_lo, int64_t row_hi, int64_t *row_ptr,
                                    int64_t *nnz_out, void *stream) {
  if (points != 7 && points != 27) return PTAP_ERR_VALUE;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t nr = row_hi - row_lo;
  if (nr > 0) k_stencil_count<<<nb(nr), 256, 0, st>>>(points, n, row_lo, row_hi, row_ptr + 1);
  if (cudaGetLastError() != cudaSuccess) return PTAP_ERR_CUDA;
  return finish_rowptr(row_ptr, nr, nnz_out, st);
}

ptap_status ptap_gen_stencil_fill(int points, int kind, uint64_t seed, int64_t n, int64_t row_lo, int64_t row_hi,
                                  const int64_t *row_ptr, int32_t *col, double *val, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  int64_t nr = row_hi - row_lo;
  if (nr > 0) k_stencil_fill<<<nb(nr), 256, 0, st>>>(points, kind, seed, n, row_lo, row_hi, row_ptr, col, val);
  return cudaGetLastError() == cudaSuccess ? PTAP_OK : PTAP_ERR_CUDA;
}

ptap_status ptap_gen_trilinear_rowptr(int64_t nc, int64_t row_lo, int64_t row_hi, int64_t *row_ptr, int64_t *nnz_out,
                                      void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  int64_t nr = row_hi - row_lo;
  if (nr > 0) k_trilinear_count<<<nb(nr), 256, 0, st>>>(nc, row_lo, row_hi, row_ptr + 1);
  if (cudaGetLastError() != cudaSuccess) return PTAP_ERR_CUDA;
  return finish_rowptr(row_ptr, nr, nnz_out, st);
}

ptap_status ptap_gen_trilinear_fill(int64_t nc, int64_t row_lo, int64_t row_hi, const int64_t *row_ptr, int32_t *col,
                                    double *val, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  int64_t nr = row_hi - row_lo;
  if (nr > 0) k_trilinear_fill<<<nb(nr), 256, 0, st>>>(nc, row_lo, row_hi, row_ptr, col, val);
  return cudaGetLastError() == cudaSuccess ? PTAP_OK : PTAP_ERR_CUDA;
}

}  // extern "C"
