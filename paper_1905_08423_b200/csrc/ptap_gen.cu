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


// ---------------------------------------------------------------------------
// config 4: block transport (problems_amg.block_transport).  Row = node * ncomp
// + component; a node's entries in ascending column order are its z-, y-, x-
// neighbours (same component), its own dense block, then x+, y+, z+.
// ---------------------------------------------------------------------------
struct BtNode {
  long long node, x, y, z;
  int c;
  long long nbr[6];  // z-, y-, x-, x+, y+, z+ node ids, -1 outside the grid
};
__device__ __forceinline__ BtNode bt_node(long long i, long long nn, int ncomp) {
  BtNode b;
  b.node = i / ncomp;
  b.c = (int)(i - b.node * ncomp);
  b.x = b.node % nn;
  b.y = (b.node / nn) % nn;
  b.z = b.node / (nn * nn);
  b.nbr[0] = b.z > 0 ? b.node - nn * nn : -1;
  b.nbr[1] = b.y > 0 ? b.node - nn : -1;
  b.nbr[2] = b.x > 0 ? b.node - 1 : -1;
  b.nbr[3] = b.x < nn - 1 ? b.node + 1 : -1;
  b.nbr[4] = b.y < nn - 1 ? b.node + nn : -1;
  b.nbr[5] = b.z < nn - 1 ? b.node + nn * nn : -1;
  return b;
}
__device__ __forceinline__ long long bt_agg(long long node, long long nn, long long ag, long long na) {
  const long long x = node % nn, y = (node / nn) % nn, z = node / (nn * nn);
  return (x / ag) + na * ((y / ag) + na * (z / ag));
}

__global__ void k_bt_count(long long nn, int ncomp, long long ag, long long lo, long long hi, int64_t *cnt_a,
                           int64_t *cnt_p) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= hi - lo) return;
  const BtNode b = bt_node(lo + r, nn, ncomp);
  const long long na = (nn + ag - 1) / ag, mine = bt_agg(b.node, nn, ag, na);
  int ca = ncomp, cp = ncomp;
  for (int q = 0; q < 6; ++q)
    if (b.nbr[q] >= 0) {
      ++ca;
      if (bt_agg(b.nbr[q], nn, ag, na) != mine) ++cp;
    }
  cnt_a[r] = ca;
  if (cnt_p) cnt_p[r] = cp;
}

__global__ void k_bt_fill_a(long long nn, int ncomp, unsigned long long seed, long long lo, long long hi,
                            const int64_t *rp, int32_t *col, double *val) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= hi - lo) return;
  const long long i = lo + r;
  const BtNode b = bt_node(i, nn, ncomp);
  const unsigned long long N = (unsigned long long)(nn * nn * nn) * (unsigned long long)ncomp;
  int64_t e = rp[r], diag_pos = -1;
  double acc = 0.0;
  auto spatial = [&](int q) {
    if (b.nbr[q] < 0) return;
    const long long j = b.nbr[q] * ncomp + b.c;
    const double v = -__dadd_rn(0.5, edge_uniform(i, j, N, seed));
    col[e] = (int32_t)j;
    val[e] = v;
    acc = __dadd_rn(acc, fabs(v));
    ++e;
  };
  spatial(0); spatial(1); spatial(2);
  for (int c2 = 0; c2 < ncomp; ++c2) {
    const long long j = b.node * ncomp + c2;
    col[e] = (int32_t)j;
    if (c2 == b.c) {
      diag_pos = e;
    } else {
      const double v = __dadd_rn(-0.1, __dmul_rn(0.2, edge_uniform(i, j, N, seed)));
      val[e] = v;
      acc = __dadd_rn(acc, fabs(v));
    }
    ++e;
  }
  spatial(3); spatial(4); spatial(5);
  val[diag_pos] = __dadd_rn(acc, 1e-2);
}

// w = D^-1 A v (power iteration for lambda_max; rows [0, n) with global columns)
__global__ void k_spmv_dinv(long long n, const int64_t *rp, const int32_t *col, const double *val, const double *v,
                            double *w) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0, d = 1.0;
  for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
    if (col[e] == i) d = val[e];
    s += val[e] * v[col[e]];
  }
  w[i] = s / d;
}

// P = P_tent - omega D^-1 A P_tent, structural pattern, scipy's operation order
// (da = dinv * a; sums of da in ascending column order from 0; omega * sum;
// 1 - that on the tentative entry, its negation elsewhere)
__global__ void k_bt_fill_p(long long nn, int ncomp, long long ag, double omega, long long lo, long long hi,
                            const int64_t *a_rp, const double *a_val, const int64_t *p_rp, int32_t *p_col,
                            double *p_val) {
  long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= hi - lo) return;
  const long long i = lo + r;
  const BtNode b = bt_node(i, nn, ncomp);
  const long long na = (nn + ag - 1) / ag, mine = bt_agg(b.node, nn, ag, na);
  // A's row: [z- y- x-] block [x+ y+ z+]; find the diagonal first
  int nlow = 0;
  for (int q = 0; q < 3; ++q) nlow += b.nbr[q] >= 0;
  const int64_t a0 = a_rp[r];
  const double dinv = __ddiv_rn(1.0, a_val[a0 + nlow + b.c]);
  int64_t e = p_rp[r], ea = a0;
  double own = 0.0;  // sum over the same-component entries inside the own aggregate, ascending column
  for (int q = 0; q < 3; ++q)
    if (b.nbr[q] >= 0) {
      const double da = __dmul_rn(dinv, a_val[ea++]);
      const long long g = bt_agg(b.nbr[q], nn, ag, na);
      if (g == mine) {
        own = __dadd_rn(own, da);
      } else {
        p_col[e] = (int32_t)(g * ncomp + b.c);
        p_val[e] = -__dmul_rn(omega, da);
        ++e;
      }
    }
  const int64_t eblock = e;
  for (int c2 = 0; c2 < ncomp; ++c2) {
    const double da = __dmul_rn(dinv, a_val[ea++]);
    p_col[e] = (int32_t)(mine * ncomp + c2);
    if (c2 == b.c) own = __dadd_rn(own, da);
    else p_val[e] = -__dmul_rn(omega, da);
    ++e;
  }
  for (int q = 3; q < 6; ++q)
    if (b.nbr[q] >= 0) {
      const double da = __dmul_rn(dinv, a_val[ea++]);
      const long long g = bt_agg(b.nbr[q], nn, ag, na);
      if (g == mine) {
        own = __dadd_rn(own, da);
      } else {
        p_col[e] = (int32_t)(g * ncomp + b.c);
        p_val[e] = -__dmul_rn(omega, da);
        ++e;
      }
    }
  p_val[eblock + b.c] = __dsub_rn(1.0, __dmul_rn(omega, own));
}


// ---------------------------------------------------------------------------
// config 5: k nearest neighbours of points in the unit cube (the directed
// edges of problems_amg.knn_laplacian's graph; scipy's cKDTree there).  The
// points are sorted by cell of a G^3 grid (the caller sorts them); a thread
// scans the cube of cells around its point, growing it until the K-th
// distance is no larger than the distance to the cube's nearest inner face.
// Squared distances fold x, y, z in order with individually rounded
// operations (the same values whichever endpoint computes them).
// ---------------------------------------------------------------------------
constexpr int KNN_MAX = 32;

__global__ void __launch_bounds__(128) k_knn_cells(long long n, const double *__restrict__ pts,
                                                   const long long *__restrict__ cell_start, int G, int K,
                                                   int32_t *__restrict__ out_idx, double *__restrict__ out_d2) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const double px = pts[3 * t], py = pts[3 * t + 1], pz = pts[3 * t + 2];
  const double h = 1.0 / (double)G;
  const int cx = min(G - 1, (int)(px * G)), cy = min(G - 1, (int)(py * G)), cz = min(G - 1, (int)(pz * G));
  double bd[KNN_MAX];
  int32_t bi[KNN_MAX];
  for (int R = 1;; ++R) {
    int cnt = 0;
    const int x0 = max(0, cx - R), x1 = min(G - 1, cx + R), y0 = max(0, cy - R), y1 = min(G - 1, cy + R);
    const int z0 = max(0, cz - R), z1 = min(G - 1, cz + R);
    for (int z = z0; z <= z1; ++z)
      for (int y = y0; y <= y1; ++y) {
        const long long c0 = ((long long)z * G + y) * G + x0, c1 = ((long long)z * G + y) * G + x1;
        const long long q0 = cell_start[c0], q1 = cell_start[c1 + 1];  // the x-run of cells is contiguous
        for (long long q = q0; q < q1; ++q) {
          if (q == t) continue;
          const double dx = __dsub_rn(px, pts[3 * q]), dy = __dsub_rn(py, pts[3 * q + 1]);
          const double dz = __dsub_rn(pz, pts[3 * q + 2]);
          const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
          if (cnt == K && d2 >= bd[K - 1]) continue;
          int pos = cnt < K ? cnt : K - 1;  // insertion into the ascending list
          while (pos > 0 && bd[pos - 1] > d2) {
            bd[pos] = bd[pos - 1];
            bi[pos] = bi[pos - 1];
            --pos;
          }
          bd[pos] = d2;
          bi[pos] = (int32_t)q;
          if (cnt < K) ++cnt;
        }
      }
    // inner faces of the scanned cube (a face on the domain boundary excludes nothing)
    double margin = 2.0;
    if (x0 > 0) margin = fmin(margin, px - x0 * h);
    if (x1 < G - 1) margin = fmin(margin, (x1 + 1) * h - px);
    if (y0 > 0) margin = fmin(margin, py - y0 * h);
    if (y1 < G - 1) margin = fmin(margin, (y1 + 1) * h - py);
    if (z0 > 0) margin = fmin(margin, pz - z0 * h);
    if (z1 < G - 1) margin = fmin(margin, (z1 + 1) * h - pz);
    const bool whole = x0 == 0 && y0 == 0 && z0 == 0 && x1 == G - 1 && y1 == G - 1 && z1 == G - 1;
    if (whole || (cnt == K && bd[K - 1] < margin * margin * (1.0 - 1e-12))) {
      for (int k = 0; k < K; ++k) {
        out_idx[t * K + k] = k < cnt ? bi[k] : -1;
        out_d2[t * K + k] = k < cnt ? bd[k] : 0.0;
      }
      return;
    }
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

// config 4 (block transport): row offsets of A and P for rows [row_lo, row_hi)
ptap_status ptap_gen_block_transport_rowptr(int64_t nn, int ncomp, int64_t agg, int64_t row_lo, int64_t row_hi,
                                            int64_t *a_row_ptr, int64_t *a_nnz_out, int64_t *p_row_ptr,
                                            int64_t *p_nnz_out, void *stream) {
  if (nn <= 0 || ncomp <= 0 || agg <= 0) return PTAP_ERR_VALUE;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t nr = row_hi - row_lo;
  if (nr > 0) k_bt_count<<<nb(nr), 256, 0, st>>>(nn, ncomp, agg, row_lo, row_hi, a_row_ptr + 1, p_row_ptr + 1);
  if (cudaGetLastError() != cudaSuccess) return PTAP_ERR_CUDA;
  ptap_status s = finish_rowptr(a_row_ptr, nr, a_nnz_out, st);
  if (s != PTAP_OK) return s;
  return finish_rowptr(p_row_ptr, nr, p_nnz_out, st);
}

ptap_status ptap_gen_block_transport_a(int64_t nn, int ncomp, uint64_t seed, int64_t row_lo, int64_t row_hi,
                                       const int64_t *row_ptr, int32_t *col, double *val, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  int64_t nr = row_hi - row_lo;
  if (nr > 0) k_bt_fill_a<<<nb(nr), 256, 0, st>>>(nn, ncomp, seed, row_lo, row_hi, row_ptr, col, val);
  return cudaGetLastError() == cudaSuccess ? PTAP_OK : PTAP_ERR_CUDA;
}

ptap_status ptap_gen_spmv_dinv(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *val,
                               const double *v, double *w, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n > 0) k_spmv_dinv<<<nb(n), 256, 0, st>>>(n, row_ptr, col, val, v, w);
  return cudaGetLastError() == cudaSuccess ? PTAP_OK : PTAP_ERR_CUDA;
}

ptap_status ptap_gen_block_transport_p(int64_t nn, int ncomp, int64_t agg, double omega, int64_t row_lo,
                                       int64_t row_hi, const int64_t *a_row_ptr, const double *a_val,
                                       const int64_t *p_row_ptr, int32_t *p_col, double *p_val, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  int64_t nr = row_hi - row_lo;
  if (nr > 0)
    k_bt_fill_p<<<nb(nr), 256, 0, st>>>(nn, ncomp, agg, omega, row_lo, row_hi, a_row_ptr, a_val, p_row_ptr, p_col,
                                        p_val);
  return cudaGetLastError() == cudaSuccess ? PTAP_OK : PTAP_ERR_CUDA;
}

// config 5: K nearest neighbours (K <= 32) of n points sorted by cell of a G^3
// grid (pts: xyz per point; cell_start: G^3 + 1 offsets into the sorted
// points).  out_idx / out_d2: [n * K] neighbour (sorted index) and squared
// distance, ascending; -1 pads when fewer than K other points exist.
ptap_status ptap_gen_knn(int64_t n, const double *pts, const int64_t *cell_start, int G, int K, int32_t *out_idx,
                         double *out_d2, void *stream) {
  if (K <= 0 || K > KNN_MAX || G <= 0) return PTAP_ERR_VALUE;
  cudaStream_t st = (cudaStream_t)stream;
  if (n > 0)
    k_knn_cells<<<(int)((n + 127) / 128), 128, 0, st>>>(n, pts, (const long long *)cell_start, G, K, out_idx, out_d2);
  return cudaGetLastError() == cudaSuccess ? PTAP_OK : PTAP_ERR_CUDA;
}

}  // extern "C"
