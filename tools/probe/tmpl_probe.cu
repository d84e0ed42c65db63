// Speed probe (not product code): row-class ("template") numeric kernel for the
// 27-point / trilinear shape at 256^3 -> 128^3.  Synthetic data with the real
// access pattern: lane = fine row of one parity class, tile = 64 consecutive
// rows, P values of the tile's 9 neighbour line segments staged in shared
// memory, AP row accumulated in registers (uniform switch) or in shared memory.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)

constexpr int NX = 256, NC = 128;
constexpr int R = 64;          // rows per tile
constexpr int NA = 27;
constexpr int HALO = 2560;     // doubles
struct Tmpl { int nA, nap, nP, npairs; uint8_t plen[32]; uint8_t slot[128]; uint8_t pmap[8 * 32]; };
__constant__ Tmpl c_T[8];

__host__ __device__ inline int plen1(int c) { return (c & 1) ? 2 : 1; }
__device__ inline int clampi(int v) { return v < 0 ? 0 : (v > NX - 1 ? NX - 1 : v); }

__global__ void k_prow_len(int64_t n, int64_t *len) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; if (i >= n) return;
  int x = i % NX, y = (i / NX) % NX, z = i / (NX * NX);
  len[i] = plen1(x) * plen1(y) * plen1(z);
}
// P columns: coarse coords per dim (odd c -> (c-1)/2,(c+1)/2 clamped)
__global__ void k_pcol(int64_t n, const int64_t *prp, int32_t *pcol) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; if (i >= n) return;
  int x = i % NX, y = (i / NX) % NX, z = i / (NX * NX);
  int64_t q = prp[i];
  for (int a = 0; a < plen1(z); ++a) for (int b = 0; b < plen1(y); ++b) for (int c = 0; c < plen1(x); ++c) {
    int cz = min((z >> 1) + a, NC - 1), cy = min((y >> 1) + b, NC - 1), cx = min((x >> 1) + c, NC - 1);
    pcol[q++] = (cz * NC + cy) * NC + cx;
  }
}
// hoff of every A entry (tile-local halo position) + tile halo segments
__global__ void k_hoff(int64_t n, const int64_t *prp, uint16_t *hoff, int *bad) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; if (i >= n) return;
  int x = i % NX, y = (i / NX) % NX, z = i / (NX * NX);
  int x0 = x & ~(R - 1);
  int xl = max(x0 - 1, 0), xh = min(x0 + R + 1, NX);
  int base[9]; int acc = 0;
  for (int s = 0; s < 9; ++s) {
    int zz = clampi(z + s / 3 - 1), yy = clampi(y + s % 3 - 1);
    int64_t r0 = ((int64_t)zz * NX + yy) * NX + xl, r1 = ((int64_t)zz * NX + yy) * NX + xh;
    base[s] = acc; acc += (int)(prp[r1] - prp[r0]);
  }
  if (acc > HALO) atomicAdd(bad, 1);
  int e = 0;
  for (int dz = -1; dz <= 1; ++dz) for (int dy = -1; dy <= 1; ++dy) for (int dx = -1; dx <= 1; ++dx, ++e) {
    int s = (dz + 1) * 3 + dy + 1;
    int zz = clampi(z + dz), yy = clampi(y + dy), xx = clampi(x + dx);
    int64_t r0 = ((int64_t)zz * NX + yy) * NX + xl, k = ((int64_t)zz * NX + yy) * NX + xx;
    hoff[i * NA + e] = (uint16_t)(base[s] + prp[k] - prp[r0]);
  }
}
__global__ void k_tile_segs(int64_t ntiles, const int64_t *prp, int64_t *seg_src, int32_t *seg_len) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; if (t >= ntiles) return;
  int64_t i = t * R;
  int x = i % NX, y = (i / NX) % NX, z = i / (NX * NX);
  int xl = max(x - 1, 0), xh = min(x + R + 1, NX);
  for (int s = 0; s < 9; ++s) {
    int zz = clampi(z + s / 3 - 1), yy = clampi(y + s % 3 - 1);
    int64_t r0 = ((int64_t)zz * NX + yy) * NX + xl, r1 = ((int64_t)zz * NX + yy) * NX + xh;
    seg_src[t * 9 + s] = prp[r0]; seg_len[t * 9 + s] = (int)(prp[r1] - prp[r0]);
  }
}
__global__ void k_fill(int64_t n, double *v, uint64_t seed) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; if (i >= n) return;
  uint64_t h = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed; h ^= h >> 29; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 32;
  v[i] = 0.5 + (double)(h >> 11) * (1.0 / 9007199254740992.0);
}

#define ACC_CASES(X) X(0) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) \
  X(16) X(17) X(18) X(19) X(20) X(21) X(22) X(23) X(24) X(25) X(26) X(27) X(28) X(29) X(30) X(31)

template <int MODE, int PH = 7>  // 0: register accumulators via uniform switch, 1: shared accumulators
__global__ void __launch_bounds__(64) k_tmpl(int64_t ntiles, const double *__restrict__ aval,
    const uint16_t *__restrict__ hoff, const double *__restrict__ pval, const int64_t *__restrict__ prp,
    const int32_t *__restrict__ pcol, const int64_t *__restrict__ seg_src, const int32_t *__restrict__ seg_len,
    double *cval) {
  extern __shared__ __align__(16) unsigned char smem[];
  double *halo = (double *)smem;
  double *sa = halo + HALO;
  uint16_t *sh = (uint16_t *)(sa + R * NA);
  int (*scb0)[8][32] = (int (*)[8][32])((double (*)[8][32])(sh + R * NA) + 2);
  double (*acc_sh)[32][33] = (PH & 1) ? (double (*)[32][33])sa : (double (*)[32][33])(scb0 + 2);  // aliases sa/sh after the folds
  double (*spv)[8][32] = (double (*)[8][32])(sh + R * NA);
  int (*scb)[8][32] = (int (*)[8][32])(spv + 2);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    __syncthreads();
    int hb = 0;
    if ((PH & 1) || t == blockIdx.x) for (int s = 0; s < 9; ++s) {
      const int64_t src = seg_src[t * 9 + s]; const int len = seg_len[t * 9 + s];
      for (int q = threadIdx.x; q < len; q += 64) halo[hb + q] = pval[src + q];
      hb += len;
    }
    const int64_t a0 = t * R * NA;
    if ((PH & 1) || t == blockIdx.x) for (int q = threadIdx.x; q < R * NA; q += 64) { sa[q] = aval[a0 + q]; sh[q] = hoff[a0 + q]; }
    const int64_t i0 = t * R;
    const int y = (i0 / NX) % NX, z = i0 / (NX * NX);
    const Tmpl &T = c_T[(z & 1) * 4 + (y & 1) * 2 + w];
    const int lr = 2 * lane + w;
    const int64_t i = i0 + lr;
    const int nP = T.nP, nap = T.nap;
    {  // own P row: targets
      const int64_t p0 = prp[i];
      for (int j = 0; j < nP; ++j) { spv[w][j][lane] = pval[p0 + j]; scb[w][j][lane] = pcol[p0 + j] * 27; }
    }
    __syncthreads();
    const int off = lr * NA;
    if (!(PH & 2)) { } else if (MODE == 0) {
#define DECL(k) double r##k = 0.0;
      ACC_CASES(DECL)
      int pj = 0;
      for (int e = 0; e < T.nA; ++e) {
        const double a = sa[off + e];
        const int h = sh[off + e];
        const int pl = T.plen[e];
        for (int q = 0; q < pl; ++q, ++pj) {
          const double p = halo[h + q];
          switch (T.slot[pj]) {
#define CASE(k) case k: r##k = fma(a, p, r##k); break;
            ACC_CASES(CASE)
          }
        }
      }
      __syncthreads();
#define STORE(k) if (k < nap) acc_sh[w][lane][k] = r##k;
      ACC_CASES(STORE)
    } else {
      double (*acc2)[33] = (double (*)[33])(scb + 2) + w * 32;  // separate region
      for (int s = 0; s < nap; ++s) acc2[lane][s] = 0.0;
      int pj = 0;
      for (int e = 0; e < T.nA; ++e) {
        const double a = sa[off + e];
        const int h = sh[off + e];
        const int pl = T.plen[e];
        for (int q = 0; q < pl; ++q, ++pj) {
          const double p = halo[h + q];
          double *ac = &acc2[lane][T.slot[pj]];
          *ac = fma(a, p, *ac);
        }
      }
      __syncthreads();
      for (int s = 0; s < nap; ++s) acc_sh[w][lane][s] = acc2[lane][s];
    }
    __syncwarp();
    // outer: flat (row, target, slot) over lanes
    int r = 0, j = 0, s = lane;
    while (s >= nap) { s -= nap; if (++j == nP) { j = 0; ++r; } }
    if (PH & 4) for (; r < 32;) {
      atomicAdd(cval + scb[w][j][r] + T.pmap[j * 32 + s], spv[w][j][r] * acc_sh[w][r][s]);
      s += 32;
      while (s >= nap) { s -= nap; if (++j == nP) { j = 0; ++r; } }
    }
  }
}

__global__ void k_stream(int64_t n, const double *a, const uint16_t *h, double *out) {
  double s = 0; int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += st) s += a[i] + h[i];
  if (s == 1.2345) out[0] = s;
}

static void build_templates() {
  Tmpl T[8];
  for (int cls = 0; cls < 8; ++cls) {
    int px = cls & 1, py = (cls >> 1) & 1, pz = (cls >> 2) & 1;
    int x = 20 + px, y = 20 + py, z = 20 + pz;
    auto pr = [&](int xx, int yy, int zz) {
      std::vector<int> c;
      for (int a = 0; a < plen1(zz); ++a) for (int b = 0; b < plen1(yy); ++b) for (int d = 0; d < plen1(xx); ++d)
        c.push_back((((zz >> 1) + a) * NC + (yy >> 1) + b) * NC + (xx >> 1) + d);
      return c;
    };
    std::vector<int> all; std::vector<std::vector<int>> rows;
    for (int dz = -1; dz <= 1; ++dz) for (int dy = -1; dy <= 1; ++dy) for (int dx = -1; dx <= 1; ++dx) {
      rows.push_back(pr(x + dx, y + dy, z + dz)); for (int c : rows.back()) all.push_back(c);
    }
    std::sort(all.begin(), all.end()); all.erase(std::unique(all.begin(), all.end()), all.end());
    Tmpl &t = T[cls]; memset(&t, 0, sizeof t);
    t.nA = 27; t.nap = (int)all.size(); int pj = 0;
    for (int e = 0; e < 27; ++e) { t.plen[e] = rows[e].size();
      for (int c : rows[e]) t.slot[pj++] = std::lower_bound(all.begin(), all.end(), c) - all.begin(); }
    t.npairs = pj;
    std::vector<int> own = pr(x, y, z); t.nP = own.size();
    for (int j = 0; j < t.nP; ++j) {
      int J = own[j], jx = J % NC, jy = (J / NC) % NC, jz = J / (NC * NC);
      for (int s = 0; s < t.nap; ++s) { int G = all[s], gx = G % NC, gy = (G / NC) % NC, gz = G / (NC * NC);
        t.pmap[j * 32 + s] = ((gz - jz + 1) * 3 + gy - jy + 1) * 3 + gx - jx + 1; }
    }
    printf("class %d: nap %d pairs %d nP %d\n", cls, t.nap, t.npairs, t.nP);
  }
  CK(cudaMemcpyToSymbol(c_T, T, sizeof T));
}

int main() {
  const int64_t n = (int64_t)NX * NX * NX, m = (int64_t)NC * NC * NC, ntiles = n / R;
  build_templates();
  int64_t *prp, *len; CK(cudaMalloc(&prp, (n + 1) * 8)); CK(cudaMalloc(&len, n * 8));
  k_prow_len<<<(n + 255) / 256, 256>>>(n, len);
  std::vector<int64_t> hl(n); CK(cudaMemcpy(hl.data(), len, n * 8, cudaMemcpyDeviceToHost));
  std::vector<int64_t> hp(n + 1, 0); for (int64_t i = 0; i < n; ++i) hp[i + 1] = hp[i] + hl[i];
  CK(cudaMemcpy(prp, hp.data(), (n + 1) * 8, cudaMemcpyHostToDevice));
  const int64_t pnnz = hp[n]; printf("nnz(P) %lld\n", (long long)pnnz);
  int32_t *pcol; double *pval, *aval, *cval; uint16_t *hoff; int64_t *seg_src; int32_t *seg_len; int *bad;
  CK(cudaMalloc(&pcol, pnnz * 4)); CK(cudaMalloc(&pval, pnnz * 8)); CK(cudaMalloc(&aval, n * NA * 8));
  CK(cudaMalloc(&hoff, n * NA * 2)); CK(cudaMalloc(&cval, m * 27 * 8)); CK(cudaMalloc(&seg_src, ntiles * 9 * 8));
  CK(cudaMalloc(&seg_len, ntiles * 9 * 4)); CK(cudaMalloc(&bad, 4)); CK(cudaMemset(bad, 0, 4));
  k_pcol<<<(n + 255) / 256, 256>>>(n, prp, pcol);
  k_fill<<<(pnnz + 255) / 256, 256>>>(pnnz, pval, 1); k_fill<<<(n * NA + 255) / 256, 256>>>(n * NA, aval, 2);
  k_hoff<<<(n + 255) / 256, 256>>>(n, prp, hoff, bad);
  k_tile_segs<<<(ntiles + 255) / 256, 256>>>(ntiles, prp, seg_src, seg_len);
  CK(cudaDeviceSynchronize()); int hb; CK(cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost)); printf("halo overflow rows %d\n", hb);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int dev; cudaGetDevice(&dev); int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  auto run = [&](const char *name, auto launch) {
    for (int w = 0; w < 3; ++w) launch();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); for (int k = 0; k < 10; ++k) launch(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); printf("%-28s %.3f ms\n", name, ms / 10);
  };
  run("stream A vals+hoff", [&] { k_stream<<<nsm * 8, 256>>>(n * NA, aval, hoff, cval); });
  const size_t SM0 = HALO * 8 + R * NA * 10 + 2 * 8 * 32 * 12, SM1 = SM0 + 2 * 32 * 33 * 8;
  CK(cudaFuncSetAttribute(k_tmpl<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM0));
  CK(cudaFuncSetAttribute(k_tmpl<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM1));
  CK(cudaFuncSetAttribute(k_tmpl<0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM1));
  CK(cudaFuncSetAttribute(k_tmpl<0, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM1));
  CK(cudaFuncSetAttribute(k_tmpl<0, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM1));
  CK(cudaFuncSetAttribute(k_tmpl<0, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM1));
  CK(cudaFuncSetAttribute(k_tmpl<1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM1));
  for (int per : {3}) {
    run("stage only", [&] { k_tmpl<0, 1><<<nsm * per, 64, SM1>>>(ntiles, aval, hoff, pval, prp, pcol, seg_src, seg_len, cval); });
    run("fold only (reg)", [&] { k_tmpl<0, 2><<<nsm * per, 64, SM1>>>(ntiles, aval, hoff, pval, prp, pcol, seg_src, seg_len, cval); });
    run("outer only", [&] { k_tmpl<0, 4><<<nsm * per, 64, SM1>>>(ntiles, aval, hoff, pval, prp, pcol, seg_src, seg_len, cval); });
    run("fold+outer (reg)", [&] { k_tmpl<0, 6><<<nsm * per, 64, SM1>>>(ntiles, aval, hoff, pval, prp, pcol, seg_src, seg_len, cval); });
    run("fold only (smem)", [&] { k_tmpl<1, 2><<<nsm * 3, 64, SM1>>>(ntiles, aval, hoff, pval, prp, pcol, seg_src, seg_len, cval); });

    int occ0, occ1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ0, k_tmpl<0>, 64, SM0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, k_tmpl<1>, 64, SM1);
    if (per == 4) printf("occupancy: reg %d CTAs/SM, smem %d CTAs/SM\n", occ0, occ1);
    char b[64];
    snprintf(b, 64, "tmpl reg-acc grid %dx", per); run(b, [&] { k_tmpl<0><<<nsm * per, 64, SM0>>>(ntiles, aval, hoff, pval, prp, pcol, seg_src, seg_len, cval); });
    snprintf(b, 64, "tmpl smem-acc grid %dx", per); run(b, [&] { k_tmpl<1><<<nsm * per, 64, SM1>>>(ntiles, aval, hoff, pval, prp, pcol, seg_src, seg_len, cval); });
  }
  CK(cudaGetLastError());
  return 0;
}
