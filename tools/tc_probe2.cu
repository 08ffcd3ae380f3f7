// Probe of the tcgen05 kind::tf32 building blocks for the micro-batch (M=16) path:
//  (1) forward  D[r][m] = sum_c W[r][c] X[m][c]: W tile by TMA 2-D (box 128 rows x 32 cols,
//      SWIZZLE_128B) = UMMA A K-major SW128; X by SIMT into the no-swizzle K-major layout.
//  (2) backward E[c][m] = sum_r W[r][c] Y[m][r]: the same W region by TMA with
//      SWIZZLE_128B_ATOM_32B = UMMA A MN-major SWIZZLE_128B_BASE32B; Y no-swizzle K-major.
//  (3) TMA 2-D store of the ATOM_32B tile (round trip through global).
// Small-integer values, exact in tf32: any layout error shows as a mismatch.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_probe2 tools/tc_probe2.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2210_09147_b200/csrc/pt_ptx.cuh"
#include "../paper_2210_09147_b200/csrc/pt_tc.cuh"
using namespace pt;

constexpr int R = 128, C = 128, MB = 16;

__global__ void __launch_bounds__(128, 1) probe(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_mn,
                                               const __grid_constant__ CUtensorMap tm_out, const float* X, const float* Y,
                                               float* D, float* E, int variant, float* raw) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = smraw;
  float* sWk = reinterpret_cast<float*>(sm);               // 4 boxes x 16 KB (K-major SW128)
  float* sWm = reinterpret_cast<float*>(sm + 65536);       // 4 boxes x 16 KB (MN-major SW128_32B)
  float* sX = reinterpret_cast<float*>(sm + 131072);       // 16 x 128 no-swizzle K-major (8 KB)
  float* sY = reinterpret_cast<float*>(sm + 139264);       // 16 x 128
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 147456);
  uint32_t* taddr_s = reinterpret_cast<uint32_t*>(bar + 4);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < MB * C; i += blockDim.x) {
    const int m = i / C, k = i % C;
    sX[tc_kmajor_noswz_off(m, k, C) / 4] = X[i];
    sY[tc_kmajor_noswz_off(m, k, C) / 4] = Y[i];
  }
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  fence_proxy_async_shared();
  __syncthreads();
  if (warp == 0) tmem_alloc(taddr_s, 64);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *taddr_s;
  if (tid == 0) {
    mbar_arrive_expect_tx(&bar[0], 2 * 65536);
    for (int b = 0; b < 4; ++b) {
      tma_load_2d(sWk + b * 4096, &tm_k, b * 32, 0, &bar[0]);
      tma_load_2d(sWm + b * 4096, &tm_mn, b * 32, 0, &bar[0]);
    }
    while (!mbar_try_wait(&bar[0], 0)) {
    }
    tc_fence_after();
    // forward: A = W (M = 128 rows, K-major SW128), B = X (N = 16, K-major no swizzle)
    const uint32_t idf = tc_idesc_tf32(128, 16, false, false);
    for (int ks = 0; ks < C / 8; ++ks) {
      const uint64_t da = tc_desc_kmajor_sw128(sWk + (ks / 4) * 4096, (ks % 4) * 32);
      const uint64_t db = tc_desc_kmajor_noswz(sX, ks, C);
      tc_mma_tf32(tbase, da, db, idf, ks > 0);
    }
    // backward: A = W^T (M = 128 cols, MN-major SW128_32B), B = Y (N = 16, K = rows)
    const uint32_t idb = tc_idesc_tf32(128, 16, true, false);
    for (int ks = 0; ks < R / 8; ++ks) {
      const uint64_t da = tc_desc_mn_sw128b32(sWm, ks * 8, 16384);
      const uint64_t db = tc_desc_kmajor_noswz(sY, ks, R);
      tc_mma_tf32(tbase + 16, da, db, idb, ks > 0);
    }
    tc_commit(&bar[1]);
  }
  __syncwarp();
  while (!mbar_try_wait(&bar[1], 0)) {
  }
  tc_fence_after();
  {
    float v[32];
    tmem_ld_32x32b_x32(tbase + ((uint32_t(warp) * 32) << 16), v);
    const int row = warp * 32 + lane;
    for (int j = 0; j < 16; ++j) D[row * 16 + j] = v[j];
    for (int j = 0; j < 16; ++j) E[row * 16 + j] = v[16 + j];
  }
  for (int i = tid; i < 4 * 4096; i += blockDim.x) raw[i] = sWm[i];
  // (3) negate the MN tile in smem and store it back through the ATOM_32B map
  __syncthreads();
  for (int i = tid; i < 4 * 4096; i += blockDim.x) sWm[i] = -sWm[i];
  fence_proxy_async_shared();
  __syncthreads();
  if (tid == 0) {
    for (int b = 0; b < 4; ++b) tma_store_2d(&tm_out, sWm + b * 4096, b * 32, 0);
    bulk_commit();
    bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free(tbase, 64);
}

int main() {
  std::vector<float> W(R * C), X(MB * C), Y(MB * R), D(R * 16), E(C * 16), Wo(R * C);
  srand(1);
  for (auto& v : W) v = float(rand() % 7 - 3);
  for (auto& v : X) v = float(rand() % 5 - 2);
  for (auto& v : Y) v = float(rand() % 5 - 2);
  float *dW, *dX, *dY, *dD, *dE, *dWo;
  cudaMalloc(&dW, W.size() * 4);
  cudaMalloc(&dWo, W.size() * 4);
  cudaMalloc(&dX, X.size() * 4);
  cudaMalloc(&dY, Y.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMalloc(&dE, E.size() * 4);
  cudaMemcpy(dW, W.data(), W.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dY, Y.data(), Y.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap tk, tmn, tout;
  if (tc_make_tmap_2d(&tk, dW, C, R, 32, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
      tc_make_tmap_2d(&tmn, dW, C, R, 32, 128, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) ||
      tc_make_tmap_2d(&tout, dWo, C, R, 32, 128, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) {
    printf("tensor map encode failed\n");
    return 2;
  }
  const int smem = 147456 + 64;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  float* dRaw;
  cudaMalloc(&dRaw, 4 * 4096 * 4);
  probe<<<1, 128, smem>>>(tk, tmn, tout, dX, dY, dD, dE, 0, dRaw);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(E.data(), dE, E.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(Wo.data(), dWo, Wo.size() * 4, cudaMemcpyDeviceToHost);
  std::vector<float> raw(4 * 4096);
  cudaMemcpy(raw.data(), dRaw, raw.size() * 4, cudaMemcpyDeviceToHost);
  // ATOM_32B smem pattern: element (r, 32b + 8g + e) at b*4096 + r*32 + 8*(g ^ f(r)) + e
  for (int hyp = 0; hyp < 3; ++hyp) {
    int bad = 0;
    for (int b = 0; b < 4; ++b)
      for (int r = 0; r < 128; ++r)
        for (int g = 0; g < 4; ++g)
          for (int e = 0; e < 8; ++e) {
            const int f = hyp == 0 ? (r & 3) : hyp == 1 ? ((r >> 1) & 3) : 0;
            bad += raw[b * 4096 + r * 32 + 8 * (g ^ f) + e] != W[r * C + 32 * b + 8 * g + e];
          }
    printf("ATOM_32B layout hypothesis %d (%s): %d mismatches\n", hyp, hyp == 0 ? "g ^ (r & 3)" : hyp == 1 ? "g ^ ((r>>1) & 3)" : "no swizzle", bad);
  }
  int bad_d = 0, bad_e = 0, bad_w = 0;
  for (int r = 0; r < R; ++r)
    for (int m = 0; m < 16; ++m) {
      float ref = 0;
      for (int k = 0; k < C; ++k) ref += W[r * C + k] * X[m * C + k];
      if (ref != D[r * 16 + m] && bad_d++ < 4) printf("D[%d][%d] = %g ref %g\n", r, m, D[r * 16 + m], ref);
    }
  for (int c = 0; c < C; ++c)
    for (int m = 0; m < 16; ++m) {
      float ref = 0;
      for (int r = 0; r < R; ++r) ref += W[r * C + c] * Y[m * R + r];
      if (ref != E[c * 16 + m] && bad_e++ < 4) printf("E[%d][%d] = %g ref %g\n", c, m, E[c * 16 + m], ref);
    }
  for (int i = 0; i < R * C; ++i) bad_w += Wo[i] != -W[i];
  printf("forward (K-major SW128) mismatches %d / %d; backward (MN-major SW128_32B) mismatches %d / %d; "
         "store round trip mismatches %d / %d\n", bad_d, R * 16, bad_e, C * 16, bad_w, R * C);
  return (bad_d || bad_e || bad_w) ? 1 : 0;
}
