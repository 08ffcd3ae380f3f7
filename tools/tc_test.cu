// Stand-alone validation of the tcgen05 kind::tf32 building blocks used by the M>1 path:
//  - W tile stored as 8-row x 16-byte core matrices (block(rg, kq) at rg*S_rg + kq*S_kq)
//  - forward:  D[r][m]  = sum_k W[r][k] * X[m][k]   (A = W   K-major, B = X K-major)
//  - backward: E[c][m]  = sum_r W[r][c] * Y[m][r]   (A = W^T MN-major on the SAME smem, B = Y K-major)
//  - TMEM alloc / commit-to-mbarrier / tcgen05.ld 32x32b readback
// Values are small integers (exact in tf32) so any layout error shows as a mismatch.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2210_09147_b200/csrc/pt_ptx.cuh"
using namespace pt;

constexpr int R = 128, C = 128, MB = 16;  // W is R x C, batch MB

__device__ __forceinline__ uint64_t sdesc(const void* p, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((smem_u32(p) >> 4) & 0x3FFF);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;  // version 1 (sm100)
  return d;                // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
}
__device__ __forceinline__ uint32_t idesc_tf32(int M, int N, int a_mn, int b_mn) {
  uint32_t d = 0;
  d |= 1u << 4;             // c_format F32
  d |= 2u << 7;             // a_format TF32
  d |= 2u << 10;            // b_format TF32
  d |= uint32_t(a_mn) << 15;
  d |= uint32_t(b_mn) << 16;
  d |= uint32_t(N >> 3) << 17;
  d |= uint32_t(M >> 4) << 24;
  return d;
}

__global__ void tc_kernel(const float* W, const float* X, const float* Y, float* D, float* E, int variant) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float* sW = reinterpret_cast<float*>(sm);                  // 64 KB blocked
  float* sX = sW + R * C;                                    // 16 x 128 blocked (8 KB)
  float* sY = sX + MB * C;                                   // 16 x 128 blocked
  uint64_t* bar = reinterpret_cast<uint64_t*>(sY + MB * R);
  uint32_t* taddr_s = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // blocked store: element (row, k) of a [rows x K] matrix -> block(row/8, k/4)
  const int S_kq_W = 128, S_rg_W = (C / 4) * 128;
  for (int i = tid; i < R * C; i += blockDim.x) {
    const int r = i / C, k = i % C;
    sW[((r / 8) * S_rg_W + (k / 4) * S_kq_W + (r % 8) * 16 + (k % 4) * 4) / 4] = W[i];
  }
  const int S_kq_X = 128, S_ng_X = (C / 4) * 128;
  for (int i = tid; i < MB * C; i += blockDim.x) {
    const int m = i / C, k = i % C;
    sX[((m / 8) * S_ng_X + (k / 4) * S_kq_X + (m % 8) * 16 + (k % 4) * 4) / 4] = X[i];
    sY[((m / 8) * S_ng_X + (k / 4) * S_kq_X + (m % 8) * 16 + (k % 4) * 4) / 4] = Y[i];
  }
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = *taddr_s;
  if (tid == 0) {
    // forward: D (cols 0..15) = W[128 x 128] * X^T, 16 K-steps of 8
    const uint32_t idf = idesc_tf32(128, 16, 0, 0);
    for (int ks = 0; ks < C / 8; ++ks) {
      const uint64_t da = sdesc(reinterpret_cast<char*>(sW) + ks * 2 * S_kq_W, S_kq_W, S_rg_W);
      const uint64_t db = sdesc(reinterpret_cast<char*>(sX) + ks * 2 * S_kq_X, S_kq_X, S_ng_X);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tbase),
                   "l"(da), "l"(db), "r"(idf), "r"(ks));
    }
    // backward: E (cols 16..31) = W^T[128 c x 128 r] * Y^T, A MN-major on the same smem
    const uint32_t idb = idesc_tf32(128, 16, variant == 3 ? 0 : 1, 0);
    for (int ks = 0; ks < R / 8; ++ks) {
      uint32_t lbo = S_rg_W, sbo = S_kq_W;
      if (variant == 1) { lbo = S_kq_W; sbo = S_rg_W; }
      if (variant == 2) { lbo = S_kq_W * 2; sbo = S_rg_W; }
      if (variant == 4) { lbo = 128; sbo = 128; }
      const uint64_t da = sdesc(reinterpret_cast<char*>(sW) + ks * S_rg_W, lbo, sbo);
      const uint64_t db = sdesc(reinterpret_cast<char*>(sY) + ks * 2 * S_kq_X, S_kq_X, S_ng_X);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tbase + 16),
                   "l"(da), "l"(db), "r"(idb), "r"(ks));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
  }
  while (!mbar_try_wait(bar, 0)) {
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < 4) {
    uint32_t v[32];
    const uint32_t ta = tbase + ((uint32_t(warp) * 32) << 16);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int row = warp * 32 + lane;
    for (int j = 0; j < 16; ++j) D[row * 16 + j] = __uint_as_float(v[j]);
    for (int j = 0; j < 16; ++j) E[row * 16 + j] = __uint_as_float(v[16 + j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tbase));
}

int main(int argc, char** argv) {
  std::vector<float> W(R * C), X(MB * C), Y(MB * R), D(R * 16), E(C * 16);
  srand(1);
  for (auto& v : W) v = float(rand() % 7 - 3);
  for (auto& v : X) v = float(rand() % 5 - 2);
  for (auto& v : Y) v = float(rand() % 5 - 2);
  float *dW, *dX, *dY, *dD, *dE;
  cudaMalloc(&dW, W.size() * 4); cudaMalloc(&dX, X.size() * 4); cudaMalloc(&dY, Y.size() * 4);
  cudaMalloc(&dD, D.size() * 4); cudaMalloc(&dE, E.size() * 4);
  cudaMemcpy(dW, W.data(), W.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dY, Y.data(), Y.size() * 4, cudaMemcpyHostToDevice);
  const int smem = (R * C + 2 * MB * C) * 4 + 64;
  cudaFuncSetAttribute(tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int variant = argc > 1 ? atoi(argv[1]) : 0;
  tc_kernel<<<1, 256, smem>>>(dW, dX, dY, dD, dE, variant);
  cudaError_t e = cudaDeviceSynchronize();
  printf("variant %d kernel: %s\n", variant, cudaGetErrorString(e));
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(E.data(), dE, E.size() * 4, cudaMemcpyDeviceToHost);
  int bad_d = 0, bad_e = 0;
  for (int r = 0; r < R; ++r)
    for (int m = 0; m < 16; ++m) {
      float ref = 0;
      for (int k = 0; k < C; ++k) ref += W[r * C + k] * X[m * C + k];
      if (ref != D[r * 16 + m] && bad_d++ < 5) printf("D[%d][%d] = %f ref %f\n", r, m, D[r * 16 + m], ref);
    }
  for (int c = 0; c < C; ++c)
    for (int m = 0; m < 16; ++m) {
      float ref = 0;
      for (int r = 0; r < R; ++r) ref += W[r * C + c] * Y[m * R + r];
      if (ref != E[c * 16 + m] && bad_e++ < 5) printf("E[%d][%d] = %f ref %f\n", c, m, E[c * 16 + m], ref);
    }
  // diagnose: is E a permutation of the reference?
  if (bad_e) {
    int nz = 0; for (auto v : E) nz += v != 0.f;
    printf("nonzero E entries: %d\n", nz);
    // try E as [c][m] vs reference transposed layouts
    for (int c = 0; c < 4; ++c) { printf("E row %d:", c); for (int m = 0; m < 6; ++m) printf(" %g", E[c * 16 + m]); printf("\n"); }
    for (int c = 0; c < 4; ++c) { printf("ref row %d:", c); for (int m = 0; m < 6; ++m) { float ref = 0; for (int r = 0; r < R; ++r) ref += W[r * C + c] * Y[m * R + r]; printf(" %g", ref);} printf("\n"); }
  }
  printf("forward mismatches %d / %d, backward (MN-major) mismatches %d / %d\n", bad_d, R * 16, bad_e, C * 16);
  return (bad_d || bad_e) ? 1 : 0;
}
