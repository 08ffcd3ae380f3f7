// Throughput of back-to-back tcgen05.mma kind::tf32 (M=64/128, K=8) for several N, A from
// smem (K-major SW128) or TMEM, one thread issuing, one CTA per SM (148 CTAs).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_rate tools/mma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2210_09147_b200/csrc/pt_tc.cuh"
using namespace pt;

__global__ void __launch_bounds__(128, 1) mma_rate(int n_iter, int M, int N, int a_tmem, int warp_issue, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 163840);
  uint32_t* taddr = reinterpret_cast<uint32_t*>(bar + 2);
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 163840 / 4; i += 128) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (tid == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  fence_proxy_async_shared();
  __syncthreads();
  if (warp == 0) tmem_alloc(taddr, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = *taddr;
  const uint32_t id = tc_idesc_tf32(M, N, false, false);
  unsigned long long t0 = 0, t1 = 0;
  if (warp == 0 && (warp_issue || (tid & 31) == 0)) {
    const uint64_t da = tc_desc_kmajor_sw128(sm, 0);
    const uint64_t db = tc_desc_kmajor_noswz(sm + 32768, 0, 64);
    t0 = globaltimer();
    for (int i = 0; i < n_iter; ++i) {
      const int ks = i & 7;
      if (!warp_issue || (tid & 31) == 0) {
        if (a_tmem) tc_mma_tf32_ts(tb, tb + 256 + ks * 8, db + ks * 16, id, i > 0);
        else tc_mma_tf32(tb, da + (ks >> 2) * 1024 + (ks & 3) * 2, db + ks * 16, id, i > 0);
      }
      if (warp_issue) __syncwarp();
    }
    if ((tid & 31) == 0) tc_commit(bar);
    if (warp_issue) __syncwarp();
    while (!mbar_try_wait(bar, 0)) {}
    t1 = globaltimer();
    if ((tid & 31) == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free(tb, 512);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 163840 + 64);
  for (int M : {128, 64})
  for (int wi : {0})
    for (int at : {0, 1})
      for (int N : {16, 32, 64, 128, 256}) {
        const int n = 4096;
        if (M == 64 && at) continue;
        mma_rate<<<148, 128, 163840 + 64>>>(n, M, N, at, wi, d);
        cudaDeviceSynchronize();
        mma_rate<<<148, 128, 163840 + 64>>>(n, M, N, at, wi, d);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long ns;
        cudaMemcpy(&ns, d, 8, cudaMemcpyDeviceToHost);
        printf("%s M=%3d A=%s N=%3d: %.1f ns/MMA  (%.0f TFLOP/s chip-wide tf32)  %s\n", wi ? "warp-issue " : "lane-issue ", M,
               at ? "tmem" : "smem", N, double(ns) / n, 2.0 * M * N * 8 * n * 148 / (ns * 1e-9) / 1e12,
               e ? cudaGetErrorString(e) : "");
      }
  return 0;
}
