// Micro-benchmark: can a per-SM TMA bulk-copy ring stream HBM at full rate?
// Variants: chunk bytes, slots, contiguous-per-CTA vs interleaved chunk assignment.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2210_09147_b200/csrc/pt_ptx.cuh"
using namespace pt;

__device__ int g_stall_ns = 0, g_pf_mode = 0, g_pf_dist = 0, g_barrier = 0;
__device__ unsigned long long g_bar_cnt = 0;
template <int NSLOT>
__global__ void __launch_bounds__(288, 1) ring_kernel(const float* __restrict__ W, size_t total_bytes, int chunk_bytes,
                                                     int interleave, float* out, int use_policy) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + size_t(NSLOT) * chunk_bytes);
  uint64_t* empty = full + NSLOT;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < NSLOT; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 8); }
    fence_mbar_init();
  }
  __syncthreads();
  const size_t nchunks_total = total_bytes / chunk_bytes;
  size_t per_cta = nchunks_total / gridDim.x;
  // interleave == 2: the tick kernel's pattern. 2048x2048 fp32 layers, CTA c owns rows
  // [2048c/G, 2048(c+1)/G) of every layer, chunks of up to 4 rows (last one shorter).
  const int r0 = int(2048LL * blockIdx.x / gridDim.x), r1 = int(2048LL * (blockIdx.x + 1) / gridDim.x);
  const int rpc = chunk_bytes / 8192;
  const int cpl = (r1 - r0 + rpc - 1) / rpc;
  const size_t nlayers = total_bytes / (2048ull * 2048 * 4);
  if (interleave == 2) per_cta = nlayers * cpl;
  auto chunk_addr = [&](size_t i) -> const char* {
    if (interleave == 2) {
      size_t layer = i / cpl, k = i % cpl;
      return reinterpret_cast<const char*>(W) + layer * (2048ull * 2048 * 4) + size_t(r0 + rpc * k) * 8192;
    }
    size_t g = interleave ? (i * gridDim.x + blockIdx.x) : (blockIdx.x * per_cta + i);
    return reinterpret_cast<const char*>(W) + g * chunk_bytes;
  };
  auto chunk_len = [&](size_t i) -> int {
    if (interleave == 2) { int k = int(i % cpl); return min(rpc, r1 - r0 - rpc * k) * 8192; }
    return chunk_bytes;
  };
  if (warp == 8) {
    const int pfm = g_pf_mode, pfd = g_pf_dist;
    size_t pfi = 0;
    auto top = [&](size_t i) {
      while (pfi < per_cta && pfi < i + pfd) {
        if (pfm == 1) { if (lane == 0) prefetch_l2(chunk_addr(pfi), chunk_len(pfi)); }
        else if (pfm == 2) { const char* a = chunk_addr(pfi); for (int o = lane * 128; o < chunk_len(pfi); o += 4096) prefetch_line_l2(a + o); }
        ++pfi;
      }
    };
    {
      uint64_t pol = policy_evict_first();
      for (size_t i = 0; i < per_cta; ++i) {
        int slot = i % NSLOT;
        uint32_t use = i / NSLOT;
        if (pfm) top(i);
        if (use > 0) while (true) { int ok = lane == 0 ? mbar_try_wait(&empty[slot], (use - 1) & 1) : 0; ok = __shfl_sync(~0u, ok, 0); if (ok) break; if (pfm) top(i); }
        if (lane != 0) { __syncwarp(); continue; }
        const int len = chunk_len(i);
        mbar_arrive_expect_tx(&full[slot], len);
        if (use_policy)
          bulk_g2s(sm + size_t(slot) * chunk_bytes, chunk_addr(i), len, &full[slot], pol);
        else
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(smem_u32(sm + size_t(slot) * chunk_bytes)), "l"(chunk_addr(i)), "r"(len),
                       "r"(smem_u32(&full[slot])) : "memory");
        __syncwarp();
      }
    }
    return;
  }
  float acc = 0.f;
  for (size_t i = 0; i < per_cta; ++i) {
    int slot = i % NSLOT;
    while (!mbar_try_wait(&full[slot], (i / NSLOT) & 1)) {}
    const float4* b = reinterpret_cast<const float4*>(sm + size_t(slot) * chunk_bytes);
    const int len = chunk_len(i);
    for (int j = tid; j < len / 16; j += 256) { float4 v = b[j]; acc += v.x + v.y + v.z + v.w; }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
    if (interleave == 2 && (i % cpl) == cpl - 1 && g_stall_ns) {  // layer end: emulate the sync phase
      uint64_t t0 = globaltimer(); while (globaltimer() - t0 < uint64_t(g_stall_ns)) {}
    }
    if (interleave == 2 && (i % cpl) == cpl - 1 && g_barrier) {  // layer end: grid barrier (polling)
      asm volatile("bar.sync 1, 256;");
      const unsigned long long target = (unsigned long long)gridDim.x * (i / cpl + 1);
      if (tid == 0) {
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" :: "l"(&g_bar_cnt) : "memory");
        while (ld_acquire_gpu(&g_bar_cnt) < target) {}
      }
      asm volatile("bar.sync 1, 256;");
    }
  }
  if (acc == 12345.f) out[0] = acc;
}

__global__ void ldg_kernel(const float4* __restrict__ W, size_t n4, float* out) {
  float acc = 0.f;
  size_t stride = size_t(gridDim.x) * blockDim.x;
  size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n4; i += 4 * stride) {
    float4 a = __ldcs(W + i), b = __ldcs(W + i + stride), c = __ldcs(W + i + 2 * stride), d = __ldcs(W + i + 3 * stride);
    acc += a.x + b.y + c.z + d.w;
  }
  if (acc == 12345.f) out[0] = acc;
}

__global__ void copy_kernel(const float4* __restrict__ A, float4* __restrict__ B, size_t n4) {
  size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) B[i] = A[i];
}

template <int NSLOT>
float run_ring(const float* W, size_t bytes, int chunk, int inter, float* out, int pol) {
  size_t smem = size_t(NSLOT) * chunk + 2 * NSLOT * 8;
  cudaFuncSetAttribute(ring_kernel<NSLOT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 4; ++r) {
    cudaEventRecord(a);
    ring_kernel<NSLOT><<<148, 288, smem>>>(W, bytes, chunk, inter, out, pol);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (r) best = fminf(best, ms);
  }
  cudaError_t e = cudaGetLastError(); if (e) printf("err %s\n", cudaGetErrorString(e));
  return bytes / (best * 1e-3) / 1e9;
}

int main() {
  size_t bytes = size_t(148) * 64 * 32768 * 4;  // ~1.24 GB
  float *W, *out, *W2;
  cudaMalloc(&W, bytes); cudaMalloc(&W2, bytes); cudaMalloc(&out, 64);
  cudaMemset(W, 0, bytes);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  for (int r = 0; r < 3; ++r) { cudaEventRecord(a); ldg_kernel<<<148 * 4, 512>>>((float4*)W, bytes / 16, out); cudaEventRecord(b); cudaEventSynchronize(b); }
  cudaEventElapsedTime(&ms, a, b); printf("LDG stream read: %.0f GB/s\n", bytes / (ms * 1e-3) / 1e9);
  for (int r = 0; r < 3; ++r) { cudaEventRecord(a); copy_kernel<<<148 * 4, 512>>>((float4*)W, (float4*)W2, bytes / 16); cudaEventRecord(b); cudaEventSynchronize(b); }
  cudaEventElapsedTime(&ms, a, b); printf("copy (r+w): %.0f GB/s\n", 2 * bytes / (ms * 1e-3) / 1e9);
  size_t lbytes = 32ull * 2048 * 2048 * 4;
  for (int bar : {1}) {
    int z = 0; cudaMemcpyToSymbol(g_barrier, &bar, 4);
    auto runb = [&](auto kern, int nslot, int cb) {
      unsigned long long zz = 0;
      float best = 1e9;
      size_t smem = size_t(nslot) * cb + 2 * nslot * 8;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      for (int r = 0; r < 3; ++r) {
        cudaMemcpyToSymbol(g_bar_cnt, &zz, 8);
        cudaEventRecord(a); kern<<<148, 288, smem>>>(W, lbytes, cb, 2, out, 1); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); best = fminf(best, ms);
      }
      cudaError_t e = cudaGetLastError(); if (e) printf("err %s\n", cudaGetErrorString(e));
      printf("  ring %2d x %2dK = %3d KB: %.0f GB/s (%.2f us/layer)\n", nslot, cb / 1024, nslot * cb / 1024,
             lbytes / (best * 1e-3) / 1e9, best * 1e3 / 32);
    };
    printf("layered + grid barrier per layer:\n");
    for (int pfm : {0, 1, 2}) for (int pfd : {4, 8, 12, 20}) {
      if (pfm == 0 && pfd != 4) continue;
      cudaMemcpyToSymbol(g_pf_mode, &pfm, 4); cudaMemcpyToSymbol(g_pf_dist, &pfd, 4);
      printf(" pf_mode=%d dist=%d:", pfm, pfd);
      runb(ring_kernel<4>, 4, 32768);
    }
    { int zz0 = 0; cudaMemcpyToSymbol(g_pf_mode, &zz0, 4); }
    cudaMemcpyToSymbol(g_barrier, &z, 4); cudaMemcpyToSymbol(g_stall_ns, &z, 4);
  }
  for (int stall : {0}) for (int pfm : {0}) for (int pfd : {4}) {
    if (pfm == 0 && pfd != 4) continue;
    cudaMemcpyToSymbol(g_stall_ns, &stall, 4); cudaMemcpyToSymbol(g_pf_mode, &pfm, 4); cudaMemcpyToSymbol(g_pf_dist, &pfd, 4);
    printf("layered stall=%dns pf_mode=%d dist=%d: 5x32K %.0f GB/s\n", stall, pfm, pfd, run_ring<5>(W, lbytes, 32768, 2, out, 1) * 1.0);
  }
  { int z = 0; cudaMemcpyToSymbol(g_stall_ns, &z, 4); cudaMemcpyToSymbol(g_pf_mode, &z, 4); }
  for (int pol = 0; pol < 1; ++pol)
    for (int inter = 0; inter < 2; ++inter) {
      printf("pol=%d inter=%d  5x32K: %.0f  6x32K: %.0f  10x16K: %.0f  12x16K: %.0f  20x8K: %.0f  24x8K: %.0f GB/s\n", pol, inter,
             run_ring<5>(W, bytes, 32768, inter, out, pol), run_ring<6>(W, bytes, 32768, inter, out, pol),
             run_ring<10>(W, bytes, 16384, inter, out, pol), run_ring<12>(W, bytes, 16384, inter, out, pol),
             run_ring<20>(W, bytes, 8192, inter, out, pol), run_ring<24>(W, bytes, 8192, inter, out, pol));
    }
  return 0;
}
