// Micro-benchmark for the M=1 tick structure: 32 layers of 2048 x 2048 fp32 weights,
// streamed through a per-SM bulk-copy ring, with a grid-wide dependency (polling
// barrier) after every layer. Question: what limits HBM throughput under the per-layer
// dependency -- ring depth, row-to-CTA assignment (partition camping), chunk order?
//   mode 0: CTA c owns a contiguous row block, chunks of rpc contiguous rows (tick kernel)
//   mode 1: CTA c owns rows c, c+G, c+2G, ... (strided); a chunk = rpc separate row copies
//   mode 2: contiguous block, chunk order rotated by c
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dep_bench tools/dep_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2210_09147_b200/csrc/pt_ptx.cuh"
using namespace pt;

constexpr int WIDTH = 2048, ROWB = WIDTH * 4, NL = 32;
__device__ unsigned long long g_bar = 0;
__device__ unsigned long long g_flags[160 * 16];
__device__ unsigned long long g_ck[3][1024];  // CTA 0: per chunk issue, landed (seen by consumer), consumed  // barrier mode 2: one 128-B line per CTA
__device__ unsigned long long g_ev[148 * NL * 4];  // per CTA, layer: arrive, leave, first-chunk-ready, last-chunk-ready

__global__ void __launch_bounds__(288, 1) dep_kernel(const float* __restrict__ W, int nslot, int slot_bytes, int mode,
                                                    int barrier, int stall_ns, int maxfly, int pfl, float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + size_t(nslot) * slot_bytes);
  uint64_t* empty = full + nslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, G = gridDim.x, c = blockIdx.x;
  if (tid == 0) {
    for (int s = 0; s < nslot; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 8); }
    fence_mbar_init();
  }
  __syncthreads();
  const int rpc = slot_bytes / ROWB;
  // rows of this CTA
  int nrows;
  if (mode == 1) nrows = (WIDTH - c + G - 1) / G;
  else nrows = int(WIDTH * (c + 1LL) / G) - int(WIDTH * (long long)c / G);
  const int r0 = int(WIDTH * (long long)c / G);
  const int cpl = (nrows + rpc - 1) / rpc;
  auto row_of = [&](int k) { return mode == 1 ? c + G * k : r0 + k; };  // k-th own row
  auto chunk_k = [&](int j) { return mode == 2 ? (j + c) % cpl : j; };  // j-th chunk in walk order
  const int total = NL * cpl;
  if (warp == 8) {
    if (lane != 0) return;
    const uint64_t pol = policy_evict_first();
    for (int i = 0; i < total; ++i) {
      const int slot = i % nslot, use = i / nslot;
      if (use > 0) while (!mbar_try_wait(&empty[slot], (use - 1) & 1)) {}
      if (maxfly > 0 && i >= maxfly) {  // at most maxfly chunks in flight
        const int o = i - maxfly;
        while (!mbar_try_wait(&full[o % nslot], (o / nslot) & 1)) {}
      }
      const int layer = i / cpl, k0 = chunk_k(i % cpl) * rpc, nr = min(rpc, nrows - k0);
      if (pfl > 0 && (i % cpl) == 0 && layer + pfl < NL && mode == 0) {  // L2 prefetch of a whole later layer block
        const char* pb = reinterpret_cast<const char*>(W) + size_t(layer + pfl) * WIDTH * ROWB + size_t(r0) * ROWB;
        prefetch_l2(pb, uint32_t(nrows) * ROWB);
      }
      if (pfl > 0 && i == 0 && mode == 0)
        for (int q = 1; q < pfl && q < NL; ++q)
          prefetch_l2(reinterpret_cast<const char*>(W) + size_t(q) * WIDTH * ROWB + size_t(r0) * ROWB, uint32_t(nrows) * ROWB);
      if (c == 0 && i < 1024) g_ck[0][i] = globaltimer();
      mbar_arrive_expect_tx(&full[slot], uint32_t(nr) * ROWB);
      const char* base = reinterpret_cast<const char*>(W) + size_t(layer) * WIDTH * ROWB;
      char* dst = reinterpret_cast<char*>(sm + size_t(slot) * slot_bytes);
      if (mode == 1) {
        for (int r = 0; r < nr; ++r)
          bulk_g2s(dst + r * ROWB, base + size_t(row_of(k0 + r)) * ROWB, ROWB, &full[slot], pol);
      } else {
        bulk_g2s(dst, base + size_t(row_of(k0)) * ROWB, uint32_t(nr) * ROWB, &full[slot], pol);
      }
    }
    return;
  }
  float acc = 0.f;
  for (int i = 0; i < total; ++i) {
    const int slot = i % nslot;
    while (!mbar_try_wait(&full[slot], (i / nslot) & 1)) {}
    if (tid == 0 && c == 0 && i < 1024) g_ck[1][i] = globaltimer();
    if (tid == 0 && (i % cpl) == 0) g_ev[(c * NL + i / cpl) * 4 + 2] = globaltimer();
    if (tid == 0 && (i % cpl) == cpl - 1) g_ev[(c * NL + i / cpl) * 4 + 3] = globaltimer();
    const int k0 = chunk_k(i % cpl) * rpc, nr = min(rpc, nrows - k0);
    const float4* b = reinterpret_cast<const float4*>(sm + size_t(slot) * slot_bytes);
    for (int j = tid; j < nr * ROWB / 16; j += 256) { float4 v = b[j]; acc += v.x + v.y + v.z + v.w; }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
    if (tid == 0 && c == 0 && i < 1024) g_ck[2][i] = globaltimer();
    if ((i % cpl) == cpl - 1) {
      if (stall_ns) { uint64_t t0 = globaltimer(); while (globaltimer() - t0 < uint64_t(stall_ns)) {} }
      if (barrier) {
        asm volatile("bar.sync 1, 256;");
        if (tid == 0) g_ev[(c * NL + i / cpl) * 4 + 0] = globaltimer();
        const unsigned long long target = (unsigned long long)G * (i / cpl + 1);
        if (barrier == 2) {
          const unsigned long long want = i / cpl + 1;
          if (tid == 0) asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(&g_flags[c * 16]), "l"(want) : "memory");
          if (tid < G) {
            unsigned long long v;
            do { asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(&g_flags[tid * 16]) : "memory"); } while (v < want);
          }
          asm volatile("bar.sync 1, 256;");
          if (tid == 0) g_ev[(c * NL + i / cpl) * 4 + 1] = globaltimer();
        } else if (tid == 0) {
          asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(&g_bar) : "memory");
          while (ld_acquire_gpu(&g_bar) < target) {}
          g_ev[(c * NL + i / cpl) * 4 + 1] = globaltimer();
        }
        asm volatile("bar.sync 1, 256;");
      }
    }
  }
  if (acc == 12345.f) out[0] = acc;
}

int main() {
  const size_t bytes = size_t(NL) * WIDTH * ROWB;
  float *W, *out;
  cudaMalloc(&W, bytes);
  cudaMalloc(&out, 64);
  cudaMemset(W, 0, bytes);
  // flush buffer larger than L2
  char* flush;
  const size_t fb = 256ull << 20;
  cudaMalloc(&flush, fb);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](int nslot, int slot_kb, int mode, int barrier, int stall, int maxfly = 0, int pfl = 0) {
    const int sb = slot_kb * 1024;
    const size_t smem = size_t(nslot) * sb + 2 * nslot * 8;
    cudaFuncSetAttribute(dep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    float best = 1e9;
    for (int r = 0; r < 4; ++r) {
      unsigned long long z = 0;
      cudaMemcpyToSymbol(g_bar, &z, 8);
      static unsigned long long zf[160 * 16];
      cudaMemcpyToSymbol(g_flags, zf, sizeof(zf));
      cudaMemset(flush, r, fb);
      cudaEventRecord(a);
      dep_kernel<<<148, 288, smem>>>(W, nslot, sb, mode, barrier, stall, maxfly, pfl, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (r) best = fminf(best, ms);
    }
    cudaError_t e = cudaGetLastError();
    if (e) printf("err %s\n", cudaGetErrorString(e));
    printf("pfl %d mode %d barrier %d stall %4d ns maxfly %d ring %2d x %2d KB (%3d KB): %5.0f GB/s  %.2f us/layer\n", pfl, mode, barrier,
           stall, maxfly, nslot, slot_kb, nslot * slot_kb, bytes / (best * 1e-3) / 1e9, best * 1e3 / NL);
  };
  const int shapes[][3] = {{32, 4, 0}, {32, 6, 1}, {32, 6, 2}, {32, 6, 3}, {48, 4, 1}, {48, 4, 2}, {64, 3, 1},
                           {64, 3, 2}, {96, 2, 1}, {112, 2, 1}, {40, 5, 1}, {40, 5, 2}, {24, 8, 2}, {24, 8, 3}};
  for (int barrier : {2, 0})
    for (auto& sh : shapes) run(sh[1], sh[0], 0, barrier, 0, sh[2], 0);
  return 0;
}
