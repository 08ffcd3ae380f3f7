// Micro-benchmark: what does one dependent batch-1 step cost, and what bounds it?
// A chain of S steps over 2048 x 2048 fp32 weights (32 distinct layers, 537 MB > L2),
// one CTA per SM owning a row block, every CTA needing the previous step's result.
// Two step kinds, as in the tick:
//   F  z = W a for own rows; the output vector is all-gathered (every CTA polls all
//      2048 tagged words {value, step+1}).
//   B  g = W^T delta over own rows, for all 2048 columns; the per-CTA partials are
//      reduce-scattered (every CTA sums 148 tagged partials of its own rows).
// Weight supply:
//   ring      TMA bulk-copy ring (one producer thread), gated by the dependency
//   resident  this CTA's rows stay in smem (no HBM): the sync + compute floor
//   wb        every chunk is bulk-stored back to HBM as soon as it lands (before the
//             dependency: the deferred-update F step reads and writes each weight)
//   nodep     ring without the dependency (the ring's pure streaming rate)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/step_bench tools/step_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2210_09147_b200/csrc/pt_ptx.cuh"
using namespace pt;

constexpr int WD = 2048, ROWB = WD * 4, NL = 32;
constexpr int NCW = 8, NCT = 256, NRM = 16;  // consumer warps / threads, max rows per CTA

enum { K_F = 0, K_B = 1 };
enum { S_RING = 0, S_RES = 1, S_WB = 2, S_NODEP = 3 };

struct Args {
  const float* W;
  float* Wout;
  u64* vec;   // F: [4][WD] tagged outputs; B: [4][G][WD] tagged partials
  int nslot, slot_bytes, kind, supply, steps;
  u64* ev;    // per CTA per step: dep ready, chunks done, published
  int nev;
};

__device__ __forceinline__ float dot4(float4 a, float4 b) {
  return fmaf(a.w, b.w, fmaf(a.z, b.z, fmaf(a.y, b.y, a.x * b.x)));
}

// v[16] per lane -> lane l holds sum over the warp of v[l & 15] (16 shuffles)
__device__ __forceinline__ float transpose_reduce16(float (&v)[NRM]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int s = 8; s >= 1; s >>= 1) {
    const bool up = lane & s;
#pragma unroll
    for (int j = 0; j < s; ++j) {
      const float send = up ? v[j] : v[j + s];
      const float keep = up ? v[j + s] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 16);
}

__global__ void __launch_bounds__(288, 1) step_kernel(const __grid_constant__ Args A) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const int ring_bytes = A.nslot * A.slot_bytes;
  float* act = reinterpret_cast<float*>(sm + ring_bytes);  // [WD] F: input vector
  float* red = act + WD;                                     // [NCW][NRM]
  float* dlt = red + 16 * NRM;                               // [NRM] B: own delta
  float* pl = dlt + NRM;                                     // [NRM][NCT] F: per-lane row partials
  uint64_t* full = reinterpret_cast<uint64_t*>(pl + NRM * NCT);
  uint64_t* empty = full + A.nslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, G = gridDim.x, c = blockIdx.x;
  const int r0 = int((long long)WD * c / G), r1 = int((long long)WD * (c + 1) / G), nrows = r1 - r0;
  const int rpc = A.slot_bytes / ROWB;
  const int cpl = (nrows + rpc - 1) / rpc;  // chunks per step
  if (tid == 0) {
    for (int s = 0; s < A.nslot; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const bool resident = A.supply == S_RES;
  if (resident) {
    for (int j = tid; j < nrows * WD / 4; j += blockDim.x)
      reinterpret_cast<float4*>(sm)[j] = reinterpret_cast<const float4*>(A.W + size_t(r0) * WD)[j];
    __syncthreads();
  }
  if (warp == NCW) {
    if (lane != 0 || resident) return;
    const uint64_t pol = policy_evict_first();
    const int total = A.steps * cpl;
    for (int i = 0; i < total; ++i) {
      const int slot = i % A.nslot, use = i / A.nslot;
      if (use > 0) {
        while (!mbar_try_wait(&empty[slot], (use - 1) & 1)) {
        }
        if (A.supply == S_WB) bulk_wait_read_all();
      }
      const int s = i / cpl, k0 = (i % cpl) * rpc, nr = min(rpc, nrows - k0);
      const size_t off = size_t(s % NL) * WD * WD + size_t(r0 + k0) * WD;
      mbar_arrive_expect_tx(&full[slot], uint32_t(nr) * ROWB);
      bulk_g2s(sm + size_t(slot) * A.slot_bytes, A.W + off, uint32_t(nr) * ROWB, &full[slot], pol);
      const bool wbs = A.supply == S_WB && (A.kind != 2 || (s % 64) < 32);
      if (wbs) {
        // store the chunk back as soon as it has landed (the deferred update applies the
        // pending rank-1 step on arrival, before the dependency resolves)
        while (!mbar_try_wait(&full[slot], use & 1)) {
        }
        bulk_s2g(A.Wout + off, sm + size_t(slot) * A.slot_bytes, uint32_t(nr) * ROWB);
        bulk_commit();
      }
    }
    bulk_wait_all();
    return;
  }
  uint32_t chunk = 0;
  const int c0 = warp * 256 + lane * 4;  // this lane's 8 columns: c0..c0+3, c0+128..c0+131
  for (int s = 0; s < A.steps; ++s) {
    const uint32_t tag = uint32_t(s);
    // kind 2 = tick: 32 F steps (read + write back) then 32 B steps (read only)
    const bool kindF = A.kind == K_F || (A.kind == 2 && (s % 64) < 32);
    // ---------------------------------------------------------------- dependency
    const bool prevF = A.kind == 2 ? ((s + 63) % 64) < 32 : kindF;  // tick mode: the step before
    if (A.supply != S_NODEP && s > 0 && prevF == kindF) {
      if (kindF) {
        // all-gather: every thread issues its 4 pair loads, then checks
        const u64* src = A.vec + size_t(s & 3) * G * G * NRM;
        u64 v[8];
#pragma unroll
        for (int k = 0; k < 4; ++k) ld2_tv_gpu(src + tid * 2 + k * 512, v[2 * k], v[2 * k + 1]);
        // re-poll every stale pair together: one round trip per round, not one per pair
        for (;;) {
          bool stale = false;
#pragma unroll
          for (int k = 0; k < 4; ++k) stale |= tv_tag(v[2 * k]) != tag || tv_tag(v[2 * k + 1]) != tag;
          if (!stale) break;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (tv_tag(v[2 * k]) != tag || tv_tag(v[2 * k + 1]) != tag)
              ld2_tv_gpu(src + tid * 2 + k * 512, v[2 * k], v[2 * k + 1]);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          act[tid * 2 + k * 512] = tv_val(v[2 * k]) * 1e-3f + 1.f;
          act[tid * 2 + k * 512 + 1] = tv_val(v[2 * k + 1]) * 1e-3f + 1.f;
        }
      } else {
        // reduce-scatter over the blocked partials [consumer][producer][NRM]: thread
        // (row = tid & 15, group = tid >> 4) sums producers group, group+16, ...
        const u64* src = A.vec + size_t(s & 3) * G * G * NRM + size_t(c) * G * NRM;
        const int row = tid & 15, grp = tid >> 4;
        float sum = 0.f;
        if (row < nrows) {
          u64 v[10];
#pragma unroll
          for (int j = 0; j < 10; ++j) {
            const int pc = grp + 16 * j;
            v[j] = pc < G ? ld_tv_gpu(src + size_t(pc) * NRM + row) : pack_tv(0.f, tag);
          }
          for (;;) {
            bool stale = false;
#pragma unroll
            for (int j = 0; j < 10; ++j) stale |= tv_tag(v[j]) != tag;
            if (!stale) break;
#pragma unroll
            for (int j = 0; j < 10; ++j)
              if (tv_tag(v[j]) != tag) v[j] = ld_tv_gpu(src + size_t(grp + 16 * j) * NRM + row);
          }
#pragma unroll
          for (int j = 0; j < 10; ++j) sum += tv_val(v[j]);
        }
        red[grp * NRM + row] = sum;
        cons_sync(NCT);
        if (tid < nrows) {
          float d = 0.f;
          for (int g2 = 0; g2 < 16; ++g2) d += red[g2 * NRM + tid];
          dlt[tid] = d * 1e-3f + 1.f;
        }
      }
    } else if (s == 0 || prevF != kindF) {
      for (int j = tid; j < WD; j += NCT) act[j] = 1.f;
      if (tid < NRM) dlt[tid] = 1.f;
    }
    cons_sync(NCT);
    if (tid == 0 && A.ev && s < A.nev) A.ev[(size_t(c) * A.nev + s) * 3 + 0] = globaltimer();
    // ---------------------------------------------------------------- chunks
    float4 g0 = make_float4(0.f, 0.f, 0.f, 0.f), g1 = g0;
    const float4 a0 = lds4(act + c0), a1 = lds4(act + c0 + 128);
    for (int k = 0; k < cpl; ++k) {
      const int k0 = k * rpc, nr = min(rpc, nrows - k0);
      const float* wb;
      if (resident) {
        wb = reinterpret_cast<const float*>(sm) + size_t(k0) * WD;
      } else {
        const int slot = chunk % A.nslot;
        while (!mbar_try_wait(&full[slot], (chunk / A.nslot) & 1)) {
        }
        wb = reinterpret_cast<const float*>(sm + size_t(slot) * A.slot_bytes);
      }
      if (kindF) {
        // per-lane row partials go to smem [row][warp][lane]; reduced once per step
        for (int r = 0; r < nr; ++r)
          pl[(k0 + r) * NCT + tid] = dot4(lds4(wb + r * WD + c0), a0) + dot4(lds4(wb + r * WD + c0 + 128), a1);
      } else {
        for (int r = 0; r < nr; ++r) {
          {
            const float d = dlt[k0 + r];
            const float4 w0 = lds4(wb + r * WD + c0), w1 = lds4(wb + r * WD + c0 + 128);
            g0.x = fmaf(w0.x, d, g0.x); g0.y = fmaf(w0.y, d, g0.y); g0.z = fmaf(w0.z, d, g0.z); g0.w = fmaf(w0.w, d, g0.w);
            g1.x = fmaf(w1.x, d, g1.x); g1.y = fmaf(w1.y, d, g1.y); g1.z = fmaf(w1.z, d, g1.z); g1.w = fmaf(w1.w, d, g1.w);
          }
        }
      }
      if (!resident) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[chunk % A.nslot]);
        ++chunk;
      }
    }
    if (tid == 0 && A.ev && s < A.nev) A.ev[(size_t(c) * A.nev + s) * 3 + 1] = globaltimer();
    // ---------------------------------------------------------------- publish
    if (kindF) {
      cons_sync(NCT);
      for (int rr = warp; rr < nrows; rr += NCW) {
        float z = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) z += pl[rr * NCT + lane + 32 * j];
        z = warp_sum(z);
        if (lane == 0) red[rr] = z;
      }
      cons_sync(NCT);
      if (tid < nrows) {
        const float z = red[tid];
        st_tv_gpu(A.vec + size_t((s + 1) & 3) * G * G * NRM + r0 + tid, pack_tv(z, tag + 1));
      }
    } else {
      // blocked partials: column col goes to its owner's block [owner][c][col - r0(owner)]
      u64* dst = A.vec + size_t((s + 1) & 3) * G * G * NRM;
      const float gv[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int col = c0 + (j & 3) + (j >> 2) * 128;
        const int own = ((col + 1) * G - 1) / WD;
        const int o0 = int((long long)WD * own / G);
        st_tv_gpu(dst + (size_t(own) * G + c) * NRM + (col - o0), pack_tv(gv[j], tag + 1));
      }
    }
    cons_sync(NCT);  // red / dlt are rewritten by the next step
    if (tid == 0 && A.ev && s < A.nev) A.ev[(size_t(c) * A.nev + s) * 3 + 2] = globaltimer();
  }
}

int main(int argc, char** argv) {
  const int steps = 256;
  const size_t wbytes = size_t(NL) * WD * WD * 4;
  float *W, *Wout;
  u64 *vec, *ev;
  cudaMalloc(&W, wbytes);
  cudaMalloc(&Wout, wbytes);
  const size_t vec_bytes = size_t(4) * 148 * 148 * NRM * 8;
  cudaMalloc(&vec, vec_bytes);
  const int nev = 64;
  cudaMalloc(&ev, size_t(148) * nev * 3 * 8);
  cudaMemset(W, 0, wbytes);
  char* flush;
  const size_t fb = 256ull << 20;
  cudaMalloc(&flush, fb);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* kname[] = {"F", "B", "T"};
  const char* sname[] = {"ring", "resident", "wb", "nodep"};
  auto run = [&](int kind, int supply, int nslot, int slot_kb, bool dump) {
    Args A;
    A.W = W;
    A.Wout = Wout;
    A.vec = vec;
    A.nslot = nslot;
    A.slot_bytes = slot_kb * 1024;
    A.kind = kind;
    A.supply = supply;
    A.steps = steps;
    A.ev = ev;
    A.nev = nev;
    const size_t smem = size_t(nslot) * A.slot_bytes + (WD + 16 * NRM + NRM + NRM * NCT) * 4 + 2 * nslot * 8 + 64;
    if (smem > 227 * 1024) return;
    cudaFuncSetAttribute(step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaMemset(vec, 0, vec_bytes);
      cudaMemset(flush, r, fb);
      cudaEventRecord(e0);
      step_kernel<<<148, 288, smem>>>(A);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r) best = fminf(best, ms);
    }
    cudaError_t e = cudaGetLastError();
    if (e) printf("err %s\n", cudaGetErrorString(e));
    const double us = best * 1e3 / steps;
    const double gbs = (supply == S_RES ? 0.0 : double(WD) * WD * 4 * (supply == S_WB ? 2 : 1)) / (us * 1e-6) / 1e9;
    printf("%s %-8s ring %2d x %2d KB: %6.2f us/step %6.0f GB/s", kname[kind], sname[supply], nslot, slot_kb, us, gbs);
    if (dump) {
      static unsigned long long h[148 * 64 * 3];
      cudaMemcpy(h, ev, sizeof(h), cudaMemcpyDeviceToHost);
      double sp = 0, cmp = 0, pub = 0, lag = 0;
      int n = 0;
      for (int s = 32; s < 63; ++s) {
        unsigned long long dmin = ~0ull, dmax = 0, emax = 0, nmin = ~0ull;
        double cm = 0, pb = 0;
        for (int c = 0; c < 148; ++c) {
          const unsigned long long* q = h + (size_t(c) * 64 + s) * 3;
          dmin = q[0] < dmin ? q[0] : dmin;
          dmax = q[0] > dmax ? q[0] : dmax;
          emax = q[2] > emax ? q[2] : emax;
          cm += double(q[1] - q[0]);
          pb += double(q[2] - q[1]);
          const unsigned long long* q2 = h + (size_t(c) * 64 + s + 1) * 3;
          nmin = q2[0] < nmin ? q2[0] : nmin;
        }
        sp += double(dmax - dmin);
        cmp += cm / 148;
        pub += pb / 148;
        lag += double(nmin) - double(emax);
        ++n;
      }
      printf("  | ready spread %.2f, chunks %.2f, publish %.2f, last publish->first ready %.2f us", sp / n / 1e3,
             cmp / n / 1e3, pub / n / 1e3, lag / n / 1e3);
    }
    printf("\n");
  };
  run(2, S_WB, 3, 64, true);
  run(2, S_WB, 6, 32, true);
  run(2, S_WB, 1, 192, true);
  run(2, S_WB, 2, 96, true);
  for (int kind : {K_F, K_B}) {
    run(kind, S_RES, 4, 32, true);
    const int shapes[][2] = {{4, 32}, {6, 32}, {3, 64}, {2, 96}, {1, 192}};
    for (int supply : {S_RING, S_NODEP, S_WB})
      for (auto& s : shapes) run(kind, supply, s[0], s[1], supply != S_NODEP && (s[0] == 4 || s[0] == 6 || s[0] == 3));
  }
  return 0;
}
