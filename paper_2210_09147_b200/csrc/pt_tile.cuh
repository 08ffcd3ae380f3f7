// pt_tile.cuh: the micro-batch (M >= 16) PARTIME tick kernel on the tcgen05 tensor cores.
//
// Same tick contract as pt::tick_kernel (
// PAPER.md Alg. 1, Eqs. 6-10), different execution: at M = 16 a dense layer is a real
// contraction (8 flop/B), so each step is a swap-AB GEMM on the tensor core with the
// weights as the 128-row A operand and the micro-batch as N:
//   F_i : Z[r][m]  = sum_c W[r][c] a[m][c]   A = W  tile, K-major SWIZZLE_128B (TMA)
//   B_i : G[c][m]  = sum_r W[r][c] d[m][r]   A = W^T tile, MN-major SWIZZLE_128B_BASE32B
//                                             (TMA, the same row-major weights, no transpose)
//         W[r][c] -= lr sum_m d[m][r] a[m][c] fused SIMT epilogue on the same smem tile,
//                                             written back by TMA store
// fp32 parity: 3xTF32 (hi*hi + hi*lo + lo*hi). The SIMT warps split every tile into
// hi = tf32(w) (in place) and lo = w - hi (second buffer); the update rebuilds w = hi + lo
// exactly before applying the SGD step.
//
// Work split (one CTA per SM, G <= 148, cooperative launch):
//   F step of a layer [n_out x n_in]: units (128-row block, column quarter); CTA c takes
//   units c, c+G, ...; a unit streams 64-column chunks (two 32 KB TMA boxes).
//   B step: units (128-column block, row quarter), 64-row chunks (four 8 KB boxes).
//   Each unit leaves a partial (over its quarter) in TMEM; the 4 partials are summed in a
//   fixed order by a distributed finalize after a grid barrier (bias, activation, loss,
//   delta, stage exchange), then a second grid barrier publishes the result. All
//   reductions are fixed-order: runs are bitwise reproducible.
// Warp roles: warp 0 = TMA producer (runs ahead across steps and ticks, stores updated
// tiles back), warp 1 = MMA issuer (one thread), warps 2..9 = SIMT (split, operand
// staging, TMEM epilogue, update, finalize, grid barrier).
// Stages may live on other GPUs/processes: their plain fp32 slots sit in an IPC-exported
// tile comm block (TileComm) with tick counters (see partime_capi.cu).
#pragma once
#include "pt_kernels.cuh"
#include "pt_tc.cuh"

namespace pt {

constexpr int T_THREADS = 320;
constexpr int T_SIMT0 = 64;            // first SIMT thread
constexpr int T_NS = 256;              // SIMT threads
constexpr int T_SLOT_FLOATS = 8192;
constexpr int T_CK = 64;               // F: chunk columns; B: chunk rows
#ifndef PT_TQ
#define PT_TQ 4
#endif
constexpr int T_Q = PT_TQ;             // quarters (columns in F, rows in B)
constexpr int T_NACC = 1;              // independent accumulators per unit (K-step % T_NACC)
constexpr int T_TMEM_COLS = 512;
// Per micro-batch size TM (16, 32 or 64; the batch is the MMA's N side, so a larger TM issues
// the same F/B MMAs with a larger N): ring slots, operand / lo-tile buffers in flight (NB),
// update-product buffers (NUB), and the TMEM plan = two unit accumulators of 2 TM columns,
// NB 64-column lo tiles, NUB 128-column update products.
// build-time overrides of the per-size plan, digits (ring slots, NB, NUB) (tools/variants experiments);
// Adam (OPT = 1) holds a ring slot longer per backward chunk and runs best one slot shallower
#ifndef PT_T16_PLAN
#define PT_T16_PLAN 432
#endif
#ifndef PT_T32_PLAN
#define PT_T32_PLAN 322
#endif
#ifndef PT_T64_PLAN
#define PT_T64_PLAN 211
#endif
#ifndef PT_T16_PLAN_ADAM
#define PT_T16_PLAN_ADAM 332
#endif
#ifndef PT_T32_PLAN_ADAM
#define PT_T32_PLAN_ADAM 222
#endif
#ifndef PT_T64_PLAN_ADAM
#define PT_T64_PLAN_ADAM 211
#endif
template <int TM, int OPT = 0>
struct TCfg {
  static constexpr int plan = OPT == 1 ? (TM == 16 ? PT_T16_PLAN_ADAM : TM == 32 ? PT_T32_PLAN_ADAM : PT_T64_PLAN_ADAM)
                                       : (TM == 16 ? PT_T16_PLAN : TM == 32 ? PT_T32_PLAN : PT_T64_PLAN);
  static constexpr int NSLOT = plan / 100;     // weight ring slots of 32 KB
  static constexpr int NB = plan / 10 % 10;    // chunks in flight between SIMT and MMA
  static constexpr int NUB = plan % 10;        // update-product buffers
  static constexpr int ACC_COLS = 2 * T_NACC * 2 * TM;
  static constexpr int LO_COL = ACC_COLS;
  static constexpr int UPD_COL = ACC_COLS + NB * T_CK;
  // dynamic shared memory: alignment slack, ring, operands (hi, lo), update operands,
  // reduction scratch (TM floats), mbarriers, TMEM address
  static constexpr int smem_bytes() {
    return 1024 + NSLOT * T_SLOT_FLOATS * 4 + NB * 2 * TM * T_CK * 4 + NB * 2 * T_CK * TM * 4 + 2 * 128 * TM * 4 +
           TM * 4 + (3 * NSLOT + 5 * NB + 4) * 8 + 16;
  }
};
template <int TM, int OPT>
constexpr bool tcfg_fits() {
  using C = TCfg<TM, OPT>;
  return C::UPD_COL + C::NUB * 128 <= T_TMEM_COLS && C::smem_bytes() <= 227 * 1024;
}
static_assert(tcfg_fits<16, 0>() && tcfg_fits<32, 0>() && tcfg_fits<64, 0>() && tcfg_fits<16, 1>() &&
                  tcfg_fits<32, 1>() && tcfg_fits<64, 1>(),
              "tile kernel TMEM / shared-memory plan");
constexpr int T_DTS = 24;              // dT row stride (floats): conflict-free staging, 16-B rows

struct TLayer {
  const CUtensorMap* tmf;  // box [128 rows][32 cols], SWIZZLE_128B
  const CUtensorMap* tmb;  // box [64 rows][32 cols], SWIZZLE_128B_ATOM_32B
  float* b;
  float *mW, *vW, *mb, *vb;  // Adam moments (m, v blocked like W: [n_out/128][n_in/64][128][64]); null for SGD
  int ld;
  int n_in, n_out, act;
  int a_in, a_out;  // offsets (floats) of a_i, a_{i+1} in a stage cache slot ([M][n] each)
};

struct TStage {
  int h, first, k, n0, nk;
  float* cache[2];       // a_0 (private copy of the stage input) .. a_k, per tick parity
  float* inslot[2];      // [M][n0], written by the upstream stage
  float* gslot[2];       // [M][nk], written by the downstream stage
  float* down_inslot[2]; // downstream stage's inslot (h < D)
  float* up_gslot[2];    // upstream stage's gslot (h > 1)
  // neighbour in another process (one stage per GPU, CUDA IPC over NVLink): the grid
  // barriers do not order its accesses, so tick counters do (TileComm in partime_capi.cu)
  int up_remote, down_remote;
  u64* in_ready;         // own: inslot ticks published by upstream
  u64* g_ready;          // own: gslot ticks published by downstream
  u64* act_credit;       // own: inslot ticks downstream has finished reading
  u64* g_credit;         // own: gslot ticks upstream has finished reading
  u64* peer_in_ready;    // downstream's in_ready
  u64* peer_g_credit;    // downstream's g_credit
  u64* peer_g_ready;     // upstream's g_ready
  u64* peer_act_credit;  // upstream's act_credit
};

struct TParams {
  const TStage* stages;
  const TLayer* layers;
  int n_stages, M, D, learn, act_delay, F, G;
  float lr;
  int opt, loss, Fy;         // optimizer (0 SGD, 1 Adam), loss (0 MSE, 1 softmax-CE), target width
  float b1, b2, eps, omb1, omb2;  // Adam, as in pt::Params
  double b1d, b2d;
  float* ce;                 // softmax-CE: per-CTA (max, sum exp) partials [G][M][2]
  long long* bad_target;     // first sample whose class index is not in [0, F)
  const float* xs;  // [n][M][ldx]
  int ldx;
  const float* ys;  // [n][M][F]
  const float* yhist;
  int yh;
  float* outs;       // [n][M][F]
  float* loss_part;  // [n][G]
  long long t0;
  int n;
  float* part;   // [T_Q][M][max_n] unit partials
  float* delta;  // [M][max_n] delta of the current B layer
  int max_n;
  u64* gbar;     // grid barrier counter (monotonic)
  u64* wbar;     // per-tick "weights written back" counter (monotonic)
  u64 gbar_base, wbar_base;
  int* status;
  unsigned long long timeout_ns;
  u64* trace;  // diagnostics: (code << 56) | globaltimer of SIMT thread 0 of CTA trace_cta
  int trace_cap, trace_cta;
  int jitter, jitter_mask;  // diagnostics: random sleeps of up to `jitter` ns at every trace
                            // point of every role on 1 in (jitter_mask + 1) calls (race detector)
};

// SIMT group A thread 0 writes [0, cap/4), group B thread 0 [cap/4, cap/2), the MMA
// thread [cap/2, 3cap/4), the producer [3cap/4, cap)
__device__ __forceinline__ void t_jitter(const TParams& P, int code) {
  uint32_t x = uint32_t(globaltimer()) ^ (blockIdx.x * 0x9E3779B9u) ^ ((threadIdx.x >> 5) * 0x85EBCA6Bu) ^
               (uint32_t(code) * 0xC2B2AE35u);
  x ^= x >> 16;
  x *= 0x7FEB352Du;
  x ^= x >> 15;
  if ((x & uint32_t(P.jitter_mask)) == 0) {
    const uint64_t t0 = globaltimer(), d = (x >> 8) % uint32_t(P.jitter);
    while (globaltimer() - t0 < d) __nanosleep(1000);
  }
}

__device__ __forceinline__ void t_trace(const TParams& P, int& idx, int code) {
#ifdef PT_JITTER_BUILD
  if (P.jitter > 0) t_jitter(P, code);
#endif
  if (P.trace == nullptr || blockIdx.x != P.trace_cta) return;
  const int tid = threadIdx.x, q = P.trace_cap / 4;
  int lo;
  if (tid == T_SIMT0) lo = 0;
  else if (tid == T_SIMT0 + 128) lo = q;
  else if (tid == 32) lo = 2 * q;
  else if (tid == 0) lo = 3 * q;
  else return;
  if (idx < q) P.trace[lo + idx++] = (u64(code) << 56) | (globaltimer() & 0x00FFFFFFFFFFFFFFull);
}

// ------------------------------------------------------------------ schedule
// The producer, the MMA issuer and the SIMT warps walk the same sequence of
// (tick, stage, step, unit, chunk); chunk j uses ring slot j % C::NSLOT and operand /
// lo buffer j % 2.
struct TStep {
  int L;        // layer index
  bool fwd;
  int nunits, nchunks;
};
__device__ __forceinline__ TStep t_step(const TParams& P, const TStage& S, int st) {
  TStep s;
  s.fwd = st < S.k;
  const int i = s.fwd ? st : 2 * S.k - 1 - st;
  s.L = S.first + i;
  const TLayer& L = P.layers[s.L];
  if (s.fwd) {
    s.nunits = (L.n_out / 128) * T_Q;
    s.nchunks = L.n_in / T_Q / T_CK;
  } else {
    s.nunits = (L.n_in / 128) * T_Q;
    s.nchunks = L.n_out / T_Q / T_CK;
  }
  return s;
}
__device__ __forceinline__ int t_nsteps(const TParams& P, const TStage& S) { return P.learn ? 2 * S.k : S.k; }
__device__ __forceinline__ bool t_upd(const TParams& P, long long t, int h) {
  return P.learn && P.lr != 0.f && t >= 2LL * P.D - h - 1;  // warm-up gate SPEC.md:254
}

// --------------------------------------------------------------- small helpers
__device__ __forceinline__ bool t_watch(const TParams& P, uint64_t t_start) {
  if (ld_volatile_s32(P.status) != ST_OK) return true;
  if (globaltimer() - t_start > P.timeout_ns) {
    atomicCAS(P.status, ST_OK, ST_TIMEOUT);
    return true;
  }
  return false;
}
// one SIMT thread per CTA waits until a (possibly remote) tick counter reaches `target`
__device__ void t_wait_cnt(const TParams& P, const u64* p, u64 target) {
  if (threadIdx.x == T_SIMT0 + 0 && target > 0) {
    if (ld_acquire_sys(p) < target) {
      const uint64_t t0 = globaltimer();
      for (unsigned it = 1;; ++it) {
        if (ld_acquire_sys(p) >= target) break;
        if ((it & 63u) == 0 && t_watch(P, t0)) break;
      }
    }
  }
}

__device__ __forceinline__ void t_wait(uint64_t* bar, uint32_t parity, const TParams& P) {
  if (mbar_try_wait(bar, parity)) return;
  const uint64_t t0 = globaltimer();
  while (!mbar_try_wait(bar, parity))
    if (t_watch(P, t0)) return;
}
__device__ __forceinline__ void simt_sync() { asm volatile("bar.sync 1, %0;" ::"n"(T_NS) : "memory"); }
// SIMT group A (warps 2-5: operands, lo tiles, accumulator epilogue) and group B (warps 6-9:
// SGD write-back of backward tiles); each covers the four TMEM lane quarters once
constexpr int T_GRP = T_NS / 2;
__device__ __forceinline__ void grp_sync(int g) {
  if (g == 0) asm volatile("bar.sync 2, %0;" ::"n"(T_GRP) : "memory");
  else asm volatile("bar.sync 3, %0;" ::"n"(T_GRP) : "memory");
}
__device__ __forceinline__ float t_ld(const float* p) { return __ldcg(p); }
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

// grid barrier among the SIMT groups of all CTAs (counter never reset: target = G * k)
__device__ void t_grid_sync(const TParams& P, u64& gen) {
  simt_sync();
  ++gen;
  if (threadIdx.x == T_SIMT0) {
    red_release_gpu(P.gbar, 1);
    const u64 target = P.gbar_base + u64(P.G) * gen;
    if (ld_acquire_gpu(P.gbar) < target) {
      const uint64_t t0 = globaltimer();
      for (unsigned it = 1;; ++it) {
        if (ld_acquire_gpu(P.gbar) >= target) break;
        if ((it & 63u) == 0 && t_watch(P, t0)) break;
      }
    }
  }
  simt_sync();
}

struct TSmem {
  float* ring;      // C::NSLOT x 32 KB (1024-B aligned)
  float* opnd;      // 2 x (hi, lo) x [M][64] no-swizzle K-major
  float* dop;       // B: update MMA B operand [delta_hi; delta_lo]^T per chunk, [2][128][16]
  float* aop;       // B: update MMA A operand a^T (hi, lo) of the unit's 128 columns, [2][128][16]
  float* red;       // TM floats
  uint64_t* full;   // [C::NSLOT]
  uint64_t* sfree;  // [C::NSLOT] forward chunk in the slot consumed (MMA commit)
  uint64_t* bfree;  // [C::NSLOT] backward chunk in the slot updated in place (4 write-back warps)
  uint64_t* opnd_rdy; // [2] operand chunk staged
  uint64_t* prep;   // [C::NB] lo tile written (group A; the whole tile in B, K half 0 in F)
  uint64_t* prep2;  // [C::NB] forward chunks: K half 1 of the lo tile written (group B)
  uint64_t* mhi;    // [2] hi MMAs of the chunk done (raw tile no longer read)
  uint64_t* mdone;  // [2] all MMAs of the chunk done
  uint64_t* afree;  // [2] accumulator read by the epilogue
  uint64_t* applied;  // [2] update product of a backward chunk consumed (TMEM buffer free)
  uint32_t* tmem;
};

// ------------------------------------------------------------------ producer
template <int TM, int OPT>
__device__ void t_producer(const TParams& P, const TSmem& sm) {
  using C = TCfg<TM, OPT>;
  const int c = blockIdx.x, G = P.G;
  uint32_t j = 0;
  for (int s = 0; s < P.n_stages; ++s)
    for (int i = P.stages[s].first; i < P.stages[s].first + P.stages[s].k; ++i) {
      tma_fence_desc_acquire(P.layers[i].tmf);
      tma_fence_desc_acquire(P.layers[i].tmb);
    }
  // per slot: kind of the chunk it holds (1 forward: released by the MMA commit on sfree,
  // 2 backward: released by the 4 write-back warps on bfree), completions consumed, and a
  // pending write-back (layer, row, col) of an updated backward tile
  int kind[C::NSLOT];
  uint32_t fcnt[C::NSLOT], bcnt[C::NSLOT];
  int pend_l[C::NSLOT], pend_r[C::NSLOT], pend_c[C::NSLOT];
  bool pend[C::NSLOT];
  for (int s = 0; s < C::NSLOT; ++s) {
    pend[s] = false;
    kind[s] = 0;
    fcnt[s] = bcnt[s] = 0;
  }
  bool dead = false;
  int tr = 0;
  auto release = [&](int s) {
    if (kind[s] == 1) t_wait(&sm.sfree[s], fcnt[s]++ & 1, P);
    else if (kind[s] == 2) t_wait(&sm.bfree[s], bcnt[s]++ & 1, P);
    kind[s] = 0;
  };
  auto flush = [&](int s) {
    if (!pend[s]) return;
    release(s);
    const CUtensorMap* tm = P.layers[pend_l[s]].tmb;
    float* base = sm.ring + size_t(s) * T_SLOT_FLOATS;
    for (int b = 0; b < 4; ++b) {
      const int cc = pend_c[s] + 32 * b, rr = pend_r[s];
      tma_store_4d(tm, base + b * 2048, cc & 63, rr & 127, cc >> 6, rr >> 7);
    }
    pend[s] = false;
  };
  for (int ti = 0; ti < P.n && !dead; ++ti) {
    const long long t = P.t0 + ti;
    if (P.learn && ti > 0) {
      // weights of tick t-1 are written back by every CTA before any tile of tick t is read
      const u64 target = P.wbar_base + u64(G) * u64(ti);
      const uint64_t t0 = globaltimer();
      while (ld_acquire_gpu(P.wbar) < target)
        if (t_watch(P, t0)) {
          dead = true;
          break;
        }
      fence_proxy_async_global();
    }
    for (int s = 0; s < P.n_stages && !dead; ++s) {
      const TStage& S = P.stages[s];
      const bool upd = t_upd(P, t, S.h);
      for (int st = 0; st < t_nsteps(P, S); ++st) {
        const TStep sp = t_step(P, S, st);
        const TLayer& L = P.layers[sp.L];
        for (int u = c; u < sp.nunits; u += G) {
          const int blk = u / T_Q, q = u % T_Q;
          for (int ch = 0; ch < sp.nchunks; ++ch, ++j) {
            const int slot = j % C::NSLOT;
            if (pend[slot]) {
              flush(slot);
              bulk_commit();
              bulk_wait_read_all();
            } else {
              release(slot);
            }
            kind[slot] = sp.fwd ? 1 : 2;
            float* dst = sm.ring + size_t(slot) * T_SLOT_FLOATS;
            t_trace(P, tr, 30);
            mbar_arrive_expect_tx(&sm.full[slot], T_SLOT_FLOATS * 4);
            if (sp.fwd) {
              const int r0 = blk * 128, c0 = q * (L.n_in / T_Q) + ch * T_CK;
              // blocked weights: coordinates {column in block, row in block, column block, row block}
              tma_load_4d(dst, L.tmf, c0 & 63, 0, c0 >> 6, r0 >> 7, &sm.full[slot]);
              tma_load_4d(dst + 4096, L.tmf, (c0 + 32) & 63, 0, (c0 + 32) >> 6, r0 >> 7, &sm.full[slot]);
            } else {
              const int c0 = blk * 128, r0 = q * (L.n_out / T_Q) + ch * T_CK;
              for (int b = 0; b < 4; ++b) {
                const int cc = c0 + 32 * b;
                tma_load_4d(dst + b * 2048, L.tmb, cc & 63, r0 & 127, cc >> 6, r0 >> 7, &sm.full[slot]);
              }
              if (upd) {
                if (L.mW) {
                  // Adam: pull this chunk's moments into L2 now, a ring's depth before the
                  // write-back group's update reads them (rows r0.. of two 128 x 64 blocks:
                  // 16 KB contiguous each)
                  const size_t o = (size_t(r0 >> 7) * (L.n_in >> 6) + (c0 >> 6)) * 8192 + size_t(r0 & 127) * 64;
                  prefetch_l2(L.mW + o, 16384);
                  prefetch_l2(L.mW + o + 8192, 16384);
                  prefetch_l2(L.vW + o, 16384);
                  prefetch_l2(L.vW + o + 8192, 16384);
                }
                pend[slot] = true;
                pend_l[slot] = sp.L;
                pend_r[slot] = r0;
                pend_c[slot] = c0;
              }
            }
            if (ld_volatile_s32(P.status) != ST_OK) dead = true;
          }
        }
      }
    }
    if (P.learn) {
      // end of tick: write back every updated tile still in the ring, then publish
      for (uint32_t k = 0; k < C::NSLOT; ++k) flush(int((j + k) % C::NSLOT));
      bulk_commit();
      bulk_wait_all();
      fence_proxy_async_global();
      red_release_gpu(P.wbar, 1);
    }
  }
}

// ------------------------------------------------------------------ MMA issuer
template <int TM, int OPT>
__device__ void t_mma(const TParams& P, const TSmem& sm, uint32_t tbase) {
  using C = TCfg<TM, OPT>;
  // Per K-step two MMAs: hi(W) x [a_hi; a_lo] (N = 2M) and lo(W) x a_hi (N = M), both into
  // the unit accumulator: columns [0, M) collect hi*a_hi + lo*a_hi, [M, 2M) hi*a_lo.
  // The hi MMAs read the raw TMA tile (the tensor core uses its top 19 bits = tf32(w)),
  // so they start as soon as the tile lands; the lo MMAs wait for the SIMT split.
  const int c = blockIdx.x, G = P.G, M = P.M;
  uint32_t j = 0, uc = 0, bj = 0, fj = 0;  // chunk, unit, backward-chunk, forward-chunk counters
  int tr = 0;
  for (int ti = 0; ti < P.n; ++ti) {
    for (int s = 0; s < P.n_stages; ++s) {
      const TStage& S = P.stages[s];
      for (int st = 0; st < t_nsteps(P, S); ++st) {
        const TStep sp = t_step(P, S, st);
        const uint32_t id2 = tc_idesc_tf32(128, 2 * M, !sp.fwd, false);
        const uint32_t id1 = tc_idesc_tf32(128, M, false, false);  // A = lo tile in TMEM, K-major
        const uint32_t idu2 = tc_idesc_tf32(128, 2 * T_CK, false, false), idu1 = tc_idesc_tf32(128, T_CK, false, false);
        const bool upd = t_upd(P, P.t0 + ti, S.h);
        for (int u = c; u < sp.nunits; u += G, ++uc) {
          const uint32_t acc = tbase + (uc & 1) * uint32_t(T_NACC * 2 * M);
          if (uc >= 2) t_wait(&sm.afree[uc & 1], ((uc - 2) >> 1) & 1, P);
          for (int ch = 0; ch < sp.nchunks; ++ch, ++j) {
            const int slot = j % C::NSLOT, b = j % C::NB;
            const float* hi = sm.ring + size_t(slot) * T_SLOT_FLOATS;
            const float* opn = sm.opnd + size_t(b) * 2 * M * T_CK;
            t_wait(&sm.opnd_rdy[b], (j / C::NB) & 1, P);  // operands (group B)
            t_wait(&sm.full[slot], (j / C::NSLOT) & 1, P);
            t_wait(&sm.prep[b], (j / C::NB) & 1, P);  // lo tile in TMEM (group A)
            if (sp.fwd) {
              t_wait(&sm.prep2[fj % C::NB], (fj / C::NB) & 1, P);  // its second K half (group B)
              ++fj;
            }
            t_trace(P, tr, 20);
            tc_fence_after();
            // descriptors advance by constants per K-step (start-address field, 16-B units):
            // K-major SW128: +32 B inside the 128-B atom, +16 KB to the next 32-column box;
            // MN-major SW128_32B: +8 rows = 1 KB; operand (no swizzle): +256 B
            const uint64_t da = sp.fwd ? tc_desc_kmajor_sw128(hi, 0) : tc_desc_mn_sw128b32(hi, 0, 8192);
            const uint64_t db = tc_desc_kmajor_noswz(opn, 0, T_CK);
            const uint32_t lot = tbase + C::LO_COL + uint32_t(b) * T_CK;  // lo tile in TMEM
#pragma unroll
            for (int ks = 0; ks < T_CK / 8; ++ks) {
              const uint64_t dak = sp.fwd ? da + uint64_t((ks >> 2) * 1024 + (ks & 3) * 2) : da + uint64_t(ks * 64);
              tc_mma_tf32(acc, dak, db + uint64_t(ks * 16), id2, ch > 0 || ks > 0);
              tc_mma_tf32_ts(acc, lot + ks * 8, db + uint64_t(ks * 16), id1, true);
            }
            if (!sp.fwd) {
              // the update product goes to TMEM buffer bj % NUB, free once group B applied bj - NUB
              const uint32_t ubuf = bj % C::NUB;
              if (bj >= C::NUB) t_wait(&sm.applied[ubuf], ((bj - C::NUB) / C::NUB) & 1, P);
              tc_fence_after();
              if (upd) {
                // D[c][r] = sum_m a[m][c] delta[m][r] over K = m (2 K-steps):
                // a_hi x [delta_hi; delta_lo] (N = 128) and a_lo x delta_hi (N = 64)
                const uint64_t ua = tc_desc_kmajor_noswz(sm.aop, 0, TM);
                const uint64_t ual = tc_desc_kmajor_noswz(sm.aop + 128 * TM, 0, TM);
                const uint64_t ub = tc_desc_kmajor_noswz(sm.dop + size_t(b) * 2 * T_CK * TM, 0, TM);
                const uint32_t ud = tbase + C::UPD_COL + ubuf * 128;
#pragma unroll
                for (int kk = 0; kk < TM / 8; ++kk)
                  tc_mma_tf32(ud, ua + uint64_t(kk * 16), ub + uint64_t(kk * 16), idu2, kk > 0);
#pragma unroll
                for (int kk = 0; kk < TM / 8; ++kk)
                  tc_mma_tf32(ud, ual + uint64_t(kk * 16), ub + uint64_t(kk * 16), idu1, true);
              }
              ++bj;
            }
            tc_commit(&sm.mdone[b]);
            if (sp.fwd) tc_commit(&sm.sfree[slot]);
            t_trace(P, tr, 21);
          }
        }
      }
    }
  }
}

// ------------------------------------------------------------------ SIMT side
// Operand chunk [M][64] fp32 (rows m, 64 consecutive k), staged as tf32 hi / lo in the
// no-swizzle K-major layout. Two phases so the L2 loads of chunk j+1 are in flight while
// chunk j is processed: fetch() issues the loads into registers, put() stores them.
// With dT != nullptr (B chunks), the exact values are also kept as dT[k][m] for the update.
template <int TM>
struct TOpnd {
  // group B thread -> TM / 2 elements (m, k): lane = (m % 8) * 4 + k % 4, so every warp store
  // of the no-swizzle core-matrix layout hits 32 distinct banks (TM / 8 row groups x 16
  // k-quads, split over the 4 warps)
  static constexpr int NQ = TM / 2, MG = TM / 8;
  float v[NQ];
  __device__ __forceinline__ void fetch(const float* src, int ld, int) {
    const int st = (threadIdx.x - T_SIMT0) & (T_GRP - 1), lane = st & 31, w = st >> 5;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int idx = w * NQ + q, m = (idx % MG) * 8 + (lane >> 2), k = (idx / MG) * 4 + (lane & 3);
      v[q] = __ldcg(src + size_t(m) * ld + k);
    }
  }
  // dop != nullptr (B chunks): also the update MMA's B operand [delta_hi; delta_lo]^T, rows
  // r (64 hi + 64 lo) x K = m (TM), no-swizzle K-major
  __device__ __forceinline__ void put(float* ohi, float* olo, float* dop, int) const {
    const int st = (threadIdx.x - T_SIMT0) & (T_GRP - 1), lane = st & 31, w = st >> 5;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int idx = w * NQ + q, mg = idx % MG, kq = idx / MG;
      const int off = mg * 512 + kq * 32 + lane;  // == tc_kmajor_noswz_off(m, k, 64) / 4
      const float h = tf32_hi(v[q]);
      ohi[off] = h;
      olo[off] = v[q] - h;
      if (dop) {
        const int r = kq * 4 + (lane & 3), m = mg * 8 + (lane >> 2);
        const int o2 = int(tc_kmajor_noswz_off(r, m, TM) >> 2);
        dop[o2] = h;
        dop[o2 + T_CK * TM] = v[q] - h;
      }
    }
  }
};

// The lo tile (w - tf32(w)) goes straight from registers to TMEM (tcgen05.st), where the
// lo MMAs read it as their A operand: lane = M row, column = K element. A group-A warp
// owns TMEM lanes 32 * (warp % 4) .. +31 and both 32-deep K halves of the 64-deep chunk.
//
// F chunk (K-major SWIZZLE_128B tile, 2 boxes [128 rows][32 cols]): thread = W row r.
__device__ __forceinline__ void t_lo_pass_f(const float* tile, uint32_t lo_tmem, int kh0, int kh1) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = 32 * (warp & 3) + lane;
  for (int kh = kh0; kh < kh1; ++kh) {
    const float* row = tile + kh * 4096 + r * 32;
    float v[32];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float4 w = *reinterpret_cast<const float4*>(row + ((c ^ (r & 7)) << 2));
      v[4 * c + 0] = w.x - tf32_hi(w.x);
      v[4 * c + 1] = w.y - tf32_hi(w.y);
      v[4 * c + 2] = w.z - tf32_hi(w.z);
      v[4 * c + 3] = w.w - tf32_hi(w.w);
    }
    tmem_st_32x32b_x32(lo_tmem + ((uint32_t(32 * (warp & 3))) << 16) + uint32_t(32 * kh), v);
  }
  tmem_st_wait();
}

// B chunk on the ATOM_32B tile [64 rows][4 boxes x 32 cols]: thread = W column c (the A row
// of W^T), 64 rows; the swizzle permutes 32-B granules by row & 3.
constexpr int T_UPR = 32;  // rows per TMEM store
__device__ __forceinline__ int t_bofs(int cl, int r) {
  const int box = cl >> 5, g = (cl >> 3) & 3, e = cl & 7;
  return box * 2048 + r * 32 + ((g ^ (r & 3)) << 3) + e;
}
__device__ __forceinline__ void t_lo_pass_b(const float* tile, uint32_t lo_tmem) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cl = 32 * (warp & 3) + lane;
  const float* colp[4];
#pragma unroll
  for (int x = 0; x < 4; ++x) colp[x] = tile + t_bofs(cl, x);
#pragma unroll
  for (int rh = 0; rh < 2; ++rh) {
    float v[32];
#pragma unroll
    for (int rr = 0; rr < T_UPR; ++rr) {
      const float w = colp[rr & 3][(rh * T_UPR + rr - (rr & 3)) * 32];
      v[rr] = w - tf32_hi(w);
    }
    tmem_st_32x32b_x32(lo_tmem + ((uint32_t(32 * (warp & 3))) << 16) + uint32_t(32 * rh), v);
  }
  tmem_st_wait();
}
// In-place SGD step on a B chunk once all its MMAs are done (group B): the tensor core has
// computed D[c][r] = sum_m a[m][c] delta[m][r] (3xTF32, columns [0,64) hi*hi + lo*hi,
// [64,128) hi*lo); thread = column c (its TMEM lane), 64 rows: w' = w - lr * (d0 + d1).
// Adam step on one weight (the same arithmetic as pt::adam1)
__device__ __forceinline__ float t_adam1(float w, float g, float& m, float& v, const TParams& P, float c1, float c2) {
  m = fmaf(P.b1, m, P.omb1 * g);
  v = fmaf(P.b2, v, P.omb2 * g * g);
  return w - P.lr * adam_quot(m * c1, v * c2, P.eps);
}

// Adam step of a B chunk: 16-row quarters, so the update products, weights
// and moments of one quarter (80 values) stay in registers. mrow / vrow: the chunk's first
// row of the unit's column block, in the blocked moment layout; thread cl reads its column,
// so a warp's loads are 128 B contiguous and a chunk's moments are two 16 KB runs each.
__device__ __forceinline__ void t_apply_adam(float* tile, uint32_t upd_tmem, const TParams& P, float* mrow,
                                             float* vrow, int, float c1, float c2) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cl = 32 * (warp & 3) + lane;
  mrow += (cl >> 6) * 8192 + (cl & 63);  // column block blk * 2 + cl / 64 of the unit
  vrow += (cl >> 6) * 8192 + (cl & 63);
  constexpr int ld = 64;
  const uint32_t ta = upd_tmem + ((uint32_t(32 * (warp & 3))) << 16);
#pragma unroll 1
  for (int rq = 0; rq < T_CK / 16; ++rq) {
    float mm[16], vv[16], d0[16], d1[16], w[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      mm[q] = __ldcg(mrow + size_t(16 * rq + q) * ld);
      vv[q] = __ldcg(vrow + size_t(16 * rq + q) * ld);
    }
    tmem_ld_32x32b_x16(ta + uint32_t(16 * rq), d0);         // hi*hi + lo*hi
    tmem_ld_32x32b_x16(ta + uint32_t(T_CK + 16 * rq), d1);  // hi*lo
#pragma unroll
    for (int q = 0; q < 16; ++q) w[q] = tile[t_bofs(cl, 16 * rq + q)];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      tile[t_bofs(cl, 16 * rq + q)] = t_adam1(w[q], d0[q] + d1[q], mm[q], vv[q], P, c1, c2);
      __stcg(mrow + size_t(16 * rq + q) * ld, mm[q]);
      __stcg(vrow + size_t(16 * rq + q) * ld, vv[q]);
    }
  }
}

template <bool ADAM>
__device__ __forceinline__ void t_apply_update(float* tile, uint32_t upd_tmem, float nlr, const TParams& P,
                                               float* mrow, float* vrow, int ld, float c1, float c2) {
  if (ADAM) {
    t_apply_adam(tile, upd_tmem, P, mrow, vrow, ld, c1, c2);
    return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cl = 32 * (warp & 3) + lane;
  float* colp[4];
#pragma unroll
  for (int x = 0; x < 4; ++x) colp[x] = tile + t_bofs(cl, x);
#pragma unroll
  for (int rh = 0; rh < 2; ++rh) {
    const uint32_t ta = upd_tmem + ((uint32_t(32 * (warp & 3))) << 16) + uint32_t(32 * rh);
    float d0[32], d1[32];
    tmem_ld_2x32(ta, ta + T_CK, d0, d1);
    // all loads before any store: the compiler cannot prove the rows distinct, and a
    // load-after-store chain would serialize on shared-memory latency
    float w[T_UPR];
#pragma unroll
    for (int rr = 0; rr < T_UPR; ++rr) w[rr] = colp[rr & 3][(rh * T_UPR + rr - (rr & 3)) * 32];
#pragma unroll
    for (int rr = 0; rr < T_UPR; ++rr)
      colp[rr & 3][(rh * T_UPR + rr - (rr & 3)) * 32] = fmaf(nlr, d0[rr] + d1[rr], w[rr]);
  }
}

// Softmax cross-entropy at the network's output (the tick kernel's formula):
// delta[m][r] = (softmax(z_m)[r] - onehot(y_m)[r]) / M * act'(a), loss = sum_m (lse_m - z_m[y_m])
// (the epilogue divides by M). The outputs of every CTA are in the stage cache once the first
// grid barrier passes; each CTA reduces (max, sum exp) over its slice of rows per sample, and
// after the second barrier every CTA combines the G partials in the same fixed order.
__device__ __noinline__ void t_softmax_ce(const TParams& P, const TLayer& L, const float* Ccur, const float* y, long long sid, int ti,
                             u64& gen, int gtid, int gthreads, int st_id, float* s_lse) {
  const int M = P.M, G = P.G, c = blockIdx.x, n = L.n_out;
  const float* z = Ccur + L.a_out;  // [M][n]
  t_grid_sync(P, gen);
  const int per = (n + G - 1) / G, r0 = min(n, c * per), r1 = min(n, r0 + per);
  if (st_id < M) {
    const int m = st_id;
    float mx = -INFINITY;
    for (int r = r0; r < r1; ++r) mx = fmaxf(mx, t_ld(z + size_t(m) * n + r));
    float se = 0.f;
    if (r1 > r0)
      for (int r = r0; r < r1; ++r) se += expf(t_ld(z + size_t(m) * n + r) - mx);
    P.ce[(size_t(c) * M + m) * 2] = mx;
    P.ce[(size_t(c) * M + m) * 2 + 1] = se;
  }
  t_grid_sync(P, gen);
  if (st_id < M) {
    const int m = st_id;
    float mx = -INFINITY;
    for (int k = 0; k < G; ++k) mx = fmaxf(mx, t_ld(P.ce + (size_t(k) * M + m) * 2));
    float se = 0.f;
    for (int k = 0; k < G; ++k) {
      const float pm = t_ld(P.ce + (size_t(k) * M + m) * 2), ps = t_ld(P.ce + (size_t(k) * M + m) * 2 + 1);
      if (ps > 0.f) se += ps * expf(pm - mx);
    }
    s_lse[m] = mx + logf(se);
  }
  simt_sync();
  float lsum = 0.f;
  for (int e = gtid; e < M * n; e += gthreads) {
    const int m = e / n, r = e - m * n;
    const float a = t_ld(z + size_t(m) * n + r);
    const int tgt = y ? int(y[m]) : -1;
    const float g = y ? (expf(a - s_lse[m]) - (r == tgt ? 1.f : 0.f)) / float(M) : 0.f;
    if (P.learn) P.delta[size_t(m) * P.max_n + r] = g * dact_fn(L.act, a);
  }
  if (c == 0 && st_id == 0) {
    for (int m = 0; m < M && y; ++m) {
      const int tgt = int(y[m]);
      if (!(y[m] >= 0.f && y[m] < float(P.F) && float(tgt) == y[m])) {
        atomicMin(P.bad_target, sid);
        continue;
      }
      lsum += s_lse[m] - t_ld(z + size_t(m) * n + tgt);
    }
  }
  if (st_id == 0) P.loss_part[size_t(ti) * G + c] = (c == 0) ? lsum : 0.f;
}

// layout conversion of the tile kernel's blocked weights (pt_set_params / pt_get_params):
// element (r, c) of [n_out][n_in] at ((r / 128) * (n_in / 64) + c / 64) * 8192 + (r % 128) * 64 + c % 64
__global__ void tl_to_blocks(const float* __restrict__ src, float* __restrict__ dst, int n_out, int n_in) {
  const size_t total = size_t(n_out) * n_in;
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    const int r = int(e / n_in), c = int(e % n_in);
    dst[(size_t(r >> 7) * (n_in >> 6) + (c >> 6)) * 8192 + (r & 127) * 64 + (c & 63)] = src[e];
  }
}
__global__ void tl_from_blocks(const float* __restrict__ src, float* __restrict__ dst, int n_out, int n_in) {
  const size_t total = size_t(n_out) * n_in;
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    const int r = int(e / n_in), c = int(e % n_in);
    dst[e] = src[(size_t(r >> 7) * (n_in >> 6) + (c >> 6)) * 8192 + (r & 127) * 64 + (c & 63)];
  }
}

// OPT: 0 SGD, 1 Adam (separate instantiations: the Adam moments' registers stay out of the
// SGD kernel)
template <int OPT, int TM>
__global__ void __launch_bounds__(T_THREADS, 1) tile_kernel(const __grid_constant__ TParams P) {
  using C = TCfg<TM, OPT>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-B alignment of the swizzled tiles
  // (pointer arithmetic on smem_raw, not integer casts, so the compiler keeps the shared
  // state space and emits LDS/STS instead of generic loads)
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  TSmem sm;
  const int M = P.M, G = P.G, c = blockIdx.x;
  const int ob = M * T_CK;
  sm.ring = reinterpret_cast<float*>(base);
  sm.opnd = sm.ring + C::NSLOT * T_SLOT_FLOATS;
  sm.dop = sm.opnd + C::NB * 2 * ob;
  sm.aop = sm.dop + C::NB * 2 * T_CK * TM;
  sm.red = sm.aop + 2 * 128 * TM;
  sm.full = reinterpret_cast<uint64_t*>(sm.red + TM);
  sm.sfree = sm.full + C::NSLOT;
  sm.bfree = sm.sfree + C::NSLOT;
  sm.opnd_rdy = sm.bfree + C::NSLOT;
  sm.prep = sm.opnd_rdy + C::NB;
  sm.prep2 = sm.prep + C::NB;
  sm.mhi = sm.prep2 + C::NB;
  sm.mdone = sm.mhi + C::NB;
  sm.afree = sm.mdone + C::NB;
  sm.applied = sm.afree + 2;
  sm.tmem = reinterpret_cast<uint32_t*>(sm.applied + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    // barriers arrived by a SIMT group count its 4 warps (one arrival per warp, no group
    // barrier needed); tensor-core commits and the producer arrive once
    for (int s = 0; s < C::NSLOT; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.sfree[s], 1);
      mbar_init(&sm.bfree[s], 4);
    }
    for (int b = 0; b < C::NB; ++b) {
      mbar_init(&sm.opnd_rdy[b], 4);
      mbar_init(&sm.mhi[b], 1);
      mbar_init(&sm.prep[b], 4);
      mbar_init(&sm.prep2[b], 4);
      mbar_init(&sm.mdone[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.afree[b], 4);
      mbar_init(&sm.applied[b], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(sm.tmem, T_TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *sm.tmem;

  if (warp == 0) {
    if (lane == 0) t_producer<TM, OPT>(P, sm);
  } else if (warp == 1) {
    if (lane == 0) t_mma<TM, OPT>(P, sm, tbase);
  } else {
    // ================================================================ SIMT
    const int st_id = tid - T_SIMT0;           // 0..255
    const int gtid = c * T_NS + st_id, gthreads = G * T_NS;
    const float nlr = -P.lr;
    const float inv_mf = 1.f / float(M * P.F);
    uint32_t j = 0, uc = 0, bj = 0, fj = 0;
    u64 gen = 0;
    int tr = 0;
    for (int ti = 0; ti < P.n; ++ti) {
      const long long t = P.t0 + ti;
      const int cur = int(t & 1), prv = cur ^ 1;
      for (int s = 0; s < P.n_stages; ++s) {
        const TStage& S = P.stages[s];
        const int h = S.h;
        const bool is_last = (h == P.D);
        const bool upd = t_upd(P, t, h);
        // Adam bias corrections of this stage's k-th update (k counts from the warm-up gate;
        // in double, as pt::tick_kernel)
        float c1 = 1.f, c2 = 1.f;
        if (OPT == 1 && upd) {
          const double k = double(t - (2LL * P.D - h - 1) + 1);
          c1 = float(1.0 / (1.0 - pow(P.b1d, k)));
          c2 = float(1.0 / (1.0 - pow(P.b2d, k)));
        }
        float* Ccur = S.cache[cur];
        const float* Cb = (h < P.D && P.act_delay) ? S.cache[prv] : S.cache[cur];  // backward cache
        // stage input: x_t (h = 1) or inslot[(t-1) % 2]
        const float* in;
        int ld_in0;
        if (h == 1) {
          in = P.xs + size_t(ti) * M * P.ldx;
          ld_in0 = P.ldx;
        } else {
          in = S.inslot[prv];
          ld_in0 = S.n0;
        }
        if (S.up_remote) {
          // the upstream process has published its tick t-1 activations into inslot
          t_wait_cnt(P, S.in_ready, u64(t));
          simt_sync();
        }
        // private copy of the stage input (inslot is overwritten at t+1 before B reads it)
        for (int e = gtid; e < M * S.n0; e += gthreads) {
          const int m = e / S.n0, k = e - m * S.n0;
          Ccur[size_t(m) * S.n0 + k] = t_ld(in + size_t(m) * ld_in0 + k);
        }
        for (int st = 0; st < t_nsteps(P, S); ++st) {
          const TStep sp = t_step(P, S, st);
          const TLayer& L = P.layers[sp.L];
          const int i = sp.L - S.first;
          // ---------------------------------------------------- compute
          if (!sp.fwd && upd) {
            // bias of this layer, rows spread over the grid: b -= lr * sum_m delta
            for (int r = gtid; r < L.n_out; r += gthreads) {
              float dv[TM];
#pragma unroll
              for (int m = 0; m < TM; ++m) dv[m] = m < M ? t_ld(P.delta + size_t(m) * P.max_n + r) : 0.f;
              float sd = 0.f;
#pragma unroll
              for (int m = 0; m < TM; ++m) sd += dv[m];
              if (OPT == 1) {
                float mm = t_ld(L.mb + r), vv = t_ld(L.vb + r);
                L.b[r] = t_adam1(t_ld(L.b + r), sd, mm, vv, P, c1, c2);
                L.mb[r] = mm;
                L.vb[r] = vv;
              } else {
                L.b[r] = fmaf(nlr, sd, t_ld(L.b + r));
              }
            }
          }
          t_trace(P, tr, 1);
          const int grp = warp < 6 ? 0 : 1;
          for (int u = c; u < sp.nunits; u += G, ++uc) {
            const int blk = u / T_Q, q = u % T_Q;
            if (grp == 0) {
              // ===================== group A: lo tiles (TMEM), accumulator epilogue
              for (int ch = 0; ch < sp.nchunks; ++ch, ++j) {
                const int slot = j % C::NSLOT, b = j % C::NB;
                const float* tile = sm.ring + size_t(slot) * T_SLOT_FLOATS;
                const uint32_t lot = tbase + C::LO_COL + uint32_t(b) * T_CK;  // lo tile in TMEM
                t_trace(P, tr, 6);
                if (j >= C::NB) t_wait(&sm.mdone[b], ((j - C::NB) / C::NB) & 1, P);  // lo buffer free
                tc_fence_after();
                t_wait(&sm.full[slot], (j / C::NSLOT) & 1, P);
                t_trace(P, tr, 7);
                if (sp.fwd) t_lo_pass_f(tile, lot, 0, 1);
                else t_lo_pass_b(tile, lot);
                t_trace(P, tr, 13);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.prep[b]);
              }
              // unit epilogue: last chunk's MMAs complete -> accumulator -> quarter partials
              const uint32_t jl = j - 1;
              t_wait(&sm.mdone[jl % C::NB], (jl / C::NB) & 1, P);
              tc_fence_after();
              {
                const int lq = warp & 3;
                const uint32_t ta = tbase + (uc & 1) * uint32_t(T_NACC * 2 * M) + ((uint32_t(lq) * 32) << 16);
                const int rowcol = blk * 128 + lq * 32 + lane;  // F: output row; B: input column
                float* dst = P.part + size_t(q) * M * P.max_n + rowcol;
                if constexpr (TM == 16) {
                  float vv[32];
                  tmem_ld_32x32b_x32(ta, vv);  // one load + wait: columns [0,16) and [16,32)
#pragma unroll
                  for (int m = 0; m < 16; ++m) dst[size_t(m) * P.max_n] = vv[m] + vv[16 + m];  // (hi + lo) * a_hi + hi * a_lo
                } else {
#pragma unroll
                  for (int hh = 0; hh < TM / 32; ++hh) {
                    float v0[32], v1[32];
                    tmem_ld_2x32(ta + 32 * hh, ta + TM + 32 * hh, v0, v1);  // columns of samples 32 hh.. in [0, TM) and [TM, 2 TM)
#pragma unroll
                    for (int m = 0; m < 32; ++m) dst[size_t(32 * hh + m) * P.max_n] = v0[m] + v1[m];
                  }
                }
              }
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&sm.afree[uc & 1]);
            } else {
              // ===================== group B: operands (smem), SGD write-back of backward tiles
              const int gst = st_id - T_GRP;
              if (!sp.fwd && upd) {
                // A operand of the update MMAs: a_i^T of the unit's 128 columns (backward
                // cache), tf32 hi / lo, no-swizzle K-major [128][16]; published with chunk
                // 0's operands. The previous unit's MMAs are complete (its last apply waited).
                const int cbase = blk * 128;
                for (int e = gst; e < 128 * TM; e += T_GRP) {
                  const int m = e >> 7, cc = e & 127;
                  const float x = t_ld(Cb + L.a_in + size_t(m) * L.n_in + cbase + cc);
                  const int o = int(tc_kmajor_noswz_off(cc, m, TM) >> 2);
                  const float h = tf32_hi(x);
                  sm.aop[o] = h;
                  sm.aop[128 * TM + o] = x - h;
                }
              }
              // operand source of chunk ch: F = a_i[:, cols], B = delta[:, rows]
              const float* osrc;
              int old;
              if (sp.fwd) {
                const int c0 = q * (L.n_in / T_Q);
                osrc = (i == 0) ? in + c0 : Ccur + L.a_in + c0;
                old = (i == 0) ? ld_in0 : L.n_in;
              } else {
                osrc = P.delta + q * (L.n_out / T_Q);
                old = P.max_n;
              }
              TOpnd<TM> op;
              op.fetch(osrc, old, M);
              auto apply = [&](uint32_t jj, uint32_t bb, int chn) {
                // chunk jj: all its MMAs are done -> SGD step in place -> producer stores the tile
                const int pslot = jj % C::NSLOT;
                t_wait(&sm.mdone[jj % C::NB], (jj / C::NB) & 1, P);
                tc_fence_after();
                t_trace(P, tr, 9);
                if (upd) {
                  // Adam: this chunk's rows r0.. and the unit's 128 columns c0.. of the moments
                  const int mr0 = q * (L.n_out / T_Q) + chn * T_CK;  // blocked moments (see TLayer)
                  const size_t mo = (size_t(mr0 >> 7) * (L.n_in >> 6) + size_t(blk) * 2) * 8192 + size_t(mr0 & 127) * 64;
                  t_apply_update<OPT == 1>(sm.ring + size_t(pslot) * T_SLOT_FLOATS, tbase + C::UPD_COL + (bb % C::NUB) * 128, nlr, P,
                                 OPT == 1 ? L.mW + mo : nullptr, OPT == 1 ? L.vW + mo : nullptr, L.ld, c1, c2);
                  fence_proxy_async_shared();  // W' -> the producer's TMA store
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                  mbar_arrive(&sm.bfree[pslot]);
                  mbar_arrive(&sm.applied[bb % C::NUB]);
                }
                t_trace(P, tr, 10);
              };
              for (int ch = 0; ch < sp.nchunks; ++ch, ++j) {
                const int b = j % C::NB;
                float* ohi = sm.opnd + size_t(b) * 2 * ob;
                float* dopb = sm.dop + size_t(b) * 2 * T_CK * TM;
                t_trace(P, tr, 8);
                if (j >= C::NB) t_wait(&sm.mdone[b], ((j - C::NB) / C::NB) & 1, P);  // operand buffers free
                tc_fence_after();
                op.put(ohi, ohi + ob, sp.fwd ? nullptr : dopb, M);
                if (ch + 1 < sp.nchunks) op.fetch(osrc + (ch + 1) * T_CK, old, M);
                fence_proxy_async_shared();  // operands -> the tensor core (async proxy)
                if (sp.fwd) {
                  // forward: group B also writes K half 1 of the lo tile
                  const int slot = j % C::NSLOT;
                  t_wait(&sm.full[slot], (j / C::NSLOT) & 1, P);
                  t_lo_pass_f(sm.ring + size_t(slot) * T_SLOT_FLOATS, tbase + C::LO_COL + uint32_t(b) * T_CK, 1, 2);
                  tc_fence_before();
                }
                __syncwarp();
                if (lane == 0) {
                  mbar_arrive(&sm.opnd_rdy[b]);
                  if (sp.fwd) mbar_arrive(&sm.prep2[fj % C::NB]);
                }
                if (sp.fwd) ++fj;
                if (!sp.fwd) {
                  if (ch > 0) apply(j - 1, bj, ch - 1);
                  if (ch > 0) ++bj;
                }
              }
              if (!sp.fwd) {
                apply(j - 1, bj, sp.nchunks - 1);
                ++bj;
              }
            }
          }
          t_trace(P, tr, 2);
          t_grid_sync(P, gen);
          t_trace(P, tr, 3);
          // ---------------------------------------------------- cross-process stage exchange
          const bool last_fwd = sp.fwd && (i == S.k - 1) && h < P.D;   // writes down_inslot, reads gslot
          const bool first_bwd = !sp.fwd && i == 0 && h > 1;            // writes up_gslot
          if (sp.fwd && i == 0 && S.up_remote && c == 0 && st_id == 0)
            red_release_sys(S.peer_act_credit, 1);  // every read of inslot[(t-1)%2] is done
          if (last_fwd && S.down_remote) {
            t_wait_cnt(P, S.act_credit, u64(t));          // downstream read what I sent at t-2
            if (P.learn) t_wait_cnt(P, S.g_ready, u64(t));  // downstream's tick t-1 gradient is in
            simt_sync();
          }
          if (first_bwd && S.up_remote) {
            t_wait_cnt(P, S.g_credit, u64(t));  // upstream read the gradient I sent at t-2
            simt_sync();
          }
          // ---------------------------------------------------- finalize
          if (sp.fwd) {
            const bool last_layer = (i == S.k - 1);
            const bool last_of_net = last_layer && is_last;
            const long long sid = t - (P.D - 1);
            const float* y = nullptr;
            if (last_of_net && sid >= 0) {
              if (sid >= P.t0) y = P.ys ? P.ys + size_t(sid - P.t0) * M * P.Fy : nullptr;
              else if (P.yhist) y = P.yhist + size_t(sid % P.yh) * M * P.Fy;
            }
            const bool ce = last_of_net && P.loss == 1;
            float lacc = 0.f;
            const int n = L.n_out;
            for (int e = gtid; e < M * n; e += gthreads) {
              const int m = e / n, r = e - m * n;
              float z = 0.f;
#pragma unroll
              for (int qq = 0; qq < T_Q; ++qq) z += t_ld(P.part + (size_t(qq) * M + m) * P.max_n + r);
              z += t_ld(L.b + r);
              const float a = act_fn(L.act, z);
              Ccur[L.a_out + size_t(m) * n + r] = a;
              if (last_layer && h < P.D) S.down_inslot[cur][size_t(m) * n + r] = a;
              if (ce) {
                P.outs[(size_t(ti) * M + m) * P.F + r] = a;  // softmax-CE: delta and loss below
              } else if (last_of_net) {
                P.outs[(size_t(ti) * M + m) * P.F + r] = a;
                float g = 0.f;
                if (y) {
                  const float d = a - y[size_t(m) * P.F + r];
                  lacc = fmaf(d, d, lacc);
                  g = 2.f * d * inv_mf;
                }
                if (P.learn) P.delta[size_t(m) * P.max_n + r] = g * dact_fn(L.act, a);
              } else if (last_layer && P.learn) {
                // delta of the stage's last layer from the downstream gradient sent at t-1
                const float ao = (P.act_delay) ? t_ld(Cb + L.a_out + size_t(m) * n + r) : a;
                P.delta[size_t(m) * P.max_n + r] = t_ld(S.gslot[prv] + size_t(m) * n + r) * dact_fn(L.act, ao);
              }
            }
            if (ce) t_softmax_ce(P, L, Ccur, y, sid, ti, gen, gtid, gthreads, st_id, sm.red);
            if (last_of_net && !ce) {
              // fixed-order CTA sum of the loss partials
              float v = warp_sum(lacc);
              if (lane == 0) sm.red[warp - 2] = v;
              simt_sync();
              if (st_id == 0) {
                float sacc = 0.f;
                for (int w = 0; w < T_NS / 32; ++w) sacc += sm.red[w];
                P.loss_part[size_t(ti) * G + c] = sacc;
              }
            }
          } else {
            const int n = L.n_in;
            for (int e = gtid; e < M * n; e += gthreads) {
              const int m = e / n, col = e - m * n;
              float g = 0.f;
#pragma unroll
              for (int qq = 0; qq < T_Q; ++qq) g += t_ld(P.part + (size_t(qq) * M + m) * P.max_n + col);
              if (i > 0) {
                const float ai = t_ld(Cb + L.a_in + size_t(m) * n + col);
                const TLayer& Lp = P.layers[sp.L - 1];
                P.delta[size_t(m) * P.max_n + col] = g * dact_fn(Lp.act, ai);
              } else if (h > 1) {
                S.up_gslot[cur][size_t(m) * n + col] = g;
              }
            }
          }
          t_trace(P, tr, 4);
          if ((last_fwd && S.down_remote) || (first_bwd && S.up_remote)) __threadfence_system();
          t_grid_sync(P, gen);
          if (c == 0 && st_id == 0) {
            if (last_fwd && S.down_remote) {
              red_release_sys(S.peer_in_ready, 1);                // tick t activations published
              if (P.learn) red_release_sys(S.peer_g_credit, 1);  // tick t-1 gradient consumed
            }
            if (first_bwd && S.up_remote) red_release_sys(S.peer_g_ready, 1);  // tick t gradient published
          }
          t_trace(P, tr, 5);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_free(tbase, T_TMEM_COLS);
}

}  // namespace pt
