// pt_panel.cuh: the batch-1 panel kernel for sm_100a (SGD or Adam; MSE or softmax-CE).
//
// Same tick contract as pt::tick_kernel (reference SPEC.md:217-225,
// 253-257), with a weight layout and work split that take the backward's
// cross-CTA reduction off the critical path (profiles/round2_step_bench.md).
//
// Weight layout. Layer l is a grid of R x C tiles of 16 x 16 fp32 (1 KB), row-block major:
// tile (rb, cb) at ((rb * C) + cb) * 256 floats, row-major inside the tile. Padding rows and
// columns are zero and stay zero. Two buffers per layer (see "deferred update").
//
// Work split. CTA k owns row blocks rows_of(R, k, G) in the forward and column blocks
// rows_of(C, k, G) in the backward:
//   F_l : z[rows of rb] = W[rb, :] a       reads row block rb (C contiguous tiles, 1-D bulk)
//   B_l : g[cols of cb] = W[:, cb]^T delta  reads column panel cb (R tiles, 1 KB each, 3-D
//                                           TMA tensor copies of 32 tiles)
// Both steps end in an all-gather of a tagged vector (every CTA needs the whole previous
// vector); no step has a cross-CTA reduction.
//
// Update placement. B_l(t) reads W^(t) (the pre-update weights g_in needs), applies the
// rank-1 step W^(t+1) = W^(t) - lr delta_t a_hat_t^T in registers and stores W^(t+1) into the
// other buffer; F_l(t+1) then reads it (4 + 8 B/weight per tick). The network's first layer has
// no g_in and hence no backward weight read, so with SGD its update is deferred: F_0(t+1)
// applies it to each chunk as it lands in shared memory, before the input vector is there
// ("update-ahead"), and stores W^(t+1) (8 B/weight); the pending update of a run's last tick is
// applied by the next run's forward, or by pt_get_params. With Adam every layer updates in its
// backward, and the moments stream through the ring beside W (PLayer::mW).
//
// Backward vectors. The CTA that publishes g_in of layer l+1 for its columns multiplies by
// act'(a_l) itself, so the published vector IS delta_l (tagged, tick parity). It is the
// dependency of B_l(t) and, one tick later, the deferred update's delta (F_l(t+1): own rows;
// B_l(t+1): all rows). A stage's last layer keeps its delta in L.dst (from the loss or from
// the downstream stage's gradient).
//
// Synchronisation (cross-CTA data are tagged words {value, tick+1}, as in the tick kernel):
//   - tick barrier (learning): a CTA starts tick t once every CTA finished tick t-1. It orders
//     the weight stores of F(t) (buffer t&1) after every B(t-1) read of that buffer, and it
//     bounds every ring of per-tick data (cache mod 4, delta mod 2) to one tick of lag;
//   - the producer issues tick-t backward loads (column panels from every CTA's F(t-1)
//     stores) once tick t-1 is finished everywhere (same counter), and forward loads of its
//     own rows once its consumers have fenced the previous tick's stores of that layer;
//   - stage exchange: the tick kernel's tagged inslot / gslot words and credit counters, so
//     neighbouring stages may live in another process / on another GPU (IPC, NVLink).
#pragma once
#include <cuda.h>

#include "pt_kernels.cuh"
#include "pt_tc.cuh"

namespace pt {

constexpr int PN_TS = 16;                       // tile side
constexpr int PN_TILE = PN_TS * PN_TS;          // floats per tile (1 KB)
constexpr int PN_CT = 32;                       // tiles per chunk (one 32 KB ring slot)
constexpr int PN_SLOT_FLOATS = PN_CT * PN_TILE;
constexpr int PN_MAXSLOT = 8;

struct PLayer {
  float* W[2];               // tiled weights, two buffers
  const CUtensorMap* tm[2];  // 3-D maps {256 floats, C, R} of W[0] / W[1]: column-panel boxes of 32 tiles
  float* b;                  // bias [n_out] (the owner CTA keeps its rows in smem during a launch)
  u64* gin[2];               // tagged delta of the previous layer = act' * g_in, [C*16] per tick parity
  float* dpl;                // plain copy of this layer's delta, [2][R*16] per tick parity (read at t+1)
  float *mW, *vW;            // Adam moments, 16 x 16 tiles in column-panel-major order (tile (rb, cb) at
                             // (cb * R + rb) * 256): only the backward touches them, one column
                             // panel per CTA, so a chunk is 32 KB contiguous (one bulk copy)
  float *mb, *vb;            // Adam moments of the bias [n_out]
  int n_in, n_out, R, C, act;
  int bw;                    // learning, and the backward reads W: it applies the update and stores
                             // W^(t+1) (buffer (t+1)&1); else the forward applies it (deferred)
  int cache_in, cache_out;   // word offsets of a_{l-1}, a_l in a stage cache slot
  long long set_tick;        // pt_set_params at this tick discarded the pending update of earlier ticks
};

struct PStage {
  int h, first, k;
  int G_up, G_down, up_remote, down_remote;
  int ld0, ldk;              // stage slot strides (words)
  u64* cache[4];             // tagged activation cache slots, tick mod 4
  float* pcache[4];          // plain copies (read one tick or more later: a_hat, act')
  u64* inslot[2];
  u64* gslot[2];
  u64* peer_inslot[2];
  u64* peer_gslot[2];
  u64* act_credit;
  u64* g_credit;
  u64* peer_act_credit;
  u64* peer_g_credit;
};

struct PParams {
  const PStage* stages;
  const PLayer* layers;
  int n_stages, n_layers, D, learn, act_delay, G, F, loss;
  float lr;
  float b1, b2, eps, omb1, omb2;  // Adam, as pt::Params
  double b1d, b2d;
  int adam;  // Adam: an updating backward chunk occupies three ring slots (W, m, v)
  const float* xs;  // padded [n][ldx] (stage 1 local)
  int ldx;
  const float* ys;  // [n][Fy] targets of this run
  const float* yhist;
  int yh;
  float* outs;      // [n][F]
  float* loss_part; // [n][G]
  long long t0;
  int n;
  u64* tick_end;    // cumulative CTA-ticks since create
  int* status;
  long long* bad_target;
  unsigned long long timeout_ns;
  int nslot, va_off, vb_off, sown_off, sah_off, red_off, bar_off, desc_off, bias_off;
  int policy;
  int pf_chunks;    // L2 prefetch distance of the producer (chunks)
  int psleep;       // producer spin back-off (ns)
  int dbg;          // experiments: bit0 = no per-step store fence, bit1 = no update-ahead
  u64* trace;
  int trace_cap, trace_cta;
  int jitter, jitter_mask;
  // Resident per-sample mode (pt_step with host buffers): one launch serves every step until
  // the host posts PN_STOP. The host writes x_t / gamma_t into mapped rings and then
  // hreq = t + 1; CTA 0 relays hreq to the other CTAs through a device word; each CTA copies
  // its slice of x_t into the tagged stage input xin[t & 1]; outputs go to the mapped
  // rout[t & 1], and the CTA that arrives last at the end of tick t sums the loss partials (in
  // the epilogue kernel's order) and publishes the PResDone record. No launch, no copy and no
  // host round trip besides the two mapped words per step.
  int resident;
  int res_last;           // this launch owns stage D: it copies targets and writes the record
  const long long* hreq;  // host-mapped: ticks requested (t + 1), or PN_STOP
  const int* hflag;       // host-mapped: 1 iff the step passed a target
  long long* relay;       // device: CTA 0's copy of hreq for the other CTAs
  const float* rx;        // host-mapped x ring [rring][ldx] (zero padded)
  const float* ry;        // host-mapped target ring [rring][Fy]
  int rring;
  u64* xin;               // device: tagged stage-1 input [2][ldx]
  u64* ytag;              // device: tagged targets [rring][ldy] (copied by CTA slices at the
  int ldy;                //   tick they are posted; the loss reads them D-1 ticks later)
  float* rout;            // host-mapped outputs [2][F]
  struct PResDone* rdone; // host-mapped completion record
};

constexpr long long PN_STOP = -1;

// completion record of one resident step (written by the last CTA, read by the host)
struct PResDone {
  long long tick;        // t + 1 once the fields below belong to tick t
  long long bad_loss;    // t if the loss was not finite, else -1
  long long bad_target;  // first sample whose softmax-CE target is not a class index (int64 max: none)
  float loss;
  int valid;
  int status;
  int pad_;
  unsigned long long req_ns, done_ns;  // diagnostics: globaltimer when CTA 0 saw the request / at the record
};

__device__ __forceinline__ int cmod4(long long t) { return int(t & 3); }  // two's complement: -1 -> 3

__device__ __forceinline__ bool pn_upd(const PParams& P, int h, long long t) {
  return P.learn && P.lr != 0.f && t >= 2LL * P.D - h - 1;  // warm-up gate SPEC.md:254
}
// the update of tick t-1 is still to be applied to layer L at tick t
__device__ __forceinline__ bool pn_pending(const PParams& P, const PLayer& L, int h, long long t) {
  return pn_upd(P, h, t - 1) && t - 1 >= L.set_tick && !(P.dbg & 8);
}
// weight buffer the forward of tick t reads: W^(t) (backward-written layers), W^(t-1) (the
// forward applies the pending update), or the only buffer (inference)
__device__ __forceinline__ int pn_fbuf(const PParams& P, const PLayer& L, long long t) {
  return !P.learn ? 0 : L.bw ? int(t & 1) : int((t - 1) & 1);
}
// the cache tick whose activations B(t) uses (act_delay reading)
__device__ __forceinline__ long long pn_ct(const PParams& P, int h, long long t) {
  return (h < P.D && P.act_delay) ? t - 1 : t;
}

__device__ __forceinline__ long long ld_acquire_sys_s64(const long long* p) {
  long long v;
  asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ long long ld_acquire_gpu_s64(const long long* p) {
  long long v;
  asm volatile("ld.acquire.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu_s64(long long* p, long long v) {
  asm volatile("st.release.gpu.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ float ld_volatile_f32(const float* p) {
  float v;
  asm volatile("ld.volatile.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}
// resident mode: wait until the host requested tick t (value >= t + 1) or posted a stop.
// CTA 0 polls the mapped host word and relays it; the others poll the relay in L2.
__device__ __forceinline__ bool pn_wait_request(const PParams& P, long long t, bool poll_host) {
  long long r;
  if (poll_host) {
    while ((r = ld_acquire_sys_s64(P.hreq)) < t + 1 && r != PN_STOP) __nanosleep(64);
    P.rdone->req_ns = globaltimer();
    if (ld_acquire_gpu_s64(P.relay) != r) st_release_gpu_s64(P.relay, r);
  } else {
    while ((r = ld_acquire_gpu_s64(P.relay)) < t + 1 && r != PN_STOP) __nanosleep(32);
  }
  return r != PN_STOP;
}

__device__ __forceinline__ bool pn_watchdog(const PParams& P, uint64_t t_start) {
  if (ld_volatile_s32(P.status) != ST_OK) return true;
  if (globaltimer() - t_start > P.timeout_ns) {
    atomicCAS(P.status, ST_OK, ST_TIMEOUT);
    return true;
  }
  return false;
}

__device__ __noinline__ void pn_wait_cnt(const u64* p, u64 target, const PParams& P) {
  if (p == nullptr || target == 0) return;
  if (ld_acquire_sys(p) >= target) return;
  const uint64_t t_start = globaltimer();
  for (unsigned it = 1;; ++it) {
    if (ld_acquire_sys(p) >= target) return;
    if ((it & 63u) == 0 && pn_watchdog(P, t_start)) return;
  }
}

__device__ __forceinline__ u64 pn_ld(const u64* p, bool sys) { return sys ? ld_tv_sys(p) : ld_tv_gpu(p); }

// resolve one tagged word (re-poll until its tag matches)
__device__ __forceinline__ float pn_resolve(const u64* p, u64 v, uint32_t tag, bool sys, const PParams& P) {
  if (tv_tag(v) == tag) return tv_val(v);
  const uint64_t t_start = globaltimer();
  for (unsigned it = 1;; ++it) {
    v = pn_ld(p, sys);
    if (tv_tag(v) == tag) break;
    if ((it & 31u) == 0 && pn_watchdog(P, t_start)) break;
  }
  return tv_val(v);
}

__device__ __forceinline__ void pn_trace(const PParams& P, int& idx, int limit, int code) {
  if (P.trace != nullptr && blockIdx.x == P.trace_cta && idx < limit)
    P.trace[idx++] = (u64(code) << 56) | (globaltimer() & 0x00FFFFFFFFFFFFFFull);
}
// race detector: random stalls at the step phases (compiled into libpartime_b200_jitter.so only)
__device__ __forceinline__ void pn_jitter(const PParams& P, int code) {
#ifdef PT_JITTER_BUILD
  if (P.jitter <= 0) return;
  uint32_t x = uint32_t(globaltimer()) ^ (blockIdx.x * 0x9E3779B9u) ^ ((threadIdx.x >> 5) * 0x85EBCA6Bu) ^
               (uint32_t(code) * 0xC2B2AE35u);
  x ^= x >> 16;
  x *= 0x7FEB352Du;
  x ^= x >> 15;
  if ((x & uint32_t(P.jitter_mask)) == 0) {
    const uint64_t t0 = globaltimer(), d = (x >> 8) % uint32_t(P.jitter);
    while (globaltimer() - t0 < d) __nanosleep(1000);
  }
#else
  (void)P;
  (void)code;
#endif
}

// tagged words [n] at p into dst[0..n) (scaled) by the consumer threads; the first NCT loads
// were issued earlier (v0 = the value this thread loaded from p[tid], when tid < n)
__device__ __forceinline__ void pn_small(const u64* p, int n, u64 v0, uint32_t tag, float scale, float* dst,
                                         const PParams& P) {
  for (int j = threadIdx.x; j < n; j += NCT) {
    const u64 v = j < NCT ? v0 : ld_tv_gpu(p + j);
    dst[j] = scale * pn_resolve(p + j, v, tag, false, P);
  }
}

// A plain fp32 vector written in an earlier tick (visible after the tick barrier), loaded by the
// consumer threads into registers first (issue, together with a step's other loads) and put
// into shared memory later (store). Words [0, 2048) take one round trip.
struct PPlain {
  float4 v[2];
  __device__ __forceinline__ void issue(const float* p, int n) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int j = int(threadIdx.x) * 4 + NCT * 4 * q;
      v[q] = j < n ? ldcg4(reinterpret_cast<const float4*>(p + j)) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  __device__ __forceinline__ void store(const float* p, int n, float scale, float* dst) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int j = int(threadIdx.x) * 4 + NCT * 4 * q;
      if (j < n) *reinterpret_cast<float4*>(dst + j) = make_float4(scale * v[q].x, scale * v[q].y, scale * v[q].z, scale * v[q].w);
    }
    for (int j = int(threadIdx.x) * 4 + NCT * 8; j < n; j += NCT * 4) {
      const float4 u = ldcg4(reinterpret_cast<const float4*>(p + j));
      *reinterpret_cast<float4*>(dst + j) = make_float4(scale * u.x, scale * u.y, scale * u.z, scale * u.w);
    }
  }
};

struct PV {
  const u64* p;  // null: not gathered (values read as 0)
  uint32_t tag;
  int sys;
};

// Pairs of words a consumer thread gathers per batch: j = base + 2 tid + 2 NCT q, q < 4.
// issue() puts the loads in flight; stale() re-polls every stale pair together, so a round
// costs one L2 round trip however many words were late.
struct PBatch {
  u64 w[8];
  __device__ __forceinline__ void issue(const PV& v, int n, int base) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = base + 2 * int(threadIdx.x) + 2 * NCT * q;
      if (j < n && v.p) {
        if (v.sys) ld2_tv_sys(v.p + j, w[2 * q], w[2 * q + 1]);
        else ld2_tv_gpu(v.p + j, w[2 * q], w[2 * q + 1]);
      } else {
        w[2 * q] = w[2 * q + 1] = pack_tv(0.f, v.tag);
      }
    }
  }
  __device__ __forceinline__ bool stale(const PV& v, int base) {
    bool st = false;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = base + 2 * int(threadIdx.x) + 2 * NCT * q;
      if (tv_tag(w[2 * q]) != v.tag || tv_tag(w[2 * q + 1]) != v.tag) {
        st = true;
        if (v.sys) ld2_tv_sys(v.p + j, w[2 * q], w[2 * q + 1]);
        else ld2_tv_gpu(v.p + j, w[2 * q], w[2 * q + 1]);
      }
    }
    return st;
  }
  __device__ __forceinline__ void settle(const PV& v, int base, const PParams& P) {
    uint64_t t_start = 0;
    for (unsigned it = 0; stale(v, base); ++it) {
      if (it == 0) t_start = globaltimer();
      if ((it & 15u) == 15u && pn_watchdog(P, t_start)) break;
    }
  }
};

// All-gather of up to NV tagged vectors [n] (n even); put(j, x) receives words j, j+1 of each
template <int NV, class Put>
__device__ __forceinline__ void pn_gather(const PV (&v)[NV], int n, const PParams& P, Put&& put) {
  for (int base = 0; base < n; base += 4 * 2 * NCT) {
    PBatch b[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) b[k].issue(v[k], n, base);
    uint64_t t_start = 0;
    for (unsigned it = 0;; ++it) {
      bool st = false;
#pragma unroll
      for (int k = 0; k < NV; ++k) st |= b[k].stale(v[k], base);
      if (!st) break;
      if (it == 0) t_start = globaltimer();
      if ((it & 15u) == 15u && pn_watchdog(P, t_start)) break;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = base + 2 * int(threadIdx.x) + 2 * NCT * q;
      if (j < n) {
        float x[NV][2];
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          x[k][0] = tv_val(b[k].w[2 * q]);
          x[k][1] = tv_val(b[k].w[2 * q + 1]);
        }
        put(j, x);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// producer: every chunk of every step in the consumers' order, plus an L2 prefetch cursor
// pf_chunks ahead
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pn_tma_load_3d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2,
                                               uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void pn_tma_prefetch_3d(const CUtensorMap* tm, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(tm), "r"(c0), "r"(c1),
               "r"(c2)
               : "memory");
}

// Schedule cursor: this CTA's chunks in the consumers' exact order (ticks x local stages x
// [F_0..F_{k-1}, B_{k-1}..B_0] x own blocks x chunks); backward steps without weight reads
// (stage 1, layer 0) have no chunks. fstep counts forward steps from the launch start.
struct PCursor {
  const int* tbl;           // per-layer block ranges of this CTA (PSmem::blk)
  int ti, s, st, blk, off;  // tick, stage, step, own block, chunk offset (tiles) in the block
  int b0, b1, len, nsteps, k, fstep;
  int lim;  // last tick (launch-relative) the cursor may enter: a resident launch parks the
            // cursor at the boundary of a tick the host has not requested (a CTA with no chunks
            // would otherwise walk through every future tick)
  bool done;
  __device__ __forceinline__ bool parked() const { return ti > lim; }
  const PLayer* L;
  __device__ __forceinline__ bool fwd() const { return st < k; }
  __device__ void begin_step(const PParams& P, const PStage* stages, const PLayer* layers) {
    const PStage& S = stages[s];
    k = S.k;
    nsteps = P.learn ? 2 * S.k : S.k;
    const int i = st < S.k ? st : 2 * S.k - 1 - st;
    L = &layers[S.first + i];
    Rows R;
    const int* b = tbl + 6 * (S.first + i);
    if (st < S.k) {
      R = Rows{b[0], b[1]};
      len = L->C;
    } else {
      R = (S.h == 1 && i == 0 && !L->bw) ? Rows{0, 0} : Rows{b[2], b[3]};
      len = L->R;
    }
    b0 = R.r0;
    b1 = R.r1;
    blk = b0;
    off = 0;
  }
  __device__ void next_step(const PParams& P, const PStage* stages, const PLayer* layers) {
    if (st < k) ++fstep;
    if (++st == nsteps) {
      st = 0;
      if (++s == P.n_stages) {
        s = 0;
        if (++ti == P.n) {
          done = true;
          return;
        }
      }
    }
    begin_step(P, stages, layers);
  }
  __device__ void settle(const PParams& P, const PStage* stages, const PLayer* layers) {
    while (!done && !parked() && blk >= b1) next_step(P, stages, layers);
  }
  __device__ void init(const PParams& P, const PStage* stages, const PLayer* layers) {
    ti = s = st = fstep = 0;
    lim = P.resident ? -1 : 0x7fffffff;
    done = P.n <= 0;
    if (done) return;
    begin_step(P, stages, layers);
    settle(P, stages, layers);
  }
  __device__ void advance(const PParams& P, const PStage* stages, const PLayer* layers) {
    off += PN_CT;
    if (off >= len) {
      off = 0;
      ++blk;
      settle(P, stages, layers);
    }
  }
  __device__ __forceinline__ long long t(const PParams& P) const { return P.t0 + ti; }
  __device__ __forceinline__ int ntiles() const { return min(PN_CT, len - off); }
  __device__ __forceinline__ size_t foff() const { return (size_t(blk) * L->C + off) * PN_TILE; }
};

// Weight write-back is the consumers' (st.global from registers, fenced for the async proxy).
// The producer issues a tick's forward loads of its own rows once its consumers have fenced
// the previous tick's stores of that layer (fwd_fenced: forward steps fenced, counted from the
// launch start), and a tick's backward loads (column panels holding every CTA's stores) once
// every CTA finished the previous tick.
template <int OPT>
__device__ void pn_producer(const PParams& P, const PLayer* layers, const PStage* stages, float* ring,
                            uint64_t* full, uint64_t* empty, const int* fwd_fenced, int nF, const int* tbl) {
  const uint64_t pol = P.policy == 1 ? policy_evict_normal() : policy_evict_first();
  const int G = P.G, nslot = P.nslot;
  uint32_t chunk = 0;
  bool dead = false;
  int tr = P.trace_cap / 2;
  PCursor cur, pf;
  cur.tbl = pf.tbl = tbl;
  cur.init(P, stages, layers);
  pf.init(P, stages, layers);
  uint32_t pf_idx = 0;
  auto top_up = [&]() {
    while (!pf.done && !pf.parked() && pf_idx < chunk + uint32_t(P.pf_chunks)) {
      const long long t = pf.t(P);
      if (pf.fwd()) {
        prefetch_l2(pf.L->W[pn_fbuf(P, *pf.L, t)] + pf.foff(), uint32_t(pf.ntiles()) * PN_TILE * 4u);
      } else {
        pn_tma_prefetch_3d(pf.L->tm[int(t & 1)], 0, pf.blk, pf.off);
        if (OPT == 1 && pn_upd(P, stages[pf.s].h, t)) {
          const size_t o = (size_t(pf.blk) * pf.L->R + pf.off) * PN_TILE;
          prefetch_l2(pf.L->mW + o, uint32_t(pf.ntiles()) * PN_TILE * 4u);
          prefetch_l2(pf.L->vW + o, uint32_t(pf.ntiles()) * PN_TILE * 4u);
        }
      }
      pf.advance(P, stages, layers);
      ++pf_idx;
    }
  };
  top_up();
  int raw_ti = 0;  // backward loads of ticks <= raw_ti may start (every CTA finished tick ti-1)
  while (!cur.done && !dead) {
    if (cur.parked()) {
      // resident mode: no load of a tick the host has not requested (at a stop, nothing is in
      // flight)
      if (!pn_wait_request(P, cur.t(P), false)) break;
      cur.lim = pf.lim = cur.ti;
      cur.settle(P, stages, layers);
      pf.settle(P, stages, layers);
      top_up();
      continue;
    }
    const int ti = cur.ti;
    const long long t = cur.t(P);
    if (P.learn && ti > 0) {
      if (cur.fwd() && !cur.L->bw) {
        // forward-written layer: my consumers stored my rows at tick ti-1; fenced yet?
        const int need = cur.fstep - nF + 1;  // the same layer's forward step of tick ti-1
        if (ld_acquire_cta_s32(fwd_fenced) < need) {
          const uint64_t t0 = globaltimer();
          while (ld_acquire_cta_s32(fwd_fenced) < need) {
            top_up();
            if (P.psleep) __nanosleep(P.psleep);
            if (pn_watchdog(P, t0)) {
              dead = true;
              break;
            }
          }
        }
      } else if (ti > raw_ti) {
        // backward-written weights: every CTA's tick ti-1 stores (fenced before its tick arrival)
        pn_wait_cnt(P.tick_end, u64(G) * u64(t), P);
        fence_proxy_async_global();
        raw_ti = ti;
      }
    }
    // an updating Adam backward chunk loads W, m and v into three consecutive ring slots
    const int nparts = (OPT == 1 && !cur.fwd() && pn_upd(P, stages[cur.s].h, t)) ? 3 : 1;
    for (int part = 0; part < nparts && !dead; ++part) {
      const int slot = int(chunk % uint32_t(nslot));
      const uint32_t use = chunk / uint32_t(nslot);
      if (use > 0) {
        const uint64_t t0 = globaltimer();
        while (!dead && !mbar_try_wait(&empty[slot], (use - 1) & 1u)) {
          top_up();
          if (P.psleep) __nanosleep(P.psleep);  // leave issue slots to the consumer warps of this SMSP
          if (pn_watchdog(P, t0)) dead = true;
        }
      }
      if (dead) break;
      float* sdst = ring + size_t(slot) * PN_SLOT_FLOATS;
      if (cur.fwd()) {
        pn_trace(P, tr, P.trace_cap - P.trace_cap / 4, 40);
        pn_jitter(P, 40);
        const uint32_t bytes = uint32_t(cur.ntiles()) * PN_TILE * 4u;
        mbar_arrive_expect_tx(&full[slot], bytes);
        bulk_g2s(sdst, cur.L->W[pn_fbuf(P, *cur.L, t)] + cur.foff(), bytes, &full[slot], pol);
      } else {
        pn_trace(P, tr, P.trace_cap - P.trace_cap / 4, 41);
        pn_jitter(P, 41);
        if (part == 0) {
          mbar_arrive_expect_tx(&full[slot], uint32_t(PN_SLOT_FLOATS) * 4u);
          pn_tma_load_3d(sdst, cur.L->tm[int(t & 1)], 0, cur.blk, cur.off, &full[slot], pol);
        } else {
          // Adam moments: the chunk is contiguous in their column-panel-major layout
          const uint32_t bytes = uint32_t(cur.ntiles()) * PN_TILE * 4u;
          const float* src = (part == 1 ? cur.L->mW : cur.L->vW) + (size_t(cur.blk) * cur.L->R + cur.off) * PN_TILE;
          mbar_arrive_expect_tx(&full[slot], bytes);
          bulk_g2s(sdst, src, bytes, &full[slot], pol);
        }
      }
      if (part + 1 < nparts) ++chunk;
    }
    if (dead) break;
    ++chunk;
    cur.advance(P, stages, layers);
    top_up();
  }
  if (dead) {
    const uint64_t t0 = globaltimer();
    while (globaltimer() - t0 < 2000000ull) {
    }
  }
}

// ---------------------------------------------------------------------------
// consumers
// ---------------------------------------------------------------------------
struct PSmem {
  float* ring;
  float* va;    // F: input a          B: delta
  float* vb;    // F: a_hat (pending)  B: -lr * delta_{t-1} (pending)
  float* sown;  // F: -lr * delta_{t-1} of own rows
  float* sah;   // B: a_hat_{t-1} of own columns
  float* red;   // 2 x 128 floats
  float* scal;  // 64 floats
  float* bias;  // own forward rows of every local layer's bias, resident for the launch
  int* boff;    // per layer: offset of its rows in `bias`
  int* blk;     // per layer: this CTA's row blocks [0, 1), column blocks [2, 3), input words [4, 5)
  int* flags;   // 32 ints: [0] forward steps whose weight stores are fenced (producer's RAW
                // wait), [1] resident mode: the host posted a stop
  uint64_t* full;
  uint64_t* empty;
};

__device__ __forceinline__ void pn_fma4(float4& w, float s, float4 a) {
  w.x = fmaf(s, a.x, w.x);
  w.y = fmaf(s, a.y, w.y);
  w.z = fmaf(s, a.z, w.z);
  w.w = fmaf(s, a.w, w.w);
}

// Forward thread mapping: thread (f4, rg, tg) = (tid & 3, (tid >> 2) & 3, tid >> 4) takes
// float4 f4 of rows rg + 4r (r < 4) of tiles tg and tg + 16 of a chunk, so one load of the
// input vector serves four weight loads (a 128-bit shared load costs four crossbar phases even
// when it is a broadcast). A quarter warp reads two whole consecutive tile rows (128 B).
// Update half: W^(t) = W^(t-1) + sc[r] * a_hat, into the slot (for the dot) and to buffer t&1.
template <bool PEND, bool FULL>
__device__ __forceinline__ void pn_fupdate(float* wb, float* gdst, const float* vb, const float (&sc)[4], int nt,
                                           int tg, bool nostore = false) {
  float4 w[2][4], ah[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int tt = tg + 16 * q;
    const bool ok = FULL || tt < nt;
    ah[q] = (PEND && ok) ? lds4(vb + tt * PN_TS) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int r = 0; r < 4; ++r) w[q][r] = ok ? lds4(wb + tt * PN_TILE + r * 64) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int tt = tg + 16 * q;
    if (FULL || tt < nt) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        if (PEND) {
          pn_fma4(w[q][r], sc[r], ah[q]);
          *reinterpret_cast<float4*>(wb + tt * PN_TILE + r * 64) = w[q][r];
        }
        if (!nostore) __stcs(reinterpret_cast<float4*>(gdst + tt * PN_TILE + r * 64), w[q][r]);
      }
    }
  }
}

// Dot half: z[r] += W[row rg + 4r][this thread's columns] . a (fixed order)
template <bool FULL>
__device__ __forceinline__ void pn_fdot(const float* wb, const float* va, int nt, int tg, float (&z)[4]) {
  float4 w[2][4], a[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int tt = tg + 16 * q;
    const bool ok = FULL || tt < nt;
    a[q] = ok ? lds4(va + tt * PN_TS) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int r = 0; r < 4; ++r) w[q][r] = ok ? lds4(wb + tt * PN_TILE + r * 64) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int r = 0; r < 4; ++r) z[r] += dot4(w[q][r], a[q]);
}

// Backward chunk: acc += W^(t)[rows][own 4 columns] * delta[rows] (this thread: float4 f4 of
// row tr of tiles tg, tg+4, ...), and W^(t+1) = W^(t) - lr delta[row] a_hat[col] stored to the
// next buffer (UPD; the plain copy otherwise, during the warm-up)
__device__ __forceinline__ float pn_adam1(float w, float g, float& m, float& v, const PParams& P, float c1, float c2) {
  m = fmaf(P.b1, m, P.omb1 * g);
  v = fmaf(P.b2, v, P.omb2 * g * g);
  return w - P.lr * adam_quot(m * c1, v * c2, P.eps);
}
__device__ __forceinline__ void pn_adam4(float4& w, float d, float4 ah, float4& m, float4& v, const PParams& P,
                                         float c1, float c2) {
  w.x = pn_adam1(w.x, d * ah.x, m.x, v.x, P, c1, c2);
  w.y = pn_adam1(w.y, d * ah.y, m.y, v.y, P, c1, c2);
  w.z = pn_adam1(w.z, d * ah.z, m.z, v.z, P, c1, c2);
  w.w = pn_adam1(w.w, d * ah.w, m.w, v.w, P, c1, c2);
}

// Backward chunk with the Adam step: g_in from the pre-update W as in pn_bchunk,
// then per weight g = delta_r * a_hat_c and the moments of the same tiled position, read and
// written in place (their loads are issued before the shared-memory tile is read). GIN: this
// layer publishes g_in (else: the network's first layer, update only).
template <bool FULL, bool GIN>
__device__ __forceinline__ void pn_bchunk_adam(const float* wb, const float* dl, float4 ah4, float* gdst, const float* ms,
                                               const float* vs, float* mdst, float* vdst, int C, int nt, int tg,
                                               float4& acc, const PParams& P, float c1, float c2) {
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    float4 w[4];
    float d[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int tt = (hh * 4 + q) * 4 + tg;
      const bool ok = FULL || tt < nt;
      w[q] = ok ? lds4(wb + tt * PN_TILE) : make_float4(0.f, 0.f, 0.f, 0.f);
      d[q] = ok ? dl[tt * PN_TS] : 0.f;
    }
    if (GIN) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        acc.x = fmaf(w[q].x, d[q], acc.x);
        acc.y = fmaf(w[q].y, d[q], acc.y);
        acc.z = fmaf(w[q].z, d[q], acc.z);
        acc.w = fmaf(w[q].w, d[q], acc.w);
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int tt = (hh * 4 + q) * 4 + tg;
      if (FULL || tt < nt) {
        float4 m = lds4(ms + tt * PN_TILE), v = lds4(vs + tt * PN_TILE);
        pn_adam4(w[q], d[q], ah4, m, v, P, c1, c2);
        __stcs(reinterpret_cast<float4*>(gdst + size_t(tt) * C * PN_TILE), w[q]);
        __stcg(reinterpret_cast<float4*>(mdst + size_t(tt) * PN_TILE), m);  // consecutive tiles
        __stcg(reinterpret_cast<float4*>(vdst + size_t(tt) * PN_TILE), v);
      }
    }
  }
}

template <bool UPD, bool FULL>
__device__ __forceinline__ void pn_bchunk(const float* wb, const float* dl, float nlr, float4 ah4, float* gdst,
                                          int C, int nt, int tg, float4& acc) {
  float4 w[8];
  float d[8];
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const int tt = p * 4 + tg;
    const bool ok = FULL || tt < nt;
    w[p] = ok ? lds4(wb + tt * PN_TILE) : make_float4(0.f, 0.f, 0.f, 0.f);
    d[p] = ok ? dl[tt * PN_TS] : 0.f;
  }
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    acc.x = fmaf(w[p].x, d[p], acc.x);
    acc.y = fmaf(w[p].y, d[p], acc.y);
    acc.z = fmaf(w[p].z, d[p], acc.z);
    acc.w = fmaf(w[p].w, d[p], acc.w);
  }
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const int tt = p * 4 + tg;
    if (FULL || tt < nt) {
      if (UPD) pn_fma4(w[p], nlr * d[p], ah4);
      __stcs(reinterpret_cast<float4*>(gdst + size_t(tt) * C * PN_TILE), w[p]);
    }
  }
}

// deterministic CTA-wide max / sum over the consumer threads (result on every thread)
__device__ __forceinline__ float pn_cta_red(float v, bool is_max, const PSmem& sm) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float u = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmaxf(v, u) : v + u;
  }
  cons_sync(NCT);
  if (lane == 0) sm.scal[warp] = v;
  cons_sync(NCT);
  float r = sm.scal[0];
  for (int w = 1; w < NCW; ++w) r = is_max ? fmaxf(r, sm.scal[w]) : r + sm.scal[w];
  cons_sync(NCT);
  return r;
}

// target row of sample sid (stage D): the run's ys or the target history ring
__device__ __forceinline__ const float* pn_target(const PParams& P, long long sid, int Fy) {
  if (sid < 0) return nullptr;
  if (sid >= P.t0 && P.resident) return P.ry + size_t(sid % P.rring) * Fy;
  if (sid >= P.t0) return P.ys ? P.ys + size_t(sid - P.t0) * Fy : nullptr;
  return P.yhist ? P.yhist + size_t(sid % P.yh) * Fy : nullptr;
}

// resident mode: the tagged device copy of sample sid's target, when it was posted during this
// launch (earlier targets come from the target history ring, as in pt_run)
__device__ __forceinline__ const u64* pn_ytag(const PParams& P, long long sid) {
  return (P.resident && sid >= P.t0) ? P.ytag + size_t(sid % P.rring) * P.ldy : nullptr;
}
__device__ __forceinline__ float pn_y(const PParams& P, const float* y, const u64* yt, long long sid, int j) {
  return yt ? pn_resolve(yt + j, ld_tv_gpu(yt + j), tag_of_tick(sid), false, P) : y[j];
}

// output row and loss partials of tick ti: per-run arrays, or two-tick rings (resident)
__device__ __forceinline__ float* pn_outs(const PParams& P, int ti) {
  return P.resident ? P.rout + size_t((P.t0 + ti) & 1) * P.F : P.outs + size_t(ti) * P.F;  // host reads rout[t & 1]
}
__device__ __forceinline__ float* pn_lpart(const PParams& P, int ti) {
  return P.loss_part + size_t(P.resident ? (ti & 1) : ti) * P.G;
}

// wait for one ring slot's data (consumer threads); the slot / phase cursor advances
__device__ __forceinline__ int pn_take(const PSmem& sm, int& cslot, uint32_t& cphase, const PParams& P) {
  const int slot = cslot;
  const uint32_t ph = cphase;
  if (++cslot == P.nslot) {
    cslot = 0;
    cphase ^= 1u;
  }
  if (!mbar_try_wait(&sm.full[slot], ph)) {
    const uint64_t t0 = globaltimer();
    while (!mbar_try_wait(&sm.full[slot], ph))
      if (pn_watchdog(P, t0)) break;
  }
  return slot;
}

// Resident mode, last CTA of tick t (warp 0): the epilogue kernel's loss (same summation
// order: lane-strided partial sums, then warp_sum), validity, the non-finite check, then the
// record's tick word last.
__device__ __noinline__ void pn_resident_done(const PParams& P, long long t, int ti, int lane) {
  __threadfence();
  const bool have = ld_volatile_s32(P.hflag) != 0;
  const bool v = t >= P.D - 1;
  const float* lp = pn_lpart(P, ti);
  float s = 0.f;
  for (int c = lane; c < P.G; c += 32) s += ldcg(lp + c);
  s = warp_sum(s) * (P.loss == 1 ? 1.f : 1.f / float(P.F));
  if (lane != 0) return;
  PResDone* d = P.rdone;
  d->loss = (v && have) ? s : __int_as_float(0x7fc00000);
  d->valid = v ? 1 : 0;
  d->bad_loss = (v && have && !isfinite(s)) ? t : -1;
  d->bad_target = *reinterpret_cast<volatile long long*>(P.bad_target);
  d->status = ld_volatile_s32(P.status);
  d->done_ns = globaltimer();
  __threadfence_system();
  *reinterpret_cast<volatile long long*>(&d->tick) = t + 1;
}

// OPT: 0 SGD, 1 Adam (every layer then updates in its backward, the network's first included)
template <int OPT>
__global__ void __launch_bounds__(NTHREADS, 1) panel_kernel(const __grid_constant__ PParams P) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  PSmem sm;
  sm.ring = reinterpret_cast<float*>(smem_raw);
  sm.va = reinterpret_cast<float*>(smem_raw + P.va_off);
  sm.vb = reinterpret_cast<float*>(smem_raw + P.vb_off);
  sm.sown = reinterpret_cast<float*>(smem_raw + P.sown_off);
  sm.sah = reinterpret_cast<float*>(smem_raw + P.sah_off);
  sm.red = reinterpret_cast<float*>(smem_raw + P.red_off);
  sm.scal = sm.red + 256;
  sm.flags = reinterpret_cast<int*>(sm.scal + 64);
  sm.full = reinterpret_cast<uint64_t*>(smem_raw + P.bar_off);
  sm.empty = sm.full + P.nslot;
  PLayer* s_layers = reinterpret_cast<PLayer*>(smem_raw + P.desc_off);
  PStage* s_stages = reinterpret_cast<PStage*>(s_layers + P.n_layers);
  sm.boff = reinterpret_cast<int*>(s_stages + P.n_stages);
  sm.blk = sm.boff + P.n_layers;
  sm.bias = reinterpret_cast<float*>(smem_raw + P.bias_off);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int c = blockIdx.x, G = P.G;
  if (tid == 0) {
    for (int s = 0; s < P.nslot; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], NCW);
    }
    sm.flags[0] = 0;
    fence_mbar_init();
  }
  {
    const int* src = reinterpret_cast<const int*>(P.layers);
    int* dst = reinterpret_cast<int*>(s_layers);
    for (int j = tid; j < P.n_layers * int(sizeof(PLayer) / 4); j += NTHREADS) dst[j] = src[j];
    src = reinterpret_cast<const int*>(P.stages);
    dst = reinterpret_cast<int*>(s_stages);
    for (int j = tid; j < P.n_stages * int(sizeof(PStage) / 4); j += NTHREADS) dst[j] = src[j];
  }
  __syncthreads();
  int nF = 0;  // forward steps per tick
  for (int s = 0; s < P.n_stages; ++s) nF += s_stages[s].k;
  for (int l = tid; l < P.n_layers; l += NTHREADS) {  // block ranges (no divisions in the tick loop)
    const Rows RB = rows_of(s_layers[l].R, c, G), CB = rows_of(s_layers[l].C, c, G);
    const Rows Q = rows_of(s_layers[l].C * PN_TS, c, G);
    int* b = sm.blk + 6 * l;
    b[0] = RB.r0;
    b[1] = RB.r1;
    b[2] = CB.r0;
    b[3] = CB.r1;
    b[4] = Q.r0;
    b[5] = Q.r1;
  }
  __syncthreads();
  if (tid == 0) {
    int off = 0;
    for (int l = 0; l < P.n_layers; ++l) {
      sm.boff[l] = off;
      off += (sm.blk[6 * l + 1] - sm.blk[6 * l]) * PN_TS;
    }
  }
  __syncthreads();
  for (int l = 0; l < P.n_layers; ++l) {
    const PLayer& L = s_layers[l];
    const Rows RB{sm.blk[6 * l], sm.blk[6 * l + 1]};
    for (int j = tid; j < (RB.r1 - RB.r0) * PN_TS; j += NTHREADS) {
      const int row = RB.r0 * PN_TS + j;
      sm.bias[sm.boff[l] + j] = row < L.n_out ? L.b[row] : 0.f;
    }
  }
  __syncthreads();
  if (warp == NCW) {
    if (lane == 0) {
      // maps written by the host: acquire them for the async proxy (a new handle may reuse a
      // freed handle's map address; see pt_tc.cuh)
      for (int l = 0; l < P.n_layers && P.learn; ++l)
        for (int b = 0; b < 2; ++b) {
          tma_fence_desc_acquire(s_layers[l].tm[b]);
          tma_prefetch_desc(s_layers[l].tm[b]);

        }
      pn_producer<OPT>(P, s_layers, s_stages, sm.ring, sm.full, sm.empty, sm.flags, nF, sm.blk);
    }
    return;
  }
  // backward: float4 f4 of row tr of tiles tg, tg+4, ... (8 tiles of a chunk); forward: see
  // pn_fupdate (float4 f4 of rows fr + 4r of tiles fg, fg + 16)
  const int f4 = tid & 3, tr = (tid >> 2) & 15, tg = tid >> 6;
  const int toff = tr * PN_TS + f4 * 4;  // this thread's float4 inside a tile (backward)
  const int fr = (tid >> 2) & 3, fg = tid >> 4;
  const int foff = fr * PN_TS + f4 * 4;  // forward: row fr of the tile, float4 f4
  int fdone = 0;  // forward steps of this launch whose weight stores are issued
  int cslot = 0;        // ring slot of the next chunk
  uint32_t cphase = 0;  // its full-barrier phase parity
  int tri = 0;
  int trc = P.trace_cap - P.trace_cap / 4;  // chunk-ready events: last quarter of the trace buffer
  const int trl = P.trace_cap / 2;
  int ev_all = 0;
#define PN_TR(code)                                                                                \
  pn_jitter(P, (code));                                                                            \
  if (tid == 0 && P.trace != nullptr) {                                                            \
    if (c == P.trace_cta && tri < trl)                                                             \
      P.trace[tri++] = (u64(code) << 56) | (globaltimer() & 0x00FFFFFFFFFFFFFFull);                \
    if (P.trace_cta < 0 && ((code) == 4 || (code) == 14)) {                                        \
      if ((ev_all + 1) * G <= P.trace_cap) P.trace[ev_all * G + c] = globaltimer();               \
      ++ev_all;                                                                                    \
    }                                                                                              \
  }
#define PN_TRC(code)                                                                               \
  if (tid == 0 && P.trace != nullptr && c == P.trace_cta && trc < P.trace_cap)                     \
    P.trace[trc++] = (u64(code) << 56) | (globaltimer() & 0x00FFFFFFFFFFFFFFull);
  for (int ti = 0; ti < P.n; ++ti) {
    const long long t = P.t0 + ti;
    const uint32_t tag_t = tag_of_tick(t);
    if (P.resident) {
      if (tid == 0) sm.flags[1] = pn_wait_request(P, t, c == 0) ? 0 : 1;
      cons_sync(NCT);
      if (sm.flags[1]) break;
      if (s_stages[0].h == 1) {
        // this CTA's slice of x_t: mapped host memory -> the tagged stage-1 input
        const int* bk0 = sm.blk + 6 * s_stages[0].first;
        const float* xr = P.rx + size_t(t % P.rring) * P.ldx;
        u64* xd = P.xin + size_t(t & 1) * P.ldx;
        for (int j = bk0[4] + tid; j < bk0[5]; j += NCT) st_tv_gpu(xd + j, pack_tv(ld_volatile_f32(xr + j), tag_t));
      }
      if (P.res_last) {
        // this CTA's slice of gamma_t: mapped host memory -> the tagged target ring (padding
        // words up to ldy are tagged zeros, so the loss gather can poll whole rows)
        const Rows Y = rows_of(P.ldy, c, G);
        const int Fy = P.loss == 1 ? 1 : P.F;
        const float* yr = P.ry + size_t(t % P.rring) * Fy;
        u64* yd = P.ytag + size_t(t % P.rring) * P.ldy;
        for (int j = Y.r0 + tid; j < Y.r1; j += NCT) st_tv_gpu(yd + j, pack_tv(j < Fy ? ld_volatile_f32(yr + j) : 0.f, tag_t));
      }
    }
    // tick barrier: every CTA finished tick t-1. It orders this tick's weight stores after
    // every read of their buffer (learning) and keeps the per-tick rings (cache slots mod 4,
    // delta and input parities) at most one tick deep. The counter is cumulative, so only
    // the full barrier bounds the skew: a lagged test (G * (t - 1) at tick t) can be met by
    // the arrivals of CTAs running ahead while one CTA is several ticks behind (the jitter
    // race detector stalled one CTA and the others overwrote cache slots it had not read).
    if (tid == 0) {
      if (t >= 1) pn_wait_cnt(P.tick_end, u64(G) * u64(t), P);
      __threadfence();
    }
    for (int s = 0; s < P.n_stages; ++s) {
      const PStage& S = s_stages[s];
      const int h = S.h;
      u64* Ccur = S.cache[cmod4(t)];
      // ------------------------------------------------------------------ forward
      for (int i = 0; i < S.k; ++i) {
        const PLayer& L = s_layers[S.first + i];
        const int nin = L.C * PN_TS;
        const int* bk = sm.blk + 6 * (S.first + i);
        const Rows RB{bk[0], bk[1]};
        const int nown = (RB.r1 - RB.r0) * PN_TS;
        const int nch = (L.C + PN_CT - 1) / PN_CT;  // chunks per row block
        const bool last = i == S.k - 1;
        const bool fw = P.learn && !L.bw;  // this forward applies the deferred update and stores W^(t)
        const bool pend = fw && pn_pending(P, L, h, t);
        const long long Cp = pn_ct(P, h, t - 1);
        PN_TR(1);
        // every weight store of earlier forward steps is fenced for the producer's loads
        if (P.learn && !(P.dbg & 1)) fence_proxy_async_global();
        // the input vector (the dependency): loads in flight now, resolved after the update
        PV vin{nullptr, 0u, 0};
        if (i == 0 && h > 1) vin = PV{S.inslot[(t - 1) & 1], tag_of_tick(t - 1), S.up_remote};
        else if (i == 0 && P.resident) vin = PV{P.xin + size_t(t & 1) * P.ldx, tag_t, 0};
        else if (i > 0) vin = PV{Ccur + L.cache_in, tag_t, 0};
        PBatch dep;
        dep.issue(vin, nin, 0);
        if (pend) {
          // a_hat_{t-1} and delta_{t-1} of own rows: plain copies from earlier ticks, loaded
          // together with the input's words
          const float* ap = S.pcache[cmod4(Cp)] + L.cache_in;
          const float* dp = L.dpl + size_t((t - 1) & 1) * (L.R * PN_TS) + RB.r0 * PN_TS;
          PPlain ahr;
          ahr.issue(ap, nin);
          const float so = tid < nown ? ldcg(dp + tid) : 0.f;
          ahr.store(ap, nin, 1.f, sm.vb);
          if (tid < nown) sm.sown[tid] = -P.lr * so;
          for (int j = tid + NCT; j < nown; j += NCT) sm.sown[j] = -P.lr * ldcg(dp + j);
        }
        cons_sync(NCT);
        if (P.learn && tid == 0) st_release_cta_s32(&sm.flags[0], fdone);
        PN_TR(2);
        // update-ahead: the pending update of the chunks the ring can hold, before the input
        // is there; W^(t) goes to the slot and to buffer t&1
        const int nck = nch * (RB.r1 - RB.r0);
        const int ua = (fw && !(P.dbg & 2)) ? min(nck, P.nslot) : 0;
        float* Wn = L.W[int(t & 1)];
        {
          int k = 0;
          int us = cslot;
          uint32_t up = cphase;
          for (int rb = RB.r0; rb < RB.r1 && k < ua; ++rb) {
            float sc[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) sc[r] = pend ? sm.sown[(rb - RB.r0) * PN_TS + fr + 4 * r] : 0.f;
            for (int c0 = 0; c0 < L.C && k < ua; c0 += PN_CT, ++k) {
              const int nt = min(PN_CT, L.C - c0);
              const int slot = pn_take(sm, us, up, P);
              PN_TRC(7);
              float* wb = sm.ring + size_t(slot) * PN_SLOT_FLOATS + foff;
              float* gd = Wn + (size_t(rb) * L.C + c0) * PN_TILE + foff;
              const float* vb = sm.vb + c0 * PN_TS + f4 * 4;
              if (pend) {
                if (nt == PN_CT) pn_fupdate<true, true>(wb, gd, vb, sc, nt, fg, (P.dbg & 4) != 0);
                else pn_fupdate<true, false>(wb, gd, vb, sc, nt, fg, (P.dbg & 4) != 0);
              } else {
                if (nt == PN_CT) pn_fupdate<false, true>(wb, gd, vb, sc, nt, fg, (P.dbg & 4) != 0);
                else pn_fupdate<false, false>(wb, gd, vb, sc, nt, fg, (P.dbg & 4) != 0);
              }
            }
          }
        }
        // the input
        if (i == 0 && h == 1 && !P.resident) {
          const float* x = P.xs + size_t(ti) * P.ldx;
          for (int j = tid * 4; j < nin; j += NCT * 4)
            *reinterpret_cast<float4*>(sm.va + j) = ldcg4(reinterpret_cast<const float4*>(x + j));
        } else {
          dep.settle(vin, 0, P);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int j = 2 * tid + 2 * NCT * q;
            if (j < nin) {
              sm.va[j] = tv_val(dep.w[2 * q]);
              sm.va[j + 1] = tv_val(dep.w[2 * q + 1]);
            }
          }
          if (nin > 4 * 2 * NCT) {  // beyond the first batch
            PV rest[1] = {vin};
            pn_gather<1>(rest, nin, P, [&](int j, const float (&x)[1][2]) {
              if (j >= 4 * 2 * NCT) {
                sm.va[j] = x[0][0];
                sm.va[j + 1] = x[0][1];
              }
            });
          }
        }
        cons_sync(NCT);
        if (i == 0) {
          // private copy of the stage input in the cache (inslot is rewritten at t+1)
          const Rows Q{bk[4], bk[5]};
          float* pc = S.pcache[cmod4(t)] + L.cache_in;
          for (int j = Q.r0 + tid; j < Q.r1; j += NCT) {
            st_tv_gpu(Ccur + L.cache_in + j, pack_tv(sm.va[j], tag_t));
            pc[j] = sm.va[j];
          }
          if (h > 1 && tid == 0) red_relaxed_sys(S.peer_act_credit, 1);  // inslot read (all threads: cons_sync above)
        }
        PN_TR(3);
        const bool net_last = last && h == P.D;
        const long long sid = t - (P.D - 1);
        const float* y = net_last ? pn_target(P, sid, P.loss == 1 ? 1 : P.F) : nullptr;
        const u64* yt = net_last ? pn_ytag(P, sid) : nullptr;
        float lsum = 0.f;
        int k = 0;
        for (int rb = RB.r0; rb < RB.r1; ++rb) {
          float sc[4];
#pragma unroll
          for (int r = 0; r < 4; ++r) sc[r] = pend ? sm.sown[(rb - RB.r0) * PN_TS + fr + 4 * r] : 0.f;
          float z[4] = {0.f, 0.f, 0.f, 0.f};
          for (int c0 = 0; c0 < L.C; c0 += PN_CT, ++k) {
            const int nt = min(PN_CT, L.C - c0);
            const int slot = pn_take(sm, cslot, cphase, P);
            if (k >= ua) PN_TRC(7);
            float* wb = sm.ring + size_t(slot) * PN_SLOT_FLOATS + foff;
            const float* va = sm.va + c0 * PN_TS + f4 * 4;
            if (k >= ua && fw) {
              // beyond the update-ahead window: update (and store) here
              float* gd = Wn + (size_t(rb) * L.C + c0) * PN_TILE + foff;
              const float* vb = sm.vb + c0 * PN_TS + f4 * 4;
              if (pend) pn_fupdate<true, false>(wb, gd, vb, sc, nt, fg, (P.dbg & 4) != 0);
              else pn_fupdate<false, false>(wb, gd, vb, sc, nt, fg, (P.dbg & 4) != 0);
            }
            if (nt == PN_CT) pn_fdot<true>(wb, va, nt, fg, z);
            else pn_fdot<false>(wb, va, nt, fg, z);
            PN_TRC(9);
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.empty[slot]);
          }
          // row rg + 4r: sum over f4 (lane bits 0-1) and fg (lane bit 4, then the warps)
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            z[r] += __shfl_xor_sync(0xffffffffu, z[r], 1);
            z[r] += __shfl_xor_sync(0xffffffffu, z[r], 2);
            z[r] += __shfl_xor_sync(0xffffffffu, z[r], 16);
          }
          float* rd = sm.red + ((rb - RB.r0) & 1) * 128;
          if ((lane & 19) == 0) {
#pragma unroll
            for (int r = 0; r < 4; ++r) rd[warp * PN_TS + fr + 4 * r] = z[r];
          }
          cons_sync(NCT);
          PN_TRC(10);
          if (tid < PN_TS) {
            const int row = rb * PN_TS + tid;
            float a = 0.f;
            if (row < L.n_out) {
              float zz = 0.f;
#pragma unroll
              for (int w = 0; w < NCW; ++w) zz += rd[w * PN_TS + tid];
              a = act_fn(L.act, zz + sm.bias[sm.boff[S.first + i] + (rb - RB.r0) * PN_TS + tid]);
            }
            const u64 w = pack_tv(a, tag_t);
            st_tv_gpu(Ccur + L.cache_out + row, w);
            if (last && h < P.D) {
              if (rb == RB.r0) {
                if (tid == 0) pn_wait_cnt(S.act_credit, u64(S.G_down) * u64(t), P);  // downstream read slot t&1 at t-1
                __syncwarp(0xffffu);
              }
              if (S.down_remote) st_tv_sys(S.peer_inslot[t & 1] + row, w);
              else st_tv_gpu(S.peer_inslot[t & 1] + row, w);
            }
            if (net_last && row < P.F) {
              pn_outs(P, ti)[row] = a;
              if (P.loss == 0 && y) {
                const float d = a - pn_y(P, y, yt, sid, row);
                lsum = fmaf(d, d, lsum);
              }
            }
          }
        }
        ++fdone;
        if (RB.r0 == RB.r1) cons_sync(NCT);  // no chunk loop: every read of va (input copy) is done
        if (net_last && warp == 0) {
          // MSE: this CTA's partial of sum (a - y)^2 (the epilogue divides by M*F); softmax-CE:
          // CTA 0 writes the loss after the full output is gathered (backward, or below)
          lsum = warp_sum(lsum);
          if (lane == 0) pn_lpart(P, ti)[c] = lsum;
        }
        PN_TR(4);
        if (net_last && P.loss == 1 && !P.learn && c == 0 && y) {
          // inference wave with softmax-CE: CTA 0 gathers the output for the loss
          PV vo[1] = {PV{Ccur + L.cache_out, tag_t, 0}};
          pn_gather<1>(vo, L.C * PN_TS, P, [&](int j, const float (&x)[1][2]) {
            sm.va[j] = x[0][0];
            sm.va[j + 1] = x[0][1];
          });
          cons_sync(NCT);
          float mx = -INFINITY;
          for (int f = tid; f < P.F; f += NCT) mx = fmaxf(mx, sm.va[f]);
          mx = pn_cta_red(mx, true, sm);
          float se = 0.f;
          for (int f = tid; f < P.F; f += NCT) se += expf(sm.va[f] - mx);
          se = pn_cta_red(se, false, sm);
          if (tid == 0) {
            const float y0 = pn_y(P, y, yt, sid, 0);
            const int tgt = int(y0);
            if (!(y0 >= 0.f && y0 < float(P.F) && float(tgt) == y0)) {
              atomicMin(P.bad_target, sid);
              pn_lpart(P, ti)[0] = 0.f;
            } else {
              pn_lpart(P, ti)[0] = mx + logf(se) - sm.va[tgt];
            }
          }
        }
      }
      if (!P.learn) continue;
      // ----------------------------------------------------------------- backward
      const bool upd_now = pn_upd(P, h, t);
      const long long Ct = pn_ct(P, h, t);
      u64* Cc = S.cache[cmod4(Ct)];
      // Adam bias corrections of this stage's k-th update (k counts from the warm-up gate;
      // in double, as pt::tick_kernel)
      float c1 = 1.f, c2 = 1.f;
      if (OPT == 1 && upd_now) {
        const double k = double(t - (2LL * P.D - h - 1) + 1);
        c1 = float(1.0 / (1.0 - pow(P.b1d, k)));
        c2 = float(1.0 / (1.0 - pow(P.b2d, k)));
      }
      for (int i = S.k - 1; i >= 0; --i) {
        const PLayer& L = s_layers[S.first + i];
        const int nout = L.R * PN_TS;
        const int* bk = sm.blk + 6 * (S.first + i);
        const Rows RB{bk[0], bk[1]};
        const Rows CB{bk[2], bk[3]};
        const int ncol = (CB.r1 - CB.r0) * PN_TS;
        const bool need_gin = !(h == 1 && i == 0);  // the network's first layer publishes no g_in
        // weight chunks: every layer with a g_in, and the first layer when it updates in the
        // backward (Adam); SGD defers the first layer's update to the next forward (L.bw == 0)
        const bool do_chunks = need_gin || (OPT == 1 && L.bw);
        const bool stage_last = i == S.k - 1;
        const bool loss_src = stage_last && h == P.D;
        PN_TR(11);
        // a_hat_t of own columns (this layer's input at the cache tick): loads issued here,
        // resolved after the gather
        const u64* ahp = (do_chunks && upd_now) ? Cc + L.cache_in + CB.r0 * PN_TS : nullptr;
        const u64 ah = (ahp && tid < ncol) ? ld_tv_gpu(ahp + tid) : 0ull;
        // delta_l(t): the next layer's published vector, or (stage's last layer) the loss
        // gradient / the downstream stage's g_in times act'; delta_l(t-1) for the rebuild
        PV vg[2];
        vg[0] = PV{nullptr, 0u, 0};
        vg[1] = PV{nullptr, 0u, 0};
        if (loss_src) {
          vg[0] = PV{Cc + L.cache_out, tag_t, 0};  // the output a_L(t) (Ct = t at stage D)
        } else if (stage_last) {
          vg[0] = PV{S.gslot[(t - 1) & 1], tag_of_tick(t - 1), S.down_remote};
          vg[1] = PV{Cc + L.cache_out, tag_of_tick(Ct), 0};
        } else {
          vg[0] = PV{s_layers[S.first + i + 1].gin[t & 1], tag_t, 0};
        }
        const long long sid = t - (P.D - 1);
        const float* y = loss_src ? pn_target(P, sid, P.loss == 1 ? 1 : P.F) : nullptr;
        const u64* yt = loss_src ? pn_ytag(P, sid) : nullptr;
        // resident MSE: the targets join the gather as a second tagged vector
        if (loss_src && yt && P.loss == 0) vg[1] = PV{yt, tag_of_tick(sid), 0};
        const float g_scale = 2.f / float(P.F);  // d mse / d a (M = 1)
        const float nlr = -P.lr;
        pn_gather<2>(vg, nout, P, [&](int j, const float (&x)[2][2]) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            float d;
            if (loss_src) {
              const float a = x[0][e];
              if (P.loss == 1) d = a;  // raw output: softmax below
              else d = (y && j + e < P.F) ? g_scale * (a - (yt ? x[1][e] : y[j + e])) * dact_fn(L.act, a) : 0.f;
            } else if (stage_last) {
              d = x[0][e] * dact_fn(L.act, x[1][e]);
            } else {
              d = x[0][e];
            }
            sm.va[j + e] = d;
          }
        });
        if (ahp) pn_small(ahp, ncol, ah, tag_of_tick(Ct), 1.f, sm.sah, P);
        cons_sync(NCT);
        if (stage_last && !loss_src && tid == 0) red_relaxed_sys(S.peer_g_credit, 1);  // gslot read
        if (loss_src && P.loss == 1) {
          // softmax cross-entropy: every CTA derives the whole delta in the
          // same fixed order; CTA 0 records -log softmax[target]
          float mx = -INFINITY;
          for (int f = tid; f < P.F; f += NCT) mx = fmaxf(mx, sm.va[f]);
          mx = pn_cta_red(mx, true, sm);
          float se = 0.f;
          for (int f = tid; f < P.F; f += NCT) se += expf(sm.va[f] - mx);
          se = pn_cta_red(se, false, sm);
          const float lse = mx + logf(se);
          int tgt = -1;
          bool ok = false;
          if (y) {
            const float y0 = pn_y(P, y, yt, sid, 0);
            tgt = int(y0);
            ok = y0 >= 0.f && y0 < float(P.F) && float(tgt) == y0;
          }
          if (c == 0 && tid == 0 && y) {
            if (!ok) atomicMin(P.bad_target, sid);
            pn_lpart(P, ti)[0] = ok ? lse - sm.va[tgt] : 0.f;
          }
          cons_sync(NCT);  // thread 0 read va[tgt] before it is rewritten
          for (int f = tid; f < nout; f += NCT) {
            const float a = sm.va[f];
            sm.va[f] = (y && f < P.F) ? (expf(a - lse) - (f == tgt ? 1.f : 0.f)) * dact_fn(L.act, a) : 0.f;
          }
          cons_sync(NCT);
        }
        // the stage's last layer keeps its delta for the next tick (own forward rows); the bias step
        for (int j = RB.r0 * PN_TS + tid; j < RB.r1 * PN_TS; j += NCT) {
          const float d = sm.va[j];
          if (stage_last && !L.bw) L.dpl[size_t(t & 1) * nout + j] = d;  // forward-applied update at t+1
          if (upd_now && j < L.n_out) {
            float* bp = sm.bias + sm.boff[S.first + i] + (j - RB.r0 * PN_TS);
            if (OPT == 1) {
              float mm = __ldcg(L.mb + j), vv = __ldcg(L.vb + j);
              *bp = pn_adam1(*bp, d, mm, vv, P, c1, c2);
              __stcg(L.mb + j, mm);
              __stcg(L.vb + j, vv);
            } else {
              *bp = fmaf(nlr, d, *bp);
            }
          }
        }
        PN_TR(13);
        if (do_chunks) {
          const bool to_peer = (i == 0);  // first layer of stage h > 1: g_in goes upstream (no act')
          const PLayer* Lp = to_peer ? nullptr : &s_layers[S.first + i - 1];
          for (int cb = CB.r0; cb < CB.r1; ++cb) {
            // a_{l-1}(Ct) of the 16 published columns (rows of layer l-1), for act'
            u64 ap = 0;
            const u64* app = nullptr;
            if (!to_peer && tid < PN_TS) {
              app = Cc + L.cache_in + cb * PN_TS + tid;
              ap = ld_tv_gpu(app);
            }
            const float4 ah4 = upd_now ? lds4(sm.sah + (cb - CB.r0) * PN_TS + f4 * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            float* Wn = L.W[int((t + 1) & 1)] + size_t(cb) * PN_TILE + toff;  // W^(t+1), this column panel
            // Adam moments of this column panel (column-panel-major: consecutive tiles)
            float* Mn = OPT == 1 ? L.mW + size_t(cb) * L.R * PN_TILE + toff : nullptr;
            float* Vn = OPT == 1 ? L.vW + size_t(cb) * L.R * PN_TILE + toff : nullptr;
            for (int j0 = 0; j0 < L.R; j0 += PN_CT) {
              const int nt = min(PN_CT, L.R - j0);
              const int slot = pn_take(sm, cslot, cphase, P);
              PN_TRC(8);
              const float* wb = sm.ring + size_t(slot) * PN_SLOT_FLOATS + toff;
              const float* dl = sm.va + j0 * PN_TS + tr;
              float* gd = Wn + size_t(j0) * L.C * PN_TILE;
              if (OPT == 1 && upd_now) {
                // the chunk's moments arrived in the next two ring slots (pn_producer)
                const int mslot = pn_take(sm, cslot, cphase, P);
                const int vslot = pn_take(sm, cslot, cphase, P);
                PN_TRC(50);
                const float* ms = sm.ring + size_t(mslot) * PN_SLOT_FLOATS + toff;
                const float* vs = sm.ring + size_t(vslot) * PN_SLOT_FLOATS + toff;
                float* md = Mn + size_t(j0) * PN_TILE;
                float* vd = Vn + size_t(j0) * PN_TILE;
                if (need_gin) {
                  if (nt == PN_CT) pn_bchunk_adam<true, true>(wb, dl, ah4, gd, ms, vs, md, vd, L.C, nt, tg, acc, P, c1, c2);
                  else pn_bchunk_adam<false, true>(wb, dl, ah4, gd, ms, vs, md, vd, L.C, nt, tg, acc, P, c1, c2);
                } else {
                  if (nt == PN_CT) pn_bchunk_adam<true, false>(wb, dl, ah4, gd, ms, vs, md, vd, L.C, nt, tg, acc, P, c1, c2);
                  else pn_bchunk_adam<false, false>(wb, dl, ah4, gd, ms, vs, md, vd, L.C, nt, tg, acc, P, c1, c2);
                }
                PN_TRC(51);
                __syncwarp();
                if (lane == 0) {
                  mbar_arrive(&sm.empty[mslot]);
                  mbar_arrive(&sm.empty[vslot]);
                }
              } else if (upd_now) {
                if (nt == PN_CT) pn_bchunk<true, true>(wb, dl, nlr, ah4, gd, L.C, nt, tg, acc);
                else pn_bchunk<true, false>(wb, dl, nlr, ah4, gd, L.C, nt, tg, acc);
              } else {
                if (nt == PN_CT) pn_bchunk<false, true>(wb, dl, nlr, ah4, gd, L.C, nt, tg, acc);
                else pn_bchunk<false, false>(wb, dl, nlr, ah4, gd, L.C, nt, tg, acc);
              }
              __syncwarp();
              if (lane == 0) mbar_arrive(&sm.empty[slot]);
            }
            if (OPT == 1 && !need_gin) continue;  // the network's first layer (Adam): update only
            // column sums over tr (lane bits 2-4, warp bit 0) and tg (warp bits 1-2)
            float g[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              g[e] += __shfl_xor_sync(0xffffffffu, g[e], 4);
              g[e] += __shfl_xor_sync(0xffffffffu, g[e], 8);
              g[e] += __shfl_xor_sync(0xffffffffu, g[e], 16);
            }
            float* rd = sm.red + ((cb - CB.r0) & 1) * 128;
            if (lane < 4) {
#pragma unroll
              for (int e = 0; e < 4; ++e) rd[warp * PN_TS + lane * 4 + e] = g[e];
            }
            cons_sync(NCT);
            if (tid < PN_TS) {
              float o = 0.f;
#pragma unroll
              for (int w = 0; w < NCW; ++w) o += rd[w * PN_TS + tid];
              const int col = cb * PN_TS + tid;
              if (to_peer) {
                const u64 wv = pack_tv(o, tag_t);
                if (cb == CB.r0) {
                  if (tid == 0) pn_wait_cnt(S.g_credit, u64(S.G_up) * u64(t), P);  // upstream read slot t&1 at t-1
                  __syncwarp(0xffffu);
                }
                if (S.up_remote) st_tv_sys(S.peer_gslot[t & 1] + col, wv);
                else st_tv_gpu(S.peer_gslot[t & 1] + col, wv);
              } else {
                // delta of layer l-1: g_in * act'(a_{l-1}(Ct)) (padding columns: g_in = 0)
                const float av = pn_resolve(app, ap, tag_of_tick(Ct), false, P);
                const float d = o * dact_fn(Lp->act, av);
                st_tv_gpu(L.gin[t & 1] + col, pack_tv(d, tag_t));
                if (!Lp->bw) Lp->dpl[size_t(t & 1) * (Lp->R * PN_TS) + col] = d;  // forward-applied update at t+1
              }
            }
          }
        }
        // no chunk loop (or none with a reduction): the delta store's reads of va are done
        if (!need_gin || CB.r0 == CB.r1) cons_sync(NCT);
        PN_TR(14);
      }
    }
    // end of tick: the tick barrier arrival (this tick's plain stores, and its weight stores
    // fenced for the producers' TMA loads, are published with it)
    if (P.learn) fence_proxy_async_global();
    cons_sync(NCT);
    if (P.resident) {
      if (warp == 0) {
        // outputs went to host memory: make them visible system-wide before arriving; the
        // last CTA to arrive completes the step for the host (its warp 0 sums the loss)
        bool last = false;
        if (lane == 0) {
          __threadfence_system();
          const u64 old = atomicAdd(reinterpret_cast<unsigned long long*>(P.tick_end), 1ull);
          last = old + 1 == u64(G) * u64(t + 1);
        }
        if (__shfl_sync(0xffffffffu, last, 0) && P.res_last) pn_resident_done(P, t, ti, lane);
      }
    } else if (tid == 0) {
      __threadfence();
      red_release_gpu(P.tick_end, 1);
    }
    PN_TR(20);
  }
#undef PN_TR
#undef PN_TRC
  if (P.learn && P.lr != 0.f) {
    cons_sync(NCT);
    for (int l = 0; l < P.n_layers; ++l) {
      const PLayer& L = s_layers[l];
      const Rows RB{sm.blk[6 * l], sm.blk[6 * l + 1]};
      for (int j = tid; j < (RB.r1 - RB.r0) * PN_TS; j += NCT) {
        const int row = RB.r0 * PN_TS + j;
        if (row < L.n_out) L.b[row] = sm.bias[sm.boff[l] + j];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// layout conversion (pt_set_params / pt_get_params)
// ---------------------------------------------------------------------------
// row-major [n_out][n_in] -> tiled (zero padding)
__global__ void pn_to_tiles(const float* __restrict__ src, float* __restrict__ dst, int n_out, int n_in, int R,
                            int C) {
  const size_t total = size_t(R) * C * PN_TILE;
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    const size_t tile = e / PN_TILE;
    const int inner = int(e % PN_TILE);
    const int rb = int(tile / C), cb = int(tile % C);
    const int row = rb * PN_TS + inner / PN_TS, col = cb * PN_TS + inner % PN_TS;
    dst[e] = (row < n_out && col < n_in) ? src[size_t(row) * n_in + col] : 0.f;
  }
}
// tiled -> row-major, with the pending update of the last tick applied when sdel != null:
// w + (-lr * delta[row]) * a_hat[col], the exact fmaf the next forward would apply
__global__ void pn_from_tiles(const float* __restrict__ src, float* __restrict__ dst, int n_out, int n_in, int C,
                              const float* sdel, const float* ahat, float lr) {
  const size_t total = size_t(n_out) * n_in;
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    const int row = int(e / n_in), col = int(e % n_in);
    float w = src[(size_t(row / PN_TS) * C + col / PN_TS) * PN_TILE + (row % PN_TS) * PN_TS + col % PN_TS];
    if (sdel) w = fmaf(-lr * sdel[row], ahat[col], w);
    dst[e] = w;
  }
}

}  // namespace pt
