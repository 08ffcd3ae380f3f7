// partime_capi.cu: host side of libpartime_b200.so (C ABI in include/partime_b200.h).
//
// The handle owns, for every stage local to this process (all on one device):
//   - padded fp32 weights [n_out, ld_in] and biases, updated in place by the kernel;
//   - a comm block (stage-input slots x2, stage-output-gradient slots x2 and four
//     counters). It is cudaMalloc'd on its own so it can be exported over CUDA IPC
//     to the neighbouring process (one process per GPU; NVLink peer stores);
//   - three activation-cache slots, g_in partial buffers and step counters.
// All of it is zeroed at create: warm-up ticks read zero slots.
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <chrono>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "partime_b200.h"
#include "pt_kernels.cuh"
#include "pt_tile.cuh"
#include "pt_panel.cuh"

using pt::u64;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                            \
  do {                                                                            \
    cudaError_t e_ = (expr);                                                      \
    if (e_ != cudaSuccess)                                                        \
      return fail(PT_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define PT_TRY(expr)          \
  do {                        \
    int r_ = (expr);          \
    if (r_ != PT_OK) return r_; \
  } while (0)

constexpr int32_t PT_IPC_MAGIC = 0x50544231;  // "PTB1"

// Padded row stride: a power of two >= 128. A 32 KB chunk is then exactly 64
// (row, 128-float segment) pairs, and every column has a fixed owner thread.
int pad_dim(int n) {
  int p = 128;
  while (p < n) p <<= 1;
  return p;
}

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Comm block of one stage (lives on that stage's GPU). The layout is a pure function
// of (M, ld0, ldk), so every process can address a neighbour's block from the config.
// Slots hold tagged 8-byte words {value, tick tag}; the two credit counters sit on
// separate 128-B lines.
struct CommLayout {
  static constexpr size_t ACT_CREDIT = 0, G_CREDIT = 128, DATA = 256;
  size_t inslot_bytes = 0, gslot_bytes = 0, total = 0;
  CommLayout() = default;
  CommLayout(int M, int ld0, int ldk) {
    inslot_bytes = align_up(size_t(M) * ld0 * 8, 256);
    gslot_bytes = align_up(size_t(M) * ldk * 8, 256);
    total = DATA + 2 * inslot_bytes + 2 * gslot_bytes;
  }
  size_t inslot(int p) const { return DATA + size_t(p) * inslot_bytes; }
  size_t gslot(int p) const { return DATA + 2 * inslot_bytes + size_t(p) * gslot_bytes; }
};

// Tile-path comm block of one stage: four counters on separate 128-B lines, then plain
// fp32 slots inslot[2][M][n0] and gslot[2][M][nk]. Counters (ticks, monotonic):
// IN_READY  inslot writes published by the upstream stage;
// G_READY   gslot writes published by the downstream stage;
// ACT_CREDIT ticks whose inslot the downstream stage has finished reading (upstream's block);
// G_CREDIT   ticks whose gslot the upstream stage has finished reading (downstream's block).
struct TileComm {
  static constexpr size_t IN_READY = 0, G_READY = 128, ACT_CREDIT = 256, G_CREDIT = 384, DATA = 512;
  size_t in_bytes = 0, g_bytes = 0, total = 0;
  TileComm() = default;
  TileComm(int M, int n0, int nk) {
    in_bytes = align_up(size_t(M) * n0 * 4, 256);
    g_bytes = align_up(size_t(M) * nk * 4, 256);
    total = DATA + 2 * in_bytes + 2 * g_bytes;
  }
  size_t inslot(int j) const { return DATA + size_t(j) * in_bytes; }
  size_t gslot(int j) const { return DATA + 2 * in_bytes + size_t(j) * g_bytes; }
};

struct IpcBlob {
  int32_t magic, abi, stage, G, M, ld0, ldk, pad_;
  int64_t comm_bytes;
  int64_t pid;       // exporting process: a same-process import uses dev_ptr directly
  uint64_t dev_ptr;  // (two handles in one process, e.g. one per GPU or per stream)
  cudaIpcMemHandle_t handle;
};

struct LayerHost {
  int n_in = 0, n_out = 0, ld_in = 0, ld_out = 0, act = 0;
  float* W = nullptr;
  float* b = nullptr;
  float* mW = nullptr;  // Adam state, allocated only for the Adam optimizer
  float* vW = nullptr;
  float* mb = nullptr;
  float* vb = nullptr;
  u64* part[2] = {nullptr, nullptr};
  int rows_per_chunk = 0;
  int cache_in = 0, cache_out = 0;
  // batch-1 panel path (pt_panel.cuh): 16 x 16-tiled weights in two buffers, g_in vectors,
  // delta store, and the tick of the last pt_set_params (discards the pending update)
  int R = 0, C = 0;
  float* Wt[2] = {nullptr, nullptr};
  u64* gin[2] = {nullptr, nullptr};
  float* dpl = nullptr;
  long long set_tick = 0;
  int bw = 0;  // learning and the backward reads W: the backward applies the update (pt_panel.cuh)
};

struct StageHost {
  int h = 0;                    // 1-based global stage index
  int first_global = 0, k = 0;  // global index of first layer, layer count
  int first_local = 0;          // index into the handle's layer array
  int ld0 = 0, ldk = 0;
  char* comm = nullptr;  // own comm block
  u64* cache = nullptr;  // 3 slots of tagged activations (4 on the panel path)
  float* pcache = nullptr;  // panel path: plain copies of the 4 slots
  size_t cache_words = 0;
  char* up = nullptr;    // upstream stage's comm block (local or IPC-mapped), h > 1
  char* down = nullptr;  // downstream stage's comm block, h < D
  int G_up = 0, G_down = 0;
  bool up_remote = false, down_remote = false;
  int cta0 = 0, ncta = 0;  // the CTAs that run this stage (all, unless stages run concurrently)
  // micro-batch tile path (plain fp32 buffers): cache[2] slots of a_0..a_k, inslot[2], gslot[2]
  float* tcache = nullptr;
  size_t tcache_floats = 0;
  char* tcomm = nullptr;  // tile comm block (TileComm layout), exported over CUDA IPC
  char* tup = nullptr;    // upstream / downstream stages' tile comm blocks (local or IPC-mapped)
  char* tdown = nullptr;
  int n0 = 0, nk = 0;
};

}  // namespace

struct pt_pipeline {
  int L = 0, D = 0, M = 1, loss = 0, opt = 0, learn = 1, act_delay = 1;
  float lr = 0.f;
  std::vector<int> dims, act, sfl;
  int local_first = 0, local_count = 0;  // 0-based stage index range owned here
  int G = 0, device = 0;
  unsigned long long timeout_ns = 0;
  bool fast = true;
  std::vector<LayerHost> layers;  // local layers, global order
  int layer_base = 0;             // global index of layers[0]
  std::vector<StageHost> stages;
  pt::LayerDev* d_layers = nullptr;
  pt::StageDev* d_stages = nullptr;
  u64* d_tick_end = nullptr;
  // local stages on disjoint SM partitions (PT_CONC=0: every CTA runs every stage in turn)
  bool conc = false;
  // Work issued on the legacy default stream (cudaMemset of new buffers, cudaMemcpy of
  // parameters and descriptors) is not ordered before the handle's non-blocking stream, and
  // a pageable H2D cudaMemcpy may return before its DMA lands: the next launch waits for it.
  // Without that, a kernel could read recycled memory that still holds another pipeline's
  // tagged words (a stale tag can match a tick) or weights that are not there yet.
  bool legacy_dirty = true;
  std::vector<int> stage_cta0, stage_ncta;  // per local stage
  int layer_ncta(size_t li) const {         // CTAs sharing local layer li's rows
    for (int s = 0; s < local_count; ++s)
      if (int(li) + layer_base >= sfl[local_first + s] && int(li) + layer_base < sfl[local_first + s + 1])
        return stage_ncta[s];
    return G;
  }
  int* d_status = nullptr;
  long long* d_first_bad = nullptr;
  long long* d_bad_target = nullptr;
  float* xs_pad = nullptr;
  size_t xs_cap = 0;  // ticks
  float* ys_stage = nullptr;
  size_t ys_cap = 0;
  float* outs_stage = nullptr;
  size_t outs_cap = 0;
  float* loss_part = nullptr;
  size_t lp_cap = 0;
  float* losses_stage = nullptr;
  size_t ls_cap = 0;
  uint8_t* valid_stage = nullptr;
  size_t vs_cap = 0;
  float* yhist = nullptr;
  int yh = 1;
  cudaStream_t own_stream = nullptr, stream = nullptr;
  // pinned staging of small host-buffer calls (pt_step): pageable copies block the host for
  // each transfer; one memcpy into pinned memory and truly asynchronous copies do not
  float* pin = nullptr;
  size_t pin_floats = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  bool timed = false;
  long long t_next = 0;
  bool broken = false;
  std::atomic<int> busy{0};
  std::vector<void*> ipc_opened;
  std::vector<void*> allocs;
  u64* d_trace = nullptr;
  int trace_cap = 0, trace_cta = 0;
  int pf_chunks = 0, split_bytes = 32768, maxfly = 0, wb_mode = 0;  // tunables (env PT_PF_CHUNKS / PT_SPLIT_BYTES)
  // shared-memory plan (see pt_kernels.cuh): ring slots first, then the small buffers
  int nslot = 0, slot_floats = 0, qw = 0, act_off = 0, spart_off = 0, spart_floats = 0, delta_off = 0,
      red_off = 0, scal_off = 0, bar_off = 0, flags_off = 0, desc_off = 0, bias_off = 0, smem_bytes = 0;
  int dbg = 0;                                        // diagnostics (env PT_DBG)
  // batch-1 panel path (pt_panel.cuh): M == 1, SGD
  bool panel = false;
  pt::PLayer* d_players = nullptr;
  pt::PStage* d_pstages = nullptr;
  CUtensorMap* d_pmaps = nullptr;
  float* rowbuf = nullptr;  // row-major staging of pt_set_params / pt_get_params
  size_t rowbuf_floats = 0;
  int pn_nslot = 0, pn_va = 0, pn_vb = 0, pn_sown = 0, pn_sah = 0, pn_red = 0, pn_bar = 0, pn_desc = 0, pn_bias = 0,
      pn_smem = 0, pn_pf = 8;
  // micro-batch tensor-core path (pt_tile.cuh): M = 16, 32 or 64, widths % 256 == 0
  bool tile = false;
  int t_smem = 0, t_maxn = 0;
  float* t_part = nullptr;
  float* t_delta = nullptr;
  float* t_ce = nullptr;  // softmax-CE partials of the tile path [G][M][2]
  u64* t_bars = nullptr;  // [0] grid barrier, [16] weight write-back counter
  CUtensorMap* d_tmaps = nullptr;
  pt::TLayer* d_tlayers = nullptr;
  pt::TStage* d_tstages = nullptr;
  std::vector<pt::TLayer> t_layers_host;
  int policy = 0;                                     // weight-load L2 hint (env PT_POLICY)
  // host outputs of a PT_HOST run enqueued without waiting (multi-device handles launch every
  // part before waiting for any): copied out of the pinned staging area at finish_impl
  struct Pending {
    bool active = false;
    int64_t n = 0;
    float *outs = nullptr, *losses = nullptr, *pin_o = nullptr, *pin_l = nullptr;
    uint8_t *valid = nullptr, *pin_v = nullptr;
    size_t st_o = 0, st_l = 0, st_v = 0;
  } pend;
  // multi-device handle (pt_config.device_of_stage): one part per run of stages on one device,
  // each a complete single-device handle; the parts' neighbour stages exchange through peer
  // memory. Empty for a single-device handle.
  std::vector<pt_pipeline*> parts;
  bool group() const { return !parts.empty(); }
  // resident pt_step (pt_panel.cuh PParams::resident): one mapped host block holding the
  // completion record, the request words and the x / target / output rings
  struct Resident {
    bool on = false;
    long long t_start = 0;
    int ring = 0, ldx = 0, fy = 0;
    size_t bytes = 0;
    void* host = nullptr;
    ptrdiff_t dev_off = 0;  // device alias of the mapped block minus its host address
    pt::PResDone* done = nullptr;
    long long* req = nullptr;
    int* flag = nullptr;
    float *x = nullptr, *y = nullptr, *out = nullptr;
    u64* xin = nullptr;
    u64* ytag = nullptr;  // tagged device targets [ring][ldy]
    int ldy = 0;
    long long* relay = nullptr;
    float* lpart = nullptr;
  } res;

  bool has_first() const { return local_first == 0; }
  bool has_last() const { return local_first + local_count == D; }
  int F() const { return dims[L]; }
  // target width: the output vector for MSE, one class index per sample for softmax-CE
  int Fy() const { return loss == PT_LOSS_SOFTMAX_CE ? 1 : dims[L]; }
  int stage_ld0(int s0) const { return pad_dim(dims[sfl[s0]]); }      // s0: 0-based stage
  int stage_ldk(int s0) const { return pad_dim(dims[sfl[s0 + 1]]); }
  CommLayout layout_of(int s0) const { return CommLayout(M, stage_ld0(s0), stage_ldk(s0)); }
  TileComm tile_layout_of(int s0) const { return TileComm(M, dims[sfl[s0]], dims[sfl[s0 + 1]]); }
};

namespace {

struct BusyGuard {
  pt_pipeline* p;
  bool ok;
  explicit BusyGuard(pt_pipeline* p_) : p(p_) {
    int z = 0;
    ok = p->busy.compare_exchange_strong(z, 1);
  }
  ~BusyGuard() {
    if (ok) p->busy.store(0);
  }
};

// Every entry point runs on the handle's device, whatever the caller's current device is
// (a multi-device handle drives several devices from one thread).
struct DevGuard {
  int old = -1;
  explicit DevGuard(int dev) {
    if (cudaGetDevice(&old) != cudaSuccess) old = -1;
    if (old != dev) cudaSetDevice(dev);
  }
  ~DevGuard() {
    int cur = -1;
    if (old >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != old) cudaSetDevice(old);
  }
};

int dev_alloc(pt_pipeline* p, void** ptr, size_t bytes) {
  if (bytes == 0) bytes = 16;
  CUDA_TRY(cudaMalloc(ptr, bytes));
  CUDA_TRY(cudaMemset(*ptr, 0, bytes));
  p->legacy_dirty = true;
  p->allocs.push_back(*ptr);
  return PT_OK;
}

void dev_free(pt_pipeline* p, void* ptr) {
  if (!ptr) return;
  for (auto& a : p->allocs)
    if (a == ptr) a = nullptr;
  cudaFree(ptr);
}

// grow a staging buffer (contents not preserved; zeroed so padding stays 0)
template <typename T>
int ensure(pt_pipeline* p, T** buf, size_t* cap, size_t need, size_t elems_per) {
  if (*cap >= need && *buf) return PT_OK;
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  dev_free(p, *buf);
  *buf = nullptr;
  size_t n = std::max<size_t>(need, 64);
  PT_TRY(dev_alloc(p, reinterpret_cast<void**>(buf), n * elems_per * sizeof(T)));
  // the buffer is filled on the handle's stream right away: its zeroing (legacy stream) must
  // not land after that
  CUDA_TRY(cudaStreamSynchronize(0));
  *cap = n;
  return PT_OK;
}

int upload_panel_desc(pt_pipeline* p);
int group_finish(pt_pipeline* p);

int upload_desc(pt_pipeline* p) {
  std::vector<pt::LayerDev> ld(p->layers.size());
  for (size_t i = 0; i < p->layers.size(); ++i) {
    const LayerHost& h = p->layers[i];
    pt::LayerDev& d = ld[i];
    d.W = h.W;
    d.b = h.b;
    d.mW = h.mW;
    d.vW = h.vW;
    d.mb = h.mb;
    d.vb = h.vb;
    d.part[0] = h.part[0];
    d.part[1] = h.part[1];
    d.n_in = h.n_in;
    d.n_out = h.n_out;
    d.ld_in = h.ld_in;
    d.ld_out = h.ld_out;
    d.act = h.act;
    d.rows_per_chunk = h.rows_per_chunk;
    d.cache_in = h.cache_in;
    d.cache_out = h.cache_out;
  }
  std::vector<pt::StageDev> sd(p->stages.size());
  for (size_t s = 0; s < p->stages.size(); ++s) {
    const StageHost& h = p->stages[s];
    const int s0 = h.h - 1;
    pt::StageDev& d = sd[s];
    memset(&d, 0, sizeof(d));
    d.h = h.h;
    d.first = h.first_local;
    d.k = h.k;
    d.G_up = h.G_up;
    d.G_down = h.G_down;
    d.cta0 = h.cta0;
    d.ncta = h.ncta;
    d.up_remote = h.up_remote ? 1 : 0;
    d.down_remote = h.down_remote ? 1 : 0;
    d.ld0 = h.ld0;
    d.ldk = h.ldk;
    for (int j = 0; j < 3; ++j) d.cache[j] = h.cache + size_t(j) * h.cache_words;
    const CommLayout own = p->layout_of(s0);
    for (int j = 0; j < 2; ++j) {
      d.inslot[j] = reinterpret_cast<u64*>(h.comm + own.inslot(j));
      d.gslot[j] = reinterpret_cast<u64*>(h.comm + own.gslot(j));
    }
    d.act_credit = reinterpret_cast<u64*>(h.comm + CommLayout::ACT_CREDIT);
    d.g_credit = reinterpret_cast<u64*>(h.comm + CommLayout::G_CREDIT);
    if (h.down) {
      const CommLayout dn = p->layout_of(s0 + 1);
      for (int j = 0; j < 2; ++j) d.peer_inslot[j] = reinterpret_cast<u64*>(h.down + dn.inslot(j));
      d.peer_g_credit = reinterpret_cast<u64*>(h.down + CommLayout::G_CREDIT);
    }
    if (h.up) {
      const CommLayout upl = p->layout_of(s0 - 1);
      for (int j = 0; j < 2; ++j) d.peer_gslot[j] = reinterpret_cast<u64*>(h.up + upl.gslot(j));
      d.peer_act_credit = reinterpret_cast<u64*>(h.up + CommLayout::ACT_CREDIT);
    }
  }
  CUDA_TRY(cudaMemcpy(p->d_layers, ld.data(), ld.size() * sizeof(pt::LayerDev), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(p->d_stages, sd.data(), sd.size() * sizeof(pt::StageDev), cudaMemcpyHostToDevice));
  p->legacy_dirty = true;
  if (p->panel) return upload_panel_desc(p);
  return PT_OK;
}

int validate(const pt_config* c, std::string* why) {
  auto bad = [&](const std::string& s) {
    *why = s;
    return PT_EINVAL;
  };
  if (!c) return bad("null config");
  if (c->n_layers < 1) return bad("n_layers must be >= 1");
  if (!c->dims || !c->act || !c->stage_first_layer) return bad("dims/act/stage_first_layer must be set");
  for (int i = 0; i <= c->n_layers; ++i)
    if (c->dims[i] < 1) return bad("dims[" + std::to_string(i) + "] must be >= 1");
  for (int i = 0; i < c->n_layers; ++i)
    if (c->act[i] < PT_ACT_NONE || c->act[i] > PT_ACT_TANH)
      return bad("act[" + std::to_string(i) + "] is not a PT_ACT_* value");
  const int D = c->n_stages;
  if (D < 1) return bad("n_stages must be >= 1");
  if (D > c->n_layers)
    return bad("D=" + std::to_string(D) + " > L=" + std::to_string(c->n_layers) + " (SPEC.md:151)");
  const int32_t* b = c->stage_first_layer;
  if (b[0] != 0 || b[D] != c->n_layers) return bad("stage plan must start at layer 0 and end at layer L");
  for (int h = 0; h < D; ++h)
    if (b[h] >= b[h + 1]) return bad("stage " + std::to_string(h + 1) + " is empty or out of order");
  if (c->batch < 1 || c->batch > pt::MAXM) return bad("batch must be in [1, " + std::to_string(pt::MAXM) + "]");
  for (int i = 0; i <= c->n_layers; ++i)
    if (pad_dim(c->dims[i]) > pt::MAX_LD)
      return bad("width " + std::to_string(c->dims[i]) + " exceeds the supported maximum 8192");
  if (c->loss != PT_LOSS_MSE && c->loss != PT_LOSS_SOFTMAX_CE) return bad("unknown loss");
  if (c->optimizer != PT_OPT_SGD && c->optimizer != PT_OPT_ADAM) return bad("unknown optimizer");
  if (c->act_delay != 0 && c->act_delay != 1) return bad("act_delay must be 0 or 1");
  if (c->local_stage_count < 0 || c->local_stage_first < 0 ||
      c->local_stage_first + c->local_stage_count > D)
    return bad("local stage range out of bounds");
  return PT_OK;
}

// Shared-memory plan: the ring gets every byte the small buffers do not need.
int plan_smem(pt_pipeline* p) {
  int max_ld = 128, maxrows = 1, sp_max = 1;
  for (size_t li = 0; li < p->layers.size(); ++li) {
    const LayerHost& Lh = p->layers[li];
    const int g = p->layer_ncta(li);
    max_ld = std::max(max_ld, Lh.ld_in);
    maxrows = std::max(maxrows, (Lh.n_out + g - 1) / g);
  }
  // Ring geometry: 4 x 32 KB slots, measured best for the 2048-wide learning tick
  // (profiles/round1_ring_sweep.md). 3 x 64 KB with one copy in flight per SM streams
  // better in the stand-alone lock-step benchmark (tools/dep_bench.cu) but is slower in
  // the tick kernel, where slots also carry the weight write-back (round 1 sweep).
  // PT_SLOT_KB (16/32/64) / PT_NSLOT / PT_MAXFLY override.
  int slot_kb = 32;
  if (const char* e = getenv("PT_SLOT_KB")) slot_kb = atoi(e);
  if (slot_kb != 16 && slot_kb != 32 && slot_kb != 64) slot_kb = 32;
  if (slot_kb == 16 && max_ld > 4096) slot_kb = 32;
  int slot_bytes = slot_kb * 1024;
  p->slot_floats = slot_bytes / 4;
  p->qw = slot_kb == 16 ? 4 : 8;  // a sub-chunk is NCW * qw (row, 128-float segment) pairs
  const int sub_floats = 128 * pt::NCW * p->qw;
  int chunk_need = 0;
  for (const LayerHost& Lh : p->layers) {
    const int nseg = Lh.ld_in / 128;
    const int sp = nseg >= p->qw ? nseg / p->qw : 1;
    sp_max = std::max(sp_max, sp);
    chunk_need = std::max(chunk_need, std::max(1, sub_floats / Lh.ld_in) * sp * p->M);
  }
  const int layer_need = (maxrows * sp_max * p->M + 1) / 2;
  p->spart_floats = std::max(chunk_need, std::min(layer_need, 4096));
  const int delta_floats = p->M * maxrows;
  const int act_floats = p->fast ? max_ld : 0;
  auto a128 = [](size_t v) { return int(align_up(v, 128)); };
  int off = 0;  // ring size decided last; lay out the tail from a fixed budget
  size_t bias_rows = 0;
  for (size_t li = 0; li < p->layers.size(); ++li)
    bias_rows += (p->layers[li].n_out + p->layer_ncta(li) - 1) / p->layer_ncta(li);
  const int n_stages_local = p->local_count;
  const int desc_bytes = a128(p->layers.size() * sizeof(pt::LayerDev) + n_stages_local * sizeof(pt::StageDev) +
                              p->layers.size() * sizeof(int));
  const int bias_bytes = a128(bias_rows * 4);
  const int tail = a128(size_t(act_floats) * 4) + a128(size_t(2 * p->spart_floats) * 4) +
                   a128(size_t(delta_floats) * 4) + a128(size_t(pt::RED_FLOATS) * 4) + a128(64 * 4) +
                   a128(2 * 16 * 8) + a128(16 * 4) + desc_bytes + bias_bytes;
  p->nslot = std::min(16, (pt::SMEM_MAX - tail) / slot_bytes);
  if (p->nslot < 3 && slot_kb == 64) {
    slot_kb = 32;
    slot_bytes = 32768;
    p->slot_floats = slot_bytes / 4;
    p->nslot = std::min(16, (pt::SMEM_MAX - tail) / slot_bytes);
  }
  int want = slot_kb == 64 ? 3 : 4;
  if (const char* e = getenv("PT_NSLOT")) want = std::max(2, atoi(e));
  p->nslot = std::min(p->nslot, want);
  p->maxfly = slot_kb == 64 ? 1 : 0;
  if (const char* e = getenv("PT_MAXFLY")) p->maxfly = std::max(0, atoi(e));
  if (!getenv("PT_SPLIT_BYTES")) p->split_bytes = slot_bytes;
  if (p->nslot < 2)
    return fail(PT_EINVAL, "shared memory too small for this layer shape (rows per CTA x batch); use a larger grid");
  off = p->nslot * slot_bytes;
  p->act_off = off;
  off += a128(size_t(act_floats) * 4);
  p->spart_off = off;
  off += a128(size_t(2 * p->spart_floats) * 4);
  p->delta_off = off;
  off += a128(size_t(delta_floats) * 4);
  p->red_off = off;
  off += a128(size_t(pt::RED_FLOATS) * 4);
  p->scal_off = off;
  off += a128(64 * 4);
  p->bar_off = off;
  off += a128(2 * 16 * 8);
  p->flags_off = off;
  off += a128(16 * 4);
  p->desc_off = off;
  off += desc_bytes;
  p->bias_off = off;
  off += bias_bytes;
  p->smem_bytes = off;
  if (p->smem_bytes > pt::SMEM_MAX) return fail(PT_EINVAL, "shared-memory plan exceeds 227 KB");
  return PT_OK;
}

// Stage descriptors of the tile path (rebuilt after every IPC import).
int upload_tile_stages(pt_pipeline* p) {
  const int M = p->M;
  std::vector<pt::TStage> ts(p->stages.size());
  for (size_t s = 0; s < p->stages.size(); ++s) {
    const StageHost& S = p->stages[s];
    const int s0 = S.h - 1;
    pt::TStage& d = ts[s];
    memset(&d, 0, sizeof(d));
    d.h = S.h;
    d.first = S.first_local;
    d.k = S.k;
    d.n0 = S.n0;
    d.nk = S.nk;
    const TileComm own = p->tile_layout_of(s0);
    for (int j = 0; j < 2; ++j) {
      d.cache[j] = S.tcache + size_t(j) * S.tcache_floats;
      d.inslot[j] = reinterpret_cast<float*>(S.tcomm + own.inslot(j));
      d.gslot[j] = reinterpret_cast<float*>(S.tcomm + own.gslot(j));
    }
    d.in_ready = reinterpret_cast<u64*>(S.tcomm + TileComm::IN_READY);
    d.g_ready = reinterpret_cast<u64*>(S.tcomm + TileComm::G_READY);
    d.act_credit = reinterpret_cast<u64*>(S.tcomm + TileComm::ACT_CREDIT);
    d.g_credit = reinterpret_cast<u64*>(S.tcomm + TileComm::G_CREDIT);
    if (S.tdown) {
      const TileComm dn = p->tile_layout_of(s0 + 1);
      for (int j = 0; j < 2; ++j) d.down_inslot[j] = reinterpret_cast<float*>(S.tdown + dn.inslot(j));
      d.peer_in_ready = reinterpret_cast<u64*>(S.tdown + TileComm::IN_READY);
      d.peer_g_credit = reinterpret_cast<u64*>(S.tdown + TileComm::G_CREDIT);
      d.down_remote = S.down_remote ? 1 : 0;
    }
    if (S.tup) {
      const TileComm upl = p->tile_layout_of(s0 - 1);
      for (int j = 0; j < 2; ++j) d.up_gslot[j] = reinterpret_cast<float*>(S.tup + upl.gslot(j));
      d.peer_g_ready = reinterpret_cast<u64*>(S.tup + TileComm::G_READY);
      d.peer_act_credit = reinterpret_cast<u64*>(S.tup + TileComm::ACT_CREDIT);
      d.up_remote = S.up_remote ? 1 : 0;
    }
    (void)M;
  }
  CUDA_TRY(cudaMemcpy(p->d_tstages, ts.data(), ts.size() * sizeof(pt::TStage), cudaMemcpyHostToDevice));
  p->legacy_dirty = true;
  return PT_OK;
}

// The tile kernel instantiation of a handle: optimizer x micro-batch (16, 32 or 64).
const void* tile_fn(const pt_pipeline* p) {
  const bool adam = p->opt == PT_OPT_ADAM;
  if (p->M == 64) return adam ? (const void*)pt::tile_kernel<1, 64> : (const void*)pt::tile_kernel<0, 64>;
  if (p->M == 32) return adam ? (const void*)pt::tile_kernel<1, 32> : (const void*)pt::tile_kernel<0, 32>;
  return adam ? (const void*)pt::tile_kernel<1, 16> : (const void*)pt::tile_kernel<0, 16>;
}

// Buffers, tensor maps and descriptors of the micro-batch tile path (pt_tile.cuh).
int setup_tile(pt_pipeline* p) {
  const int M = p->M;
  int maxn = 0;
  for (int i = 0; i <= p->L; ++i) maxn = std::max(maxn, p->dims[i]);
  p->t_maxn = maxn;
  PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&p->t_part), size_t(pt::T_Q) * M * maxn * 4));
  PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&p->t_delta), size_t(M) * maxn * 4));
  PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&p->t_bars), 32 * sizeof(u64)));
  PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&p->t_ce), size_t(p->G) * M * 2 * 4));
  std::vector<CUtensorMap> maps(2 * p->layers.size());
  std::vector<pt::TLayer> tl(p->layers.size());
  PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&p->d_tmaps), maps.size() * sizeof(CUtensorMap)));
  for (size_t i = 0; i < p->layers.size(); ++i) {
    const LayerHost& Lh = p->layers[i];
    // blocked weights [n_out/128][n_in/64][128][64] (pt_tile.cuh tl_to_blocks)
    if (pt::tc_make_tmap_blocked(&maps[2 * i], Lh.W, Lh.n_in, Lh.n_out, 32, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
        pt::tc_make_tmap_blocked(&maps[2 * i + 1], Lh.W, Lh.n_in, Lh.n_out, 32, 64,
                                 CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
      return fail(PT_ECUDA, "cuTensorMapEncodeTiled failed for layer " + std::to_string(p->layer_base + i));
    tl[i].tmf = p->d_tmaps + 2 * i;
    tl[i].tmb = p->d_tmaps + 2 * i + 1;
    tl[i].b = Lh.b;
    tl[i].mW = Lh.mW;
    tl[i].vW = Lh.vW;
    tl[i].mb = Lh.mb;
    tl[i].vb = Lh.vb;
    tl[i].ld = Lh.ld_in;
    tl[i].n_in = Lh.n_in;
    tl[i].n_out = Lh.n_out;
    tl[i].act = Lh.act;
  }
  for (size_t s = 0; s < p->stages.size(); ++s) {
    StageHost& S = p->stages[s];
    S.n0 = p->dims[S.first_global];
    S.nk = p->dims[S.first_global + S.k];
    size_t off = 0;
    for (int i = 0; i < S.k; ++i) {
      pt::TLayer& t = tl[S.first_local + i];
      t.a_in = int(off);
      off += size_t(M) * t.n_in;
      t.a_out = int(off);
    }
    off += size_t(M) * S.nk;
    S.tcache_floats = align_up(off, 64);
    PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&S.tcache), 2 * S.tcache_floats * 4));
    PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&S.tcomm), p->tile_layout_of(S.h - 1).total));
  }
  // local neighbours
  for (size_t s = 0; s < p->stages.size(); ++s) {
    if (s > 0) p->stages[s].tup = p->stages[s - 1].tcomm;
    if (s + 1 < p->stages.size()) p->stages[s].tdown = p->stages[s + 1].tcomm;
  }
  PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&p->d_tlayers), tl.size() * sizeof(pt::TLayer)));
  PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&p->d_tstages), p->stages.size() * sizeof(pt::TStage)));
  CUDA_TRY(cudaMemcpy(p->d_tmaps, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(p->d_tlayers, tl.data(), tl.size() * sizeof(pt::TLayer), cudaMemcpyHostToDevice));
  p->legacy_dirty = true;
  p->t_layers_host = tl;
  PT_TRY(upload_tile_stages(p));
  // shared memory: 1 KB alignment slack, ring, operands, update operands, reductions, barriers
  if (p->opt == PT_OPT_ADAM)
    p->t_smem = M == 16 ? pt::TCfg<16, 1>::smem_bytes() : M == 32 ? pt::TCfg<32, 1>::smem_bytes() : pt::TCfg<64, 1>::smem_bytes();
  else
    p->t_smem = M == 16 ? pt::TCfg<16>::smem_bytes() : M == 32 ? pt::TCfg<32>::smem_bytes() : pt::TCfg<64>::smem_bytes();
  if (p->t_smem > pt::SMEM_MAX) return fail(PT_EINVAL, "tile path shared-memory plan exceeds 227 KB");
  CUDA_TRY(cudaFuncSetAttribute(tile_fn(p), cudaFuncAttributeMaxDynamicSharedMemorySize, p->t_smem));
  return PT_OK;
}


// ---------------------------------------------------------------- panel path (pt_panel.cuh)
// Descriptors of the panel kernel (rebuilt after pt_set_params and every IPC import).
int upload_panel_desc(pt_pipeline* p) {
  std::vector<pt::PLayer> pl(p->layers.size());
  for (size_t i = 0; i < p->layers.size(); ++i) {
    const LayerHost& h = p->layers[i];
    pt::PLayer& d = pl[i];
    memset(&d, 0, sizeof(d));
    for (int j = 0; j < 2; ++j) {
      d.W[j] = h.Wt[j] ? h.Wt[j] : h.Wt[0];
      d.tm[j] = p->d_pmaps ? p->d_pmaps + 4 * i + j : nullptr;
      d.gin[j] = h.gin[j];
    }
    d.b = h.b;
    d.dpl = h.dpl;
    d.mW = h.mW;
    d.vW = h.vW;
    d.mb = h.mb;
    d.vb = h.vb;
    d.bw = h.bw;
    d.n_in = h.n_in;
    d.n_out = h.n_out;
    d.R = h.R;
    d.C = h.C;
    d.act = h.act;
    d.cache_in = h.cache_in;
    d.cache_out = h.cache_out;
    d.set_tick = h.set_tick;
  }
  std::vector<pt::PStage> ps(p->stages.size());
  for (size_t s = 0; s < p->stages.size(); ++s) {
    const StageHost& h = p->stages[s];
    const int s0 = h.h - 1;
    pt::PStage& d = ps[s];
    memset(&d, 0, sizeof(d));
    d.h = h.h;
    d.first = h.first_local;
    d.k = h.k;
    d.G_up = h.G_up;
    d.G_down = h.G_down;
    d.up_remote = h.up_remote ? 1 : 0;
    d.down_remote = h.down_remote ? 1 : 0;
    d.ld0 = h.ld0;
    d.ldk = h.ldk;
    for (int j = 0; j < 4; ++j) {
      d.cache[j] = h.cache + size_t(j) * h.cache_words;
      d.pcache[j] = h.pcache + size_t(j) * h.cache_words;
    }
    const CommLayout own = p->layout_of(s0);
    for (int j = 0; j < 2; ++j) {
      d.inslot[j] = reinterpret_cast<u64*>(h.comm + own.inslot(j));
      d.gslot[j] = reinterpret_cast<u64*>(h.comm + own.gslot(j));
    }
    d.act_credit = reinterpret_cast<u64*>(h.comm + CommLayout::ACT_CREDIT);
    d.g_credit = reinterpret_cast<u64*>(h.comm + CommLayout::G_CREDIT);
    if (h.down) {
      const CommLayout dn = p->layout_of(s0 + 1);
      for (int j = 0; j < 2; ++j) d.peer_inslot[j] = reinterpret_cast<u64*>(h.down + dn.inslot(j));
      d.peer_g_credit = reinterpret_cast<u64*>(h.down + CommLayout::G_CREDIT);
    }
    if (h.up) {
      const CommLayout upl = p->layout_of(s0 - 1);
      for (int j = 0; j < 2; ++j) d.peer_gslot[j] = reinterpret_cast<u64*>(h.up + upl.gslot(j));
      d.peer_act_credit = reinterpret_cast<u64*>(h.up + CommLayout::ACT_CREDIT);
    }
  }
  // stream-ordered: a pt_set_params between runs must not race the next launch's descriptor read
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  CUDA_TRY(cudaMemcpy(p->d_players, pl.data(), pl.size() * sizeof(pt::PLayer), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(p->d_pstages, ps.data(), ps.size() * sizeof(pt::PStage), cudaMemcpyHostToDevice));
  p->legacy_dirty = true;
  return PT_OK;
}

// 3-D fp32 tensor map {256 floats, C, R} over tiled weights; box {256, 1, 32}: one column
// panel piece of 32 tiles (rows beyond R are zero-filled). 0 = ok
int panel_tmap(CUtensorMap* tm, const float* base, int R, int C) {
  static pt::PFN_encodeTiled fn = nullptr;
  if (fn == nullptr) {
    void* q = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &q, cudaEnableDefault, &qr) != cudaSuccess || q == nullptr)
      return -1;
    fn = reinterpret_cast<pt::PFN_encodeTiled>(q);
  }
  const cuuint64_t dims[3] = {cuuint64_t(pt::PN_TILE), cuuint64_t(C), cuuint64_t(R)};
  const cuuint64_t strides[2] = {cuuint64_t(pt::PN_TILE) * 4, cuuint64_t(C) * pt::PN_TILE * 4};
  const cuuint32_t box[3] = {cuuint32_t(pt::PN_TILE), 1, cuuint32_t(pt::PN_CT)};
  const cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : int(r);
}

// stage (1-based) owning global layer `layer`
int stage_of_layer(const pt_pipeline* p, int layer) {
  int h = 1;
  while (h < p->D && layer >= p->sfl[h]) ++h;
  return h;
}

// Buffers, tensor maps, shared-memory plan and descriptors of the panel path.
int setup_panel(pt_pipeline* p) {
  const int G = p->G;
  int maxw = 16, maxrown = 16, maxcoln = 16;
  size_t bias_rows = 0;
  for (size_t i = 0; i < p->layers.size(); ++i) {
    LayerHost& Lh = p->layers[i];
    bias_rows += size_t((Lh.R + G - 1) / G) * pt::PN_TS;
    maxw = std::max(maxw, std::max(Lh.R, Lh.C) * pt::PN_TS);
    maxrown = std::max(maxrown, (Lh.R + G - 1) / G * pt::PN_TS);
    maxcoln = std::max(maxcoln, (Lh.C + G - 1) / G * pt::PN_TS);
    const int li_global = p->layer_base + int(i);
    if (p->learn) {
      // every layer but the network's first reads W in the backward and updates it there; the
      // first layer's update is deferred to the next forward, which needs its delta a tick later
      // (plain [2][R*16]). gin: the tagged delta of the previous layer this backward publishes.
      Lh.bw = li_global != 0 || p->opt == PT_OPT_ADAM;
      if (!Lh.bw)
        PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&Lh.dpl), size_t(2) * Lh.R * pt::PN_TS * sizeof(float)));
      else
        for (int j = 0; j < 2; ++j)
          PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&Lh.gin[j]), size_t(Lh.C) * pt::PN_TS * sizeof(u64)));
    }
  }
  if (p->learn) {
    std::vector<CUtensorMap> maps(4 * p->layers.size());  // per layer: W[0], W[1] (2 spare)
    for (size_t i = 0; i < p->layers.size(); ++i) {
      const LayerHost& Lh = p->layers[i];
      const float* src[2] = {Lh.Wt[0], Lh.Wt[1]};
      for (int j = 0; j < 2; ++j)
        if (src[j] && panel_tmap(&maps[4 * i + j], src[j], Lh.R, Lh.C))
          return fail(PT_ECUDA, "cuTensorMapEncodeTiled failed for layer " + std::to_string(p->layer_base + i));
    }
    PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&p->d_pmaps), maps.size() * sizeof(CUtensorMap)));
    CUDA_TRY(cudaMemcpy(p->d_pmaps, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
  }
  PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&p->d_players), p->layers.size() * sizeof(pt::PLayer)));
  PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&p->d_pstages), p->stages.size() * sizeof(pt::PStage)));
  for (StageHost& S : p->stages)
    PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&S.pcache), 4 * S.cache_words * sizeof(float)));
  // shared memory: ring (32 KB slots) first, then the vectors and small buffers
  auto a128 = [](size_t v) { return int(align_up(v, 128)); };
  const int desc = a128(p->layers.size() * sizeof(pt::PLayer) + p->stages.size() * sizeof(pt::PStage) +
                        p->layers.size() * 7 * sizeof(int));  // + bias offsets and block ranges
  const int bias = a128(bias_rows * 4);
  const int tail = 2 * a128(size_t(maxw) * 4) + a128(size_t(maxrown) * 4) + a128(size_t(maxcoln) * 4) +
                   a128((256 + 64 + 32) * 4) + a128(3 * pt::PN_MAXSLOT * 8) + desc + bias;
  const int slot_bytes = pt::PN_SLOT_FLOATS * 4;
  int nslot = std::min(pt::PN_MAXSLOT, (pt::SMEM_MAX - tail) / slot_bytes);
  if (const char* e = getenv("PT_NSLOT")) nslot = std::min(nslot, std::max(2, atoi(e)));
  if (nslot < 2 || (p->opt == PT_OPT_ADAM && nslot < 3))  // an Adam backward chunk holds 3 slots
    return fail(PT_EINVAL, "shared memory too small for this layer shape (rows per CTA); use a larger grid");
  p->pn_nslot = nslot;
  int off = nslot * slot_bytes;
  p->pn_va = off;
  off += a128(size_t(maxw) * 4);
  p->pn_vb = off;
  off += a128(size_t(maxw) * 4);
  p->pn_sown = off;
  off += a128(size_t(maxrown) * 4);
  p->pn_sah = off;
  off += a128(size_t(maxcoln) * 4);
  p->pn_red = off;
  off += a128((256 + 64 + 32) * 4);  // red[256], scal[64], flags[32] (PSmem)
  p->pn_bar = off;
  off += a128(3 * pt::PN_MAXSLOT * 8);
  p->pn_desc = off;
  off += desc;
  p->pn_bias = off;
  off += bias;
  p->pn_smem = off;
  if (const char* e = getenv("PT_PF_CHUNKS")) p->pn_pf = std::max(0, atoi(e));
  if (p->pn_smem > pt::SMEM_MAX) return fail(PT_EINVAL, "panel shared-memory plan exceeds 227 KB");
  CUDA_TRY(cudaFuncSetAttribute(pt::panel_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, pt::SMEM_MAX));
  CUDA_TRY(cudaFuncSetAttribute(pt::panel_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, pt::SMEM_MAX));
  return PT_OK;
}

// the weight buffer the next forward reads: W^(T) (backward-updated layers) or W^(T-1), whose
// pending update the forward applies (T = t_next)
int panel_cur(const pt_pipeline* p, const LayerHost& L) {
  return !p->learn ? 0 : L.bw ? int(p->t_next & 1) : int((p->t_next - 1) & 1);
}

int panel_rowbuf(pt_pipeline* p, size_t floats) {
  if (p->rowbuf_floats >= floats && p->rowbuf) return PT_OK;
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  dev_free(p, p->rowbuf);
  p->rowbuf = nullptr;
  PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&p->rowbuf), floats * 4));
  CUDA_TRY(cudaStreamSynchronize(0));
  p->rowbuf_floats = floats;
  return PT_OK;
}


int create_impl(const pt_config* c, pt_pipeline* p) {
  std::string why;
  if (validate(c, &why) != PT_OK) return fail(PT_EINVAL, why);
  p->L = c->n_layers;
  p->D = c->n_stages;
  p->M = c->batch;
  p->loss = c->loss;
  p->opt = c->optimizer;
  p->learn = c->learn ? 1 : 0;
  p->act_delay = c->act_delay;
  p->lr = c->lr;
  p->dims.assign(c->dims, c->dims + p->L + 1);
  p->act.assign(c->act, c->act + p->L);
  p->sfl.assign(c->stage_first_layer, c->stage_first_layer + p->D + 1);
  p->local_first = c->local_stage_count ? c->local_stage_first : 0;
  p->local_count = c->local_stage_count ? c->local_stage_count : p->D;
  p->timeout_ns = (unsigned long long)(c->timeout_ms > 0 ? c->timeout_ms : 30000) * 1000000ull;
  p->fast = (p->M == 1);
  if (const char* e = getenv("PT_PF_CHUNKS")) p->pf_chunks = std::max(0, atoi(e));
  if (const char* e = getenv("PT_DBG")) p->dbg = atoi(e);
  if (const char* e = getenv("PT_POLICY")) p->policy = atoi(e);
  if (const char* e = getenv("PT_WB")) p->wb_mode = atoi(e) ? 1 : 0;
  if (const char* e = getenv("PT_SPLIT_BYTES")) p->split_bytes = std::max(1024, atoi(e)) / 16 * 16;

  CUDA_TRY(cudaGetDevice(&p->device));
  int sms = 0, coop = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device));
  CUDA_TRY(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, p->device));
  if (!coop) return fail(PT_EUNSUPPORTED, "device does not support cooperative launch");
  {
    const void* fns[] = {(const void*)pt::tick_kernel<true, 4, false>, (const void*)pt::tick_kernel<true, 8, false>,
                         (const void*)pt::tick_kernel<false, 4, false>, (const void*)pt::tick_kernel<false, 8, false>,
                         (const void*)pt::tick_kernel<true, 4, true>, (const void*)pt::tick_kernel<true, 8, true>,
                         (const void*)pt::tick_kernel<false, 4, true>, (const void*)pt::tick_kernel<false, 8, true>};
    for (const void* f : fns)
      CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, pt::SMEM_MAX));
    // Load every kernel of the library now. With lazy module loading (the CUDA default) the
    // first launch of a kernel may wait for the kernels running on the device; a persistent
    // stage kernel waiting for a neighbour (another handle, part or process) that is itself
    // blocked in such a load would only end at the watchdog.
    const void* others[] = {(const void*)pt::panel_kernel<0>, (const void*)pt::panel_kernel<1>,
                            (const void*)pt::tile_kernel<0, 16>, (const void*)pt::tl_to_blocks,
                            (const void*)pt::tl_from_blocks,
                            (const void*)pt::tile_kernel<1, 16>, (const void*)pt::tile_kernel<0, 32>,
                            (const void*)pt::tile_kernel<1, 32>, (const void*)pt::tile_kernel<0, 64>,
                            (const void*)pt::tile_kernel<1, 64>,
                            (const void*)pt::epilogue_kernel, (const void*)pt::pn_to_tiles,
                            (const void*)pt::pn_from_tiles};
    cudaFuncAttributes fa;
    for (const void* f : others) CUDA_TRY(cudaFuncGetAttributes(&fa, f));
  }
  int per_sm = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pt::tick_kernel<true, 8, false>, pt::NTHREADS,
                                                         pt::SMEM_MAX));
  if (per_sm < 1) return fail(PT_EUNSUPPORTED, "tick kernel does not fit on one SM");
  p->G = c->grid > 0 ? c->grid : sms;
  if (p->G > sms * per_sm) return fail(PT_EINVAL, "grid exceeds co-resident CTA capacity");
  {
    // micro-batch tensor-core path: every width a multiple of 256, M = 16, 32 or 64
    bool ok = p->M == 16 || p->M == 32 || p->M == 64;  // SGD or Adam, MSE or softmax-CE
    int units = 0;
    for (int i = 0; i <= p->L && ok; ++i) ok = (p->dims[i] % 256) == 0;
    for (int i = 0; i < p->L && ok; ++i) units = std::max(units, std::max(p->dims[i + 1], p->dims[i]) / 128 * pt::T_Q);
    if (const char* e = getenv("PT_TILE")) ok = ok && atoi(e) != 0;
    if (ok) {
      p->tile = true;
      p->G = std::min(c->grid > 0 ? c->grid : sms, units);
    }
  }
  {
    // batch-1 panel path (pt_panel.cuh): SGD, any widths; stages in turn on every CTA.
    // PT_PANEL=0 keeps the row-owned tick kernel.
    bool ok = !p->tile && p->M == 1;  // SGD or Adam
    if (const char* e = getenv("PT_PANEL")) ok = ok && atoi(e) != 0;
    if (ok) {
      p->panel = true;
      p->G = c->grid > 0 ? c->grid : std::min(sms, 128);  // 2048-wide layers: one 16-row block per CTA
    }
  }

  // local layers
  const int s_lo = p->local_first, s_hi = p->local_first + p->local_count;
  p->layer_base = p->sfl[s_lo];
  const int l_hi = p->sfl[s_hi];
  for (int l = p->layer_base; l < l_hi; ++l) {
    LayerHost Lh;
    Lh.n_in = p->dims[l];
    Lh.n_out = p->dims[l + 1];
    Lh.ld_in = pad_dim(Lh.n_in);
    Lh.ld_out = pad_dim(Lh.n_out);
    Lh.act = p->act[l];
    Lh.R = (Lh.n_out + pt::PN_TS - 1) / pt::PN_TS;
    Lh.C = (Lh.n_in + pt::PN_TS - 1) / pt::PN_TS;
    if (p->panel) {
      const size_t tiled = size_t(Lh.R) * Lh.C * pt::PN_TILE * 4;
      PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&Lh.Wt[0]), tiled));
      if (p->learn) PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&Lh.Wt[1]), tiled));
    } else {
      PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&Lh.W), size_t(Lh.n_out) * Lh.ld_in * 4));
    }
    PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&Lh.b), size_t(Lh.n_out) * 4));
    if (p->opt == PT_OPT_ADAM && p->learn) {
      // moments: row-major [n_out][ld_in] (tick kernel), the panel path's tiles, or the tile
      // path's blocked [n_out/128][n_in/64][128][64] (within the same allocation size)
      const size_t nm = p->panel ? size_t(Lh.R) * Lh.C * pt::PN_TILE : size_t(Lh.n_out) * Lh.ld_in;
      PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&Lh.mW), nm * 4));
      PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&Lh.vW), nm * 4));
      PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&Lh.mb), size_t(Lh.n_out) * 4));
      PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&Lh.vb), size_t(Lh.n_out) * 4));
    }
    p->layers.push_back(Lh);
  }
  // Local stages are independent within a tick (each reads only tick t-1 data), so with
  // several of them on this GPU they run concurrently on disjoint CTA ranges, sized by their
  // weight bytes, and exchange through L2 exactly as separate GPUs would through NVLink
  p->stage_cta0.assign(p->local_count, 0);
  p->stage_ncta.assign(p->local_count, p->G);
  p->conc = p->local_count > 1 && !p->tile && !p->panel && p->G >= 2 * p->local_count;
  // uniform widths only: with uneven layers (C5) a byte-proportional split leaves the stage
  // with the most lock-step steps per byte behind, measured slower than running in turn
  for (const LayerHost& Lh : p->layers)
    p->conc = p->conc && Lh.n_in == p->layers[0].n_in && Lh.n_out == p->layers[0].n_out;
  if (const char* e = getenv("PT_CONC")) p->conc = p->conc && atoi(e) != 0;
  if (p->conc) {
    std::vector<double> w(p->local_count, 0.0);
    double tot = 0.0;
    for (int s = 0; s < p->local_count; ++s) {
      for (int l = p->sfl[p->local_first + s]; l < p->sfl[p->local_first + s + 1]; ++l)
        w[s] += double(p->dims[l]) * double(p->dims[l + 1]);
      tot += w[s];
    }
    std::vector<double> frac(p->local_count);
    int used = 0;
    for (int s = 0; s < p->local_count; ++s) {
      const double x = p->G * w[s] / tot;
      p->stage_ncta[s] = std::max(1, int(x));
      frac[s] = x - int(x);
      used += p->stage_ncta[s];
    }
    while (used < p->G) {  // largest remainders first
      int best = 0;
      for (int s = 1; s < p->local_count; ++s)
        if (frac[s] > frac[best]) best = s;
      ++p->stage_ncta[best];
      frac[best] = -1.0;
      ++used;
    }
    while (used > p->G) {  // (minimum-1 rounding overshoot) take from the largest
      int big = 0;
      for (int s = 1; s < p->local_count; ++s)
        if (p->stage_ncta[s] > p->stage_ncta[big]) big = s;
      --p->stage_ncta[big];
      --used;
    }
    for (int s = 1; s < p->local_count; ++s) p->stage_cta0[s] = p->stage_cta0[s - 1] + p->stage_ncta[s - 1];
    if (plan_smem(p) != PT_OK) {  // rows per CTA too many for shared memory: run in turn
      p->conc = false;
      p->stage_cta0.assign(p->local_count, 0);
      p->stage_ncta.assign(p->local_count, p->G);
    }
  }
  if (!p->panel) {
    PT_TRY(plan_smem(p));
    for (LayerHost& Lh : p->layers) Lh.rows_per_chunk = p->slot_floats / Lh.ld_in;
  }
  // local stages
  for (int s0 = s_lo; s0 < s_hi; ++s0) {
    StageHost S;
    S.h = s0 + 1;
    S.first_global = p->sfl[s0];
    S.k = p->sfl[s0 + 1] - p->sfl[s0];
    S.first_local = S.first_global - p->layer_base;
    S.ld0 = p->stage_ld0(s0);
    S.ldk = p->stage_ldk(s0);
    S.cta0 = p->stage_cta0[s0 - s_lo];
    S.ncta = p->stage_ncta[s0 - s_lo];
    // cache slot: a_0 .. a_k, each [M][ld]
    size_t off = 0;
    for (int i = 0; i < S.k; ++i) {
      LayerHost& Lh = p->layers[S.first_local + i];
      Lh.cache_in = int(off);
      off += size_t(p->M) * Lh.ld_in;
      Lh.cache_out = int(off);
    }
    off += size_t(p->M) * p->layers[S.first_local + S.k - 1].ld_out;
    S.cache_words = align_up(off, 64);
    // cache slots: tick mod 3 (tick kernel) or mod 4 (panel kernel: a slot is read as the
    // deferred update's a_hat up to two ticks after it was written)
    PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&S.cache), (p->panel ? 4 : 3) * S.cache_words * sizeof(u64)));
    const CommLayout cl = p->layout_of(s0);
    PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&S.comm), cl.total));
    // g_in partials: needed by every layer except stage 1's first
    if (p->learn && !p->tile && !p->panel) {
      for (int i = 0; i < S.k; ++i) {
        if (S.h == 1 && i == 0) continue;
        LayerHost& Lh = p->layers[S.first_local + i];
        for (int j = 0; j < 2; ++j)
          PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&Lh.part[j]), size_t(p->G) * p->M * Lh.ld_in * sizeof(u64)));
      }
    }
    p->stages.push_back(S);
  }
  // wire local neighbours
  for (size_t s = 0; s < p->stages.size(); ++s) {
    StageHost& S = p->stages[s];
    if (s > 0) {
      S.up = p->stages[s - 1].comm;
      S.G_up = p->stages[s - 1].ncta;
    }
    if (s + 1 < p->stages.size()) {
      S.down = p->stages[s + 1].comm;
      S.G_down = p->stages[s + 1].ncta;
    }
  }
  PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&p->d_layers), p->layers.size() * sizeof(pt::LayerDev)));
  PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&p->d_stages), p->stages.size() * sizeof(pt::StageDev)));
  PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&p->d_tick_end), sizeof(u64)));
  PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&p->d_status), sizeof(int)));
  PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&p->d_first_bad), sizeof(long long)));
  PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&p->d_bad_target), sizeof(long long)));
  const long long big = std::numeric_limits<long long>::max();
  CUDA_TRY(cudaMemcpy(p->d_first_bad, &big, sizeof(big), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(p->d_bad_target, &big, sizeof(big), cudaMemcpyHostToDevice));
  p->yh = std::max(1, p->D);
  if (p->has_last()) PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&p->yhist), size_t(p->yh) * p->M * p->Fy() * 4));
  CUDA_TRY(cudaStreamCreateWithFlags(&p->own_stream, cudaStreamNonBlocking));
  p->stream = p->own_stream;
  CUDA_TRY(cudaEventCreate(&p->ev0));
  CUDA_TRY(cudaEventCreate(&p->ev1));
  if (p->tile) PT_TRY(setup_tile(p));
  if (p->panel) PT_TRY(setup_panel(p));
  PT_TRY(upload_desc(p));
  CUDA_TRY(cudaDeviceSynchronize());
  return PT_OK;
}

LayerHost* local_layer(pt_pipeline* p, int layer, std::string* why) {
  const int li = layer - p->layer_base;
  if (layer < 0 || layer >= p->L) {
    *why = "layer index " + std::to_string(layer) + " out of range";
    return nullptr;
  }
  if (li < 0 || li >= int(p->layers.size())) {
    *why = "layer " + std::to_string(layer) + " is not owned by this process";
    return nullptr;
  }
  return &p->layers[li];
}

int check_ready(pt_pipeline* p) {
  if (p->broken) return fail(PT_ESTATE, "pipeline unusable after an earlier device-side failure");
  for (const StageHost& S : p->stages) {
    if (p->tile) {
      if ((S.h > 1 && !S.tup) || (S.h < p->D && !S.tdown))
        return fail(PT_EINVAL, "stage " + std::to_string(S.h) + ": neighbour stage not imported (pt_ipc_import)");
      continue;
    }
    if (S.h > 1 && !S.up)
      return fail(PT_EINVAL, "stage " + std::to_string(S.h) + ": upstream stage not imported (pt_ipc_import)");
    if (S.h < p->D && !S.down)
      return fail(PT_EINVAL, "stage " + std::to_string(S.h) + ": downstream stage not imported (pt_ipc_import)");
  }
  return PT_OK;
}

int read_status(pt_pipeline* p) {
  int st = 0;
  long long bad = 0;
  CUDA_TRY(cudaMemcpy(&st, p->d_status, sizeof(int), cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(&bad, p->d_first_bad, sizeof(long long), cudaMemcpyDeviceToHost));
  if (st != pt::ST_OK) {
    p->broken = true;
    return fail(PT_ETIMEOUT, "a stage waited longer than timeout_ms for a neighbour; pipeline state is lost");
  }
  long long badt = std::numeric_limits<long long>::max();
  CUDA_TRY(cudaMemcpy(&badt, p->d_bad_target, sizeof(long long), cudaMemcpyDeviceToHost));
  const long long big = std::numeric_limits<long long>::max();
  if (badt != big) {
    CUDA_TRY(cudaMemcpy(p->d_bad_target, &big, sizeof(big), cudaMemcpyHostToDevice));
    p->legacy_dirty = true;
    return fail(PT_EINVAL, "target out of class range for cross-entropy (sample " + std::to_string(badt) + ")");
  }
  if (bad != big) {
    CUDA_TRY(cudaMemcpy(p->d_first_bad, &big, sizeof(big), cudaMemcpyHostToDevice));
    p->legacy_dirty = true;
    return fail(PT_ENONFINITE, "non-finite loss at step " + std::to_string(bad));
  }
  return PT_OK;
}

// Wait for the handle's stream, copy pending host outputs out of the pinned staging area and
// report deferred device-side errors.
int finish_impl(pt_pipeline* p) {
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  if (p->pend.active) {
    pt_pipeline::Pending& q = p->pend;
    if (q.st_o) memcpy(q.outs, q.pin_o, q.st_o * 4);
    if (q.st_l) memcpy(q.losses, q.pin_l, q.st_l * 4);
    if (q.st_v) memcpy(q.valid, q.pin_v, size_t(q.n));
    q.active = false;
  }
  return read_status(p);
}

// Launch parameters of the panel kernel shared by pt_run and the resident pt_step.
void panel_common(pt_pipeline* p, pt::PParams& Q) {
  memset(&Q, 0, sizeof(Q));
  Q.stages = p->d_pstages;
  Q.layers = p->d_players;
  Q.n_stages = int(p->stages.size());
  Q.n_layers = int(p->layers.size());
  Q.D = p->D;
  Q.learn = p->learn;
  Q.act_delay = p->act_delay;
  Q.G = p->G;
  Q.F = p->F();
  Q.loss = p->loss;
  Q.lr = p->lr;
  Q.b1 = 0.9f;  // Adam (oracle/netcore.py Adam), as the tick kernel
  Q.b2 = 0.999f;
  Q.b1d = 0.9;
  Q.b2d = 0.999;
  Q.omb1 = float(1.0 - 0.9);
  Q.omb2 = float(1.0 - 0.999);
  Q.eps = 1e-8f;
  Q.adam = p->opt == PT_OPT_ADAM && p->learn ? 1 : 0;
  Q.ldx = p->stage_ld0(0);
  Q.yhist = p->yhist;
  Q.yh = p->yh;
  Q.tick_end = p->d_tick_end;
  Q.status = p->d_status;
  Q.bad_target = p->d_bad_target;
  Q.timeout_ns = p->timeout_ns;
  Q.nslot = p->pn_nslot;
  Q.va_off = p->pn_va;
  Q.vb_off = p->pn_vb;
  Q.sown_off = p->pn_sown;
  Q.sah_off = p->pn_sah;
  Q.red_off = p->pn_red;
  Q.bar_off = p->pn_bar;
  Q.desc_off = p->pn_desc;
  Q.bias_off = p->pn_bias;
  Q.pf_chunks = p->pn_pf;
  Q.psleep = getenv("PT_PSLEEP") ? atoi(getenv("PT_PSLEEP")) : 0;
  Q.dbg = getenv("PT_PN_DBG") ? atoi(getenv("PT_PN_DBG")) : 0;
  Q.policy = p->policy;
  Q.trace = p->d_trace;
  Q.trace_cap = p->trace_cap;
  Q.trace_cta = p->trace_cta;
  Q.jitter_mask = 3;
}

// ---------------------------------------------------------------- resident pt_step
// The per-sample drop-in (pipeline_step; Pipeline.forward)
// without a launch per sample: PAPER.md:600-605 removed the per-tick enqueue cost with CUDA
// Graphs; here one persistent panel-kernel launch serves consecutive pt_step calls (see
// PParams::resident in pt_panel.cuh). Any other entry point stops it first (resident_stop).
// A resident launch holds its SMs until the host posts a stop. Another handle's cooperative
// launch on the same device could then never become co-resident, so every launch first stops
// the resident launches of the other handles on its device (process-wide registry).
std::mutex g_res_mu;
std::vector<pt_pipeline*> g_resident;
int resident_stop(pt_pipeline* p);

void resident_register(pt_pipeline* p, bool on) {
  std::lock_guard<std::mutex> lk(g_res_mu);
  auto it = std::find(g_resident.begin(), g_resident.end(), p);
  if (on && it == g_resident.end()) g_resident.push_back(p);
  if (!on && it != g_resident.end()) g_resident.erase(it);
}

int stop_foreign_residents(pt_pipeline* self) {
  std::vector<pt_pipeline*> others;
  {
    std::lock_guard<std::mutex> lk(g_res_mu);
    for (pt_pipeline* q : g_resident) {
      if (q == self) continue;
      bool same = q->device == self->device;
      for (const pt_pipeline* m : q->parts) same = same || (m->device == self->device && m != self);
      if (same) others.push_back(q);
    }
  }
  for (pt_pipeline* q : others) {
    // the owner may be inside a step of its own: wait for the handle (single driver)
    const auto t_begin = std::chrono::steady_clock::now();
    int z = 0;
    while (!q->busy.compare_exchange_strong(z, 1)) {
      z = 0;
      if (std::chrono::steady_clock::now() - t_begin > std::chrono::nanoseconds(self->timeout_ns))
        return fail(PT_EBUSY, "another pipeline's resident pt_step launch holds the device");
      std::this_thread::yield();
    }
    int r;
    {
      DevGuard dg(q->device);
      r = resident_stop(q);
    }
    q->busy.store(0);
    if (r != PT_OK) return r;
  }
  return PT_OK;
}

// The handles that execute a driver's resident launch: the handle itself, or a multi-device
// handle's parts (one resident launch per device; the parts exchange through peer memory as
// in pt_run, and all of them poll the same mapped request word).
std::vector<pt_pipeline*> resident_members(pt_pipeline* p) {
  if (p->group()) return p->parts;
  return {p};
}

bool resident_eligible(const pt_pipeline* p) {
  if (!p->has_first() || !p->has_last() || p->M != 1) return false;
  if (p->group()) {
    for (const pt_pipeline* q : p->parts)
      if (!q->panel) return false;
  } else if (!p->panel) {
    return false;
  }
  const char* e = getenv("PT_RESIDENT");
  return !(e && atoi(e) == 0);
}

// The driver's mapped host block: completion record, request words, x / target / output rings.
int resident_alloc_host(pt_pipeline* p) {
  pt_pipeline::Resident& r = p->res;
  if (r.host) return PT_OK;
  r.ring = p->D + 2;
  r.ldx = p->stage_ld0(0);
  r.fy = p->Fy();
  const size_t nx = size_t(r.ring) * r.ldx, ny = size_t(r.ring) * r.fy, no = size_t(2) * p->F();
  r.bytes = align_up(sizeof(pt::PResDone), 64) + 64 + (nx + ny + no) * 4;
  // portable: every device of a multi-device handle maps it
  CUDA_TRY(cudaHostAlloc(&r.host, r.bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(r.host, 0, r.bytes);
  char* h = static_cast<char*>(r.host);
  r.done = reinterpret_cast<pt::PResDone*>(h);
  h += align_up(sizeof(pt::PResDone), 64);
  r.req = reinterpret_cast<long long*>(h);
  r.flag = reinterpret_cast<int*>(h + 8);
  h += 64;
  r.x = reinterpret_cast<float*>(h);
  r.y = r.x + nx;
  r.out = r.y + ny;
  return PT_OK;
}

// A member's device buffers and its device alias of the driver's host block.
int resident_alloc_dev(pt_pipeline* q, const pt_pipeline* drv) {
  pt_pipeline::Resident& r = q->res;
  void* dh = nullptr;
  CUDA_TRY(cudaHostGetDevicePointer(&dh, drv->res.host, 0));
  r.dev_off = static_cast<char*>(dh) - static_cast<char*>(drv->res.host);
  if (r.relay) return PT_OK;
  PT_TRY(dev_alloc(q, reinterpret_cast<void**>(&r.xin), size_t(2) * drv->res.ldx * sizeof(u64)));
  r.ldy = (q->F() + pt::PN_TS - 1) / pt::PN_TS * pt::PN_TS;  // the loss gather's row length
  PT_TRY(dev_alloc(q, reinterpret_cast<void**>(&r.ytag), size_t(drv->res.ring) * r.ldy * sizeof(u64)));
  PT_TRY(dev_alloc(q, reinterpret_cast<void**>(&r.relay), 64));
  PT_TRY(dev_alloc(q, reinterpret_cast<void**>(&r.lpart), size_t(2) * q->G * sizeof(float)));
  return PT_OK;
}

template <class T>
T* to_dev(const pt_pipeline* q, T* hptr) {
  return reinterpret_cast<T*>(reinterpret_cast<char*>(hptr) + q->res.dev_off);
}

int resident_launch(pt_pipeline* q, const pt_pipeline* drv) {
  const pt_pipeline::Resident& h = drv->res;
  pt_pipeline::Resident& r = q->res;
  CUDA_TRY(cudaMemsetAsync(r.relay, 0, 64, q->stream));
  pt::PParams Q;
  panel_common(q, Q);
  Q.t0 = q->t_next;
  Q.n = std::numeric_limits<int>::max();
  Q.loss_part = r.lpart;
  Q.resident = 1;
  Q.res_last = q->has_last() ? 1 : 0;
  Q.hreq = to_dev(q, h.req);
  Q.hflag = to_dev(q, h.flag);
  Q.relay = r.relay;
  Q.rx = to_dev(q, h.x);
  Q.ry = to_dev(q, h.y);
  Q.rring = h.ring;
  Q.xin = r.xin;
  Q.ytag = r.ytag;
  Q.ldy = r.ldy;
  Q.rout = to_dev(q, h.out);
  Q.rdone = to_dev(q, h.done);
  if (q->d_trace) CUDA_TRY(cudaMemsetAsync(q->d_trace, 0, size_t(q->trace_cap) * sizeof(u64), q->stream));
  void* qargs[] = {&Q};
  CUDA_TRY(cudaLaunchCooperativeKernel(q->opt == PT_OPT_ADAM ? (const void*)pt::panel_kernel<1> : (const void*)pt::panel_kernel<0>,
                                       dim3(q->G), dim3(pt::NTHREADS), qargs, size_t(q->pn_smem), q->stream));
  r.on = true;
  r.t_start = q->t_next;
  return PT_OK;
}

int resident_start(pt_pipeline* p) {
  const std::vector<pt_pipeline*> mem = resident_members(p);
  PT_TRY(resident_alloc_host(p));
  for (pt_pipeline* q : mem) {
    DevGuard dg(q->device);
    PT_TRY(check_ready(q));
    PT_TRY(stop_foreign_residents(q));
    PT_TRY(resident_alloc_dev(q, p));
    if (q->legacy_dirty) {
      CUDA_TRY(cudaStreamSynchronize(0));
      q->legacy_dirty = false;
    }
  }
  pt_pipeline::Resident& r = p->res;
  *reinterpret_cast<volatile long long*>(r.req) = p->t_next;  // nothing requested yet
  *reinterpret_cast<volatile long long*>(&r.done->tick) = -1;
  for (pt_pipeline* q : mem) {
    DevGuard dg(q->device);
    PT_TRY(resident_launch(q, p));
  }
  r.on = true;
  r.t_start = p->t_next;
  resident_register(p, true);
  return PT_OK;
}

// Post a stop, wait for every member's launch to drain, and queue the last D-1 posted targets
// for the next pt_run (target queue).
int resident_stop(pt_pipeline* p) {
  pt_pipeline::Resident& r = p->res;
  if (!r.on) return PT_OK;
  resident_register(p, false);
  std::atomic_thread_fence(std::memory_order_seq_cst);
  *reinterpret_cast<volatile long long*>(r.req) = pt::PN_STOP;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  r.on = false;
  const auto t_begin = std::chrono::steady_clock::now();
  int first_err = PT_OK;
  std::string msg;
  for (pt_pipeline* q : resident_members(p)) {
    DevGuard dg(q->device);
    q->res.on = false;
    q->t_next = p->t_next;
    // the launch ends at its next tick boundary; never block without a bound on it
    cudaError_t e;
    while ((e = cudaStreamQuery(q->stream)) == cudaErrorNotReady) {
      if (std::chrono::steady_clock::now() - t_begin > std::chrono::nanoseconds(2 * q->timeout_ns)) {
        long long relay = 0;
        cudaMemcpy(&relay, q->res.relay, sizeof(relay), cudaMemcpyDeviceToHost);
        q->broken = p->broken = true;
        return fail(PT_ETIMEOUT, "resident launch did not stop (relay " + std::to_string(relay) + ", tick " +
                                     std::to_string(p->t_next) + ")");
      }
      std::this_thread::yield();
    }
    if (e != cudaSuccess) return fail(PT_ECUDA, std::string("resident launch failed: ") + cudaGetErrorString(e));
    if (q->has_last()) {
      const int Fy = q->Fy();
      for (long long s = std::max(r.t_start, p->t_next - (p->D - 1)); s < p->t_next; ++s)
        CUDA_TRY(cudaMemcpyAsync(q->yhist + size_t(s % q->yh) * Fy, r.y + size_t(s % r.ring) * Fy, size_t(Fy) * 4,
                                 cudaMemcpyHostToDevice, q->stream));
      CUDA_TRY(cudaStreamSynchronize(q->stream));
    }
    const int rs = read_status(q);
    if (rs != PT_OK && first_err == PT_OK) {
      first_err = rs;
      msg = g_err;
    }
  }
  if (first_err != PT_OK) g_err = msg;
  return first_err;
}

// One tick through the resident launch(es): write x_t and gamma_t into the mapped rings, post
// the request, wait for the completion record (written by the member that owns stage D).
int resident_step(pt_pipeline* p, const float* x, const float* y, float* out, float* loss, int32_t* valid) {
  if (!x) return fail(PT_EINVAL, "x is required on the process that owns stage 1");
  if (p->learn && !y) return fail(PT_EINVAL, "targets are required for online learning (stage D)");
  if (!p->res.on) PT_TRY(resident_start(p));
  pt_pipeline::Resident& r = p->res;
  const std::vector<pt_pipeline*> mem = resident_members(p);
  const long long t = p->t_next;
  const int n0 = p->dims[0], Fy = p->Fy(), F = p->F();
  memcpy(r.x + size_t(t % r.ring) * r.ldx, x, size_t(n0) * 4);
  if (y) memcpy(r.y + size_t(t % r.ring) * Fy, y, size_t(Fy) * 4);
  else memset(r.y + size_t(t % r.ring) * Fy, 0, size_t(Fy) * 4);
  *reinterpret_cast<volatile int*>(r.flag) = y ? 1 : 0;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  *reinterpret_cast<volatile long long*>(r.req) = t + 1;
  volatile long long* dt = &r.done->tick;
  const auto t_begin = std::chrono::steady_clock::now();
  unsigned spins = 0;
  while (*dt != t + 1) {
    if ((++spins & 0xFFFu) == 0) {
      for (pt_pipeline* q : mem) {
        DevGuard dg(q->device);
        const cudaError_t e = cudaStreamQuery(q->stream);
        if (e != cudaErrorNotReady) {  // a launch ended without completing the step
          resident_register(p, false);
          r.on = false;
          for (pt_pipeline* o : mem) o->res.on = false;
          if (e != cudaSuccess) return fail(PT_ECUDA, std::string("resident launch failed: ") + cudaGetErrorString(e));
          PT_TRY(read_status(q));
          return fail(PT_ESTATE, "resident launch ended before completing step " + std::to_string(t));
        }
      }
      if (std::chrono::steady_clock::now() - t_begin > std::chrono::nanoseconds(4 * p->timeout_ns)) {
        p->broken = true;
        return fail(PT_ETIMEOUT, "resident step " + std::to_string(t) + " did not complete");
      }
    }
  }
  std::atomic_thread_fence(std::memory_order_seq_cst);
  p->t_next = t + 1;
  for (pt_pipeline* q : mem) q->t_next = t + 1;
  const pt::PResDone d = *const_cast<const pt::PResDone*>(r.done);
  static const bool dbg = getenv("PT_RESIDENT_DEBUG") != nullptr;  // diagnostics: per-step timing
  if (dbg) {
    static double dev_sum = 0, host_sum = 0;
    static long cnt = 0;
    dev_sum += double(d.done_ns - d.req_ns) * 1e-3;
    host_sum += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_begin).count();
    if (++cnt % 100 == 0)
      fprintf(stderr, "resident: %ld steps, device request->record %.1f us, host post->done %.1f us\n", cnt,
              dev_sum / cnt, host_sum / cnt);
  }
  if (out) memcpy(out, r.out + size_t(t & 1) * F, size_t(F) * 4);
  if (loss) *loss = d.loss;
  if (valid) *valid = d.valid;
  if (d.status != pt::ST_OK) {
    PT_TRY(resident_stop(p));
    return fail(PT_ETIMEOUT, "a stage waited longer than timeout_ms; pipeline state is lost");
  }
  if (d.bad_target != std::numeric_limits<long long>::max()) {
    PT_TRY(resident_stop(p));  // read_status reports and clears the device flag
    return PT_EINVAL;
  }
  if (d.bad_loss >= 0) return fail(PT_ENONFINITE, "non-finite loss at step " + std::to_string(d.bad_loss));
  return PT_OK;
}

int run_impl(pt_pipeline* p, const float* xs, const float* ys, int64_t n, float* outs, float* losses,
             uint8_t* valid, int where, bool wait = true) {
  PT_TRY(check_ready(p));
  PT_TRY(stop_foreign_residents(p));
  if (p->pend.active) return fail(PT_EBUSY, "contract violation: previous run not finished (pt_sync)");
  if (n <= 0) return PT_OK;
  if (p->legacy_dirty) {
    CUDA_TRY(cudaStreamSynchronize(0));
    p->legacy_dirty = false;
  }
  if (n > (1 << 30)) return fail(PT_EINVAL, "too many ticks in one call");
  if (where != PT_HOST && where != PT_DEVICE) return fail(PT_EINVAL, "where must be PT_HOST or PT_DEVICE");
  const cudaMemcpyKind h2d = where == PT_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  const cudaMemcpyKind d2h = where == PT_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  const int M = p->M, F = p->F(), Fy = p->Fy();
  const bool first = p->has_first(), last = p->has_last();
  if (first && !xs) return fail(PT_EINVAL, "xs is required on the process that owns stage 1");
  if (last && p->learn && !ys) return fail(PT_EINVAL, "targets are required for online learning (stage D)");
  const int n0 = p->dims[0], ld0 = p->stage_ld0(0);

  // small host-buffer calls (pt_step and short pt_run) go through a pinned staging area:
  // [xs n*M*n0 | ys n*M*Fy | outs n*M*F | losses n | valid n (bytes, as floats)]
  const size_t st_x = first ? size_t(n) * M * n0 : 0, st_y = (last && ys) ? size_t(n) * M * Fy : 0;
  const size_t st_o = (last && outs) ? size_t(n) * M * F : 0, st_l = (last && losses) ? size_t(n) : 0;
  const size_t st_v = (last && valid) ? (size_t(n) + 3) / 4 : 0;
  const size_t st_total = st_x + st_y + st_o + st_l + st_v;
  const bool staged = where == PT_HOST && st_total <= (size_t(1) << 16);
  float* pin_x = nullptr;
  float* pin_y = nullptr;
  float* pin_o = nullptr;
  float* pin_l = nullptr;
  uint8_t* pin_v = nullptr;
  if (staged) {
    if (p->pin_floats < st_total) {
      CUDA_TRY(cudaStreamSynchronize(p->stream));
      if (p->pin) CUDA_TRY(cudaFreeHost(p->pin));
      p->pin = nullptr;
      p->pin_floats = 0;
      CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&p->pin), std::max<size_t>(st_total, 4096) * 4,
                             cudaHostAllocDefault));
      p->pin_floats = std::max<size_t>(st_total, 4096);
    }
    pin_x = p->pin;
    pin_y = pin_x + st_x;
    pin_o = pin_y + st_y;
    pin_l = pin_o + st_o;
    pin_v = reinterpret_cast<uint8_t*>(pin_l + st_l);
    if (st_x) memcpy(pin_x, xs, st_x * 4);
    if (st_y) memcpy(pin_y, ys, st_y * 4);
    if (st_x) xs = pin_x;
    if (st_y) ys = pin_y;
  }
  if (first) {
    PT_TRY(ensure(p, &p->xs_pad, &p->xs_cap, size_t(n), size_t(M) * ld0));
    CUDA_TRY(cudaMemcpy2DAsync(p->xs_pad, size_t(ld0) * 4, xs, size_t(n0) * 4, size_t(n0) * 4, size_t(n) * M,
                               h2d, p->stream));
  }
  const float* ys_dev = nullptr;
  float* outs_dev = nullptr;
  float* losses_dev = nullptr;
  uint8_t* valid_dev = nullptr;
  if (last) {
    if (ys) {
      if (where == PT_HOST) {
        PT_TRY(ensure(p, &p->ys_stage, &p->ys_cap, size_t(n), size_t(M) * Fy));
        CUDA_TRY(cudaMemcpyAsync(p->ys_stage, ys, size_t(n) * M * Fy * 4, h2d, p->stream));
        ys_dev = p->ys_stage;
      } else {
        ys_dev = ys;
      }
    }
    if (where == PT_DEVICE && outs) {
      outs_dev = outs;
    } else {
      PT_TRY(ensure(p, &p->outs_stage, &p->outs_cap, size_t(n), size_t(M) * F));
      outs_dev = p->outs_stage;
    }
    PT_TRY(ensure(p, &p->loss_part, &p->lp_cap, size_t(n), size_t(p->G)));
    if (where == PT_DEVICE) {
      losses_dev = losses;
      valid_dev = valid;
    }
    if (!losses_dev) {
      PT_TRY(ensure(p, &p->losses_stage, &p->ls_cap, size_t(n), 1));
      losses_dev = p->losses_stage;
    }
    if (!valid_dev) {
      PT_TRY(ensure(p, &p->valid_stage, &p->vs_cap, size_t(n), 1));
      valid_dev = p->valid_stage;
    }
  }

  pt::Params P;
  memset(&P, 0, sizeof(P));
  P.stages = p->d_stages;
  P.layers = p->d_layers;
  P.n_stages = int(p->stages.size());
  P.M = M;
  P.D = p->D;
  P.learn = p->learn;
  P.act_delay = p->act_delay;
  P.G = p->G;
  P.F = F;
  int nB = 0;
  for (const StageHost& S : p->stages) nB += S.k;
  P.nB = p->learn ? nB : 0;
  P.lr = p->lr;
  P.loss = p->loss;
  P.opt = p->opt;
  P.Fy = Fy;
  P.b1 = 0.9f;  // Adam (oracle/netcore.py Adam)
  P.b2 = 0.999f;
  P.b1d = 0.9;
  P.b2d = 0.999;
  P.omb1 = float(1.0 - 0.9);
  P.omb2 = float(1.0 - 0.999);
  P.eps = 1e-8f;
  P.xs = first ? p->xs_pad : nullptr;
  P.ys = ys_dev;
  P.yhist = p->yhist;
  P.yh = p->yh;
  P.outs = outs_dev;
  P.loss_part = last ? p->loss_part : nullptr;
  P.t0 = p->t_next;
  P.n = int(n);
  P.tick_end = p->d_tick_end;
  P.status = p->d_status;
  P.bad_target = p->d_bad_target;
  P.timeout_ns = p->timeout_ns;
  P.nslot = p->nslot;
  P.slot_floats = p->slot_floats;
  P.act_off = p->act_off;
  P.spart_off = p->spart_off;
  P.spart_floats = p->spart_floats;
  P.delta_off = p->delta_off;
  P.red_off = p->red_off;
  P.scal_off = p->scal_off;
  P.bar_off = p->bar_off;
  P.flags_off = p->flags_off;
  P.desc_off = p->desc_off;
  P.bias_off = p->bias_off;
  P.n_layers = int(p->layers.size());
  P.pf_chunks = p->pf_chunks;
  P.split_bytes = p->split_bytes;
  P.maxfly = p->maxfly;
  P.wb_mode = p->wb_mode;
  P.dbg = p->dbg;
  P.policy = p->policy;
  P.trace = p->d_trace;
  P.trace_cap = p->trace_cap;
  P.trace_cta = p->trace_cta;
  if (const char* e = getenv("PT_JITTER")) P.jitter = atoi(e);
  P.jitter_mask = 3;
  if (const char* e = getenv("PT_JITTER_MASK")) P.jitter_mask = atoi(e);
  if (p->d_trace) CUDA_TRY(cudaMemsetAsync(p->d_trace, 0, size_t(p->trace_cap) * sizeof(u64), p->stream));

  if (p->panel) {
    pt::PParams Q;
    panel_common(p, Q);
    Q.xs = first ? p->xs_pad : nullptr;
    Q.ldx = ld0;
    Q.ys = ys_dev;
    Q.outs = outs_dev;
    Q.loss_part = last ? p->loss_part : nullptr;
    Q.t0 = p->t_next;
    Q.n = int(n);
    Q.jitter = P.jitter;
    Q.jitter_mask = P.jitter_mask;
    void* qargs[] = {&Q};
    CUDA_TRY(cudaEventRecord(p->ev0, p->stream));
    CUDA_TRY(cudaLaunchCooperativeKernel(p->opt == PT_OPT_ADAM ? (const void*)pt::panel_kernel<1> : (const void*)pt::panel_kernel<0>,
                                       dim3(p->G), dim3(pt::NTHREADS), qargs,
                                         size_t(p->pn_smem), p->stream));
    CUDA_TRY(cudaEventRecord(p->ev1, p->stream));
  } else if (p->tile) {
    pt::TParams T;
    memset(&T, 0, sizeof(T));
    T.stages = p->d_tstages;
    T.layers = p->d_tlayers;
    T.n_stages = int(p->stages.size());
    T.M = M;
    T.D = p->D;
    T.learn = p->learn;
    T.act_delay = p->act_delay;
    T.F = F;
    T.G = p->G;
    T.lr = p->lr;
    T.opt = p->opt;
    T.loss = p->loss;
    T.Fy = Fy;
    T.b1 = P.b1;
    T.b2 = P.b2;
    T.b1d = P.b1d;
    T.b2d = P.b2d;
    T.omb1 = P.omb1;
    T.omb2 = P.omb2;
    T.eps = P.eps;
    T.ce = p->t_ce;
    T.bad_target = p->d_bad_target;
    T.xs = p->xs_pad;
    T.ldx = ld0;
    T.ys = ys_dev;
    T.yhist = p->yhist;
    T.yh = p->yh;
    T.outs = outs_dev;
    T.loss_part = p->loss_part;
    T.t0 = p->t_next;
    T.n = int(n);
    T.part = p->t_part;
    T.delta = p->t_delta;
    T.max_n = p->t_maxn;
    T.gbar = p->t_bars;
    T.wbar = p->t_bars + 16;
    T.status = p->d_status;
    T.timeout_ns = p->timeout_ns;
    T.trace = p->d_trace;
    T.trace_cap = p->trace_cap;
    T.trace_cta = p->trace_cta;
    if (const char* e = getenv("PT_JITTER")) T.jitter = atoi(e);
    T.jitter_mask = 3;
    if (const char* e = getenv("PT_JITTER_MASK")) T.jitter_mask = atoi(e);
    if (p->d_trace) CUDA_TRY(cudaMemsetAsync(p->d_trace, 0, size_t(p->trace_cap) * sizeof(u64), p->stream));
    CUDA_TRY(cudaMemsetAsync(p->t_bars, 0, 32 * sizeof(u64), p->stream));
    void* targs[] = {&T};
    CUDA_TRY(cudaEventRecord(p->ev0, p->stream));
    CUDA_TRY(cudaLaunchCooperativeKernel(tile_fn(p), dim3(p->G), dim3(pt::T_THREADS), targs,
                                         size_t(p->t_smem), p->stream));
    CUDA_TRY(cudaEventRecord(p->ev1, p->stream));
  } else {
    void* args[] = {&P};
    CUDA_TRY(cudaEventRecord(p->ev0, p->stream));
    const void* fn;
    if (p->conc)
      fn = p->fast ? (p->qw == 8 ? (const void*)pt::tick_kernel<true, 8, true> : (const void*)pt::tick_kernel<true, 4, true>)
                   : (p->qw == 8 ? (const void*)pt::tick_kernel<false, 8, true> : (const void*)pt::tick_kernel<false, 4, true>);
    else
      fn = p->fast ? (p->qw == 8 ? (const void*)pt::tick_kernel<true, 8, false> : (const void*)pt::tick_kernel<true, 4, false>)
                   : (p->qw == 8 ? (const void*)pt::tick_kernel<false, 8, false> : (const void*)pt::tick_kernel<false, 4, false>);
    CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(p->G), dim3(pt::NTHREADS), args, size_t(p->smem_bytes), p->stream));
    CUDA_TRY(cudaEventRecord(p->ev1, p->stream));
  }
  p->timed = true;

  if (last) {
    const int threads = 256, warps_per_block = threads / 32;
    const int blocks = int((n + warps_per_block - 1) / warps_per_block);
    pt::epilogue_kernel<<<blocks, threads, 0, p->stream>>>(p->loss_part, p->G, int(n), p->t_next, p->D,
                                                           p->loss == PT_LOSS_SOFTMAX_CE ? 1.f / float(M) : 1.f / float(M * F),
                                                           ys_dev != nullptr ? 1 : 0,
                                                           losses_dev, valid_dev, p->d_first_bad);
    CUDA_TRY(cudaGetLastError());
    // queue the last D-1 targets for the next call (target queue)
    if (ys_dev) {
      for (long long s = std::max<long long>(p->t_next, p->t_next + n - (p->D - 1)); s < p->t_next + n; ++s)
        CUDA_TRY(cudaMemcpyAsync(p->yhist + size_t(s % p->yh) * M * Fy, ys_dev + size_t(s - p->t_next) * M * Fy,
                                 size_t(M) * Fy * 4, cudaMemcpyDeviceToDevice, p->stream));
    }
    if (outs && outs != outs_dev)
      CUDA_TRY(cudaMemcpyAsync(staged ? pin_o : outs, outs_dev, size_t(n) * M * F * 4, d2h, p->stream));
    if (losses && losses != losses_dev)
      CUDA_TRY(cudaMemcpyAsync(staged ? pin_l : losses, losses_dev, size_t(n) * 4, d2h, p->stream));
    if (valid && valid != valid_dev)
      CUDA_TRY(cudaMemcpyAsync(staged ? pin_v : valid, valid_dev, size_t(n), d2h, p->stream));
  }
  p->t_next += n;
  if (where == PT_HOST) {
    if (staged && last) {
      p->pend.n = n;
      p->pend.outs = outs;
      p->pend.losses = losses;
      p->pend.valid = valid;
      p->pend.pin_o = pin_o;
      p->pend.pin_l = pin_l;
      p->pend.pin_v = pin_v;
      p->pend.st_o = st_o;
      p->pend.st_l = st_l;
      p->pend.st_v = st_v;
      p->pend.active = true;
    }
    if (!wait) return PT_OK;
    return finish_impl(p);
  }
  return PT_OK;
}


// ---------------------------------------------------------------- multi-device handles
// pt_config.device_of_stage spreads the local stages over several devices of this process
// (SURVEY.md §8(b)). Each maximal run of stages on one device becomes a part:
// a complete single-device handle with local_stage_first/count = that run. Neighbouring parts
// import each other's comm blocks by device pointer (peer access enabled), so the kernels
// store activations, gradients and credits straight into the neighbour's memory with
// system-scope stores, exactly as across processes with CUDA IPC.
//
// PT_VIRTUAL_DEVICES=1 (testing on a one-GPU box): device ordinals are taken modulo the device
// count, and parts that land on one physical device split its SMs (grid = SMs / parts there),
// so their cooperative launches are co-resident.

pt_pipeline* part_of_layer(pt_pipeline* p, int layer) {
  for (pt_pipeline* q : p->parts)
    if (layer >= q->layer_base && layer < q->layer_base + int(q->layers.size())) return q;
  return nullptr;
}

int connect_parts(pt_pipeline* a, pt_pipeline* b) {
  // a owns stages [.., s], b owns [s+1, ..] (1-based s = a->local_first + a->local_count)
  const int s = a->local_first + a->local_count;
  char blob[256];
  size_t len = 0;
  if (a->device != b->device) {
    int ab = 0, ba = 0;
    CUDA_TRY(cudaDeviceCanAccessPeer(&ab, a->device, b->device));
    CUDA_TRY(cudaDeviceCanAccessPeer(&ba, b->device, a->device));
    if (!ab || !ba)
      return fail(PT_EUNSUPPORTED, "devices " + std::to_string(a->device) + " and " + std::to_string(b->device) +
                                       " have no peer access (one process per GPU: dist.build_distributed)");
    for (int k = 0; k < 2; ++k) {
      DevGuard dg(k ? b->device : a->device);
      cudaError_t e = cudaDeviceEnablePeerAccess(k ? a->device : b->device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
      } else if (e != cudaSuccess) {
        return fail(PT_ECUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
      }
    }
  }
  PT_TRY(pt_ipc_export(a, s, blob, sizeof(blob), &len));
  PT_TRY(pt_ipc_import(b, blob, len));
  PT_TRY(pt_ipc_export(b, s + 1, blob, sizeof(blob), &len));
  PT_TRY(pt_ipc_import(a, blob, len));
  return PT_OK;
}

int create_group(const pt_config* c, pt_pipeline* p) {
  std::string why;
  if (validate(c, &why) != PT_OK) return fail(PT_EINVAL, why);
  const int D = c->n_stages;
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  const char* ve = getenv("PT_VIRTUAL_DEVICES");
  const bool virt = ve && atoi(ve) != 0;
  std::vector<int> dev(D);
  for (int h = 0; h < D; ++h) {
    const int d = c->device_of_stage[h];
    if (d < 0 || (!virt && d >= ndev))
      return fail(PT_EINVAL, "device_of_stage[" + std::to_string(h) + "] = " + std::to_string(d) +
                                 " is not a device of this process (" + std::to_string(ndev) + " visible)");
    dev[h] = d;
  }
  for (int h = 1; h < D; ++h)
    for (int g = 0; g + 1 < h; ++g)
      if (dev[g] == dev[h] && dev[h - 1] != dev[h])
        return fail(PT_EINVAL, "stages of one device must be contiguous (device " + std::to_string(dev[h]) +
                                   " holds stages " + std::to_string(g + 1) + " and " + std::to_string(h + 1) + ")");
  const int lo = c->local_stage_count ? c->local_stage_first : 0;
  const int hi = c->local_stage_count ? lo + c->local_stage_count : D;
  std::vector<std::pair<int, int>> runs;  // (first stage, count), 0-based
  for (int h = lo; h < hi; ++h) {
    if (runs.empty() || dev[h] != dev[runs.back().first]) runs.push_back({h, 0});
    ++runs.back().second;
  }
  std::vector<int> phys(runs.size());
  std::vector<int> share(std::max(ndev, 1), 0);
  for (size_t i = 0; i < runs.size(); ++i) {
    phys[i] = dev[runs[i].first] % std::max(ndev, 1);
    ++share[phys[i]];
  }
  p->L = c->n_layers;
  p->D = D;
  p->M = c->batch;
  p->loss = c->loss;
  p->learn = c->learn ? 1 : 0;
  p->dims.assign(c->dims, c->dims + p->L + 1);
  p->sfl.assign(c->stage_first_layer, c->stage_first_layer + D + 1);
  p->local_first = lo;
  p->local_count = hi - lo;
  p->device = phys[0];
  p->timeout_ns = (unsigned long long)(c->timeout_ms > 0 ? c->timeout_ms : 30000) * 1000000ull;
  for (size_t i = 0; i < runs.size(); ++i) {
    pt_config sub = *c;
    sub.device_of_stage = nullptr;
    sub.local_stage_first = runs[i].first;
    sub.local_stage_count = runs[i].second;
    if (sub.grid == 0 && share[phys[i]] > 1) {
      int sms = 0;
      CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, phys[i]));
      sub.grid = sms / share[phys[i]];
    }
    DevGuard dg(phys[i]);
    pt_pipeline* q = nullptr;
    PT_TRY(pt_create(&sub, &q));
    p->parts.push_back(q);
  }
  for (size_t i = 0; i + 1 < p->parts.size(); ++i) PT_TRY(connect_parts(p->parts[i], p->parts[i + 1]));
  return PT_OK;
}

// Enqueue n ticks on every part (stage-1 part first; none waits), then, for host buffers,
// wait for all of them. Inputs go to the part that owns stage 1, targets and outputs to the
// part that owns stage D.
int group_run(pt_pipeline* p, const float* xs, const float* ys, int64_t n, float* outs, float* losses,
              uint8_t* valid, int where) {
  if (n <= 0) return PT_OK;
  if (p->has_first() && !xs) return fail(PT_EINVAL, "xs is required on the process that owns stage 1");
  if (p->has_last() && p->learn && !ys) return fail(PT_EINVAL, "targets are required for online learning (stage D)");
  for (pt_pipeline* q : p->parts) PT_TRY(check_ready(q));
  for (pt_pipeline* q : p->parts) {
    DevGuard dg(q->device);
    const bool f = q->has_first(), l = q->has_last();
    const int r = run_impl(q, f ? xs : nullptr, l ? ys : nullptr, n, l ? outs : nullptr, l ? losses : nullptr,
                           l ? valid : nullptr, where, false);
    if (r != PT_OK) {
      // the parts already launched wait for this one until their watchdog fires (timeout_ms)
      for (pt_pipeline* o : p->parts) o->broken = true;
      return r;
    }
  }
  p->t_next += n;
  if (where == PT_HOST) return group_finish(p);
  return PT_OK;
}

int group_finish(pt_pipeline* p) {
  int first_err = PT_OK;
  std::string msg;
  for (pt_pipeline* q : p->parts) {
    DevGuard dg(q->device);
    const int r = finish_impl(q);
    if (r != PT_OK && first_err == PT_OK) {
      first_err = r;
      msg = g_err;
    }
  }
  if (first_err != PT_OK) g_err = msg;
  return first_err;
}

}  // namespace

extern "C" {

int32_t pt_abi_version(void) { return PT_ABI_VERSION; }

const char* pt_last_error(void) { return g_err.c_str(); }

int pt_create(const pt_config* cfg, pt_pipeline** out) {
  if (!out) return fail(PT_EINVAL, "out is null");
  *out = nullptr;
  pt_pipeline* p = new pt_pipeline();
  int r;
  if (cfg && cfg->device_of_stage) {
    // one device for every local stage: a plain handle on that device; several: a group
    const int lo = cfg->local_stage_count ? cfg->local_stage_first : 0;
    const int hi = cfg->local_stage_count ? lo + cfg->local_stage_count : cfg->n_stages;
    bool one = true;
    for (int h = lo + 1; h < hi && h < cfg->n_stages && lo >= 0; ++h)
      one = one && cfg->device_of_stage[h] == cfg->device_of_stage[lo];
    const char* ve = getenv("PT_VIRTUAL_DEVICES");
    if (one && lo >= 0 && lo < cfg->n_stages && cfg->n_stages >= 1) {
      int ndev = 1;
      cudaGetDeviceCount(&ndev);
      int d = cfg->device_of_stage[lo];
      if (ve && atoi(ve) != 0 && ndev > 0) d %= ndev;
      if (d < 0 || d >= ndev) {
        r = fail(PT_EINVAL, "device_of_stage[" + std::to_string(lo) + "] = " + std::to_string(d) +
                                " is not a device of this process");
      } else {
        pt_config sub = *cfg;
        sub.device_of_stage = nullptr;
        DevGuard dg(d);
        r = create_impl(&sub, p);
      }
    } else {
      r = create_group(cfg, p);
    }
  } else {
    r = create_impl(cfg, p);
  }
  if (r != PT_OK) {
    std::string keep = g_err;
    pt_destroy(p);
    g_err = keep;
    return r;
  }
  *out = p;
  return PT_OK;
}

void pt_destroy(pt_pipeline* p) {
  if (!p) return;
  if (p->group()) {
    resident_stop(p);
    if (p->res.host) cudaFreeHost(p->res.host);
    for (pt_pipeline* q : p->parts) {
      DevGuard dg(q->device);
      cudaStreamSynchronize(q->stream);
    }
    for (pt_pipeline* q : p->parts) pt_destroy(q);
    delete p;
    return;
  }
  DevGuard dg(p->device);
  resident_stop(p);
  cudaDeviceSynchronize();
  if (p->res.host) cudaFreeHost(p->res.host);
  for (void* q : p->ipc_opened) cudaIpcCloseMemHandle(q);
  for (void* a : p->allocs)
    if (a) cudaFree(a);
  if (p->ev0) cudaEventDestroy(p->ev0);
  if (p->ev1) cudaEventDestroy(p->ev1);
  if (p->own_stream) cudaStreamDestroy(p->own_stream);
  if (p->pin) cudaFreeHost(p->pin);
  delete p;
}

int pt_set_params(pt_pipeline* p, int32_t layer, const float* W, const float* b, int32_t where) {
  if (!p) return fail(PT_EINVAL, "null handle");
  BusyGuard g(p);
  if (!g.ok) return fail(PT_EBUSY, "contract violation: handle used concurrently");
  if (p->group()) {
    PT_TRY(resident_stop(p));
    pt_pipeline* q = part_of_layer(p, layer);
    if (!q) return fail(PT_EINVAL, "layer " + std::to_string(layer) + " is not owned by this process");
    return pt_set_params(q, layer, W, b, where);
  }
  DevGuard dg(p->device);
  PT_TRY(resident_stop(p));
  std::string why;
  LayerHost* Lh = local_layer(p, layer, &why);
  if (!Lh) return fail(PT_EINVAL, why);
  const cudaMemcpyKind k = where == PT_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  if (p->panel) {
    // row-major staging -> the tiled buffer the next forward reads; the pending update of
    // earlier ticks no longer applies to this layer
    if (W) {
      const size_t nw = size_t(Lh->n_out) * Lh->n_in;
      PT_TRY(panel_rowbuf(p, nw));
      CUDA_TRY(cudaMemcpyAsync(p->rowbuf, W, nw * 4, k, p->stream));
      pt::pn_to_tiles<<<592, 256, 0, p->stream>>>(p->rowbuf, Lh->Wt[panel_cur(p, *Lh)], Lh->n_out, Lh->n_in, Lh->R,
                                                  Lh->C);
      CUDA_TRY(cudaGetLastError());
      Lh->set_tick = p->t_next;
    }
    if (b) CUDA_TRY(cudaMemcpyAsync(Lh->b, b, size_t(Lh->n_out) * 4, k, p->stream));
    CUDA_TRY(cudaStreamSynchronize(p->stream));
    return W ? upload_panel_desc(p) : PT_OK;
  }
  if (p->tile) {
    // row-major staging -> the tile kernel's blocked layout
    if (W) {
      const size_t nw = size_t(Lh->n_out) * Lh->n_in;
      PT_TRY(panel_rowbuf(p, nw));
      CUDA_TRY(cudaMemcpyAsync(p->rowbuf, W, nw * 4, k, p->stream));
      pt::tl_to_blocks<<<592, 256, 0, p->stream>>>(p->rowbuf, Lh->W, Lh->n_out, Lh->n_in);
      CUDA_TRY(cudaGetLastError());
    }
    if (b) CUDA_TRY(cudaMemcpyAsync(Lh->b, b, size_t(Lh->n_out) * 4, k, p->stream));
    CUDA_TRY(cudaStreamSynchronize(p->stream));
    return PT_OK;
  }
  if (W)
    CUDA_TRY(cudaMemcpy2D(Lh->W, size_t(Lh->ld_in) * 4, W, size_t(Lh->n_in) * 4, size_t(Lh->n_in) * 4,
                          size_t(Lh->n_out), k));
  if (b) CUDA_TRY(cudaMemcpy(Lh->b, b, size_t(Lh->n_out) * 4, k));
  p->legacy_dirty = true;
  return PT_OK;
}

int pt_get_params(pt_pipeline* p, int32_t layer, float* W, float* b, int32_t where) {
  if (!p) return fail(PT_EINVAL, "null handle");
  BusyGuard g(p);
  if (!g.ok) return fail(PT_EBUSY, "contract violation: extract called mid-step (SPEC.md:239)");
  if (p->group()) {
    PT_TRY(resident_stop(p));
    pt_pipeline* q = part_of_layer(p, layer);
    if (!q) return fail(PT_EINVAL, "layer " + std::to_string(layer) + " is not owned by this process");
    PT_TRY(group_finish(p));  // every part idle: the weights are a consistent tick
    return pt_get_params(q, layer, W, b, where);
  }
  DevGuard dg(p->device);
  PT_TRY(resident_stop(p));
  std::string why;
  LayerHost* Lh = local_layer(p, layer, &why);
  if (!Lh) return fail(PT_EINVAL, why);
  const cudaMemcpyKind k = where == PT_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  if (p->panel) {
    if (W) {
      // W^(T) = the stored W^(T-1) plus the update of tick T-1, if the next forward would apply it
      const long long T = p->t_next;
      const int h = stage_of_layer(p, layer);
      const bool pend = p->learn && !Lh->bw && p->lr != 0.f && T - 1 >= 2LL * p->D - h - 1 && T - 1 >= Lh->set_tick;
      const float* sdel = nullptr;
      const float* ahat = nullptr;
      if (pend) {
        const StageHost& S = p->stages[h - 1 - p->local_first];
        const long long Cp = (h < p->D && p->act_delay) ? T - 2 : T - 1;
        sdel = Lh->dpl + size_t((T - 1) & 1) * Lh->R * pt::PN_TS;
        ahat = S.pcache + size_t(Cp & 3) * S.cache_words + Lh->cache_in;
      }
      const size_t nw = size_t(Lh->n_out) * Lh->n_in;
      PT_TRY(panel_rowbuf(p, nw));
      pt::pn_from_tiles<<<592, 256, 0, p->stream>>>(Lh->Wt[panel_cur(p, *Lh)], p->rowbuf, Lh->n_out, Lh->n_in, Lh->C, sdel,
                                                    ahat, p->lr);
      CUDA_TRY(cudaGetLastError());
      CUDA_TRY(cudaMemcpyAsync(W, p->rowbuf, nw * 4, k, p->stream));
    }
    if (b) CUDA_TRY(cudaMemcpyAsync(b, Lh->b, size_t(Lh->n_out) * 4, k, p->stream));
    CUDA_TRY(cudaStreamSynchronize(p->stream));
    return PT_OK;
  }
  if (p->tile) {
    if (W) {
      const size_t nw = size_t(Lh->n_out) * Lh->n_in;
      PT_TRY(panel_rowbuf(p, nw));
      pt::tl_from_blocks<<<592, 256, 0, p->stream>>>(Lh->W, p->rowbuf, Lh->n_out, Lh->n_in);
      CUDA_TRY(cudaGetLastError());
      CUDA_TRY(cudaMemcpyAsync(W, p->rowbuf, nw * 4, k, p->stream));
    }
    if (b) CUDA_TRY(cudaMemcpyAsync(b, Lh->b, size_t(Lh->n_out) * 4, k, p->stream));
    CUDA_TRY(cudaStreamSynchronize(p->stream));
    return PT_OK;
  }
  if (W)
    CUDA_TRY(cudaMemcpy2D(W, size_t(Lh->n_in) * 4, Lh->W, size_t(Lh->ld_in) * 4, size_t(Lh->n_in) * 4,
                          size_t(Lh->n_out), k));
  if (b) CUDA_TRY(cudaMemcpy(b, Lh->b, size_t(Lh->n_out) * 4, k));
  return PT_OK;
}

int pt_run(pt_pipeline* p, const float* xs, const float* ys, int64_t n, float* outs, float* losses,
           uint8_t* valid, int32_t where) {
  if (!p) return fail(PT_EINVAL, "null handle");
  BusyGuard g(p);
  if (!g.ok) return fail(PT_EBUSY, "contract violation: pipeline_step called concurrently (SPEC.md:221)");
  if (where != PT_HOST && where != PT_DEVICE) return fail(PT_EINVAL, "where must be PT_HOST or PT_DEVICE");
  if (p->group()) {
    PT_TRY(resident_stop(p));
    return group_run(p, xs, ys, n, outs, losses, valid, where);
  }
  DevGuard dg(p->device);
  PT_TRY(resident_stop(p));
  return run_impl(p, xs, ys, n, outs, losses, valid, where);
}

int pt_step(pt_pipeline* p, const float* x, const float* y, float* out, float* loss, int32_t* valid,
            int32_t where) {
  if (!p) return fail(PT_EINVAL, "null handle");
  BusyGuard g(p);
  if (!g.ok) return fail(PT_EBUSY, "contract violation: pipeline_step called concurrently (SPEC.md:221)");
  uint8_t v8 = 0;
  int r;
  const bool grp = p->group();
  pt_pipeline* last = grp ? p->parts.back() : p;
  DevGuard dg(grp ? p->parts.front()->device : p->device);
  if (where == PT_HOST && resident_eligible(p)) return resident_step(p, x, y, out, loss, valid);
  PT_TRY(resident_stop(p));
  if (where == PT_HOST) {
    r = grp ? group_run(p, x, y, 1, out, loss, valid ? &v8 : nullptr, PT_HOST)
            : run_impl(p, x, y, 1, out, loss, valid ? &v8 : nullptr, PT_HOST);
    if (valid) *valid = v8;
  } else {
    // device I/O: valid is int32 on the caller side; go through the staging byte
    r = grp ? group_run(p, x, y, 1, out, loss, nullptr, PT_DEVICE) : run_impl(p, x, y, 1, out, loss, nullptr, PT_DEVICE);
    if (r == PT_OK) {
      r = grp ? group_finish(p) : finish_impl(p);
      if (valid && last->has_last()) {
        DevGuard dl(last->device);
        uint8_t hv = 0;
        if (cudaMemcpy(&hv, last->valid_stage, 1, cudaMemcpyDeviceToHost) != cudaSuccess)
          return fail(PT_ECUDA, "valid copy failed");
        int32_t v32 = hv;
        if (cudaMemcpy(valid, &v32, 4, cudaMemcpyHostToDevice) != cudaSuccess)
          return fail(PT_ECUDA, "valid copy failed");
      }
    }
  }
  return r;
}

int pt_sync(pt_pipeline* p) {
  if (!p) return fail(PT_EINVAL, "null handle");
  BusyGuard g(p);
  if (!g.ok) return fail(PT_EBUSY, "contract violation: handle used concurrently");
  if (p->group()) {
    PT_TRY(resident_stop(p));
    return group_finish(p);
  }
  DevGuard dg(p->device);
  PT_TRY(resident_stop(p));
  return finish_impl(p);
}

int pt_set_stream(pt_pipeline* p, void* stream) {
  if (!p) return fail(PT_EINVAL, "null handle");
  if (p->group()) {
    if (stream) return fail(PT_EUNSUPPORTED, "a multi-device handle runs one private stream per device");
    return PT_OK;
  }
  DevGuard dg(p->device);
  PT_TRY(resident_stop(p));
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  p->stream = stream ? reinterpret_cast<cudaStream_t>(stream) : p->own_stream;
  return PT_OK;
}

int pt_get_stream(const pt_pipeline* p, void** stream) {
  if (!p || !stream) return fail(PT_EINVAL, "null argument");
  // multi-device handle: the stream of the part that owns stage D (where outputs are written)
  *stream = reinterpret_cast<void*>(p->group() ? p->parts.back()->stream : p->stream);
  return PT_OK;
}

int pt_last_kernel_ms(pt_pipeline* p, float* ms) {
  if (!p || !ms) return fail(PT_EINVAL, "null argument");
  if (p->group()) {  // the slowest device
    float worst = 0.f;
    for (pt_pipeline* q : p->parts) {
      float m = 0.f;
      PT_TRY(pt_last_kernel_ms(q, &m));
      worst = std::max(worst, m);
    }
    *ms = worst;
    return PT_OK;
  }
  DevGuard dg(p->device);
  if (!p->timed) return fail(PT_EINVAL, "no kernel has run yet");
  CUDA_TRY(cudaEventSynchronize(p->ev1));
  CUDA_TRY(cudaEventElapsedTime(ms, p->ev0, p->ev1));
  return PT_OK;
}

int64_t pt_tick(pt_pipeline* p) { return p ? p->t_next : -1; }

int32_t pt_stage_device(const pt_pipeline* p, int32_t stage) {
  if (!p) return fail(PT_EINVAL, "null handle");
  if (p->group()) {
    for (const pt_pipeline* q : p->parts)
      if (stage - 1 >= q->local_first && stage - 1 < q->local_first + q->local_count) return q->device;
    return -1;
  }
  return (stage - 1 >= p->local_first && stage - 1 < p->local_first + p->local_count) ? p->device : -1;
}

int32_t pt_kernel_path(const pt_pipeline* p) {
  if (!p) return fail(PT_EINVAL, "null handle");
  if (p->group()) return pt_kernel_path(p->parts.front());
  return p->tile ? PT_PATH_TILE : p->panel ? PT_PATH_PANEL : PT_PATH_TICK;
}

int pt_set_trace(pt_pipeline* p, int32_t cta, int32_t cap) {
  if (!p) return fail(PT_EINVAL, "null handle");
  if (p->group()) {
    PT_TRY(resident_stop(p));
    return pt_set_trace(p->parts.front(), cta, cap);  // the stage-1 device
  }
  DevGuard dg(p->device);
  PT_TRY(resident_stop(p));
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  dev_free(p, p->d_trace);
  p->d_trace = nullptr;
  p->trace_cap = 0;
  if (cap > 0) {
    if (cta < -1 || cta >= p->G) return fail(PT_EINVAL, "trace CTA out of range (-1 = all CTAs, step ends)");
    PT_TRY(dev_alloc(p, reinterpret_cast<void**>(&p->d_trace), size_t(cap) * sizeof(u64)));
    p->trace_cap = cap;
    p->trace_cta = cta;
  }
  return PT_OK;
}

int pt_get_trace(pt_pipeline* p, uint64_t* out, int32_t cap) {
  if (!p || !out) return fail(PT_EINVAL, "null argument");
  if (p->group()) {
    PT_TRY(resident_stop(p));
    return pt_get_trace(p->parts.front(), out, cap);
  }
  DevGuard dg(p->device);
  PT_TRY(resident_stop(p));
  if (!p->d_trace) return fail(PT_EINVAL, "tracing is off (pt_set_trace)");
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  const int n = std::min(cap, p->trace_cap);
  CUDA_TRY(cudaMemcpy(out, p->d_trace, size_t(n) * sizeof(u64), cudaMemcpyDeviceToHost));
  return PT_OK;
}

int pt_ipc_export(pt_pipeline* p, int32_t stage, void* buf, size_t cap, size_t* len) {
  if (!p || !buf || !len) return fail(PT_EINVAL, "null argument");
  if (cap < sizeof(IpcBlob)) return fail(PT_EINVAL, "buffer too small");
  if (p->group()) return fail(PT_EUNSUPPORTED, "export a stage of a single-device handle");
  DevGuard dg(p->device);
  PT_TRY(resident_stop(p));
  const int s = stage - 1 - p->local_first;
  if (s < 0 || s >= int(p->stages.size())) return fail(PT_EINVAL, "stage is not local");
  const StageHost& S = p->stages[s];
  IpcBlob b;
  memset(&b, 0, sizeof(b));
  b.magic = PT_IPC_MAGIC;
  b.abi = PT_ABI_VERSION;
  b.stage = stage;
  b.G = S.ncta > 0 ? S.ncta : p->G;
  b.M = p->M;
  b.ld0 = S.ld0;
  b.ldk = S.ldk;
  char* block = p->tile ? S.tcomm : S.comm;
  b.comm_bytes = int64_t(p->tile ? p->tile_layout_of(stage - 1).total : p->layout_of(stage - 1).total);
  b.pid = int64_t(getpid());
  b.dev_ptr = uint64_t(reinterpret_cast<uintptr_t>(block));
  CUDA_TRY(cudaIpcGetMemHandle(&b.handle, block));
  memcpy(buf, &b, sizeof(b));
  *len = sizeof(b);
  return PT_OK;
}

int pt_ipc_import(pt_pipeline* p, const void* buf, size_t len) {
  if (!p || !buf) return fail(PT_EINVAL, "null argument");
  if (len < sizeof(IpcBlob)) return fail(PT_EINVAL, "IPC blob too short");
  if (p->group()) return fail(PT_EUNSUPPORTED, "import into a single-device handle");
  DevGuard dg(p->device);
  PT_TRY(resident_stop(p));
  IpcBlob b;
  memcpy(&b, buf, sizeof(b));
  if (b.magic != PT_IPC_MAGIC || b.abi != PT_ABI_VERSION) return fail(PT_EINVAL, "not a partime IPC blob");
  const int s0 = b.stage - 1;
  if (s0 < 0 || s0 >= p->D) return fail(PT_EINVAL, "IPC blob stage out of range");
  if (b.M != p->M || b.ld0 != p->stage_ld0(s0) || b.ldk != p->stage_ldk(s0) ||
      b.comm_bytes != int64_t(p->tile ? p->tile_layout_of(s0).total : p->layout_of(s0).total))
    return fail(PT_EINVAL, "IPC blob shape does not match this pipeline's config");
  const int lo = p->local_first, hi = p->local_first + p->local_count;  // [lo, hi)
  if (s0 >= lo && s0 < hi) return fail(PT_EINVAL, "stage is local; nothing to import");
  if (s0 != lo - 1 && s0 != hi) return fail(PT_EINVAL, "stage is not a neighbour of the local stages");
  void* ptr = nullptr;
  if (b.pid == int64_t(getpid())) {
    ptr = reinterpret_cast<void*>(uintptr_t(b.dev_ptr));  // same process: CUDA IPC cannot reopen it
  } else {
    CUDA_TRY(cudaIpcOpenMemHandle(&ptr, b.handle, cudaIpcMemLazyEnablePeerAccess));
    p->ipc_opened.push_back(ptr);
  }
  if (p->tile) {
    if (s0 == lo - 1) {
      p->stages.front().tup = static_cast<char*>(ptr);
      p->stages.front().up_remote = true;
    } else {
      p->stages.back().tdown = static_cast<char*>(ptr);
      p->stages.back().down_remote = true;
    }
    return upload_tile_stages(p);
  }
  if (s0 == lo - 1) {
    p->stages.front().up = static_cast<char*>(ptr);
    p->stages.front().G_up = b.G;
    p->stages.front().up_remote = true;
  } else {
    p->stages.back().down = static_cast<char*>(ptr);
    p->stages.back().G_down = b.G;
    p->stages.back().down_remote = true;
  }
  return upload_desc(p);
}

}  // extern "C"
