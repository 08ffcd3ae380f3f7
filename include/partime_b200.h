/*
 * partime_b200.h: C ABI of the B200 PARTIME per-tick pipeline engine.
 *
 * The reference has no FFI. Its boundary for this path is Python only:
 *   - SPEC engine API (reference SPEC.md:208-243): pipeline_build / pipeline_step /
 *     pipeline_run / pipeline_extract_weights;
 *   - paper API (reference PAPER.md:640-672): partime.pipeline.Pipeline(...).forward(inp, target).
 * Each entry point below names the reference operation it replaces. The Python
 * mirrors (the `pipestream` package = paper_2210_09147_b200.engine and friends, and the
 * `partime` package = paper_2210_09147_b200.partime) bind this header through ctypes
 * (see INTEGRATION.md).
 *
 * Conventions
 *   - return 0 on success, a negative PT_E* code on error; pt_last_error() gives a
 *     thread-local message;
 *   - plain pointers and sizes; no torch types. `where` says whether caller
 *     buffers are host (PT_HOST) or device (PT_DEVICE) memory;
 *   - a handle is single-driver (reference SPEC.md:261). Concurrent calls on one
 *     handle return PT_EBUSY ("step called concurrently").
 *
 * Layout
 *   - weights W[l] are row-major [dims[l+1], dims[l]] fp32 (out x in);
 *   - activations are [M, dims[*]] fp32, where M is the micro-batch (1 = per-sample stream).
 *   Padding is internal; callers always see dense arrays.
 */
#ifndef PARTIME_B200_H
#define PARTIME_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PT_ABI_VERSION 2

/* error codes */
#define PT_OK            0
#define PT_EINVAL       -1   /* bad argument / plan / shape */
#define PT_EUNSUPPORTED -2   /* valid in the reference, not implemented on this path */
#define PT_ECUDA        -3   /* CUDA runtime error */
#define PT_EBUSY        -4   /* concurrent use of one handle */
#define PT_ENONFINITE   -5   /* non-finite loss; message names the first bad tick */
#define PT_ETIMEOUT     -6   /* a stage waited past cfg.timeout_ms for a neighbour (device watchdog) */
#define PT_ESTATE       -7   /* handle unusable after an earlier device-side failure */

/* memory location of caller buffers */
#define PT_HOST   0
#define PT_DEVICE 1

/* activation applied after each dense layer (the dense+act pair is the fusion unit) */
#define PT_ACT_NONE 0
#define PT_ACT_RELU 1
#define PT_ACT_TANH 2

#define PT_LOSS_MSE 0        /* mean over M*F elements */
#define PT_LOSS_SOFTMAX_CE 1 /* mean over M of -log softmax[target]; y holds one
                                class index per sample; a target outside [0, F) -> PT_EINVAL */

#define PT_OPT_SGD 0
#define PT_OPT_ADAM 1        /* beta = (0.9, 0.999), eps = 1e-8; the step count
                                starts at the stage's warm-up gate t >= 2D-h-1 */

typedef struct pt_pipeline pt_pipeline;

/* Pipeline description. It replaces the arguments of pipeline_build
 * and Pipeline.__init__. All arrays are copied. */
typedef struct pt_config {
  int32_t n_layers;                  /* L dense layers */
  const int32_t* dims;               /* L+1 widths: dims[0] = input, dims[L] = F */
  const int32_t* act;                /* L activations (PT_ACT_*) */
  int32_t loss;                      /* PT_LOSS_* */
  int32_t optimizer;                 /* PT_OPT_* */
  float lr;                          /* learning rate (SGD / Adam step size) */
  int32_t n_stages;                  /* D */
  const int32_t* stage_first_layer;  /* D+1 layer indices; [0] = 0, [D] = L (StagePlan) */
  int32_t batch;                     /* M rows per tick (1..64) */
  int32_t learn;                     /* 1: forward+backward+update; 0: inference wave */
  int32_t act_delay;                 /* 1: SPEC reading (stages h<D backprop the previous tick's
                                        cache); 0: paper reading (current tick) */
  int32_t local_stage_first;         /* stages owned by this process, all on the current */
  int32_t local_stage_count;         /*   device; count 0 = all stages (single process) */
  int32_t grid;                      /* CTAs per device; 0 = one per SM */
  int32_t timeout_ms;                /* device watchdog for cross-stage waits; 0 = 30000 */
  const int32_t* device_of_stage;    /* D CUDA device ordinals ("the list of available
                                        GPU devices ... it can be smaller, making multiple stages
                                        execute on the same device"), or NULL = the current device.
                                        Stages of one device must be contiguous. When the local
                                        stages span several devices the handle drives one part per
                                        device from this process: peer access is enabled and the
                                        parts exchange activations / gradients by peer stores over
                                        NVLink (same tagged-slot + credit protocol as CUDA IPC) */
} pt_config;

/* pipeline_build: allocate all buffers, zero slots/caches, init nothing
 * else; weights are zero until pt_set_params. */
int pt_create(const pt_config* cfg, pt_pipeline** out);

/* Upload/download one dense layer's parameters (layer = global index, must be local).
 * W: [dims[l+1], dims[l]], b: [dims[l+1]]. pt_get_params is pipeline_extract_weights
 * (SPEC.md:235-243); it synchronises the handle's stream first. */
int pt_set_params(pt_pipeline* p, int32_t layer, const float* W, const float* b, int32_t where);
int pt_get_params(pt_pipeline* p, int32_t layer, float* W, float* b, int32_t where);

/* pipeline_step / Pipeline.forward: one tick, synchronous.
 * x: [M, dims[0]] (needed iff stage 1 is local), y: [M, F] (MSE) or [M] class indices
 * (softmax-CE) target of the SAME tick
 * (queued internally for D-1 ticks). out: [M, F] output of sample t-(D-1),
 * loss: scalar (NaN when invalid), valid: t >= D-1. Any of out/loss/valid may be NULL. */
int pt_step(pt_pipeline* p, const float* x, const float* y, float* out, float* loss,
            int32_t* valid, int32_t where);

/* pipeline_run over n ticks with no per-tick host round trip.
 * xs: [n, M, dims[0]], ys: [n, M, F], outs: [n, M, F], losses: [n], valid: [n].
 * With where == PT_DEVICE the call is asynchronous on the handle's stream; errors such as
 * PT_ENONFINITE surface at pt_sync. With PT_HOST it copies in, runs and copies out. */
int pt_run(pt_pipeline* p, const float* xs, const float* ys, int64_t n, float* outs,
           float* losses, uint8_t* valid, int32_t where);

/* Wait for queued work and report deferred device-side errors. */
int pt_sync(pt_pipeline* p);

/* Use an external CUDA stream (cudaStream_t as void*); NULL restores the private stream. */
int pt_set_stream(pt_pipeline* p, void* stream);

/* The stream the handle enqueues on (its private non-blocking stream unless pt_set_stream
 * chose another). Callers passing PT_DEVICE buffers written on another stream must order that
 * stream before pt_run/pt_step (cudaStreamWaitEvent), as the Python engine does. */
int pt_get_stream(const pt_pipeline* p, void** stream);

/* Device time (ms) of the tick kernel of the last pt_run/pt_step, from CUDA events on the
 * handle's stream; valid after pt_sync. */
int pt_last_kernel_ms(pt_pipeline* p, float* ms);

/* Device ordinal that runs 1-based `stage` (device_of_stage, or the creating device); -1 if
 * the stage is not local. Device-buffer callers of a multi-device handle pass xs on stage 1's
 * device and ys / outs / losses / valid on stage D's. */
int32_t pt_stage_device(const pt_pipeline* p, int32_t stage);

/* Next global tick index (number of ticks executed so far). */
int64_t pt_tick(pt_pipeline* p);

/* Which device path the handle runs (no reference counterpart; the engine picks it at
 * pt_create): PT_PATH_PANEL = batch-1 panel kernel (16 x 16-tiled weights, column-owned
 * backward; SGD or Adam; PT_PANEL=0 disables), PT_PATH_TILE = tcgen05 tensor-core tile kernel
 * (batch 16, 32 or 64, widths % 256 == 0; SGD or Adam, MSE or softmax-CE; PT_TILE=0 disables),
 * PT_PATH_TICK = row-owned SIMT tick kernel (every other batch and shape). All three run one
 * stage per process / GPU or several stages in one process. Negative = error. */
#define PT_PATH_TICK 0
#define PT_PATH_TILE 1
#define PT_PATH_PANEL 2
int32_t pt_kernel_path(const pt_pipeline* p);

/* Diagnostics (no reference counterpart): record device timestamps of one CTA's step
 * phases during each run, (code << 56) | globaltimer ns. The first cap/2 entries hold
 * consumer events, the rest producer events. cap = 0 turns tracing off. */
int pt_set_trace(pt_pipeline* p, int32_t cta, int32_t cap);
int pt_get_trace(pt_pipeline* p, uint64_t* out, int32_t cap);

/* Multi-process (one process per GPU): export the inbound-slot block of a local stage
 * (a CUDA IPC handle plus shapes), and import a neighbour's block so the kernel can store
 * activations/gradients and ready flags straight into the peer's memory over NVLink. */
int pt_ipc_export(pt_pipeline* p, int32_t stage, void* buf, size_t cap, size_t* len);
int pt_ipc_import(pt_pipeline* p, const void* buf, size_t len);

void pt_destroy(pt_pipeline* p);
const char* pt_last_error(void);
int32_t pt_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PARTIME_B200_H */
