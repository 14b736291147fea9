/*
 * ptq_b200.h -- C ABI of the B200 PTQ-configuration evaluator.
 *
 * Drop-in boundary for the reference's evaluator plug point
 *   Evaluator = Callable[[QuantConfig], float]            (ptqtune/tuner.py:44)
 *   make_accuracy_evaluator(g, d, seed, profile)          (ptqtune/tuner.py:434-444)
 * ("ptqtune/" = /root/reference/pkg/src/ptqtune/).  The reference is pure
 * Python, so the binding a maintainer adds is a ctypes stub;
 * paper_2202_05048_b200/_lib.py is exactly that stub.
 *
 * Conventions: plain C types only, host pointers in and out, caller owns all
 * host buffers; every entry point returns 0 on success or a negative
 * PTQ_E* status and never throws across the boundary; ptq_last_error()
 * describes the most recent failure of the calling thread.  One context is
 * bound to one CUDA device and is not safe for concurrent calls (the Python
 * wrapper serialises calls with a lock, tuner.py:192-203 may call from
 * threads).
 */
#ifndef PTQ_B200_H
#define PTQ_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PTQ_OK 0
#define PTQ_EINVAL (-1)   /* bad argument / unsupported graph (GraphError, ValueError) */
#define PTQ_ECUDA (-2)    /* CUDA runtime or kernel failure */
#define PTQ_ESTATE (-3)   /* call out of order (e.g. eval before ranges are set) */
#define PTQ_ENOMEM (-4)   /* device allocation failed */

#define PTQ_NBINS 2048
#define PTQ_NWINDOWS 1921 /* KL candidate windows i = 128..2048 (clipping.py:78) */

/* node kinds: the reference IR vocabulary (ptqtune/ir.py:31-33) */
enum ptq_node_kind {
  PTQ_CONV = 0, PTQ_DWCONV = 1, PTQ_PWCONV = 2, PTQ_FC = 3, PTQ_RELU = 4,
  PTQ_MAXPOOL = 5, PTQ_AVGPOOL = 6, PTQ_ADD = 7, PTQ_CONCAT = 8, PTQ_SOFTMAX = 9
};

#define PTQ_MAX_INPUTS 8

/* One IR node (ptqtune/ir.py:40-64).  Tensor ids: 0 = graph input, i+1 = output
 * of node i (so tensor ids equal the calibration-cache order, calibration.py:81). */
typedef struct {
  int32_t kind;
  int32_t n_inputs;                 /* data inputs */
  int32_t inputs[PTQ_MAX_INPUTS];   /* tensor ids */
  int32_t weight;                   /* index into weights[] or -1 */
  int32_t bias;                     /* index into weights[] or -1 */
  int32_t kernel, stride, pad;      /* conv/pool attributes (ir.py:119-150) */
} ptq_node_desc;

typedef struct {
  const float* data;                /* host fp32, reference layout (OIHW / (O, F) / (O,)) */
  int64_t shape[4];
  int32_t ndim;
} ptq_weight_desc;

typedef struct {
  int32_t n_nodes;
  const ptq_node_desc* nodes;
  int32_t n_weights;
  const ptq_weight_desc* weights;
  int32_t in_c, in_h, in_w;         /* Graph.input_shape */
  int32_t n_classes;                /* Graph.output_classes */
} ptq_graph_desc;

/* QuantConfig (ptqtune/quantize.py:54-84) as small integers, in the reference's
 * enumeration order: cache {S1,S2,S3}, scheme {Asymmetric, Symmetric,
 * SymmetricUint8, SymmetricPower2}, clipping {Max, KL}, granularity {Tensor,
 * Channel}, mixed {Off, FirstLastFp32}, fusion {0,1} (numerically neutral). */
typedef struct {
  int32_t cache, scheme, clipping, granularity, mixed, fusion;
} ptq_config;

typedef struct ptq_ctx ptq_ctx;

const char* ptq_last_error(void);
int ptq_version(void);

/* Upload graph, images (N, C, H, W fp32, calibration pool first) and the eval
 * labels (n_images - n_calib int64) to device `device`.  Replaces the state the
 * reference builds inside make_accuracy_evaluator (tuner.py:434-438).
 * Returns once the calibration images are resident; the evaluation images keep
 * uploading in the background (overlapping calibration), so `images` must stay
 * valid until ptq_destroy (the first call that needs them waits for the copy). */
int ptq_create(ptq_ctx** out, int device, const ptq_graph_desc* g, const float* images,
               const int64_t* eval_labels, int64_t n_images, int64_t n_calib);
int ptq_destroy(ptq_ctx* ctx);

/* Number of histogram tensors T (graph input + one per node). */
int ptq_num_tensors(const ptq_ctx* ctx, int32_t* T);

/* Calibrate the three caches (calibration.py:57-112 with select_images ids
 * supplied by the host, tuner.py:438): one fp32 forward over the union of the
 * image ids, exact per-tensor min/max, 2048-bin histograms.  ids: concatenated
 * calibration-pool indices of cache 0..n_caches-1, sizes in cache_sizes.
 * Outputs (may be NULL): ranges [n_caches][T][2] fp32 (min_seen, max_seen),
 * counts [n_caches][T][2048] int64, n_samples [n_caches][T]. */
int ptq_calibrate(ptq_ctx* ctx, int32_t n_caches, const int32_t* cache_sizes, const int64_t* ids,
                  float* ranges, int64_t* counts, int64_t* n_samples);

/* The same in two phases, for calibration images sharded across ranks: phase 1
 * runs the fp32 forward over this rank's ids and returns the local per-cache
 * ranges (+inf/-inf for a cache with no local images); the host MIN/MAX-reduces
 * them across ranks; phase 2 bins the retained activations with the global
 * ranges (the host SUM-reduces the counts).  sizes may contain zeros. */
int ptq_calib_forward(ptq_ctx* ctx, int32_t n_caches, const int32_t* cache_sizes,
                      const int64_t* ids, float* local_ranges);
int ptq_calib_histogram(ptq_ctx* ctx, const float* ranges, int64_t* counts);

/* KL sweep (clipping.py:55-86): kl[h][w] for window width 128+w of histogram h;
 * +inf for infeasible windows and for histograms the reference does not sweep
 * (min == max or empty).  counts [n_hist][2048], ranges [n_hist][2] as above. */
int ptq_kl_sweep(ptq_ctx* ctx, int32_t n_hist, const int64_t* counts, const float* ranges,
                 double* kl);

/* EXTENSION (not in the reference: clipped_range rejects "Percentile", clipping.py:91-92;
 * parity unpinned -- checked against oracle.percentile_range only).  Percentile clipping
 * of n_hist histograms on the device, one CTA per histogram: out[h] = (edge[lo_idx],
 * edge[hi_idx + 1]) with hi_idx = first bin whose cumulative count >= fl(q N), lo_idx =
 * first bin whose cumulative count > fl(fl(1 - q) N), q = pct / 100, edges as numpy's
 * histogram (calibration.py:81-91); lo == hi or empty histograms keep (lo, hi).  counts
 * [n_hist][2048], ranges [n_hist][2] fp32, out [n_hist][2] fp64 -- the format
 * ptq_set_clip_ranges takes. */
int ptq_percentile_ranges(ptq_ctx* ctx, int32_t n_hist, const int64_t* counts, const float* ranges,
                          double pct, double* out);

/* Install the clipped ranges (clipped_range, clipping.py:89-96) for
 * (cache, clipping): ranges [T][2] fp64 (lo, hi). */
int ptq_set_clip_ranges(ptq_ctx* ctx, int32_t cache, int32_t clipping, const double* ranges);

/* Device-side preparation that every config shares: activation params for all
 * 24 (cache, scheme, clipping) variants, the 8 (scheme, granularity) weight
 * variants and, for FirstLastFp32, the config-invariant fp32 first layer of the
 * eval set.  Called implicitly by ptq_eval_configs when needed. */
int ptq_prepare(ptq_ctx* ctx);

/* Evaluate configs (quantize_model + evaluate_quantized, quantize.py:133-211,
 * intexec.py:337-366): correct[i] = number of eval images whose top-1 matches. */
int ptq_eval_configs(ptq_ctx* ctx, const ptq_config* cfgs, int32_t n_cfg, int64_t* correct);

/* Parity probes (tests): int8 codes of tensor `tensor` for one config over the
 * eval set in NCHW order [n_eval][C][H][W] (fp32-domain tensors return
 * PTQ_EINVAL).  Returns the element count through *n_out when out == NULL. */
/* Quantized state of one int8 compute node under `cfg`, in the reference's layouts, for the
 * .qtm8 emitter (replaces the QuantizedGraph fields quantize.py:133-211 builds and
 * save_quantized, quantize.py:254-300, writes): weight codes [cout][cin][k][k] (depthwise
 * [C][1][k][k], fc [cout][features]), per-output-channel weight scale / zero point (the same
 * value repeated for per-tensor granularity) and int32 bias codes (if the node has a bias). */
int ptq_export_layer(ptq_ctx* ctx, const ptq_config* cfg, int32_t node, int8_t* codes, float* wscale,
                     int32_t* wzp, int32_t* bias);
int ptq_probe_codes(ptq_ctx* ctx, const ptq_config* cfg, int32_t tensor, int8_t* out,
                    int64_t* n_out);
/* Parity probes over a subset of eval images (imgs: eval-set indices, n_imgs of them); every
 * output is in the reference's NCHW layout, image-major in the order of imgs.
 *  ptq_probe_tensors  int8 codes of n_tensors tensors after one evaluation of cfg (the codes the
 *                     reference's run_quantized sink sees, intexec.py:148-301): out holds
 *                     [n_imgs][C][H][W] per tensor, back to back; found[k] = 0 for tensors the
 *                     fused epilogues never materialise (fusion option on).
 *  ptq_probe_acc      the int32-saturated accumulator acc + bias of int8 compute node `node`
 *                     (intexec.py:177-190), taken from the same tcgen05 / depthwise kernel launch
 *                     with an accumulator-storing epilogue: [n_imgs][Cout][OH][OW] ([n_imgs][Cout]
 *                     for fc).
 *  ptq_probe_output   run_quantized's return value (intexec.py:337-351): dequantize_array of the
 *                     output codes (schemes.py:153-155, on the device) or the fp32 scores when
 *                     the last layer runs in fp32: [n_imgs][classes].
 *  ptq_probe_f32      an fp32-domain tensor of cfg (FirstLastFp32 layers, intexec.py:304-334).
 *  ptq_minmax_host    the calibration min/max kernels (calibration.py:67-76) over a host array
 *                     [n_img][elems]: range = (min, max) as fp32. */
int ptq_probe_tensors(ptq_ctx* ctx, const ptq_config* cfg, int32_t n_tensors, const int32_t* tensors,
                      int32_t n_imgs, const int64_t* imgs, int8_t* out, int32_t* found);
int ptq_probe_acc(ptq_ctx* ctx, const ptq_config* cfg, int32_t node, int32_t n_imgs, const int64_t* imgs,
                  int32_t* out);
int ptq_probe_output(ptq_ctx* ctx, const ptq_config* cfg, int32_t n_imgs, const int64_t* imgs, float* out);
int ptq_probe_f32(ptq_ctx* ctx, const ptq_config* cfg, int32_t tensor, int32_t n_imgs, const int64_t* imgs,
                  float* out);
int ptq_minmax_host(ptq_ctx* ctx, const float* x, int32_t n_img, int64_t elems, float* range);
/* Activation params the device derived for one variant: scale/zp [T]. */
int ptq_probe_act_params(ptq_ctx* ctx, int32_t cache, int32_t scheme, int32_t clipping,
                         float* scale, int32_t* zp);
/* Histogram a host array exactly like np.histogram(x.astype(f64), 2048, (lo, hi)). */
int ptq_histogram_host(ptq_ctx* ctx, const float* x, int64_t n, float lo, float hi,
                       int64_t* counts);
/* Runtime options: "conv_ref" (1 = CUDA-core reference conv instead of tcgen05,
 * tests only), "fusion" (0 = materialise every tensor so each can be probed),
 * "eval_chunk" (images per eval pass; default = whole eval set), "time_conv" (N =
 * record CUDA events around the int8 conv launches of the first N configs of each
 * ptq_eval_configs call, for ptq_last_stats),
 * "reset_stats" (zero the cumulative kernel-launch counter).  A/B switches for tests, each
 * path bit-identical to its fallback: "tma" (0 = gather A operand), "kwr" (kw-reuse slabs),
 * "subsample" (0 = strided 1x1 convs gather directly), "dwconv_v4" (2 register-tap 3x3,
 * 1 four-channel, 0 scalar depthwise), "concat_v16" (0 = per-byte concat requant),
 * "fx" (0 = fp64 requant epilogue instead of the exact fixed-point one), "tio" (0 = direct
 * global epilogue stores instead of shared tiles + TMA), "hist_multi" (0 = one histogram
 * launch per tensor), "rs_mma" (0 = weight-zero-point row sums from the row-sum warp /
 * pixel-sum passes instead of the MMA's K-indicator columns), "skip_pf" (0 = no L2 prefetch
 * of the fused-add operand tiles). */
int ptq_set_option(ptq_ctx* ctx, const char* key, int64_t value);
/* Statistics: cumulative kernel launches (option "reset_stats" zeroes it) and, for the
 * last ptq_eval_configs call, the summed CUDA-event time of the int8 conv launches of
 * the first "time_conv" configs, their algorithmic int8 ops (2*M*N*K, unpadded dims),
 * the number of timed conv launches and the total number of conv launches. */
int ptq_last_stats(const ptq_ctx* ctx, int64_t* kernel_launches, double* conv_ms_event,
                   double* conv_ops, int64_t* conv_launches, int64_t* conv_launches_total);
/* Per-launch CUDA-event times (ms) of the timed conv launches of the last
 * ptq_eval_configs call, in launch order; *n = number available. */
int ptq_conv_timings(const ptq_ctx* ctx, float* ms, int64_t cap, int64_t* n);
/* The CUDA stream (cudaStream_t) every kernel of this context runs on. */
int ptq_stream(const ptq_ctx* ctx, void** stream);

#ifdef __cplusplus
}
#endif
#endif /* PTQ_B200_H */
