// ptq_b200 runtime: graph lowering, device memory, and the C ABI
// (include/ptq_b200.h).  Host C++ only; every FLOP runs in the kernels of
// k_calib.cu (F1, F2), k_quant.cu (F3), k_conv_tc.cu (F4) and k_fp32.cu.
//
// The quantize_model domain/parameter rules restated here follow
// /root/reference/pkg/src/ptqtune/quantize.py:116-202:
//   * every tensor's params come from one calibration histogram ("psrc");
//   * a compute/add node whose output feeds exactly one relu takes the relu
//     output's histogram (narrowing, :125-130);
//   * relu/maxpool/avgpool/softmax adopt their input's params (:198-202);
//   * FirstLastFp32 keeps the first and last compute nodes in fp32 (:143-147);
//     the graph input and the last layer's output stay unquantized.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <stdexcept>
#include <string>
#include <array>
#include <thread>
#include <atomic>
#include <vector>

#include "kernels.h"
#include "ptq_b200.h"

using namespace ptq;

namespace {

thread_local std::string g_err;

// PTQ_TRACE=1: device-synchronised wall time of every runtime phase on stderr
struct Trace {
  const char* name;
  std::chrono::steady_clock::time_point t0;
  bool on;
  explicit Trace(const char* n) : name(n), on(std::getenv("PTQ_TRACE") != nullptr) {
    if (on) {
      cudaDeviceSynchronize();
      t0 = std::chrono::steady_clock::now();
    }
  }
  ~Trace() {
    if (!on) return;
    cudaDeviceSynchronize();
    double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    std::fprintf(stderr, "[ptq-trace] %-28s %9.3f ms\n", name, ms);
  }
};

struct Err {
  int code;
  std::string msg;
};

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess)                                                               \
      throw Err{e_ == cudaErrorMemoryAllocation ? PTQ_ENOMEM : PTQ_ECUDA,                \
                std::string(#x) + " -> " + cudaGetErrorString(e_)};                      \
  } while (0)
#define REQ(cond, msg)                                   \
  do {                                                   \
    if (!(cond)) throw Err{PTQ_EINVAL, std::string(msg)}; \
  } while (0)

inline int rup(int x, int m) { return (x + m - 1) / m * m; }

struct NodeI {
  int kind;
  std::vector<int> in;
  int out;
  int weight, bias, k, stride, pad;
};
struct TensorI {
  int c, h, w;
  int64_t elems;
  int producer = -1;
  std::vector<int> consumers;
};

bool is_compute(int k) { return k == PTQ_CONV || k == PTQ_DWCONV || k == PTQ_PWCONV || k == PTQ_FC; }
bool is_tc(int k) { return k == PTQ_CONV || k == PTQ_PWCONV || k == PTQ_FC; }

// per-compute-node device weights
struct WeightsDev {
  int cout = 0, cin = 0, k = 1, fc_hw = 0, cin_p = 0;
  int bn = 0, n_kiter = 0, n_chunks = 0, kreal = 0;
  int brows_mask = 0;           // variants whose B tiles carry 16 K-indicator rows (rs_mma)
  int var_rows[8] = {};         // B rows per tile of each variant (bn, or bn + 16)
  int64_t var_off[9] = {};      // byte offset of each variant's codes (var_off[8] = total)
  bool im2col = false;          // few-channel conv: packed im2col + 1x1 tensor-core GEMM
  bool sub1x1 = false;          // strided 1x1 conv: subsampled input + stride-1 pointwise GEMM
  int im_cp = 0;                // im2col row pitch (k*k*Cin rounded up to 16)
  int q_cin_p = 0, q_k = 1, q_fc_hw = 0;   // weight-quantizer view of the K layout
  float* f32_gemm = nullptr;    // [K][cout] fp32 (NHWC K order) for the fp32 path, or dw [C][k*k]
  float* f32_bias = nullptr;
  int8_t* codes = nullptr;      // 8 variants back to back (var_off)
  int64_t bytes_per_variant = 0;  // largest variant (dw: every variant)
  float* scale = nullptr;       // [8][cout]
  int* zp = nullptr;            // [8][cout]
  int* wsum = nullptr;          // [8][cout]
  bool has_wzp[8] = {};
  double* mult = nullptr;       // [cout]
  int* biasq = nullptr;         // [cout]
  LayerRt* rt = nullptr;
  EpiParam* ep = nullptr;       // [cout] tensor-core epilogue constants
  int8_t* addtab = nullptr;     // [PTQ_ADDTAB_BYTES] fused-add lookup table (layers with a fused add)
};

struct Plan {
  bool built = false;
  int mixed = 0;
  std::vector<int> psrc;         // per tensor: histogram id or -1 (fp32 domain)
  std::vector<char> fp32node;    // per node
  std::vector<char> skip;        // node fused into an earlier one
  std::vector<int> mat;          // per compute node: tensor id materialised by its epilogue
  std::vector<int> relu_hist, add_node, add_other, add_is_a, add_relu_hist;
  int prefix_end = -1;           // mixed: last node index of the config-invariant fp32 prefix
  std::vector<int> layer_of;     // node -> index into d_layers (int8 compute nodes) or -1
  std::vector<LayerSt> h_layers;
  LayerSt* d_layers = nullptr;
};

}  // namespace

struct ptq_ctx {
  int dev = 0;
  cudaStream_t st = nullptr;
  std::vector<void*> allocs;
  // graph
  std::vector<NodeI> nodes;
  std::vector<TensorI> tens;
  int T = 0, out_tensor = -1, n_classes = 0;
  std::vector<float*> d_wt;              // device copies of the weights (reference layout)
  std::vector<std::vector<int64_t>> wshape;
  std::vector<WeightsDev> W;             // per node (compute nodes only)
  int first_compute = -1, last_compute = -1;
  // space-to-depth stem: the graph input feeds only a stride-2 kxk conv on <= 4 channels with
  // odd padding (k-1)/2; its int8 codes are stored s2d (H/2 x W/2 pixels of 16 bytes) and
  // the conv runs as a stride-1 k'xk' conv, k' = (k+1)/2, halo (pad+1)/2
  int s2d_node = -1, s2d_k = 0, s2d_halo = 0;
  // data
  float* d_imgs = nullptr;
  long long* d_labels = nullptr;
  int64_t n_images = 0, n_calib = 0, n_eval = 0;
  // ranges and parameters
  std::vector<double> clip;              // [3 caches][2 clippings][T][2]
  std::vector<char> clip_set;            // [3][2]
  float* d_act_scale = nullptr;          // [24][T]
  int* d_act_zp = nullptr;
  uint64_t act_gen = 0;                  // bumped whenever the activation-parameter table is rewritten
  // the graph input's codes currently in d_codes[0]: (variant, act_gen, first image, images,
  // buffer) -- configs that share the input's quantization parameters reuse them
  struct CodesKey { int v = -1; uint64_t gen = 0; int64_t img0 = -1; int B = -1; const int8_t* buf = nullptr; };
  CodesKey inq;
  CodesKey pq;                           // the same for the folded FirstLastFp32 prefix codes
  bool prepared = false;
  bool static_ready = false;             // weight variants + eval buffers + mixed prefix enqueued
  bool wzp_pending = false;              // h_zp holds weight zero points not yet scanned
  int* h_zp = nullptr;                   // pinned [sum of 8*cout] weight zero points
  // eval buffers
  int64_t chunk = 0;
  // evaluation images upload in the background while calibration runs (ptq_create returns
  // once the calibration images are resident); ensure_upload() joins it before first use
  std::thread up_thread;
  cudaStream_t st_up = nullptr;
  cudaEvent_t ev_up = nullptr;
  std::string up_err;
  std::vector<int8_t*> d_codes;          // per tensor int8 view buffer (or null)
  // (variant, act_gen, zero-point source, first image, images) each halo was last filled with
  std::vector<std::array<int64_t, 5>> halo_key;
  std::vector<int> halo, cpad;
  std::vector<float*> d_f32;             // per tensor fp32 eval buffer (mixed tail)
  float* d_prefix = nullptr;             // mixed: fp32 output of the first compute node, all eval imgs
  // mixed + first compute -> relu -> maxpool: maxpool(relu(prefix)) in fp32, config-invariant;
  // quantization is monotone, so quantizing it equals max-pooling the relu'd codes
  int pool_fold = -1;                    // the folded maxpool node, or -1
  float* d_prefix_pool = nullptr;
  int* d_P = nullptr;                    // pixel sums scratch
  int8_t* d_im2col = nullptr;            // packed im2col scratch (few-channel convs)
  int64_t P_cap = 0;
  unsigned long long* d_correct = nullptr;
  Plan plans[2];
  // calibration state kept between ptq_calib_forward and ptq_calib_histogram
  std::vector<float*> cal_bufs;
  std::vector<int*> cal_slots;
  std::vector<int> cal_sizes;
  // options
  int conv_ref = 0, fusion = 1, time_conv = 0, ablate = 0, tma = 1, subsample = 1;
  int dwconv_variant = 3, concat_v16 = 1, kwr = 0;   // A/B switches (per context)
  int fx = 1;                            // exact fixed-point conv epilogue (0: fp64 epilogue)
  int tio = 1;                           // tile I/O through shared memory + TMA (flat conv layers)
  int rs_mma = 1;                        // A-row sums for weight zero points from the MMA (bn <= 128)
  int skip_pf = 1;                       // L2 prefetch of the fused-add operand tiles
  int hist_multi = 1;                    // batched histogram launch (0: one launch per histogram, A/B)
  int64_t opt_chunk = 0;
  // stats
  int64_t launches = 0;
  double conv_ms = 0.0, conv_ops = 0.0;
  int cur_cfg = 0;
  int64_t conv_launches_total = 0;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;

  template <typename T>
  // stream-ordered allocations from the device's default memory pool, which keeps freed
  // blocks (release threshold = max) so the 30 GB calibration activations and the eval
  // buffers are recycled across steps and across evaluator instances instead of being
  // mapped and unmapped each time
  T* dalloc(size_t n) {
    void* p = nullptr;
    if (n == 0) n = 1;
    CK(cudaMallocAsync(&p, n * sizeof(T), st));
    allocs.push_back(p);
    return static_cast<T*>(p);
  }
  void dfree(void* p) {
    if (!p) return;
    auto it = std::find(allocs.begin(), allocs.end(), p);
    if (it != allocs.end()) allocs.erase(it);
    cudaFreeAsync(p, st);
  }
};

namespace {

void check_launch(ptq_ctx* c) {
  ++c->launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Err{PTQ_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e)};
}

// A device fault (illegal address, trap, ...) leaves the CUDA context of the process unusable:
// every later call would fail with the same error or, worse, appear to work on garbage.  The
// first such fault poisons the library; from then on every entry point fails fast with
// PTQ_ECUDA and the original message, so each later trial is reported as failed (the
// reference's _safe_eval records it, tuner.py:173-177) instead of returning wrong accuracies.
// Recovery needs a new process (an in-process device reset would destroy every other context
// of the process, e.g. PyTorch's).
static std::atomic<int> g_poisoned{0};
static std::string g_poison_msg;
static bool sticky_cuda_error(cudaError_t e) {
  switch (e) {
    case cudaErrorIllegalAddress: case cudaErrorLaunchFailure: case cudaErrorHardwareStackError:
    case cudaErrorIllegalInstruction: case cudaErrorMisalignedAddress: case cudaErrorInvalidAddressSpace:
    case cudaErrorInvalidPc: case cudaErrorLaunchTimeout: case cudaErrorAssert: case cudaErrorECCUncorrectable:
      return true;
    default:
      return false;
  }
}
template <typename F>
int guarded(F&& f) {
  if (g_poisoned.load()) {
    g_err = "CUDA context unusable after an earlier device fault (" + g_poison_msg +
            "); start a new process";
    return PTQ_ECUDA;
  }
  try {
    f();
    return PTQ_OK;
  } catch (const Err& e) {
    g_err = e.msg;
    if (e.code == PTQ_ECUDA && sticky_cuda_error(cudaGetLastError())) {
      g_poison_msg = e.msg;
      g_poisoned.store(1);
    }
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PTQ_EINVAL;
  } catch (...) {
    g_err = "unknown error";
    return PTQ_EINVAL;
  }
}

// ---------------------------------------------------------------- graph import
void import_graph(ptq_ctx* c, const ptq_graph_desc* g) {
  Trace tr("import_graph");
  REQ(g && g->n_nodes > 0 && g->nodes, "empty graph");
  c->nodes.resize(g->n_nodes);
  c->tens.assign(g->n_nodes + 1, TensorI{});
  c->tens[0] = TensorI{g->in_c, g->in_h, g->in_w, (int64_t)g->in_c * g->in_h * g->in_w, -1, {}};
  c->n_classes = g->n_classes;
  for (int i = 0; i < g->n_nodes; ++i) {
    const ptq_node_desc& d = g->nodes[i];
    NodeI& n = c->nodes[i];
    n.kind = d.kind;
    REQ(d.n_inputs >= 1 && d.n_inputs <= PTQ_MAX_INPUTS, "bad input count");
    for (int j = 0; j < d.n_inputs; ++j) {
      REQ(d.inputs[j] >= 0 && d.inputs[j] <= i, "node input used before definition");
      n.in.push_back(d.inputs[j]);
    }
    n.out = i + 1;
    n.weight = d.weight;
    n.bias = d.bias;
    n.k = d.kernel;
    n.stride = d.stride < 1 ? 1 : d.stride;
    n.pad = d.pad;
    const TensorI& x = c->tens[n.in[0]];
    TensorI& y = c->tens[n.out];
    y.producer = i;
    switch (n.kind) {
      case PTQ_CONV: case PTQ_PWCONV: case PTQ_DWCONV: {
        REQ(n.weight >= 0 && n.weight < g->n_weights, "conv without weight");
        const ptq_weight_desc& w = g->weights[n.weight];
        REQ(w.ndim == 4 && w.shape[2] == w.shape[3], "conv weight must be (O,I,k,k)");
        n.k = (int)w.shape[2];
        if (n.kind == PTQ_DWCONV) REQ(w.shape[1] == 1 && w.shape[0] == x.c, "depthwise weight must be (C,1,k,k)");
        else REQ(w.shape[1] == x.c, "conv weight/input channel mismatch");
        y.c = (int)w.shape[0];
        y.h = (x.h + 2 * n.pad - n.k) / n.stride + 1;
        y.w = (x.w + 2 * n.pad - n.k) / n.stride + 1;
        REQ(y.h >= 1 && y.w >= 1, "conv does not fit input");
        break;
      }
      case PTQ_FC: {
        REQ(n.weight >= 0 && n.weight < g->n_weights, "fc without weight");
        const ptq_weight_desc& w = g->weights[n.weight];
        REQ(w.ndim == 2 && w.shape[1] == x.elems, "fc weight/input mismatch");
        y.c = (int)w.shape[0]; y.h = 1; y.w = 1;
        break;
      }
      case PTQ_MAXPOOL: case PTQ_AVGPOOL:
        REQ(n.k >= 1, "bad pool kernel");
        y.c = x.c;
        y.h = (x.h - n.k) / n.stride + 1;
        y.w = (x.w - n.k) / n.stride + 1;
        REQ(y.h >= 1 && y.w >= 1, "pool does not fit input");
        break;
      case PTQ_RELU: y.c = x.c; y.h = x.h; y.w = x.w; break;
      case PTQ_SOFTMAX:
        REQ(x.h == 1 && x.w == 1, "softmax supported on per-image vectors only");
        y.c = x.c; y.h = 1; y.w = 1;
        break;
      case PTQ_ADD:
        REQ(n.in.size() == 2, "add takes two inputs");
        REQ(c->tens[n.in[1]].c == x.c && c->tens[n.in[1]].h == x.h && c->tens[n.in[1]].w == x.w,
            "add shape mismatch");
        y.c = x.c; y.h = x.h; y.w = x.w;
        break;
      case PTQ_CONCAT: {
        int cs = 0;
        for (int t : n.in) {
          REQ(c->tens[t].h == x.h && c->tens[t].w == x.w, "concat spatial mismatch");
          cs += c->tens[t].c;
        }
        y.c = cs; y.h = x.h; y.w = x.w;
        break;
      }
      default: REQ(false, "unknown node kind");
    }
    y.elems = (int64_t)y.c * y.h * y.w;
    if (is_compute(n.kind)) {
      if (c->first_compute < 0) c->first_compute = i;
      c->last_compute = i;
    }
  }
  c->T = g->n_nodes + 1;
  for (int i = 0; i < g->n_nodes; ++i)
    for (int t : c->nodes[i].in) c->tens[t].consumers.push_back(i);
  int outs = 0;
  for (int t = 1; t < c->T; ++t)
    if (c->tens[t].consumers.empty()) { c->out_tensor = t; ++outs; }
  REQ(outs == 1, "graph must have exactly one output");
  REQ(c->first_compute >= 0, "graph has no weighted layers");
  const TensorI& o = c->tens[c->out_tensor];
  REQ(o.h == 1 && o.w == 1, "graph output must be a per-image score vector");

  // weights: device copies + the fp32 GEMM / depthwise forms
  c->d_wt.assign(g->n_weights, nullptr);
  c->wshape.assign(g->n_weights, {});
  for (int i = 0; i < g->n_weights; ++i) {
    const ptq_weight_desc& w = g->weights[i];
    int64_t n = 1;
    for (int d = 0; d < w.ndim; ++d) { n *= w.shape[d]; c->wshape[i].push_back(w.shape[d]); }
    c->d_wt[i] = c->dalloc<float>(n);
    CK(cudaMemcpyAsync(c->d_wt[i], w.data, n * sizeof(float), cudaMemcpyHostToDevice, c->st));
  }
  c->W.assign(g->n_nodes, WeightsDev{});
  for (int i = 0; i < g->n_nodes; ++i) {
    const NodeI& n = c->nodes[i];
    if (!is_compute(n.kind)) continue;
    WeightsDev& wd = c->W[i];
    const TensorI& x = c->tens[n.in[0]];
    const ptq_weight_desc& w = g->weights[n.weight];
    wd.cout = c->tens[n.out].c;
    if (n.bias >= 0) {
      REQ(g->weights[n.bias].ndim == 1 && g->weights[n.bias].shape[0] == wd.cout, "bias length mismatch");
      wd.f32_bias = c->d_wt[n.bias];
    }
    if (n.kind == PTQ_DWCONV) {
      wd.cin = x.c; wd.k = n.k;
      wd.f32_gemm = c->d_wt[n.weight];                  // (C,1,k,k) == [C][k*k]
      wd.bytes_per_variant = (int64_t)wd.cout * n.k * n.k;
    } else {
      // fp32 GEMM weight [K][cout], K in NHWC order (built on the device)
      const int kk = n.kind == PTQ_FC ? 1 : n.k;
      const int64_t K = n.kind == PTQ_FC ? x.elems : (int64_t)kk * kk * x.c;
      wd.f32_gemm = c->dalloc<float>((size_t)(K * wd.cout));
      launch_gemm_weight(c->d_wt[n.weight], wd.cout, x.c, kk, n.kind == PTQ_FC ? x.h * x.w : 0,
                         wd.f32_gemm, c->st);
      check_launch(c);
      // int8 tensor-core form
      wd.cin = x.c;
      wd.k = kk;
      wd.cin_p = rup(x.c, 16);
      wd.fc_hw = n.kind == PTQ_FC ? x.h * x.w : 0;
      wd.n_chunks = n.kind == PTQ_FC ? x.h * x.w * wd.cin_p / 16 : kk * kk * wd.cin_p / 16;
      wd.kreal = n.kind == PTQ_FC ? (int)x.elems : kk * kk * x.c;
      wd.q_cin_p = wd.cin_p;
      wd.q_k = kk;
      wd.q_fc_hw = wd.fc_hw;
      const bool s2d = n.kind == PTQ_CONV && n.in[0] == 0 && c->tens[0].consumers.size() == 1 &&
                       kk > 1 && x.c <= 4 && n.stride == 2 && n.pad == (kk - 1) / 2 && (n.pad & 1) &&
                       x.h % 2 == 0 && x.w % 2 == 0;
      if (s2d) {
        c->s2d_node = i;
        c->s2d_k = (kk + 1) / 2;
        c->s2d_halo = (n.pad + 1) / 2;
        wd.n_chunks = c->s2d_k * c->s2d_k;      // one 16-byte s2d pixel per tap
        wd.q_k = kk;
        wd.q_fc_hw = -c->s2d_k;
      } else if (n.kind != PTQ_FC && kk > 1 && x.c < 16) {
        // per-tap channel padding would inflate K (RGB stem: 49 x 16 vs 147 bytes): gather a
        // packed (kh, kw, c) im2col row per output pixel instead and run a 1x1 GEMM over it;
        // the weight quantizer sees it as an fc over k*k "pixels" of Cin unpadded channels
        wd.im2col = true;
        wd.im_cp = rup(kk * kk * x.c, 16);
        wd.n_chunks = wd.im_cp / 16;
        wd.q_cin_p = x.c;
        wd.q_k = 1;
        wd.q_fc_hw = kk * kk;
      }
      if (!s2d && !wd.im2col && n.kind == PTQ_CONV && kk == 1 && n.stride > 1 && n.pad == 0 &&
          x.c % 16 == 0 && wd.cin_p == x.c) {
        // same K layout as a pointwise conv (kb = ch), so the weight tiles need no change
        wd.sub1x1 = true;
        wd.im_cp = x.c;
      }
      wd.n_kiter = (wd.n_chunks + 7) / 8;
      REQ(wd.cout <= conv_tc_max_cout(), "conv / fc output channels exceed the tensor-core conv limit (2048)");
      wd.bn = conv_tc_bn_for(wd.cout);
      // a conv whose residual add is fused into its epilogue (its output only feeds the add, and
      // the add's other operand is produced earlier) keeps the 66 KB add table in shared memory;
      // with B streamed (Cout > 256) BN = 128 leaves room for the tile-I/O buffers.  Only for
      // K <= 512: deeper layers re-read A once per n-tile, which costs more than tile I/O saves
      // (ResNet-50: poin37 0.39 -> 0.33 ms, conv102 K=1024 0.14 -> 0.17 ms)
      const TensorI& ot = c->tens[n.out];
      bool fused_add = false;
      if (ot.consumers.size() == 1 && c->nodes[ot.consumers[0]].kind == PTQ_ADD) {
        const NodeI& an = c->nodes[ot.consumers[0]];
        const int other = an.in[0] == n.out ? an.in[1] : an.in[0];
        int prod = -1;
        for (int j = 0; j < g->n_nodes; ++j)
          if (c->nodes[j].out == other) prod = j;
        fused_add = prod < i;
      }
      if (wd.bn == 256 && wd.cout > 256 && wd.n_kiter <= 4 && fused_add) wd.bn = 128;
      // shallow (K <= 128) wide layers without a fused add whose width is a multiple of 128:
      // 128-wide tiles (3 accumulators in flight, group pairs) drain faster and the second A
      // pass is one stage per row (ResNet-50 poin7 0.300 -> 0.287, poin29 0.158 -> 0.148 ms,
      // MobileNet-v2 384-wide 0.060 -> 0.048).  A partial last 128-wide tile costs more than it
      // saves (MobileNet-v2 144 / 192 / 576-wide: 0.29 -> 0.49, 0.093 -> 0.131, 0.072 -> 0.085),
      // and with a fused add the 256-wide tile stays faster (poin8 0.461 vs 0.484)
      if (wd.bn == 256 && wd.n_kiter <= 1 && !fused_add && wd.cout % 128 == 0) wd.bn = 128;
      // narrow tiles of the variants with weight zero points (scheme 0 = Asymmetric, both
      // granularities) carry 16 K-indicator rows: the MMA also yields the A-row sums (N = bn + 16
      // <= 144; bn = 256 tiles fill TMEM and keep the row-sum warp).  The other variants keep
      // bn-row tiles (no extra B bytes or MMA columns)
      wd.brows_mask = wd.bn <= 128 ? 0x3 : 0;
      int ntiles = (wd.cout + wd.bn - 1) / wd.bn;
      for (int v = 0; v < 8; ++v) {
        wd.var_rows[v] = (wd.brows_mask >> v & 1) ? wd.bn + 16 : wd.bn;
        const int64_t vb = (int64_t)ntiles * wd.n_kiter * 8 * wd.var_rows[v] * 16;
        wd.var_off[v + 1] = wd.var_off[v] + vb;
        wd.bytes_per_variant = std::max(wd.bytes_per_variant, vb);
      }
    }
    if (n.kind == PTQ_DWCONV)
      for (int v = 0; v < 8; ++v) {
        wd.var_rows[v] = 0;
        wd.var_off[v + 1] = wd.var_off[v] + wd.bytes_per_variant;
      }
    wd.codes = c->dalloc<int8_t>(wd.var_off[8]);
    wd.scale = c->dalloc<float>(8 * wd.cout);
    wd.zp = c->dalloc<int>(8 * wd.cout);
    wd.wsum = c->dalloc<int>(8 * wd.cout);
    wd.mult = c->dalloc<double>(wd.cout);
    wd.biasq = c->dalloc<int>(wd.cout);
    wd.rt = c->dalloc<LayerRt>(1);
    // SoA block (kernels.h EpiParam) + the same again as k_layer_params' FX scratch
    wd.ep = c->dalloc<EpiParam>(2 * rup(wd.cout, 16));
  }
}

// ---------------------------------------------------------------- fp32 forward
// bufs[t] = [n][h][w][c] fp32; computes nodes [from, to]
void run_fp32(ptq_ctx* c, int n, std::vector<float*>& bufs, int from, int to) {
  for (int i = from; i <= to; ++i) {
    const NodeI& nd = c->nodes[i];
    const TensorI& x = c->tens[nd.in[0]];
    const TensorI& y = c->tens[nd.out];
    const float* xb = bufs[nd.in[0]];
    float* yb = bufs[nd.out];
    REQ(xb && yb, "fp32 buffer missing");
    switch (nd.kind) {
      case PTQ_CONV: case PTQ_PWCONV:
        launch_conv_f32(xb, n, x.h, x.w, x.c, c->W[i].f32_gemm, c->W[i].f32_bias, y.c, nd.k,
                        nd.stride, nd.pad, y.h, y.w, yb, c->st);
        break;
      case PTQ_FC:
        launch_conv_f32(xb, n, 1, 1, (int)x.elems, c->W[i].f32_gemm, c->W[i].f32_bias, y.c, 1, 1, 0,
                        1, 1, yb, c->st);
        break;
      case PTQ_DWCONV:
        launch_dwconv_f32(xb, n, x.h, x.w, x.c, c->W[i].f32_gemm, c->W[i].f32_bias, nd.k, nd.stride,
                          nd.pad, y.h, y.w, yb, c->st);
        break;
      case PTQ_RELU: launch_relu_f32(xb, yb, (int64_t)n * y.elems, c->st); break;
      case PTQ_MAXPOOL: case PTQ_AVGPOOL:
        launch_pool_f32(xb, n, x.h, x.w, x.c, nd.k, nd.stride, y.h, y.w,
                        nd.kind == PTQ_AVGPOOL, yb, c->st);
        break;
      case PTQ_ADD: launch_add_f32(xb, bufs[nd.in[1]], yb, (int64_t)n * y.elems, c->st); break;
      case PTQ_CONCAT: {
        int coff = 0;
        for (int t : nd.in) {
          launch_concat_f32(bufs[t], (int64_t)n * y.h * y.w, c->tens[t].c, y.c, coff, yb, c->st);
          coff += c->tens[t].c;
        }
        break;
      }
      case PTQ_SOFTMAX: launch_softmax_f32(xb, n, y.c, yb, c->st); break;
    }
    check_launch(c);
  }
}

// ---------------------------------------------------------------- plans (quantize_model rules)
int narrowed(ptq_ctx* c, int node) {
  const TensorI& t = c->tens[c->nodes[node].out];
  if (t.consumers.size() == 1 && c->nodes[t.consumers[0]].kind == PTQ_RELU)
    return c->nodes[t.consumers[0]].out;
  return c->nodes[node].out;
}

void build_plan(ptq_ctx* c, int mixed) {
  Plan& P = c->plans[mixed];
  if (P.built) return;
  const int N = (int)c->nodes.size();
  P.mixed = mixed;
  P.psrc.assign(c->T, -1);
  P.fp32node.assign(N, 0);
  P.skip.assign(N, 0);
  P.mat.assign(N, -1);
  P.relu_hist.assign(N, -1);
  P.add_node.assign(N, -1);
  P.add_other.assign(N, -1);
  P.add_is_a.assign(N, 0);
  P.add_relu_hist.assign(N, -1);
  P.layer_of.assign(N, -1);
  if (mixed) {
    P.fp32node[c->first_compute] = 1;
    P.fp32node[c->last_compute] = 1;
    P.prefix_end = c->first_compute;
  }
  P.psrc[0] = mixed ? -1 : 0;
  for (int i = 0; i < N; ++i) {
    const NodeI& n = c->nodes[i];
    bool all = true, any = false;
    for (int t : n.in) { bool q = P.psrc[t] >= 0; all &= q; any |= q; }
    if (is_compute(n.kind)) {
      if (P.fp32node[i]) {
        P.psrc[n.out] = (i == c->last_compute) ? -1 : narrowed(c, i);
        continue;
      }
      REQ(all, "quantized layer fed by fp32 tensor");
      P.psrc[n.out] = narrowed(c, i);
    } else if (n.kind == PTQ_ADD || n.kind == PTQ_CONCAT) {
      if (all) P.psrc[n.out] = n.kind == PTQ_ADD ? narrowed(c, i) : n.out;
      else REQ(!any, "mixed int8/fp32 operands");
    } else {
      P.psrc[n.out] = P.psrc[n.in[0]];
    }
  }
  if (mixed) {
    for (int i = 0; i < c->first_compute; ++i)
      for (int t : c->nodes[i].in) REQ(P.psrc[t] < 0, "unsupported mixed prefix");
  }
  // fusion of relu / add(+relu) into int8 compute epilogues (and relu into the mixed prefix quantize)
  std::vector<char> materialized(c->T, 0);
  materialized[0] = 1;
  for (int i = 0; i < N; ++i) {
    const NodeI& n = c->nodes[i];
    if (P.skip[i]) continue;
    if (!is_compute(n.kind)) {
      materialized[n.out] = 1;
      continue;
    }
    P.mat[i] = n.out;
    struct MarkMat {
      std::vector<char>& m;
      Plan& P;
      int i;
      ~MarkMat() { m[P.mat[i]] = 1; }
    } mark{materialized, P, i};
    const bool int8_out = P.psrc[n.out] >= 0;
    if (!int8_out || !c->fusion) continue;
    if (P.fp32node[i] && i != c->first_compute) continue;
    const TensorI& t = c->tens[n.out];
    if (t.consumers.size() != 1) continue;
    const int cn = t.consumers[0];
    const NodeI& cons = c->nodes[cn];
    if (cons.kind == PTQ_RELU && P.psrc[cons.out] >= 0) {
      P.relu_hist[i] = P.psrc[cons.out];
      P.skip[cn] = 1;
      P.mat[i] = cons.out;
    } else if (cons.kind == PTQ_ADD && P.psrc[cons.out] >= 0 && (n.kind == PTQ_CONV || n.kind == PTQ_PWCONV) &&
               !P.fp32node[i]) {
      const int other = cons.in[0] == n.out ? cons.in[1] : cons.in[0];
      if (other == n.out) continue;
      // the other operand must already be materialised when this conv runs
      if (!materialized[other]) continue;
      P.add_node[i] = cn;
      P.add_other[i] = other;
      P.add_is_a[i] = cons.in[0] == n.out;
      P.skip[cn] = 1;
      P.mat[i] = cons.out;
      const TensorI& at = c->tens[cons.out];
      if (at.consumers.size() == 1 && c->nodes[at.consumers[0]].kind == PTQ_RELU &&
          P.psrc[c->nodes[at.consumers[0]].out] >= 0) {
        P.add_relu_hist[i] = P.psrc[c->nodes[at.consumers[0]].out];
        P.skip[at.consumers[0]] = 1;
        P.mat[i] = c->nodes[at.consumers[0]].out;
      }
    }
  }
  // per-layer static descriptors for the int8 compute nodes
  P.h_layers.clear();
  for (int i = 0; i < N; ++i) {
    const NodeI& n = c->nodes[i];
    if (!is_compute(n.kind) || P.fp32node[i]) continue;
    WeightsDev& wd = c->W[i];
    LayerSt L{};
    L.cout = wd.cout;
    L.in_hist = P.psrc[n.in[0]];
    L.out_hist = P.psrc[n.out];
    L.relu_hist = P.relu_hist[i];
    L.add_a_hist = L.add_b_hist = L.add_o_hist = -1;
    if (P.add_node[i] >= 0) {
      const NodeI& an = c->nodes[P.add_node[i]];
      L.add_a_hist = P.psrc[an.in[0]];
      L.add_b_hist = P.psrc[an.in[1]];
      L.add_o_hist = P.psrc[an.out];
    }
    L.add_relu_hist = P.add_relu_hist[i];
    L.bias = wd.f32_bias;
    L.wscale = wd.scale;
    L.mult = wd.mult;
    L.biasq = wd.biasq;
    L.rt = wd.rt;
    L.wzp8 = wd.zp;
    L.wsum8 = wd.wsum;
    L.kreal = wd.kreal;
    L.ep = wd.ep;
    L.dw = n.kind == PTQ_DWCONV;
    L.addtab = nullptr;
    L.add_conv_is_a = P.add_is_a[i];
    if (P.add_node[i] >= 0 && L.ep && !L.dw) {
      if (!wd.addtab) wd.addtab = c->dalloc<int8_t>(PTQ_ADDTAB_BYTES);
      L.addtab = wd.addtab;
    }
    P.layer_of[i] = (int)P.h_layers.size();
    P.h_layers.push_back(L);
  }
  if (!P.h_layers.empty()) {
    P.d_layers = c->dalloc<LayerSt>(P.h_layers.size());
    CK(cudaMemcpyAsync(P.d_layers, P.h_layers.data(), P.h_layers.size() * sizeof(LayerSt),
                       cudaMemcpyHostToDevice, c->st));
  }
  P.built = true;
}

// ---------------------------------------------------------------- eval buffers
View view_of(ptq_ctx* c, int t, int n) {
  const TensorI& x = c->tens[t];
  if (t == 0 && c->s2d_node >= 0) return View{c->d_codes[0], n, x.h / 2, x.w / 2, 4 * x.c, 16, c->s2d_halo};
  return View{c->d_codes[t], n, x.h, x.w, x.c, c->cpad[t], c->halo[t]};
}

void ensure_eval_buffers(ptq_ctx* c) {
  Trace tr("ensure_eval_buffers");
  int64_t chunk = c->opt_chunk > 0 ? std::min<int64_t>(c->opt_chunk, c->n_eval) : c->n_eval;
  if (c->chunk == chunk && !c->d_codes.empty()) return;
  for (auto p : c->d_codes) c->dfree(p);
  for (auto p : c->d_f32) c->dfree(p);
  c->dfree(c->d_P);
  c->d_P = nullptr;
  c->chunk = chunk;
  const int T = c->T;
  c->halo.assign(T, 0);
  c->cpad.assign(T, 16);
  for (int t = 0; t < T; ++t) {
    c->cpad[t] = rup(c->tens[t].c, 16);
    for (int ci : c->tens[t].consumers) {
      const NodeI& n = c->nodes[ci];
      if (n.kind == PTQ_CONV || n.kind == PTQ_DWCONV || n.kind == PTQ_PWCONV)
        c->halo[t] = std::max(c->halo[t], n.pad);
    }
  }
  if (c->s2d_node >= 0) {
    c->halo[0] = c->s2d_halo;
    c->cpad[0] = 16;
  }
  // fc inputs are read as one flattened pixel: they must not carry a halo
  for (const NodeI& n : c->nodes)
    if (n.kind == PTQ_FC) REQ(c->halo[n.in[0]] == 0, "fc input also feeds a padded conv");
  c->d_codes.assign(T, nullptr);
  c->halo_key.clear();
  c->d_f32.assign(T, nullptr);
  std::set<int> need8, need32;
  for (int m = 0; m < 2; ++m) {
    build_plan(c, m);
    const Plan& P = c->plans[m];
    need8.insert(0);
    for (int i = 0; i < (int)c->nodes.size(); ++i) {
      const NodeI& n = c->nodes[i];
      if (P.skip[i]) continue;
      if (is_compute(n.kind)) {
        if (P.psrc[P.mat[i]] >= 0) need8.insert(P.mat[i]);
        else need32.insert(n.out);
        if (P.fp32node[i] && i == c->last_compute) need32.insert(n.in[0]);
      } else if (P.psrc[n.out] >= 0) {
        need8.insert(n.out);
      } else if (!(m == 1 && i < c->first_compute)) {
        need32.insert(n.out);
        for (int t : n.in) need32.insert(t);
      }
    }
  }
  int64_t maxP = 0;
  for (int t : need8) {
    const TensorI& x = c->tens[t];
    const int h = (t == 0 && c->s2d_node >= 0) ? x.h / 2 : x.h, w = (t == 0 && c->s2d_node >= 0) ? x.w / 2 : x.w;
    int64_t bytes = chunk * (int64_t)(h + 2 * c->halo[t]) * (w + 2 * c->halo[t]) * c->cpad[t];
    // the stem's slab copies (k_conv_tc A mode 67) of the last tile read up to one tile plus
    // k-1 padded rows past the grid
    const int64_t slack = (t == 0 && c->s2d_node >= 0)
                              ? ((int64_t)c->s2d_k * (w + 2 * c->halo[t]) + 2 * 128) * c->cpad[t] : 0;
    c->d_codes[t] = c->dalloc<int8_t>(bytes + slack);
    CK(cudaMemsetAsync(c->d_codes[t], 0, bytes, c->st));
    maxP = std::max<int64_t>(maxP, chunk * (int64_t)(h + 2 * c->halo[t]) * (w + 2 * c->halo[t]));
  }
  if (c->s2d_node >= 0) {                        // per-output-pixel window sums of the stem
    const TensorI& y = c->tens[c->nodes[c->s2d_node].out];
    maxP = std::max<int64_t>(maxP, chunk * (int64_t)y.h * y.w);
  }
  for (int t : need32) c->d_f32[t] = c->dalloc<float>(chunk * c->tens[t].elems);
  int64_t im_bytes = 0;
  for (int i = 0; i < (int)c->nodes.size(); ++i)
    if (c->W[i].im2col || c->W[i].sub1x1)
      im_bytes = std::max<int64_t>(im_bytes, chunk * (int64_t)c->tens[c->nodes[i].out].h *
                                                 c->tens[c->nodes[i].out].w * c->W[i].im_cp);
  c->dfree(c->d_im2col);
  c->d_im2col = im_bytes ? c->dalloc<int8_t>(im_bytes) : nullptr;
  for (int i = 0; i < (int)c->nodes.size(); ++i)
    if (c->W[i].im2col || c->W[i].sub1x1)
      maxP = std::max<int64_t>(maxP, chunk * (int64_t)c->tens[c->nodes[i].out].h * c->tens[c->nodes[i].out].w);
  c->d_P = c->dalloc<int>(maxP);
  c->P_cap = maxP;
}

// ---------------------------------------------------------------- prepare
void prepare_static(ptq_ctx* c);

void prepare(ptq_ctx* c) {
  if (c->prepared) return;
  Trace tr("prepare");
  for (int i = 0; i < 6; ++i) REQ(c->clip_set[i], "clip ranges not set for every (cache, clipping)");
  const int T = c->T;
  // activation params: variant v = (cache*4 + scheme)*2 + clip
  std::vector<double> r((size_t)24 * T * 2);
  std::vector<int> vs(24);
  for (int cache = 0; cache < 3; ++cache)
    for (int sch = 0; sch < 4; ++sch)
      for (int cl = 0; cl < 2; ++cl) {
        int v = (cache * 4 + sch) * 2 + cl;
        vs[v] = sch;
        std::memcpy(&r[(size_t)v * T * 2], &c->clip[((size_t)(cache * 2 + cl)) * T * 2], sizeof(double) * T * 2);
      }
  double* d_r = c->dalloc<double>(r.size());
  int* d_vs = c->dalloc<int>(24);
  CK(cudaMemcpyAsync(d_r, r.data(), r.size() * sizeof(double), cudaMemcpyHostToDevice, c->st));
  CK(cudaMemcpyAsync(d_vs, vs.data(), 24 * sizeof(int), cudaMemcpyHostToDevice, c->st));
  if (!c->d_act_scale) {
    c->d_act_scale = c->dalloc<float>((size_t)24 * T);
    c->d_act_zp = c->dalloc<int>((size_t)24 * T);
  }
  launch_act_params(d_r, d_vs, 24, T, c->d_act_scale, c->d_act_zp, c->st);
  ++c->act_gen;
  check_launch(c);
  prepare_static(c);
  CK(cudaStreamSynchronize(c->st));
  if (c->wzp_pending) {
    size_t off = 0;
    for (auto& wd : c->W) {
      if (!wd.cout) continue;
      for (int v = 0; v < 8; ++v) {
        wd.has_wzp[v] = false;
        for (int o = 0; o < wd.cout; ++o) wd.has_wzp[v] |= c->h_zp[off + (size_t)v * wd.cout + o] != 0;
      }
      off += (size_t)8 * wd.cout;
    }
    c->wzp_pending = false;
  }
  c->dfree(d_r);
  c->dfree(d_vs);
  c->prepared = true;
}

// clip-range independent part of prepare(): weight variants, eval buffers, the mixed
// prefix.  Only enqueued (no sync), so ptq_kl_sweep can start it while the host picks the
// KL windows.
void prepare_static(ptq_ctx* c) {
  if (c->static_ready) return;
  // weights: 8 variants (scheme, granularity) per compute node
  Trace trw("prepare.weights");
  unsigned int* d_mm = nullptr;
  int maxc = 1;
  for (auto& wd : c->W) maxc = std::max(maxc, wd.cout);
  d_mm = c->dalloc<unsigned int>(2 * (size_t)maxc + 2);
  for (int i = 0; i < (int)c->nodes.size(); ++i) {
    const NodeI& n = c->nodes[i];
    if (!is_compute(n.kind)) continue;
    WeightsDev& wd = c->W[i];
    const float* w = c->d_wt[n.weight];
    int64_t per_ch = 1;
    for (size_t d = 1; d < c->wshape[n.weight].size(); ++d) per_ch *= c->wshape[n.weight][d];
    launch_weight_prepare8(w, wd.cout, per_ch, n.kind == PTQ_DWCONV, wd.cin, n.kind == PTQ_DWCONV ? wd.k : wd.q_k,
                           wd.q_fc_hw, wd.q_cin_p, wd.bn, wd.brows_mask, wd.n_kiter, wd.bytes_per_variant, d_mm, wd.scale,
                           wd.zp, wd.codes, wd.wsum, c->st);
    check_launch(c);
  }
  // weight zero points to the host asynchronously (scanned for has_wzp in prepare())
  size_t nzp = 0;
  for (auto& wd : c->W) nzp += (size_t)8 * wd.cout;
  if (!c->h_zp) CK(cudaMallocHost(&c->h_zp, std::max<size_t>(nzp, 1) * sizeof(int)));
  size_t off = 0;
  for (auto& wd : c->W) {
    if (!wd.cout) continue;
    CK(cudaMemcpyAsync(c->h_zp + off, wd.zp, (size_t)8 * wd.cout * sizeof(int), cudaMemcpyDeviceToHost, c->st));
    off += (size_t)8 * wd.cout;
  }
  c->wzp_pending = true;
  c->dfree(d_mm);
  ensure_eval_buffers(c);
  // mixed prefix: config-invariant fp32 output of the first compute node for all eval images
  {
    Trace trp("prepare.mixed_prefix");
    const int fc_ = c->first_compute;
    const int tout = c->nodes[fc_].out;
    if (!c->d_prefix) c->d_prefix = c->dalloc<float>((size_t)c->n_eval * c->tens[tout].elems);
    std::vector<float*> bufs(c->T, nullptr);
    int64_t pc = std::min<int64_t>(c->n_eval, 256);
    std::vector<int> need;
    for (int i = 0; i <= fc_; ++i) {
      need.push_back(c->nodes[i].out);
      for (int t : c->nodes[i].in) need.push_back(t);
    }
    std::sort(need.begin(), need.end());
    need.erase(std::unique(need.begin(), need.end()), need.end());
    for (int t : need)
      if (t != tout) bufs[t] = c->dalloc<float>(pc * c->tens[t].elems);
    const TensorI& in = c->tens[0];
    for (int64_t s = 0; s < c->n_eval; s += pc) {
      int nn = (int)std::min<int64_t>(pc, c->n_eval - s);
      launch_nchw_to_nhwc(c->d_imgs + (c->n_calib + s) * in.elems, nullptr, nn, in.c, in.h, in.w,
                          bufs[0], c->st);
      check_launch(c);
      bufs[tout] = c->d_prefix + s * c->tens[tout].elems;
      run_fp32(c, nn, bufs, 0, fc_);
    }
    for (int t : need)
      if (t != tout) c->dfree(bufs[t]);
    // fold relu + maxpool into the prefix (see pool_fold)
    c->pool_fold = -1;
    const TensorI& t1 = c->tens[tout];
    if (t1.consumers.size() == 1 && c->nodes[t1.consumers[0]].kind == PTQ_RELU) {
      const NodeI& r = c->nodes[t1.consumers[0]];
      const TensorI& t2 = c->tens[r.out];
      if (t2.consumers.size() == 1 && c->nodes[t2.consumers[0]].kind == PTQ_MAXPOOL) {
        const int pi = t2.consumers[0];
        const NodeI& pn = c->nodes[pi];
        const TensorI& tp = c->tens[pn.out];
        if (!c->d_prefix_pool) c->d_prefix_pool = c->dalloc<float>((size_t)c->n_eval * tp.elems);
        for (int64_t s0 = 0; s0 < c->n_eval; s0 += pc) {
          const int nn = (int)std::min<int64_t>(pc, c->n_eval - s0);
          launch_pool_f32(c->d_prefix + s0 * t1.elems, nn, t1.h, t1.w, t1.c, pn.k, pn.stride, tp.h, tp.w, 0,
                          c->d_prefix_pool + s0 * tp.elems, c->st);
          check_launch(c);
        }
        // relu after the max (both monotone: relu(max x) == max relu(x)); d_prefix stays
        // intact for probes of the unfolded tensors
        launch_relu_f32(c->d_prefix_pool, c->d_prefix_pool, (int64_t)c->n_eval * tp.elems, c->st);
        check_launch(c);
        c->pool_fold = pi;
      }
    }
  }
  c->static_ready = true;
}

// ---------------------------------------------------------------- one config
// Parity probes (tests only; the timed path passes pr == nullptr).  Images `imgs` (eval-set
// indices) of one evaluation are copied to the host in the reference's NCHW layouts:
//   codes   int8 codes of each tensor in `tensors` ([n_imgs][C][H][W] at code_out[k]); found[k]
//           = 1 when the tensor was materialised (fused-away tensors stay 0)
//   acc     the clipped int32 accumulator of compute node acc_node ([n_imgs][Cout][OH][OW])
//   logits  what run_quantized returns (intexec.py:337-351): dequantized output codes, or the
//           fp32 output when the last layer runs in fp32 ([n_imgs][classes])
//   f32     an fp32-domain tensor (FirstLastFp32 layers) ([n_imgs][C][H][W])
struct ProbeReq {
  std::vector<int64_t> imgs;
  std::vector<int> tensors;
  std::vector<int8_t*> code_out;
  std::vector<int> found;
  int acc_node = -1;
  int32_t* acc_out = nullptr;
  bool acc_found = false;
  float* logit_out = nullptr;
  int f32_tensor = -1;
  float* f32_out = nullptr;
  bool f32_found = false;
};

// host copy of the selected images of a [B][h][w][c] device array (element size E) into
// out[j] = image imgs[j] in NCHW order; sel = (output slot j, local image index)
template <typename T>
void copy_nchw(ptq_ctx* c, const T* dev, int64_t img_stride, int h, int w, int ch, int64_t pitch_px,
               int halo, int cp, const std::vector<std::pair<int, int>>& sel, T* out) {
  const int Hp = h + 2 * halo, Wp = w + 2 * halo;
  std::vector<T> tmp((size_t)Hp * Wp * cp);
  for (auto [j, n] : sel) {
    CK(cudaMemcpyAsync(tmp.data(), dev + (int64_t)n * img_stride, tmp.size() * sizeof(T), cudaMemcpyDeviceToHost,
                       c->st));
    CK(cudaStreamSynchronize(c->st));
    T* o = out + (size_t)j * ch * h * w;
    for (int k = 0; k < ch; ++k)
      for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x)
          o[((size_t)k * h + y) * w + x] = tmp[((size_t)(y + halo) * Wp + x + halo) * cp + k];
    (void)pitch_px;
  }
}

// ---------------------------------------------------------------- one config
void eval_one(ptq_ctx* c, const ptq_config& cfg, unsigned long long* d_correct, ProbeReq* pr) {
  REQ(cfg.cache >= 0 && cfg.cache < 3 && cfg.scheme >= 0 && cfg.scheme < 4 && cfg.clipping >= 0 &&
          cfg.clipping < 2 && cfg.granularity >= 0 && cfg.granularity < 2 && cfg.mixed >= 0 &&
          cfg.mixed < 2,
      "config field out of range");
  Plan& P = c->plans[cfg.mixed];
  const int v = (cfg.cache * 4 + cfg.scheme) * 2 + cfg.clipping;
  const int wv = cfg.scheme * 2 + cfg.granularity;
  const float* as = c->d_act_scale + (size_t)v * c->T;
  const int* az = c->d_act_zp + (size_t)v * c->T;
  launch_layer_params(P.d_layers, (int)P.h_layers.size(), as, az, wv, c->fx, c->st);
  check_launch(c);
  const int N = (int)c->nodes.size();
  std::vector<int> alias(c->T);
  for (int t = 0; t < c->T; ++t) alias[t] = t;

  for (int64_t img0 = 0; img0 < c->n_eval; img0 += c->chunk) {
    const int B = (int)std::min<int64_t>(c->chunk, c->n_eval - img0);
    auto V = [&](int t) { return view_of(c, alias[t], B); };
    std::vector<std::pair<int, int>> sel;          // (probe slot, local image) in this chunk
    if (pr)
      for (int j = 0; j < (int)pr->imgs.size(); ++j)
        if (pr->imgs[j] >= img0 && pr->imgs[j] < img0 + B) sel.push_back({j, (int)(pr->imgs[j] - img0)});
    auto probe = [&](int t) {
      if (!pr || sel.empty()) return;
      int k = -1;
      for (int q = 0; q < (int)pr->tensors.size(); ++q)
        if (pr->tensors[q] == t) k = q;
      if (k < 0) return;
      pr->found[k] = 1;
      View pv = V(t);
      const TensorI& x = c->tens[t];
      int8_t* out = pr->code_out[k];
      if (t == 0 && c->s2d_node >= 0) {                // space-to-depth input view
        const int Wq = pv.W + 2 * pv.halo, Hq = pv.H + 2 * pv.halo;
        std::vector<int8_t> h2((size_t)Hq * Wq * pv.Cp);
        for (auto [j, n] : sel) {
          CK(cudaMemcpyAsync(h2.data(), pv.p + (size_t)n * h2.size(), h2.size(), cudaMemcpyDeviceToHost, c->st));
          CK(cudaStreamSynchronize(c->st));
          int8_t* o = out + (size_t)j * x.elems;
          for (int ch = 0; ch < x.c; ++ch)
            for (int y = 0; y < x.h; ++y)
              for (int xx = 0; xx < x.w; ++xx)
                o[((size_t)ch * x.h + y) * x.w + xx] =
                    h2[((size_t)(y / 2 + pv.halo) * Wq + xx / 2 + pv.halo) * pv.Cp + ((y & 1) * 2 + (xx & 1)) * x.c + ch];
        }
        return;
      }
      const int64_t per_img = (int64_t)(x.h + 2 * pv.halo) * (x.w + 2 * pv.halo) * pv.Cp;
      copy_nchw<int8_t>(c, pv.p, per_img, x.h, x.w, x.c, 0, pv.halo, pv.Cp, sel, out);
    };
    // every int8 tensor buffer is dedicated and no producer writes its halo, so all halos of
    // this config are filled up front in one launch -- and only those whose zero point (or
    // image range) changed since they were last filled
    {
      HaloBatch hb{};
      if (c->halo_key.size() != (size_t)c->T) c->halo_key.assign(c->T, std::array<int64_t, 5>{-1, -1, -1, -1, -1});
      for (int t = 0; t < c->T && hb.n < 48; ++t) {
        if (!c->d_codes[t] || P.psrc[t] < 0) continue;
        const View vv = V(t);
        if (vv.halo <= 0 || vv.p == nullptr) continue;
        const std::array<int64_t, 5> key = {(int64_t)v, (int64_t)c->act_gen, (int64_t)P.psrc[t], img0, (int64_t)B};
        if (c->halo_key[t] == key) continue;
        c->halo_key[t] = key;
        hb.v[hb.n] = vv;
        hb.hist[hb.n] = P.psrc[t];
        ++hb.n;
      }
      if (hb.n) {
        launch_halo_fill_multi(hb, az, c->st);
        check_launch(c);
      }
    }
    auto halo_fill = [&](int t) { (void)t; };
    // graph input / mixed prefix
    int start = 0;
    if (!cfg.mixed) {
      // the input codes depend only on the activation-parameter variant (its input entry):
      // consecutive Mixed=Off configs of one (cache, scheme, clipping) quantize it once
      const bool reuse = c->inq.v == v && c->inq.gen == c->act_gen && c->inq.img0 == img0 && c->inq.B == B &&
                         c->inq.buf == c->d_codes[0] && P.psrc[0] == 0;
      if (!reuse) {
        if (c->s2d_node >= 0)
          launch_quant_input_s2d(c->d_imgs, c->n_calib + img0, c->tens[0].c, V(0), as, az, P.psrc[0], c->st);
        else
          launch_quant_input(c->d_imgs, c->n_calib + img0, V(0), as, az, P.psrc[0], c->st);
        check_launch(c);
        halo_fill(0);
        c->inq.v = v; c->inq.gen = c->act_gen; c->inq.img0 = img0; c->inq.B = B; c->inq.buf = c->d_codes[0];
      }
      c->pq.v = -1;                                // this plan writes the prefix's pooled codes
      probe(0);
    } else {
      const int fc_ = c->first_compute;
      const int mt = P.mat[fc_];
      const int pf = c->pool_fold;
      if (pf >= 0 && P.psrc[c->nodes[pf].out] == P.psrc[c->nodes[fc_].out] && !pr) {
        // quantize maxpool(relu(prefix)) straight into the maxpool's output codes
        const int tp = c->nodes[pf].out;
        const View vt = V(tp);
        if (!(c->pq.v == v && c->pq.gen == c->act_gen && c->pq.img0 == img0 && c->pq.B == B && c->pq.buf == vt.p)) {
          launch_quant_nhwc(c->d_prefix_pool + img0 * c->tens[tp].elems, vt, as, az,
                            P.psrc[c->nodes[fc_].out], -1, c->st);
          check_launch(c);
          halo_fill(tp);
          c->pq.v = v; c->pq.gen = c->act_gen; c->pq.img0 = img0; c->pq.B = B; c->pq.buf = vt.p;
        }
        probe(tp);
        start = pf + 1;
      } else {
        c->pq.v = -1;
        launch_quant_nhwc(c->d_prefix + img0 * c->tens[c->nodes[fc_].out].elems, V(mt), as, az,
                          P.psrc[c->nodes[fc_].out], P.relu_hist[fc_], c->st);
        check_launch(c);
        halo_fill(mt);
        probe(mt);
        start = fc_ + 1;
      }
    }
    for (int i = start; i < N; ++i) {
      if (P.skip[i]) continue;
      const NodeI& n = c->nodes[i];
      const int tin = n.in[0];
      if (is_compute(n.kind) && !P.fp32node[i]) {
        WeightsDev& wd = c->W[i];
        const int tout = P.mat[i];
        const LayerSt& L = P.h_layers[P.layer_of[i]];
        const TensorI& yo = c->tens[n.out];
        const bool acc_probe = pr && pr->acc_node == i && !sel.empty();
        int* d_acc = acc_probe ? c->dalloc<int>((size_t)B * yo.elems) : nullptr;
        if (n.kind == PTQ_DWCONV) {
          // the dp4a kernel takes the weight zero points only when this variant has any
          const bool dp4 = c->dwconv_variant == 3;
          launch_dwconv_i8(V(tin), V(tout), wd.codes + wd.var_off[wv],
                           (dp4 && !wd.has_wzp[wv]) ? nullptr : wd.zp + (size_t)wv * wd.cout, n.k, n.stride,
                           n.pad, L, c->st, d_acc, c->dwconv_variant);
          check_launch(c);
        } else {
          ConvTcArgs a{};
          View vin = V(tin);
          const TensorI& x = c->tens[tin];
          if (n.kind == PTQ_FC) {
            vin.H = 1; vin.W = 1; vin.C = x.h * x.w * vin.Cp; vin.Cp = vin.C; vin.halo = 0;
            a.k = 1; a.stride = 1; a.pad = 0; a.OH = 1; a.OW = 1;
          } else if (wd.im2col || (wd.sub1x1 && c->subsample)) {
            const TensorI& y = c->tens[n.out];
            launch_im2col(vin, n.k, n.stride, n.pad, y.h, y.w, c->d_im2col, wd.im_cp, c->st);
            check_launch(c);
            vin = View{c->d_im2col, B, y.h, y.w, wd.kreal, wd.im_cp, 0};
            a.k = 1; a.stride = 1; a.pad = 0; a.OH = y.h; a.OW = y.w;
          } else if (i == c->s2d_node) {            // stride-1 k'xk' conv over the s2d input
            a.k = c->s2d_k; a.stride = 1; a.pad = c->s2d_halo;
            a.OH = c->tens[n.out].h; a.OW = c->tens[n.out].w;
          } else {
            a.k = n.k; a.stride = n.stride; a.pad = n.pad;
            a.OH = c->tens[n.out].h; a.OW = c->tens[n.out].w;
          }
          a.in = vin;
          a.out = V(tout);
          a.wB = wd.codes + wd.var_off[wv];
          a.b_rows = wd.var_rows[wv];
          a.n_kiter = wd.n_kiter;
          a.n_chunks = wd.n_chunks;
          a.wzp = wd.zp + (size_t)wv * wd.cout;
          a.wsum = wd.wsum + (size_t)wv * wd.cout;
          a.kreal = wd.kreal;
          a.has_wzp = wd.has_wzp[wv];
          a.rs_mma = a.has_wzp && c->rs_mma && a.b_rows > wd.bn && !c->conv_ref;
          if (a.has_wzp && !a.rs_mma && i == c->s2d_node) {
            REQ((int64_t)B * a.OH * a.OW <= c->P_cap, "stem rowsum buffer too small");
            launch_stem_rowsum(vin, n.k, c->tens[0].c, a.OH, a.OW, c->d_P, c->st);
            check_launch(c);
            a.Rpix = c->d_P;
          }
          a.L = L;
          a.skip = View{nullptr, 0, 0, 0, 0, 0, 0};
          if (P.add_node[i] >= 0) {
            a.skip = V(P.add_other[i]);
            a.conv_is_a = P.add_is_a[i];
          }
          a.addtab = L.addtab;
          a.ablate = c->ablate;
          a.allow_tma = c->tma;
          a.kwr_mode = c->kwr;
          a.tio_mode = c->tio;
          a.skip_pf = c->skip_pf;
          if (a.has_wzp && !a.rs_mma && !a.Rpix && (c->conv_ref || !conv_tc_tma_rowsum(a, wd.bn))) {
            launch_pixsum(vin, c->d_P, c->st);       // gather-mode convs sum input pixels first
            check_launch(c);
            a.P = c->d_P;
          }
          cudaEvent_t ea = nullptr, eb = nullptr;
          const bool timed = c->cur_cfg < c->time_conv;   // instrument only the leading configs
          ++c->conv_launches_total;
          if (timed) {
            while (c->ev_pool.size() < c->ev_used + 2) {
              cudaEvent_t e;
              CK(cudaEventCreate(&e));
              c->ev_pool.push_back(e);
            }
            ea = c->ev_pool[c->ev_used++];
            eb = c->ev_pool[c->ev_used++];
            CK(cudaEventRecord(ea, c->st));
          }
          if (c->conv_ref) launch_conv_i8_ref(a, wd.bn, c->st);
          else launch_conv_tc(a, wd.bn, c->st);
          check_launch(c);
          if (d_acc) {                               // probe: the same tcgen05 launch, acc epilogue
            REQ(!c->conv_ref, "accumulator probes need the tensor-core conv");
            ConvTcArgs b = a;
            b.acc_out = d_acc;
            launch_conv_tc(b, wd.bn, c->st);
            check_launch(c);
          }
          if (timed) {
            CK(cudaEventRecord(eb, c->st));
            c->conv_ops += 2.0 * (double)B * a.OH * a.OW * (double)wd.cout * (double)wd.kreal;
          }
        }
        if (d_acc) {
          copy_nchw<int>(c, d_acc, yo.elems, yo.h, yo.w, yo.c, 0, 0, yo.c, sel, pr->acc_out);
          pr->acc_found = true;
          c->dfree(d_acc);
        }
        halo_fill(tout);
        probe(tout);
        continue;
      }
      if (is_compute(n.kind)) {                      // fp32 last layer (mixed)
        const int tout = n.out;
        float* xin = c->d_f32[tin];
        if (P.psrc[tin] >= 0) {
          launch_dequant(V(tin), as, az, P.psrc[tin], xin, c->st);
          check_launch(c);
        }
        std::vector<float*> bufs(c->T, nullptr);
        bufs[tin] = xin;
        bufs[tout] = c->d_f32[tout];
        run_fp32(c, B, bufs, i, i);
        if (P.psrc[tout] >= 0) {
          launch_quant_nhwc(c->d_f32[tout], V(tout), as, az, P.psrc[tout], -1, c->st);
          check_launch(c);
          halo_fill(tout);
        }
        continue;
      }
      const int tout = n.out;
      if (P.psrc[tout] < 0) {                        // fp32-domain tail
        std::vector<float*> bufs(c->T, nullptr);
        for (int t : n.in) bufs[t] = c->d_f32[t];
        bufs[tout] = c->d_f32[tout];
        run_fp32(c, B, bufs, i, i);
        continue;
      }
      switch (n.kind) {
        case PTQ_RELU: launch_relu_codes(V(tin), V(tout), az, P.psrc[tout], c->st); break;
        case PTQ_MAXPOOL: case PTQ_AVGPOOL:
          launch_pool_codes(V(tin), V(tout), n.k, n.stride, n.kind == PTQ_AVGPOOL, az, P.psrc[tout], c->st);
          break;
        case PTQ_ADD:
          launch_add_codes(V(n.in[0]), V(n.in[1]), V(tout), as, az, P.psrc[n.in[0]], P.psrc[n.in[1]],
                           P.psrc[tout], c->st);
          break;
        case PTQ_CONCAT: {
          int coff = 0;
          for (int t : n.in) {
            launch_concat_codes(V(t), V(tout), coff, as, az, P.psrc[t], P.psrc[tout], c->st, c->concat_v16);
            check_launch(c);
            coff += c->tens[t].c;
          }
          break;
        }
        case PTQ_SOFTMAX:                            // monotone: identity on codes (intexec.py:290-292)
          alias[tout] = alias[tin];
          probe(tout);
          continue;
      }
      check_launch(c);
      halo_fill(tout);
      probe(tout);
    }
    const int ot = c->out_tensor;
    if (P.psrc[ot] >= 0) launch_argmax_codes(V(ot), c->d_labels + img0, d_correct, c->st);
    else launch_argmax_f32(c->d_f32[ot], B, c->tens[ot].c, c->d_labels + img0, d_correct, c->st);
    check_launch(c);
    if (pr && !sel.empty() && pr->logit_out) {       // run_quantized's return value
      const TensorI& o = c->tens[ot];
      if (P.psrc[ot] >= 0) {                         // dequantize_array of the output codes (F3)
        float* d_y = c->dalloc<float>((size_t)B * o.elems);
        launch_dequant(V(ot), as, az, P.psrc[ot], d_y, c->st);
        check_launch(c);
        copy_nchw<float>(c, d_y, o.elems, 1, 1, o.c, 0, 0, o.c, sel, pr->logit_out);
        c->dfree(d_y);
      } else {
        copy_nchw<float>(c, c->d_f32[ot], o.elems, 1, 1, o.c, 0, 0, o.c, sel, pr->logit_out);
      }
    }
    if (pr && !sel.empty() && pr->f32_tensor >= 0) { // an fp32-domain tensor of this config
      const int t = pr->f32_tensor;
      const TensorI& x = c->tens[t];
      const float* src = nullptr;
      int64_t stride = x.elems;
      if (cfg.mixed && t == c->nodes[c->first_compute].out) src = c->d_prefix + img0 * x.elems;
      else if (P.psrc[t] < 0 && c->d_f32[t]) src = c->d_f32[t];
      REQ(src, "tensor is not an fp32-domain tensor of this config");
      copy_nchw<float>(c, src, stride, x.h, x.w, x.c, 0, 0, x.c, sel, pr->f32_out);
      pr->f32_found = true;
    }
  }
}

}  // namespace

// ================================================================ C ABI
extern "C" {

const char* ptq_last_error(void) { return g_err.c_str(); }
// the background upload of the evaluation images has landed (and the host buffer is no
// longer read); the context stream waits for it
static void ensure_upload(ptq_ctx* c) {
  if (c->up_thread.joinable()) {
    c->up_thread.join();
    if (!c->up_err.empty()) throw Err{PTQ_ECUDA, "evaluation image upload: " + c->up_err};
    CK(cudaStreamWaitEvent(c->st, c->ev_up, 0));
  }
}

int ptq_version(void) { return 1; }

int ptq_create(ptq_ctx** out, int device, const ptq_graph_desc* g, const float* images,
               const int64_t* eval_labels, int64_t n_images, int64_t n_calib) {
  ptq_ctx* c = new ptq_ctx();
  int rc = guarded([&] {
    REQ(out && g && images, "null argument");
    REQ(n_calib >= 0 && n_calib <= n_images, "bad calibration split");
    c->dev = device;
    CK(cudaSetDevice(device));
    int major = 0, minor = 0;
    CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    CK(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
    REQ(major == 10 && minor == 0, "ptq_b200 requires an sm_100 (B200) device");
    CK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
    {
      cudaMemPool_t pool;
      CK(cudaDeviceGetDefaultMemPool(&pool, device));
      uint64_t thr = UINT64_MAX;
      CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    }
    import_graph(c, g);
    c->n_images = n_images;
    c->n_calib = n_calib;
    c->n_eval = n_images - n_calib;
    const TensorI& in = c->tens[0];
    c->d_imgs = c->dalloc<float>((size_t)n_images * in.elems);
    // calibration pool now; the evaluation images (3.4x the bytes at 300/1000) stream in a
    // background thread on their own stream while the calibration forward runs
    CK(cudaMemcpyAsync(c->d_imgs, images, (size_t)n_calib * in.elems * sizeof(float),
                       cudaMemcpyHostToDevice, c->st));
    if (n_images > n_calib) {
      CK(cudaStreamSynchronize(c->st));          // d_imgs allocated (stream-ordered) before the copy
      CK(cudaStreamCreateWithFlags(&c->st_up, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&c->ev_up, cudaEventDisableTiming));
      float* dst = c->d_imgs + (size_t)n_calib * in.elems;
      const float* src = images + (size_t)n_calib * in.elems;
      const size_t bytes = (size_t)(n_images - n_calib) * in.elems * sizeof(float);
      c->up_thread = std::thread([c, dst, src, bytes] {
        cudaError_t e = cudaSetDevice(c->dev);
        if (e == cudaSuccess) e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->st_up);
        if (e == cudaSuccess) e = cudaEventRecord(c->ev_up, c->st_up);
        if (e == cudaSuccess) e = cudaStreamSynchronize(c->st_up);
        if (e != cudaSuccess) c->up_err = cudaGetErrorString(e);
      });
    }
    c->d_labels = c->dalloc<long long>(std::max<int64_t>(c->n_eval, 1));
    if (c->n_eval > 0 && eval_labels)
      CK(cudaMemcpyAsync(c->d_labels, eval_labels, c->n_eval * sizeof(long long),
                         cudaMemcpyHostToDevice, c->st));
    c->d_correct = c->dalloc<unsigned long long>(4096);
    c->clip.assign((size_t)6 * c->T * 2, 0.0);
    c->clip_set.assign(6, 0);
    CK(cudaStreamSynchronize(c->st));
    *out = c;
  });
  if (rc != PTQ_OK) {
    if (c->up_thread.joinable()) c->up_thread.join();
    for (void* p : c->allocs) cudaFreeAsync(p, c->st);
    if (c->st) cudaStreamSynchronize(c->st);
    if (c->st) cudaStreamDestroy(c->st);
    delete c;
  }
  return rc;
}

int ptq_destroy(ptq_ctx* c) {
  if (!c) return PTQ_OK;
  if (c->up_thread.joinable()) c->up_thread.join();
  cudaSetDevice(c->dev);
  if (c->st) cudaStreamSynchronize(c->st);
  for (void* p : c->allocs) cudaFreeAsync(p, c->st);
  if (c->st) cudaStreamSynchronize(c->st);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  if (c->h_zp) cudaFreeHost(c->h_zp);
  if (c->st) cudaStreamDestroy(c->st);
  if (c->st_up) cudaStreamDestroy(c->st_up);
  if (c->ev_up) cudaEventDestroy(c->ev_up);
  delete c;
  return PTQ_OK;
}

int ptq_num_tensors(const ptq_ctx* c, int32_t* T) {
  if (!c || !T) { g_err = "null argument"; return PTQ_EINVAL; }
  *T = c->T;
  return PTQ_OK;
}

int ptq_calib_forward(ptq_ctx* c, int32_t n_caches, const int32_t* sizes, const int64_t* ids,
                      float* local_ranges) {
  return guarded([&] {
    Trace tr("calib_forward");
    REQ(c && n_caches >= 1 && sizes, "null argument");
    CK(cudaSetDevice(c->dev));
    c->static_ready = false;                     // a new calibration rebuilds the evaluator state
    for (auto p : c->cal_bufs) c->dfree(p);
    for (auto p : c->cal_slots) c->dfree(p);
    c->cal_bufs.clear();
    c->cal_slots.clear();
    c->cal_sizes.assign(sizes, sizes + n_caches);
    int64_t tot = 0;
    for (int k = 0; k < n_caches; ++k) {
      REQ(sizes[k] >= 0, "negative cache size");
      tot += sizes[k];
    }
    REQ(tot == 0 || ids, "null ids");
    std::vector<int64_t> uni(ids, ids + tot);
    for (int64_t v : uni) REQ(v >= 0 && v < c->n_calib, "calibration id out of range");
    std::sort(uni.begin(), uni.end());
    uni.erase(std::unique(uni.begin(), uni.end()), uni.end());
    const int nu = (int)uni.size();
    std::map<int64_t, int> slot;
    for (int i = 0; i < nu; ++i) slot[uni[i]] = i;
    const int T = c->T;
    float* d_rng = c->dalloc<float>((size_t)n_caches * T * 2);
    unsigned int* d_mm = c->dalloc<unsigned int>((size_t)T * std::max(nu, 1) * 2);
    if (nu > 0) {
      // fp32 forward over the union of the caches' images (one batch)
      c->cal_bufs.assign(T, nullptr);
      for (int t = 0; t < T; ++t) c->cal_bufs[t] = c->dalloc<float>((size_t)nu * c->tens[t].elems);
      std::vector<int> uid(uni.begin(), uni.end());
      int* d_uid = c->dalloc<int>(nu);
      CK(cudaMemcpyAsync(d_uid, uid.data(), nu * sizeof(int), cudaMemcpyHostToDevice, c->st));
      const TensorI& in = c->tens[0];
      launch_nchw_to_nhwc(c->d_imgs, d_uid, nu, in.c, in.h, in.w, c->cal_bufs[0], c->st);
      check_launch(c);
      run_fp32(c, nu, c->cal_bufs, 0, (int)c->nodes.size() - 1);
      // F1a: exact per-image min/max of every tensor
      launch_fill_minmax(d_mm, (int64_t)T * nu, c->st);
      check_launch(c);
      for (int t = 0; t < T; ++t) {
        launch_minmax_per_image(c->cal_bufs[t], c->tens[t].elems, nu, d_mm + (size_t)t * nu * 2, c->st);
        check_launch(c);
      }
      CK(cudaStreamSynchronize(c->st));
      c->dfree(d_uid);
    }
    int64_t off = 0;
    for (int k = 0; k < n_caches; ++k) {
      std::vector<int> sl(sizes[k]);
      for (int j = 0; j < sizes[k]; ++j) sl[j] = slot[ids[off + j]];
      off += sizes[k];
      int* ds = c->dalloc<int>(std::max<size_t>(sl.size(), 1));
      c->cal_slots.push_back(ds);
      if (!sl.empty())
        CK(cudaMemcpyAsync(ds, sl.data(), sl.size() * sizeof(int), cudaMemcpyHostToDevice, c->st));
      launch_minmax_reduce_cache(d_mm, T, std::max(nu, 1), ds, sizes[k], d_rng + (size_t)k * T * 2, c->st);
      check_launch(c);
    }
    if (local_ranges)
      CK(cudaMemcpyAsync(local_ranges, d_rng, (size_t)n_caches * T * 2 * sizeof(float),
                         cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    c->dfree(d_mm);
    c->dfree(d_rng);
  });
}

int ptq_calib_histogram(ptq_ctx* c, const float* ranges, int64_t* counts) {
  return guarded([&] {
    Trace tr("calib_histogram");
    REQ(c && ranges && counts, "null argument");
    REQ(c->cal_sizes.size() == c->cal_slots.size(), "ptq_calib_forward must run first");
    CK(cudaSetDevice(c->dev));
    const int T = c->T, nk = (int)c->cal_sizes.size();
    float* d_rng = c->dalloc<float>((size_t)nk * T * 2);
    unsigned long long* d_cnt = c->dalloc<unsigned long long>((size_t)nk * T * PTQ_NBINS);
    CK(cudaMemcpyAsync(d_rng, ranges, (size_t)nk * T * 2 * sizeof(float), cudaMemcpyHostToDevice, c->st));
    CK(cudaMemsetAsync(d_cnt, 0, (size_t)nk * T * PTQ_NBINS * 8, c->st));
    // F1b: every histogram (cache k, tensor t) with the cache's global (lo, hi), one batched launch
    std::vector<HistItem> items;
    for (int k = 0; k < nk; ++k) {
      if (c->cal_sizes[k] == 0) continue;
      for (int t = 0; t < T; ++t)
        items.push_back(HistItem{c->cal_bufs[t], c->tens[t].elems, c->cal_slots[k], c->cal_sizes[k],
                                 d_rng + ((size_t)k * T + t) * 2, d_cnt + ((size_t)k * T + t) * PTQ_NBINS, 0});
    }
    const int64_t n_chunks = hist_items_chunk0(items.data(), (int)items.size());
    HistItem* d_items = c->dalloc<HistItem>(items.size() ? items.size() : 1);
    if (c->hist_multi) {
      CK(cudaMemcpyAsync(d_items, items.data(), items.size() * sizeof(HistItem), cudaMemcpyHostToDevice, c->st));
      launch_histogram_multi(d_items, (int)items.size(), n_chunks, c->st);
      check_launch(c);
    } else {
      for (const HistItem& it : items) {
        launch_histogram(it.x, it.elems, it.slots, it.n_slots, it.range, it.counts, c->st);
        check_launch(c);
      }
    }
    CK(cudaMemcpyAsync(counts, d_cnt, (size_t)nk * T * PTQ_NBINS * 8, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    for (auto p : c->cal_bufs) c->dfree(p);
    for (auto p : c->cal_slots) c->dfree(p);
    c->cal_bufs.clear();
    c->cal_slots.clear();
    c->cal_sizes.clear();
    c->dfree(d_rng);
    c->dfree(d_cnt);
    c->dfree(d_items);
  });
}

int ptq_calibrate(ptq_ctx* c, int32_t n_caches, const int32_t* sizes, const int64_t* ids,
                  float* ranges, int64_t* counts, int64_t* n_samples) {
  if (!c || n_caches < 1 || !sizes) { g_err = "null argument"; return PTQ_EINVAL; }
  std::vector<float> r((size_t)n_caches * c->T * 2);
  std::vector<int64_t> cnt((size_t)n_caches * c->T * PTQ_NBINS);
  int rc = ptq_calib_forward(c, n_caches, sizes, ids, r.data());
  if (rc != PTQ_OK) return rc;
  rc = ptq_calib_histogram(c, r.data(), cnt.data());
  if (rc != PTQ_OK) return rc;
  if (ranges) std::memcpy(ranges, r.data(), r.size() * sizeof(float));
  if (counts) std::memcpy(counts, cnt.data(), cnt.size() * sizeof(int64_t));
  if (n_samples)
    for (int k = 0; k < n_caches; ++k)
      for (int t = 0; t < c->T; ++t) n_samples[(size_t)k * c->T + t] = (int64_t)sizes[k] * c->tens[t].elems;
  return PTQ_OK;
}

int ptq_kl_sweep(ptq_ctx* c, int32_t n_hist, const int64_t* counts, const float* ranges, double* kl) {
  return guarded([&] {
    Trace tr("kl_sweep");
    REQ(c && counts && ranges && kl && n_hist >= 0, "null argument");
    if (n_hist == 0) return;
    CK(cudaSetDevice(c->dev));
    long long* d_c = c->dalloc<long long>((size_t)n_hist * PTQ_NBINS);
    float* d_r = c->dalloc<float>((size_t)n_hist * 2);
    double* d_cum = c->dalloc<double>((size_t)n_hist * PTQ_NBINS);
    int* d_nz = c->dalloc<int>((size_t)n_hist * PTQ_NBINS);
    double* d_log = c->dalloc<double>((size_t)n_hist * PTQ_NBINS);
    double* d_kl = c->dalloc<double>((size_t)n_hist * PTQ_NWINDOWS);
    CK(cudaMemcpyAsync(d_c, counts, (size_t)n_hist * PTQ_NBINS * 8, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(d_r, ranges, (size_t)n_hist * 2 * sizeof(float), cudaMemcpyHostToDevice, c->st));
    launch_kl_sweep(d_c, d_r, n_hist, d_cum, d_nz, d_log, d_kl, c->st);
    check_launch(c);
    CK(cudaMemcpyAsync(kl, d_kl, (size_t)n_hist * PTQ_NWINDOWS * 8, cudaMemcpyDeviceToHost, c->st));
    cudaEvent_t done;
    CK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    CK(cudaEventRecord(done, c->st));
    for (void* p : {(void*)d_c, (void*)d_r, (void*)d_cum, (void*)d_nz, (void*)d_log, (void*)d_kl}) c->dfree(p);
    // the clip-range independent preparation runs on the GPU while the caller picks windows
    if (!c->static_ready && c->W.size()) prepare_static(c);
    CK(cudaEventSynchronize(done));
    CK(cudaEventDestroy(done));
  });
}

int ptq_percentile_ranges(ptq_ctx* c, int32_t n_hist, const int64_t* counts, const float* ranges, double pct,
                          double* out) {
  return guarded([&] {
    REQ(c && counts && ranges && out && n_hist >= 0, "null argument");
    REQ(pct > 0.0 && pct <= 100.0, "percentile must be in (0, 100]");
    if (n_hist == 0) return;
    CK(cudaSetDevice(c->dev));
    long long* d_c = c->dalloc<long long>((size_t)n_hist * PTQ_NBINS);
    float* d_r = c->dalloc<float>((size_t)n_hist * 2);
    double* d_o = c->dalloc<double>((size_t)n_hist * 2);
    CK(cudaMemcpyAsync(d_c, counts, (size_t)n_hist * PTQ_NBINS * 8, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(d_r, ranges, (size_t)n_hist * 2 * sizeof(float), cudaMemcpyHostToDevice, c->st));
    launch_percentile(d_c, d_r, n_hist, pct / 100.0, d_o, c->st);
    check_launch(c);
    CK(cudaMemcpyAsync(out, d_o, (size_t)n_hist * 2 * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    for (void* p : {(void*)d_c, (void*)d_r, (void*)d_o}) c->dfree(p);
  });
}

int ptq_set_clip_ranges(ptq_ctx* c, int32_t cache, int32_t clipping, const double* ranges) {
  return guarded([&] {
    REQ(c && ranges && cache >= 0 && cache < 3 && clipping >= 0 && clipping < 2, "bad argument");
    std::memcpy(&c->clip[((size_t)(cache * 2 + clipping)) * c->T * 2], ranges, sizeof(double) * c->T * 2);
    c->clip_set[cache * 2 + clipping] = 1;
    c->prepared = false;
  });
}

int ptq_prepare(ptq_ctx* c) {
  return guarded([&] {
    if (c) ensure_upload(c);
    REQ(c, "null context");
    CK(cudaSetDevice(c->dev));
    prepare(c);
  });
}

int ptq_eval_configs(ptq_ctx* c, const ptq_config* cfgs, int32_t n_cfg, int64_t* correct) {
  return guarded([&] {
    if (c) ensure_upload(c);
    Trace tr("eval_configs");
    REQ(c && cfgs && correct && n_cfg >= 0, "null argument");
    CK(cudaSetDevice(c->dev));
    prepare(c);
    ensure_eval_buffers(c);
    c->conv_ops = 0.0;
    c->conv_ms = 0.0;
    c->ev_used = 0;
    c->conv_launches_total = 0;
    for (int32_t b0 = 0; b0 < n_cfg; b0 += 4096) {
      const int nb = std::min<int32_t>(4096, n_cfg - b0);
      CK(cudaMemsetAsync(c->d_correct, 0, nb * sizeof(unsigned long long), c->st));
      // evaluation order: grouped by (mixed, cache, scheme, clipping) so configs that share
      // the quantized graph input / prefix reuse it (results land in the caller's order)
      std::vector<int> order(nb);
      for (int i = 0; i < nb; ++i) order[i] = i;
      auto key = [&](int i) {
        const ptq_config& f = cfgs[b0 + i];
        return ((f.mixed * 3 + f.cache) * 4 + f.scheme) * 2 + f.clipping;
      };
      std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return key(x) < key(y); });
      for (int i : order) {
        c->cur_cfg = b0 + i;
        eval_one(c, cfgs[b0 + i], c->d_correct + i, nullptr);
      }
      c->cur_cfg = 0;
      std::vector<unsigned long long> h(nb);
      CK(cudaMemcpyAsync(h.data(), c->d_correct, nb * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->st));
      CK(cudaStreamSynchronize(c->st));
      for (int i = 0; i < nb; ++i) correct[b0 + i] = (int64_t)h[i];
    }
    for (size_t e = 0; e + 1 < c->ev_used; e += 2) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, c->ev_pool[e], c->ev_pool[e + 1]));
      c->conv_ms += ms;
    }
  });
}

int ptq_probe_codes(ptq_ctx* c, const ptq_config* cfg, int32_t tensor, int8_t* out, int64_t* n_out) {
  return guarded([&] {
    if (c) ensure_upload(c);
    REQ(c && cfg && tensor >= 0 && tensor < c->T, "bad argument");
    const int64_t n = c->n_eval * c->tens[tensor].elems;
    if (n_out) *n_out = n;
    if (!out) return;
    CK(cudaSetDevice(c->dev));
    prepare(c);
    ensure_eval_buffers(c);
    REQ(c->plans[cfg->mixed].psrc[tensor] >= 0, "tensor is in the fp32 domain for this config");
    REQ(c->d_codes[tensor], "tensor is fused away (set option fusion=0 to probe it)");
    ProbeReq pr;
    for (int64_t i = 0; i < c->n_eval; ++i) pr.imgs.push_back(i);
    pr.tensors = {tensor};
    pr.code_out = {out};
    pr.found = {0};
    CK(cudaMemsetAsync(c->d_correct, 0, 8, c->st));
    eval_one(c, *cfg, c->d_correct, &pr);
    CK(cudaStreamSynchronize(c->st));
    REQ(pr.found[0], "tensor is fused away (set option fusion=0 to probe it)");
  });
}

static void probe_images(ptq_ctx* c, ProbeReq& pr, int32_t n_imgs, const int64_t* imgs) {
  REQ(n_imgs > 0 && imgs, "no probe images");
  for (int i = 0; i < n_imgs; ++i) {
    REQ(imgs[i] >= 0 && imgs[i] < c->n_eval, "probe image out of range");
    pr.imgs.push_back(imgs[i]);
  }
}

int ptq_probe_tensors(ptq_ctx* c, const ptq_config* cfg, int32_t n_tensors, const int32_t* tensors,
                      int32_t n_imgs, const int64_t* imgs, int8_t* out, int32_t* found) {
  return guarded([&] {
    if (c) ensure_upload(c);
    REQ(c && cfg && tensors && out && found && n_tensors > 0, "null argument");
    CK(cudaSetDevice(c->dev));
    prepare(c);
    ensure_eval_buffers(c);
    ProbeReq pr;
    probe_images(c, pr, n_imgs, imgs);
    int64_t off = 0;
    for (int k = 0; k < n_tensors; ++k) {
      REQ(tensors[k] >= 0 && tensors[k] < c->T, "bad tensor id");
      pr.tensors.push_back(tensors[k]);
      pr.code_out.push_back(out + off);
      pr.found.push_back(0);
      off += (int64_t)n_imgs * c->tens[tensors[k]].elems;
    }
    CK(cudaMemsetAsync(c->d_correct, 0, 8, c->st));
    eval_one(c, *cfg, c->d_correct, &pr);
    CK(cudaStreamSynchronize(c->st));
    for (int k = 0; k < n_tensors; ++k) found[k] = pr.found[k];
  });
}

int ptq_probe_acc(ptq_ctx* c, const ptq_config* cfg, int32_t node, int32_t n_imgs, const int64_t* imgs,
                  int32_t* out) {
  return guarded([&] {
    if (c) ensure_upload(c);
    REQ(c && cfg && out, "null argument");
    REQ(node >= 0 && node < (int)c->nodes.size() && is_compute(c->nodes[node].kind), "not a compute node");
    CK(cudaSetDevice(c->dev));
    prepare(c);
    ensure_eval_buffers(c);
    REQ(!c->plans[cfg->mixed].fp32node[node], "node runs in fp32 under this config");
    ProbeReq pr;
    probe_images(c, pr, n_imgs, imgs);
    pr.acc_node = node;
    pr.acc_out = out;
    CK(cudaMemsetAsync(c->d_correct, 0, 8, c->st));
    eval_one(c, *cfg, c->d_correct, &pr);
    CK(cudaStreamSynchronize(c->st));
    REQ(pr.acc_found, "accumulator probe did not run");
  });
}

int ptq_probe_output(ptq_ctx* c, const ptq_config* cfg, int32_t n_imgs, const int64_t* imgs, float* out) {
  return guarded([&] {
    if (c) ensure_upload(c);
    REQ(c && cfg && out, "null argument");
    CK(cudaSetDevice(c->dev));
    prepare(c);
    ensure_eval_buffers(c);
    ProbeReq pr;
    probe_images(c, pr, n_imgs, imgs);
    pr.logit_out = out;
    CK(cudaMemsetAsync(c->d_correct, 0, 8, c->st));
    eval_one(c, *cfg, c->d_correct, &pr);
    CK(cudaStreamSynchronize(c->st));
  });
}

int ptq_probe_f32(ptq_ctx* c, const ptq_config* cfg, int32_t tensor, int32_t n_imgs, const int64_t* imgs,
                  float* out) {
  return guarded([&] {
    if (c) ensure_upload(c);
    REQ(c && cfg && out && tensor >= 0 && tensor < c->T, "bad argument");
    CK(cudaSetDevice(c->dev));
    prepare(c);
    ensure_eval_buffers(c);
    ProbeReq pr;
    probe_images(c, pr, n_imgs, imgs);
    pr.f32_tensor = tensor;
    pr.f32_out = out;
    CK(cudaMemsetAsync(c->d_correct, 0, 8, c->st));
    eval_one(c, *cfg, c->d_correct, &pr);
    CK(cudaStreamSynchronize(c->st));
    REQ(pr.f32_found, "tensor is not an fp32-domain tensor of this config");
  });
}

int ptq_minmax_host(ptq_ctx* c, const float* x, int32_t n_img, int64_t elems, float* range) {
  return guarded([&] {
    REQ(c && x && range && n_img > 0 && elems > 0, "bad argument");
    CK(cudaSetDevice(c->dev));
    float* d_x = c->dalloc<float>((size_t)n_img * elems);
    unsigned int* d_mm = c->dalloc<unsigned int>((size_t)n_img * 2);
    int* d_s = c->dalloc<int>(n_img);
    float* d_r = c->dalloc<float>(2);
    std::vector<int> sl(n_img);
    for (int i = 0; i < n_img; ++i) sl[i] = i;
    CK(cudaMemcpyAsync(d_x, x, (size_t)n_img * elems * sizeof(float), cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(d_s, sl.data(), n_img * sizeof(int), cudaMemcpyHostToDevice, c->st));
    launch_fill_minmax(d_mm, n_img, c->st);
    check_launch(c);
    launch_minmax_per_image(d_x, elems, n_img, d_mm, c->st);   // F1a, as in ptq_calib_forward
    check_launch(c);
    launch_minmax_reduce_cache(d_mm, 1, n_img, d_s, n_img, d_r, c->st);
    check_launch(c);
    CK(cudaMemcpyAsync(range, d_r, 2 * sizeof(float), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    for (void* p : {(void*)d_x, (void*)d_mm, (void*)d_s, (void*)d_r}) c->dfree(p);
  });
}

int ptq_probe_act_params(ptq_ctx* c, int32_t cache, int32_t scheme, int32_t clipping, float* scale,
                         int32_t* zp) {
  return guarded([&] {
    REQ(c && scale && zp, "null argument");
    CK(cudaSetDevice(c->dev));
    prepare(c);
    const int v = (cache * 4 + scheme) * 2 + clipping;
    CK(cudaMemcpy(scale, c->d_act_scale + (size_t)v * c->T, c->T * sizeof(float), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(zp, c->d_act_zp + (size_t)v * c->T, c->T * sizeof(int), cudaMemcpyDeviceToHost));
  });
}

int ptq_export_layer(ptq_ctx* c, const ptq_config* cfg, int32_t node, int8_t* codes, float* wscale,
                     int32_t* wzp, int32_t* bias) {
  return guarded([&] {
    if (c) ensure_upload(c);
    REQ(c && cfg && codes && wscale && wzp, "null argument");
    REQ(node >= 0 && node < (int)c->nodes.size() && is_compute(c->nodes[node].kind), "not a compute node");
    CK(cudaSetDevice(c->dev));
    prepare(c);
    Plan& P = c->plans[cfg->mixed];
    REQ(!P.fp32node[node], "node runs in fp32 under this config");
    const NodeI& n = c->nodes[node];
    WeightsDev& wd = c->W[node];
    const int wv = cfg->scheme * 2 + cfg->granularity;
    const int v = (cfg->cache * 4 + cfg->scheme) * 2 + cfg->clipping;
    // per-config layer constants (bias codes) exactly as an evaluation computes them
    launch_layer_params(P.d_layers, (int)P.h_layers.size(), c->d_act_scale + (size_t)v * c->T,
                        c->d_act_zp + (size_t)v * c->T, wv, c->fx, c->st);
    check_launch(c);
    CK(cudaMemcpyAsync(wscale, wd.scale + (size_t)wv * wd.cout, wd.cout * sizeof(float), cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(wzp, wd.zp + (size_t)wv * wd.cout, wd.cout * sizeof(int), cudaMemcpyDeviceToHost, c->st));
    if (bias && wd.f32_bias)
      CK(cudaMemcpyAsync(bias, wd.biasq, wd.cout * sizeof(int), cudaMemcpyDeviceToHost, c->st));
    std::vector<int8_t> tiled((size_t)(wd.var_off[wv + 1] - wd.var_off[wv]));
    CK(cudaMemcpyAsync(tiled.data(), wd.codes + wd.var_off[wv], tiled.size(),
                       cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    if (n.kind == PTQ_DWCONV) {                      // [C][k*k], stored as is
      std::memcpy(codes, tiled.data(), (size_t)wd.cout * wd.k * wd.k);
      return;
    }
    // inverse of the B-tile layout [nt][ki][8][BN][16] (see wsrc in k_quant.cu)
    const int k = n.kind == PTQ_FC ? 1 : n.k, cin = wd.cin;
    const int64_t per_o = n.kind == PTQ_FC ? (int64_t)cin * wd.q_fc_hw : (int64_t)cin * k * k;
    for (int o = 0; o < wd.cout; ++o)
      for (int64_t e = 0; e < per_o; ++e) {
        int64_t kb;
        if (n.kind == PTQ_FC) {                      // e = ch*hw + pix  ->  kb = pix*cin_p + ch
          const int64_t ch = e / wd.q_fc_hw, pix = e - ch * wd.q_fc_hw;
          kb = pix * wd.q_cin_p + ch;
        } else {
          const int ch = (int)(e / (k * k)), t = (int)(e % (k * k)), kh = t / k, kw = t % k;
          if (wd.q_fc_hw < 0) {                      // s2d stem: tap (kh', kw'), sub-pixel (a, b)
            const int k2 = -wd.q_fc_hw, a = (kh + 1) & 1, b = (kw + 1) & 1;
            kb = (((kh + 1) >> 1) * k2 + ((kw + 1) >> 1)) * 16 + (2 * a + b) * cin + ch;
          } else if (wd.im2col) {                    // packed (kh, kw, c) row
            kb = (int64_t)(kh * k + kw) * cin + ch;
          } else {
            kb = (int64_t)(kh * k + kw) * wd.cin_p + ch;
          }
        }
        const int nt = o / wd.bn, row = o % wd.bn;
        const int64_t it = kb >> 7, j = (kb >> 4) & 7, b = kb & 15;
        codes[(int64_t)o * per_o + e] = tiled[(size_t)((((int64_t)nt * wd.n_kiter + it) * 8 + j) * wd.var_rows[wv] + row) * 16 + b];
      }
  });
}

int ptq_histogram_host(ptq_ctx* c, const float* x, int64_t n, float lo, float hi, int64_t* counts) {
  return guarded([&] {
    REQ(c && x && counts && n > 0, "bad argument");
    CK(cudaSetDevice(c->dev));
    float* d_x = c->dalloc<float>(n);
    float* d_r = c->dalloc<float>(2);
    int* d_s = c->dalloc<int>(1);
    unsigned long long* d_c = c->dalloc<unsigned long long>(PTQ_NBINS);
    float hr[2] = {lo, hi};
    int zero = 0;
    CK(cudaMemcpyAsync(d_x, x, n * sizeof(float), cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(d_r, hr, sizeof(hr), cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(d_s, &zero, sizeof(int), cudaMemcpyHostToDevice, c->st));
    CK(cudaMemsetAsync(d_c, 0, PTQ_NBINS * 8, c->st));
    launch_histogram(d_x, n, d_s, 1, d_r, d_c, c->st);
    check_launch(c);
    CK(cudaMemcpyAsync(counts, d_c, PTQ_NBINS * 8, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    for (void* p : {(void*)d_x, (void*)d_r, (void*)d_s, (void*)d_c}) c->dfree(p);
  });
}

int ptq_set_option(ptq_ctx* c, const char* key, int64_t value) {
  return guarded([&] {
    REQ(c && key, "null argument");
    std::string k(key);
    if (k == "conv_ref") c->conv_ref = (int)value;
    else if (k == "ablate") c->ablate = (int)value;
    else if (k == "tma") c->tma = (int)value;
    else if (k == "subsample") c->subsample = (int)value;
    else if (k == "dwconv_v4") c->dwconv_variant = (int)value;
    else if (k == "concat_v16") c->concat_v16 = (int)value;
    else if (k == "kwr") c->kwr = (int)value;
    else if (k == "fx") c->fx = (int)value;
    else if (k == "rs_mma") c->rs_mma = (int)value;
    else if (k == "skip_pf") c->skip_pf = (int)value;
    else if (k == "tio") c->tio = (int)value;
    else if (k == "hist_multi") c->hist_multi = (int)value;
    else if (k == "time_conv") c->time_conv = (int)value;
    else if (k == "reset_stats") c->launches = 0;
    else if (k == "fusion") {
      if (c->fusion != (int)value) {
        c->fusion = (int)value;
        for (auto& P : c->plans) { if (P.d_layers) c->dfree(P.d_layers); P = Plan{}; }
        for (auto p : c->d_codes) c->dfree(p);
        c->d_codes.clear();
        c->halo_key.clear();
        c->static_ready = false;
        c->prepared = false;
      }
    } else if (k == "eval_chunk") {
      c->opt_chunk = value;
      c->static_ready = false;
      c->prepared = false;
    } else {
      REQ(false, "unknown option " + k);
    }
  });
}

int ptq_last_stats(const ptq_ctx* c, int64_t* launches, double* conv_ms, double* conv_ops,
                   int64_t* conv_launches, int64_t* conv_launches_total) {
  if (!c) { g_err = "null context"; return PTQ_EINVAL; }
  if (launches) *launches = c->launches;
  if (conv_ms) *conv_ms = c->conv_ms;
  if (conv_ops) *conv_ops = c->conv_ops;
  if (conv_launches) *conv_launches = (int64_t)(c->ev_used / 2);
  if (conv_launches_total) *conv_launches_total = c->conv_launches_total;
  return PTQ_OK;
}

int ptq_conv_timings(const ptq_ctx* c, float* ms, int64_t cap, int64_t* n) {
  if (!c || !n) { g_err = "null argument"; return PTQ_EINVAL; }
  *n = (int64_t)(c->ev_used / 2);
  for (int64_t i = 0; ms && i < *n && i < cap; ++i) {
    float v = 0.f;
    if (cudaEventElapsedTime(&v, c->ev_pool[2 * i], c->ev_pool[2 * i + 1]) != cudaSuccess) {
      g_err = "event timing unavailable";
      return PTQ_ECUDA;
    }
    ms[i] = v;
  }
  return PTQ_OK;
}

int ptq_stream(const ptq_ctx* c, void** stream) {
  if (!c || !stream) { g_err = "null argument"; return PTQ_EINVAL; }
  *stream = (void*)c->st;
  return PTQ_OK;
}

}  // extern "C"
