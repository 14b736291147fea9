// Host-side launch wrappers for every ptq_b200 kernel family, plus the small
// POD structs shared between the runtime and the kernels.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace ptq {

// int8 activation tensor in HBM: NHWC, channel pitch Cp (multiple of 16), optional
// spatial halo filled with the tensor's zero-point code (so convs never test bounds).
struct View {
  int8_t* p;
  int N, H, W, C, Cp, halo;
};

// fused-add lookup table geometry (rows padded against shared-memory bank conflicts)
#define PTQ_ADDTAB_ROW 260
#define PTQ_ADDTAB_BYTES (256 * PTQ_ADDTAB_ROW)

// per-config, per-int8-layer scalars written on device by k_layer_params
struct LayerRt {
  int zx, zy;          // input / output zero points (output = the conv's own quant params)
  int relu_zp;         // zero point used by a fused relu (or INT32_MIN for none)
  int za, zb, zo;      // fused add: operand zps and add output zp
  double ra, rb;       // fused add: s_a / s_o and s_b / s_o (operand order of the add node)
  int add_relu_zp;     // relu fused after the add (or INT32_MIN)
  int slow;            // 1: the fast epilogue's range preconditions fail -> exact 64-bit path
  int aclamp;          // fast path clamps acc to [-aclamp, aclamp]: beyond it every channel
                       // saturates (|acc*m| > 300) and |acc*m| stays < 2^30 for the floor trick
  double mg_zy, mg_zo; // 1.5*2^52 + zp: floor(r) + zp via one round-down add
  int noclamp;         // max m < 0.5: |acc*m| < 2^30 for any int32 acc, no clamp needed
  int uni;             // every channel has the same m and zw (per-tensor weights): m0 / zw0
  double m0;
  int zw0;
  // exact fixed-point requant (k_layer_params, "FX"): code = (v'*M_c + B'_c) >> (32 + fx_s)
  // reproduces clip(floor(fl(fl(acc*m_c) + 0.5)) + zy) for every int32 accumulator, with
  // v' = dot - zw*rowsum (acc = v' + cc).  fx = 1 when every channel's (M_c, B'_c) was found;
  // the EpiParam SoA then holds B'_c (int64) in the m slot and M_c in the cc slot.
  int fx;
  int fx_s;            // S - 32 (per layer)
  int fx_m0;           // M of per-tensor layers (uni)
};

// per-config, per-output-channel epilogue constants of the tensor-core conv:
//   acc = dot - zw*rowsum + cc  (cc = bias - zx*sum(w) + K*zx*zw), out = requant(acc, m)
// stored as a structure of arrays in a block of cs = roundup(cout, 16) EpiParam slots
// (16 * cs bytes): m[cs] fp64 at byte 0, cc[cs] at byte 8*cs, zw[cs] at byte 12*cs.
//   cc is cc + 2^31 (mod 2^32); valid when the layer's rt.slow == 0 (|cc| < 2^30, no int32
//   clip possible).  The bias lets acc + 2^31 feed i2d directly.
//   With rt.fx = 1 the same block holds the fixed-point constants instead: B'_c (int64) at
//   byte 0, M_c (int32) at byte 8*cs, zw at 12*cs.
struct alignas(16) EpiParam {
  double m;
  int cc;
  int zw;
};

// static description of one int8 compute layer (conv / pointwise / depthwise / fc)
struct LayerSt {
  int cout;
  int in_hist, out_hist;        // act-param sources (histogram ids) of input and output
  int relu_hist;                // -1 or hist id whose zp the fused relu clamps to
  int add_a_hist, add_b_hist, add_o_hist;  // -1 when no fused add
  int add_relu_hist;            // -1 or hist id of a relu fused after the add
  const float* bias;            // fp32 bias (device) or nullptr
  const float* wscale;          // [8 variants][cout]
  double* mult;                 // [cout] per-config requant multipliers (out)
  int* biasq;                   // [cout] per-config int32 bias codes (out)
  LayerRt* rt;                  // per-config scalars (out)
  const int* wzp8;              // [8][cout] weight zero points (tensor-core layers)
  const int* wsum8;             // [8][cout] sum of weight codes
  int kreal;                    // real K = k*k*Cin
  EpiParam* ep;                 // [roundup(cout,16)] per-config epilogue constants (SoA, out), or nullptr
  int8_t* addtab;               // fused residual add: [256 skip codes][260: conv code + 128]
                                // -> add output code (out, per config), or nullptr
  int add_conv_is_a;            // 1 if the conv output is operand 0 of the fused add
  int dw;                       // depthwise layer: cc = bias code only (the kernel sums the rest)
};

// ---------------------------------------------------------------- F1 / F2 (k_calib.cu)
void launch_minmax_per_image(const float* x, int64_t elems, int n_img, unsigned int* out_ord,
                             cudaStream_t s);
void launch_fill_minmax(unsigned int* p, int64_t n_pairs, cudaStream_t s);
void launch_minmax_reduce_cache(const unsigned int* per_img, int n_tensors, int n_img_total,
                                const int* slots, int n_slots, float* ranges, cudaStream_t s);
void launch_histogram(const float* x, int64_t elems, const int* slots, int n_slots,
                      const float* range, unsigned long long* counts, cudaStream_t s);
// one histogram of the batched launch: values x[slots[j]][e], range (lo, hi), 2048 int64 counts
struct HistItem {
  const float* x;
  int64_t elems;
  const int* slots;
  int n_slots;
  const float* range;
  unsigned long long* counts;
  int64_t chunk0;          // first chunk index of this item (hist_items_chunk0)
};
int64_t hist_items_chunk0(HistItem* items, int n);      // fills chunk0, returns the chunk count
void launch_histogram_multi(const HistItem* d_items, int n_items, int64_t n_chunks, cudaStream_t s);
void launch_percentile(const long long* counts, const float* ranges, int n_hist, double q, double* out,
                       cudaStream_t s);
void launch_kl_sweep(const long long* counts, const float* ranges, int n_hist, double* cum,
                     int* nzc, double* logc, double* kl_out, cudaStream_t s);

// ---------------------------------------------------------------- fp32 forward (k_fp32.cu)
void launch_nchw_to_nhwc(const float* src, const int* ids, int n, int C, int H, int W, float* dst,
                         cudaStream_t s);
void launch_conv_f32(const float* x, int N, int H, int W, int Cin, const float* Bw,
                     const float* bias, int Cout, int k, int stride, int pad, int OH, int OW,
                     float* y, cudaStream_t s);
void launch_dwconv_f32(const float* x, int N, int H, int W, int C, const float* w,
                       const float* bias, int k, int stride, int pad, int OH, int OW, float* y,
                       cudaStream_t s);
void launch_gemm_weight(const float* w, int cout, int cin, int k, int hw, float* out, cudaStream_t s);
void launch_relu_f32(const float* x, float* y, int64_t n, cudaStream_t s);
void launch_add_f32(const float* a, const float* b, float* y, int64_t n, cudaStream_t s);
void launch_pool_f32(const float* x, int N, int H, int W, int C, int k, int stride, int OH, int OW,
                     int mode, float* y, cudaStream_t s);
void launch_concat_f32(const float* x, int64_t npix, int Cx, int Cy, int coff, float* y,
                       cudaStream_t s);
void launch_softmax_f32(const float* x, int64_t rows, int C, float* y, cudaStream_t s);

// ---------------------------------------------------------------- F3 (k_quant.cu)
void launch_act_params(const double* ranges /*[n_var][T][2]*/, const int* var_scheme, int n_var,
                       int T, float* scale, int* zp, cudaStream_t s);
// all 8 (scheme, granularity) variants of one weight tensor: params, codes, code sums
void launch_weight_prepare8(const float* w, int cout, int64_t per_ch, bool depthwise, int cin, int k,
                            int fc_hw, int cin_p, int bn, int rows_mask, int n_kiter, int64_t bytes_per_variant,
                            unsigned int* mnmx, float* scale, int* zp, int8_t* codes, int* wsum,
                            cudaStream_t s);
// fx: 1 = also derive the exact fixed-point epilogue constants (LayerRt::fx), 0 = fp64 only
void launch_layer_params(const LayerSt* d_layers, int n_layers, const float* act_scale,
                         const int* act_zp, int wvar, int fx, cudaStream_t s);
void launch_quant_input(const float* imgs_nchw, int64_t img0, View out, const float* act_scale,
                        const int* act_zp, int hist, cudaStream_t s);
void launch_quant_input_s2d(const float* imgs_nchw, int64_t img0, int C0, View out,
                            const float* act_scale, const int* act_zp, int hist, cudaStream_t s);
void launch_stem_rowsum(View in_s2d, int k, int C0, int OH, int OW, int* R, cudaStream_t s);
void launch_quant_nhwc(const float* x, View out, const float* act_scale, const int* act_zp,
                       int hist, int relu_hist, cudaStream_t s);
void launch_dequant(View in, const float* act_scale, const int* act_zp, int hist, float* y,
                    cudaStream_t s);
void launch_halo_fill(View v, const int* act_zp, int hist, cudaStream_t s);
// the halos of up to 48 tensors with their zero-point codes act_zp[hist[i]], one launch
struct HaloBatch {
  int n;
  View v[48];
  int hist[48];
  int64_t unit0[48];
  int64_t total;
};
void launch_halo_fill_multi(HaloBatch& hb, const int* act_zp, cudaStream_t s);
void launch_relu_codes(View in, View out, const int* act_zp, int hist, cudaStream_t s);
void launch_pool_codes(View in, View out, int k, int stride, int mode, const int* act_zp,
                       int hist, cudaStream_t s);
void launch_add_codes(View a, View b, View out, const float* act_scale, const int* act_zp,
                      int ha, int hb, int ho, cudaStream_t s);
// v16: 1 = per-block 256-entry requant table, 16 codes per thread; 0 = per-byte fp64 (A/B)
void launch_concat_codes(View in, View out, int coff, const float* act_scale, const int* act_zp,
                         int hin, int hout, cudaStream_t s, int v16 = 1);
void launch_pixsum(View in, int* P, cudaStream_t s);
// variant: 2 = k x k register-tap kernel, 1 = four channels per thread, 0 = scalar (A/B)
void launch_dwconv_i8(View in, View out, const int8_t* w, const int* wzp, int k, int stride,
                      int pad, LayerSt L, cudaStream_t s, int* acc_out = nullptr, int variant = 2);
void launch_argmax_codes(View in, const long long* labels, unsigned long long* correct,
                         cudaStream_t s);
void launch_argmax_f32(const float* x, int64_t rows, int C, const long long* labels,
                       unsigned long long* correct, cudaStream_t s);

// ---------------------------------------------------------------- F4 (k_conv_tc.cu)
// n / d and n % d for 0 <= n < 2^31 with a multiply-high (CUTLASS-style round-up magic)
struct FastDiv {
  uint32_t d, mul, shr;
  static FastDiv make(uint32_t d) {
    FastDiv f{d, 0u, 0u};
    if (d > 1) {
      uint32_t l = 0;
      while ((1u << l) < d) ++l;                 // ceil(log2 d)
      const uint32_t p = 31 + l;
      f.mul = (uint32_t)(((1ull << p) + d - 1) / d);
      f.shr = p - 32;
    }
    return f;
  }
#ifdef __CUDACC__
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    return d == 1 ? n : (__umulhi(n, mul) >> shr);
  }
#endif
};

// packed im2col for convs with few input channels (the RGB stem): row m of `out` holds
// the k*k*C codes of output pixel m in (kh, kw, c) order, zero padded to out_cp bytes
void launch_im2col(View in, int k, int stride, int pad, int OH, int OW, int8_t* out, int out_cp,
                   cudaStream_t s);

struct ConvTcArgs {
  CUtensorMap tmA;        // TMA map of the A operand (tma_a != 0); 64-byte aligned first member
  CUtensorMap tmO, tmS;   // tile I/O (tio): output / fused-add operand as [pixels][Cp] maps
  int tma_a;              // 0: cp.async implicit-im2col gather; 64 / 128: TMA tile loads of
                          // 128 flat padded pixels x 64 / 128 channel bytes (SWIZZLE_64B / 128B)
  int OHr, OWr;           // real output dims (TMA mode computes over the padded grid OH x OW)
  int allow_tma;          // runtime option: TMA A loads for eligible layers
  View in, out;
  int k, stride, pad, OH, OW;
  const int8_t* wB;       // tiled weights [n_tiles][n_kiter][8][b_rows][16]
  int b_rows;             // B rows per tile: BN, or BN + 16 when the tiles carry the 16 K-indicator
                          // rows (1 at every real K position) used by rs_mma
  int rs_mma;             // set by the runtime (has_wzp, b_rows > BN): the MMA runs over N = BN + 16
                          // and the extra accumulator columns are the A-row sums sum_k x[row][k]
                          // (no row-sum warp, pixel-sum pass or stem window-sum pass)
  int n_kiter;            // K stages of 128 bytes
  int n_chunks;           // real 16-byte K chunks = k*k*Cp/16
  const int* wzp;         // [cout] weight zero points (variant)
  const int* wsum;        // [cout] sum of weight codes over real K (variant)
  int kreal;              // k*k*C
  const int* P;           // per-padded-input-pixel channel sums (only when has_wzp)
  const int* Rpix;        // per-output-pixel window sums (s2d stem with has_wzp) or nullptr
  int tma_rowsum;         // set by the launcher: TMA mode with has_wzp -> row sums of the A
                          // tiles are taken from shared memory (no pixel-sum pass)
  int has_wzp;
  LayerSt L;              // holds device pointers: mult / biasq / rt
  View skip;              // fused add operand (p == nullptr when none)
  int conv_is_a;          // 1 if the conv output is operand 0 of the fused add
  FastDiv div_ow, div_oh, div_nt;   // m -> (n, oh, ow) and tile -> (m-tile, n-tile)
  int ablate;             // profiling only: 1 = skip epilogue math, 2 = skip A gathers
  const int8_t* addtab;   // fused add lookup table (LayerSt::addtab) or nullptr
  int n_stages;           // smem pipeline depth (set by the launcher)
  int b_res;              // set by the launcher: the whole B operand (one n-tile) stays resident
                          // in shared memory instead of streaming with every tile
  int kwr;                // set by the launcher: 3x3 Cp=64 TMA conv loads one 136-row slab per kh
                          // and feeds its 3 kw taps as row-shifted descriptors (A bytes / 3)
  int a_iters;            // A pipeline stages per tile (n_kiter, or 3 kh slabs with kwr)
  int flat;               // set by the launcher: GEMM row m is flat pixel m of the output (and of
                          // the add operand) -- halo-free TMA-mode layers skip the row geometry
  int kwr_mode;           // runtime option: -1 disables the kw-reuse slabs and the stem slab
  int tio_mode;           // runtime option: 0 disables tile I/O
  int skip_pf;            // runtime option: L2 prefetch of the fused-add operand tiles (tile I/O)
  int tio;                // set by the launcher (flat layers): the epilogue writes codes into a
                          // swizzled shared tile stored by TMA, and reads the fused-add operand from
                          // a tile a producer loads by TMA, instead of per-row 16-byte global accesses
  int io_w;               // tile I/O box width in bytes (64 or 128 = the swizzle span)
  int* acc_out;           // parity probe (ptq_probe_acc): when set, the epilogue stores the exact
                          // int32-clipped accumulator acc + bias (intexec.py:177-190) of every real
                          // output as [pixel][cout] int32 instead of requantized codes
};
int conv_tc_bn_for(int cout);     // BN tile width the kernel uses for this Cout
int conv_tc_max_cout();           // largest Cout the tensor-core conv supports
void launch_conv_tc(const ConvTcArgs& a, int bn, cudaStream_t s);
// true when launch_conv_tc will load A with TMA and (with has_wzp) sum the rows itself
bool conv_tc_tma_rowsum(const ConvTcArgs& a, int bn);
// CUDA-core reference of the same contract (tests / cross-checks only)
void launch_conv_i8_ref(const ConvTcArgs& a, int bn, cudaStream_t s);

}  // namespace ptq
