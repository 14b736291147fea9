// fp32 forward kernels (calibration observer pass and mixed-precision
// FirstLastFp32 layers).  Layout NHWC, batch-major.  These restate the
// reference's fp32 interpreter (/root/reference/pkg/src/ptqtune/fp32.py:41-114)
// but accumulate in a different order than OpenBLAS sgemm, so activations
// agree to ~1e-6 relative, not bitwise (SURVEY.md 8(c) staged parity).
#include "common.cuh"
#include "kernels.h"

namespace ptq {

// images NCHW (host layout) -> NHWC, gathering image ids
__global__ void k_nchw_to_nhwc(const float* __restrict__ src, const int* __restrict__ ids, int n,
                               int C, int H, int W, float* __restrict__ dst) {
  int64_t total = (int64_t)n * C * H * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int c = i % C;
    int64_t r = i / C;
    int w = r % W; r /= W;
    int h = r % H;
    int img = (int)(r / H);
    int64_t sid = ids ? ids[img] : img;
    dst[i] = __ldg(src + ((sid * C + c) * H + h) * W + w);
  }
}

// Implicit-GEMM direct conv, fp32 SIMT.
// out[m][co] = bias[co] + sum_k A[m][k] * Bw[k][co];  m = (n, oh, ow); k = (kh, kw, ci).
// Bw is [K][Cout] (prepared on device).  Also used for fully-connected layers
// (1x1 "image" whose channel axis is the NHWC-flattened feature vector).
constexpr int CF_BM = 128, CF_BN = 64, CF_BK = 8;
__global__ void __launch_bounds__(256) k_conv_f32(const float* __restrict__ x, int N, int H, int W,
                                                  int Cin, const float* __restrict__ Bw,
                                                  const float* __restrict__ bias, int Cout, int k,
                                                  int stride, int pad, int OH, int OW,
                                                  float* __restrict__ y) {
  __shared__ float As[CF_BK][CF_BM + 4];
  __shared__ float Bs[CF_BK][CF_BN];
  const int tid = threadIdx.x;
  const int64_t M = (int64_t)N * OH * OW;
  const int K = k * k * Cin;
  const int64_t m0 = (int64_t)blockIdx.x * CF_BM;
  const int n0 = blockIdx.y * CF_BN;
  // loader mapping: A: kk = tid % 8, rows r = tid/8 + 32*j
  const int a_k = tid & 7;
  int a_ih0[4], a_iw0[4];
  int64_t a_base[4];
  bool a_ok[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    int64_t m = m0 + (tid >> 3) + 32 * j;
    a_ok[j] = m < M;
    int64_t mm = a_ok[j] ? m : 0;
    int ow = mm % OW;
    int64_t t = mm / OW;
    int oh = t % OH;
    int nimg = (int)(t / OH);
    a_ih0[j] = oh * stride - pad;
    a_iw0[j] = ow * stride - pad;
    a_base[j] = (int64_t)nimg * H * W;
  }
  const int b_k = tid >> 5, b_n = (tid & 31) * 2;  // 8 x 64 tile, 2 per thread
  const int tm = tid >> 4, tn = tid & 15;           // compute: rows tm*8.., cols tn*4..
  float acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int k0 = 0; k0 < K; k0 += CF_BK) {
    {
      int kk = k0 + a_k;
      int tap = kk / Cin, ci = kk - tap * Cin;
      int kh = tap / k, kw = tap - kh * k;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float v = 0.f;
        int ih = a_ih0[j] + kh, iw = a_iw0[j] + kw;
        if (a_ok[j] && kk < K && ih >= 0 && ih < H && iw >= 0 && iw < W)
          v = __ldg(x + ((a_base[j] + (int64_t)ih * W + iw) * Cin + ci));
        As[a_k][(tid >> 3) + 32 * j] = v;
      }
      int kb = k0 + b_k;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        int nn = n0 + b_n + j;
        Bs[b_k][b_n + j] = (kb < K && nn < Cout) ? __ldg(Bw + (int64_t)kb * Cout + nn) : 0.f;
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < CF_BK; ++kk) {
      float a[8], b[4];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = As[kk][tm * 8 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tn * 4 + j];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int64_t m = m0 + tm * 8 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int nn = n0 + tn * 4 + j;
      if (nn < Cout) y[m * Cout + nn] = acc[i][j] + (bias ? __ldg(bias + nn) : 0.f);
    }
  }
}

// Register-blocked implicit-GEMM conv for Cin % 8 == 0 (every layer but the RGB stem):
// 128 x BN block tile, BK = 8 (one tap, 8 consecutive channels), 256 threads each owning
// an 8 x (BN/16) register tile, double-buffered shared tiles with the next K slice
// prefetched into registers (float4 global loads) while the current one is multiplied.
template <int BN, int BK>
__global__ void __launch_bounds__(256, 2) k_conv_f32_rb(const float* __restrict__ x, int N, int H, int W,
                                                     int Cin, const float* __restrict__ Bw,
                                                     const float* __restrict__ bias, int Cout, int k,
                                                     int stride, int pad, int OH, int OW,
                                                     float* __restrict__ y) {
  constexpr int BM = 128, TN = BN / 16;           // TN = 8 (BN 128) or 4 (BN 64)
  constexpr int NA = BK / 8;                       // float4 A loads per thread per K slice
  constexpr int NB = (BK * BN / 4 + 255) / 256;    // float4 B loads per thread per K slice
  __shared__ __align__(16) float As[2][BK][BM + 4];
  __shared__ __align__(16) float Bs[2][BK][BN];
  const int tid = threadIdx.x;
  const int64_t M = (int64_t)N * OH * OW;
  const int K = k * k * Cin;
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;
  // A loader: row ar = tid / 2, channels 4 * (tid & 1) + 8 j .. +4 of the current tap
  const int ar = tid >> 1, ah = (tid & 1) * 4;
  const int64_t am = m0 + ar;
  const bool aok = am < M;
  int aih0 = 0, aiw0 = 0;
  int64_t abase = 0;
  {
    const int64_t mm = aok ? am : 0;
    const int ow = (int)(mm % OW);
    const int64_t t = mm / OW;
    const int oh = (int)(t % OH);
    aih0 = oh * stride - pad;
    aiw0 = ow * stride - pad;
    abase = (t / OH) * H * W;
  }
  // B loader: float4 index q = tid + 256 i over the BK x BN slice
  const int tm = tid >> 4, tn = tid & 15;
  float acc[8][TN];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

  auto load_a = [&](int k0, float4 (&r)[NA]) {
    const int tap = k0 / Cin, ci = k0 - tap * Cin + ah;
    const int kh = tap / k, kw = tap - kh * k;
    const int ih = aih0 + kh, iw = aiw0 + kw;
    const bool ok = aok && ih >= 0 && ih < H && iw >= 0 && iw < W;
    const float4* src = reinterpret_cast<const float4*>(x + (abase + (int64_t)ih * W + iw) * Cin + ci);
#pragma unroll
    for (int j = 0; j < NA; ++j) r[j] = ok ? __ldg(src + 2 * j) : make_float4(0.f, 0.f, 0.f, 0.f);
  };
  auto load_b = [&](int k0, float4 (&r)[NB]) {
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const int q = tid + 256 * i, bk = q / (BN / 4), bc = (q % (BN / 4)) * 4;
      const int nn = n0 + bc;
      r[i] = (bk < BK && nn < Cout) ? __ldg(reinterpret_cast<const float4*>(Bw + (int64_t)(k0 + bk) * Cout + nn))
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  float4 ra[NA], rb[NB];
  load_a(0, ra);
  load_b(0, rb);
  int buf = 0;
  for (int k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
    for (int j = 0; j < NA; ++j) {
      As[buf][ah + 8 * j + 0][ar] = ra[j].x;
      As[buf][ah + 8 * j + 1][ar] = ra[j].y;
      As[buf][ah + 8 * j + 2][ar] = ra[j].z;
      As[buf][ah + 8 * j + 3][ar] = ra[j].w;
    }
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const int q = tid + 256 * i, bk = q / (BN / 4), bc = (q % (BN / 4)) * 4;
      if (bk < BK) *reinterpret_cast<float4*>(&Bs[buf][bk][bc]) = rb[i];
    }
    __syncthreads();
    if (k0 + BK < K) {                               // prefetch the next K slice
      load_a(k0 + BK, ra);
      load_b(k0 + BK, rb);
    }
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][tm * 8]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][tm * 8 + 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      float b[TN];
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tn * TN]);
      b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w;
      if (TN == 8) {
        const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tn * TN + 4]);
        b[4 % TN] = b1.x; b[5 % TN] = b1.y; b[6 % TN] = b1.z; b[7 % TN] = b1.w;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    buf ^= 1;
  }
  const int cn = n0 + tn * TN;
  float bv[TN];
#pragma unroll
  for (int j = 0; j < TN; ++j) bv[j] = (bias && cn + j < Cout) ? __ldg(bias + cn + j) : 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t m = m0 + tm * 8 + i;
    if (m >= M || cn >= Cout) continue;
    float* dst = y + m * Cout + cn;
#pragma unroll
    for (int j = 0; j < TN; j += 4)
      *reinterpret_cast<float4*>(dst + j) =
          make_float4(acc[i][j] + bv[j], acc[i][j + 1] + bv[j + 1], acc[i][j + 2] + bv[j + 2], acc[i][j + 3] + bv[j + 3]);
  }
}

// fully-connected layers with few outputs (the classifier): one warp per output element,
// lanes stride over K (the generic tiled kernel would run a handful of CTAs over K)
__global__ void k_fc_f32_small(const float* __restrict__ x, int64_t rows, int K, const float* __restrict__ Bw,
                               const float* __restrict__ bias, int Cout, float* __restrict__ y) {
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= rows * Cout) return;
  const int64_t r = wid / Cout;
  const int co = (int)(wid - r * Cout);
  const float* xr = x + r * K;
  float acc = 0.f;
  for (int kk = lane; kk < K; kk += 32) acc = fmaf(__ldg(xr + kk), __ldg(Bw + (int64_t)kk * Cout + co), acc);
  for (int d = 16; d; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
  if (lane == 0) y[wid] = acc + (bias ? __ldg(bias + co) : 0.f);
}

// depthwise conv: w is [C][k*k]
__global__ void k_dwconv_f32(const float* __restrict__ x, int N, int H, int W, int C,
                             const float* __restrict__ w, const float* __restrict__ bias, int k,
                             int stride, int pad, int OH, int OW, float* __restrict__ y) {
  int64_t total = (int64_t)N * OH * OW * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int c = i % C;
    int64_t r = i / C;
    int ow = r % OW; r /= OW;
    int oh = r % OH;
    int n = (int)(r / OH);
    float acc = 0.f;
    for (int kh = 0; kh < k; ++kh) {
      int ih = oh * stride - pad + kh;
      if (ih < 0 || ih >= H) continue;
      for (int kw = 0; kw < k; ++kw) {
        int iw = ow * stride - pad + kw;
        if (iw < 0 || iw >= W) continue;
        acc = fmaf(__ldg(x + (((int64_t)n * H + ih) * W + iw) * C + c), __ldg(w + c * k * k + kh * k + kw), acc);
      }
    }
    y[i] = acc + (bias ? __ldg(bias + c) : 0.f);
  }
}

__global__ void k_relu_f32(const float* __restrict__ x, float* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = fmaxf(x[i], 0.f);
}

__global__ void k_add_f32(const float* __restrict__ a, const float* __restrict__ b,
                          float* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = a[i] + b[i];
}

// mode 0 = max, 1 = avg (sum in fp32 then / area)
__global__ void k_pool_f32(const float* __restrict__ x, int N, int H, int W, int C, int k,
                           int stride, int OH, int OW, int mode, float* __restrict__ y) {
  int64_t total = (int64_t)N * OH * OW * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int c = i % C;
    int64_t r = i / C;
    int ow = r % OW; r /= OW;
    int oh = r % OH;
    int n = (int)(r / OH);
    float acc = mode ? 0.f : -INFINITY;
    for (int kh = 0; kh < k; ++kh)
      for (int kw = 0; kw < k; ++kw) {
        float v = __ldg(x + (((int64_t)n * H + oh * stride + kh) * W + ow * stride + kw) * C + c);
        acc = mode ? acc + v : fmaxf(acc, v);
      }
    y[i] = mode ? acc / (float)(k * k) : acc;
  }
}

// copy x [n][HW][Cx] into y [n][HW][Cy] at channel offset coff
__global__ void k_concat_f32(const float* __restrict__ x, int64_t npix, int Cx, int Cy, int coff,
                             float* __restrict__ y) {
  int64_t total = npix * Cx;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = i / Cx;
    int c = i - p * Cx;
    y[p * Cy + coff + c] = x[i];
  }
}

// softmax over the last axis of [rows][C] (one warp per row)
__global__ void k_softmax_f32(const float* __restrict__ x, int64_t rows, int C, float* __restrict__ y) {
  int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float* p = x + r * C;
  float mx = -INFINITY;
  for (int c = lane; c < C; c += 32) mx = fmaxf(mx, p[c]);
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float s = 0.f;
  for (int c = lane; c < C; c += 32) s += expf(p[c] - mx);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  for (int c = lane; c < C; c += 32) y[r * C + c] = expf(p[c] - mx) / s;
}

// fp32 GEMM weight [K][cout] (K in NHWC order) from the reference layout: conv OIHW
// (K = (kh*k + kw)*cin + c) or fc (O, C*H*W) flattened NCHW (K = p*cin + c, p = h*W + w)
__global__ void k_gemm_weight(const float* __restrict__ w, int cout, int cin, int k, int hw,
                              float* __restrict__ out, int64_t total) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int o = (int)(i % cout);
    const int64_t kidx = i / cout;
    const int ci = (int)(kidx % cin);
    const int64_t t = kidx / cin;
    int64_t src;
    if (hw > 0) {
      src = ((int64_t)o * cin + ci) * hw + t;
    } else {
      const int a = (int)(t / k), b = (int)(t % k);
      src = (((int64_t)o * cin + ci) * k + a) * k + b;
    }
    out[i] = __ldg(w + src);
  }
}

// ---------------------------------------------------------------- launch wrappers
static inline int gblk(int64_t n) {
  int64_t b = (n + 255) / 256;
  return (int)(b < 1 ? 1 : (b > 148 * 32 ? 148 * 32 : b));
}
void launch_nchw_to_nhwc(const float* src, const int* ids, int n, int C, int H, int W, float* dst,
                         cudaStream_t s) {
  k_nchw_to_nhwc<<<gblk((int64_t)n * C * H * W), 256, 0, s>>>(src, ids, n, C, H, W, dst);
}
void launch_conv_f32(const float* x, int N, int H, int W, int Cin, const float* Bw,
                     const float* bias, int Cout, int k, int stride, int pad, int OH, int OW,
                     float* y, cudaStream_t s) {
  int64_t M = (int64_t)N * OH * OW;
  if (k == 1 && H == 1 && W == 1 && OH == 1 && OW == 1 && Cout < 64) {
    const int64_t warps = M * Cout;
    k_fc_f32_small<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(x, M, Cin, Bw, bias, Cout, y);
    return;
  }
  if (Cin % 8 == 0 && Cout % 64 == 0) {              // register-blocked path (float4 operands)
    const bool bk16 = Cin % 16 == 0;                 // 16-deep K slices: half the barriers
    if (Cout % 128 == 0) {
      dim3 g((unsigned)((M + 127) / 128), (unsigned)(Cout / 128));
      if (bk16) k_conv_f32_rb<128, 16><<<g, 256, 0, s>>>(x, N, H, W, Cin, Bw, bias, Cout, k, stride, pad, OH, OW, y);
      else k_conv_f32_rb<128, 8><<<g, 256, 0, s>>>(x, N, H, W, Cin, Bw, bias, Cout, k, stride, pad, OH, OW, y);
    } else {
      dim3 g((unsigned)((M + 127) / 128), (unsigned)(Cout / 64));
      if (bk16) k_conv_f32_rb<64, 16><<<g, 256, 0, s>>>(x, N, H, W, Cin, Bw, bias, Cout, k, stride, pad, OH, OW, y);
      else k_conv_f32_rb<64, 8><<<g, 256, 0, s>>>(x, N, H, W, Cin, Bw, bias, Cout, k, stride, pad, OH, OW, y);
    }
    return;
  }
  dim3 g((unsigned)((M + CF_BM - 1) / CF_BM), (unsigned)((Cout + CF_BN - 1) / CF_BN));
  k_conv_f32<<<g, 256, 0, s>>>(x, N, H, W, Cin, Bw, bias, Cout, k, stride, pad, OH, OW, y);
}
// four channels per thread (float4 loads / stores); per channel the same fmaf chain in the
// same (kh, kw) order as k_dwconv_f32, so the results are bit-identical
__global__ void k_dwconv_f32_v4(const float* __restrict__ x, int N, int H, int W, int C,
                                const float* __restrict__ w, const float* __restrict__ bias, int k,
                                int stride, int pad, int OH, int OW, float* __restrict__ y) {
  const int cq = C >> 2;
  const int64_t total = (int64_t)N * OH * OW * cq;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c0 = (int)(i % cq) * 4;
    const int p = (int)(i / cq);
    const int ow = p % OW, t = p / OW;
    const int oh = t % OH, n = t / OH;
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    for (int kh = 0; kh < k; ++kh) {
      const int ih = oh * stride - pad + kh;
      if (ih < 0 || ih >= H) continue;
      for (int kw = 0; kw < k; ++kw) {
        const int iw = ow * stride - pad + kw;
        if (iw < 0 || iw >= W) continue;
        const float4 v = __ldg(reinterpret_cast<const float4*>(x + (((int64_t)n * H + ih) * W + iw) * C + c0));
        const int tap = kh * k + kw;
        a0 = fmaf(v.x, __ldg(w + (c0 + 0) * k * k + tap), a0);
        a1 = fmaf(v.y, __ldg(w + (c0 + 1) * k * k + tap), a1);
        a2 = fmaf(v.z, __ldg(w + (c0 + 2) * k * k + tap), a2);
        a3 = fmaf(v.w, __ldg(w + (c0 + 3) * k * k + tap), a3);
      }
    }
    if (bias) {
      a0 += __ldg(bias + c0); a1 += __ldg(bias + c0 + 1);
      a2 += __ldg(bias + c0 + 2); a3 += __ldg(bias + c0 + 3);
    } else {
      a0 += 0.f; a1 += 0.f; a2 += 0.f; a3 += 0.f;
    }
    *reinterpret_cast<float4*>(y + (int64_t)p * C + c0) = make_float4(a0, a1, a2, a3);
  }
}

void launch_dwconv_f32(const float* x, int N, int H, int W, int C, const float* w,
                       const float* bias, int k, int stride, int pad, int OH, int OW, float* y,
                       cudaStream_t s) {
  if (C % 4 == 0 && ((uintptr_t)x & 15) == 0 && ((uintptr_t)y & 15) == 0) {
    k_dwconv_f32_v4<<<gblk((int64_t)N * OH * OW * (C / 4)), 256, 0, s>>>(x, N, H, W, C, w, bias, k,
                                                                        stride, pad, OH, OW, y);
    return;
  }
  k_dwconv_f32<<<gblk((int64_t)N * OH * OW * C), 256, 0, s>>>(x, N, H, W, C, w, bias, k, stride,
                                                             pad, OH, OW, y);
}
void launch_gemm_weight(const float* w, int cout, int cin, int k, int hw, float* out, cudaStream_t s) {
  const int64_t total = (int64_t)cout * cin * (hw > 0 ? hw : k * k);
  k_gemm_weight<<<gblk(total), 256, 0, s>>>(w, cout, cin, k, hw, out, total);
}
void launch_relu_f32(const float* x, float* y, int64_t n, cudaStream_t s) {
  k_relu_f32<<<gblk(n), 256, 0, s>>>(x, y, n);
}
void launch_add_f32(const float* a, const float* b, float* y, int64_t n, cudaStream_t s) {
  k_add_f32<<<gblk(n), 256, 0, s>>>(a, b, y, n);
}
void launch_pool_f32(const float* x, int N, int H, int W, int C, int k, int stride, int OH, int OW,
                     int mode, float* y, cudaStream_t s) {
  k_pool_f32<<<gblk((int64_t)N * OH * OW * C), 256, 0, s>>>(x, N, H, W, C, k, stride, OH, OW, mode, y);
}
void launch_concat_f32(const float* x, int64_t npix, int Cx, int Cy, int coff, float* y,
                       cudaStream_t s) {
  k_concat_f32<<<gblk(npix * Cx), 256, 0, s>>>(x, npix, Cx, Cy, coff, y);
}
void launch_softmax_f32(const float* x, int64_t rows, int C, float* y, cudaStream_t s) {
  k_softmax_f32<<<(int)((rows * 32 + 255) / 256), 256, 0, s>>>(x, rows, C, y);
}

}  // namespace ptq
