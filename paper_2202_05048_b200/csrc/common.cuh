// Shared device helpers for the ptq_b200 kernels (sm_100a only).
//
// Exact-arithmetic contract: every fp64 step that the
// reference performs in numpy is evaluated here in the same order with
// explicit round-to-nearest intrinsics (__dmul_rn/__dadd_rn/__ddiv_rn), which
// nvcc never contracts into FMAs.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "ptq_b200 kernels target sm_100a only (compile with -gencode arch=compute_100a,code=sm_100a)"
#endif

#define PTQ_QMIN (-128)
#define PTQ_QMAX 127
#define PTQ_NBINS 2048
#define PTQ_LEVELS 128
#define PTQ_NWIN (PTQ_NBINS - PTQ_LEVELS + 1)

namespace ptq {

// ---------------------------------------------------------------- rounding
// RHA = sign(x) * floor(|x| + 0.5)   (ref schemes.py:61-64)
__host__ __device__ __forceinline__ double rha(double x) {
#ifdef __CUDA_ARCH__
  double a = floor(__dadd_rn(fabs(x), 0.5));
#else
  double a = floor(fabs(x) + 0.5);
#endif
  return x > 0.0 ? a : (x < 0.0 ? -a : 0.0);
}

// RHU = floor(x + 0.5)   (ref intexec.py:67-69)
__device__ __forceinline__ double rhu(double x) { return floor(__dadd_rn(x, 0.5)); }

__host__ __device__ __forceinline__ int clip8(double v) {
  return v < PTQ_QMIN ? PTQ_QMIN : (v > PTQ_QMAX ? PTQ_QMAX : (int)v);
}
__host__ __device__ __forceinline__ int clip8i(long long v) {
  return v < PTQ_QMIN ? PTQ_QMIN : (v > PTQ_QMAX ? PTQ_QMAX : (int)v);
}
__host__ __device__ __forceinline__ long long clip32(long long v) {
  const long long lo = -2147483648LL, hi = 2147483647LL;
  return v < lo ? lo : (v > hi ? hi : v);
}

// quantize one value: clip(RHA(x64 / s64 + zp), -128, 127)   (ref schemes.py:145-150)
__device__ __forceinline__ int quant1(float x, double s64, double zp64) {
  return clip8(rha(__dadd_rn(__ddiv_rn((double)x, s64), zp64)));
}

// Same result as quant1 with a multiply by r = fl(1/s) instead of the division: the
// fast value is within a few ulps of the reference's fl(fl(x/s) + zp), so whenever it is
// farther than that from a half-integer both round (RHA) identically; otherwise (rare)
// fall back to the exact division.
__device__ __forceinline__ int quant1_fast(float x, double r, double s64, double zp64) {
  const double t = __dadd_rn(__dmul_rn((double)x, r), zp64);
  const double a = fabs(t);
  const double fr = __dsub_rn(a, floor(a));
  if (fabs(fr - 0.5) > 1e-14 * (a + 1.0)) {
    const double q = floor(__dadd_rn(a, 0.5));
    return clip8(t < 0.0 ? -q : q);
  }
  return quant1(x, s64, zp64);
}

// quant1 on the fp32 pipe with an exactness guard: t32 = fma(x, fl32(1/s), zp) is within
// 2^-23 (2|t| + |zp|) of the reference's fl(fl(x/s) + zp).  When t32 is farther than that
// from a half-integer, RHA of the reference value equals round-to-nearest of t32 (the
// half-way tie rule never applies), and saturation follows from the clamp.  Otherwise
// (rare) the exact fp64 path.  Returns the unclamped code (callers saturate).
__device__ __forceinline__ int quant1_f32g_raw(float x, float r32, float zf, double r64, double s64, double z64) {
  const float t = __fmaf_rn(x, r32, zf);
  const float r = rintf(t);
  const float lim = __fmaf_rn(-3.0e-7f, fabsf(t), 0.4999f);   // 0.5 - margin
  if (fabsf(__fsub_rn(t, r)) < lim) return (int)r;           // exact conversion (|r| < 2^24)
  if (fabsf(t) > 300.0f) return t > 0.0f ? PTQ_QMAX : PTQ_QMIN;
  return quant1_fast(x, r64, s64, z64);
}
__device__ __forceinline__ int quant1_f32g(float x, float r32, float zf, double r64, double s64, double z64) {
  const int q = quant1_f32g_raw(x, r32, zf, r64, s64, z64);
  return q < PTQ_QMIN ? PTQ_QMIN : (q > PTQ_QMAX ? PTQ_QMAX : q);
}

// Four values through the fp32 quantizer with magic-number rounding (no conversion pipe):
// t = fma(x, fl32(1/s), zp) is within 2^-23 (2|t| + |zp|) of the reference's fl(fl(x/s) + zp);
// rm = t + 1.5*2^23 rounds to nearest (|t| < 2^22) and holds the integer in its low mantissa
// bits.  Whenever t is farther than 2e-4 from a half-integer (|t| <= 600: the approximation error
// is < 1.7e-4), round-to-nearest of t equals the reference's RHA of its own value; otherwise
// `bad` is set and the caller recomputes the four values exactly (quant1_f32g).  Saturation is a
// clamp of rm to [M - 128, M + 127]; the low bytes of the four words are the codes.
__device__ __forceinline__ uint32_t quant4_magic(float x0, float x1, float x2, float x3, float r32, float zf,
                                                 float lo, bool& bad) {
  const float M = 12582912.0f;
  const float xs[4] = {x0, x1, x2, x3};
  uint32_t w[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float t = __fmaf_rn(xs[j], r32, zf);
    float rm = __fadd_rn(t, M);
    const float d = fabsf(__fsub_rn(t, __fsub_rn(rm, M)));
    bad |= !(d < 0.4998f) && !(fabsf(t) > 600.0f);   // far outside: saturates either way
    rm = fminf(fmaxf(rm, M + lo), M + 127.0f);
    w[j] = __float_as_uint(rm);
  }
  return __byte_perm(__byte_perm(w[0], w[1], 0x0040), __byte_perm(w[2], w[3], 0x0040), 0x5410);
}

// 4 int32 -> 4 saturated int8 codes in one word (byte j = x_j)
__device__ __forceinline__ uint32_t pack4_sat(int x0, int x1, int x2, int x3) {
  uint32_t hi, out;
  asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, 0;" : "=r"(hi) : "r"(x3), "r"(x2));
  asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, %3;" : "=r"(out) : "r"(x1), "r"(x0), "r"(hi));
  return out;
}

// requantize an int32-clipped accumulator: clip(RHU(acc * m) + zp)   (ref intexec.py:72-85)
__device__ __forceinline__ int requant1(long long acc, double m, int zp) {
  return clip8(rhu(__dmul_rn((double)acc, m)) + (double)zp);
}

// ---------------------------------------------------------------- scheme params
// (scale as float32, zero point) for a (vmin, vmax) range; ref schemes.py:81-131.
// scheme: 0 Asymmetric, 1 Symmetric, 2 SymmetricUint8, 3 SymmetricPower2.
__host__ __device__ inline void params_for_range(int scheme, double vmin, double vmax,
                                                 float* scale, int* zp) {
  double max_abs = fabs(vmin) > fabs(vmax) ? fabs(vmin) : fabs(vmax);
  auto sym = [&](double m, float* s, int* z) {
    if (m == 0.0) { *s = 1.0f; *z = 0; return; }
#ifdef __CUDA_ARCH__
    *s = (float)__ddiv_rn(fabs(m), 127.0);
#else
    *s = (float)(fabs(m) / 127.0);
#endif
    *z = 0;
  };
  if (scheme == 0) {
    double lo = vmin < 0.0 ? vmin : 0.0, hi = vmax > 0.0 ? vmax : 0.0;
    if (lo == hi) { *scale = 1.0f; *zp = 0; return; }
#ifdef __CUDA_ARCH__
    double s64 = __ddiv_rn(__dsub_rn(hi, lo), 255.0);
    double q = __ddiv_rn(lo, s64);
#else
    double s64 = (hi - lo) / 255.0;
    double q = lo / s64;
#endif
    *scale = (float)s64;
    *zp = (int)(-rha(q)) - 128;
  } else if (scheme == 1) {
    sym(max_abs, scale, zp);
  } else if (scheme == 2) {
    if (vmin < 0.0) { sym(max_abs, scale, zp); return; }
    if (max_abs == 0.0) { *scale = 1.0f; *zp = -128; return; }
#ifdef __CUDA_ARCH__
    *scale = (float)__ddiv_rn(fabs(max_abs), 255.0);
#else
    *scale = (float)(fabs(max_abs) / 255.0);
#endif
    *zp = -128;
  } else {
    float s; int z;
    sym(max_abs, &s, &z);
    // ceil_log2 via frexp on the stored fp32 scale (ref schemes.py:67-72, :114-117)
    int e;
    double m = frexp((double)s, &e);
    int k = (m == 0.5) ? e - 1 : e;
    *scale = (float)ldexp(1.0, k);
    *zp = 0;
  }
}

// ---------------------------------------------------------------- numpy linspace edge
// e[k] = fl(k * fl(delta / 2048)) + lo  with e[2048] = hi  (numpy function_base.py linspace)
__host__ __device__ __forceinline__ double hist_edge(double lo, double hi, int k) {
  if (k >= PTQ_NBINS) return hi;
#ifdef __CUDA_ARCH__
  double delta = __dsub_rn(hi, lo);
  double step = __ddiv_rn(delta, (double)PTQ_NBINS);
  double y = (step == 0.0) ? __dmul_rn(__ddiv_rn((double)k, (double)PTQ_NBINS), delta)
                           : __dmul_rn((double)k, step);
  return __dadd_rn(y, lo);
#else
  double delta = hi - lo;
  double step = delta / PTQ_NBINS;
  double y = (step == 0.0) ? ((double)k / PTQ_NBINS) * delta : (double)k * step;
  return y + lo;
#endif
}

// ---------------------------------------------------------------- ordered float atomics
__device__ __forceinline__ unsigned int f2ord(float f) {
  unsigned int u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(unsigned int u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

// ---------------------------------------------------------------- PTX: barriers / async copies
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// 16-byte shared-memory load / store by 32-bit shared address
__device__ __forceinline__ int4 lds128(uint32_t a) {
  int4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, int4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, 10000000;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// arrive on `bar` once every cp.async issued so far by this thread has landed
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// 16-byte global->shared async copy; src_bytes < 16 zero-fills the rest
__device__ __forceinline__ void cp_async16(void* dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes)
               : "memory");
}
// bulk copy global->shared completing on an mbarrier (TMA bulk path, SASS UBLKCP)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// 2-D TMA tile load (box given by the tensor map) completing on an mbarrier
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// L2 prefetch of one tensor-map box (no shared-memory destination, no barrier)
__device__ __forceinline__ void tma_prefetch_2d(const void* tmap, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(tmap), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}
// bulk prefetch of [src, src + bytes) into L2 (bytes a multiple of 16)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// 2-D TMA tile store shared -> global (bulk async group of the issuing thread)
__device__ __forceinline__ void tma_store_2d(const void* tmap, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(tmap),
               "r"(c0), "r"(c1), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// wait until at most N bulk groups of this thread still read shared memory
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

}  // namespace ptq
