// F1: calibration reductions.  F2: KL-divergence threshold sweep.
//
// F1 restates the reference's two-pass calibration
// (/root/reference/pkg/src/ptqtune/calibration.py:57-106): exact fp32
// min/max per tensor, then np.histogram(x.astype(f64), 2048, range=(lo, hi))
// with numpy's uniform-bin index rule (numpy lib/_histograms_impl.py: fp64
// (x-lo)/(hi-lo)*2048, truncate, one-step decrement/increment fixup against
// the np.linspace edges).  lo == hi puts every value in bin 0 (:86-87).
//
// F2 restates clip_range_kl / _window_kl (clipping.py:38-86): 1921 candidate
// windows per histogram, one CTA per (histogram, window).  The KL sum is
// accumulated over the compacted P>0 sequence in numpy's pairwise-summation
// order (8 strided accumulators per <=128-element leaf, halving splits rounded
// to multiples of 8), so it is bit-identical to numpy whenever the log values
// agree; the host re-ranks near-ties with numpy (evaluator.py).
#include <atomic>

#include "common.cuh"
#include "kernels.h"

namespace ptq {

// ---------------------------------------------------------------- F1a: per-image min/max
// x: [n_img][elems] fp32.  out_ord: [n_img][2] ordered-uint (min, max), pre-initialised.
__global__ void k_minmax_per_image(const float* __restrict__ x, int64_t elems,
                                   unsigned int* __restrict__ out_ord) {
  const int img = blockIdx.y;
  const float* p = x + (int64_t)img * elems;
  float lo = INFINITY, hi = -INFINITY;
  // 16-byte vector body when the per-image slice is 16B aligned
  const bool vec = ((((uintptr_t)p) & 15) == 0);
  int64_t n4 = vec ? (elems >> 2) : 0;
  const float4* p4 = reinterpret_cast<const float4*>(p);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 v = __ldg(p4 + i);
    lo = fminf(lo, fminf(fminf(v.x, v.y), fminf(v.z, v.w)));
    hi = fmaxf(hi, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
  }
  for (int64_t i = (n4 << 2) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < elems;
       i += (int64_t)gridDim.x * blockDim.x) {
    float v = __ldg(p + i);
    lo = fminf(lo, v);
    hi = fmaxf(hi, v);
  }
  // warp shuffle reduction, then one atomic per warp
  for (int o = 16; o > 0; o >>= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  __shared__ float slo[32], shi[32];
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { slo[w] = lo; shi[w] = hi; }
  __syncthreads();
  if (w == 0) {
    int nw = blockDim.x >> 5;
    lo = l < nw ? slo[l] : INFINITY;
    hi = l < nw ? shi[l] : -INFINITY;
    for (int o = 16; o > 0; o >>= 1) {
      lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (l == 0 && elems > 0) {
      atomicMin(out_ord + 2 * img, f2ord(lo));
      atomicMax(out_ord + 2 * img + 1, f2ord(hi));
    }
  }
}

__global__ void k_fill_u32(unsigned int* p, int64_t n, unsigned int a, unsigned int b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (i & 1) ? b : a;
}

// per-cache reduction of per-image (min,max): slots[j] are image slots of the cache
__global__ void k_minmax_reduce_cache(const unsigned int* __restrict__ per_img, int n_tensors,
                                      int n_img_total, const int* __restrict__ slots, int n_slots,
                                      float* __restrict__ ranges /*[T][2]*/) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_tensors) return;
  if (n_slots == 0) {  // identity element for the cross-rank MIN/MAX allreduce
    ranges[2 * t] = INFINITY;
    ranges[2 * t + 1] = -INFINITY;
    return;
  }
  unsigned int lo = 0xffffffffu, hi = 0u;
  for (int j = 0; j < n_slots; ++j) {
    const unsigned int* q = per_img + ((int64_t)t * n_img_total + slots[j]) * 2;
    lo = min(lo, q[0]);
    hi = max(hi, q[1]);
  }
  ranges[2 * t] = ord2f(lo);
  ranges[2 * t + 1] = ord2f(hi);
}

// ---------------------------------------------------------------- F1b: histogram
// numpy uniform-bin index for x in [lo, hi] (lo < hi), exact.
__device__ __forceinline__ int np_bin(double x, double lo, double hi, double denom) {
  double f = __dmul_rn(__ddiv_rn(__dsub_rn(x, lo), denom), (double)PTQ_NBINS);
  int idx = (int)f;
  if (idx >= PTQ_NBINS) idx = PTQ_NBINS - 1;
  if (x < hist_edge(lo, hi, idx)) idx -= 1;
  if (idx != PTQ_NBINS - 1 && x >= hist_edge(lo, hi, idx + 1)) idx += 1;
  return idx;
}

// Fast path: an approximate position fe = (x - lo) * fl(2048 / (hi - lo)) is within a
// few ulps of numpy's f-index, and numpy's edges are within a few ulps of the exact
// bin edges.  When fe's fractional part keeps a margin `eps` (in bin units) from both
// neighbouring edges, numpy's truncation and both fixups provably leave floor(fe)
// unchanged, so only near-edge values pay for the exact division + edge checks.
__device__ __forceinline__ int np_bin_fast(double x, double lo, double hi, double denom,
                                           double rc, double eps) {
  const double fe = __dmul_rn(__dsub_rn(x, lo), rc);
  const int k = (int)fe;
  const double frac = __dsub_rn(fe, (double)k);
  if (k < PTQ_NBINS && frac > eps && frac < 1.0 - eps) return k;
  return np_bin(x, lo, hi, denom);
}

// fp32 pre-filter: fe32 = fl32(fl32(x - lo) * fl32(2048 / (hi - lo))) is within
// 3 * 2^-24 * 2048 = 3.7e-4 bins of the true position (three relative fp32 roundings on a
// value <= 2048; numpy's own fp64 position and edges are 1e-12 away); when its fractional
// part keeps a 5e-4 margin from both neighbouring integers (|frac - 0.5| < 0.4995) the bin is
// settled on the fp32 pipe, otherwise np_bin_fast decides in fp64.  A position at or past 2048
// (x at hi) has frac ~ 0 and takes the fp64 path.
// floor of the fp32 position without the conversion pipe: fe + 1.5*2^23 rounded down holds
// floor(fe) in its low mantissa bits (-2^22 < fe < 2^22); the fractional part is exact
__device__ __forceinline__ int f32_floor_frac(float fe, float& frac) {
  const float rm = __fadd_rd(fe, 12582912.0f);
  frac = __fsub_rn(fe, __fsub_rn(rm, 12582912.0f));
  return (int)(__float_as_uint(rm) - 0x4B400000u);
}
__device__ __forceinline__ int np_bin_f32g(float x, float lo32, float rc32, double lo, double hi, double denom,
                                           double rc, double eps) {
  const float fe = __fmul_rn(__fsub_rn(x, lo32), rc32);
  float frac;
  const int k = f32_floor_frac(fe, frac);
  if (fabsf(__fsub_rn(frac, 0.5f)) < 0.4995f) return k;
  return np_bin_fast((double)x, lo, hi, denom, rc, eps);
}

// x: [n_img_total][elems]; slots: image slots of this cache; range: lo, hi (fp32 values).
// counts: [2048] int64 (accumulated).  One shared sub-histogram per warp keeps the atomics
// warp-private; exact zeros (post-ReLU tensors pile up there) go straight to the zero bin.
#ifndef HIST_COPIES
#define HIST_COPIES 8              // one private sub-histogram per warp: no cross-warp atomics
#endif
#define HIST_BLOCKS_PER_SM (HIST_COPIES == 8 ? 3 : 8)
__global__ void __launch_bounds__(256) k_histogram(const float* __restrict__ x, int64_t elems,
                                                   const int* __restrict__ slots, int n_slots,
                                                   const float* __restrict__ range,
                                                   unsigned long long* __restrict__ counts) {
  extern __shared__ unsigned int sh[];       // HIST_COPIES sub-histograms, one per warp
  for (int i = threadIdx.x; i < HIST_COPIES * PTQ_NBINS; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const double lo = (double)range[0], hi = (double)range[1];
  const double denom = __dsub_rn(hi, lo);
  const bool degenerate = !(lo < hi);
  const double rc = degenerate ? 0.0 : __ddiv_rn((double)PTQ_NBINS, denom);
  const double mag = fmax(fabs(lo), fabs(hi));
  const double eps = degenerate ? 1.0 : 16.0 * 2.220446049250313e-16 * mag * rc + 1e-9;
  if (degenerate) {                       // lo == hi: every value lands in bin 0 (:86-87)
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(counts, (unsigned long long)(elems * n_slots));
    return;
  }
  const int z0 = (lo <= 0.0 && 0.0 <= hi) ? np_bin(0.0, lo, hi, denom) : -1;
  unsigned int* my = sh + ((threadIdx.x >> 5) % HIST_COPIES) * PTQ_NBINS;
  unsigned int zc = 0;
  const float lo32 = range[0], rc32 = (float)rc;
  auto put = [&](float v) {
    if (v == 0.0f && z0 >= 0) ++zc;
    else atomicAdd(&my[np_bin_f32g(v, lo32, rc32, lo, hi, denom, rc, eps)], 1u);
  };
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // every per-image slice is 16-byte aligned (elems % 4 == 0) except for tiny tensors:
  // flatten (image, float4) work items so small tensors still spread over all blocks
  const bool vec = (elems & 3) == 0 && ((((uintptr_t)x) & 15) == 0);
  if (vec) {
    // (image, float4) cursors advanced by the grid stride with 32-bit adds (the flat index
    // split costs one 64-bit division per thread, not one per load)
    const int64_t nv = elems >> 2;
    const unsigned nvu = (unsigned)nv;           // < 2^31: r + sr never wraps
    const int sj = (int)(stride / nv);
    const unsigned sr = (unsigned)(stride % nv);
    const int64_t w0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int j = (int)(w0 / nv);
    unsigned r = (unsigned)(w0 % nv);
    auto adv = [&](int& jj, unsigned& rr) {
      rr += sr;
      jj += sj;
      if (rr >= nvu) { rr -= nvu; ++jj; }
    };
    auto at = [&](int jj, unsigned rr) -> float4 {
      return __ldg(reinterpret_cast<const float4*>(x + (int64_t)__ldg(slots + jj) * elems) + rr);
    };
    // four loads in flight per thread, then 16 values binned without branches: the fp32
    // bin and a needs-fp64 mask for all 16, one (rarely taken) branch for the near-edge
    // values, then 16 unconditional shared atomics
    const bool zero_in = z0 >= 0;
    for (;;) {
      int j1 = j, j2, j3;
      unsigned r1 = r, r2, r3;
      adv(j1, r1); j2 = j1; r2 = r1; adv(j2, r2); j3 = j2; r3 = r2; adv(j3, r3);
      if (j3 >= n_slots) break;
      const float4 q0 = at(j, r), q1 = at(j1, r1), q2 = at(j2, r2), q3 = at(j3, r3);
      j = j3; r = r3;
      adv(j, r);
      const float v[16] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w,
                           q2.x, q2.y, q2.z, q2.w, q3.x, q3.y, q3.z, q3.w};
      int k[16];
      unsigned slow = 0;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const float fe = __fmul_rn(__fsub_rn(v[e], lo32), rc32);
        float frac;
        k[e] = f32_floor_frac(fe, frac);
        const bool ok = fabsf(__fsub_rn(frac, 0.5f)) < 0.4995f;
        const bool z = zero_in && v[e] == 0.0f;   // exact zeros: the zero bin, no fp64
        if (z) k[e] = z0;
        slow |= (unsigned)(!ok && !z) << e;
      }
      if (slow) {
#pragma unroll
        for (int e = 0; e < 16; ++e)
          if (slow & (1u << e)) k[e] = np_bin_fast((double)v[e], lo, hi, denom, rc, eps);
      }
#pragma unroll
      for (int e = 0; e < 16; ++e)
        atomicAdd(&my[k[e]], 1u);      // ATOMS.POPC.INC: same-address lanes aggregate
    }
    for (; j < n_slots; adv(j, r)) {
      const float4 v = at(j, r);
      put(v.x); put(v.y); put(v.z); put(v.w);
    }
  } else {                                // scalar path (element count not a multiple of 4)
    const int64_t total = elems * n_slots;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += stride) {
      const int j = (int)(i / elems);
      put(__ldg(x + (int64_t)slots[j] * elems + (i - (int64_t)j * elems)));
    }
  }
  for (int d = 16; d; d >>= 1) zc += __shfl_xor_sync(0xffffffffu, zc, d);
  if ((threadIdx.x & 31) == 0 && zc) atomicAdd(&sh[z0], zc);
  __syncthreads();
  for (int i = threadIdx.x; i < PTQ_NBINS; i += blockDim.x) {
    unsigned int t = 0;
#pragma unroll
    for (int c = 0; c < HIST_COPIES; ++c) t += sh[c * PTQ_NBINS + i];
    if (t) atomicAdd(counts + i, (unsigned long long)t);
  }
}

// ---------------------------------------------------------------- F1b, batched
// All histograms of a calibration in one launch: the (cache, tensor) items are cut into
// chunks of HIST_CHUNK values of their (image slot, element) space; a persistent grid walks the
// chunk list, bins each chunk into the block's private shared sub-histograms and flushes them
// to the item's int64 counts.  Small tensors no longer cost a launch each (366 launches per
// calibration before), and every chunk keeps all SMs busy.
constexpr int64_t HIST_CHUNK = 1 << 20;
__global__ void __launch_bounds__(256) k_histogram_multi(const HistItem* __restrict__ items, int n_items,
                                                         int64_t n_chunks) {
  extern __shared__ unsigned int sh[];
  unsigned int* my = sh + ((threadIdx.x >> 5) % HIST_COPIES) * PTQ_NBINS;
  for (int64_t ch = blockIdx.x; ch < n_chunks; ch += gridDim.x) {
    // item of this chunk: binary search over the chunk prefix
    int lo_i = 0, hi_i = n_items - 1;
    while (lo_i < hi_i) {
      const int mid = (lo_i + hi_i + 1) >> 1;
      if (items[mid].chunk0 <= ch) lo_i = mid; else hi_i = mid - 1;
    }
    const HistItem it = items[lo_i];
    const int64_t total = it.elems * it.n_slots;
    const int64_t f0 = (ch - it.chunk0) * HIST_CHUNK;
    const int64_t f1 = f0 + HIST_CHUNK < total ? f0 + HIST_CHUNK : total;
    const double lo = (double)it.range[0], hi = (double)it.range[1];
    if (!(lo < hi)) {                                // lo == hi: every value lands in bin 0 (:86-87)
      if (threadIdx.x == 0) atomicAdd(it.counts, (unsigned long long)(f1 - f0));
      continue;
    }
    for (int i = threadIdx.x; i < HIST_COPIES * PTQ_NBINS; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const double denom = __dsub_rn(hi, lo);
    const double rc = __ddiv_rn((double)PTQ_NBINS, denom);
    const double mag = fmax(fabs(lo), fabs(hi));
    const double eps = 16.0 * 2.220446049250313e-16 * mag * rc + 1e-9;
    const int z0 = (lo <= 0.0 && 0.0 <= hi) ? np_bin(0.0, lo, hi, denom) : -1;
    const float lo32 = it.range[0], rc32 = (float)rc;
    unsigned int zc = 0;
    auto put = [&](float v) {
      if (v == 0.0f && z0 >= 0) ++zc;
      else atomicAdd(&my[np_bin_f32g(v, lo32, rc32, lo, hi, denom, rc, eps)], 1u);
    };
    const bool vec = (it.elems & 3) == 0 && ((((uintptr_t)it.x) & 15) == 0);
    if (vec) {
      // float4 index u of the chunk -> (slot j, float4 r) cursors advanced by the block stride
      const int64_t nv = it.elems >> 2;
      const unsigned nvu = (unsigned)nv;
      const int64_t u0 = (f0 >> 2) + threadIdx.x, u1 = f1 >> 2;
      const int sj = (int)(blockDim.x / nv);
      const unsigned sr = (unsigned)(blockDim.x % nv);
      int j = (int)(u0 / nv);
      unsigned r = (unsigned)(u0 % nv);
      int64_t u = u0;
      auto adv = [&](int& jj, unsigned& rr) {
        rr += sr;
        jj += sj;
        if (rr >= nvu) { rr -= nvu; ++jj; }
      };
      auto at = [&](int jj, unsigned rr) -> float4 {
        return __ldg(reinterpret_cast<const float4*>(it.x + (int64_t)__ldg(it.slots + jj) * it.elems) + rr);
      };
      const bool zero_in = z0 >= 0;
      const int64_t st = blockDim.x;
      for (; u + 3 * st < u1; u += 4 * st) {
        int j1 = j, j2, j3;
        unsigned r1 = r, r2, r3;
        adv(j1, r1); j2 = j1; r2 = r1; adv(j2, r2); j3 = j2; r3 = r2; adv(j3, r3);
        const float4 q0 = at(j, r), q1 = at(j1, r1), q2 = at(j2, r2), q3 = at(j3, r3);
        j = j3; r = r3;
        adv(j, r);
        const float v[16] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w,
                             q2.x, q2.y, q2.z, q2.w, q3.x, q3.y, q3.z, q3.w};
        int k[16];
        unsigned slow = 0;
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float fe = __fmul_rn(__fsub_rn(v[e], lo32), rc32);
          float frac;
          k[e] = f32_floor_frac(fe, frac);
          const bool ok = fabsf(__fsub_rn(frac, 0.5f)) < 0.4995f;
          const bool z = zero_in && v[e] == 0.0f;
          if (z) k[e] = z0;
          slow |= (unsigned)(!ok && !z) << e;
        }
        if (slow) {
#pragma unroll
          for (int e = 0; e < 16; ++e)
            if (slow & (1u << e)) k[e] = np_bin_fast((double)v[e], lo, hi, denom, rc, eps);
        }
#pragma unroll
        for (int e = 0; e < 16; ++e) atomicAdd(&my[k[e]], 1u);
      }
      for (; u < u1; u += st, adv(j, r)) {
        const float4 v = at(j, r);
        put(v.x); put(v.y); put(v.z); put(v.w);
      }
    } else {
      for (int64_t i = f0 + threadIdx.x; i < f1; i += blockDim.x) {
        const int jj = (int)(i / it.elems);
        put(__ldg(it.x + (int64_t)it.slots[jj] * it.elems + (i - (int64_t)jj * it.elems)));
      }
    }
    for (int d = 16; d; d >>= 1) zc += __shfl_xor_sync(0xffffffffu, zc, d);
    if ((threadIdx.x & 31) == 0 && zc) atomicAdd(&sh[z0], zc);
    __syncthreads();
    for (int i = threadIdx.x; i < PTQ_NBINS; i += blockDim.x) {
      unsigned int t = 0;
#pragma unroll
      for (int c = 0; c < HIST_COPIES; ++c) t += sh[c * PTQ_NBINS + i];
      if (t) atomicAdd(it.counts + i, (unsigned long long)t);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- F2: KL sweep
// Per histogram h we precompute (k_kl_prep): cum[j] = sum counts[0..j] (fp64 of exact
// integers: any summation order gives the same value below 2^53), nzc[j] = #(counts[0..j] > 0),
// logc[j] = log(counts[j]) (0 where empty).  One 256-thread block per histogram: 8 bins per
// thread, a block scan of the per-thread sums, logs in parallel.
__global__ void __launch_bounds__(256) k_kl_prep(const long long* __restrict__ counts, int n_hist,
                                                 double* __restrict__ cum, int* __restrict__ nzc,
                                                 double* __restrict__ logc) {
  const int h = blockIdx.x, t = threadIdx.x;
  if (h >= n_hist) return;
  __shared__ long long ps[256];
  __shared__ int pz[256];
  const long long* c = counts + (int64_t)h * PTQ_NBINS;
  long long v[8], s = 0;
  int z = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    v[j] = c[t * 8 + j];
    s += v[j];
    z += v[j] > 0;
  }
  ps[t] = s;
  pz[t] = z;
  __syncthreads();
  for (int d = 1; d < 256; d <<= 1) {                 // inclusive Hillis-Steele scan
    const long long a = t >= d ? ps[t - d] : 0;
    const int b = t >= d ? pz[t - d] : 0;
    __syncthreads();
    ps[t] += a;
    pz[t] += b;
    __syncthreads();
  }
  long long run = ps[t] - s;
  int nz = pz[t] - z;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int k = t * 8 + j;
    run += v[j];
    nz += v[j] > 0;
    cum[(int64_t)h * PTQ_NBINS + k] = (double)run;
    nzc[(int64_t)h * PTQ_NBINS + k] = nz;
    logc[(int64_t)h * PTQ_NBINS + k] = v[j] > 0 ? log((double)v[j]) : 0.0;
  }
}

// numpy pairwise sum of t[0..n) (numpy loops_utils.h pairwise_sum, PW_BLOCKSIZE 128),
// evaluated from the per-leaf partial sums computed in parallel.
__device__ double pw_leaf(const double* t, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, t[i]);
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = t[j];
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], t[i + j]);
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, t[i]);
  return res;
}

// leaves of the pairwise recursion over [0, n): enumerate in order
__device__ int pw_leaves(int n, int* lstart, int* llen) {
  // iterative DFS with an explicit stack; depth <= 6 for n <= 2048
  int stack_s[16], stack_n[16], sp = 0, cnt = 0;
  stack_s[sp] = 0; stack_n[sp] = n; ++sp;
  while (sp) {
    --sp;
    int s = stack_s[sp], m = stack_n[sp];
    if (m <= 128) { lstart[cnt] = s; llen[cnt] = m; ++cnt; continue; }
    int m2 = m / 2; m2 -= m2 % 8;
    // push right then left so left is processed first
    stack_s[sp] = s + m2; stack_n[sp] = m - m2; ++sp;
    stack_s[sp] = s; stack_n[sp] = m2; ++sp;
  }
  return cnt;
}

__device__ double pw_combine(int n, const double* leafsum, int* leaf_idx) {
  if (n <= 128) return leafsum[(*leaf_idx)++];
  int m2 = n / 2; m2 -= m2 % 8;
  double a = pw_combine(m2, leafsum, leaf_idx);
  double b = pw_combine(n - m2, leafsum, leaf_idx);
  return __dadd_rn(a, b);
}

// grid: (1921 windows, n_hist); block 128 threads (one per quantization level / group)
// out: kl[h][w] (inf when infeasible or not applicable)
__global__ void __launch_bounds__(128) k_kl_sweep(const long long* __restrict__ counts,
                                                  const float* __restrict__ ranges,
                                                  const double* __restrict__ cum_all,
                                                  const int* __restrict__ nzc_all,
                                                  const double* __restrict__ logc_all,
                                                  double* __restrict__ kl_out) {
  __shared__ double terms[PTQ_NBINS];
  __shared__ int gcount[PTQ_LEVELS + 1];
  __shared__ double leafsum[40];
  __shared__ int lstart[40], llen[40], nleaves;
  __shared__ int infeasible, wtot[4];

  const int w = blockIdx.x, h = blockIdx.y, g = threadIdx.x;
  const int i = w + PTQ_LEVELS;                    // window width in bins
  const long long* c = counts + (int64_t)h * PTQ_NBINS;
  const double* cum = cum_all + (int64_t)h * PTQ_NBINS;
  const int* nzc = nzc_all + (int64_t)h * PTQ_NBINS;
  const double* logc = logc_all + (int64_t)h * PTQ_NBINS;
  const double lo = (double)ranges[2 * h], hi = (double)ranges[2 * h + 1];
  const double total = cum[PTQ_NBINS - 1];
  double* out = kl_out + (int64_t)h * PTQ_NWIN + w;
  if (!(lo < hi) || !(total > 0.0)) {              // clip_range_kl early returns (:63-69)
    if (g == 0) *out = INFINITY;
    return;
  }
  const bool is_signed = lo < 0.0;
  int zero_bin = 0;
  if (is_signed) {
    double width = __ddiv_rn(__dsub_rn(hi, lo), (double)PTQ_NBINS);
    zero_bin = (int)__ddiv_rn(-lo, width);         // int((0.0 - lo) / width), lo < 0
  }
  int start = 0;
  if (is_signed) {
    start = zero_bin - i / 2;
    start = start < 0 ? 0 : start;
    start = start > PTQ_NBINS - i ? PTQ_NBINS - i : start;
  }
  const int end = start + i;
  // merged reference P: outliers folded into the window edge bins (:77-80)
  const double ref_first = (double)c[start] + (start > 0 ? cum[start - 1] : 0.0);
  const double ref_last_add = __dsub_rn(total, cum[end - 1]);
  // group layout: m = i // 128, group g covers [g*m, (g+1)*m), last absorbs remainder
  const int m = i / PTQ_LEVELS;
  const int gs = g * m, ge = (g == PTQ_LEVELS - 1) ? i : (g + 1) * m;
  auto refv = [&](int j) -> double {               // ref value at window-relative bin j
    double v = (double)c[start + j];
    if (j == 0) v = ref_first;
    if (j == i - 1) v = __dadd_rn(v, ref_last_add);
    return v;
  };
  // unmerged group sum (exact integer arithmetic in fp64) and P>0 count
  double gsum = __dsub_rn(cum[start + ge - 1], (start + gs > 0) ? cum[start + gs - 1] : 0.0);
  int gnz = nzc[start + ge - 1] - ((start + gs > 0) ? nzc[start + gs - 1] : 0);
  // the two edge bins use the merged flags
  if (gs == 0) gnz += (refv(0) > 0.0) - (c[start] > 0);
  if (ge == i && i - 1 != 0) gnz += (refv(i - 1) > 0.0) - (c[start + i - 1] > 0);
  if (g == 0) infeasible = 0;
  gcount[g + 1] = gnz;
  __syncthreads();
  if (gnz > 0 && gsum == 0.0) infeasible = 1;      // Q = 0 under P > 0 -> inf (:49-50)
  // exclusive scan of gnz over the 128 groups: warp shuffle scans + the 4 warp totals
  {
    const int lane = g & 31, wi = g >> 5;
    int x = gnz;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    if (lane == 31) wtot[wi] = x;
    __syncthreads();
    int off = 0;
    for (int w2 = 0; w2 < wi; ++w2) off += wtot[w2];
    gcount[g + 1] = x + off;                         // inclusive prefix at g + 1
    if (g == 0) gcount[0] = 0;
  }
  __syncthreads();
  if (infeasible) {
    if (g == 0) *out = INFINITY;
    return;
  }
  // terms p * (log p - log q) written at their compacted positions
  if (gnz > 0) {
    double q = __ddiv_rn(gsum, (double)gnz);
    double lq = log(q);
    int pos = gcount[g];
    for (int j = gs; j < ge; ++j) {
      double p = refv(j);
      if (p > 0.0) {
        bool edge = (j == 0) || (j == i - 1);
        double lp = edge ? log(p) : logc[start + j];
        terms[pos++] = __dmul_rn(p, __dsub_rn(lp, lq));
      }
    }
  }
  const int n = gcount[PTQ_LEVELS];
  if (g == 0) nleaves = pw_leaves(n, lstart, llen);
  __syncthreads();
  if (g < nleaves) leafsum[g] = pw_leaf(terms + lstart[g], llen[g]);
  __syncthreads();
  if (g == 0) {
    int li = 0;
    double s = (n == 0) ? 0.0 : __dadd_rn(0.0, pw_combine(n, leafsum, &li));
    *out = __ddiv_rn(s, total);                    // / ref.sum() == total (:52)
  }
}

// ---------------------------------------------------------------- launch wrappers
static inline int nblocks(int64_t n, int t, int cap) {
  int64_t b = (n + t - 1) / t;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}
void launch_fill_minmax(unsigned int* p, int64_t n_pairs, cudaStream_t s) {
  k_fill_u32<<<nblocks(2 * n_pairs, 256, 4096), 256, 0, s>>>(p, 2 * n_pairs, 0xffffffffu, 0u);
}
void launch_minmax_per_image(const float* x, int64_t elems, int n_img, unsigned int* out_ord,
                             cudaStream_t s) {
  int bx = nblocks(elems / 4 + 1, 256, 512);
  int want = (148 * 8 + n_img - 1) / n_img;
  if (bx > want) bx = want < 1 ? 1 : want;
  dim3 g(bx, n_img);
  k_minmax_per_image<<<g, 256, 0, s>>>(x, elems, out_ord);
}
void launch_minmax_reduce_cache(const unsigned int* per_img, int n_tensors, int n_img_total,
                                const int* slots, int n_slots, float* ranges, cudaStream_t s) {
  k_minmax_reduce_cache<<<(n_tensors + 127) / 128, 128, 0, s>>>(per_img, n_tensors, n_img_total,
                                                               slots, n_slots, ranges);
}
void launch_histogram(const float* x, int64_t elems, const int* slots, int n_slots,
                      const float* range, unsigned long long* counts, cudaStream_t s) {
  int64_t total = elems * n_slots;
  constexpr int smem = HIST_COPIES * PTQ_NBINS * 4;
  // per-device function attribute, raised once per device (a failure surfaces as a failed launch)
  static std::atomic<uint64_t> attr{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr.load() & bit) &&
      cudaFuncSetAttribute(k_histogram, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess)
    attr.fetch_or(bit);
  k_histogram<<<nblocks(total, 256, 148 * HIST_BLOCKS_PER_SM), 256, smem, s>>>(x, elems, slots, n_slots, range,
                                                                               counts);
}
int64_t hist_items_chunk0(HistItem* items, int n) {
  int64_t c = 0;
  for (int i = 0; i < n; ++i) {
    items[i].chunk0 = c;
    c += (items[i].elems * items[i].n_slots + HIST_CHUNK - 1) / HIST_CHUNK;
  }
  return c;
}
void launch_histogram_multi(const HistItem* d_items, int n_items, int64_t n_chunks, cudaStream_t s) {
  if (n_items <= 0 || n_chunks <= 0) return;
  constexpr int smem = HIST_COPIES * PTQ_NBINS * 4;
  static std::atomic<uint64_t> attr{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr.load() & bit) &&
      cudaFuncSetAttribute(k_histogram_multi, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess)
    attr.fetch_or(bit);
  const int grid = (int)(n_chunks < 148 * HIST_BLOCKS_PER_SM ? n_chunks : 148 * HIST_BLOCKS_PER_SM);
  k_histogram_multi<<<grid, 256, smem, s>>>(d_items, n_items, n_chunks);
}
// ---------------------------------------------------------------- F2b: percentile clipping
// Extension (not in the reference, which rejects "Percentile": clipping.py:91-92): the
// clipped range of a histogram keeps the central q = pct/100 of its mass.  With N = sum(c),
// cum_i = c_0 + ... + c_i (exact int64):  hi_idx = first i with cum_i >= fl(q N),
// lo_idx = first i with cum_i > fl(fl(1 - q) N);  range = (edge[lo_idx], edge[hi_idx + 1])
// on numpy's linspace edges.  Histograms the KL sweep skips (lo == hi, N == 0) keep (lo, hi).
// One CTA per histogram: 256 threads own 8 consecutive bins each, a block scan of the
// per-thread sums, then each thread scans its bins and offers candidates by atomicMin.
__global__ void __launch_bounds__(256) k_percentile(const long long* __restrict__ counts,
                                                    const float* __restrict__ ranges, double q,
                                                    double* __restrict__ out) {
  __shared__ long long part[256];
  __shared__ int idx[2];
  const int h = blockIdx.x, t = threadIdx.x;
  const long long* c = counts + (int64_t)h * PTQ_NBINS;
  const double lo = (double)ranges[2 * h], hi = (double)ranges[2 * h + 1];
  long long v[8], s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) { v[j] = c[t * 8 + j]; s += v[j]; }
  part[t] = s;
  if (t == 0) { idx[0] = PTQ_NBINS; idx[1] = PTQ_NBINS; }
  __syncthreads();
  for (int d = 1; d < 256; d <<= 1) {                 // inclusive Hillis-Steele scan
    const long long a = t >= d ? part[t - d] : 0;
    __syncthreads();
    part[t] += a;
    __syncthreads();
  }
  const long long total = part[255];
  if (total == 0 || !(lo < hi)) {
    if (t == 0) { out[2 * h] = lo; out[2 * h + 1] = hi; }
    return;
  }
  const double thr_hi = __dmul_rn(q, (double)total);
  const double thr_lo = __dmul_rn(__dsub_rn(1.0, q), (double)total);
  long long cum = part[t] - s;
  bool got_lo = false, got_hi = false;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    cum += v[j];
    const double cd = (double)cum;                   // exact: total < 2^53
    if (!got_lo && cd > thr_lo) { atomicMin(&idx[0], t * 8 + j); got_lo = true; }
    if (!got_hi && cd >= thr_hi) { atomicMin(&idx[1], t * 8 + j); got_hi = true; }
  }
  __syncthreads();
  if (t == 0) {
    const int li = idx[0] < PTQ_NBINS ? idx[0] : PTQ_NBINS - 1;
    const int hj = idx[1] < PTQ_NBINS ? idx[1] : PTQ_NBINS - 1;
    out[2 * h] = hist_edge(lo, hi, li);
    out[2 * h + 1] = hist_edge(lo, hi, hj + 1);
  }
}
void launch_percentile(const long long* counts, const float* ranges, int n_hist, double q, double* out,
                       cudaStream_t s) {
  if (n_hist <= 0) return;
  k_percentile<<<n_hist, 256, 0, s>>>(counts, ranges, q, out);
}

void launch_kl_sweep(const long long* counts, const float* ranges, int n_hist, double* cum,
                     int* nzc, double* logc, double* kl_out, cudaStream_t s) {
  if (n_hist <= 0) return;
  k_kl_prep<<<n_hist, 256, 0, s>>>(counts, n_hist, cum, nzc, logc);
  dim3 g(PTQ_NWIN, n_hist);
  k_kl_sweep<<<g, 128, 0, s>>>(counts, ranges, cum, nzc, logc, kl_out);
}

}  // namespace ptq
