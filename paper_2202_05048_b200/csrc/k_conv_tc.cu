// F4: int8 implicit-GEMM convolution on the 5th-generation tensor cores.
//
// Restates the reference's integer conv/fc branch (/root/reference/pkg/src/
// ptqtune/intexec.py:170-211, _int_conv :95-105): acc = sum (x-zx)(w-zw) with
// zero padding in the shifted domain, + int32 bias, saturate to int32, then
// requantize with m = (sx*sw)/sy and round-half-up, optional relu / residual
// add on codes.  The contraction runs as D[s32] = A[s8] x B[s8] with
//   sum (x-zx)(w-zw) = sum x*w - zw*sum x - zx*sum w + K*zx*zw
// where the halo of the NHWC input holds the zero-point code (so padded taps
// contribute exactly 0), -zx*sum w + K*zx*zw + bias is a per-channel constant
// (EpiParam.cc, computed per config by k_layer_params) and sum x is a
// per-output-pixel term from per-pixel channel sums P (only when some zw != 0).
//
// Persistent, warp-specialised kernel (one CTA per SM, 512 threads = 4 warps per
// SM sub-partition, <= 128 registers each, no spills):
//   warps 0-1   A producers: two GEMM rows (output pixels) per thread; gather the
//               rows' 16-byte K chunks with cp.async into the UMMA K-major
//               no-swizzle canonical layout (8-row x 16-byte core matrices);
//               cp.async.mbarrier.arrive.noinc signals the stage's full barrier.
//   warp 2      B producer: one cp.async.bulk per stage from the pre-tiled
//               weight image (TMA bulk engine, complete_tx on the same barrier).
//   warp 3      TMEM allocator + single-thread tcgen05.mma.kind::i8 issuer
//               (M=128, N=BN, K=32 per instruction, 4 per 128-byte stage).
//               Two TMEM accumulators so tile t+1's MMAs overlap tile t's epilogue.
//   warps 4-15  epilogue, 3 column groups x 4 TMEM lane quarters: tcgen05.ld 32x32b
//               (TMEM lane = output row), int32 zero-point correction, fp64 requant
//               (explicit _rn intrinsics, reference op order), relu, fused residual
//               add as a 64 KB shared-memory lookup table, 16-byte code stores.
// The smem pipeline depth is chosen at launch from what the per-channel constants
// and the add table leave of the 227 KB.
#include <atomic>
#include <climits>
#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace ptq {

constexpr int TC_BM = 128;
// per-channel epilogue constants of the layer being run, in constant memory: the epilogue
// indexes them with warp-uniform channel bases, so they load into uniform registers through
// the constant cache and never touch the L1 data pipe (shared-memory broadcasts of these
// 16-byte records were the L1 limiter).  Written by the launcher with a stream-ordered
// device-to-device copy before every launch.
constexpr int TC_MAX_COUT = 2048;
__constant__ EpiParam c_ep[TC_MAX_COUT];    // SoA image, see ep_soa() in kernels.h

constexpr int TC_MAX_STAGES = 10;                 // smem pipeline depth cap (runtime depth: launcher)
constexpr int TC_IO_NB = 2;                       // tile I/O buffers (tio)
constexpr int TC_SMEM_MAX = 232448;                // 227 KB opt-in dynamic smem per CTA
constexpr int TC_A_STAGE = TC_BM * 128;            // 16 KB: 8 chunks x 128 rows x 16 B
#ifndef PTQ_EPI_GROUPS
#define PTQ_EPI_GROUPS 4
#endif
constexpr int TC_NG = PTQ_EPI_GROUPS;               // epilogue column groups per TMEM lane quarter
constexpr int TC_EPI_WARPS = 4 * TC_NG;             // NG per SM sub-partition
constexpr int TC_THREADS = (4 + TC_EPI_WARPS) * 32;    // + producer / MMA warps 0-3
// How the 4 epilogue column groups share tiles.  Splitting every tile over all 4 groups
// gives each warp BN/64 chunks of 16 columns per tile, so for narrow tiles the per-tile work
// (barrier waits, row geometry, arrivals) costs as much as the chunks.  Instead GPT groups
// drain one tile (BN/(16*GPT) = 4 chunks per warp whenever BN >= 64) and the 4/GPT group sets
// take the CTA's tiles in turn (slot = lt mod SLOTS), each tile in its own TMEM accumulator
// (NACC >= SLOTS + 1 buffers where TMEM allows, so the MMA can fill one ahead) and, with tile
// I/O, its own shared tile (NIO).
template <int BN> struct TcGeom {
  static constexpr int GPT = BN <= 64 ? 1 : BN == 128 ? 2 : 4;   // column groups per tile
  static constexpr int SLOTS = TC_NG / GPT;                      // tiles drained at once
  static constexpr bool GROUPED = SLOTS > 1;
  static constexpr int NACC = BN <= 64 ? 4 : BN == 128 ? 3 : 2;  // accumulator buffers
  static constexpr int NIO = BN <= 64 ? 4 : BN == 128 ? 3 : TC_IO_NB;   // tile I/O buffers
  static constexpr int ARRIVE = GPT * 4 * 32;                    // epilogue threads per tile
};
constexpr int TC_MAX_BUF = 4;                      // barrier slots per buffer kind


__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version 1 (sm_100); base offset 0; SWIZZLE_NONE
  return d;
}

// K-major swizzled layout (TMA-written A): rows of 64 / 128 bytes in 8-row atoms of
// 512 / 1024 bytes (SBO), LBO unused (1), layout type 4 (SWIZZLE_64B) / 2 (SWIZZLE_128B)
__device__ __forceinline__ uint64_t umma_desc_sw(uint32_t saddr, int swz, uint32_t base_off = 0) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(((uint32_t)(swz * 8) >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(base_off & 7u) << 49;                // matrix base offset (swizzle phase)
  d |= (uint64_t)(swz == 128 ? 2u : 4u) << 61;
  return d;
}

// instruction descriptor: D=s32, A=s8, B=s8, both K-major, N (multiple of 16, <= 256), M=128
template <int N>
__device__ __forceinline__ uint32_t idesc_i8() {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(TC_BM >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// One 128-byte K stage in one asm block, executed by the whole (convergent) MMA warp: an
// elected lane issues the stage's K=32 MMAs and commits the stage's smem barrier.  The k-step
// offsets (descriptor units = 16 bytes) are added to the start-address field (smem addresses
// are < 256 KB, so the 14-bit field never carries).  One uniform-issue region per stage instead
// of one per MMA: the single issuing warp was the pacing resource of every narrow (BN <= 128)
// layer -- ~34-46 issued instructions per MMA before, the MMA itself takes 32 cycles at N=64.
// MMAs 2 and 3 are skipped when `full` is 0 (a half stage of the s2d slab with odd k).
__device__ __forceinline__ void mma4_commit(uint32_t d, uint64_t ad, uint64_t bd, uint64_t a1, uint64_t a2,
                                            uint64_t a3, uint64_t b1, uint32_t idesc, uint32_t acc,
                                            uint32_t full, uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e, q, t, f;\n\t.reg .b64 xa, xb;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 q, %8, 0;\n\t"
      "setp.eq.b32 t, %8, %8;\n\t"
      "setp.ne.and.b32 f, %9, 0, e;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %7, q;\n\t"
      "add.s64 xa, %1, %3;\n\tadd.s64 xb, %2, %6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], xa, xb, %7, t;\n\t"
      "add.s64 xa, %1, %4;\n\tadd.s64 xb, xb, %6;\n\t"
      "@f tcgen05.mma.cta_group::1.kind::i8 [%0], xa, xb, %7, t;\n\t"
      "add.s64 xa, %1, %5;\n\tadd.s64 xb, xb, %6;\n\t"
      "@f tcgen05.mma.cta_group::1.kind::i8 [%0], xa, xb, %7, t;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%10];\n\t}" ::"r"(d),
      "l"(ad), "l"(bd), "l"(a1), "l"(a2), "l"(a3), "l"(b1), "r"(idesc), "r"(acc), "r"(full), "r"(bar)
      : "memory");
}
// kw-reuse stage: 6 MMAs (3 kw taps x 2 K=32 halves), A and B both arithmetic sequences
__device__ __forceinline__ void mma6_commit(uint32_t d, uint64_t ad, uint64_t bd, uint64_t astep, uint64_t bstep,
                                            uint32_t idesc, uint32_t acc, uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e, q, t;\n\t.reg .b64 xa, xb;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 q, %6, 0;\n\t"
      "setp.eq.b32 t, %6, %6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %5, q;\n\t"
      "add.s64 xa, %1, %3;\n\tadd.s64 xb, %2, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], xa, xb, %5, t;\n\t"
      "add.s64 xa, xa, %3;\n\tadd.s64 xb, xb, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], xa, xb, %5, t;\n\t"
      "add.s64 xa, xa, %3;\n\tadd.s64 xb, xb, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], xa, xb, %5, t;\n\t"
      "add.s64 xa, xa, %3;\n\tadd.s64 xb, xb, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], xa, xb, %5, t;\n\t"
      "add.s64 xa, xa, %3;\n\tadd.s64 xb, xb, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], xa, xb, %5, t;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%7];\n\t}" ::"r"(d),
      "l"(ad), "l"(bd), "l"(astep), "l"(bstep), "r"(idesc), "r"(acc), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ int64_t vpix(const View& v, int n, int h, int w) {
  const int Hp = v.H + 2 * v.halo, Wp = v.W + 2 * v.halo;
  return ((int64_t)n * Hp + h + v.halo) * Wp + w + v.halo;
}

// ---------------------------------------------------------------- exact epilogue pieces
// int32 -> fp64 without the (slow) conversion pipe: 2^52 + 2^31 + x is exact, then subtract
__device__ __forceinline__ double i2d(int x) {
  return __dsub_rn(__hiloint2double(0x43300000, x ^ (int)0x80000000), 4503601774854144.0);
}
// floor(r) for |r| < 2^51 on the FP64 pipe: round-down add of 1.5*2^52 leaves floor(r)
// in the low word (two's complement)
__device__ __forceinline__ int floor_i(double r) {
  return __double2loint(__dadd_rd(r, 6755399441055744.0));
}
__device__ __forceinline__ int clampi(int x, int lo, int hi) { return x < lo ? lo : (x > hi ? hi : x); }

__device__ __forceinline__ int imin(int a, int b) { return a < b ? a : b; }
__device__ __forceinline__ int imax(int a, int b) { return a > b ? a : b; }

// fp64 value of a 2^31-biased int32 (accb = acc + 2^31 mod 2^32): 2^52 + accb is exact
__device__ __forceinline__ double b2d(uint32_t accb) {
  return __dsub_rn(__hiloint2double(0x43300000, (int)accb), 4503601774854144.0);
}
// per-layer epilogue constants held in registers by every epilogue thread
struct EpiK {
  uint32_t clo, chi;   // biased acc clamp bounds 2^31 -/+ aclamp
  int lo_conv, lo_add;
  // per-tensor weight granularity (rt.uni): the requant multiplier and the weight zero point
  // are the same for every channel and live in registers; only cc is loaded per channel
  double m0;
  int zw0;
  int fxm0, fxs;       // FX: per-tensor M and the shift S - 32
};


// RHU(acc*m) + zp (unclipped) on a biased accumulator: acc clamped to the layer's
// saturation margin, then fl(fl(acc*m) + 0.5) exactly as the reference, floor and +zp in
// one round-down add
template <bool CLAMP>
__device__ __forceinline__ int requant_raw(uint32_t accb, double m, const LayerRt& rt, const EpiK& k) {
  if (CLAMP) accb = umin(umax(accb, k.clo), k.chi);      // else |acc*m| < 2^30 already
  const double r = __dadd_rn(__dmul_rn(b2d(accb), m), 0.5);
  return __double2loint(__dadd_rd(r, rt.mg_zy));
}
// 16 output channels of one row, fast path (no int32 saturation possible).  Without a fused
// add the clip to [-128, 127] is the saturating pack (a fused relu adds one max).  A fused
// residual add is one shared-memory lookup: stab[skip byte * 260 + conv code] with stab
// pointing at column 128 of the table (built exactly by k_layer_params for the config;
// operand order is baked in).
template <bool WZP, bool SKIP, bool CLAMP, bool RELU, bool PT>
__device__ __forceinline__ int4 epi_chunk16(const uint32_t (&v)[16], const uint8_t* __restrict__ sp, int cs,
                                            int cb, int rowsum, const LayerRt& rt, const EpiK& k,
                                            const int8_t* __restrict__ stab, const int4 skv) {
  // per-channel constants, structure of arrays (m[cs] fp64, cc[cs], zw[cs]): from shared
  // memory (sp), or from __constant__ c_ep for the fused-add layers whose shared-memory pipe
  // the add table saturates.  Each broadcast 16-byte load costs the L1 data pipe several
  // wavefronts, so only what the variant needs is loaded: cc always, m and zw per channel
  // unless the weights are per-tensor (PT).
  const uint8_t* cbase = SKIP ? reinterpret_cast<const uint8_t*>(c_ep) : sp;
  uint32_t packed[4];
  const uint32_t skw[4] = {(uint32_t)skv.x, (uint32_t)skv.y, (uint32_t)skv.z, (uint32_t)skv.w};
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    int4 cc4, zw4;
    double2 m01, m23;
    if (SKIP) {
      cc4 = reinterpret_cast<const int4*>(reinterpret_cast<const uint8_t*>(c_ep) + 8 * cs)[(cb >> 2) + g];
      if (WZP && !PT) zw4 = reinterpret_cast<const int4*>(reinterpret_cast<const uint8_t*>(c_ep) + 12 * cs)[(cb >> 2) + g];
      if (!PT) {
        m01 = reinterpret_cast<const double2*>(c_ep)[(cb >> 1) + 2 * g];
        m23 = reinterpret_cast<const double2*>(c_ep)[(cb >> 1) + 2 * g + 1];
      }
    } else {
      cc4 = reinterpret_cast<const int4*>(sp + 8 * cs)[(cb >> 2) + g];
      if (WZP && !PT) zw4 = reinterpret_cast<const int4*>(sp + 12 * cs)[(cb >> 2) + g];
      if (!PT) {
        m01 = reinterpret_cast<const double2*>(sp)[(cb >> 1) + 2 * g];
        m23 = reinterpret_cast<const double2*>(sp)[(cb >> 1) + 2 * g + 1];
      }
    }
    (void)cbase;
    const int ccv[4] = {cc4.x, cc4.y, cc4.z, cc4.w};
    int zwv[4] = {0, 0, 0, 0};
    double mv[4] = {k.m0, k.m0, k.m0, k.m0};
    if (!PT) {
      mv[0] = m01.x; mv[1] = m01.y; mv[2] = m23.x; mv[3] = m23.y;
      if (WZP) { zwv[0] = zw4.x; zwv[1] = zw4.y; zwv[2] = zw4.z; zwv[3] = zw4.w; }
    }
    int q[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t accb = v[g * 4 + j] + (uint32_t)ccv[j];
      if (WZP) accb -= (uint32_t)((PT ? k.zw0 : zwv[j]) * rowsum);
      q[j] = requant_raw<CLAMP>(accb, mv[j], rt, k);
      if (RELU || SKIP) q[j] = imax(q[j], k.lo_conv);
      if (SKIP) {
        q[j] = stab[(int)__byte_perm(skw[g], 0u, 0x4440u + j) * PTQ_ADDTAB_ROW + imin(q[j], PTQ_QMAX)];
      }
    }
    packed[g] = SKIP ? __byte_perm(__byte_perm((uint32_t)q[0], (uint32_t)q[1], 0x0040),
                                   __byte_perm((uint32_t)q[2], (uint32_t)q[3], 0x0040), 0x5410)
                     : pack4_sat(q[0], q[1], q[2], q[3]);
  }
  return make_int4((int)packed[0], (int)packed[1], (int)packed[2], (int)packed[3]);
}

// 16 output channels of one row, exact fixed-point requant (rt.fx, k_layer_params): code =
// hi32(v'*M_c + B'_c) >> (S - 32) with v' = dot - zw*rowsum -- one IMAD.WIDE and one shift per
// output, no fp64 and no clamp (|v'| < 2^28.5, |B'| < 2^62: the 64-bit sum cannot wrap).  The
// per-channel constants (SoA: B'[cs] int64, M[cs], zw[cs]) come from shared memory, or from
// __constant__ c_ep on the fused-add layers; per-tensor layers (PT) hold M in a register and
// fold zw*rowsum into the per-row zr.
template <bool WZP, bool SKIP, bool RELU, bool PT>
__device__ __forceinline__ int4 epi_chunk16_fx(const uint32_t (&v)[16], const uint8_t* __restrict__ sp, int cs,
                                               int cb, int rowsum, int zr, const LayerRt& rt, const EpiK& k,
                                               const int8_t* __restrict__ stab, const int4 skv) {
  const uint8_t* base = SKIP ? reinterpret_cast<const uint8_t*>(c_ep) : sp;
  uint32_t packed[4];
  const uint32_t skw[4] = {(uint32_t)skv.x, (uint32_t)skv.y, (uint32_t)skv.z, (uint32_t)skv.w};
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const longlong2 b01 = reinterpret_cast<const longlong2*>(base)[(cb >> 1) + 2 * g];
    const longlong2 b23 = reinterpret_cast<const longlong2*>(base)[(cb >> 1) + 2 * g + 1];
    const long long bv[4] = {b01.x, b01.y, b23.x, b23.y};
    int mv[4] = {k.fxm0, k.fxm0, k.fxm0, k.fxm0};
    int zwv[4] = {0, 0, 0, 0};
    if (!PT) {
      const int4 m4 = reinterpret_cast<const int4*>(base + 8 * cs)[(cb >> 2) + g];
      mv[0] = m4.x; mv[1] = m4.y; mv[2] = m4.z; mv[3] = m4.w;
      if (WZP) {
        const int4 z4 = reinterpret_cast<const int4*>(base + 12 * cs)[(cb >> 2) + g];
        zwv[0] = z4.x; zwv[1] = z4.y; zwv[2] = z4.z; zwv[3] = z4.w;
      }
    }
    int q[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int a = (int)v[g * 4 + j];
      if (WZP) a = PT ? a - zr : a - zwv[j] * rowsum;
      const long long X = (long long)a * (long long)mv[j] + bv[j];
      q[j] = (int)(X >> 32) >> k.fxs;
      if (RELU || SKIP) q[j] = imax(q[j], k.lo_conv);
      if (SKIP) {
        q[j] = stab[(int)__byte_perm(skw[g], 0u, 0x4440u + j) * PTQ_ADDTAB_ROW + imin(q[j], PTQ_QMAX)];
      }
    }
    packed[g] = SKIP ? __byte_perm(__byte_perm((uint32_t)q[0], (uint32_t)q[1], 0x0040),
                                   __byte_perm((uint32_t)q[2], (uint32_t)q[3], 0x0040), 0x5410)
                     : pack4_sat(q[0], q[1], q[2], q[3]);
  }
  return make_int4((int)packed[0], (int)packed[1], (int)packed[2], (int)packed[3]);
}

// general (slow) path: 64-bit accumulator with the reference's int32 saturation
__device__ __forceinline__ int epi_slow(long long dot, int c, long long rowsum, const ConvTcArgs& a,
                                        const LayerRt& rt) {
  long long zw = a.wzp[c];
  long long acc = dot - zw * rowsum - (long long)rt.zx * a.wsum[c] + (long long)a.kreal * rt.zx * zw;
  acc = clip32(acc + a.L.biasq[c]);
  return requant1(acc, a.L.mult[c], rt.zy);
}

__device__ __forceinline__ uint32_t tmem_ld1(uint32_t taddr) {
  uint32_t v;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  return v;
}

// exact 64-bit path for a 16-channel chunk (int32 saturation possible, or a partial chunk).
// Rare (warp-uniform branch); written as a rolled loop that re-reads one TMEM column per
// step so it holds no arrays and costs the fast path no registers.
__device__ __forceinline__ int4 epi_slow_chunk(uint32_t taddr, int cb, long long rowsum,
                                               const ConvTcArgs& a, const LayerRt& rt, int lo_conv,
                                               int lo_add, int4 skv) {
  const uint64_t sk_lo = ((uint64_t)(uint32_t)skv.y << 32) | (uint32_t)skv.x;
  const uint64_t sk_hi = ((uint64_t)(uint32_t)skv.w << 32) | (uint32_t)skv.z;
  uint64_t lo = 0, hi = 0;
#pragma unroll 1
  for (int j = 0; j < 16; ++j) {
    const uint32_t x = tmem_ld1(taddr + (uint32_t)j);
    const int c = cb + j;
    int code = 0;
    if (c < a.L.cout) {
      code = epi_slow((long long)(int)x, c, rowsum, a, rt);
      if (code < lo_conv) code = lo_conv;
      if (a.skip.p) {
        const int skc = (int)(int8_t)(((j < 8) ? sk_lo : sk_hi) >> (8 * (j & 7)));
        const int xa = a.conv_is_a ? code : skc, xb = a.conv_is_a ? skc : code;
        const double s2 = __dadd_rn(__dmul_rn(i2d(xa - rt.za), rt.ra), __dmul_rn(i2d(xb - rt.zb), rt.rb));
        code = clip8(rhu(s2) + (double)rt.zo);
        if (code < lo_add) code = lo_add;
      }
    }
    const uint64_t bits = (uint64_t)((uint32_t)code & 0xffu) << (8 * (j & 7));
    if (j < 8) lo |= bits; else hi |= bits;
  }
  return make_int4((int)(uint32_t)lo, (int)(uint32_t)(lo >> 32), (int)(uint32_t)hi, (int)(uint32_t)(hi >> 32));
}

// parity probe (ptq_probe_acc): the exact accumulators of a 16-channel chunk, acc + bias
// saturated to int32 as the reference does before requantizing (intexec.py:177-190), stored to
// dst[c] (dst = this pixel's [cout] row, or nullptr for rows outside the real output).  The
// warp-uniform loop re-reads one TMEM column per step (tcgen05.ld is .sync.aligned).
__device__ __forceinline__ void epi_acc_chunk(uint32_t taddr, int cb, long long rowsum, const ConvTcArgs& a,
                                              const LayerRt& rt, int* dst) {
#pragma unroll 1
  for (int j = 0; j < 16; ++j) {
    const uint32_t x = tmem_ld1(taddr + (uint32_t)j);
    const int c = cb + j;
    if (dst && c < a.L.cout) {
      const long long zw = a.wzp[c];
      const long long acc = (long long)(int)x - zw * rowsum - (long long)rt.zx * a.wsum[c] +
                            (long long)a.kreal * rt.zx * zw;
      dst[c] = (int)clip32(acc + a.L.biasq[c]);
    }
  }
}

__device__ __forceinline__ long long pixel_rowsum(const ConvTcArgs& a, int n, int ih0, int iw0) {
  if (!a.has_wzp) return 0;
  const int Wp = a.in.W + 2 * a.in.halo, Hp = a.in.H + 2 * a.in.halo;
  long long s = 0;
  for (int kh = 0; kh < a.k; ++kh)
    for (int kw = 0; kw < a.k; ++kw) s += a.P[((int64_t)n * Hp + ih0 + kh) * Wp + iw0 + kw];
  return s;
}

struct RowGeo {
  bool ok;
  int n, oh, ow, ih0, iw0;
};
__device__ __forceinline__ RowGeo row_geo(const ConvTcArgs& a, int m, int M) {
  RowGeo g{};
  g.ok = m < M;   // (TMA mode: also inside the real output, checked below)
  if (g.ok) {                                  // M < 2^31: multiply-high divisions
    const uint32_t t = a.div_ow.div((uint32_t)m);
    g.ow = m - (int)t * a.OW;
    const uint32_t nn = a.div_oh.div(t);
    g.oh = (int)t - (int)nn * a.OH;
    g.n = (int)nn;
  }
  g.ok = g.ok && g.oh < a.OHr && g.ow < a.OWr;
  g.ih0 = g.oh * a.stride - a.pad + a.in.halo;
  g.iw0 = g.ow * a.stride - a.pad + a.in.halo;
  return g;
}

// what the epilogue warps share across the persistent tile loop
struct EpiEnv {
  uint32_t tmem;
  uint64_t *tfull, *tempty, *rsfull;
  const int* rsum;
  const uint8_t* sp;                                 // shared-memory constants (non-add layers), SoA
  int cs;                                            // SoA channel stride = roundup(Cout, 16)
  const int8_t* stab_c;
  int q, grp, row, M, n_tiles, n_nt;
  uint8_t* sio;                                      // tile I/O buffers [NIO][128][BN] (tio)
  uint64_t *iofull, *ioempty, *ioready;
};

// persistent epilogue tile loop of one variant (GENERIC: runtime dispatch, slow layers and
// the profiling ablation).  q / grp come from a warp-uniform (shuffled) warp index, so the
// chunk loop and the channel base cb are warp-uniform: every lane of a warp loads the same
// per-channel constants (broadcast shared-memory loads, or for the fused-add layers indexed
// LDC from __constant__ c_ep, which keeps them off the L1 data pipe the add table uses).
template <int BN, bool WZP, bool SKIP, bool CLAMP, bool RELU, bool GENERIC, bool ACC = false, bool PT = false,
          bool FX = false, int TIOM = -1>
__device__ __forceinline__ void epi_tiles(const ConvTcArgs& a, const LayerRt& rt, const EpiK& k, const EpiEnv& e) {
  constexpr int NCH = BN / 16;                       // 16-column chunks per tile
  const int Cout = a.L.cout;
  // tile I/O: a compile-time choice for the FX variants (TIOM 0 / 1), so the tile-I/O loop
  // carries no direct-store / residual-load code and keeps its slot address in registers
  const bool tio = TIOM < 0 ? a.tio != 0 : TIOM == 1;
  const bool has_skip = GENERIC ? a.skip.p != nullptr : SKIP;
  using G = TcGeom<BN>;
  uint32_t lt = 0;
  int slot = 0;                                      // lt % SLOTS
  const int my_slot = e.grp / G::GPT;                // this group's tiles: slot == my_slot
  for (int tile = blockIdx.x; tile < e.n_tiles; tile += gridDim.x, ++lt, slot = slot == G::SLOTS - 1 ? 0 : slot + 1) {
    if (G::GROUPED && slot != my_slot) continue;     // warp-uniform: another group set's tile
    const uint32_t buf = lt % G::NACC, uph = (lt / G::NACC) & 1u;
    const int mt = (int)a.div_nt.div((uint32_t)tile);
    // n-tile (warp-uniform; the shuffle lets ptxas keep it, and every channel index derived
    // from it, in uniform registers)
    const int nt = __shfl_sync(0xffffffffu, tile - mt * e.n_nt, 0);
    // chunks c = first, first + GPT, ... (BN / (16 GPT) per warp: an even split)
    const int first = e.grp % G::GPT;
    constexpr int CSTEP = G::GPT;
    const int m = mt * TC_BM + e.row;
    RowGeo g;
    int8_t* orow;
    const int8_t* srow;
    if (a.flat) {                                    // row m == flat output pixel m
      g.ok = m < e.M;
      orow = g.ok ? a.out.p + (int64_t)m * a.out.Cp : nullptr;
      srow = (g.ok && has_skip) ? a.skip.p + (int64_t)m * a.skip.Cp : nullptr;
    } else {
      g = row_geo(a, m, e.M);
      orow = g.ok ? a.out.p + vpix(a.out, g.n, g.oh, g.ow) * a.out.Cp : nullptr;
      srow = (g.ok && has_skip) ? a.skip.p + vpix(a.skip, g.n, g.oh, g.ow) * a.skip.Cp : nullptr;
    }
    long long rowsum = 0;
    if ((GENERIC || WZP) && a.rs_mma) {
      // read below from the accumulator's indicator columns
    } else if ((GENERIC || WZP) && a.tma_rowsum) {
      mbar_wait(&e.rsfull[buf], uph);
      rowsum = e.rsum[buf * TC_BM + e.row];
    } else if ((GENERIC || WZP) && g.ok && first < NCH) {
      rowsum = a.Rpix ? (long long)a.Rpix[((int64_t)g.n * a.OHr + g.oh) * a.OWr + g.ow]
                      : pixel_rowsum(a, g.n, g.ih0, g.iw0);
    }
    // tile I/O: this tile's shared buffer (the fused-add operand landed by TMA, or a buffer
    // whose previous TMA store has finished reading it)
    const uint32_t ib = lt % G::NIO, iph = (lt / G::NIO) & 1u;
    uint8_t* io = e.sio + ib * (TC_BM * BN);
    const int iow = a.io_w, iosh = a.io_w == 128 ? 3 : 2;   // box width in bytes, log2(16-byte units)
    // this row's slot base (shared address) and 16-byte-unit swizzle, once per tile: per chunk
    // only the uniform box / unit offset is added and the unit XORed with the row phase
    const uint32_t io_row = smem_u32(io) + (uint32_t)(e.row * iow);
    const uint32_t io_x = (uint32_t)(iow == 128 ? (e.row & 7) : ((e.row >> 1) & 3)) << 4;
    if (tio) {
      if (has_skip) mbar_wait(&e.iofull[ib], iph);
      else mbar_wait(&e.ioempty[ib], iph ^ 1u);
    }
    mbar_wait(&e.tfull[buf], uph);
    tc_fence_after();
    const uint32_t tbase = e.tmem + ((uint32_t)(e.q * 32) << 16) + buf * (uint32_t)a.b_rows;
    if ((GENERIC || WZP) && a.rs_mma) rowsum = (int)tmem_ld1(tbase + BN);   // sum_k x[row][k]
    const int zr = (FX && PT && WZP) ? k.zw0 * (int)rowsum : 0;   // per-tensor zw * rowsum
#pragma unroll 1
    for (int c = first; c < NCH; c += CSTEP) {
      const int cb = nt * BN + c * 16;
      if (ACC) {
        if (cb >= Cout) continue;                    // warp-uniform
        const int64_t pix = a.flat ? (int64_t)m : ((int64_t)g.n * a.OHr + g.oh) * a.OWr + g.ow;
        epi_acc_chunk(tbase + (uint32_t)(c * 16), cb, rowsum, a, rt, g.ok ? a.acc_out + pix * Cout : nullptr);
        continue;
      }
      // residual operand without tile I/O (non-flat layers): a direct 16-byte load issued
      // ahead of the TMEM load it overlaps with (no cross-chunk prefetch state: those register
      // moves cost every chunk of the tile-I/O layers an extra 8 instructions)
      int4 skv = make_int4(0, 0, 0, 0);
      if (has_skip && !tio && srow && cb < a.out.Cp) skv = __ldg(reinterpret_cast<const int4*>(srow + cb));
      uint32_t v[16];
      tmem_ld16(tbase + (uint32_t)(c * 16), v);
      if (cb >= a.out.Cp) continue;                  // warp-uniform: the slow path re-reads TMEM
      // swizzled slot of (row, chunk c) in the I/O tile: box c / iocpb, 16-byte unit XOR row phase
      const uint32_t ioslot = io_row + (uint32_t)((c >> iosh) * (TC_BM * iow)) +
                              (((uint32_t)(c & ((1 << iosh) - 1)) << 4) ^ io_x);
      if (has_skip && tio) skv = lds128(ioslot);
      int4 res;
      if (GENERIC && a.ablate == 1) {
        res = make_int4((int)v[0], (int)v[1], (int)v[2], (int)v[3]);
      } else if (FX && cb + 16 <= Cout) {
        res = epi_chunk16_fx<WZP, SKIP, RELU, PT>(v, e.sp, e.cs, cb, (int)rowsum, zr, rt, k, e.stab_c, skv);
      } else if (!GENERIC && !FX && cb + 16 <= Cout) {
        res = epi_chunk16<WZP, SKIP, CLAMP, RELU, PT>(v, e.sp, e.cs, cb, (int)rowsum, rt, k, e.stab_c, skv);
      } else {
        res = epi_slow_chunk(tbase + (uint32_t)(c * 16), cb, rowsum, a, rt, k.lo_conv, k.lo_add, skv);
      }
      if (tio) sts128(ioslot, res);
      else if (g.ok) *reinterpret_cast<int4*>(orow + cb) = res;
    }
    tc_fence_before();
    mbar_arrive(&e.tempty[buf]);                     // accumulator buffer may be reused
    if (tio) {
      // this thread's codes are in the tile: hand them to the async proxy and tell the I/O
      // agent (no CTA-wide barrier: the epilogue warps stay decoupled)
      fence_proxy_async();
      mbar_arrive(&e.ioready[ib]);
    }
  }
}

// per-tensor weights (rt.uni: one requant multiplier and weight zero point for the layer)
// take the PT variant, which loads only cc per channel
template <int BN, bool WZP, bool SKIP, bool CLAMP, bool RELU>
__device__ __forceinline__ void epi_pt(const ConvTcArgs& a, const LayerRt& rt, const EpiK& k, const EpiEnv& e) {
  if (rt.uni) epi_tiles<BN, WZP, SKIP, CLAMP, RELU, false, false, true>(a, rt, k, e);
  else epi_tiles<BN, WZP, SKIP, CLAMP, RELU, false, false, false>(a, rt, k, e);
}
template <int BN, bool WZP, bool SKIP, bool RELU>
__device__ __forceinline__ void epi_fx(const ConvTcArgs& a, const LayerRt& rt, const EpiK& k, const EpiEnv& e) {
  if (a.tio) {
    if (rt.uni) epi_tiles<BN, WZP, SKIP, false, RELU, false, false, true, true, 1>(a, rt, k, e);
    else epi_tiles<BN, WZP, SKIP, false, RELU, false, false, false, true, 1>(a, rt, k, e);
  } else {
    if (rt.uni) epi_tiles<BN, WZP, SKIP, false, RELU, false, false, true, true, 0>(a, rt, k, e);
    else epi_tiles<BN, WZP, SKIP, false, RELU, false, false, false, true, 0>(a, rt, k, e);
  }
}

// BR = B rows per tile (a.b_rows): BN, or BN + 16 K-indicator rows (the MMA then runs over
// N = BR and accumulator columns BN..BN+15 are the A-row sums, rs_mma)
template <int BN, int BR>
__global__ void __launch_bounds__(TC_THREADS, 1) k_conv_tc(const __grid_constant__ ConvTcArgs a) {
  const int NS = a.n_stages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // swizzled TMA tiles need 1024-byte aligned stages (the launcher reserves the slack)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sio = smem;                              // tile I/O buffers (tio), 1024-aligned boxes
  using G = TcGeom<BN>;
  uint8_t* sA = smem + (a.tio ? G::NIO * TC_BM * BN : 0);
  uint8_t* sB = sA + NS * TC_A_STAGE;               // B ring [NS][BN][128], or resident [n_kiter][BN][128]
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + (a.b_res ? a.n_kiter : NS) * BR * 128);
  uint64_t* empty = full + NS;
  uint64_t* tfull = empty + NS;                                  // [NACC] accumulator ready
  uint64_t* tempty = tfull + TC_MAX_BUF;                         // [NACC] accumulator drained
  uint64_t* rsfull = tempty + TC_MAX_BUF;                        // [NACC] row sums of tile buffer ready
  uint64_t* bfull = rsfull + TC_MAX_BUF;                         // resident B landed
  uint64_t* iofull = bfull + 1;                                  // [NIO] operand tile landed
  uint64_t* ioempty = iofull + TC_MAX_BUF;                       // [NIO] tile buffer free
  uint64_t* ioready = ioempty + TC_MAX_BUF;                      // [NIO] epilogue wrote the tile
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ioready + TC_MAX_BUF);
  int* rsum = reinterpret_cast<int*>(ioready + TC_MAX_BUF + 1);  // [NACC][128] A-row sums (tma_rowsum)
  EpiParam* sparam = reinterpret_cast<EpiParam*>(rsum + TC_MAX_BUF * TC_BM);   // [Cout] (no fused add)
  int8_t* stab = reinterpret_cast<int8_t*>(rsum + TC_MAX_BUF * TC_BM);          // fused-add table
  // NACC accumulator buffers of BR columns (power-of-two allocation, at least 32)
  constexpr uint32_t TMEM_NEED = G::NACC * BR;
  constexpr uint32_t TMEM_COLS = TMEM_NEED <= 32 ? 32u : TMEM_NEED <= 64 ? 64u : TMEM_NEED <= 128 ? 128u
                                 : TMEM_NEED <= 256 ? 256u : 512u;
  static_assert(TMEM_NEED <= 512, "accumulator buffers exceed TMEM");

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int M = a.in.N * a.OH * a.OW;
  const int n_nt = (a.L.cout + BN - 1) / BN;
  const int n_tiles = ((M + TC_BM - 1) / TC_BM) * n_nt;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], (a.tma_a ? 1 : 64) + (a.b_res ? 0 : 1));
      mbar_init(&empty[s], a.tma_rowsum ? 2 : 1);
    }
    mbar_init(bfull, 1);
    for (int b = 0; b < G::NIO; ++b) {
      mbar_init(&iofull[b], 1);
      mbar_init(&ioempty[b], 1);
      mbar_init(&ioready[b], G::ARRIVE);
    }
    for (int b = 0; b < G::NACC; ++b) {
      mbar_init(&rsfull[b], 1);
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], G::ARRIVE);
    }
    fence_mbar_init();
  }
  if (warp == 3) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 2 && a.tma_a) {
    // ------------------------------------------------ A producer, TMA mode: the conv runs over
    // the padded output grid, so tap (kh, kw) of 128 consecutive output positions is 128
    // consecutive flat input pixels at offset kh*Wp + kw -- one tensor-map tile per tap slice
    if (warp == 0 && lane == 0) {
      if (a.tma_a != 67) prefetch_tmap(&a.tmA);
      const int Wp = a.in.W + 2 * a.in.halo;
      const int cpc = a.in.Cp >> 4, taps = a.k * a.k;
      int s = 0;
      uint32_t ph = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int p0 = (int)a.div_nt.div((uint32_t)tile) * TC_BM;
        for (int ki = 0; ki < a.a_iters; ++ki) {
          mbar_wait(&empty[s], ph ^ 1u);
          uint8_t* dst = sA + s * TC_A_STAGE;
          if (a.tma_a == 128) {                      // one tap, 128 channels per stage
            const int kk = ki * 8, tap = kk / cpc, c0 = (kk - tap * cpc) * 16;
            mbar_arrive_expect_tx(&full[s], TC_A_STAGE);
            tma_load_2d(dst, &a.tmA, c0, p0 + (tap / a.k) * Wp + tap % a.k, &full[s]);
          } else if (a.tma_a == 67) {                // s2d stem: one contiguous slab per stage
            // input pixels p0 + 2ki*Wp + [0, Wp + 131): both kh rows of the stage and their 4 kw
            // taps are this slab shifted by kh*Wp + kw pixels (16 bytes each) -- one bulk copy
            const int kh0 = 2 * ki;
            const uint32_t bytes = (uint32_t)((kh0 + 1 < a.k ? Wp : 0) + TC_BM + 3) * 16u;
            mbar_arrive_expect_tx(&full[s], bytes);
            bulk_g2s(dst, a.in.p + ((int64_t)p0 + (int64_t)kh0 * Wp) * 16, bytes, &full[s]);
          } else if (a.tma_a == 66) {                // s2d stem, 64-byte window rows: two kh
            const int t0 = 2 * ki, t1 = 2 * ki + 1;  // rows of 4 kw taps per stage
            mbar_arrive_expect_tx(&full[s], t1 < a.k ? TC_A_STAGE : TC_A_STAGE / 2);
            tma_load_2d(dst, &a.tmA, 0, p0 + t0 * Wp, &full[s]);
            if (t1 < a.k) tma_load_2d(dst + TC_A_STAGE / 2, &a.tmA, 0, p0 + t1 * Wp, &full[s]);
          } else if (a.kwr) {                        // one 136-row slab per kh (all 3 kw taps)
            mbar_arrive_expect_tx(&full[s], (TC_BM + 8) * 64);
            tma_load_2d(dst, &a.tmA, 0, p0 + ki * Wp, &full[s]);
          } else if (a.tma_a == 64) {                // Cp == 64: two taps per stage
            const int t0 = 2 * ki, t1 = 2 * ki + 1;
            mbar_arrive_expect_tx(&full[s], t1 < taps ? TC_A_STAGE : TC_A_STAGE / 2);
            tma_load_2d(dst, &a.tmA, 0, p0 + (t0 / a.k) * Wp + t0 % a.k, &full[s]);
            if (t1 < taps)
              tma_load_2d(dst + TC_A_STAGE / 2, &a.tmA, 0, p0 + (t1 / a.k) * Wp + t1 % a.k, &full[s]);
          } else {                                   // Cp == 16, k == 4 (s2d stem): 4 kw taps
            const int t0 = 2 * ki, t1 = 2 * ki + 1;  // per box, two kh rows per stage
            mbar_arrive_expect_tx(&full[s], t1 < a.k ? TC_A_STAGE : TC_A_STAGE / 2);
            tma_load_3d(dst, &a.tmA, 0, p0 + t0 * Wp, 0, &full[s]);
            if (t1 < a.k) tma_load_3d(dst + TC_A_STAGE / 2, &a.tmA, 0, p0 + t1 * Wp, 0, &full[s]);
          }
          if (++s == NS) { s = 0; ph ^= 1u; }
        }
      }
    } else if (warp == 1 && a.tma_rowsum) {
      // weight zero points need sum_k x[row][k] per GEMM row: sum the A rows straight from
      // the landed stages (halo taps hold the zero point, pad channels 0), instead of a
      // separate pixel-sum pass over the input tensor.  Lane l owns rows l + 32i; chunks are
      // visited in a lane-rotated order so every quarter-warp hits distinct banks.
      const int taps = a.k * a.k;
      int s = 0;
      uint32_t ph = 0, lt = 0;
      const int iters = a.kwr ? a.a_iters : a.n_kiter;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++lt) {
        const uint32_t buf = lt % G::NACC, uph = (lt / G::NACC) & 1u;
        int sum[4] = {0, 0, 0, 0};
        for (int ki = 0; ki < iters; ++ki) {
          mbar_wait(&full[s], ph);
          const uint8_t* st = sA + s * TC_A_STAGE;
          if (a.kwr) {
            // kw-reuse slab of one kernel row: 136 pixels x 64 channel bytes; GEMM row r takes
            // pixels r, r + 1, r + 2 (the three kw taps).  Per-pixel sums px[i] of pixels
            // lane + 32i, then the two right neighbours by shuffles
            int px[5];
#pragma unroll
            for (int i = 0; i < 5; ++i) {
              px[i] = 0;
              const int j = lane + 32 * i;
              if (j < TC_BM + 8)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  const int4 v = *reinterpret_cast<const int4*>(st + j * 64 + ((q + (lane >> 1)) & 3) * 16);
                  px[i] = __dp4a(v.x, 0x01010101, __dp4a(v.y, 0x01010101, __dp4a(v.z, 0x01010101, __dp4a(v.w, 0x01010101, px[i]))));
                }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int a1 = __shfl_down_sync(0xffffffffu, px[i], 1), b1 = __shfl_sync(0xffffffffu, px[i + 1], 0);
              const int a2 = __shfl_down_sync(0xffffffffu, px[i], 2);
              const int b2 = __shfl_sync(0xffffffffu, px[i + 1], (lane + 2) & 31);
              sum[i] += px[i] + (lane < 31 ? a1 : b1) + (lane < 30 ? a2 : b2);
            }
          } else if (a.tma_a == 128) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const int4 v = *reinterpret_cast<const int4*>(st + (lane + 32 * i) * 128 + ((j + lane) & 7) * 16);
                sum[i] = __dp4a(v.x, 0x01010101, __dp4a(v.y, 0x01010101, __dp4a(v.z, 0x01010101, __dp4a(v.w, 0x01010101, sum[i]))));
              }
          } else {
            const int halves = 2 * ki + 1 < taps ? 2 : 1;
            for (int hv = 0; hv < halves; ++hv)
#pragma unroll
              for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const int4 v = *reinterpret_cast<const int4*>(st + hv * (TC_A_STAGE / 2) + (lane + 32 * i) * 64 +
                                                                ((j + (lane >> 1)) & 3) * 16);
                  sum[i] = __dp4a(v.x, 0x01010101, __dp4a(v.y, 0x01010101, __dp4a(v.z, 0x01010101, __dp4a(v.w, 0x01010101, sum[i]))));
                }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[s]);     // this stage's A bytes are no longer needed here
          if (++s == NS) { s = 0; ph ^= 1u; }
        }
        mbar_wait(&tempty[buf], uph ^ 1u);           // the epilogue is done with rsum[buf]
#pragma unroll
        for (int i = 0; i < 4; ++i) rsum[buf * TC_BM + lane + 32 * i] = sum[i];
        __syncwarp();
        if (lane == 0) mbar_arrive(&rsfull[buf]);
      }
    }
  } else if (warp < 2) {
    // ------------------------------------------------ A producers (implicit im2col gather)
    if (a.in.Cp & 16) {
      // odd chunks per tap: the chunk pairs below would straddle taps (two pixels), so one GEMM
      // row per lane: 64 threads, rows r and r + 64, 16-byte chunks of one row in sequence
      const int r = threadIdx.x;
      const int Cp = a.in.Cp, cpc = Cp >> 4;
      const int Wp = a.in.W + 2 * a.in.halo, Hp = a.in.H + 2 * a.in.halo;
      int s = 0;
      uint32_t ph = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int mt = (int)a.div_nt.div((uint32_t)tile);
        const RowGeo g0 = row_geo(a, mt * TC_BM + r, M);
        const RowGeo g1 = row_geo(a, mt * TC_BM + r + 64, M);
        const int8_t* base0 = a.in.p + (((int64_t)g0.n * Hp + g0.ih0) * Wp + g0.iw0) * Cp;
        const int8_t* base1 = a.in.p + (((int64_t)g1.n * Hp + g1.ih0) * Wp + g1.iw0) * Cp;
        if (a.skip.p) {
          const int nt = tile - mt * n_nt;
          const int c0 = nt * BN;
          const uint32_t bytes = (uint32_t)(a.skip.Cp - c0 < BN ? a.skip.Cp - c0 : BN);
          if (g0.ok) bulk_prefetch_l2(a.skip.p + vpix(a.skip, g0.n, g0.oh, g0.ow) * a.skip.Cp + c0, bytes);
          if (g1.ok) bulk_prefetch_l2(a.skip.p + vpix(a.skip, g1.n, g1.oh, g1.ow) * a.skip.Cp + c0, bytes);
        }
        int kh = 0, kw = 0, ch = 0, kk = 0;
        for (int ki = 0; ki < a.n_kiter; ++ki) {
          mbar_wait(&empty[s], ph ^ 1u);
          uint8_t* dst = sA + s * TC_A_STAGE + r * 16;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const bool kin = kk < a.n_chunks && a.ablate != 2;
            const int64_t off = ((int64_t)kh * Wp + kw) * Cp + ch * 16;
            const bool v0 = g0.ok && kin, v1 = g1.ok && kin;
            cp_async16(dst + j * (TC_BM * 16), v0 ? base0 + off : a.in.p, v0 ? 16u : 0u);
            cp_async16(dst + j * (TC_BM * 16) + 64 * 16, v1 ? base1 + off : a.in.p, v1 ? 16u : 0u);
            ++kk;
            if (++ch == cpc) {
              ch = 0;
              if (++kw == a.k) { kw = 0; ++kh; }
            }
          }
          cp_async_mbar_arrive_noinc(&full[s]);
          if (++s == NS) { s = 0; ph ^= 1u; }
        }
      }
    } else {
      // 64 threads; a warp instruction covers 16 GEMM rows x 2 adjacent 16-byte K chunks, so the
      // two lanes of a row fill one 32-byte sector (one L2 request instead of two half-used ones;
      // the 2-way shared-memory write conflict between the two chunk planes is cheaper).  Lane l of
      // warp w: rows w*64 + 16g + l/2 (g = 0..3), chunks of parity l & 1
      const int lane2 = threadIdx.x & 31, par = lane2 & 1;
      const int rbase = (threadIdx.x >> 5) * 64 + (lane2 >> 1);
      const int Cp = a.in.Cp, cpc = Cp >> 4;
      const int Wp = a.in.W + 2 * a.in.halo, Hp = a.in.H + 2 * a.in.halo;
      int s = 0;
      uint32_t ph = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int mt = (int)a.div_nt.div((uint32_t)tile);
        const int8_t* base[4];
        bool rok[4];
  #pragma unroll
        for (int gi = 0; gi < 4; ++gi) {
          const RowGeo gg = row_geo(a, mt * TC_BM + rbase + 16 * gi, M);
          rok[gi] = gg.ok;
          base[gi] = a.in.p + (((int64_t)gg.n * Hp + gg.ih0) * Wp + gg.iw0) * Cp;
          if (a.skip.p && par == 0 && gg.ok) {
            // the fused add's operand rows for this tile: pull them into L2 now, a few tiles
            // before the epilogue reads them 16 bytes at a time
            const int nt = tile - mt * n_nt;
            const int c0 = nt * BN;
            const uint32_t bytes = (uint32_t)(a.skip.Cp - c0 < BN ? a.skip.Cp - c0 : BN);
            bulk_prefetch_l2(a.skip.p + vpix(a.skip, gg.n, gg.oh, gg.ow) * a.skip.Cp + c0, bytes);
          }
        }
        // this lane's K chunks: kk = par, par + 2, ... walked as (kh, kw, ch)
        int kh = 0, kw = 0, ch = par, kk = par;
        while (ch >= cpc) { ch -= cpc; if (++kw == a.k) { kw = 0; ++kh; } }
        for (int ki = 0; ki < a.n_kiter; ++ki) {
          mbar_wait(&empty[s], ph ^ 1u);
          uint8_t* dst = sA + s * TC_A_STAGE + rbase * 16;
  #pragma unroll
          for (int q = 0; q < 4; ++q) {
            const bool kin = kk < a.n_chunks && a.ablate != 2;
            const int64_t off = ((int64_t)kh * Wp + kw) * Cp + ch * 16;
            uint8_t* d = dst + (2 * q + par) * (TC_BM * 16);
  #pragma unroll
            for (int gi = 0; gi < 4; ++gi) {
              const bool v = rok[gi] && kin;
              cp_async16(d + gi * (16 * 16), v ? base[gi] + off : a.in.p, v ? 16u : 0u);
            }
            kk += 2;
            ch += 2;
            while (ch >= cpc) { ch -= cpc; if (++kw == a.k) { kw = 0; ++kh; } }
          }
          cp_async_mbar_arrive_noinc(&full[s]);
          if (++s == NS) { s = 0; ph ^= 1u; }
        }
      }
    }
  } else if (warp == 2) {
    // ------------------------------------------------ B producer (bulk copies of pre-tiled weights)
    if (lane == 0 && a.b_res) {                     // one n-tile: load every K stage once
      mbar_arrive_expect_tx(bfull, (uint32_t)(a.n_kiter * BR * 128));
      for (int ki = 0; ki < a.n_kiter; ++ki)
        bulk_g2s(sB + ki * BR * 128, a.wB + (int64_t)ki * BR * 128, BR * 128, bfull);
    } else if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int nt = tile - (int)a.div_nt.div((uint32_t)tile) * n_nt;
        const int8_t* gB = a.wB + (int64_t)nt * a.n_kiter * BR * 128;
        for (int ki = 0; ki < a.n_kiter; ++ki) {
          mbar_wait(&empty[s], ph ^ 1u);
          mbar_arrive_expect_tx(&full[s], BR * 128);
          bulk_g2s(sB + s * BR * 128, gB + (int64_t)ki * BR * 128, BR * 128, &full[s]);
          if (++s == NS) { s = 0; ph ^= 1u; }
        }
      }
    } else if (lane == 1 && a.tio) {
      // ---------------------------------------------- tile I/O agent (tio), lane 1 of warp 2:
      // loads the fused-add operand of a tile into its buffer (TMA), and stores each tile the
      // epilogue finished (TMA; rows past M and columns past Cp are clipped by the map); a
      // buffer is reloaded / handed back once its store has finished reading it
      const bool skip = a.skip.p != nullptr;
      const int iow = a.io_w;
      if (skip) prefetch_tmap(&a.tmS);
      prefetch_tmap(&a.tmO);
      auto load = [&](int tile, uint32_t ib) {
        const int mt = (int)a.div_nt.div((uint32_t)tile), nt = tile - mt * n_nt;
        const int nbox = (imin(BN, a.skip.Cp - nt * BN) + iow - 1) / iow;
        uint8_t* io = sio + ib * (TC_BM * BN);
        mbar_arrive_expect_tx(&iofull[ib], (uint32_t)(nbox * TC_BM * iow));
        for (int b = 0; b < nbox; ++b)
          tma_load_2d(io + b * (TC_BM * iow), &a.tmS, nt * BN + b * iow, mt * TC_BM, &iofull[ib]);
      };
      // the operand of the tile NIO loads ahead is pulled into L2 when its predecessor is
      // loaded, so the shared-memory load (issued only once a buffer's store has been read)
      // sees L2 latency, not HBM latency.  Only for 256-wide tiles (2 buffers): ResNet-50
      // poin15 0.433 -> 0.396 ms; the 128-wide grouped layers (3 buffers) lose 5 %
      const bool PF = BN == 256 && a.skip_pf;
      auto prefetch = [&](int tile) {
        if (tile >= n_tiles) return;
        const int mt = (int)a.div_nt.div((uint32_t)tile), nt = tile - mt * n_nt;
        const int nbox = (imin(BN, a.skip.Cp - nt * BN) + iow - 1) / iow;
        for (int b = 0; b < nbox; ++b) tma_prefetch_2d(&a.tmS, nt * BN + b * iow, mt * TC_BM);
      };
      if (skip) {
        for (int i = 0; i < G::NIO && blockIdx.x + i * (int)gridDim.x < n_tiles; ++i)
          load(blockIdx.x + i * gridDim.x, (uint32_t)i);
        if (PF)
          for (int i = G::NIO; i < 2 * G::NIO; ++i) prefetch(blockIdx.x + i * (int)gridDim.x);
      }
      uint32_t lt = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++lt) {
        const uint32_t ib = lt % G::NIO, iph = (lt / G::NIO) & 1u;
        const int mt = (int)a.div_nt.div((uint32_t)tile), nt = tile - mt * n_nt;
        const int nbox = (imin(BN, a.out.Cp - nt * BN) + iow - 1) / iow;
        uint8_t* io = sio + ib * (TC_BM * BN);
        mbar_wait(&ioready[ib], iph);
        for (int b = 0; b < nbox; ++b) tma_store_2d(&a.tmO, io + b * (TC_BM * iow), nt * BN + b * iow, mt * TC_BM);
        bulk_commit();
        if (skip) {
          const int next = tile + G::NIO * (int)gridDim.x;
          if (next < n_tiles) {
            bulk_wait_read<0>();
            load(next, ib);
            if (PF) prefetch(next + G::NIO * (int)gridDim.x);
          }
        } else {
          bulk_wait_read<1>();
          if (lt > 0) mbar_arrive(&ioempty[(lt - 1) % G::NIO]);
        }
      }
      bulk_wait_all();
    }
  } else if (warp == 3) {
    // ------------------------------------------------ MMA issuer
    // The whole warp walks the pipeline (uniform control flow: descriptors and stage indices
    // stay in uniform registers); one elected lane issues each stage (mma4/6_commit).
    // Descriptors are a per-mode template plus the stage's smem address; k-steps within a
    // stage are constant offsets (16-byte units):
    //   gather / s2d 3-D TMA (no swizzle, LBO = one 16-byte K plane of 128 rows): 256
    //   SWIZZLE_128B: 2          SWIZZLE_64B (two taps per stage): 0, 2, 512, 514
    //   s2d slab (no swizzle, LBO 16: the next K chunk is the next pixel): 0, 2, Wp, Wp + 2
    //   kw-reuse: A slab shifted by kw rows (4 units per kw), B resident chunk-major
    // B: no swizzle, LBO = one K plane of BN rows; K=32 step = 2 planes = 2*BN units.
    {
      // BR > BN: the MMA also covers the 16 K-indicator rows, so accumulator columns BN..BN+15
      // of every row hold that A row's sum
      const uint32_t idesc = idesc_i8<BR>();
      const int mode = a.tma_a;
      const uint32_t sa = smem_u32(sA), sb = smem_u32(sB);
      const bool nosw = mode == 0 || mode == 65;
      const uint64_t adt = a.kwr ? umma_desc_sw(0, 64)
                           : nosw ? umma_desc(0, TC_BM * 16, 128)
                           : mode == 67 ? umma_desc(0, 16, 128)
                           : mode == 128 ? umma_desc_sw(0, 128) : umma_desc_sw(0, 64);
      const uint64_t bdt = umma_desc(0, BR * 16, 128);
      const int Wp = a.in.W + 2 * a.in.halo;
      uint64_t a1, a2, a3;
      if (nosw) { a1 = 256; a2 = 512; a3 = 768; }
      else if (mode == 67) { a1 = 2; a2 = (uint64_t)Wp; a3 = (uint64_t)Wp + 2; }
      else if (mode == 128) { a1 = 2; a2 = 4; a3 = 6; }
      else { a1 = 2; a2 = 512; a3 = 514; }
      const uint64_t bstep = 2 * BR;
      if (a.b_res) mbar_wait(bfull, 0);
      int s = 0;
      uint32_t ph = 0, lt = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++lt) {
        const uint32_t buf = lt % G::NACC, uph = (lt / G::NACC) & 1u;
        mbar_wait(&tempty[buf], uph ^ 1u);           // epilogue drained this accumulator
        tc_fence_after();
        const uint32_t d = tmem + buf * (uint32_t)BR;
        for (int ki = 0; ki < a.a_iters; ++ki) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          if (mode == 0) fence_proxy_async();          // cp.async-written A -> async proxy
          const uint64_t ad = adt + ((sa + (uint32_t)s * TC_A_STAGE) >> 4);
          const uint32_t bar = smem_u32(&empty[s]);    // freed when the stage's MMAs land
          if (a.kwr) {
            // slab = input rows p0 + ki*Wp + [0, 136); tap (ki, kw) = the slab shifted by kw
            // rows (A: +4 units per kw, +2 per K half); B chunk ki*12 + kw*4 + 2*ks2
            mma6_commit(d, ad, bdt + (sb >> 4) + (uint64_t)(ki * 12 * BR), 2, bstep, idesc, ki != 0, bar);
          } else {
            const uint64_t bd = bdt + ((sb + (uint32_t)((a.b_res ? ki : s) * BR * 128)) >> 4);
            mma4_commit(d, ad, bd, a1, a2, a3, bstep, idesc, ki != 0, mode != 67 || 2 * ki + 1 < a.k, bar);
          }
          if (++s == NS) { s = 0; ph ^= 1u; }
        }
        commit_elect(&tfull[buf]);                   // accumulator ready for the epilogue
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------ epilogue warps
    // warp-uniform warp index (a shuffle from lane 0): q, grp, the chunk loop and the channel
    // base become uniform values, so the per-channel constants load into uniform registers
    const int wu = __shfl_sync(0xffffffffu, warp, 0);
    const int q = wu & 3;                            // TMEM lane quarter this warp may access
    const int grp = (wu - 4) >> 2;                   // column group (TC_NG groups per lane quarter)
    const int row = q * 32 + lane;
    const LayerRt rt = *a.L.rt;
    EpiK k;
    k.lo_conv = rt.relu_zp > PTQ_QMIN ? rt.relu_zp : PTQ_QMIN;
    k.lo_add = rt.add_relu_zp > PTQ_QMIN ? rt.add_relu_zp : PTQ_QMIN;
    k.clo = 0x80000000u - (uint32_t)rt.aclamp;
    k.chi = 0x80000000u + (uint32_t)rt.aclamp;
    const int Cout = a.L.cout;
    // stage the fused-add table (or the per-channel constants) in shared memory, then sync
    // the epilogue warps only (add layers read their constants from __constant__ c_ep)
    const int cs = (a.L.cout + 15) & ~15;
    if (!a.addtab)
      for (int i = threadIdx.x - 4 * 32; i < cs; i += TC_EPI_WARPS * 32) sparam[i] = a.L.ep[i];
    if (a.addtab)
      for (int i = threadIdx.x - 4 * 32; i < PTQ_ADDTAB_BYTES / 16; i += TC_EPI_WARPS * 32)
        reinterpret_cast<int4*>(stab)[i] = reinterpret_cast<const int4*>(a.addtab)[i];
    asm volatile("bar.sync 1, %0;" ::"n"(TC_EPI_WARPS * 32) : "memory");
    const int8_t* stab_c = stab + 128;                // column of conv code 0
    k.m0 = rt.m0;
    k.zw0 = rt.zw0;
    k.fxm0 = rt.fx_m0;
    k.fxs = rt.fx_s;

    const EpiEnv e{tmem, tfull, tempty, rsfull, rsum, reinterpret_cast<const uint8_t*>(sparam), cs, stab_c,
                   q, grp, row, M, n_tiles, n_nt, sio, iofull, ioempty, ioready};
    // one persistent tile loop per epilogue variant: the per-chunk code carries no
    // layer-level dispatch (that overhead was ~20% of the hot loop's instructions)
    const bool skip = a.skip.p != nullptr, wzp = a.has_wzp != 0, clamp = !rt.noclamp,
               relu = k.lo_conv > PTQ_QMIN;
    if (a.acc_out) epi_tiles<BN, false, false, false, false, true, true>(a, rt, k, e);
    else if (rt.fx && a.ablate != 1) {
      if (skip) { if (wzp) epi_fx<BN, true, true, false>(a, rt, k, e);
                  else epi_fx<BN, false, true, false>(a, rt, k, e); }
      else if (wzp) { if (relu) epi_fx<BN, true, false, true>(a, rt, k, e);
                      else epi_fx<BN, true, false, false>(a, rt, k, e); }
      else { if (relu) epi_fx<BN, false, false, true>(a, rt, k, e);
             else epi_fx<BN, false, false, false>(a, rt, k, e); }
    }
    else if (rt.slow || a.ablate == 1) epi_tiles<BN, false, false, false, false, true>(a, rt, k, e);
    else if (skip) {
      if (wzp) { if (clamp) epi_pt<BN, true, true, true, false>(a, rt, k, e);
                 else epi_pt<BN, true, true, false, false>(a, rt, k, e); }
      else { if (clamp) epi_pt<BN, false, true, true, false>(a, rt, k, e);
             else epi_pt<BN, false, true, false, false>(a, rt, k, e); }
    } else if (wzp) {
      if (clamp) { if (relu) epi_pt<BN, true, false, true, true>(a, rt, k, e);
                   else epi_pt<BN, true, false, true, false>(a, rt, k, e); }
      else { if (relu) epi_pt<BN, true, false, false, true>(a, rt, k, e);
             else epi_pt<BN, true, false, false, false>(a, rt, k, e); }
    } else {
      if (clamp) { if (relu) epi_pt<BN, false, false, true, true>(a, rt, k, e);
                   else epi_pt<BN, false, false, true, false>(a, rt, k, e); }
      else { if (relu) epi_pt<BN, false, false, false, true>(a, rt, k, e);
             else epi_pt<BN, false, false, false, false>(a, rt, k, e); }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 3) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------- CUDA-core reference
// Same contract, direct sum over the tiled weight image (tests / cross-checks only).
template <int BN>
__global__ void k_conv_i8_ref(const ConvTcArgs a) {
  const int M = a.in.N * a.OH * a.OW;
  const int Cout = a.L.cout;
  const int64_t total = (int64_t)M * a.out.Cp;
  const LayerRt rt = *a.L.rt;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % a.out.Cp);
    const int m = (int)(i / a.out.Cp);
    const RowGeo g = row_geo(a, m, M);
    int8_t* orow = a.out.p + vpix(a.out, g.n, g.oh, g.ow) * a.out.Cp;
    if (c >= Cout) { orow[c] = 0; continue; }
    const int Wp = a.in.W + 2 * a.in.halo, Hp = a.in.H + 2 * a.in.halo;
    const int cpc = a.in.Cp >> 4;
    const int ntile = c / BN, row = c % BN;
    long long dot = 0;
    for (int kk = 0; kk < a.n_chunks; ++kk) {
      const int tap = kk / cpc, ch = kk % cpc;
      const int kh = tap / a.k, kw = tap % a.k;
      const int8_t* xs = a.in.p + (((int64_t)g.n * Hp + g.ih0 + kh) * Wp + g.iw0 + kw) * a.in.Cp + ch * 16;
      const int8_t* ws = a.wB + (((int64_t)ntile * a.n_kiter + kk / 8) * 8 + kk % 8) * a.b_rows * 16 + row * 16;
      for (int b = 0; b < 16; ++b) dot += (long long)xs[b] * ws[b];
    }
    const long long rowsum = a.Rpix ? (long long)a.Rpix[((int64_t)g.n * a.OHr + g.oh) * a.OWr + g.ow]
                                    : pixel_rowsum(a, g.n, g.ih0, g.iw0);
    int q = epi_slow(dot, c, rowsum, a, rt);
    if (q < rt.relu_zp) q = rt.relu_zp;
    if (a.skip.p) {
      const int sk = a.skip.p[vpix(a.skip, g.n, g.oh, g.ow) * a.skip.Cp + c];
      const int xa = a.conv_is_a ? q : sk, xb = a.conv_is_a ? sk : q;
      const double s = __dadd_rn(__dmul_rn((double)(xa - rt.za), rt.ra), __dmul_rn((double)(xb - rt.zb), rt.rb));
      q = clip8(rhu(s) + (double)rt.zo);
      if (q < rt.add_relu_zp) q = rt.add_relu_zp;
    }
    orow[c] = (int8_t)q;
  }
}

int conv_tc_max_cout() { return TC_MAX_COUT; }

int conv_tc_bn_for(int cout) {
  if (cout <= 16) return 16;
  if (cout <= 32) return 32;
  if (cout <= 64) return 64;
  if (cout <= 128) return 128;
  return 256;
}


template <int BN, int BR>
static void launch_bn(const ConvTcArgs& a, cudaStream_t s) {
  // fixed part: barriers, TMEM slot, optional add table, resident B; the rest of the 227 KB
  // goes to pipeline stages (deeper for narrow tiles, at least 2)
  const int n_nt = (a.L.cout + BN - 1) / BN;
  const size_t b_bytes = (size_t)a.n_kiter * a.b_rows * 128;
  const int b_res = n_nt == 1 && b_bytes <= 64 * 1024;
  ConvTcArgs b = a;
  size_t smem = 0;
  int ns = 0;
  // tile I/O takes NIO [128][BN] buffers; without room for two pipeline stages beside
  // them the layer keeps the direct global epilogue
  for (int pass = 0; pass < 2; ++pass) {
    const size_t fixed = 1024 + (2 * TC_MAX_STAGES + 2 + 6 * TC_MAX_BUF) * 8 + TC_MAX_BUF * TC_BM * 4 + 16 +
                         (a.addtab ? PTQ_ADDTAB_BYTES : (size_t)((a.L.cout + 15) & ~15) * sizeof(EpiParam)) +
                         (b_res ? b_bytes : 0) + (b.tio ? (size_t)TcGeom<BN>::NIO * TC_BM * BN : 0);
    const size_t per_stage = (size_t)TC_A_STAGE + (b_res ? 0 : (size_t)a.b_rows * 128);
    ns = fixed < TC_SMEM_MAX ? (int)((TC_SMEM_MAX - fixed) / per_stage) : 0;
    if (ns < 2 && b.tio) { b.tio = 0; continue; }
    if (ns > TC_MAX_STAGES) ns = TC_MAX_STAGES;
    if (ns < 2) ns = 2;                // does not fit: the launch fails loudly (check_launch)
    smem = (size_t)ns * per_stage + fixed;
    break;
  }
  b.n_stages = ns;
  b.b_res = b_res;
  int dev = 0;
  cudaGetDevice(&dev);
  // the opt-in shared-memory limit is a per-device function attribute: raise it once per
  // device (a failure leaves the launch to fail loudly in check_launch)
  static std::atomic<uint64_t> configured{0};
  const uint64_t bit = 1ull << (dev & 63);
  if (!(configured.load() & bit) &&
      cudaFuncSetAttribute(k_conv_tc<BN, BR>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM_MAX) == cudaSuccess)
    configured.fetch_or(bit);
  int num_sms = 0;
  cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t M = (int64_t)a.in.N * a.OH * a.OW;
  const int64_t tiles = ((M + TC_BM - 1) / TC_BM) * ((a.L.cout + BN - 1) / BN);
  const int grid = (int)(tiles < num_sms ? tiles : num_sms);   // persistent: one CTA per SM
  // per-channel epilogue constants -> __constant__ c_ep with a stream-ordered copy right
  // before the launch.  c_ep is one per device, so launches of several contexts on one
  // device (other streams) are ordered through a per-device event: each copy waits for the
  // previous conv launch on that device to finish reading the constants.
  // cout <= TC_MAX_COUT is checked when the graph is imported (conv_tc_max_cout)
  static std::mutex mu;
  static cudaEvent_t last[64] = {};
  static cudaStream_t last_stream[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  const int d = dev & 63;
  if (!last[d]) cudaEventCreateWithFlags(&last[d], cudaEventDisableTiming);
  if (last_stream[d] && last_stream[d] != s) cudaStreamWaitEvent(s, last[d], 0);
  if (a.addtab)
    cudaMemcpyToSymbolAsync(c_ep, a.L.ep, (size_t)((a.L.cout + 15) & ~15) * sizeof(EpiParam), 0,
                            cudaMemcpyDeviceToDevice, s);
  k_conv_tc<BN, BR><<<grid, TC_THREADS, smem, s>>>(b);
  cudaEventRecord(last[d], s);
  last_stream[d] = s;
}

static ConvTcArgs with_divs(const ConvTcArgs& a0, int bn) {
  ConvTcArgs a = a0;
  if (!a.tma_a) { a.OHr = a.OH; a.OWr = a.OW; }
  a.div_ow = FastDiv::make((uint32_t)a.OW);
  a.div_oh = FastDiv::make((uint32_t)a.OH);
  a.div_nt = FastDiv::make((uint32_t)((a.L.cout + bn - 1) / bn));
  return a;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// TMA A path: stride-1 "same" convs whose input halo equals the padding (every 1x1 conv
// on a halo-free input, every 3x3 pad-1 conv) with 64 or 128k channel bytes
static bool setup_tma_a(ConvTcArgs& a) {
  const int Cp = a.in.Cp;
  if (!a.allow_tma || a.stride != 1 || a.in.halo != a.pad) return false;
  const int Hp = a.in.H + 2 * a.in.halo, Wp = a.in.W + 2 * a.in.halo;
  EncodeTiledFn fn = encode_tiled();
  if (!fn) return false;
  if (Cp == 16 && a.k == 4 && a.OH <= Hp - 3 && a.OW <= Wp - 3) {
    if (a.kwr_mode >= 0 && (Wp + TC_BM + 3) * 16 <= TC_A_STAGE) {
      // preferred: one contiguous bulk copy per stage (the input buffer carries the slack
      // the last tiles read past the grid; those rows only feed masked outputs)
      a.tma_a = 67;
      a.OHr = a.OH;
      a.OWr = a.OW;
      a.OH = Hp;
      a.OW = Wp;
      return true;
    }
    // preferred: overlapping 64-byte rows (4 consecutive 16-byte pixels) as a 2-D map with a
    // 16-byte row stride, loaded as SWIZZLE_64B boxes like the Cp == 64 path
    {
      cuuint64_t gdim[2] = {64, (cuuint64_t)a.in.N * Hp * Wp - 3};
      cuuint64_t gstride[1] = {16};
      cuuint32_t box[2] = {64, (cuuint32_t)TC_BM};
      cuuint32_t es[2] = {1, 1};
      if (fn(&a.tmA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)a.in.p, gdim, gstride, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS) {
        a.tma_a = 66;
        a.OHr = a.OH;
        a.OWr = a.OW;
        a.OH = Hp;
        a.OW = Wp;
        return true;
      }
    }
    // s2d stem: dims {16 B, pixels, 4 kw taps} with strides {16, 16} (the tap dimension
    // overlaps the pixel one): a box {16, 128, 4} lands as [tap][row][16 B], the no-swizzle
    // K-major layout of 4 K chunks, i.e. one kh row of taps for 128 GEMM rows
    cuuint64_t gdim[3] = {16, (cuuint64_t)a.in.N * Hp * Wp, 4};
    cuuint64_t gstride[2] = {16, 16};
    cuuint32_t box[3] = {16, (cuuint32_t)TC_BM, 4};
    cuuint32_t es[3] = {1, 1, 1};
    if (fn(&a.tmA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)a.in.p, gdim, gstride, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
    a.tma_a = 65;
    a.OHr = a.OH;
    a.OWr = a.OW;
    a.OH = Hp;
    a.OW = Wp;
    return true;
  }
  if (a.k != 2 * a.pad + 1) return false;
  if (!(Cp == 64 || Cp % 128 == 0) || a.OH != a.in.H || a.OW != a.in.W) return false;
  const int box0 = Cp == 64 ? 64 : 128;
  cuuint64_t gdim[2] = {(cuuint64_t)Cp, (cuuint64_t)a.in.N * Hp * Wp};
  cuuint64_t gstride[1] = {(cuuint64_t)Cp};
  cuuint32_t box[2] = {(cuuint32_t)box0, (cuuint32_t)TC_BM};
  cuuint32_t es[2] = {1, 1};
  if (fn(&a.tmA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)a.in.p, gdim, gstride, box, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, box0 == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  a.tma_a = box0;
  a.OHr = a.OH;
  a.OWr = a.OW;
  a.OH = Hp;                                         // GEMM rows = padded grid positions
  a.OW = Wp;
  return true;
}

// A-operand mode of one launch: TMA map (setup_tma_a), kw-reuse slabs, in-kernel row sums
static void plan_launch(ConvTcArgs& t, int bn) {
  t.tma_a = 0;
  setup_tma_a(t);
  t.kwr = 0;
  t.a_iters = t.n_kiter;
  if (t.tma_a == 64 && t.k == 3 && bn == 64 && t.L.cout <= 64 && t.kwr_mode >= 0 &&
      (size_t)t.n_kiter * 64 * 128 <= 64 * 1024) {    // needs the resident B of launch_bn
    // re-encode A with 136-row boxes: one slab per kh row of taps
    const int Hp = t.in.H + 2 * t.in.halo, Wp = t.in.W + 2 * t.in.halo;
    cuuint64_t gdim[2] = {64, (cuuint64_t)t.in.N * Hp * Wp};
    cuuint64_t gstride[1] = {64};
    cuuint32_t box[2] = {64, (cuuint32_t)(TC_BM + 8)};
    cuuint32_t es[2] = {1, 1};
    EncodeTiledFn fn = encode_tiled();
    if (fn && fn(&t.tmA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)t.in.p, gdim, gstride, box, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS) {
      t.kwr = 1;
      t.a_iters = 3;                                 // A stages per tile = kh rows
    }
  }
  t.tma_rowsum = t.has_wzp && !t.rs_mma && !t.Rpix && (t.tma_a == 64 || t.tma_a == 128);
  // flat rows: halo-free input and output, no padded-grid rows, halo-free add operand, and
  // row sums (when needed) taken in-kernel
  t.flat = (t.tma_a == 64 || t.tma_a == 128) && t.in.halo == 0 && t.out.halo == 0 && t.OH == t.OHr &&
           t.OW == t.OWr && (!t.skip.p || t.skip.halo == 0) &&
           (!t.has_wzp || t.tma_rowsum || t.rs_mma);
  // tile I/O for flat layers: the output (and the fused-add operand) as 2-D [pixels][Cp] maps
  // with boxes of 128 rows x io_w bytes, swizzled like the epilogue's shared tile
  t.tio = 0;
  if (t.flat && t.tio_mode && !t.acc_out && bn >= 64 && (t.out.Cp % 16) == 0) {
    EncodeTiledFn fn = encode_tiled();
    const int w = bn >= 128 ? 128 : 64;
    const int64_t M = (int64_t)t.in.N * t.OH * t.OW;
    auto enc = [&](CUtensorMap* m, const View& v) {
      cuuint64_t gdim[2] = {(cuuint64_t)v.Cp, (cuuint64_t)M};
      cuuint64_t gstride[1] = {(cuuint64_t)v.Cp};
      cuuint32_t box[2] = {(cuuint32_t)w, (cuuint32_t)TC_BM};
      cuuint32_t es[2] = {1, 1};
      return fn && fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)v.p, gdim, gstride, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, w == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    if (enc(&t.tmO, t.out) && (!t.skip.p || (t.skip.Cp == t.out.Cp && enc(&t.tmS, t.skip)))) {
      t.tio = 1;
      t.io_w = w;
    }
  }
}

bool conv_tc_tma_rowsum(const ConvTcArgs& a0, int bn) {
  ConvTcArgs t = a0;
  plan_launch(t, bn);
  return t.tma_rowsum != 0;
}

void launch_conv_tc(const ConvTcArgs& a0, int bn, cudaStream_t s) {
  ConvTcArgs t = a0;
  plan_launch(t, bn);
  const ConvTcArgs a = with_divs(t, bn);
  const bool ind = a.b_rows > bn;                   // tiles carry the K-indicator rows
  switch (bn) {
    case 16: ind ? launch_bn<16, 32>(a, s) : launch_bn<16, 16>(a, s); break;
    case 32: ind ? launch_bn<32, 48>(a, s) : launch_bn<32, 32>(a, s); break;
    case 64: ind ? launch_bn<64, 80>(a, s) : launch_bn<64, 64>(a, s); break;
    case 128: ind ? launch_bn<128, 144>(a, s) : launch_bn<128, 128>(a, s); break;
    default: launch_bn<256, 256>(a, s); break;
  }
}

void launch_conv_i8_ref(const ConvTcArgs& a0, int bn, cudaStream_t s) {
  const ConvTcArgs a = with_divs(a0, bn);
  const int64_t total = (int64_t)a.in.N * a.OH * a.OW * a.out.Cp;
  int64_t b = (total + 255) / 256;
  int blocks = (int)(b > 148 * 64 ? 148 * 64 : (b < 1 ? 1 : b));
  switch (bn) {
    case 16: k_conv_i8_ref<16><<<blocks, 256, 0, s>>>(a); break;
    case 32: k_conv_i8_ref<32><<<blocks, 256, 0, s>>>(a); break;
    case 64: k_conv_i8_ref<64><<<blocks, 256, 0, s>>>(a); break;
    case 128: k_conv_i8_ref<128><<<blocks, 256, 0, s>>>(a); break;
    default: k_conv_i8_ref<256><<<blocks, 256, 0, s>>>(a); break;
  }
}

}  // namespace ptq
