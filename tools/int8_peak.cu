// Measured int8 tensor-core peak of this B200 (the roofline denominator of F4, k_conv_tc).
//
// A persistent tcgen05 kind::i8 GEMM, C[M][N] (s32) = A[M][K] (s8) x B[N][K]^T (s8), both
// operands K-major and TMA-loaded as SWIZZLE_128B boxes (A 128 x 128 B, B 256 x 128 B per
// stage), M=128 x N=256 x K=32 per tcgen05.mma issued by one thread, two TMEM accumulators
// (512 columns) so tile t+1's MMAs overlap tile t's drain, 4 epilogue warps storing s32.
// This is the contraction the reference performs as an exact float64 dgemm
// (/root/reference/pkg/src/ptqtune/intexec.py:95-105) at its densest.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/int8_peak tools/int8_peak.cu
//   build/int8_peak [M N K] [sustain_seconds]   -> one JSON line
//
// Burst = best of 10 back-to-back launches; sustained = mean over a >= sustain_seconds loop.
// Two modes: the full GEMM (operands streamed every K stage) and mma_only (the same MMA
// stream on operand stages loaded once: the tensor-pipe rate without L2 traffic).
// Correctness: 4096 random C entries checked against a host int64 dot product.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess) {                                                             \
      std::fprintf(stderr, "%s -> %s\n", #x, cudaGetErrorString(e_));                  \
      std::exit(1);                                                                      \
    }                                                                                    \
  } while (0)

constexpr int BM = 128, BN = 256, BK = 128;   // BK in bytes (= int8 elements) per stage
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK, B_BYTES = BN * BK, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int THREADS = 256;                   // warp 0 TMA, warp 1 MMA, warps 4-7 epilogue

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, 10000000;\n\t"
      "@!P1 bra W_%=;\n\t}" ::"r"(su32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          su32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;          // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;                    // SWIZZLE_128B
  return d;
}
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

__global__ void __launch_bounds__(THREADS, 1)
    k_gemm_i8(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int32_t* C,
              int M, int N, int K, int mma_only) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = M / BM, nt = N / BN, tiles = mt * nt, kit = K / BK;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 128); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  if (warp == 0 && lane == 0 && mma_only) {
    // tensor-pipe peak: the operand stages are loaded once and re-used by every MMA, so the
    // loop measures the MMA issue rate with no L2 / TMA traffic in it
    for (int s = 0; s < STAGES; ++s) {
      uint8_t* st = smem + s * STAGE_BYTES;
      mbar_expect(&full[s], STAGE_BYTES);
      tma2d(st, &tmA, s * BK, 0, &full[s]);
      tma2d(st + A_BYTES, &tmB, s * BK, 0, &full[s]);
    }
  } else if (warp == 0 && lane == 0) {
    int s = 0;
    uint32_t ph = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      const int m0 = (t / nt) * BM, n0 = (t % nt) * BN;
      for (int k = 0; k < kit; ++k) {
        mbar_wait(&empty[s], ph ^ 1u);
        uint8_t* st = smem + s * STAGE_BYTES;
        mbar_expect(&full[s], STAGE_BYTES);
        tma2d(st, &tmA, k * BK, m0, &full[s]);
        tma2d(st + A_BYTES, &tmB, k * BK, n0, &full[s]);
        if (++s == STAGES) { s = 0; ph ^= 1u; }
      }
    }
  } else if (warp == 1 && lane == 0) {
    int s = 0;
    uint32_t ph = 0, lt = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++lt) {
      const uint32_t buf = lt & 1u, uph = (lt >> 1) & 1u;
      mbar_wait(&tempty[buf], uph ^ 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t d = tmem + buf * BN;
      for (int k = 0; k < kit; ++k) {
        if (!mma_only) mbar_wait(&full[s], ph);
        else if (lt == 0 && k < STAGES) mbar_wait(&full[s], 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t a0 = su32(smem + s * STAGE_BYTES), b0 = a0 + A_BYTES;
#pragma unroll
        for (int ks = 0; ks < BK / 32; ++ks) {
          const uint64_t ad = desc_sw128(a0 + ks * 32), bd = desc_sw128(b0 + ks * 32);
          const uint32_t acc = (k | ks) != 0;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
              "l"(ad), "l"(bd), "r"(IDESC), "r"(acc));
        }
        if (!mma_only)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           su32(&empty[s]))
                       : "memory");
        if (++s == STAGES) { s = 0; ph ^= 1u; }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       su32(&tfull[buf]))
                   : "memory");
    }
  } else if (warp >= 4) {
    const int q = warp & 3, row = q * 32 + lane;
    uint32_t lt = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++lt) {
      const uint32_t buf = lt & 1u, uph = (lt >> 1) & 1u;
      const int m0 = (t / nt) * BM, n0 = (t % nt) * BN;
      mbar_wait(&tfull[buf], uph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      int32_t* crow = C + (int64_t)(m0 + row) * N + n0;
#pragma unroll 1
      for (int c = 0; c < BN / 16; ++c) {
        uint32_t v[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(tmem + ((uint32_t)(q * 32) << 16) + buf * BN + c * 16));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 4; ++j)
          reinterpret_cast<int4*>(crow + c * 16)[j] =
              make_int4((int)v[4 * j], (int)v[4 * j + 1], (int)v[4 * j + 2], (int)v[4 * j + 3]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&tempty[buf]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static CUtensorMap make_map(EncodeFn fn, void* p, int rows, int K, int box_rows) {
  CUtensorMap m;
  cuuint64_t gdim[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t gstride[1] = {(cuuint64_t)K};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  if (fn(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, p, gdim, gstride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS) {
    std::fprintf(stderr, "cuTensorMapEncodeTiled failed\n");
    std::exit(1);
  }
  return m;
}

int main(int argc, char** argv) {
  int M = 8192, N = 8192, K = 8192;
  double sustain_s = 4.0;
  if (argc >= 4) { M = std::atoi(argv[1]); N = std::atoi(argv[2]); K = std::atoi(argv[3]); }
  if (argc >= 5) sustain_s = std::atof(argv[4]);
  if (M % BM || N % BN || K % BK) { std::fprintf(stderr, "M %% 128, N %% 256, K %% 128 required\n"); return 1; }
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  std::vector<int8_t> hA((size_t)M * K), hB((size_t)N * K);
  std::mt19937 rng(1234);
  for (auto& v : hA) v = (int8_t)(rng() & 0xff);
  for (auto& v : hB) v = (int8_t)(rng() & 0xff);
  int8_t *dA, *dB;
  int32_t* dC;
  CK(cudaMalloc(&dA, hA.size()));
  CK(cudaMalloc(&dB, hB.size()));
  CK(cudaMalloc(&dC, (size_t)M * N * 4));
  CK(cudaMemcpy(dA, hA.data(), hA.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hB.data(), hB.size(), cudaMemcpyHostToDevice));
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult qr;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &qr));
  EncodeFn enc = reinterpret_cast<EncodeFn>(fp);
  CUtensorMap tA = make_map(enc, dA, M, K, BM), tB = make_map(enc, dB, N, K, BN);
  const int smem = STAGES * STAGE_BYTES + 1024 + 256;
  CK(cudaFuncSetAttribute(k_gemm_i8, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int tiles = (M / BM) * (N / BN);
  const int grid = tiles < prop.multiProcessorCount ? tiles : prop.multiProcessorCount;
  int mma_only = 0;
  auto launch = [&] { k_gemm_i8<<<grid, THREADS, smem>>>(tA, tB, dC, M, N, K, mma_only); };
  for (int i = 0; i < 3; ++i) launch();
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  // correctness on random entries
  std::vector<int32_t> hC((size_t)M * N);
  CK(cudaMemcpy(hC.data(), dC, hC.size() * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int i = 0; i < 4096; ++i) {
    const int r = rng() % M, c = rng() % N;
    long long s = 0;
    for (int k = 0; k < K; ++k) s += (long long)hA[(size_t)r * K + k] * hB[(size_t)c * K + k];
    if ((int32_t)s != hC[(size_t)r * N + c]) ++bad;
  }
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const double ops = 2.0 * M * N * (double)K;
  auto measure = [&](double& burst_ms, double& sust_ms, int& n) {
    for (int i = 0; i < 3; ++i) launch();
    float best = 1e30f;
    for (int i = 0; i < 10; ++i) {
      CK(cudaEventRecord(e0));
      launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (ms < best) best = ms;
    }
    const int per = std::max(1, (int)(sustain_s * 1000.0 / best / 4));
    n = 0;
    float total = 0.f;
    auto t0 = std::chrono::steady_clock::now();
    while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < sustain_s) {
      CK(cudaEventRecord(e0));
      for (int i = 0; i < per; ++i) launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      total += ms;
      n += per;
    }
    CK(cudaGetLastError());
    burst_ms = best;
    sust_ms = total / n;
  };
  double gb, gs, mb, ms_;
  int gn, mn;
  measure(gb, gs, gn);
  mma_only = 1;
  measure(mb, ms_, mn);
  std::printf("{\"kernel\": \"tcgen05.mma.cta_group::1.kind::i8 M128 N256 K32, TMA SWIZZLE_128B, %d stages, "
              "persistent %d CTAs\", \"M\": %d, \"N\": %d, \"K\": %d, "
              "\"gemm\": {\"burst_ms\": %.4f, \"tops_burst\": %.1f, \"sustained_ms\": %.4f, \"tops_sustained\": %.1f, "
              "\"launches\": %d, \"note\": \"A/B streamed by TMA from L2/HBM every K stage\"}, "
              "\"mma_only\": {\"burst_ms\": %.4f, \"tops_burst\": %.1f, \"sustained_ms\": %.4f, \"tops_sustained\": %.1f, "
              "\"launches\": %d, \"note\": \"same MMAs and epilogue, operand stages loaded once (tensor-pipe issue rate)\"}, "
              "\"check_bad\": %d, \"check_n\": 4096, \"device\": \"%s\", \"sms\": %d}\n",
              STAGES, grid, M, N, K, gb, ops / (gb * 1e-3) / 1e12, gs, ops / (gs * 1e-3) / 1e12, gn, mb,
              ops / (mb * 1e-3) / 1e12, ms_, ops / (ms_ * 1e-3) / 1e12, mn, bad, prop.name, prop.multiProcessorCount);
  return bad ? 2 : 0;
}
