// TMEM -> register read bandwidth on one B200 (tcgen05.ld), the resource the k_conv_tc
// epilogue drains every int32 accumulator through.  One persistent CTA per SM allocates 512
// TMEM columns; W warps (W/4 per TMEM lane quarter) each loop over their quarter's columns with
// tcgen05.ld.sync.aligned.32x32b.xN (N = 16, 32, 64) and `inflight` loads before one
// tcgen05.wait::ld.  Prints bytes per SM-cycle (clock from SM %clock64 deltas).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_bw tools/tmem_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int N>
__device__ __forceinline__ void ld(uint32_t taddr, uint32_t (&v)[N]);
template <>
__device__ __forceinline__ void ld<16>(uint32_t t, uint32_t (&v)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                 "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
               : "r"(t));
}
template <>
__device__ __forceinline__ void ld<32>(uint32_t t, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,"
      "%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(t));
}
// 16x256b: 16 TMEM lanes x 256 bits (8 columns) per x1; x8 = 64 columns, 32 regs per thread
__device__ __forceinline__ void ld16x256b_x4(uint32_t t, uint32_t (&v)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                 "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
               : "r"(t));
}

template <int N, int MODE>
__global__ void __launch_bounds__(512, 1) k_tmem_bw(int iters, int nwarps, unsigned long long* out_cycles,
                                                    uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  uint32_t acc = 0;
  unsigned long long t0 = clock64();
  if (warp < nwarps) {
    const int q = warp & 3, grp = warp >> 2, ng = nwarps / 4;
    const uint32_t base = tmem + ((uint32_t)(q * 32) << 16);
    for (int it = 0; it < iters; ++it) {
      // this warp's share of the 512 columns, N columns per load
      for (int c = grp * N; c < 512; c += ng * N) {
        if (MODE == 0) {
          uint32_t v[N];
          ld<N>(base + c, v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < N; ++j) acc ^= v[j];
        } else {
          uint32_t v[16];
          ld16x256b_x4(base + c, v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 16; ++j) acc ^= v[j];
        }
      }
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out_cycles[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) sink[0] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, int MODE>
static void run(int nwarps, int sms, unsigned long long* d_cyc, uint32_t* d_sink) {
  const int iters = 2000;
  k_tmem_bw<N, MODE><<<sms, 512>>>(10, nwarps, d_cyc, d_sink);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { std::printf("warmup failed: %s\n", cudaGetErrorString(e)); return; }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_tmem_bw<N, MODE><<<sms, 512>>>(iters, nwarps, d_cyc, d_sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  unsigned long long cyc[256];
  cudaMemcpy(cyc, d_cyc, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  double mc = 0;
  for (int i = 0; i < sms; ++i) mc += (double)cyc[i];
  mc /= sms;
  const double bytes_per_sm = (double)iters * 128 * 512 * 4;   // 128 lanes x 512 columns x 4 B
  std::printf("{\"shape\": \"%s\", \"N\": %d, \"warps\": %d, \"ms\": %.3f, \"B_per_clk_per_sm\": %.1f, "
              "\"TB_per_s\": %.2f, \"err\": \"%s\"}\n",
              MODE == 0 ? "32x32b" : "16x256b.x4", N, nwarps, ms, bytes_per_sm / mc,
              bytes_per_sm * sms / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

#define CKE(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { std::printf("error %s at %d\n", cudaGetErrorString(e_), __LINE__); std::fflush(stdout); return 1; } } while (0)
int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  std::printf("start\n");
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d_cyc;
  uint32_t* d_sink;
  CKE(cudaMalloc(&d_cyc, 256 * sizeof(unsigned long long)));
  CKE(cudaMalloc(&d_sink, 64));
  std::printf("sms %d\n", sms);
  for (int w : {4, 8, 12, 16}) {
    run<16, 0>(w, sms, d_cyc, d_sink);
    run<32, 0>(w, sms, d_cyc, d_sink);
    run<16, 1>(w, sms, d_cyc, d_sink);
  }
  return 0;
}
