// TMEM -> register read bandwidth probe (dev tool): can tensor memory feed the
// repeated-addition kernel's bases faster than shared memory (128 B/clk/SM)?
// Each warp repeatedly loads 32 columns x 32 lanes (4 KB) of its lane quadrant
// with tcgen05.ld.32x32b.x32 and folds the registers with FADD2 chains so the
// loads cannot be elided; reports bytes/clk/SM for several warp counts, next
// to the same loop fed by ld.shared.v4 for comparison.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/tmem_probe tools/tmem_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void fold(float2* acc, const uint32_t* r) {
#pragma unroll
  for (int i = 0; i < 16; ++i)
    acc[i & 7] = __fadd2_rn(acc[i & 7], make_float2(__uint_as_float(r[2 * i]),
                                                    __uint_as_float(r[2 * i + 1])));
}

template <bool TMEM, int FOLD>
__global__ void k_probe(int iters, long long* cycles, float* sink) {
  __shared__ uint32_t tbase;
  __shared__ __align__(16) uint32_t sm[32 * 32 * 8];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 32 * 32 * 8; i += blockDim.x) sm[i] = 0;
  if (TMEM && warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t taddr = tbase + ((warp & 3u) * 32u << 16);
  float2 acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = make_float2(0.f, 0.f);
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t r[32];
    const uint32_t col = (it * 32u) & 511u;
    if (TMEM) {
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
          "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
            "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
            "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
            "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
            "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
            "=r"(r[31])
          : "r"(taddr + col));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    } else {
      const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm) + (it & 7) * 4096 + lane * 16;
#pragma unroll
      for (int g = 0; g < 8; ++g)
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r[4 * g]), "=r"(r[4 * g + 1]), "=r"(r[4 * g + 2]), "=r"(r[4 * g + 3])
                     : "r"(base + g * 512));
    }
#pragma unroll
    for (int f = 0; f < FOLD; ++f) fold(acc, r);
  }
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i].x + acc[i].y;
  if (s == 1234.5f) sink[0] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (TMEM && warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

template <bool TMEM, int FOLD>
void run(int sms, long long* cyc, float* sink) {
  const int iters = 4096;
  for (int warps : {4, 8, 16}) {
    k_probe<TMEM, FOLD><<<sms, warps * 32>>>(iters, cyc, sink);
    k_probe<TMEM, FOLD><<<sms, warps * 32>>>(iters, cyc, sink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(e));
      return;
    }
    long long h[256];
    cudaMemcpy(h, cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < sms; ++i) mean += (double)h[i];
    mean /= sms;
    const double bytes = (double)warps * iters * 4096;
    const double adds = (double)warps * 32 * iters * 32 * FOLD;
    printf("%s fold=%d warps=%2d: %.1f B/clk/SM, %.1f adds/clk/SM\n", TMEM ? "tmem" : "smem", FOLD,
           warps, bytes / mean, adds / mean);
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* cyc;
  float* sink;
  cudaMalloc(&cyc, 256 * sizeof(long long));
  cudaMalloc(&sink, 64);
  run<true, 1>(sms, cyc, sink);
  run<false, 1>(sms, cyc, sink);
  run<true, 2>(sms, cyc, sink);
  run<false, 2>(sms, cyc, sink);
  return 0;
}
