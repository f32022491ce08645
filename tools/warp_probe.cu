// FADD2 issue-rate probe: adds/clk/SM as a function of warps per SM
// sub-partition, with the product kernel's chain shape (16 independent float2
// accumulators per lane, one register-held step each). Answers "how many
// FP-phase warps does an SMSP need to keep the FMA pipe busy?" (dev tool).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/warp_probe tools/warp_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void k_fadd2(const float* __restrict__ s, float* out, int iters,
                        long long* cycles) {
  float2 acc[C], st[C];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    acc[c] = make_float2(0.f, 0.f);
    st[c] = make_float2(s[(threadIdx.x + 2 * c) & 255], s[(threadIdx.x + 2 * c + 1) & 255]);
  }
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int c = 0; c < C; ++c) acc[c] = __fadd2_rn(acc[c], st[c]);
  }
  const long long t1 = clock64();
  float r = 0.f;
#pragma unroll
  for (int c = 0; c < C; ++c) r += acc[c].x + acc[c].y;
  if (r == 1234.5f) out[0] = r;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* s;
  long long* cyc;
  cudaMalloc(&s, 1024 * sizeof(float));
  cudaMemset(s, 0, 1024 * sizeof(float));
  cudaMalloc(&cyc, sms * sizeof(long long));
  const int iters = 4096;
  for (int wps : {1, 2, 3, 4, 6, 8}) {
    const int threads = 128 * wps;  // wps warps on each of the 4 SMSPs
    for (int rep = 0; rep < 2; ++rep) k_fadd2<16><<<sms, threads>>>(s, s + 512, iters, cyc);
    cudaDeviceSynchronize();
    long long h[1024];
    cudaMemcpy(h, cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < sms; ++i) mean += (double)h[i];
    mean /= sms;
    const double adds = (double)threads * iters * 4 * 16 * 2;  // per SM
    printf("warps/SMSP %d: %.1f adds/clk/SM (%.1f%% of 128)\n", wps, adds / mean,
           100.0 * adds / mean / 128.0);
  }
  return 0;
}
