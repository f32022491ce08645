// Standalone FP-add peak probe (first-pass measurement before the library exists).
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

template <int C>
__global__ void k_fadd(const float* __restrict__ s, float* out, int iters) {
  float acc[C], st[C];
#pragma unroll
  for (int c = 0; c < C; ++c) { acc[c] = 0.f; st[c] = s[(threadIdx.x + c) & 255]; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < C; ++c) acc[c] = __fadd_rn(acc[c], st[c]);
  }
  float r = 0.f;
#pragma unroll
  for (int c = 0; c < C; ++c) r += acc[c];
  if (r == 1234.5f) out[0] = r;
}

template <int C>
__global__ void k_fadd2(const float* __restrict__ s, float* out, int iters) {
  float2 acc[C / 2], st[C / 2];
#pragma unroll
  for (int c = 0; c < C / 2; ++c) {
    acc[c] = make_float2(0.f, 0.f);
    st[c] = make_float2(s[(threadIdx.x + 2 * c) & 255], s[(threadIdx.x + 2 * c + 1) & 255]);
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < C / 2; ++c) acc[c] = __fadd2_rn(acc[c], st[c]);
  }
  float r = 0.f;
#pragma unroll
  for (int c = 0; c < C / 2; ++c) r += acc[c].x + acc[c].y;
  if (r == 1234.5f) out[0] = r;
}

template <int C>
__global__ void k_dadd(const double* __restrict__ s, double* out, int iters) {
  double acc[C], st[C];
#pragma unroll
  for (int c = 0; c < C; ++c) { acc[c] = 0.0; st[c] = s[(threadIdx.x + c) & 255]; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < C; ++c) acc[c] = __dadd_rn(acc[c], st[c]);
  }
  double r = 0.0;
#pragma unroll
  for (int c = 0; c < C; ++c) r += acc[c];
  if (r == 1234.5) out[0] = r;
}

template <class K, class T>
double run(K kern, const T* s, T* out, int blocks, int threads, int iters, double adds_per_thread_iter) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) kern<<<blocks, threads>>>(s, out, iters);
  cudaEventRecord(a);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) kern<<<blocks, threads>>>(s, out, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double adds = adds_per_thread_iter * iters * (double)blocks * threads * reps;
  return adds / (ms * 1e-3);
}

int main() {
  float* sf; double* sd; float* of; double* od;
  cudaMalloc(&sf, 1024 * 4); cudaMalloc(&sd, 1024 * 8); cudaMalloc(&of, 64); cudaMalloc(&od, 64);
  float hf[1024]; double hd[1024];
  for (int i = 0; i < 1024; ++i) { hf[i] = 1e-7f * (i + 1); hd[i] = 1e-15 * (i + 1); }
  cudaMemcpy(sf, hf, sizeof hf, cudaMemcpyHostToDevice);
  cudaMemcpy(sd, hd, sizeof hd, cudaMemcpyHostToDevice);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("sms=%d clock_khz=%d\n", sms, clk);
  const int iters = 4096;
  int tpbs[] = {128, 256, 512, 1024};
  int bpsm[] = {1, 2, 4, 8};
  for (int t : tpbs) for (int bp : bpsm) {
    if (t * bp > 2048) continue;
    int blocks = sms * bp;
    double f4 = run(k_fadd<4>, sf, of, blocks, t, iters, 16 * 4);
    double f8 = run(k_fadd<8>, sf, of, blocks, t, iters, 16 * 8);
    double f16 = run(k_fadd<16>, sf, of, blocks, t, iters, 16 * 16);
    double g8 = run(k_fadd2<8>, sf, of, blocks, t, iters, 16 * 8);
    double g16 = run(k_fadd2<16>, sf, of, blocks, t, iters, 16 * 16);
    double d4 = run(k_dadd<4>, sd, od, blocks, t, iters / 4, 16 * 4);
    double d8 = run(k_dadd<8>, sd, od, blocks, t, iters / 4, 16 * 8);
    printf("tpb=%4d bpsm=%d  FADD c4 %.3e c8 %.3e c16 %.3e | FADD2 c8 %.3e c16 %.3e | DADD c4 %.3e c8 %.3e adds/s\n",
           t, bp, f4, f8, f16, g8, g16, d4, d8);
  }
  cudaError_t e = cudaGetLastError();
  printf("err=%s\n", cudaGetErrorString(e));
  return 0;
}
