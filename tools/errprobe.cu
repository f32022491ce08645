// Dev probe: does a successful runtime call clear a pending launch error?
// (It does: cudaFuncSetAttribute resets cudaPeekAtLastError.)
//   nvcc -gencode arch=compute_100a,code=sm_100a -o build/errprobe tools/errprobe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void big(int* p) { extern __shared__ int s[]; __shared__ int t[4200]; t[threadIdx.x] = 1; s[threadIdx.x] = t[threadIdx.x]; p[threadIdx.x] = s[0]; }
__global__ void other(int* p) { p[0] = 1; }
int main() {
  int* d; cudaMalloc(&d, 4096);
  big<<<1, 32, 40000>>>(d);            // 16.8 KB static + 40 KB dynamic > 48 KB
  printf("peek after bad launch: %s\n", cudaGetErrorString(cudaPeekAtLastError()));
  cudaError_t e = cudaFuncSetAttribute(other, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024);
  printf("setattr returned: %s\n", cudaGetErrorString(e));
  printf("peek after setattr: %s\n", cudaGetErrorString(cudaPeekAtLastError()));
  e = cudaMemsetAsync(d, 0, 16, 0);
  printf("memset returned: %s; peek: %s\n", cudaGetErrorString(e), cudaGetErrorString(cudaPeekAtLastError()));
  other<<<1,1>>>(d);
  printf("get after good launch: %s\n", cudaGetErrorString(cudaGetLastError()));
  big<<<1, 32, 40000>>>(d);
  void* p; e = cudaMalloc(&p, 1 << 20);
  printf("malloc returned: %s; get: %s\n", cudaGetErrorString(e), cudaGetErrorString(cudaGetLastError()));
  return 0;
}
