// Prototype (dev tool): k_bladder -- R B-form rows per warp walking k densely
// with every row's rep (0..255) in one u64 per (group, k); per row one
// brx.idx into a fall-through ladder of 8 FADD2 steps (plus trips of 8 for
// larger reps). The mid-rep analogue of k_bgroup's jump tables: the bases of
// a k are loaded once for R rows and the per-row control is one indirect
// branch instead of k_bform's per-entry list walk / seek / rep loop.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xptxas -v \
//        -o build/ladder_proto tools/ladder_proto.cu -lcuda
//   build/ladder_proto <n> <dist: unif|const|geom|cfg5> <param>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <algorithm>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include "../paper_1308_2400_b200/csrc/common.cuh"

using namespace afmm_dev;

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

constexpr int KB = 8;
constexpr int NV = 8;        // float2 per lane per row (16 fp32 columns)
constexpr int TILE_N = 512;  // columns per CTA
constexpr int STAGE_BYTES = KB * TILE_N * 4;

__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}


#define STEP8(OP)                                                                                 \
  OP " %0, %0, %8;\n\t" OP " %1, %1, %9;\n\t" OP " %2, %2, %10;\n\t" OP " %3, %3, %11;\n\t" OP \
     " %4, %4, %12;\n\t" OP " %5, %5, %13;\n\t" OP " %6, %6, %14;\n\t" OP " %7, %7, %15;\n\t"
#define OPS8(a, b)                                                                              \
  : "+l"(a[0]), "+l"(a[1]), "+l"(a[2]), "+l"(a[3]), "+l"(a[4]), "+l"(a[5]), "+l"(a[6]),       \
    "+l"(a[7])                                                                                  \
  : "l"(b[0]), "l"(b[1]), "l"(b[2]), "l"(b[3]), "l"(b[4]), "l"(b[5]), "l"(b[6]), "l"(b[7])

// t sequential steps (any t): trips of 8, then one brx.idx into the ladder.
__device__ __forceinline__ void row_steps(unsigned long long* a, const unsigned long long (&b)[8],
                                          uint32_t t) {
#pragma unroll 1
  while (t > 8) {
    asm volatile("{\n\t" STEP8("add.rn.f32x2") STEP8("add.rn.f32x2") STEP8("add.rn.f32x2")
                     STEP8("add.rn.f32x2") STEP8("add.rn.f32x2") STEP8("add.rn.f32x2")
                         STEP8("add.rn.f32x2") STEP8("add.rn.f32x2") "}" OPS8(a, b));
    t -= 8;
  }
  const uint32_t idx = 8u - t;
  asm volatile(
      "{\n\t"
      "Lt%=: .branchtargets L8%=, L7%=, L6%=, L5%=, L4%=, L3%=, L2%=, L1%=, L0%=;\n\t"
      "brx.idx %16, Lt%=;\n\t"
      "L8%=:\n\t" STEP8("add.rn.f32x2") "L7%=:\n\t" STEP8("add.rn.f32x2") "L6%=:\n\t" STEP8(
          "add.rn.f32x2") "L5%=:\n\t" STEP8("add.rn.f32x2") "L4%=:\n\t" STEP8("add.rn.f32x2")
          "L3%=:\n\t" STEP8("add.rn.f32x2") "L2%=:\n\t" STEP8("add.rn.f32x2") "L1%=:\n\t" STEP8(
              "add.rn.f32x2") "L0%=:\n\t"
      "}" OPS8(a, b), "r"(idx));
}

template <int R, int CW, int STAGES>
__global__ void __launch_bounds__((CW + 1) * 32, 1)
    k_bladder(const __grid_constant__ CUtensorMap tb, const unsigned long long* __restrict__ reps,
              uint32_t ngroups, uint32_t nrows, uint32_t nk, float* __restrict__ out, uint64_t ld_out) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  const int32_t tile_c = blockIdx.y * TILE_N;
  const uint32_t nkb = (nk + KB - 1) / KB;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (warp == CW) {
    if (lane == 0) {
      prefetch_tensormap(&tb);
      for (uint32_t i = 0; i < nkb; ++i) {
        const uint32_t slot = i % STAGES;
        if (i >= STAGES) mbar_sleep_wait_at(smem_u32(&empty[slot]), ((i / STAGES) - 1) & 1);
        mbar_arrive_expect_tx(&full[slot], (uint32_t)STAGE_BYTES);
        unsigned char* st = base + slot * STAGE_BYTES;
        tma_load_2d(st, &tb, &full[slot], tile_c, (int32_t)(i * KB));
        tma_load_2d(st + KB * 1024, &tb, &full[slot], tile_c + 256, (int32_t)(i * KB));
      }
    }
    return;
  }
  const uint32_t g = blockIdx.x * CW + warp;
  const bool active = g < ngroups;
  const unsigned long long* __restrict__ rp = reps + (uint64_t)(active ? g : 0) * nk;
  unsigned long long acc[R * NV];
#pragma unroll
  for (int i = 0; i < R * NV; ++i) acc[i] = 0ull;
  const uint32_t ring = smem_u32(base) + lane * 16;
  uint32_t slot = 0, phase = 0;
  for (uint32_t kb = 0; kb < nkb; ++kb) {
    mbar_sleep_wait_at(smem_u32(&full[slot]), phase);
    if (active) {
      if (kb + 4 < nkb) asm volatile("prefetch.global.L1 [%0];" ::"l"(rp + (kb + 4) * KB));
      const uint32_t sa = ring + slot * STAGE_BYTES;
#pragma unroll 1
      for (int kk = 0; kk < KB; ++kk) {
        const unsigned long long rv = __ldg(rp + kb * KB + kk);
        if (rv == 0ull) continue;
        const uint32_t ra = sa + kk * 1024;
        unsigned long long b[NV];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];"
                       : "=l"(b[2 * q]), "=l"(b[2 * q + 1])
                       : "r"(ra + (q >> 1) * KB * 1024 + (q & 1) * 512));
        }
#pragma unroll
        for (int r = 0; r < R; ++r) row_steps(acc + r * NV, b, (uint32_t)(rv >> (8 * r)) & 0xffu);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive_at(smem_u32(&empty[slot]));
    if (++slot == STAGES) { slot = 0; phase ^= 1; }
  }
  if (!active) return;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const uint32_t row = g * R + r;
    if (row >= nrows) break;
    float* o = out + (uint64_t)row * ld_out + tile_c;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const unsigned long long x = acc[r * NV + 2 * q], y = acc[r * NV + 2 * q + 1];
      *reinterpret_cast<float4*>(o + (q >> 1) * 256 + (q & 1) * 128 + lane * 4) =
          make_float4(__uint_as_float((uint32_t)x), __uint_as_float((uint32_t)(x >> 32)),
                      __uint_as_float((uint32_t)y), __uint_as_float((uint32_t)(y >> 32)));
    }
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

static uint64_t rng_state = 88172645463325252ull;
static inline uint64_t xr() {
  rng_state ^= rng_state << 13; rng_state ^= rng_state >> 7; rng_state ^= rng_state << 17;
  return rng_state;
}

template <int R, int CW, int STAGES>
void run(uint32_t n, const float* dB, float* dZ, const std::vector<float>& B, const std::vector<uint8_t>& Rp,
         double adds, const char* tag) {
  const uint32_t ngroups = (n + R - 1) / R;
  std::vector<unsigned long long> reps((size_t)ngroups * n, 0ull);
  for (uint32_t g = 0; g < ngroups; ++g)
    for (int r = 0; r < R; ++r) {
      const uint32_t row = g * R + r;
      if (row >= n) break;
      for (uint32_t k = 0; k < n; ++k) reps[(size_t)g * n + k] |= (unsigned long long)Rp[(size_t)row * n + k] << (8 * r);
    }
  unsigned long long* dR;
  CK(cudaMalloc(&dR, reps.size() * 8));
  CK(cudaMemcpy(dR, reps.data(), reps.size() * 8, cudaMemcpyHostToDevice));
  auto fn = enc();
  CUtensorMap tb;
  cuuint64_t gdim[2] = {n, n};
  cuuint64_t gstr[1] = {(cuuint64_t)n * 4};
  cuuint32_t box[2] = {256, KB};
  cuuint32_t es[2] = {1, 1};
  if (fn(&tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)dB, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("tmap failed\n"); exit(1);
  }
  const size_t smem = 1024 + STAGES * STAGE_BYTES + 2 * STAGES * 8;
  auto kern = k_bladder<R, CW, STAGES>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((ngroups + CW - 1) / CW, n / TILE_N);
  CK(cudaMemset(dZ, 0xff, (size_t)n * n * 4));
  kern<<<grid, (CW + 1) * 32, smem>>>(tb, dR, ngroups, n, n, dZ, n);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> z((size_t)n);
  int bad_rows = 0;
  for (int si = 0; si < 16; ++si) {
    const uint32_t i = (uint32_t)((uint64_t)si * (n - 1) / 15);
    CK(cudaMemcpy(z.data(), dZ + (size_t)i * n, n * 4, cudaMemcpyDeviceToHost));
    std::vector<float> acc(n, 0.f);
    for (uint32_t k = 0; k < n; ++k) {
      const int t = Rp[(size_t)i * n + k];
      if (!t) continue;
      const float* brow = &B[(size_t)k * n];
      for (uint32_t j = 0; j < n; ++j) {
        float a = acc[j];
        for (int u = 0; u < t; ++u) a = a + brow[j];
        acc[j] = a;
      }
    }
    if (memcmp(acc.data(), z.data(), n * 4) != 0) ++bad_rows;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int it = 0; it < 3; ++it) {
    cudaEventRecord(e0);
    kern<<<grid, (CW + 1) * 32, smem>>>(tb, dR, ngroups, n, n, dZ, n);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = std::min(best, ms);
  }
  const double rate = adds / (best * 1e-3);
  printf("%-22s R=%d CW=%d ST=%d grid=%ux%u  %.3f ms  %.4e adds/s  frac %.3f  rows-bad %d/16\n",
         tag, R, CW, STAGES, grid.x, grid.y, best, rate, rate / 3.71e13, bad_rows);
  cudaFree(dR);
}

int main(int argc, char** argv) {
  const uint32_t n = argc > 1 ? atoi(argv[1]) : 4096;
  const char* dist = argc > 2 ? argv[2] : "unif";
  const int param = argc > 3 ? atoi(argv[3]) : 4;
  std::vector<float> B((size_t)n * n);
  std::vector<uint8_t> Rp((size_t)n * n);
  for (auto& v : B) v = (float)((double)(xr() >> 11) / 9007199254740992.0 * 2.0 - 1.0);
  double adds = 0;
  for (auto& r : Rp) {
    int t;
    const double u = (double)(xr() >> 11) / 9007199254740992.0;
    if (!strcmp(dist, "const")) t = param;
    else if (!strcmp(dist, "unif")) t = (int)(xr() % (uint64_t)(2 * param + 1));
    else if (!strcmp(dist, "cfg5")) t = u < 0.9 ? (int)(xr() % 32) : 0;
    else {  // geometric mean param capped at 64
      t = 1;
      while (t < 64 && (double)(xr() >> 11) / 9007199254740992.0 >= 1.0 / param) ++t;
    }
    r = (uint8_t)t;
    adds += t;
  }
  adds *= n;
  float *dB, *dZ;
  CK(cudaMalloc(&dB, (size_t)n * n * 4));
  CK(cudaMalloc(&dZ, (size_t)n * n * 4));
  CK(cudaMemcpy(dB, B.data(), (size_t)n * n * 4, cudaMemcpyHostToDevice));
  char tag[64];
  snprintf(tag, sizeof tag, "n=%u %s %d", n, dist, param);
  run<2, 16, 12>(n, dB, dZ, B, Rp, adds, tag);
  run<3, 16, 12>(n, dB, dZ, B, Rp, adds, tag);
  run<4, 15, 12>(n, dB, dZ, B, Rp, adds, tag);
  run<5, 15, 12>(n, dB, dZ, B, Rp, adds, tag);
  return 0;
}
