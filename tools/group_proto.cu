// Prototype (dev tool): k_bgroup -- R B-form rows per warp over merged
// group lists {k, idx}, one brx.idx jump-table dispatch per entry
// (tools/gen_jumptable.py). Each staged base row is loaded from smem once for
// R rows: at small reps the R = 1 kernel is bound by the shared-memory reads
// of the bases (4 B per add at rep 1).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xptxas -v \
//        -o build/group_proto tools/group_proto.cu -lcuda
//   build/group_proto <n> <dist: unif|const> <param>
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
#include "../paper_1308_2400_b200/csrc/jumptable.inc"

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

template <int R1, int R2, int T, int CW, int STAGES>
__global__ void __launch_bounds__((CW + 1) * 32, 1)
    k_bgroup(const __grid_constant__ CUtensorMap tb, const int2* __restrict__ lists, uint64_t cap,
             const uint32_t* __restrict__ counts, uint32_t ngroups, uint32_t nrows, uint32_t nk,
             float* __restrict__ out, uint64_t ld_out) {
  constexpr int R = R1 + R2;
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
  const uint32_t cnt = g < ngroups ? counts[g] : 0u;
  const int2* __restrict__ lp = lists + (uint64_t)(g < ngroups ? g : 0) * cap;
  unsigned long long acc[R * NV];
#pragma unroll
  for (int i = 0; i < R * NV; ++i) acc[i] = 0ull;
  const uint32_t ring = smem_u32(base) + lane * 16;
  uint32_t kb_cur = 0, slot = 0, phase = 0, stage_addr = ring;
  mbar_sleep_wait_at(smem_u32(&full[0]), 0);
  int2 e = cnt ? __ldg(lp) : make_int2(0, 0);
  for (uint32_t i = 0; i < cnt; ++i) {
    const uint32_t f = i + 1;
    const int2 ne = f < cnt ? __ldg(lp + f) : make_int2(0, 0);
    if (f + 64 < cnt) asm volatile("prefetch.global.L1 [%0];" ::"l"(lp + f + 64));
    const uint32_t k = (uint32_t)e.x;
    const uint32_t kb = k / KB;
    while (kb_cur < kb) {
      __syncwarp();
      if (lane == 0) mbar_arrive_at(smem_u32(&empty[slot]));
      ++kb_cur;
      stage_addr += STAGE_BYTES;
      if (++slot == STAGES) { slot = 0; phase ^= 1; stage_addr = ring; }
      mbar_sleep_wait_at(smem_u32(&full[slot]), phase);
    }
    const uint32_t ra = stage_addr + (k % KB) * 1024;
    unsigned long long b[NV];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 v = lds128(ra + (q >> 1) * KB * 1024 + (q & 1) * 512);
      b[2 * q] = ((unsigned long long)__float_as_uint(v.y) << 32) | __float_as_uint(v.x);
      b[2 * q + 1] = ((unsigned long long)__float_as_uint(v.w) << 32) | __float_as_uint(v.z);
    }
    if constexpr (R2 == 0) {
      jt_apply<R1, T, NV>(acc, b, (uint32_t)e.y);
    } else {
      unsigned long long* a1 = acc;
      unsigned long long* a2 = acc + R1 * NV;
      jt_apply<R1, T, NV>(*reinterpret_cast<unsigned long long(*)[R1 * NV]>(a1), b, (uint32_t)e.y & 0xffu);
      jt_apply<R2, T, NV>(*reinterpret_cast<unsigned long long(*)[R2 * NV]>(a2), b, (uint32_t)e.y >> 8);
    }
    e = ne;
  }
  while (true) {
    __syncwarp();
    if (lane == 0) mbar_arrive_at(smem_u32(&empty[slot]));
    ++kb_cur;
    if (++slot == STAGES) { slot = 0; phase ^= 1; }
    if (kb_cur >= nkb) break;
    mbar_sleep_wait_at(smem_u32(&full[slot]), phase);
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const uint32_t row = g * R + r;
    if (g >= ngroups || row >= nrows) continue;
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

template <int R1, int R2, int T, int CW, int STAGES>
void run(uint32_t n, const float* dB, float* dZ, const std::vector<float>& B, const std::vector<int8_t>& Rp,
         double adds, const char* tag) {
  constexpr int R = R1 + R2;
  // group lists
  const uint32_t ngroups = (n + R - 1) / R;
  std::vector<int2> lists((size_t)ngroups * n);
  std::vector<uint32_t> counts(ngroups);
  size_t entries = 0;
  for (uint32_t g = 0; g < ngroups; ++g) {
    uint32_t c = 0;
    for (uint32_t k = 0; k < n; ++k) {
      uint32_t idx = 0, mul = 1;
      for (int r = 0; r < R; ++r) {
        const uint32_t row = g * R + r;
        const int t = row < n ? Rp[(size_t)row * n + k] : 0;
        if (t < 0 || t > T) { printf("rep out of range\n"); exit(1); }
        if (r == R1) mul = 256;
        idx += (uint32_t)t * mul;
        mul *= (T + 1);
      }
      if (idx) lists[(size_t)g * n + c++] = make_int2((int)k, (int)idx);
    }
    counts[g] = c;
    entries += c;
  }
  int2* dL;
  uint32_t* dC;
  CK(cudaMalloc(&dL, lists.size() * 8));
  CK(cudaMalloc(&dC, counts.size() * 4));
  CK(cudaMemcpy(dL, lists.data(), lists.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dC, counts.data(), counts.size() * 4, cudaMemcpyHostToDevice));
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
  auto kern = k_bgroup<R1, R2, T, CW, STAGES>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((ngroups + CW - 1) / CW, n / TILE_N);
  CK(cudaMemset(dZ, 0xff, (size_t)n * n * 4));
  kern<<<grid, (CW + 1) * 32, smem>>>(tb, dL, n, dC, ngroups, n, n, dZ, n);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> z((size_t)n);
  int bad_rows = 0;
  for (int si = 0; si < 24; ++si) {
    const uint32_t i = (uint32_t)((uint64_t)si * (n - 1) / 23);
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
  for (int it = 0; it < 5; ++it) {
    cudaEventRecord(e0);
    kern<<<grid, (CW + 1) * 32, smem>>>(tb, dL, n, dC, ngroups, n, n, dZ, n);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = std::min(best, ms);
  }
  const double rate = adds / (best * 1e-3);
  printf("%-22s R=%d+%d T=%d CW=%d ST=%d grid=%ux%u entries/group %.0f  %.3f ms  %.4e adds/s  frac %.3f  rows-bad %d/24\n",
         tag, R1, R2, T, CW, STAGES, grid.x, grid.y, (double)entries / ngroups, best, rate, rate / 3.71e13, bad_rows);
  cudaFree(dL);
  cudaFree(dC);
}

int main(int argc, char** argv) {
  const uint32_t n = argc > 1 ? atoi(argv[1]) : 4096;
  const char* dist = argc > 2 ? argv[2] : "unif";
  const int param = argc > 3 ? atoi(argv[3]) : 1;
  std::vector<float> B((size_t)n * n);
  std::vector<int8_t> Rp((size_t)n * n);
  for (auto& v : B) v = (float)((double)(xr() >> 11) / 9007199254740992.0 * 2.0 - 1.0);
  double adds = 0;
  for (auto& r : Rp) {
    const int t = !strcmp(dist, "const") ? param : (int)(xr() % (uint64_t)(2 * param + 1));
    r = (int8_t)t;
    adds += t;
  }
  adds *= n;
  float *dB, *dZ;
  CK(cudaMalloc(&dB, (size_t)n * n * 4));
  CK(cudaMalloc(&dZ, (size_t)n * n * 4));
  CK(cudaMemcpy(dB, B.data(), (size_t)n * n * 4, cudaMemcpyHostToDevice));
  char tag[64];
  snprintf(tag, sizeof tag, "n=%u %s %d", n, dist, param);
  int maxt = 0;
  for (auto r : Rp) maxt = std::max<int>(maxt, r);
  if (maxt <= 2) {
    run<3, 0, 2, 16, 12>(n, dB, dZ, B, Rp, adds, tag);
    run<2, 2, 2, 15, 12>(n, dB, dZ, B, Rp, adds, tag);
    run<2, 2, 2, 16, 12>(n, dB, dZ, B, Rp, adds, tag);
    run<3, 1, 2, 15, 12>(n, dB, dZ, B, Rp, adds, tag);
    run<3, 2, 2, 15, 12>(n, dB, dZ, B, Rp, adds, tag);
    run<3, 3, 2, 12, 12>(n, dB, dZ, B, Rp, adds, tag);
  }
  return 0;
}
