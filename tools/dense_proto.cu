// Prototype (dev tool, not the product): a repeated-addition kernel with
// register-resident bases and TMEM-resident accumulators over a DENSE int8
// rep tile, to lift the shared-memory bound of k_bform at small reps.
//
// k_bform reads a warp's 1024 bases (4 KB) from smem for every list entry:
// at rep 1 that is 4 B per add against 1 B per add of smem bandwidth per FP
// add issue (128 B/clk vs 128 adds/clk per SM). Here a warp loads the bases of
// KSUB k rows x 512 columns into registers ONCE and applies them to RW rows
// whose accumulators live in tensor memory (tcgen05.ld/st, a separate data
// path): per (row, KSUB block) one 16-column TMEM load + store instead of KSUB
// smem base loads, and the bases are reused RW times.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
//        -fmad=false -ftz=false -Xcompiler -ffp-contract=off -o build/dense_proto tools/dense_proto.cu -lcuda
//   build/dense_proto <n> <dist> <param> [ladder] [rw]
//     dist: const r | unif mu (uniform{0..2mu}) | geom mean
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

constexpr int NV = 8;        // float2 per lane (16 fp32 columns)
constexpr int TILE_N = 512;  // columns per CTA
constexpr int KSUB = 4;      // k rows per register block

__device__ __forceinline__ void tm_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tm_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
      "%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]));
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

template <bool NEG>
__device__ __forceinline__ void step(float2 (&a)[NV], const float2 (&b)[NV]) {
#pragma unroll
  for (int c = 0; c < NV; ++c) a[c] = __fadd2_rn(a[c], NEG ? make_float2(-b[c].x, -b[c].y) : b[c]);
}

// LADDER 2: one brx.idx per k: jump into a fall-through ladder of 8 steps
// (t <= 8 after the trips of 8), so a rep costs one indirect branch.
#define F2(i) "l"(*reinterpret_cast<const unsigned long long*>(&b[i]))
template <bool NEG>
__device__ __forceinline__ void ladder8(float2 (&a)[NV], const float2 (&b)[NV], uint32_t t) {
  unsigned long long* A = reinterpret_cast<unsigned long long*>(a);
  const uint32_t idx = 8u - t;  // t in [0, 8]
#define STEP8 OP " %0, %0, %8;\n\t" OP " %1, %1, %9;\n\t" OP " %2, %2, %10;\n\t" OP " %3, %3, %11;\n\t" \
              OP " %4, %4, %12;\n\t" OP " %5, %5, %13;\n\t" OP " %6, %6, %14;\n\t" OP " %7, %7, %15;\n\t"
#define LADDER_ASM                                                                                   \
  asm volatile(                                                                                      \
      "{\n\t"                                                                                        \
      "Lt%=: .branchtargets L8%=, L7%=, L6%=, L5%=, L4%=, L3%=, L2%=, L1%=, L0%=;\n\t"               \
      "brx.idx %16, Lt%=;\n\t"                                                                       \
      "L8%=:\n\t" STEP8 "L7%=:\n\t" STEP8 "L6%=:\n\t" STEP8 "L5%=:\n\t" STEP8                         \
      "L4%=:\n\t" STEP8 "L3%=:\n\t" STEP8 "L2%=:\n\t" STEP8 "L1%=:\n\t" STEP8 "L0%=:\n\t"             \
      "}"                                                                                            \
      : "+l"(A[0]), "+l"(A[1]), "+l"(A[2]), "+l"(A[3]), "+l"(A[4]), "+l"(A[5]), "+l"(A[6]), "+l"(A[7]) \
      : F2(0), F2(1), F2(2), F2(3), F2(4), F2(5), F2(6), F2(7), "r"(idx));
  if (NEG) {
#define OP "sub.rn.f32x2"
    LADDER_ASM;
#undef OP
  } else {
#define OP "add.rn.f32x2"
    LADDER_ASM;
#undef OP
  }
}

// t sequential adds: LADDER 0 = trips of 8 + binary digits 4/2/1;
// LADDER 1 = trips of 8 + a fall-through switch (jump table).
template <bool NEG, int LADDER>
__device__ __forceinline__ void run_t(float2 (&a)[NV], const float2 (&b)[NV], uint32_t t) {
  if (LADDER == 0) {
#pragma unroll 1
    while (t >= 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) step<NEG>(a, b);
      t -= 8;
    }
    if (t & 4) { step<NEG>(a, b); step<NEG>(a, b); step<NEG>(a, b); step<NEG>(a, b); }
    if (t & 2) { step<NEG>(a, b); step<NEG>(a, b); }
    if (t & 1) step<NEG>(a, b);
  } else if (LADDER == 2) {
#pragma unroll 1
    while (t > 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) step<NEG>(a, b);
      t -= 8;
    }
    ladder8<NEG>(a, b, t);
  } else {
#pragma unroll 1
    while (t > 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) step<NEG>(a, b);
      t -= 8;
    }
    switch (t) {
      case 8: step<NEG>(a, b); [[fallthrough]];
      case 7: step<NEG>(a, b); [[fallthrough]];
      case 6: step<NEG>(a, b); [[fallthrough]];
      case 5: step<NEG>(a, b); [[fallthrough]];
      case 4: step<NEG>(a, b); [[fallthrough]];
      case 3: step<NEG>(a, b); [[fallthrough]];
      case 2: step<NEG>(a, b); [[fallthrough]];
      case 1: step<NEG>(a, b); [[fallthrough]];
      default: break;
    }
  }
}

template <int KS, int STAGES, int LADDER, int CW>
__global__ void __launch_bounds__((CW + 1) * 32, 1)
    k_dense(const __grid_constant__ CUtensorMap tb, const __grid_constant__ CUtensorMap tr,
            uint32_t nrows, uint32_t nk, uint32_t rw, float* __restrict__ out, uint64_t ld_out) {
  constexpr int BASE_BYTES = KS * TILE_N * 4;  // [2 boxes][KS][1 KB]
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t cta_rows = CW * rw;
  const uint32_t rep_bytes = KS * cta_rows;
  const uint32_t stage_bytes = BASE_BYTES + ((rep_bytes + 127) & ~127u);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + STAGES * stage_bytes);
  uint64_t* empty = full + STAGES;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(empty + STAGES);
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  const uint32_t row0 = blockIdx.x * cta_rows;
  const int32_t tile_c = blockIdx.y * TILE_N;
  const uint32_t nst = (nk + KS - 1) / KS;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = *tslot;

  if (warp == CW) {
    if (lane == 0) {
      prefetch_tensormap(&tb);
      prefetch_tensormap(&tr);
      for (uint32_t i = 0; i < nst; ++i) {
        const uint32_t slot = i % STAGES;
        if (i >= STAGES) mbar_sleep_wait_at(smem_u32(&empty[slot]), ((i / STAGES) - 1) & 1);
        mbar_arrive_expect_tx(&full[slot], (uint32_t)BASE_BYTES + rep_bytes);
        unsigned char* st = base + slot * stage_bytes;
        tma_load_2d(st, &tb, &full[slot], tile_c, (int32_t)(i * KS));
        tma_load_2d(st + KS * 1024, &tb, &full[slot], tile_c + 256, (int32_t)(i * KS));
        tma_load_2d(st + BASE_BYTES, &tr, &full[slot], (int32_t)(i * KS), (int32_t)row0);
      }
    }
  } else {
    const uint32_t taddr = pin(tbase + (((warp & 3u) * 32u) << 16) + (warp >> 2) * 128u);
    {
      uint32_t z[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) z[i] = 0u;
      for (uint32_t r = 0; r < rw; ++r) tm_st16(taddr + r * 16, z);
    }
    const uint32_t ring = smem_u32(base);
    uint32_t slot = 0, phase = 0;
    for (uint32_t s = 0; s < nst; ++s) {
      mbar_sleep_wait_at(smem_u32(&full[slot]), phase);
      const uint32_t sb = ring + slot * stage_bytes;
      const uint32_t rb = sb + BASE_BYTES + warp * rw * KS;
#pragma unroll 1
      for (int sub = 0; sub < KS / KSUB; ++sub) {
        float2 b[KSUB][NV];
#pragma unroll
        for (int kk = 0; kk < KSUB; ++kk)
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const float4 v = lds128(sb + (g >> 1) * KS * 1024 + (sub * KSUB + kk) * 1024 + (g & 1) * 512 + lane * 16);
            b[kk][2 * g] = make_float2(v.x, v.y);
            b[kk][2 * g + 1] = make_float2(v.z, v.w);
          }
        tm_wait_st();
#pragma unroll 1
        for (uint32_t r = 0; r < rw; ++r) {
          const uint32_t w4 = lds32(rb + r * KS + sub * KSUB);
          if (w4 == 0u) continue;
          uint32_t ar[16];
          tm_ld16(taddr + r * 16, ar);
          tm_wait_ld();
          float2 a[NV];
#pragma unroll
          for (int c = 0; c < NV; ++c) a[c] = make_float2(__uint_as_float(ar[2 * c]), __uint_as_float(ar[2 * c + 1]));
#pragma unroll
          for (int kk = 0; kk < KSUB; ++kk) {
            const int t = (int)(int8_t)(w4 >> (8 * kk));
            if (t > 0) run_t<false, LADDER>(a, b[kk], (uint32_t)t);
            else if (t < 0) run_t<true, LADDER>(a, b[kk], (uint32_t)(-t));
          }
#pragma unroll
          for (int c = 0; c < NV; ++c) { ar[2 * c] = __float_as_uint(a[c].x); ar[2 * c + 1] = __float_as_uint(a[c].y); }
          tm_st16(taddr + r * 16, ar);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_at(smem_u32(&empty[slot]));
      if (++slot == STAGES) { slot = 0; phase ^= 1; }
    }
    tm_wait_st();
    for (uint32_t r = 0; r < rw; ++r) {
      const uint32_t row = row0 + warp * rw + r;
      uint32_t ar[16];
      tm_ld16(taddr + r * 16, ar);
      tm_wait_ld();
      if (row < nrows) {
        float* o = out + (uint64_t)row * ld_out + tile_c;
#pragma unroll
        for (int g = 0; g < 4; ++g)
          *reinterpret_cast<float4*>(o + g * 128 + lane * 4) =
              make_float4(__uint_as_float(ar[4 * g]), __uint_as_float(ar[4 * g + 1]),
                          __uint_as_float(ar[4 * g + 2]), __uint_as_float(ar[4 * g + 3]));
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
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

template <int KS, int STAGES, int LADDER, int CW>
void run(uint32_t n, uint32_t rw, const float* dB, const int8_t* dR, float* dZ, const std::vector<float>& B,
         const std::vector<int8_t>& R, double adds, const char* tag) {
  auto fn = enc();
  CUtensorMap tb, tr;
  {
    cuuint64_t gdim[2] = {n, n};
    cuuint64_t gstr[1] = {(cuuint64_t)n * 4};
    cuuint32_t box[2] = {256, KS};
    cuuint32_t es[2] = {1, 1};
    if (fn(&tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)dB, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      printf("tmap B failed\n"); exit(1);
    }
  }
  {
    cuuint64_t gdim[2] = {n, n};
    cuuint64_t gstr[1] = {(cuuint64_t)n};
    cuuint32_t box[2] = {KS, CW * rw};
    cuuint32_t es[2] = {1, 1};
    if (fn(&tr, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)dR, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      printf("tmap R failed\n"); exit(1);
    }
  }
  const uint32_t rep_bytes = KS * CW * rw;
  const size_t stage = (size_t)KS * TILE_N * 4 + ((rep_bytes + 127) & ~127u);
  const size_t smem = 1024 + STAGES * stage + 2 * STAGES * 8 + 16;
  auto kern = k_dense<KS, STAGES, LADDER, CW>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((n + CW * rw - 1) / (CW * rw), n / TILE_N);
  CK(cudaMemset(dZ, 0xff, (size_t)n * n * 4));
  kern<<<grid, (CW + 1) * 32, smem>>>(tb, tr, n, n, rw, dZ, n);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  // check sampled rows bit for bit
  std::vector<float> z((size_t)n);
  int bad_rows = 0;
  for (int si = 0; si < 24; ++si) {
    const uint32_t i = (uint32_t)((uint64_t)si * (n - 1) / 23);
    CK(cudaMemcpy(z.data(), dZ + (size_t)i * n, n * 4, cudaMemcpyDeviceToHost));
    std::vector<float> acc(n, 0.f);
    for (uint32_t k = 0; k < n; ++k) {
      const int t = R[(size_t)i * n + k];
      if (!t) continue;
      const float* brow = &B[(size_t)k * n];
      const int m = t < 0 ? -t : t;
      for (uint32_t j = 0; j < n; ++j) {
        const float s = t < 0 ? -brow[j] : brow[j];
        float a = acc[j];
        for (int u = 0; u < m; ++u) a = a + s;
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
    kern<<<grid, (CW + 1) * 32, smem>>>(tb, tr, n, n, rw, dZ, n);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = std::min(best, ms);
  }
  const double rate = adds / (best * 1e-3);
  printf("%-28s CW=%d KS=%d ST=%d L=%d rw=%u grid=%ux%u  %.3f ms  %.4e adds/s  frac %.3f  rows-bad %d/24\n", tag, CW, KS, STAGES,
         LADDER, rw, grid.x, grid.y, best, rate, rate / 3.71e13, bad_rows);
}

int main(int argc, char** argv) {
  const uint32_t n = argc > 1 ? atoi(argv[1]) : 4096;
  const char* dist = argc > 2 ? argv[2] : "unif";
  const double param = argc > 3 ? atof(argv[3]) : 1;
  const int which = argc > 4 ? atoi(argv[4]) : -1;
  std::vector<float> B((size_t)n * n);
  std::vector<int8_t> R((size_t)n * n);
  for (auto& v : B) v = (float)((double)(xr() >> 11) / 9007199254740992.0 * 2.0 - 1.0);
  double adds = 0;
  for (auto& r : R) {
    int t;
    if (!strcmp(dist, "const")) t = (int)param;
    else if (!strcmp(dist, "unif")) t = (int)(xr() % (uint64_t)(2 * param + 1));
    else if (!strcmp(dist, "sunif")) t = (int)(xr() % (uint64_t)(2 * param + 1)) - (int)param;
    else {  // geometric mean param capped at 64
      t = 1;
      const double p = 1.0 / param;
      while (t < 64 && (double)(xr() >> 11) / 9007199254740992.0 >= p) ++t;
    }
    r = (int8_t)t;
    adds += std::abs(t);
  }
  adds *= n;  // every base lane (dense bases)
  float *dB, *dZ;
  int8_t* dR;
  CK(cudaMalloc(&dB, (size_t)n * n * 4));
  CK(cudaMalloc(&dZ, (size_t)n * n * 4));
  CK(cudaMalloc(&dR, (size_t)n * n));
  CK(cudaMemcpy(dB, B.data(), (size_t)n * n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dR, R.data(), (size_t)n * n, cudaMemcpyHostToDevice));
  char tag[64];
  snprintf(tag, sizeof tag, "n=%u %s %g", n, dist, param);
  for (uint32_t rw : {8u, 7u}) {
    if (which < 0 || which == 0) run<16, 4, 1, 16>(n, rw, dB, dR, dZ, B, R, adds, tag);
    if (which < 0 || which == 1) run<16, 4, 0, 15>(n, rw, dB, dR, dZ, B, R, adds, tag);
    if (which < 0 || which == 2) run<16, 4, 1, 15>(n, rw, dB, dR, dZ, B, R, adds, tag);
    if (which < 0 || which == 3) run<16, 4, 0, 12>(n, rw, dB, dR, dZ, B, R, adds, tag);
    if (which < 0 || which == 4) run<16, 4, 2, 16>(n, rw, dB, dR, dZ, B, R, adds, tag);
    if (which < 0 || which == 5) run<16, 4, 2, 15>(n, rw, dB, dR, dZ, B, R, adds, tag);
  }
  return 0;
}
