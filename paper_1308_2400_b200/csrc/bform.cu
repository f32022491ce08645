// bform.cu -- the repeated-addition kernel (sm_100a, CUDA cores only).
//
// Computes Z' = R' (x) B' in the reference's order-preserving form: for every
// output element, the terms arrive in increasing k and each is |rep|
// sequential `acc += step` (kernels.hpp:95-104, :148-163). "B-form" means the
// rep is uniform along an output row, which is Case B verbatim
// (kernels.hpp:142-165: rep = X[i,k], bases Y[k,:]); Case A is run through the
// same kernel on transposed operands (afmm_case_a(X,Y) = afmm_case_b(Y^T,X^T)^T,
// same per-element add sequence).
//
// Structure (one CTA = CW consumer warps + 1 TMA producer warp):
//   * CTA tile = CW output rows x TILE_N output columns; each consumer warp
//     owns one output row, each lane C columns held in registers for the
//     whole k sweep (register-resident Z tile).
//   * The producer streams KB x TILE_N tiles of the base matrix B' through a
//     STAGES-deep smem ring with cp.async.bulk.tensor (TMA) + mbarriers;
//     the tile is shared by all CW rows of the CTA (CW-fold reuse from smem).
//   * Each consumer walks its row's compacted (k, rep) list (built by the
//     prepass, zero reps already skipped), waits for the stage holding row k,
//     loads its C bases with two conflict-free 128-bit LDS and runs the
//     warp-uniform rep loop: |rep| x (C/2) FADD2 (fp32) or |rep| x C DADD
//     (fp64). Since the rep is uniform across the warp there is no
//     divergence; zero bases are added as +0/-0, which is bit-neutral
//     (the accumulator is never -0) and never counted.
//   * Warps release a stage by arriving on its empty barrier; they may drift
//     up to STAGES blocks apart, which absorbs per-row work imbalance.
#include "common.cuh"
#include "kernels.h"

namespace afmm_dev {

namespace {

constexpr unsigned FULL = 0xffffffffu;

template <class T>
struct BformCfg;

template <>
struct BformCfg<float> {
  // 8 columns per lane (4 x float2)
  static constexpr int TILE_N = 256;   // columns per CTA
};

template <>
struct BformCfg<double> {
  // 4 columns per lane (2 x double2)
  static constexpr int TILE_N = 128;
};

constexpr int KB = 16;       // k rows per stage
constexpr int STAGES = 6;    // smem ring depth
constexpr int CW = 16;       // consumer warps (output rows) per CTA

template <class T>
__host__ __device__ constexpr size_t stage_bytes() {
  return (size_t)KB * BformCfg<T>::TILE_N * sizeof(T);
}

template <class T>
__host__ __device__ constexpr size_t bform_smem_bytes() {
  return 1024 /*alignment slack*/ + STAGES * stage_bytes<T>() + 2 * STAGES * sizeof(uint64_t);
}

// ---- per-element-type inner loops -----------------------------------------

struct AccF32 {
  float2 a[4];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int c = 0; c < 4; ++c) a[c] = make_float2(0.f, 0.f);
  }
  // Lane owns columns {4l..4l+3} and {128+4l..128+4l+3} of the tile, so each
  // 128-bit LDS across the warp reads 512 contiguous bytes (no bank conflict).
  __device__ __forceinline__ void run(const float* row, uint32_t lane, int rep) {
    const float4 v0 = *reinterpret_cast<const float4*>(row + 4 * lane);
    const float4 v1 = *reinterpret_cast<const float4*>(row + 128 + 4 * lane);
    float2 b[4] = {make_float2(v0.x, v0.y), make_float2(v0.z, v0.w), make_float2(v1.x, v1.y),
                   make_float2(v1.z, v1.w)};
    uint32_t t = (uint32_t)rep;
    if (rep < 0) {
      // step = -base (kernels.hpp:97): exact negation
#pragma unroll
      for (int c = 0; c < 4; ++c) b[c] = make_float2(-b[c].x, -b[c].y);
      t = (uint32_t)(-rep);
    }
    while (t >= 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int c = 0; c < 4; ++c) a[c] = __fadd2_rn(a[c], b[c]);
      t -= 4;
    }
    if (t & 2) {
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int c = 0; c < 4; ++c) a[c] = __fadd2_rn(a[c], b[c]);
    }
    if (t & 1) {
#pragma unroll
      for (int c = 0; c < 4; ++c) a[c] = __fadd2_rn(a[c], b[c]);
    }
  }
  __device__ __forceinline__ void store(float* out_row, int32_t oc0, int32_t ncols, uint32_t lane,
                                        bool vec_ok) {
    const int32_t c0 = oc0 + 4 * (int32_t)lane;
    const int32_t c1 = oc0 + 128 + 4 * (int32_t)lane;
    const float v[8] = {a[0].x, a[0].y, a[1].x, a[1].y, a[2].x, a[2].y, a[3].x, a[3].y};
    if (vec_ok && c0 + 3 < ncols) {
      *reinterpret_cast<float4*>(out_row + c0) = make_float4(v[0], v[1], v[2], v[3]);
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (c0 + e < ncols) out_row[c0 + e] = v[e];
    }
    if (vec_ok && c1 + 3 < ncols) {
      *reinterpret_cast<float4*>(out_row + c1) = make_float4(v[4], v[5], v[6], v[7]);
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (c1 + e < ncols) out_row[c1 + e] = v[4 + e];
    }
  }
};

struct AccF64 {
  double a[4];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int c = 0; c < 4; ++c) a[c] = 0.0;
  }
  // Lane owns columns {2l, 2l+1} and {64+2l, 64+2l+1}.
  __device__ __forceinline__ void run(const double* row, uint32_t lane, int rep) {
    const double2 v0 = *reinterpret_cast<const double2*>(row + 2 * lane);
    const double2 v1 = *reinterpret_cast<const double2*>(row + 64 + 2 * lane);
    double b[4] = {v0.x, v0.y, v1.x, v1.y};
    uint32_t t = (uint32_t)rep;
    if (rep < 0) {
#pragma unroll
      for (int c = 0; c < 4; ++c) b[c] = -b[c];
      t = (uint32_t)(-rep);
    }
    while (t >= 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int c = 0; c < 4; ++c) a[c] = __dadd_rn(a[c], b[c]);
      t -= 4;
    }
    if (t & 2) {
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int c = 0; c < 4; ++c) a[c] = __dadd_rn(a[c], b[c]);
    }
    if (t & 1) {
#pragma unroll
      for (int c = 0; c < 4; ++c) a[c] = __dadd_rn(a[c], b[c]);
    }
  }
  __device__ __forceinline__ void store(double* out_row, int32_t oc0, int32_t ncols,
                                        uint32_t lane, bool vec_ok) {
    const int32_t c0 = oc0 + 2 * (int32_t)lane;
    const int32_t c1 = oc0 + 64 + 2 * (int32_t)lane;
    if (vec_ok && c0 + 1 < ncols) {
      *reinterpret_cast<double2*>(out_row + c0) = make_double2(a[0], a[1]);
    } else {
      if (c0 < ncols) out_row[c0] = a[0];
      if (c0 + 1 < ncols) out_row[c0 + 1] = a[1];
    }
    if (vec_ok && c1 + 1 < ncols) {
      *reinterpret_cast<double2*>(out_row + c1) = make_double2(a[2], a[3]);
    } else {
      if (c1 < ncols) out_row[c1] = a[2];
      if (c1 + 1 < ncols) out_row[c1 + 1] = a[3];
    }
  }
};

template <class T>
struct AccOf;
template <>
struct AccOf<float> {
  using type = AccF32;
};
template <>
struct AccOf<double> {
  using type = AccF64;
};

// lists: row b's entries at lists[b * cap .. b * cap + counts[b]) in increasing k.
// Output row b, column (col0 + c) -> out[b * ld_out + c], c < ncols.
template <class T>
__global__ void __launch_bounds__((CW + 1) * 32, 2)
    k_bform(const __grid_constant__ CUtensorMap tmap, const int2* __restrict__ lists,
            uint64_t cap, const uint32_t* __restrict__ counts, uint32_t nrows, int32_t col0,
            int32_t ncols, uint32_t nkb, T* __restrict__ out, uint64_t ld_out, int vec_ok,
            const DevStatus* __restrict__ st) {
  using Cfg = BformCfg<T>;
  extern __shared__ unsigned char smem_raw[];
  // 1024-byte aligned ring; pointer arithmetic on the smem pointer itself keeps
  // the shared address space visible to the compiler (LDS, not generic LD).
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  T* tiles = reinterpret_cast<T*>(base);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + STAGES * stage_bytes<T>());
  uint64_t* empty = full + STAGES;

  if (status_failed(st)) return;  // validation failed: compute nothing (kernels.hpp:115,144)

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t tile_c = blockIdx.y * Cfg::TILE_N;  // relative to col0

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == CW) {
    // ---- TMA producer ----
    if (lane == 0) {
      prefetch_tensormap(&tmap);
      uint32_t slot = 0, phase = 0;
      for (uint32_t kb = 0; kb < nkb; ++kb) {
        if (kb >= STAGES) mbar_wait(&empty[slot], phase ^ 1);
        mbar_arrive_expect_tx(&full[slot], (uint32_t)stage_bytes<T>());
        tma_load_2d(tiles + (size_t)slot * KB * Cfg::TILE_N, &tmap, &full[slot], col0 + tile_c,
                    (int32_t)(kb * KB));
        if (++slot == STAGES) {
          slot = 0;
          phase ^= 1;
        }
      }
    }
    return;
  }

  // ---- consumers: one output row per warp ----
  const uint32_t b = blockIdx.x * CW + warp;
  const uint32_t cnt = b < nrows ? counts[b] : 0u;
  const int2* lst = lists + (uint64_t)(b < nrows ? b : 0) * cap;

  typename AccOf<T>::type acc;
  acc.zero();

  // (kb_cur, slot, phase): the k block currently held, its ring slot and the
  // parity of that slot's current fill.
  uint32_t kb_cur = 0, slot = 0, phase = 0;
  auto advance = [&]() {
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
    ++kb_cur;
    if (++slot == STAGES) {
      slot = 0;
      phase ^= 1;
    }
  };
  mbar_wait(&full[0], 0);
  int2 cur = lane < cnt ? lst[lane] : make_int2(0, 0);
  for (uint32_t p = 0; p < cnt; p += 32) {
    const uint32_t pn = p + 32 + lane;
    const int2 nxt = pn < cnt ? lst[pn] : make_int2(0, 0);  // prefetch next chunk
    const uint32_t m = cnt - p < 32u ? cnt - p : 32u;
    for (uint32_t q = 0; q < m; ++q) {
      const int k = __shfl_sync(FULL, cur.x, q);
      const int rep = __shfl_sync(FULL, cur.y, q);
      const uint32_t kb = (uint32_t)k / KB;
      while (kb_cur < kb) {
        advance();
        mbar_wait(&full[slot], phase);
      }
      const T* row = tiles + ((size_t)slot * KB + ((uint32_t)k % KB)) * Cfg::TILE_N;
      acc.run(row, lane, rep);
    }
    cur = nxt;
  }
  // release the remaining stages in order
  while (true) {
    advance();
    if (kb_cur >= nkb) break;
    mbar_wait(&full[slot], phase);
  }

  if (b < nrows) acc.store(out + (uint64_t)b * ld_out, tile_c, ncols, lane, vec_ok != 0);
}

}  // namespace

template <class T>
int bform_tile_n() {
  return BformCfg<T>::TILE_N;
}

template <class T>
int bform_kb() {
  return KB;
}

template <class T>
cudaError_t launch_bform(const CUtensorMap* tmap, const int2* lists, uint64_t cap,
                         const uint32_t* counts, uint32_t nrows, int32_t col0, int32_t ncols,
                         uint32_t nk, T* out, uint64_t ld_out, const DevStatus* st,
                         cudaStream_t s) {
  const size_t smem = bform_smem_bytes<T>();
  // set on every call: the attribute is per device and costs ~1 us
  cudaError_t e =
      cudaFuncSetAttribute(k_bform<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const uint32_t nkb = (nk + KB - 1) / KB;
  const bool vec_ok = (ld_out * sizeof(T)) % 16 == 0 &&
                      (reinterpret_cast<uintptr_t>(out) % 16) == 0;
  dim3 grid((nrows + CW - 1) / CW, (ncols + BformCfg<T>::TILE_N - 1) / BformCfg<T>::TILE_N);
  k_bform<T><<<grid, (CW + 1) * 32, smem, s>>>(*tmap, lists, cap, counts, nrows, col0, ncols, nkb,
                                               out, ld_out, vec_ok ? 1 : 0, st);
  note_launch();
  return cudaGetLastError();
}

template int bform_tile_n<float>();
template int bform_tile_n<double>();
template int bform_kb<float>();
template int bform_kb<double>();
template cudaError_t launch_bform<float>(const CUtensorMap*, const int2*, uint64_t,
                                         const uint32_t*, uint32_t, int32_t, int32_t, uint32_t,
                                         float*, uint64_t, const DevStatus*, cudaStream_t);
template cudaError_t launch_bform<double>(const CUtensorMap*, const int2*, uint64_t,
                                          const uint32_t*, uint32_t, int32_t, int32_t, uint32_t,
                                          double*, uint64_t, const DevStatus*, cudaStream_t);

}  // namespace afmm_dev
