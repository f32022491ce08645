// bform_l1.cu -- repeated-addition kernel, decoupled-warp variant (sm_100a).
//
// Same contract and order preservation as k_bform (bform.cu): one warp owns
// one B-form output row, each lane 16 fp32 / 8 fp64 register accumulators,
// the row's compacted (k, rep) list is applied in increasing k, each entry as
// |rep| warp-uniform FADD2 / DADD steps (kernels.hpp:95-104).
//
// Difference: there is no shared smem ring and no producer warp. Each warp
// fetches its entry's bases with 128-bit read-only loads straight from
// global memory and software-pipelines them one entry ahead (the loads for
// entry e+1 are in flight while entry e's adds run). The warps of an SM read
// the same base rows k at nearly the same time, so those loads hit L1; a warp
// that drifts ahead or behind simply misses to L2 instead of stalling the
// others. ncu on the ring variant showed consumer warps spinning on stage
// barriers: per-row work is a random walk in k and the ring's hard coupling
// (the producer refills a stage only after all 16 warps released it) turned
// that drift into stalls.
#include "common.cuh"
#include "kernels.h"

namespace afmm_dev {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int WARPS = 8;  // rows per CTA
constexpr int G = 4;      // 128-bit vectors per lane per base row (2 KB per warp)

template <class T>
struct L1Cfg {
  static constexpr int V = 16 / sizeof(T);       // elements per 128-bit vector
  static constexpr int TILE_N = G * 32 * V;      // 512 fp32 / 256 fp64 columns
};

__device__ __forceinline__ float4 ldg128(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ double2 ldg128(const double* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}

struct Vec32 {
  float2 v[2 * G];
};
struct Vec64 {
  double v[2 * G];
};

template <class T>
struct Lane;

template <>
struct Lane<float> {
  using Bases = Vec32;
  float2 a[2 * G];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int c = 0; c < 2 * G; ++c) a[c] = make_float2(0.f, 0.f);
  }
  // row points at base row k, column (tile start + 4*lane); `lim` = number of
  // readable columns from the tile start for this lane's groups.
  __device__ __forceinline__ static void load(Bases& b, const float* row, int32_t avail) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
      if (g * 128 + 3 < avail) x = ldg128(row + g * 128);
      b.v[2 * g] = make_float2(x.x, x.y);
      b.v[2 * g + 1] = make_float2(x.z, x.w);
    }
  }
  __device__ __forceinline__ void run(Bases b, int rep) {
    uint32_t t = (uint32_t)rep;
    if (rep < 0) {
#pragma unroll
      for (int c = 0; c < 2 * G; ++c)
        b.v[c] = make_float2(__int_as_float(__float_as_int(b.v[c].x) ^ 0x80000000),
                             __int_as_float(__float_as_int(b.v[c].y) ^ 0x80000000));
      t = 0u - t;
    }
#pragma unroll 1
    while (t >= 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int c = 0; c < 2 * G; ++c) a[c] = __fadd2_rn(a[c], b.v[c]);
      t -= 4;
    }
#pragma unroll 1
    while (t != 0) {
#pragma unroll
      for (int c = 0; c < 2 * G; ++c) a[c] = __fadd2_rn(a[c], b.v[c]);
      t -= 1;
    }
  }
  __device__ __forceinline__ void store(float* out_row, int32_t oc0, int32_t ncols, uint32_t lane,
                                        bool vec_ok) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int32_t c = oc0 + g * 128 + 4 * (int32_t)lane;
      const float v[4] = {a[2 * g].x, a[2 * g].y, a[2 * g + 1].x, a[2 * g + 1].y};
      if (vec_ok && c + 3 < ncols) {
        *reinterpret_cast<float4*>(out_row + c) = make_float4(v[0], v[1], v[2], v[3]);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (c + e < ncols) out_row[c + e] = v[e];
      }
    }
  }
};

template <>
struct Lane<double> {
  using Bases = Vec64;
  double a[2 * G];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int c = 0; c < 2 * G; ++c) a[c] = 0.0;
  }
  __device__ __forceinline__ static void load(Bases& b, const double* row, int32_t avail) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      double2 x = make_double2(0.0, 0.0);
      if (g * 64 + 1 < avail) x = ldg128(row + g * 64);
      b.v[2 * g] = x.x;
      b.v[2 * g + 1] = x.y;
    }
  }
  __device__ __forceinline__ void run(Bases b, int rep) {
    uint32_t t = (uint32_t)rep;
    if (rep < 0) {
#pragma unroll
      for (int c = 0; c < 2 * G; ++c)
        b.v[c] = __longlong_as_double(__double_as_longlong(b.v[c]) ^ 0x8000000000000000ll);
      t = 0u - t;
    }
#pragma unroll 1
    while (t >= 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int c = 0; c < 2 * G; ++c) a[c] = __dadd_rn(a[c], b.v[c]);
      t -= 4;
    }
#pragma unroll 1
    while (t != 0) {
#pragma unroll
      for (int c = 0; c < 2 * G; ++c) a[c] = __dadd_rn(a[c], b.v[c]);
      t -= 1;
    }
  }
  __device__ __forceinline__ void store(double* out_row, int32_t oc0, int32_t ncols,
                                        uint32_t lane, bool vec_ok) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int32_t c = oc0 + g * 64 + 2 * (int32_t)lane;
      if (vec_ok && c + 1 < ncols) {
        *reinterpret_cast<double2*>(out_row + c) = make_double2(a[2 * g], a[2 * g + 1]);
      } else {
        if (c < ncols) out_row[c] = a[2 * g];
        if (c + 1 < ncols) out_row[c + 1] = a[2 * g + 1];
      }
    }
  }
};

// base: B' with leading dimension ldb (elements), readable for columns < ldb.
// Output row b, column (col0 + c) -> out[b * ld_out + c], c < ncols.
template <class T>
__global__ void __launch_bounds__(WARPS * 32, 4)
    k_bform_l1(const T* __restrict__ base, uint64_t ldb, const int2* __restrict__ lists,
               uint64_t cap, const uint32_t* __restrict__ counts, uint32_t nrows, int32_t col0,
               int32_t ncols, T* __restrict__ out, uint64_t ld_out, int vec_ok,
               const DevStatus* __restrict__ st) {
  using Cfg = L1Cfg<T>;
  if (status_failed(st)) return;  // validation failed: compute nothing (kernels.hpp:115,144)
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t b = blockIdx.x * WARPS + warp;
  if (b >= nrows) return;
  const int32_t tile_c = blockIdx.y * Cfg::TILE_N;
  const uint32_t cnt = counts[b];
  const int2* lst = lists + (uint64_t)b * cap;
  // readable columns for this lane, counted from its first element
  const int32_t avail = (int32_t)ldb - (col0 + tile_c) - (int32_t)lane * Cfg::V;
  const T* col_base = base + col0 + tile_c + lane * Cfg::V;

  Lane<T> acc;
  acc.zero();
  if (cnt > 0) {
    int2 A = lane < cnt ? lst[lane] : make_int2(0, 0);            // entries [f & ~31, +32)
    int2 B = 32 + lane < cnt ? lst[32 + lane] : make_int2(0, 0);  // the chunk after A
    typename Lane<T>::Bases cur_b, nxt_b;
    int k = __shfl_sync(FULL, A.x, 0);
    int rep = __shfl_sync(FULL, A.y, 0);
    Lane<T>::load(cur_b, col_base + (uint64_t)k * ldb, avail);
    for (uint32_t e = 0; e < cnt; ++e) {
      const uint32_t f = e + 1;
      if ((f & 31u) == 0) {
        A = B;
        const uint32_t pn = f + 32 + lane;
        B = pn < cnt ? lst[pn] : make_int2(0, 0);
      }
      int rep_n = 0;
      if (f < cnt) {
        const int kn = __shfl_sync(FULL, A.x, f & 31u);
        rep_n = __shfl_sync(FULL, A.y, f & 31u);
        Lane<T>::load(nxt_b, col_base + (uint64_t)kn * ldb, avail);  // in flight during run()
      }
      acc.run(cur_b, rep);
      cur_b = nxt_b;
      rep = rep_n;
    }
  }
  acc.store(out + (uint64_t)b * ld_out, tile_c, ncols, lane, vec_ok != 0);
}

}  // namespace

template <class T>
cudaError_t launch_bform_l1(const T* base, uint64_t ldb, const int2* lists, uint64_t cap,
                            const uint32_t* counts, uint32_t nrows, int32_t col0, int32_t ncols,
                            T* out, uint64_t ld_out, const DevStatus* st, cudaStream_t s) {
  const bool vec_ok = (ld_out * sizeof(T)) % 16 == 0 &&
                      (reinterpret_cast<uintptr_t>(out) % 16) == 0;
  dim3 grid((nrows + WARPS - 1) / WARPS, (ncols + L1Cfg<T>::TILE_N - 1) / L1Cfg<T>::TILE_N);
  k_bform_l1<T><<<grid, WARPS * 32, 0, s>>>(base, ldb, lists, cap, counts, nrows, col0, ncols,
                                            out, ld_out, vec_ok ? 1 : 0, st);
  note_launch();
  return cudaGetLastError();
}

template cudaError_t launch_bform_l1<float>(const float*, uint64_t, const int2*, uint64_t,
                                            const uint32_t*, uint32_t, int32_t, int32_t, float*,
                                            uint64_t, const DevStatus*, cudaStream_t);
template cudaError_t launch_bform_l1<double>(const double*, uint64_t, const int2*, uint64_t,
                                             const uint32_t*, uint32_t, int32_t, int32_t, double*,
                                             uint64_t, const DevStatus*, cudaStream_t);

}  // namespace afmm_dev
