// prepass.cu -- O(n^2) device prepass of the AFMM product (sm_100a).
//
// Replaces the inline zero tests and the up-front validation of the
// reference kernels (/root/reference/proj/include/afmm/kernels.hpp:25-43,
// :121-130, :150-159) with three streaming passes (one warp per matrix row,
// 128-bit loads, one read of each operand):
//
//   k_scan_stats   both operands: finite check (matrix.hpp:31-35), rep
//                  validation of the rep operand (kernels.hpp:25-43; first
//                  offender by atomicMax on the inverted row-major index), and
//                  the per-k vector the work formulas need: nnz(Y[k,:]) (Case B)
//                  or R_k = sum_j |llround Y[k,j]| (Case A)
//   k_rows         per row i of X: exact additions W_i and zero_skips (closed
//                  forms of kernels.hpp:119-134 / :148-163), the slab's OpCounts,
//                  and (Case B) the warp-scan stream compaction of the row's
//                  nonzero reps into an ordered (k, rep) list: the zero-skip of
//                  kernels.hpp:151-153 done once instead of per (i,k,j)
//   k_transpose_compact  (Case A) the same compaction for the columns of Y,
//                  through 32x33 smem tiles (the rep list of B-form row j is
//                  column j of Y)
//
// plus k_transpose (Case A operand/result transposes) and k_reduce_slices
// (fast-mode split-k combine). All are HBM-bound; none does FP arithmetic on
// the product.
#include <cuda_fp16.h>

#include "common.cuh"
#include "kernels.h"

namespace afmm_dev {

namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(FULL, v, o);
    v = w > v ? w : v;
  }
  return v;
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t v, uint32_t lane, uint32_t* total) {
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  *total = __shfl_sync(FULL, x, 31);
  return x - v;
}

// Four consecutive row elements j..j+3 (zeros beyond n). `vec` = row base and
// leading dimension allow 128-bit loads.
template <class T>
__device__ __forceinline__ void load4(const T* row, uint32_t j, uint32_t n, bool vec, T v[4]) {
  if (vec && j + 3 < n) {
    if constexpr (sizeof(T) == 4) {
      const float4 q = __ldg(reinterpret_cast<const float4*>(row + j));
      v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else {
      const double2 a = __ldg(reinterpret_cast<const double2*>(row + j));
      const double2 b = __ldg(reinterpret_cast<const double2*>(row + j + 2));
      v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    }
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] = j + e < n ? row[j + e] : T(0);
  }
}

__device__ __forceinline__ long long abs_ll(long long r) { return r < 0 ? -r : r; }

// warp task t < n: lhs row t; t >= n: rhs row t - n.
template <class T>
__global__ void k_scan_stats(const T* __restrict__ lhs, const T* __restrict__ rhs, uint64_t ld,
                             uint32_t n, int which_case, int vec, DevStatus* st,
                             uint32_t* __restrict__ nnz, unsigned long long* __restrict__ rsum) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t t = warp; t < 2ull * n; t += nwarps) {
    const bool is_rhs = t >= n;
    const uint64_t i = is_rhs ? t - n : t;
    const T* row = (is_rhs ? rhs : lhs) + i * ld;
    // Case A validates rhs (kernels.hpp:115), Case B lhs (:144)
    const bool is_rep = is_rhs == (which_case == 0);
    unsigned long long nf = 0, rb = 0, tl = 0;  // inverted keys, 0 = none
    uint32_t cnt = 0;
    unsigned long long s = 0;
    for (uint32_t j0 = 4 * lane; j0 < n; j0 += 128) {
      T v[4];
      load4(row, j0, n, vec != 0, v);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t j = j0 + e;
        if (j >= n) break;
        const double d = (double)v[e];
        const unsigned long long lin = i * (uint64_t)n + j;
        if (!isfinite(d) && nf == 0) nf = ~lin;  // ascending j: the first one is the minimum
        if (is_rep) {
          const int kind = rep_kind(d);
          if (kind && rb == 0) rb = ~((lin << 2) | (unsigned long long)kind);
          else if (!kind && tl == 0 && fabs(d) >= 2147483647.5) tl = ~lin;
        }
        if (is_rhs) {
          cnt += v[e] != T(0) ? 1u : 0u;
          if (v[e] != T(0)) s += (unsigned long long)abs_ll(llround(d));
        }
      }
    }
    if (__any_sync(FULL, (nf | rb | tl) != 0)) {
      nf = warp_max_u64(nf);
      rb = warp_max_u64(rb);
      tl = warp_max_u64(tl);
      if (lane == 0) {
        if (nf) atomicMax(is_rhs ? &st->nonfinite_rhs_inv : &st->nonfinite_lhs_inv, nf);
        if (rb) atomicMax(&st->rep_bad_inv, rb);
        if (tl) atomicMax(&st->rep_too_large_inv, tl);
      }
    }
    if (is_rhs) {
      if (which_case == 1) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(FULL, cnt, o);
        if (lane == 0) nnz[i] = cnt;
      } else {
        s = warp_sum_u64(s);
        if (lane == 0) rsum[i] = s;
      }
    }
  }
}

// Per row i of X (all n rows): W_i -> work[i]; rows in [r0, r1) add to the
// slab OpCounts and (Case B, lists != nullptr) get their compacted rep list.
// Case A: W_i = sum_{k: X[i,k] != 0} R_k, zs_i = #{k: X[i,k] == 0}
// Case B: W_i = sum_k |rep_ik| nnz_k,    zs_i = sum_{k: rep_ik != 0} (n - nnz_k)
// A rep is skipped exactly when the reference skips it: value == 0.0 or
// llround == 0 (kernels.hpp:151-153).
template <class T>
__global__ void k_rows(const T* __restrict__ x, uint64_t ld, uint32_t n, int which_case, int vec,
                       const uint32_t* __restrict__ nnz,
                       const unsigned long long* __restrict__ rsum, uint32_t r0, uint32_t r1,
                       int2* __restrict__ lists, uint64_t cap, uint32_t* __restrict__ counts,
                       unsigned long long* __restrict__ work, DevStatus* st,
                       uint32_t* __restrict__ nnz_row) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = warp; i < n; i += nwarps) {
    const T* row = x + i * ld;
    const bool in_slab = i >= r0 && i < r1;
    const bool compact = which_case == 1 && in_slab && lists != nullptr;
    int2* out = compact ? lists + (i - r0) * cap : nullptr;
    unsigned long long w = 0, z = 0;
    uint32_t base = 0;
    for (uint32_t c0 = 0; c0 < n; c0 += 128) {  // warp-uniform trip count (the scan below)
      const uint32_t j0 = c0 + 4 * lane;
      T v[4];
      load4(row, j0, n, vec != 0, v);
      long long rep[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t j = j0 + e;
        rep[e] = 0;
        if (j < n && v[e] != T(0)) rep[e] = llround((double)v[e]);
        if (which_case == 0) {
          if (j < n) {
            if (v[e] == T(0)) ++z;
            else w += rsum[j];
          }
        } else if (rep[e] != 0) {
          const unsigned long long nb = nnz[j];
          w += (unsigned long long)abs_ll(rep[e]) * nb;  // count bookkeeping, not an element product
          z += (unsigned long long)n - nb;
        }
      }
      if (compact) {
        const uint32_t mine = (rep[0] != 0) + (rep[1] != 0) + (rep[2] != 0) + (rep[3] != 0);
        uint32_t total;
        uint32_t pos = base + warp_excl_scan(mine, lane, &total);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (rep[e] != 0) out[pos++] = make_int2((int)(j0 + e), (int)rep[e]);
        base += total;
      }
    }
    w = warp_sum_u64(w);
    z = warp_sum_u64(z);
    if (lane == 0) {
      work[i] = w;
      if (in_slab) {
        if (w) atomicAdd(&st->additions, w);
        if (z) atomicAdd(&st->zero_skips, z);
        if (compact) counts[i - r0] = base;
        // Case A: nonzero bases of the row (its A-form cost)
        if (nnz_row && which_case == 0) nnz_row[i - r0] = n - (uint32_t)z;
      }
    }
  }
}

// Case A rep lists: B-form row j = column j of Y. A block owns 32 columns and
// walks k in 32-row tiles through smem; warp w compacts columns 4w..4w+3.
template <class T>
__global__ void __launch_bounds__(256) k_transpose_compact(const T* __restrict__ y, uint64_t ld,
                                                           uint32_t n, int2* __restrict__ lists,
                                                           uint64_t cap,
                                                           uint32_t* __restrict__ counts) {
  __shared__ T tile[32][33];
  const uint32_t tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const uint32_t j0 = blockIdx.x * 32;
  const unsigned lt = (1u << tx) - 1u;
  uint32_t base[4] = {0, 0, 0, 0};
  // the next 32-row tile is loaded into registers while this one is compacted
  // (the block walks k serially, so unhidden load latency is its whole cost
  // at small n)
  T pre[4];
  auto fetch = [&](uint32_t k0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t k = k0 + ty + 8 * q, j = j0 + tx;
      pre[q] = (k < n && j < n) ? y[(uint64_t)k * ld + j] : T(0);
    }
  };
  fetch(0);
  for (uint32_t k0 = 0; k0 < n; k0 += 32) {
#pragma unroll
    for (int q = 0; q < 4; ++q) tile[ty + 8 * q][tx] = pre[q];
    __syncthreads();
    if (k0 + 32 < n) fetch(k0 + 32);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t jj = ty * 4 + q, j = j0 + jj;
      const T v = tile[tx][jj];  // Y[k0 + tx, j]
      int rep = 0;
      if (v != T(0) && k0 + tx < n) rep = (int)llround((double)v);
      const unsigned m = __ballot_sync(FULL, rep != 0);
      if (rep != 0 && j < n) lists[(uint64_t)j * cap + base[q] + __popc(m & lt)] =
          make_int2((int)(k0 + tx), rep);
      base[q] += __popc(m);
    }
    __syncthreads();
  }
  if (tx == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t j = j0 + ty * 4 + q;
      if (j < n) counts[j] = base[q];
    }
  }
}

// ---- A-form prepass (k_aform, Case A with the base uniform per warp) ----

// A-form rep counts: cnt[k][j] = llround(Y[k,j]) as fp16 (exact for |rep| <=
// 2048, the A-form's eligibility bound; 0 for zero reps, kernels.hpp:128-130),
// and per (k, column tile) the largest |rep| (the warp-uniform trip count of
// the predicated add loop) with bit 15 set when the tile row holds a negative
// rep. One warp per (k, tile).
// fstats (optional): [0] nonzero reps, [1] sum of the per-(k, tile) trip counts,
// [2] reps beyond 2048, [3] sum of |rep| -- the A-form / B-form cost inputs.
template <class T>
__global__ void k_counts_f16(const T* __restrict__ y, uint64_t ld, uint32_t n, uint32_t tile_cols,
                             uint32_t ntiles, __half* __restrict__ cnt, uint64_t ldc,
                             uint16_t* __restrict__ rmax, unsigned long long* __restrict__ fstats) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t task = warp; task < (uint64_t)n * ntiles; task += nwarps) {
    const uint64_t k = task / ntiles;
    const uint32_t t = (uint32_t)(task % ntiles);
    uint32_t mx = 0, neg = 0, nz = 0, big = 0;
    unsigned long long sum = 0;
    for (uint32_t c = t * tile_cols + lane; c < (t + 1) * tile_cols && c < n; c += 32) {
      const T v = y[k * ld + c];
      long long r = v != T(0) ? llround((double)v) : 0;
      nz += r != 0 ? 1u : 0u;
      sum += (unsigned long long)abs_ll(r);
      if (r > 2048 || r < -2048) {
        big += 1;
        r = r > 0 ? 2048 : -2048;
      }
      cnt[k * ldc + c] = __int2half_rn((int)r);
      const uint32_t a = (uint32_t)(r < 0 ? -r : r);
      mx = a > mx ? a : mx;
      neg |= r < 0 ? 1u : 0u;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint32_t m = __shfl_xor_sync(FULL, mx, o);
      mx = m > mx ? m : mx;
      neg |= __shfl_xor_sync(FULL, neg, o);
      nz += __shfl_xor_sync(FULL, nz, o);
      big += __shfl_xor_sync(FULL, big, o);
    }
    sum = warp_sum_u64(sum);
    if (lane == 0) {
      rmax[k * ntiles + t] = (uint16_t)(mx | (neg ? 0x8000u : 0u));
      if (fstats) {
        if (nz) atomicAdd(&fstats[0], (unsigned long long)nz);
        if (mx) atomicAdd(&fstats[1], (unsigned long long)mx);
        if (big) atomicAdd(&fstats[2], (unsigned long long)big);
        if (sum) atomicAdd(&fstats[3], sum);
      }
    }
  }
}

// A-form lists: row i in [r0, r1) of X -> its nonzero bases (k, X[i,k]) in
// increasing k (the zero-base skip of kernels.hpp:121-125 done once).
// rows_idx (optional): task t compacts slab row rows_idx[t] (else t); lists
// and counts are indexed by slab row either way.
template <class T>
__global__ void k_acompact(const T* __restrict__ x, uint64_t ld, uint32_t n, int vec, uint32_t r0,
                           uint32_t ntask, const uint32_t* __restrict__ rows_idx,
                           typename AEntry<T>::type* __restrict__ lists, uint64_t cap,
                           uint32_t* __restrict__ counts) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t t = warp; t < ntask; t += nwarps) {
    const uint64_t q = rows_idx ? rows_idx[t] : t;  // slab row
    const T* row = x + (r0 + q) * ld;
    auto* out = lists + q * cap;
    uint32_t base = 0;
    for (uint32_t c0 = 0; c0 < n; c0 += 128) {
      const uint32_t j0 = c0 + 4 * lane;
      T v[4];
      load4(row, j0, n, vec != 0, v);
      const uint32_t mine = (v[0] != T(0)) + (v[1] != T(0)) + (v[2] != T(0)) + (v[3] != T(0));
      uint32_t total;
      uint32_t pos = base + warp_excl_scan(mine, lane, &total);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (v[e] == T(0)) continue;
        if constexpr (sizeof(T) == 4) {
          out[pos++] = make_int2((int)(j0 + e), __float_as_int((float)v[e]));
        } else {
          const double d = (double)v[e];
          out[pos++] = make_int4((int)(j0 + e), 0, __double2loint(d), __double2hiint(d));
        }
      }
      base += total;
    }
    if (lane == 0) counts[q] = base;
  }
}

// Dense int32 reps for k_bform_mr: dst[r][c] = llround(src[r][c]) or, with
// transpose, llround(src[c][r]); zero reps stay 0 (value == 0.0 or llround == 0
// both skip, kernels.hpp:128-130 / :151-153). 32x33 smem tiles.
template <class T>
__global__ void k_reps_dense(const T* __restrict__ src, uint64_t ld_src, uint32_t rows,
                             uint32_t cols, int transpose, int32_t* __restrict__ dst,
                             uint64_t ld_dst) {
  __shared__ int32_t tile[32][33];
  const uint32_t c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  // destination tile rows [r0, r0+32) x cols [c0, c0+32)
  for (uint32_t dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    int32_t v = 0;
    if (transpose) {
      // read src row (c0 + dy), columns r0 + tx  -> dst[r0 + tx][c0 + dy]
      const uint32_t sr = c0 + dy, sc = r0 + threadIdx.x;
      if (sr < cols && sc < rows) {
        const T x = src[(uint64_t)sr * ld_src + sc];
        if (x != T(0)) v = (int32_t)llround((double)x);
      }
    } else {
      const uint32_t sr = r0 + dy, sc = c0 + threadIdx.x;
      if (sr < rows && sc < cols) {
        const T x = src[(uint64_t)sr * ld_src + sc];
        if (x != T(0)) v = (int32_t)llround((double)x);
      }
    }
    tile[dy][threadIdx.x] = v;
  }
  __syncthreads();
  for (uint32_t dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const uint32_t r = r0 + dy, c = c0 + threadIdx.x;
    if (r < rows && c < cols)
      dst[(uint64_t)r * ld_dst + c] = transpose ? tile[threadIdx.x][dy] : tile[dy][threadIdx.x];
  }
}

// out[oc * ld_out + r] = in[ir * ld_in + c] for r < rows, c < cols, with
// ir = in_rows ? in_rows[r] : r and oc = out_rows ? out_rows[c] : c (the row
// maps gather / scatter the rows of a Case A split between the two kernels).
template <class T>
__global__ void k_transpose(const T* __restrict__ in, uint64_t ld_in, uint32_t rows,
                            uint32_t cols, T* __restrict__ out, uint64_t ld_out,
                            const uint32_t* __restrict__ in_rows,
                            const uint32_t* __restrict__ out_rows, const DevStatus* st) {
  // the result transpose writes Z only for a valid product (out untouched on
  // a validation error, like the kernels that write Z directly)
  if (st && status_failed(st)) return;
  __shared__ T tile[32][33];
  const uint32_t c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (uint32_t dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const uint32_t r = r0 + dy, c = c0 + threadIdx.x;
    if (r < rows && c < cols) {
      const uint64_t ir = in_rows ? in_rows[r] : r;
      tile[dy][threadIdx.x] = in[ir * ld_in + c];
    }
  }
  __syncthreads();
  for (uint32_t dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const uint32_t c = c0 + dy, r = r0 + threadIdx.x;
    if (r < rows && c < cols) {
      const uint64_t oc = out_rows ? out_rows[c] : c;
      out[oc * ld_out + r] = tile[threadIdx.x][dy];
    }
  }
}

// Fast mode: combine the k-slice partial products in ascending slice order
// (deterministic; the reassociation the fast mode allows is exactly this
// regrouping of each element's k-sum).
template <class T>
__global__ void k_reduce_slices(const T* __restrict__ part, uint64_t stride, uint64_t ld_part,
                                uint32_t splits, uint32_t rows, uint32_t cols,
                                T* __restrict__ out, uint64_t ld_out, const DevStatus* st) {
  if (status_failed(st)) return;
  const uint64_t total = (uint64_t)rows * cols;
  for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = idx / cols, c = idx % cols;
    const T* p = part + r * ld_part + c;
    T acc = p[0];
    for (uint32_t z = 1; z < splits; ++z) acc = acc + p[z * stride];
    out[r * ld_out + c] = acc;
  }
}

inline unsigned grid_for_warps(uint64_t tasks, int warps_per_block) {
  uint64_t blocks = (tasks + warps_per_block - 1) / warps_per_block;
  if (blocks > 148ull * 16) blocks = 148ull * 16;
  if (blocks < 1) blocks = 1;
  return (unsigned)blocks;
}

template <class T>
int vec_ok(const T* p, uint64_t ld) {
  return (reinterpret_cast<uintptr_t>(p) % 16 == 0 && (ld * sizeof(T)) % 16 == 0) ? 1 : 0;
}

}  // namespace

// ---- launchers ---------------------------------------------------------------

template <class T>
void launch_scan_stats(const T* lhs, const T* rhs, uint64_t ld, uint32_t n, int which_case,
                       DevStatus* st, uint32_t* nnz, unsigned long long* rsum, cudaStream_t s) {
  const int vec = vec_ok(lhs, ld) & vec_ok(rhs, ld);
  k_scan_stats<T><<<grid_for_warps(2ull * n, 8), 256, 0, s>>>(lhs, rhs, ld, n, which_case, vec,
                                                               st, nnz, rsum);
  note_launch();
}

template <class T>
void launch_rows(const T* x, uint64_t ld, uint32_t n, int which_case, const uint32_t* nnz,
                 const unsigned long long* rsum, uint32_t r0, uint32_t r1, int2* lists,
                 uint64_t cap, uint32_t* counts, unsigned long long* work, DevStatus* st,
                 cudaStream_t s, uint32_t* nnz_row) {
  k_rows<T><<<grid_for_warps(n, 8), 256, 0, s>>>(x, ld, n, which_case, vec_ok(x, ld), nnz, rsum,
                                                  r0, r1, lists, cap, counts, work, st, nnz_row);
  note_launch();
}

template <class T>
void launch_counts_f16(const T* y, uint64_t ld, uint32_t n, uint32_t tile_cols, __half* cnt,
                       uint64_t ldc, uint16_t* rmax, unsigned long long* fstats, cudaStream_t s) {
  const uint32_t ntiles = (n + tile_cols - 1) / tile_cols;
  k_counts_f16<T><<<grid_for_warps((uint64_t)n * ntiles, 8), 256, 0, s>>>(
      y, ld, n, tile_cols, ntiles, cnt, ldc, rmax, fstats);
  note_launch();
}

template <class T>
void launch_acompact(const T* x, uint64_t ld, uint32_t n, uint32_t r0, uint32_t ntask,
                     const uint32_t* rows_idx, typename AEntry<T>::type* lists, uint64_t cap,
                     uint32_t* counts, cudaStream_t s) {
  k_acompact<T><<<grid_for_warps(ntask, 8), 256, 0, s>>>(x, ld, n, vec_ok(x, ld), r0, ntask,
                                                         rows_idx, lists, cap, counts);
  note_launch();
}

template <class T>
void launch_transpose_compact(const T* y, uint64_t ld, uint32_t n, int2* lists, uint64_t cap,
                              uint32_t* counts, cudaStream_t s) {
  k_transpose_compact<T><<<(n + 31) / 32, 256, 0, s>>>(y, ld, n, lists, cap, counts);
  note_launch();
}

template <class T>
void launch_transpose(const T* in, uint64_t ld_in, uint32_t rows, uint32_t cols, T* out,
                      uint64_t ld_out, cudaStream_t s, const uint32_t* in_rows,
                      const uint32_t* out_rows, const DevStatus* st) {
  dim3 grid((cols + 31) / 32, (rows + 31) / 32);
  k_transpose<T><<<grid, dim3(32, 8), 0, s>>>(in, ld_in, rows, cols, out, ld_out, in_rows,
                                               out_rows, st);
  note_launch();
}

template <class T>
void launch_reps_dense(const T* src, uint64_t ld_src, uint32_t rows, uint32_t cols,
                       int transpose, int32_t* dst, uint64_t ld_dst, cudaStream_t s) {
  dim3 grid((cols + 31) / 32, (rows + 31) / 32);
  k_reps_dense<T><<<grid, dim3(32, 8), 0, s>>>(src, ld_src, rows, cols, transpose, dst, ld_dst);
  note_launch();
}

template <class T>
void launch_reduce_slices(const T* part, uint64_t stride, uint64_t ld_part, uint32_t splits,
                          uint32_t rows, uint32_t cols, T* out, uint64_t ld_out,
                          const DevStatus* st, cudaStream_t s) {
  uint64_t blocks = ((uint64_t)rows * cols + 255) / 256;
  if (blocks > 148ull * 16) blocks = 148ull * 16;
  if (blocks < 1) blocks = 1;
  k_reduce_slices<T><<<(unsigned)blocks, 256, 0, s>>>(part, stride, ld_part, splits, rows, cols,
                                                      out, ld_out, st);
  note_launch();
}

#define INSTANTIATE(T)                                                                         \
  template void launch_scan_stats<T>(const T*, const T*, uint64_t, uint32_t, int, DevStatus*,  \
                                     uint32_t*, unsigned long long*, cudaStream_t);            \
  template void launch_rows<T>(const T*, uint64_t, uint32_t, int, const uint32_t*,             \
                               const unsigned long long*, uint32_t, uint32_t, int2*, uint64_t, \
                               uint32_t*, unsigned long long*, DevStatus*, cudaStream_t,       \
                               uint32_t*);                                                     \
  template void launch_counts_f16<T>(const T*, uint64_t, uint32_t, uint32_t, __half*, uint64_t, \
                                     uint16_t*, unsigned long long*, cudaStream_t);            \
  template void launch_acompact<T>(const T*, uint64_t, uint32_t, uint32_t, uint32_t,           \
                                   const uint32_t*, typename AEntry<T>::type*, uint64_t,      \
                                   uint32_t*, cudaStream_t);                                   \
  template void launch_transpose_compact<T>(const T*, uint64_t, uint32_t, int2*, uint64_t,     \
                                            uint32_t*, cudaStream_t);                          \
  template void launch_transpose<T>(const T*, uint64_t, uint32_t, uint32_t, T*, uint64_t,      \
                                    cudaStream_t, const uint32_t*, const uint32_t*,            \
                                    const DevStatus*);                                         \
  template void launch_reps_dense<T>(const T*, uint64_t, uint32_t, uint32_t, int, int32_t*,    \
                                     uint64_t, cudaStream_t);                                  \
  template void launch_reduce_slices<T>(const T*, uint64_t, uint64_t, uint32_t, uint32_t,     \
                                        uint32_t, T*, uint64_t, const DevStatus*,             \
                                        cudaStream_t);

INSTANTIATE(float)
INSTANTIATE(double)

}  // namespace afmm_dev
