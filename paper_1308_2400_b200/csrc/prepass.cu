// prepass.cu -- O(n^2) device prepass of the AFMM product (sm_100a).
//
// Replaces the inline zero tests and the up-front validation of the
// reference kernels (/root/reference/proj/include/afmm/kernels.hpp:25-43,
// :121-130, :150-159) with streaming passes (one warp per matrix row,
// 128-bit loads, one read of each operand):
//
//   k_scan_stats   rows of both operands: finite check (matrix.hpp:31-35), rep
//                  validation of the rep operand (kernels.hpp:25-43; first
//                  offender by atomicMax on the inverted row-major index), and
//                  the per-k vector the work formulas need: nnz(Y[k,:]) (Case B)
//                  or R_k = sum_j |llround Y[k,j]| (Case A)
//   k_rows         rows of X: exact additions W_i and zero_skips (closed forms
//                  of kernels.hpp:119-134 / :148-163), the slab's OpCounts, and
//                  (Case B, one row per list) the warp-scan stream compaction of
//                  the row's nonzero reps into an ordered (k, rep) list: the
//                  zero-skip of kernels.hpp:151-153 done once instead of per (i,k,j)
//   k_transpose_compact  (Case A) the same compaction for the columns of Y,
//                  through 32x33 smem tiles (the rep list of B-form row j is
//                  column j of Y)
//   k_counts_f16, k_choose, k_acompact  the A-form inputs and the device-side
//                  A-form / B-form choice (costmodel.h)
//
// plus k_transpose (Case A operand/result transposes) and k_reduce_slices
// (fast-mode split-k combine). All are HBM-bound; none does FP arithmetic on
// the product.
#include <cuda_fp16.h>

#include "common.cuh"
#include "costmodel.h"
#include "kernels.h"

namespace afmm_dev {

namespace {

constexpr unsigned FULL = 0xffffffffu;
// Largest |rep| one list entry {k, int32 rep} holds.
constexpr unsigned long long kMaxRep = 0x7fffffffull;

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

__device__ __forceinline__ unsigned long long abs_ll(long long r) {
  return r < 0 ? 0ull - (unsigned long long)r : (unsigned long long)r;
}

// The rep of an element as the reference reads it: value == 0.0 or
// llround == 0 both mean "no term" (kernels.hpp:128-130, :151-153).
template <class T>
__device__ __forceinline__ long long rep_of(T v) {
  return v != T(0) ? llround((double)v) : 0ll;
}

// rep_of for an operand that passed validation: an fp32 rep is then an exact
// integer or rounds to 0 (|v| <= 1e-9; float spacing near integers >= 1 is
// far wider than 1e-9), so truncation equals llround without FP64 work.
template <class T>
__device__ __forceinline__ long long rep_valid(T v) {
  if constexpr (sizeof(T) == 4) return (long long)v;
  else return rep_of(v);
}

// List entries a term of magnitude a needs when an entry holds at most M.
__device__ __forceinline__ uint32_t entries_for(unsigned long long a, unsigned long long M) {
  if (a <= M) return a != 0 ? 1u : 0u;
  const unsigned long long c = (a + M - 1) / M;
  return c > 0x00ffffffull ? 0x00ffffffu : (uint32_t)c;  // saturates: such a list cannot be allocated
}

// Part c of a term split into entries of at most M: the first parts are M.
__device__ __forceinline__ long long part_of(long long r, uint32_t c, unsigned long long M) {
  const unsigned long long a = abs_ll(r), done = (unsigned long long)c * M;
  if (a <= done) return 0;
  const unsigned long long p = a - done < M ? a - done : M;
  return r < 0 ? -(long long)p : (long long)p;
}

// Record the length of a list that does not fit (the runtime re-runs with it).
__device__ __forceinline__ void note_list(DevStatus* st, unsigned long long len, uint64_t cap) {
  if (len > cap) atomicMax(&st->list_need, len);
}

// One element as the validation sees it (kernels.hpp:25-43 on the widened
// value; matrix.hpp:31-35 for the finite check): *kind = 0 ok, 1 not
// integer-valued, 2 beyond the exact integer range; *rep = llround (0 for a
// zero or a value that rounds to 0). NaN: kind 0, rep 0 (reported apart).
__device__ __forceinline__ void classify(double d, int* kind, long long* rep) {
  *kind = rep_kind(d);
  *rep = (*kind == 0 && d == d && d != 0.0) ? llround(d) : 0ll;
}
// fp32 without double arithmetic: a float is integer-valued within 1e-9
// exactly when it is integral (float spacing is >= 2^-24 at |v| >= 0.5) or
// |v| <= 1e-9 (then it rounds to 0); integral floats convert exactly. (The
// FP64 rounding of the generic path made k_scan_stats FP64-bound: 108 us at
// n = 4096 for 128 MB.)
__device__ __forceinline__ void classify(float v, int* kind, long long* rep) {
  const float a = fabsf(v);
  if (rintf(v) == v) {  // integral, +-0 and +-inf included
    *kind = a > 9007199254740992.0f ? 2 : 0;
    *rep = *kind == 0 ? (long long)v : 0ll;
  } else {
    *kind = (double)a > 1e-9 ? 1 : 0;  // NaN compares false: kind 0
    *rep = 0;
  }
}

// Per-lane state of one row scan (k_scan_stats). Offenders are kept as the
// lane's first column (its columns ascend), turned into inverted row-major
// keys once per row.
struct ScanState {
  uint32_t nf_j = ~0u;                // first non-finite element
  uint32_t rb_j = ~0u, rb_kind = 0;   // first rep that fails kernels.hpp:31-40
  uint32_t rn_j = ~0u;                // first NaN rep
  uint32_t cnt = 0;                   // nonzero elements (Case B rhs: nnz_k)
  uint32_t rmx = 0, rneg = 0;         // rep operand: max |rep| (saturated at 255), any < 0
  uint32_t nzr = 0, big = 0, tmx = 0; // Case A statistics: nonzero reps, > 2048, tile max
  unsigned long long s = 0;           // Case A: sum |rep| (R_k)
};

// One element, every check spelled out (fp64, and fp32 elements that leave
// the fast path below).
template <class T>
__device__ __forceinline__ void scan_elem(T x, uint32_t j, bool check_finite, bool is_rep,
                                          bool is_rhs, bool stats, ScanState& S) {
  if (check_finite && !isfinite(x) && S.nf_j == ~0u) S.nf_j = j;
  if (is_rhs) S.cnt += x != T(0) ? 1u : 0u;
  if (!is_rep) return;
  int kind;
  long long r;
  classify(x, &kind, &r);
  // (an infinite rep: kind 2, as in the reference)
  if (kind && S.rb_j == ~0u) {
    S.rb_j = j;
    S.rb_kind = (uint32_t)kind;
  }
  if (isnan(x) && S.rn_j == ~0u) S.rn_j = j;
  const unsigned long long a = abs_ll(r);
  S.rmx = max(S.rmx, a >= 255ull ? 255u : (uint32_t)a);
  S.rneg |= r < 0 ? 1u : 0u;
  if (is_rhs && isfinite(x)) {  // Case A (rhs = the reps): R_k; statistics
    S.s += a;
    if (stats) {
      S.nzr += a != 0 ? 1u : 0u;
      S.big += a > 2048ull ? 1u : 0u;
      S.tmx = max(S.tmx, a > 2048ull ? 2048u : (uint32_t)a);
    }
  }
}

// Four consecutive elements j0..j0+3 (all < n). fp32 fast path: when the four
// are finite (and, for the rep operand, integral with |rep| <= 2^24) every
// check passes and the rep statistics are plain 32-bit arithmetic; anything
// else takes scan_elem. (k_scan_stats was issue bound at ~60 instructions per
// element with the generic checks, 86 us for 128 MB at n = 4096.)
template <class T>
__device__ __forceinline__ void scan4(const T (&v)[4], uint32_t j0, uint32_t n, bool check_finite,
                                      bool is_rep, bool is_rhs, bool stats, ScanState& S) {
  if constexpr (sizeof(T) == 4) {
    if (j0 + 3 < n) {
      bool good = true;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float x = v[e], a = fabsf(x);
        good = good && (is_rep ? (x == rintf(x) && a <= 16777216.0f) : a <= 3.402823466e38f);
      }
      if (good) {
        uint32_t sum = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float x = v[e];
          if (is_rhs) S.cnt += x != 0.0f ? 1u : 0u;
          if (is_rep) {
            const uint32_t a = (uint32_t)fabsf(x);
            S.rmx = max(S.rmx, min(a, 255u));
            S.rneg |= x < 0.0f ? 1u : 0u;
            sum += a;
            if (stats) {
              S.nzr += a != 0 ? 1u : 0u;
              S.big += a > 2048u ? 1u : 0u;
              S.tmx = max(S.tmx, min(a, 2048u));
            }
          }
        }
        if (is_rep && is_rhs) S.s += sum;
        return;
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e)
    if (j0 + e < n) scan_elem(v[e], j0 + e, check_finite, is_rep, is_rhs, stats, S);
}

// warp task t < (l1 - l0): lhs row l0 + t; then rhs rows q0 .. q1 - 1.
// fstats (Case A, optional; accumulated): the cost-model statistics of the
// rhs rows -- nonzero reps, sum over (row, atile-column tile) of the tile's
// max |rep| (clamped to 2048), reps beyond 2048, sum of |rep| (as
// k_counts_f16 computes them, so the A-form counts can be built after the
// choice, only when some row takes the A-form).
template <class T>
__global__ void k_scan_stats(const T* __restrict__ lhs, const T* __restrict__ rhs, uint64_t ld,
                             uint32_t n, int which_case, int vec, int check_finite, uint32_t l0,
                             uint32_t l1, uint32_t q0, uint32_t q1, DevStatus* st,
                             uint32_t* __restrict__ nnz, unsigned long long* __restrict__ rsum,
                             unsigned long long* __restrict__ fstats, uint32_t atile) {
  constexpr uint32_t U = 4;          // 16-byte loads in flight per lane
  constexpr uint32_t W = 128 * U;    // columns per warp iteration
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t ntl = l1 - l0, ntask = ntl + (q1 - q0);
  for (uint64_t t = warp; t < ntask; t += nwarps) {
    const bool is_rhs = t >= ntl;
    const uint64_t i = is_rhs ? q0 + (t - ntl) : l0 + t;
    const T* row = (is_rhs ? rhs : lhs) + i * ld;
    // Case A validates rhs (kernels.hpp:115), Case B lhs (:144)
    const bool is_rep = is_rhs == (which_case == 0);
    const bool stats = is_rhs && which_case == 0 && fstats != nullptr;
    ScanState S;
    unsigned long long trip = 0;
    for (uint32_t c0 = 0; c0 < n; c0 += W) {  // warp-uniform trip count
      T v[U][4];
#pragma unroll
      for (uint32_t u = 0; u < U; ++u) load4(row, c0 + u * 128 + 4 * lane, n, vec != 0, v[u]);
#pragma unroll
      for (uint32_t u = 0; u < U; ++u)
        scan4(v[u], c0 + u * 128 + 4 * lane, n, check_finite != 0, is_rep, is_rhs, stats, S);
      // per-tile max |rep| (A-form trip counts): tiles of atile columns
      if (stats && ((c0 + W) % atile == 0 || c0 + W >= n)) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) S.tmx = max(S.tmx, __shfl_xor_sync(FULL, S.tmx, o));
        trip += S.tmx;
        S.tmx = 0;
      }
    }
    const unsigned long long base = i * (uint64_t)n;
    unsigned long long nf = S.nf_j != ~0u ? ~(base + S.nf_j) : 0ull;  // inverted keys, 0 = none
    unsigned long long rb =
        S.rb_j != ~0u ? ~(((base + S.rb_j) << 2) | (unsigned long long)S.rb_kind) : 0ull;
    unsigned long long rn = S.rn_j != ~0u ? ~(base + S.rn_j) : 0ull;
    if (__any_sync(FULL, (nf | rb | rn) != 0)) {
      nf = warp_max_u64(nf);
      rb = warp_max_u64(rb);
      rn = warp_max_u64(rn);
      if (lane == 0) {
        if (nf) atomicMax(is_rhs ? &st->nonfinite_rhs_inv : &st->nonfinite_lhs_inv, nf);
        if (rb) atomicMax(&st->rep_bad_inv, rb);
        if (rn) atomicMax(&st->rep_nan_inv, rn);
      }
    }
    if (is_rep && __any_sync(FULL, (S.rmx > kGroupMaxRep) || S.rneg != 0)) {
      uint32_t rmx = S.rmx, rneg = S.rneg;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        rmx = max(rmx, __shfl_xor_sync(FULL, rmx, o));
        rneg |= __shfl_xor_sync(FULL, rneg, o);
      }
      if (lane == 0) {
        if (rmx > kGroupMaxRep) atomicMax(&st->rep_max, rmx);
        if (rneg) atomicOr(&st->rep_neg, 1u);
      }
    }
    if (is_rhs) {
      if (which_case == 1) {
        uint32_t cnt = S.cnt;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(FULL, cnt, o);
        if (lane == 0) nnz[i] = cnt;
      } else {
        const unsigned long long sum = warp_sum_u64(S.s);
        if (lane == 0) rsum[i] = sum;
        if (stats) {
          uint32_t nzr = S.nzr, big = S.big;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            nzr += __shfl_xor_sync(FULL, nzr, o);
            big += __shfl_xor_sync(FULL, big, o);
          }
          if (lane == 0) {
            if (nzr) atomicAdd(&fstats[0], (unsigned long long)nzr);
            if (trip) atomicAdd(&fstats[1], trip);
            if (big) atomicAdd(&fstats[2], (unsigned long long)big);
            if (sum) atomicAdd(&fstats[3], sum);
          }
        }
      }
    }
  }
}

// Rows i in [a0, a1) of X: W_i -> work[i] (when work != nullptr); rows in the
// slab [r0, r1) add to the slab OpCounts and get (Case B, lists != nullptr)
// their compacted rep list / (Case A, nnz_row != nullptr) their nonzero-base
// count.
// Case A: W_i = sum_{k: X[i,k] != 0} R_k, zs_i = #{k: X[i,k] == 0}
// Case B: W_i = sum_k |rep_ik| nnz_k,    zs_i = sum_{k: rep_ik != 0} (n - nnz_k)
template <class T>
__global__ void k_rows(const T* __restrict__ x, uint64_t ld, uint32_t n, int which_case, int vec,
                       const uint32_t* __restrict__ nnz,
                       const unsigned long long* __restrict__ rsum, uint32_t a0, uint32_t a1,
                       uint32_t r0, uint32_t r1, int2* __restrict__ lists, uint64_t cap,
                       uint32_t* __restrict__ counts, unsigned long long* __restrict__ work,
                       DevStatus* st, uint32_t* __restrict__ nnz_row, int group_allow) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  // group mode: k_bgroup reads the dense group index instead of the lists
  const bool lists_needed = lists != nullptr && !group_mode(st, group_allow);
  const bool packed = packed_mode(st, group_allow);  // 4-byte entries (every |rep| <= 127)
  for (uint64_t i = a0 + warp; i < a1; i += nwarps) {
    const T* row = x + i * ld;
    const bool in_slab = i >= r0 && i < r1;
    const bool compact = which_case == 1 && in_slab && lists_needed;
    int2* out = compact ? lists + (i - r0) * cap : nullptr;
    unsigned long long w = 0, z = 0, base = 0;
    // warp-uniform trip count (the scan below); 4 loads in flight per lane
    for (uint32_t c1 = 0; c1 < n; c1 += 512) {
      T vv[4][4];
#pragma unroll
      for (uint32_t u = 0; u < 4; ++u) load4(row, c1 + u * 128 + 4 * lane, n, vec != 0, vv[u]);
#pragma unroll
      for (uint32_t u = 0; u < 4; ++u) {
        const uint32_t c0 = c1 + u * 128;
        const uint32_t j0 = c0 + 4 * lane;
        const T* v = vv[u];
        long long rep[4];
        // Case A: R_k of the four columns as two 16-byte loads (a load per
        // nonzero element kept k_rows on long-scoreboard stalls)
        unsigned long long rs[4] = {0ull, 0ull, 0ull, 0ull};
        if (which_case == 0) {
          if (j0 + 3 < n) {
            const ulonglong2 a = __ldg(reinterpret_cast<const ulonglong2*>(rsum + j0));
            const ulonglong2 b = __ldg(reinterpret_cast<const ulonglong2*>(rsum + j0 + 2));
            rs[0] = a.x; rs[1] = a.y; rs[2] = b.x; rs[3] = b.y;
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) rs[e] = j0 + e < n ? rsum[j0 + e] : 0ull;
          }
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t j = j0 + e;
          rep[e] = (which_case == 1 && j < n) ? rep_of(v[e]) : 0;
          if (which_case == 0) {
            if (j < n) {
              if (v[e] == T(0)) ++z;
              else w += rs[e];
            }
          } else if (rep[e] != 0) {
            const unsigned long long nb = nnz[j];
            w += abs_ll(rep[e]) * nb;  // count bookkeeping, not an element product
            z += (unsigned long long)n - nb;
          }
        }
        if (compact) {
          uint32_t ne[4], mine = 0;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            ne[e] = entries_for(abs_ll(rep[e]), kMaxRep);
            mine += ne[e];
          }
          uint32_t total;
          unsigned long long pos = base + warp_excl_scan(mine, lane, &total);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (ne[e] == 1) {
              if (pos < cap) {
                if (packed) reinterpret_cast<uint32_t*>(out)[pos] = pack_entry(j0 + e, rep[e]);
                else out[pos] = make_int2((int)(j0 + e), (int)rep[e]);
              }
              ++pos;
            } else {
              for (uint32_t c = 0; c < ne[e]; ++c, ++pos)
                if (pos < cap)
                  out[pos] = make_int2((int)(j0 + e), (int)part_of(rep[e], c, kMaxRep));
            }
          }
          base += total;
        }
      }
    }
    w = warp_sum_u64(w);
    z = warp_sum_u64(z);
    if (lane == 0) {
      if (work) work[i] = w;
      if (in_slab) {
        if (w) atomicAdd(&st->additions, w);
        if (z) atomicAdd(&st->zero_skips, z);
        if (compact) {
          counts[i - r0] = (uint32_t)(base < 0xffffffffull ? base : 0xffffffffull);
          note_list(st, base, cap);
        }
        // Case A: nonzero bases of the row (its A-form cost)
        if (nnz_row && which_case == 0) nnz_row[i - r0] = n - (uint32_t)z;
      }
    }
  }
}

// Case A rep lists: B-form row j = column j of Y. A block owns 32 columns and
// walks k in 32-row tiles through smem; warp w compacts columns 4w..4w+3.
// skip (optional): nothing to do when *skip == 0 (the device-side Case A
// choice gave every row to the A-form).
template <class T>
__global__ void __launch_bounds__(256)
    k_transpose_compact(const T* __restrict__ y, uint64_t ld, uint32_t n, int2* __restrict__ lists,
                        uint64_t cap, uint32_t* __restrict__ counts, DevStatus* st,
                        const uint32_t* __restrict__ skip, int group_allow) {
  if (skip && *skip == 0) return;
  if (group_mode(st, group_allow)) return;  // k_bgroup runs: no lists
  const bool packed = packed_mode(st, group_allow);  // 4-byte entries (every |rep| <= 127)
  __shared__ T tile[32][33];
  const uint32_t tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const uint32_t j0 = blockIdx.x * 32;
  unsigned long long base[4] = {0, 0, 0, 0};
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
    const uint32_t k = k0 + tx;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t j = j0 + ty * 4 + q;
      const long long rep = k < n ? rep_of(tile[tx][ty * 4 + q]) : 0;  // Y[k, j]
      const uint32_t ne = entries_for(abs_ll(rep), kMaxRep);
      uint32_t total;
      unsigned long long pos = base[q] + warp_excl_scan(ne, tx, &total);
      if (j < n) {
        if (packed) {  // (ne <= 1: no rep is split)
          if (ne && pos < cap)
            reinterpret_cast<uint32_t*>(lists + (uint64_t)j * cap)[pos] = pack_entry(k, rep);
          pos += ne;
        } else {
          for (uint32_t c = 0; c < ne; ++c, ++pos)
            if (pos < cap)
              lists[(uint64_t)j * cap + pos] =
                  make_int2((int)k, (int)(ne == 1 ? rep : part_of(rep, c, kMaxRep)));
        }
      }
      base[q] += total;
    }
    __syncthreads();
  }
  if (tx == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t j = j0 + ty * 4 + q;
      if (j < n) {
        counts[j] = (uint32_t)(base[q] < 0xffffffffull ? base[q] : 0xffffffffull);
        note_list(st, base[q], cap);
      }
    }
  }
}

// ---- group index of the small-rep group kernel (k_bgroup, bform.cu) ----
//
// B-form rows 5g .. 5g+4 form group g; gidx[g][k] = (t0 + 3 t1 + 9 t2) |
// (t3 + 3 t4) << 8, t_r = the row's rep at k (0..kGroupMaxRep in group mode,
// 0 past the last row and for k >= n up to the padded ldg). Dense: one u16
// per (group, k), so both builders are plain parallel passes (no compaction);
// k_bgroup skips the k with index 0. Both exit unless the device-side status
// chose group mode.
// A rep of a validated group-mode operand (fp32, 0..kGroupMaxRep): the float
// is an exact small integer or rounds to 0 (|v| <= 1e-9), so truncation is
// llround (kernels.hpp:128-130) without the FP64 conversion.
template <class T>
__device__ __forceinline__ uint32_t group_rep(T v) {
  if constexpr (sizeof(T) == 4) return (uint32_t)(int)v;
  else return (uint32_t)rep_of(v);
}

__device__ __forceinline__ uint32_t group_digit(int r) {
  return r == 0 ? 1u : r == 1 ? 3u : r == 2 ? 9u : r == 3 ? 256u : 768u;
}

// Case B: groups of slab rows r0 + 5g .. of X; one warp per group.
template <class T>
__global__ void k_group_idx_rows(const T* __restrict__ x, uint64_t ld, uint32_t n, int vec,
                                 uint32_t r0, uint32_t rows, uint16_t* __restrict__ gidx,
                                 uint64_t ldg, const DevStatus* st, int allow) {
  if (!group_mode(st, allow) || status_failed(st)) return;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t ngroups = (rows + kGroupRows - 1) / kGroupRows;
  for (uint64_t g = warp; g < ngroups; g += nwarps) {
    for (uint64_t c0 = 0; c0 < ldg; c0 += 128) {
      const uint32_t j0 = (uint32_t)c0 + 4 * lane;
      uint32_t idx[4] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int r = 0; r < kGroupRows; ++r) {
        const uint64_t q = g * kGroupRows + r;
        if (q >= rows) break;
        T v[4];
        load4(x + (r0 + q) * ld, j0, n, vec != 0, v);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (j0 + e < n) idx[e] += group_rep(v[e]) * group_digit(r);
      }
      if (j0 < ldg)  // ldg % 8 == 0: the 4 entries are in range together
        *reinterpret_cast<ushort4*>(gidx + g * ldg + j0) =
            make_ushort4((unsigned short)idx[0], (unsigned short)idx[1], (unsigned short)idx[2],
                         (unsigned short)idx[3]);
    }
  }
}

// Case A: groups of columns 5g .. of Y (B-form row j = column j of Y), through
// 32 k x 160 column smem tiles (32 groups per block).
template <class T>
__global__ void __launch_bounds__(256)
    k_group_idx_cols(const T* __restrict__ y, uint64_t ld, uint32_t n, int vec,
                     uint16_t* __restrict__ gidx, uint64_t ldg, const DevStatus* st, int allow,
                     const uint32_t* __restrict__ skip) {
  if (!group_mode(st, allow) || status_failed(st)) return;
  if (skip && *skip == 0) return;  // the Case A choice left the B-form no rows
  constexpr uint32_t GC = 32 * kGroupRows;  // columns per block
  __shared__ uint8_t tile[32][GC + 1];
  const uint32_t j0 = blockIdx.x * GC, k0 = blockIdx.y * 32;
  if (vec && j0 + GC <= n && k0 + 32 <= n) {
    // whole tile: 16-byte loads, all of a thread's issued before any is used
    constexpr uint32_t Q = 32 * GC / 4 / 256;  // 16-byte quads per thread (5)
    T q[Q][4];
#pragma unroll
    for (uint32_t u = 0; u < Q; ++u) {
      const uint32_t idx = threadIdx.x + u * 256, r = idx / (GC / 4), c = (idx % (GC / 4)) * 4;
      load4(y + (uint64_t)(k0 + r) * ld + j0, c, GC, true, q[u]);
    }
#pragma unroll
    for (uint32_t u = 0; u < Q; ++u) {
      const uint32_t idx = threadIdx.x + u * 256, r = idx / (GC / 4), c = (idx % (GC / 4)) * 4;
#pragma unroll
      for (int e = 0; e < 4; ++e) tile[r][c + e] = (uint8_t)group_rep(q[u][e]);
    }
  } else {
    for (uint32_t i = threadIdx.x; i < 32 * GC; i += blockDim.x) {
      const uint32_t r = i / GC, c = i % GC, k = k0 + r, j = j0 + c;
      tile[r][c] = (k < n && j < n) ? (uint8_t)group_rep(y[(uint64_t)k * ld + j]) : (uint8_t)0;
    }
  }
  __syncthreads();
  const uint32_t gl = threadIdx.x >> 3, kq = (threadIdx.x & 7) * 4;
  const uint64_t g = (uint64_t)blockIdx.x * 32 + gl;
  const uint32_t ngroups = (n + kGroupRows - 1) / kGroupRows;
  if (g >= ngroups || k0 + kq >= ldg) return;
  uint32_t idx[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    uint32_t v = 0;
#pragma unroll
    for (int r = 0; r < kGroupRows; ++r) v += (uint32_t)tile[kq + e][gl * kGroupRows + r] * group_digit(r);
    idx[e] = v;
  }
  *reinterpret_cast<ushort4*>(gidx + g * ldg + k0 + kq) =
      make_ushort4((unsigned short)idx[0], (unsigned short)idx[1], (unsigned short)idx[2],
                   (unsigned short)idx[3]);
}

// ---- A-form prepass (k_aform, Case A with the base uniform per warp) ----

// A-form rep counts: cnt[k][j] = llround(Y[k,j]) as fp16 (exact for |rep| <=
// 2048, the A-form's eligibility bound; 0 for zero reps, kernels.hpp:128-130),
// and per (k, column tile) the largest |rep| (the warp-uniform trip count of
// the predicated add loop) with bit 15 set when the tile row holds a negative
// rep. One warp per (k, tile).
// fstats (accumulated): [0] nonzero reps, [1] sum of the per-(k, tile) trip
// counts, [2] reps beyond 2048, [3] sum of |rep| -- the cost-model inputs.
template <class T>
__global__ void k_counts_f16(const T* __restrict__ y, uint64_t ld, uint32_t n, int vec,
                             uint32_t tile_cols, uint32_t ntiles, __half* __restrict__ cnt,
                             uint64_t ldc,
                             uint16_t* __restrict__ rmax, unsigned long long* __restrict__ fstats,
                             const uint32_t* __restrict__ need) {
  if (need && *need == 0) return;  // the device-side choice gave the A-form no rows
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t task = warp; task < (uint64_t)n * ntiles; task += nwarps) {
    const uint64_t k = task / ntiles;
    const uint32_t t = (uint32_t)(task % ntiles);
    uint32_t mx = 0, neg = 0, nz = 0, big = 0;
    unsigned long long sum = 0;
    // 4 columns per lane per 16-byte load, all of the tile's loads in flight
    // (scalar loads left this pass at ~1.2 TB/s)
    const uint32_t cb = t * tile_cols, ce = min(cb + tile_cols, n);
    constexpr uint32_t U = 8;
    for (uint32_t c1 = cb; c1 < ce; c1 += 128 * U) {
      T v[U][4];
#pragma unroll
      for (uint32_t u = 0; u < U; ++u) load4(y + k * ld, c1 + u * 128 + 4 * lane, ce, vec != 0, v[u]);
#pragma unroll
      for (uint32_t u = 0; u < U; ++u) {
        const uint32_t c = c1 + u * 128 + 4 * lane;
        if (c >= ce) break;
        __half h[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          long long r = c + e < ce ? rep_valid(v[u][e]) : 0ll;
          nz += r != 0 ? 1u : 0u;
          sum += abs_ll(r);
          if (r > 2048 || r < -2048) {
            big += 1;
            r = r > 0 ? 2048 : -2048;
          }
          h[e] = __int2half_rn((int)r);
          const uint32_t a = (uint32_t)(r < 0 ? -r : r);
          mx = a > mx ? a : mx;
          neg |= r < 0 ? 1u : 0u;
        }
        __half* dst = cnt + k * ldc + c;  // ldc % 64 == 0: 8-byte aligned
        if (c + 3 < ce) {
          const __half2 p[2] = {__halves2half2(h[0], h[1]), __halves2half2(h[2], h[3])};
          *reinterpret_cast<uint2*>(dst) = *reinterpret_cast<const uint2*>(p);
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (c + e < ce) dst[e] = h[e];
        }
      }
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
      if (!fstats) continue;
      if (nz) atomicAdd(&fstats[0], (unsigned long long)nz);
      if (mx) atomicAdd(&fstats[1], (unsigned long long)mx);
      if (big) atomicAdd(&fstats[2], (unsigned long long)big);
      if (sum) atomicAdd(&fstats[3], sum);
    }
  }
}

// Device-side Case A choice (one CTA): from the slab rows' nonzero-base
// counts and the statistics of Y, evaluate the cost model (costmodel.h) and
// write plan[0] = m (A-form rows), plan[1] = rows - m (B-form rows), and the
// row order ridx: the A rows first (the m sparsest, by nonzero count, ties in
// row order), then the B rows in ascending order (identity unless split).
// scratch: 3 * (n + 2) words.
constexpr int kChooseThreads = 1024;
// Dynamic shared memory of k_choose: its scratch when that fits next to the
// static arrays (n <= 12000: 192 KB), else 0 (global scratch).
__host__ __device__ inline size_t choose_smem_bytes(uint64_t n) {
  const size_t b = (4 * (n + 2) + 2) * sizeof(uint32_t);
  return n <= 12000 ? b : 0;
}
constexpr int kChooseCands = 1024;  // split candidates evaluated (j < 1024 B tiles)

__global__ void __launch_bounds__(kChooseThreads)
    k_choose(CaseAModel md, uint32_t rows, int variant, const uint32_t* __restrict__ nnz_row,
             const unsigned long long* __restrict__ fstats, uint32_t* __restrict__ scratch,
             uint32_t* __restrict__ plan, uint32_t* __restrict__ ridx, DevStatus* st) {
  __shared__ double s_pre[kChooseCands + 1];
  __shared__ double s_split[kChooseCands + 1];  // modeled cost of the split with c B tiles
  __shared__ uint32_t s_m, s_vstar, s_tstar;
  __shared__ uint32_t s_wsum[32];
  const uint32_t tid = threadIdx.x, n = (uint32_t)md.n;
  const uint32_t nb = n + 2;  // values 0..n, plus one past the end
  // the histogram and its prefix sums live in shared memory when they fit
  // (the launcher sizes the dynamic smem; global scratch otherwise): the
  // binary searches over `cum` below are serial dependent loads, ~30 cycles
  // each from smem against ~600 from L2 (k_choose took 54 us at n = 4096)
  extern __shared__ __align__(8) uint32_t s_dyn[];
  if (choose_smem_bytes(n)) scratch = s_dyn;
  uint32_t* hist = scratch;             // count of rows per nonzero-base value
  uint32_t* cum = scratch + nb;         // rows with value < v (then: next A slot of value v)
  unsigned long long* csum = reinterpret_cast<unsigned long long*>(scratch + 2 * nb);  // 8-byte aligned
  md.nnz_y = fstats[0];
  md.trip_sum = fstats[1];
  md.rep_sum = fstats[3];
  md.group = group_mode(st, md.group_allow);  // the B part runs k_bgroup
  const bool a_ok = fstats[2] == 0;  // every |rep| <= 2048 (exact fp16 counts)

  for (uint32_t v = tid; v < nb; v += kChooseThreads) hist[v] = 0;
  __syncthreads();
  // warp-aggregated: rows of equal density (all of them when X is dense) would
  // otherwise serialise on one counter
  for (uint32_t i0 = 0; i0 < rows; i0 += kChooseThreads) {
    const uint32_t i = i0 + tid;
    const uint32_t v = i < rows ? min(nnz_row[i], n) : 0xffffffffu;
    const unsigned peers = __match_any_sync(FULL, v);
    if (v != 0xffffffffu && (tid & 31) == (uint32_t)(__ffs(peers) - 1))
      atomicAdd(&hist[v], (uint32_t)__popc(peers));
  }
  __syncthreads();
  // exclusive scans over the values: each thread a contiguous chunk
  const uint32_t per = (nb + kChooseThreads - 1) / kChooseThreads;
  const uint32_t v0 = min(tid * per, nb), v1 = min(v0 + per, nb);
  uint32_t lc = 0;
  unsigned long long ls = 0;
  for (uint32_t v = v0; v < v1; ++v) {
    lc += hist[v];
    ls += (unsigned long long)hist[v] * v;
  }
  // block exclusive scan of (lc, ls): warp scans + warp totals
  const uint32_t lane = tid & 31, wid = tid >> 5;
  uint32_t xc = lc;
  unsigned long long xs = ls;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t yc = __shfl_up_sync(FULL, xc, o);
    const unsigned long long ys = __shfl_up_sync(FULL, xs, o);
    if (lane >= (uint32_t)o) {
      xc += yc;
      xs += ys;
    }
  }
  __shared__ unsigned long long s_wsum_s[32];
  if (lane == 31) {
    s_wsum[wid] = xc;
    s_wsum_s[wid] = xs;
  }
  __syncthreads();
  if (wid == 0) {
    uint32_t c = s_wsum[lane];
    unsigned long long sm = s_wsum_s[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t yc = __shfl_up_sync(FULL, c, o);
      const unsigned long long ys = __shfl_up_sync(FULL, sm, o);
      if (lane >= (uint32_t)o) {
        c += yc;
        sm += ys;
      }
    }
    s_wsum[lane] = c - s_wsum[lane];        // exclusive warp offsets
    s_wsum_s[lane] = sm - s_wsum_s[lane];
  }
  __syncthreads();
  uint32_t rc = s_wsum[wid] + xc - lc;
  unsigned long long rs = s_wsum_s[wid] + xs - ls;
  for (uint32_t v = v0; v < v1; ++v) {
    cum[v] = rc;
    csum[v] = rs;
    rc += hist[v];
    rs += (unsigned long long)hist[v] * v;
  }
  __syncthreads();
  // nonzero bases of the m sparsest rows: value v* with cum[v*] <= m < cum[v*+1]
  auto pre_of = [&](uint64_t m, uint32_t* vstar) -> double {
    uint32_t lo = 0, hi = n + 1;  // largest v with cum[v] <= m
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) >> 1;
      if (cum[mid] <= m) lo = mid;
      else hi = mid - 1;
    }
    if (vstar) *vstar = lo;
    return (double)csum[lo] + (double)lo * (double)(m - cum[lo]);
  };
  const uint64_t tb = md.tile_rows();
  // candidate c: c = 0 -> m = rows (pure A), c = j >= 1 -> m = rows - j * tb;
  // each thread prices its own split (thread 0 alone took ~20 us: 64-bit
  // divisions in the wave quantisation of every candidate)
  for (uint32_t c = tid; c <= kChooseCands; c += kChooseThreads) {
    const uint64_t m = c == 0 ? rows : (uint64_t)rows - (uint64_t)c * tb;
    const bool ok = c == 0 || (uint64_t)c * tb < rows;
    s_pre[c] = ok ? pre_of(m, nullptr) : 0.0;
    s_split[c] = (ok && c > 0) ? md.cost_a(m, s_pre[c]) + md.cost_b(c) : 0.0;
  }
  __syncthreads();
  if (tid == 0) {
    uint64_t m = 0;
    if (a_ok && rows > 0 && (rows - 1) / tb < (uint64_t)kChooseCands) {
      m = choose_aform_rows(
          md, rows, variant,
          [&](uint64_t mm) { return mm == rows ? s_pre[0] : s_pre[(rows - mm) / tb]; }, nullptr,
          s_split);
    }
    s_m = (uint32_t)m;
    plan[0] = (uint32_t)m;
    plan[1] = rows - (uint32_t)m;
    st->a_rows = (uint32_t)m;
    st->form_rows = rows;
    uint32_t vstar = 0;
    if (m > 0 && m < rows) pre_of(m, &vstar);
    s_vstar = vstar;
    s_tstar = (m > 0 && m < rows) ? (uint32_t)(m - cum[vstar]) : 0u;
  }
  __syncthreads();
  const uint32_t m = s_m;
  if (m == 0 || m == rows) {
    for (uint32_t i = tid; i < rows; i += kChooseThreads) ridx[i] = i;
    return;
  }
  // split: a stable counting sort of the A rows, B rows in ascending order
  // (one warp walks the rows in order; cum[v] becomes the next slot of value v)
  if (wid != 0) return;
  const uint32_t vstar = s_vstar, tstar = s_tstar;
  uint32_t run_eq = 0, run_b = 0;
  for (uint32_t i0 = 0; i0 < rows; i0 += 32) {
    const uint32_t i = i0 + lane;
    const bool valid = i < rows;
    const uint32_t v = valid ? min(nnz_row[i], n) : 0u;
    const unsigned lt = (1u << lane) - 1u;
    const bool is_eq = valid && v == vstar;
    const unsigned eq_mask = __ballot_sync(FULL, is_eq);
    const uint32_t rank_eq = run_eq + __popc(eq_mask & lt);
    const bool is_a = valid && (v < vstar || (is_eq && rank_eq < tstar));
    const bool is_b = valid && !is_a;
    const unsigned b_mask = __ballot_sync(FULL, is_b);
    const uint32_t key = is_a ? v : (0x80000000u | lane);
    const unsigned peers = __match_any_sync(FULL, key);
    const uint32_t leader = __ffs(peers) - 1;
    uint32_t slot = 0;
    if (is_a && lane == leader) {
      slot = cum[v];
      cum[v] = slot + __popc(peers);
    }
    slot = __shfl_sync(FULL, slot, leader);
    if (is_a) ridx[slot + __popc(peers & lt)] = i;
    if (is_b) ridx[m + run_b + __popc(b_mask & lt)] = i;
    run_eq += __popc(eq_mask);
    run_b += __popc(b_mask);
    __syncwarp();
  }
}

// A-form lists: tasks t < ntask (or *dyn_ntask) compact slab row q = rows_idx[t]
// (or t) of X -> its nonzero bases (k, X[r0 + q, k]) in increasing k (the
// zero-base skip of kernels.hpp:121-125 done once); lists / counts are indexed
// by slab row.
template <class T>
__global__ void k_acompact(const T* __restrict__ x, uint64_t ld, uint32_t n, int vec, uint32_t r0,
                           uint32_t ntask, const uint32_t* __restrict__ dyn_ntask,
                           const uint32_t* __restrict__ rows_idx,
                           typename AEntry<T>::type* __restrict__ lists, uint64_t cap,
                           uint32_t* __restrict__ counts) {
  const uint32_t ntotal = ntask;
  if (dyn_ntask) ntask = *dyn_ntask;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  // the rows the choice left to the B-form: empty lists, so that the warps of
  // the last A-form CTA that fall on them add nothing (k_aform)
  if (rows_idx)
    for (uint64_t t = ntask + warp * 32 + lane; t < ntotal; t += nwarps * 32) counts[rows_idx[t]] = 0;
  for (uint64_t t = warp; t < ntask; t += nwarps) {
    const uint64_t q = rows_idx ? rows_idx[t] : t;  // slab row
    const T* row = x + (r0 + q) * ld;
    auto* out = lists + q * cap;
    uint32_t base = 0;
    for (uint32_t c1 = 0; c1 < n; c1 += 512) {  // 4 loads in flight per lane
      T vv[4][4];
#pragma unroll
      for (uint32_t u = 0; u < 4; ++u) load4(row, c1 + u * 128 + 4 * lane, n, vec != 0, vv[u]);
#pragma unroll
      for (uint32_t u = 0; u < 4; ++u) {
        const uint32_t j0 = c1 + u * 128 + 4 * lane;
        const T* v = vv[u];
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
    }
    if (lane == 0) counts[q] = base;
  }
}

// out[oc * ld_out + r] = in[ir * ld_in + c] for r < rows, c < cols, with
// ir = in_rows ? in_rows[r] : r and oc = out_rows ? out_rows[c] : c (the row
// maps gather / scatter the rows of a Case A split between the two kernels).
// plan (optional, the device-side choice): dyn = 1 -> rows = plan[1] and
// in_rows += plan[0]; dyn = 2 -> cols = plan[1] and out_rows += plan[0].
template <class T>
__global__ void k_transpose(const T* __restrict__ in, uint64_t ld_in, uint32_t rows,
                            uint32_t cols, T* __restrict__ out, uint64_t ld_out,
                            const uint32_t* __restrict__ in_rows,
                            const uint32_t* __restrict__ out_rows, const DevStatus* st,
                            const uint32_t* __restrict__ plan, int dyn) {
  // the result transpose writes Z only for a valid product (out untouched on
  // a validation error, like the kernels that write Z directly)
  if (st && status_failed(st)) return;
  if (dyn == 1) {
    rows = plan[1];
    in_rows += plan[0];
  } else if (dyn == 2) {
    cols = plan[1];
    out_rows += plan[0];
  }
  const uint32_t c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  if (c0 >= cols || r0 >= rows) return;
  __shared__ T tile[32][33];
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
      if (st) AFMM_CHECK(st, !out_rows || oc < (uint64_t)gridDim.x * 32 + (dyn == 2 ? plan[0] : 0));
      out[oc * ld_out + r] = tile[threadIdx.x][dy];
    }
  }
}

// Fast mode: combine the k-slice partial products in ascending slice order
// (deterministic; the reassociation the fast mode allows is exactly this
// regrouping of each element's k-sum). dyn_cols (optional): cols on the device.
template <class T>
__global__ void k_reduce_slices(const T* __restrict__ part, uint64_t stride, uint64_t ld_part,
                                uint32_t splits, uint32_t rows, uint32_t cols,
                                T* __restrict__ out, uint64_t ld_out, const DevStatus* st,
                                const uint32_t* __restrict__ dyn_cols) {
  if (status_failed(st)) return;
  if (dyn_cols) cols = *dyn_cols;
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
                       uint32_t l0, uint32_t l1, uint32_t q0, uint32_t q1, DevStatus* st,
                       uint32_t* nnz, unsigned long long* rsum, cudaStream_t s, int check_finite,
                       unsigned long long* fstats) {
  const int vec = vec_ok(lhs, ld) & vec_ok(rhs, ld);
  const uint64_t tasks = (uint64_t)(l1 - l0) + (q1 - q0);
  if (tasks == 0) return;
  k_scan_stats<T><<<grid_for_warps(tasks, 8), 256, 0, s>>>(
      lhs, rhs, ld, n, which_case, vec, check_finite, l0, l1, q0, q1, st, nnz, rsum, fstats,
      aform_tile_cols<T>());
  note_launch();
}

template <class T>
void launch_rows(const T* x, uint64_t ld, uint32_t n, int which_case, const uint32_t* nnz,
                 const unsigned long long* rsum, uint32_t a0, uint32_t a1, uint32_t r0,
                 uint32_t r1, int2* lists, uint64_t cap, uint32_t* counts,
                 unsigned long long* work, DevStatus* st, cudaStream_t s, uint32_t* nnz_row,
                 int group_allow) {
  if (a1 <= a0) return;
  k_rows<T><<<grid_for_warps(a1 - a0, 8), 256, 0, s>>>(x, ld, n, which_case, vec_ok(x, ld), nnz,
                                                        rsum, a0, a1, r0, r1, lists, cap, counts,
                                                        work, st, nnz_row, group_allow);
  note_launch();
}

template <class T>
void launch_group_idx(const T* rep, uint64_t ld, uint32_t n, int which_case, uint32_t r0,
                      uint32_t rows, uint16_t* gidx, uint64_t ldg, const DevStatus* st, int allow,
                      cudaStream_t s, const uint32_t* skip) {
  if (which_case == 1) {
    const uint32_t ngroups = (rows + kGroupRows - 1) / kGroupRows;
    if (ngroups == 0) return;
    k_group_idx_rows<T><<<grid_for_warps(ngroups, 8), 256, 0, s>>>(rep, ld, n, vec_ok(rep, ld), r0,
                                                                  rows, gidx, ldg, st, allow);
  } else {
    const uint32_t ngroups = (n + kGroupRows - 1) / kGroupRows;
    dim3 grid((ngroups + 31) / 32, (uint32_t)((ldg + 31) / 32));
    k_group_idx_cols<T><<<grid, 256, 0, s>>>(rep, ld, n, vec_ok(rep, ld), gidx, ldg, st, allow,
                                             skip);
  }
  note_launch();
}

template <class T>
void launch_counts_f16(const T* y, uint64_t ld, uint32_t n, uint32_t tile_cols, __half* cnt,
                       uint64_t ldc, uint16_t* rmax, unsigned long long* fstats, cudaStream_t s,
                       const uint32_t* need) {
  const uint32_t ntiles = (n + tile_cols - 1) / tile_cols;
  k_counts_f16<T><<<grid_for_warps((uint64_t)n * ntiles, 8), 256, 0, s>>>(
      y, ld, n, vec_ok(y, ld), tile_cols, ntiles, cnt, ldc, rmax, fstats, need);
  note_launch();
}

size_t choose_scratch_bytes(uint64_t n) { return (4 * (n + 2) + 2) * sizeof(uint32_t); }

cudaError_t launch_choose(const CaseAModel& md, uint32_t rows, int variant, const uint32_t* nnz_row,
                   const unsigned long long* fstats, uint32_t* scratch, uint32_t* plan,
                   uint32_t* ridx, DevStatus* st, cudaStream_t s) {
  // the static arrays (16.8 KB) count against the default 48 KB as well: set
  // the opt-in size for every dynamic size (a first call at n = 2100 -- 33.6
  // KB dynamic -- failed to launch before any call had raised the limit)
  const size_t smem = choose_smem_bytes(md.n);
  if (smem > 0) {
    const cudaError_t e =
        cudaFuncSetAttribute(k_choose, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k_choose<<<1, kChooseThreads, smem, s>>>(md, rows, variant, nnz_row, fstats, scratch, plan, ridx,
                                           st);
  note_launch();
  return cudaGetLastError();
}

template <class T>
void launch_acompact(const T* x, uint64_t ld, uint32_t n, uint32_t r0, uint32_t ntask,
                     const uint32_t* dyn_ntask, const uint32_t* rows_idx,
                     typename AEntry<T>::type* lists, uint64_t cap, uint32_t* counts,
                     cudaStream_t s) {
  if (ntask == 0) return;
  k_acompact<T><<<grid_for_warps(ntask, 8), 256, 0, s>>>(x, ld, n, vec_ok(x, ld), r0, ntask,
                                                         dyn_ntask, rows_idx, lists, cap, counts);
  note_launch();
}

template <class T>
void launch_transpose_compact(const T* y, uint64_t ld, uint32_t n, int2* lists, uint64_t cap,
                              uint32_t* counts, DevStatus* st, const uint32_t* skip,
                              cudaStream_t s, int group_allow) {
  k_transpose_compact<T><<<(n + 31) / 32, 256, 0, s>>>(y, ld, n, lists, cap, counts, st, skip,
                                                       group_allow);
  note_launch();
}

template <class T>
void launch_transpose(const T* in, uint64_t ld_in, uint32_t rows, uint32_t cols, T* out,
                      uint64_t ld_out, cudaStream_t s, const uint32_t* in_rows,
                      const uint32_t* out_rows, const DevStatus* st, const uint32_t* plan,
                      int dyn) {
  if (rows == 0 || cols == 0) return;
  dim3 grid((cols + 31) / 32, (rows + 31) / 32);
  k_transpose<T><<<grid, dim3(32, 8), 0, s>>>(in, ld_in, rows, cols, out, ld_out, in_rows,
                                               out_rows, st, plan, dyn);
  note_launch();
}

template <class T>
void launch_reduce_slices(const T* part, uint64_t stride, uint64_t ld_part, uint32_t splits,
                          uint32_t rows, uint32_t cols, T* out, uint64_t ld_out,
                          const DevStatus* st, const uint32_t* dyn_cols, cudaStream_t s) {
  uint64_t blocks = ((uint64_t)rows * cols + 255) / 256;
  if (blocks > 148ull * 16) blocks = 148ull * 16;
  if (blocks < 1) blocks = 1;
  k_reduce_slices<T><<<(unsigned)blocks, 256, 0, s>>>(part, stride, ld_part, splits, rows, cols,
                                                      out, ld_out, st, dyn_cols);
  note_launch();
}

#define INSTANTIATE(T)                                                                         \
  template void launch_scan_stats<T>(const T*, const T*, uint64_t, uint32_t, int, uint32_t,    \
                                     uint32_t, uint32_t, uint32_t, DevStatus*, uint32_t*,      \
                                     unsigned long long*, cudaStream_t, int,                   \
                                     unsigned long long*);                                     \
  template void launch_rows<T>(const T*, uint64_t, uint32_t, int, const uint32_t*,             \
                               const unsigned long long*, uint32_t, uint32_t, uint32_t,        \
                               uint32_t, int2*, uint64_t, uint32_t*, unsigned long long*,      \
                               DevStatus*, cudaStream_t, uint32_t*, int);                      \
  template void launch_group_idx<T>(const T*, uint64_t, uint32_t, int, uint32_t, uint32_t,     \
                                    uint16_t*, uint64_t, const DevStatus*, int, cudaStream_t,  \
                                    const uint32_t*);                                          \
  template void launch_counts_f16<T>(const T*, uint64_t, uint32_t, uint32_t, __half*, uint64_t, \
                                     uint16_t*, unsigned long long*, cudaStream_t,             \
                                     const uint32_t*);                                         \
  template void launch_acompact<T>(const T*, uint64_t, uint32_t, uint32_t, uint32_t,           \
                                   const uint32_t*, const uint32_t*,                           \
                                   typename AEntry<T>::type*, uint64_t, uint32_t*,             \
                                   cudaStream_t);                                              \
  template void launch_transpose_compact<T>(const T*, uint64_t, uint32_t, int2*, uint64_t,     \
                                            uint32_t*, DevStatus*, const uint32_t*,            \
                                            cudaStream_t, int);                                \
  template void launch_transpose<T>(const T*, uint64_t, uint32_t, uint32_t, T*, uint64_t,      \
                                    cudaStream_t, const uint32_t*, const uint32_t*,            \
                                    const DevStatus*, const uint32_t*, int);                   \
  template void launch_reduce_slices<T>(const T*, uint64_t, uint64_t, uint32_t, uint32_t,     \
                                        uint32_t, T*, uint64_t, const DevStatus*,             \
                                        const uint32_t*, cudaStream_t);

INSTANTIATE(float)
INSTANTIATE(double)

}  // namespace afmm_dev
