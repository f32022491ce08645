// common.cuh -- shared device helpers for the AFMM sm_100a kernels:
// mbarrier + TMA (cp.async.bulk.tensor) inline PTX, rep conversion, status.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace afmm_dev {

// Device-side status of one product call: first offenders, the exact counts,
// list overflow and the Case A form chosen on the device, all written by the
// prepass. Offenders are stored INVERTED (~key, reduced with atomicMax) so
// that an all-zero struct means "no error, zero counts" and one memset
// initialises everything.
struct DevStatus {
  unsigned long long nonfinite_lhs_inv;  // ~(linear index) of first non-finite lhs element
  unsigned long long nonfinite_rhs_inv;
  unsigned long long rep_bad_inv;        // ~((linear index << 2) | kind) of first bad rep
  // Longest rep list the product needs when it exceeds the list capacity (0 =
  // every list fits). Reps beyond an entry's range (|rep| > 2^31 - 1 in the
  // int2 lists, > 32767 in the quad lists) are split into consecutive entries
  // at the same k -- the element's |rep| sequential adds stay consecutive, so
  // the result is unchanged -- and such lists can outgrow the n-entry
  // capacity; the runtime then re-runs the product with this capacity.
  unsigned long long list_need;
  unsigned long long additions;
  unsigned long long zero_skips;
  uint32_t a_rows;     // Case A: slab rows the device-side choice gave the A-form
  uint32_t form_rows;  // Case A: slab rows seen by the choice (0: no choice made)
  unsigned long long rep_nan_inv;  // ~(linear index) of the first NaN rep (kernel semantics)
  // checked build (-DAFMM_CHECKED, `make checked`): bound-check violations
  // counted by the kernels (AFMM_CHECK); always 0 in the product build
  unsigned long long check_violations;
  // Rep statistics for the small-rep group kernel (k_bgroup): the largest
  // |rep| of the rep operand (saturated at 255) and whether any rep is
  // negative. Both are reduced over every shard of a multi-device call.
  uint32_t rep_max;
  uint32_t rep_neg;
  unsigned long long pad[6];
};
static_assert(sizeof(DevStatus) == 128, "DevStatus is a 128-byte record");

// Bound checks of the checked build (compute-sanitizer is not available on
// this pool): a violated condition is counted in the call's status (the
// runtime reports it as an error) instead of faulting the context.
#ifdef AFMM_CHECKED
#define AFMM_CHECK(st, cond)                                                              \
  do {                                                                                    \
    if (!(cond)) atomicAdd(const_cast<unsigned long long*>(&(st)->check_violations), 1ull); \
  } while (0)
#else
#define AFMM_CHECK(st, cond) \
  do {                       \
  } while (0)
#endif

// A-form list entry: (k, base) of a nonzero base X[i,k] (k_aform).
template <class T>
struct AEntry;
template <>
struct AEntry<float> {
  using type = int2;  // {k, float bits}
};
template <>
struct AEntry<double> {
  using type = int4;  // {k, 0, low word, high word}
};

// Validation failed or a list overflowed: the compute kernels do nothing.
__device__ __forceinline__ bool status_failed(const DevStatus* st) {
  return (st->nonfinite_lhs_inv | st->nonfinite_rhs_inv | st->rep_bad_inv | st->list_need |
          st->rep_nan_inv) != 0ull;
}

// Largest |rep| (and no negative rep) the group kernel takes: its jump tables
// cover reps 0..kGroupMaxRep (tools/gen_jumptable.py).
constexpr uint32_t kGroupMaxRep = 2;
constexpr int kGroupRows = 5;  // B-form rows per group (one warp)

// The product runs the small-rep group kernel (k_bgroup) instead of k_bform:
// decided on the device from the validated rep statistics, so the choice needs
// no host round trip. `allow` is the host's half (fp32, order-preserving mode,
// no forced k_bform shape).
// (`allow` carries the host's half of two device-side decisions as bits.)
constexpr int kAllowGroup = 1;  // the small-rep group kernel may run
constexpr int kAllowPack = 2;   // the rep lists may be written as packed 4-byte entries
__device__ __forceinline__ bool group_mode(const DevStatus* st, int allow) {
  return (allow & kAllowGroup) && st->rep_max <= kGroupMaxRep && st->rep_neg == 0;
}

// Packed rep lists: when every |rep| of the validated rep operand is <=
// kPackMaxRep (rep_max saturates at 255) a list entry is one 32-bit word
// (k << 8) | (rep & 0xff) instead of an int2 {k, rep} -- the lists are re-read
// once per column tile, so they are most of the repeated-addition kernel's
// DRAM traffic (cfg5: 31 of 40 GB per launch). Decided on the device like
// group_mode; the host's half (kAllowPack) requires k < 2^24, the
// order-preserving mode and a problem large enough to matter.
constexpr uint32_t kPackMaxRep = 127;
__device__ __forceinline__ bool packed_mode(const DevStatus* st, int allow) {
  return (allow & kAllowPack) && st->rep_max <= kPackMaxRep;
}
__device__ __forceinline__ uint32_t pack_entry(uint32_t k, long long rep) {
  return (k << 8) | ((uint32_t)(int)rep & 0xffu);
}
__device__ __forceinline__ int2 unpack_entry(uint32_t e) {
  return make_int2((int)(e >> 8), (int)(e << 24) >> 24);
}

// kernels.hpp:31-40 on the widened value: 0 ok, 1 not integer-valued,
// 2 exceeds the exact integer range. round() is std::round (half away from
// zero). NaN passes both tests exactly as in the reference; non-finite
// elements are rejected separately (the DenseMatrix ctor, matrix.hpp:31-35).
__device__ __forceinline__ int rep_kind(double v) {
  if (fabs(v - round(v)) > 1e-9) return 1;
  if (fabs(v) > 9007199254740992.0) return 2;
  return 0;
}

// Lane index that the compiler cannot rematerialise (an asm volatile result
// stays in its register instead of being re-read from SR_TID in hot loops).
__device__ __forceinline__ uint32_t lane_id() {
  uint32_t l;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(l));
  return l;
}

// Make a value opaque to the compiler so it stays in a register instead of
// being re-derived (S2UR SR_CTAID / SR_CgaCtaId + address math) in hot loops.
__device__ __forceinline__ uint32_t pin(uint32_t v) {
  asm volatile("" : "+r"(v));
  return v;
}

// ---- mbarrier --------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\t"
      "mbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\t"
      "mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// Same operations on a precomputed shared-memory address.
__device__ __forceinline__ void mbar_arrive_at(uint32_t addr) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\t"
      "mbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(addr)
      : "memory");
}

__device__ __forceinline__ void mbar_wait_at(uint32_t addr, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
  }
}

// Blocking wait that suspends the warp in hardware until the phase completes
// (or SUSPEND_NS elapse) instead of re-polling: a polling try_wait returns
// after a short system time limit and the retry loop costs issue slots that
// the FP-bound warps on the same SM sub-partition need (ncu source view: the
// producer's empty-barrier loop was 11% of all issued instructions).
constexpr uint32_t SUSPEND_NS = 1000000;

__device__ __forceinline__ void mbar_sleep_wait_at(uint32_t addr, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity), "n"(SUSPEND_NS)
        : "memory");
  }
}

// Non-blocking probe: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// ---- TMA -------------------------------------------------------------------

// 2D tiled tensor load global -> shared, completion via mbarrier tx bytes.
// c0 = innermost (column) coordinate, c1 = row coordinate, in elements.
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map,
                                            uint64_t* bar, int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void prefetch_tensormap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

}  // namespace afmm_dev
