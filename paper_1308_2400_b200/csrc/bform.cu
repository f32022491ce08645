// bform.cu -- the repeated-addition kernels (sm_100a, CUDA cores only).
//
// Computes Z' = R' (x) B' in the reference's order-preserving form: for every
// output element, the terms arrive in increasing k and each is |rep|
// sequential `acc += step` (kernels.hpp:95-104, :148-163). "B-form" means the
// rep is uniform along an output row, which is Case B verbatim
// (kernels.hpp:142-165: rep = X[i,k], bases Y[k,:]); Case A is run through the
// same kernel on transposed operands (afmm_case_a(X,Y) = afmm_case_b(Y^T,X^T)^T,
// same per-element add sequence). "A-form" (k_aform, below) is
// Case A in its own orientation, base uniform per warp, for sparse X.
//
// Contents: k_bform (the product kernel, three tile shapes), k_bform_tm
// (opt-in TMEM-fed variant), k_aform (A-form), k_bform_mr (opt-in dense-rep
// multi-row variant), and their launchers.
//
// k_bform (one CTA = CW consumer warps, each owning one output row, + 1 TMA
// producer warp):
//   * CTA tile = CW output rows x TILE_N output columns; each lane holds
//     8*G fp32 / 4*G fp64 columns in registers for the whole k sweep
//     (register-resident Z tile).
//   * KB x TILE_N tiles of the base matrix B' stream through a STAGES-deep
//     smem ring with cp.async.bulk.tensor (TMA) + mbarriers; the tile is
//     shared by all CW rows of the CTA (CW-fold reuse from smem).
//   * Each warp walks its row's compacted (k, rep) list (built by the
//     prepass, zero reps already skipped), waits for the stage holding row k,
//     loads its bases with conflict-free 128-bit LDS and runs the
//     warp-uniform rep loop: |rep| x 4G FADD2 (fp32) or |rep| x 4G DADD
//     (fp64). The rep is uniform across the warp, so there is no divergence;
//     zero bases are added as +0/-0, which is bit-neutral (the accumulator is
//     never -0) and never counted.
//   * Warps release a stage by arriving on its empty barrier; they may drift
//     up to STAGES blocks apart.
//
// Issue-slot budget: FADD2 and DADD occupy their pipe for 2 cycles per warp
// instruction, so one non-FP instruction per FP instruction issues for free.
// The entry path uses ALU/LSU instructions (SHF/LOP3, LDS, a uniform LDG) and
// the rep loop has no predicated FP tail (a predicated-off FADD2 still
// occupies the pipe). The next entry's (k, rep) load is issued before the
// current rep loop so its latency is hidden. Wider tiles (G = 8: 1024 fp32
// columns, 32 accumulators per lane) amortise the per-entry overhead over
// twice the adds, which matters for small reps (tools/sweep.py).
#include "common.cuh"
#include "kernels.h"

namespace afmm_dev {

namespace {

constexpr unsigned FULL = 0xffffffffu;

#ifndef AFMM_EXP_KB
constexpr int KB = 8;  // k rows per stage
#else
constexpr int KB = AFMM_EXP_KB;  // timing experiments (Makefile exp-%)
#endif
#ifndef AFMM_EXP_REP_UNROLL
// rep loop: trips of 8 steps, then the remainder (< 8) by its binary digits
// (4, 2, 1 steps) with no loop. Measured against 4-step trips + a 1-step
// remainder loop: cfg5 1845 -> 1809 ms, rep 16 0.901 -> 0.912 of peak, and 88
// registers instead of 96 + an 8-byte spill (ptxas); the loop counter and
// back-edge instructions it removes issue on the FMA pipe (VIADD) or stall on
// branch resolution.
constexpr int REP_UNROLL = 8;  // rep-loop unroll (adds per column per trip)
#else
constexpr int REP_UNROLL = AFMM_EXP_REP_UNROLL;
#endif
#ifndef AFMM_EXP_REP_BIN
constexpr bool REP_BIN = true;  // remainder by binary digits instead of a loop
#else
constexpr bool REP_BIN = AFMM_EXP_REP_BIN != 0;
#endif
static_assert(!REP_BIN || (REP_UNROLL & (REP_UNROLL - 1)) == 0,
              "a binary remainder needs a power-of-two unroll");
#ifndef AFMM_EXP_WIDE_STAGES
#define AFMM_EXP_WIDE_STAGES 6
#endif
#ifndef AFMM_EXP_WIDE_MINB
#define AFMM_EXP_WIDE_MINB kWideCtasPerSm
#endif
#ifndef AFMM_EXP_WIDE_G
#define AFMM_EXP_WIDE_G 8
#endif
#ifndef AFMM_EXP_WIDE_CW
#define AFMM_EXP_WIDE_CW kWideRows
#endif
// Producer-less ring (experiment): no TMA warp; the consumer warp that
// releases a stage last refills it (smem counter per slot), so 16 consumer
// warps per SM get the 128-register budget of 16 warps.
#ifndef AFMM_EXP_NOPROD
#define AFMM_EXP_NOPROD 0
#endif
constexpr bool kNoProd = AFMM_EXP_NOPROD != 0;
constexpr uint32_t kListPrefetch = 64;  // list entries ahead prefetched into L1
constexpr int kProdWarps = kNoProd ? 0 : 1;

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// A TMA box is at most 256 elements wide, so a stage is G/2 boxes of
// KB x BOX_BYTES laid out box-major: [box][k row][BOX_BYTES].
constexpr int BOX_BYTES = 1024;

// smem byte offset of 128-bit group g of a k row, relative to the row's address
// in box 0 (each 1 KB box row holds two warp-wide 512-byte groups).
__device__ __forceinline__ constexpr uint32_t group_off(int g) {
  return (uint32_t)((g >> 1) * KB * BOX_BYTES + (g & 1) * 512);
}

template <class T, int G>
struct Geo {
  static constexpr int ROW_BYTES = G * 512;                // one k row of the CTA tile
  static constexpr int STAGE_BYTES = KB * ROW_BYTES;
  static constexpr int TILE_N = ROW_BYTES / sizeof(T);     // columns per CTA
  static constexpr int BOX_N = BOX_BYTES / sizeof(T);      // columns per TMA box
  static constexpr int NBOX = ROW_BYTES / BOX_BYTES;
};

__device__ __forceinline__ float4 lds128f(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}

__device__ __forceinline__ double2 lds128d(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

// Lane l owns, for g = 0..G-1, the 16-byte column group at byte
// (g>>1)*KB*BOX_BYTES + (g&1)*512 + l*16 of each staged k row: every 128-bit
// LDS across the warp reads 512 contiguous bytes (no bank conflict). In
// output columns that is tile_col + g*128 + 4l (fp32) / g*64 + 2l (fp64).
// ---- tensor memory (TMEM) ---------------------------------------------------

// 32 lanes x 32 columns of 32-bit words -> 32 registers per thread (lane t of
// the warp's TMEM lane quadrant, 32 consecutive columns), then wait.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}

__device__ __forceinline__ void tmem_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// smem -> TMEM copy of a 32-row x 16-byte matrix, replicated into all four
// 32-lane quadrants (row r -> lane r of every quadrant, 4 columns).
__device__ __forceinline__ void tmem_cp_32x128b_x4(uint32_t taddr, uint64_t desc) {
  asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(taddr), "l"(desc)
               : "memory");
}

// Arrive on an mbarrier once all previously issued tcgen05 async operations of
// this thread (here: the copies) have completed.
__device__ __forceinline__ void tmem_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}

// tcgen05 shared-memory matrix descriptor, no swizzle: 8-row x 16-byte core
// matrices stored contiguously (128 B apart), version 1 (sm_100).
__device__ __forceinline__ uint64_t smem_desc_128(uint32_t saddr) {
  const uint64_t start = (saddr >> 4) & 0x3fffu;
  const uint64_t lbo = 128u >> 4, sbo = 128u >> 4;
  return start | (lbo << 16) | (sbo << 32) | (1ull << 46);
}

template <class T, int G>
struct Acc;

template <int G>
struct Acc<float, G> {
  struct Bases {
    float2 b[2 * G];
  };
  float2 a[2 * G];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int c = 0; c < 2 * G; ++c) a[c] = make_float2(0.f, 0.f);
  }
  __device__ __forceinline__ static Bases load_bases(uint32_t row_addr) {
    Bases s;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float4 v = lds128f(row_addr + group_off(g));
      s.b[2 * g] = make_float2(v.x, v.y);
      s.b[2 * g + 1] = make_float2(v.z, v.w);
    }
    return s;
  }
  // t sequential `acc += step` per column; NEG: step = -base (kernels.hpp:97),
  // applied as the FADD2 operand-negate modifier (exact), so the shared bases
  // are never copied or rewritten.
  template <bool NEG>
  __device__ __forceinline__ void add_n(const Bases& s, uint32_t t) {
#pragma unroll 1
    while (t >= 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int c = 0; c < 2 * G; ++c)
          a[c] = __fadd2_rn(a[c], NEG ? make_float2(-s.b[c].x, -s.b[c].y) : s.b[c]);
      t -= 4;
    }
#pragma unroll 1
    while (t != 0) {
#pragma unroll
      for (int c = 0; c < 2 * G; ++c)
        a[c] = __fadd2_rn(a[c], NEG ? make_float2(-s.b[c].x, -s.b[c].y) : s.b[c]);
      t -= 1;
    }
  }
  // |rep| sequential `acc += step` per column, step = rep >= 0 ? base : -base
  // (kernels.hpp:95-104).
  __device__ __forceinline__ void add(const Bases& s, int rep) {
    if (rep >= 0) add_n<false>(s, (uint32_t)rep);
    else add_n<true>(s, 0u - (uint32_t)rep);
  }
  // The same on column groups [G0, G1) only, with just those bases live.
  template <bool NEG, int G0, int G1>
  __device__ __forceinline__ void add_range(const float2* b, uint32_t t) {
#pragma unroll 1
    while (t >= REP_UNROLL) {
#pragma unroll
      for (int u = 0; u < REP_UNROLL; ++u)
#pragma unroll
        for (int c = 2 * G0; c < 2 * G1; ++c)
          a[c] = __fadd2_rn(a[c], NEG ? make_float2(-b[c - 2 * G0].x, -b[c - 2 * G0].y)
                                      : b[c - 2 * G0]);
      t -= REP_UNROLL;
    }
    if (REP_BIN) {  // remainder t < REP_UNROLL by its binary digits, no loop
#pragma unroll
      for (int bit = REP_UNROLL / 2; bit >= 1; bit >>= 1)
        if (t & (uint32_t)bit) {
#pragma unroll
          for (int u = 0; u < bit; ++u)
#pragma unroll
            for (int c = 2 * G0; c < 2 * G1; ++c)
              a[c] = __fadd2_rn(a[c], NEG ? make_float2(-b[c - 2 * G0].x, -b[c - 2 * G0].y)
                                          : b[c - 2 * G0]);
        }
      return;
    }
#pragma unroll 1
    while (t != 0) {
#pragma unroll
      for (int c = 2 * G0; c < 2 * G1; ++c)
        a[c] = __fadd2_rn(a[c], NEG ? make_float2(-b[c - 2 * G0].x, -b[c - 2 * G0].y)
                                    : b[c - 2 * G0]);
      t -= 1;
    }
  }
  template <int G0, int G1>
  __device__ __forceinline__ void run_range(uint32_t row_addr, int rep) {
    float2 b[2 * (G1 - G0)];
#pragma unroll
    for (int g = G0; g < G1; ++g) {
      const float4 v = lds128f(row_addr + group_off(g));
      b[2 * (g - G0)] = make_float2(v.x, v.y);
      b[2 * (g - G0) + 1] = make_float2(v.z, v.w);
    }
    if (rep >= 0) add_range<false, G0, G1>(b, (uint32_t)rep);
    else add_range<true, G0, G1>(b, 0u - (uint32_t)rep);
  }
  // One list entry, all G column groups in one rep loop. (Splitting wide tiles
  // into two half-width loops to save 16 base registers was measured 3% slower.)
  __device__ __forceinline__ void run(uint32_t row_addr, int rep) { run_range<0, G>(row_addr, rep); }
  // The same entry with the bases read from tensor memory (k_bform_tm): the
  // lane's 4G words sit in 4G consecutive TMEM columns in LDS order.
  __device__ __forceinline__ void run_tm(uint32_t taddr, int rep) {
    static_assert(G == 8, "TMEM bases: 32 columns per lane");
    uint32_t r[32];
    tmem_ld32(taddr, r);
    float2 b[2 * G];
#pragma unroll
    for (int c = 0; c < 2 * G; ++c)
      b[c] = make_float2(__uint_as_float(r[2 * c]), __uint_as_float(r[2 * c + 1]));
    if (rep >= 0) add_range<false, 0, G>(b, (uint32_t)rep);
    else add_range<true, 0, G>(b, 0u - (uint32_t)rep);
  }
  __device__ __forceinline__ void store(float* out_row, int32_t oc0, int32_t ncols, uint32_t lane,
                                        bool vec_ok) const {
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

template <int G>
struct Acc<double, G> {
  double a[2 * G];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int c = 0; c < 2 * G; ++c) a[c] = 0.0;
  }
  struct Bases {
    double b[2 * G];
  };
  __device__ __forceinline__ static Bases load_bases(uint32_t row_addr) {
    Bases s;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const double2 v = lds128d(row_addr + group_off(g));
      s.b[2 * g] = v.x;
      s.b[2 * g + 1] = v.y;
    }
    return s;
  }
  template <bool NEG>
  __device__ __forceinline__ void add_n(const Bases& s, uint32_t t) {
#pragma unroll 1
    while (t >= 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int c = 0; c < 2 * G; ++c) a[c] = __dadd_rn(a[c], NEG ? -s.b[c] : s.b[c]);
      t -= 4;
    }
#pragma unroll 1
    while (t != 0) {
#pragma unroll
      for (int c = 0; c < 2 * G; ++c) a[c] = __dadd_rn(a[c], NEG ? -s.b[c] : s.b[c]);
      t -= 1;
    }
  }
  __device__ __forceinline__ void add(const Bases& s, int rep) {
    if (rep >= 0) add_n<false>(s, (uint32_t)rep);
    else add_n<true>(s, 0u - (uint32_t)rep);
  }
  template <bool NEG, int G0, int G1>
  __device__ __forceinline__ void add_range(const double* b, uint32_t t) {
#pragma unroll 1
    while (t >= REP_UNROLL) {
#pragma unroll
      for (int u = 0; u < REP_UNROLL; ++u)
#pragma unroll
        for (int c = 2 * G0; c < 2 * G1; ++c)
          a[c] = __dadd_rn(a[c], NEG ? -b[c - 2 * G0] : b[c - 2 * G0]);
      t -= REP_UNROLL;
    }
    if (REP_BIN) {
#pragma unroll
      for (int bit = REP_UNROLL / 2; bit >= 1; bit >>= 1)
        if (t & (uint32_t)bit) {
#pragma unroll
          for (int u = 0; u < bit; ++u)
#pragma unroll
            for (int c = 2 * G0; c < 2 * G1; ++c)
              a[c] = __dadd_rn(a[c], NEG ? -b[c - 2 * G0] : b[c - 2 * G0]);
        }
      return;
    }
#pragma unroll 1
    while (t != 0) {
#pragma unroll
      for (int c = 2 * G0; c < 2 * G1; ++c)
        a[c] = __dadd_rn(a[c], NEG ? -b[c - 2 * G0] : b[c - 2 * G0]);
      t -= 1;
    }
  }
  template <int G0, int G1>
  __device__ __forceinline__ void run_range(uint32_t row_addr, int rep) {
    double b[2 * (G1 - G0)];
#pragma unroll
    for (int g = G0; g < G1; ++g) {
      const double2 v = lds128d(row_addr + group_off(g));
      b[2 * (g - G0)] = v.x;
      b[2 * (g - G0) + 1] = v.y;
    }
    if (rep >= 0) add_range<false, G0, G1>(b, (uint32_t)rep);
    else add_range<true, G0, G1>(b, 0u - (uint32_t)rep);
  }
  __device__ __forceinline__ void run(uint32_t row_addr, int rep) { run_range<0, G>(row_addr, rep); }
  __device__ __forceinline__ void run_tm(uint32_t taddr, int rep) {
    static_assert(G == 8, "TMEM bases: 32 columns per lane");
    uint32_t r[32];
    tmem_ld32(taddr, r);
    double b[2 * G];
#pragma unroll
    for (int c = 0; c < 2 * G; ++c)
      b[c] = __hiloint2double((int)r[2 * c + 1], (int)r[2 * c]);
    if (rep >= 0) add_range<false, 0, G>(b, (uint32_t)rep);
    else add_range<true, 0, G>(b, 0u - (uint32_t)rep);
  }
  __device__ __forceinline__ void store(double* out_row, int32_t oc0, int32_t ncols,
                                        uint32_t lane, bool vec_ok) const {
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

// Rows per CTA (<= cw) that minimise (waves x rows per CTA), i.e. the busiest
// SM's share of rows when every SM holds `per_sm` CTAs: a last wave that is
// mostly empty costs as much as a full one (n = 1024 fp64, 16-row CTAs, 4
// column tiles: 256 CTAs on 296 slots; 14-row CTAs fill exactly one wave).
// Keeps cw unless trimming gains more than 3%.
inline uint32_t balanced_rows(uint32_t nrows, uint32_t tiles, uint32_t cw, uint32_t per_sm) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);  // per call: contexts may drive GPUs of different sizes
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      sms <= 0) {
    cudaGetLastError();
    sms = 148;
  }
  const uint64_t slots = (uint64_t)sms * per_sm;
  auto cost = [&](uint32_t r) {
    const uint64_t ctas = (uint64_t)((nrows + r - 1) / r) * tiles;
    return ((ctas + slots - 1) / slots) * (uint64_t)r;
  };
  uint32_t best = cw;
  uint64_t best_cost = cost(cw);
  for (uint32_t r = cw - 1; r >= 1 && 2 * r >= cw; --r) {
    const uint64_t c = cost(r);
    if (c * 100 < best_cost * 97) {
      best = r;
      best_cost = c;
    }
  }
  return best;
}

template <class T, int G, int STAGES>
__host__ __device__ constexpr size_t ring_smem_bytes() {
  return 128 /*alignment slack*/ + (size_t)STAGES * Geo<T, G>::STAGE_BYTES +
         2 * STAGES * sizeof(uint64_t);
}

// TMA issue logic of the producer warp (lane 0). pump() issues, without
// blocking, every load whose ring slot has been released by all consumers:
// the i-th block of the slice (k block kb_lo + i) goes to slot i % STAGES
// once the block STAGES earlier is released. The producer alternates pump()
// with a suspending wait on the next slot's empty barrier. (An in-consumer
// variant that let warp 0 pump between its own entries was measured 2-3x
// slower: the pumping warp becomes the ring's slowest consumer.)
template <class T, int G, int STAGES>
struct Pump {
  using Gm = Geo<T, G>;
  const CUtensorMap* tmap;
  const CUtensorMap* rmap;  // optional dense-rep map (k_bform_mr)
  unsigned char* ring;
  unsigned char* rring;
  uint64_t* full;
  uint64_t* empty;
  int32_t col;
  int32_t rrow;
  uint32_t nkb;
  uint32_t kb_lo;
  uint32_t rep_stage_bytes;
  uint32_t next;
  __device__ __forceinline__ void pump() {
    while (next < nkb) {
      const uint32_t slot = next % STAGES;
      if (next >= STAGES && !mbar_test_wait(&empty[slot], ((next / STAGES) - 1) & 1)) return;
      mbar_arrive_expect_tx(&full[slot], (uint32_t)Gm::STAGE_BYTES + rep_stage_bytes);
      const int32_t krow = (int32_t)((kb_lo + next) * KB);
#pragma unroll
      for (int h = 0; h < Gm::NBOX; ++h)
        tma_load_2d(ring + slot * Gm::STAGE_BYTES + h * KB * BOX_BYTES, tmap, &full[slot],
                    col + h * Gm::BOX_N, krow);
      if (rmap) tma_load_2d(rring + slot * rep_stage_bytes, rmap, &full[slot], rrow, krow);
      ++next;
    }
  }
};

// First list index with k >= key (lists are sorted by k); every lane computes
// the same answer from broadcast loads.
__device__ __forceinline__ uint32_t lower_bound_k(const int2* lst, uint32_t cnt, uint32_t key) {
  uint32_t lo = 0, hi = cnt;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if ((uint32_t)lst[mid].x < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// lists: row b's entries at lists[b * cap .. b * cap + counts[b]) in increasing k.
// Output row b, column (col0 + c) -> out[b * ld_out + c], c < ncols.
// k slice: blockIdx.z selects slice z = [z*slice_blocks, (z+1)*slice_blocks)
// of the nkb_total k blocks and writes to out + z * slice_stride (fast-mode
// split-k; one slice = the whole k range in order-preserving mode).
template <class T, int G, int CW, int STAGES, int MINB, bool SPLIT>
__global__ void __launch_bounds__((CW + kProdWarps) * 32, MINB)
    k_bform(const __grid_constant__ CUtensorMap tmap, const int2* __restrict__ lists,
            uint64_t cap, const uint32_t* __restrict__ counts, uint32_t nrows, uint32_t rpc,
            int32_t col0, int32_t ncols, uint32_t nkb_total, uint32_t slice_blocks, uint64_t slice_stride,
            T* __restrict__ out, uint64_t ld_out, int vec_ok, const DevStatus* __restrict__ st) {
  using Gm = Geo<T, G>;
  extern __shared__ unsigned char smem_raw[];
  // 128-byte aligned ring (TMA destination without swizzle); pointer arithmetic
  // on the smem pointer itself keeps the shared address space visible to the
  // compiler.
  unsigned char* base = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + STAGES * Gm::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  const uint32_t ring = smem_u32(base);

  if (status_failed(st)) return;  // validation failed: compute nothing (kernels.hpp:115,144)

  // %laneid through asm volatile: under register pressure ptxas otherwise
  // re-derives the lane from S2R SR_TID inside the entry loop (a ~30-cycle
  // stall per entry, ncu source view at rep 1).
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  const int32_t tile_c = blockIdx.y * Gm::TILE_N;  // relative to col0
  // SPLIT = false (order-preserving mode): one slice, k_lo = 0 at compile time
  // (a runtime k_lo was rematerialised from S2UR SR_CTAID.Z + LDC every entry).
  const uint32_t kb_lo = SPLIT ? blockIdx.z * slice_blocks : 0u;
  const uint32_t kb_hi = min(nkb_total, kb_lo + slice_blocks);
  const uint32_t nkb = kb_hi - kb_lo;
  if (SPLIT) out += blockIdx.z * slice_stride;

  // refill of ring slot `sl` with block `blk` of the slice (one thread)
  auto refill = [&](uint32_t sl, uint32_t blk) {
    mbar_arrive_expect_tx(&full[sl], (uint32_t)Gm::STAGE_BYTES);
    const int32_t krow = (int32_t)((kb_lo + blk) * KB);
#pragma unroll
    for (int h = 0; h < Gm::NBOX; ++h)
      tma_load_2d(base + sl * Gm::STAGE_BYTES + h * KB * BOX_BYTES, &tmap, &full[sl],
                  col0 + tile_c + h * Gm::BOX_N, krow);
  };
  uint32_t* released = reinterpret_cast<uint32_t*>(empty);  // kNoProd: arrivals per slot
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      if (kNoProd) released[s] = 0;
      else mbar_init(&empty[s], CW);
    }
    fence_barrier_init();
    if (kNoProd)
      for (uint32_t s = 0; s < (uint32_t)STAGES && s < nkb; ++s) refill(s, s);
  }
  __syncthreads();

  if (!kNoProd && warp == CW) {
    // ---- dedicated TMA producer warp ----
    // (Unlike k_bform_mr, the list-walking warps progress unevenly; an
    // in-warp pump makes warp 0 the ring's bottleneck: measured 2-3x slower.)
    if (lane == 0) {
      Pump<T, G, STAGES> pump{&tmap, nullptr, base, nullptr, full, empty, col0 + tile_c, 0,
                              nkb, kb_lo, 0, 0};
      prefetch_tensormap(&tmap);
      while (true) {
        pump.pump();
        if (pump.next >= nkb) break;
        mbar_sleep_wait_at(smem_u32(&empty[pump.next % STAGES]), ((pump.next / STAGES) - 1) & 1);
      }
    }
    return;
  }

  // ---- consumers: one output row per warp ----
  // rpc <= CW rows per CTA (the launcher trims it to balance the last wave);
  // warps past it walk no entries but still release every stage.
  const uint32_t b = warp < rpc ? blockIdx.x * rpc + warp : nrows;
  uint32_t cnt = b < nrows ? counts[b] : 0u;
  const int2* lst = lists + (uint64_t)(b < nrows ? b : 0) * cap;
  if (SPLIT) {
    // this slice's entries: [lower_bound(kb_lo*KB), lower_bound(kb_hi*KB))
    const uint32_t p0 = lower_bound_k(lst, cnt, kb_lo * KB);
    const uint32_t p1 = kb_hi == nkb_total ? cnt : lower_bound_k(lst, cnt, kb_hi * KB);
    lst += p0;
    cnt = p1 - p0;
  }

  Acc<T, G> acc;
  acc.zero();
  const uint32_t k_lo = kb_lo * KB;
  const uint32_t full0 = smem_u32(full), empty0 = smem_u32(empty);

  // (kb_cur, slot, phase): the k block currently held, its ring slot and the
  // parity of that slot's current fill; stage_addr = smem address of the slot
  // plus this lane's first 16-byte column group.
  uint32_t kb_cur = 0, slot = 0, phase = 0;
  uint32_t stage_addr = ring + lane * 16;
  auto advance = [&]() {
    __syncwarp();
    if (lane == 0) {
      if (kNoProd) {
        // the last of the CW warps to release this use of the slot refills it
        const uint32_t old = atomicAdd(&released[slot], 1u);
        if (old % CW == CW - 1 && kb_cur + STAGES < nkb) {
          fence_proxy_async_smem();  // order the warps' smem reads before the TMA write
          refill(slot, kb_cur + STAGES);
        }
      } else {
        mbar_arrive_at(empty0 + slot * 8);
      }
    }
    ++kb_cur;
    stage_addr += Gm::STAGE_BYTES;
    if (++slot == STAGES) {
      slot = 0;
      phase ^= 1;
      stage_addr -= STAGES * Gm::STAGE_BYTES;
    }
  };
  mbar_sleep_wait_at(full0, 0);
  // Entry e + 1 = (k, rep) is read by a warp-uniform load (L1 broadcast)
  // while entry e runs, and the list line 64 entries ahead is prefetched into
  // L1. (Measured against one coalesced 32-entry load per chunk + SHFL
  // broadcasts: equal at cfg5, cfg3 mu = 4 +2.6%, cfg4 +1%, rep 1 -2%; fewer
  // instructions and branches per entry.)
  const int2* __restrict__ lp = lst;
  const int2 e0 = cnt ? __ldg(lp) : make_int2(0, 0);
  uint32_t k = (uint32_t)e0.x;
  int rep = e0.y;
  for (uint32_t e = 0; e < cnt; ++e) {
    const uint32_t f = e + 1;
    const int2 ne = f < cnt ? __ldg(lp + f) : make_int2(0, 0);
    if (f + kListPrefetch < cnt)
      asm volatile("prefetch.global.L1 [%0];" ::"l"(lp + f + kListPrefetch));
    const uint32_t kb = (k - k_lo) / KB;  // block index within the slice
    while (kb_cur < kb) {
      advance();
      mbar_sleep_wait_at(full0 + slot * 8, phase);
    }
    acc.run(stage_addr + (k % KB) * BOX_BYTES, rep);
    k = (uint32_t)ne.x;
    rep = ne.y;
  }
  // release the remaining stages in order
  while (true) {
    advance();
    if (kb_cur >= nkb) break;
    mbar_sleep_wait_at(full0 + slot * 8, phase);
  }

  if (b < nrows) acc.store(out + (uint64_t)b * ld_out, tile_c, ncols, lane, vec_ok != 0);
}

// ---------------------------------------------------------------------------
// k_bform_tm: k_bform with the bases served from tensor memory.
//
// At small reps k_bform is bound by the shared-memory data pipe (ncu at rep 1:
// L1TEX wavefronts 97%, FMA pipe 28%): each of the CTA's warps re-reads every
// staged base row with 128-bit LDS at 128 B/clk/SM. TMEM reads into registers
// run at >= 450 B/clk/SM (tools/tmem_probe.cu), so here
//   * warp CW (TMA) streams KB x 1024-byte-row tiles of B' into an SST-deep
//     smem ring (as in k_bform);
//   * warp CW+1 (copy) moves each landed tile into one of TST TMEM stages with
//     tcgen05.cp 32x128b.warpx4 (each 512-byte column group -> 4 columns of all
//     128 lanes, i.e. one copy per lane quadrant), then tcgen05.commit arrives on
//     the stage's full barrier and on the smem slot's empty barrier;
//   * the CW consumer warps walk their rows' lists as in k_bform but fetch an
//     entry's 32 bases per lane with one tcgen05.ld 32x32b.x32 from their lane
//     quadrant, releasing TMEM stages through per-stage empty barriers.
// CW = 14 consumers + 2 producers (4 warps per SM sub-partition, 128-register
// budget), one CTA per SM owning all 512 TMEM columns: TM_TST = 4 stages of
// TM_TKB = 4 k rows x 32 columns. Per element the order is unchanged (one
// chain, k ascending, |rep| adds).
//
// Measured (tools/exp_time.py): equal to k_bform at rep >= 4 and slower at
// rep 1-2 (0.20 vs 0.23 of peak): the replicating copy (one 32x128b.warpx4
// per 512 bytes) cannot refill TMEM as fast as 14 warps drain it, so the
// consumers wait on the stage-full barrier (ncu: 32% of warp samples). Kept
// as an opt-in variant (AFMM_BFORM=tmem) with full parity coverage.
// ---------------------------------------------------------------------------

constexpr int TM_TKB = 4;           // k rows per TMEM stage (half an smem stage)
constexpr int TM_TST = 4;           // TMEM stages
constexpr int TM_COLS = 512;        // TMEM columns allocated (whole SM)
constexpr int TM_STAGE_COLS = TM_TKB * 32;
static_assert(KB % TM_TKB == 0, "TMEM stage must divide the smem stage");

template <class T, int CW, int SST>
__host__ __device__ constexpr size_t tm_smem_bytes() {
  return 128 + (size_t)SST * Geo<T, 8>::STAGE_BYTES +
         (2 * SST + 2 * TM_TST) * sizeof(uint64_t) + 16;
}

template <class T, int CW, int SST, bool SPLIT>
__global__ void __launch_bounds__((CW + 2) * 32, 1)
    k_bform_tm(const __grid_constant__ CUtensorMap tmap, const int2* __restrict__ lists,
               uint64_t cap, const uint32_t* __restrict__ counts, uint32_t nrows, uint32_t rpc,
               int32_t col0, int32_t ncols, uint32_t nkb_total, uint32_t slice_blocks, uint64_t slice_stride,
               T* __restrict__ out, uint64_t ld_out, int vec_ok,
               const DevStatus* __restrict__ st) {
  constexpr int G = 8;
  using Gm = Geo<T, G>;
  static_assert(TM_TST * TM_STAGE_COLS <= TM_COLS, "TMEM stages");
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  uint64_t* sfull = reinterpret_cast<uint64_t*>(base + SST * Gm::STAGE_BYTES);
  uint64_t* sempty = sfull + SST;
  uint64_t* tfull = sempty + SST;
  uint64_t* tempty = tfull + TM_TST;
  uint32_t* tbase_slot = reinterpret_cast<uint32_t*>(tempty + TM_TST);
  const uint32_t ring = smem_u32(base);

  if (status_failed(st)) return;  // validation failed: compute nothing (kernels.hpp:115,144)

  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  const int32_t tile_c = blockIdx.y * Gm::TILE_N;
  const uint32_t kb_lo = SPLIT ? blockIdx.z * slice_blocks : 0u;
  const uint32_t kb_hi = min(nkb_total, kb_lo + slice_blocks);
  const uint32_t nkb = kb_hi - kb_lo;
  if (SPLIT) out += blockIdx.z * slice_stride;

  if (threadIdx.x == 0) {
    for (int i = 0; i < SST; ++i) {
      mbar_init(&sfull[i], 1);
      mbar_init(&sempty[i], 1);
    }
    for (int i = 0; i < TM_TST; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], CW);
    }
    fence_barrier_init();
  }
  if (warp == CW + 1) {  // the copy warp owns the TMEM allocation
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tbase_slot)),
                 "n"(TM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = *tbase_slot;

  if (warp == CW) {
    // ---- TMA producer: global -> smem ring ----
    if (lane == 0) {
      prefetch_tensormap(&tmap);
      for (uint32_t i = 0; i < nkb; ++i) {
        const uint32_t slot = i % SST;
        if (i >= SST) mbar_sleep_wait_at(smem_u32(&sempty[slot]), ((i / SST) - 1) & 1);
        mbar_arrive_expect_tx(&sfull[slot], (uint32_t)Gm::STAGE_BYTES);
        const int32_t krow = (int32_t)((kb_lo + i) * KB);
#pragma unroll
        for (int h = 0; h < Gm::NBOX; ++h)
          tma_load_2d(base + slot * Gm::STAGE_BYTES + h * KB * BOX_BYTES, &tmap, &sfull[slot],
                      col0 + tile_c + h * Gm::BOX_N, krow);
      }
    }
    return;
  }

  if (warp == CW + 1) {
    // ---- copy warp: smem ring -> TMEM stages ----
    if (lane == 0) {
      for (uint32_t i = 0; i < nkb; ++i) {
        const uint32_t slot = i % SST;
        mbar_sleep_wait_at(smem_u32(&sfull[slot]), (i / SST) & 1);
        const uint32_t src = ring + slot * Gm::STAGE_BYTES;
#pragma unroll 1
        for (int h = 0; h < KB / TM_TKB; ++h) {
          const uint32_t j = i * (KB / TM_TKB) + h, ts = j % TM_TST;
          if (j >= TM_TST) mbar_sleep_wait_at(smem_u32(&tempty[ts]), ((j / TM_TST) - 1) & 1);
          tmem_fence_after();
          const uint32_t dst = tbase + ts * TM_STAGE_COLS;
#pragma unroll 1
          for (int kk = 0; kk < TM_TKB; ++kk)
#pragma unroll
            for (int g = 0; g < G; ++g)
              tmem_cp_32x128b_x4(
                  dst + kk * 32 + g * 4,
                  smem_desc_128(src + group_off(g) + (h * TM_TKB + kk) * BOX_BYTES));
          tmem_commit(smem_u32(&tfull[ts]));
        }
        tmem_commit(smem_u32(&sempty[slot]));
      }
    }
    __syncwarp();
    // wait for the consumers, then free TMEM
    asm volatile("bar.sync 1, %0;" ::"n"((CW + 1) * 32) : "memory");
    tmem_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(TM_COLS)
                 : "memory");
    return;
  }

  // ---- consumers: one output row per warp ----
  // rpc <= CW rows per CTA (the launcher trims it to balance the last wave);
  // warps past it walk no entries but still release every stage.
  const uint32_t b = warp < rpc ? blockIdx.x * rpc + warp : nrows;
  uint32_t cnt = b < nrows ? counts[b] : 0u;
  const int2* lst = lists + (uint64_t)(b < nrows ? b : 0) * cap;
  if (SPLIT) {
    const uint32_t p0 = lower_bound_k(lst, cnt, kb_lo * KB);
    const uint32_t p1 = kb_hi == nkb_total ? cnt : lower_bound_k(lst, cnt, kb_hi * KB);
    lst += p0;
    cnt = p1 - p0;
  }

  Acc<T, G> acc;
  acc.zero();
  const uint32_t k_lo = kb_lo * KB;
  const uint32_t tfull0 = smem_u32(tfull), tempty0 = smem_u32(tempty);
  // this warp's lane quadrant of the current TMEM stage
  const uint32_t tq = tbase + (((warp & 3u) * 32u) << 16);
  uint32_t kb_cur = 0, ts = 0, phase = 0;
  uint32_t stage_t = tq;
  auto advance = [&]() {
    tmem_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive_at(tempty0 + ts * 8);
    ++kb_cur;
    stage_t += TM_STAGE_COLS;
    if (++ts == TM_TST) {
      ts = 0;
      phase ^= 1;
      stage_t = tq;
    }
  };
  mbar_sleep_wait_at(tfull0, 0);
  tmem_fence_after();
  int2 cur = lane < cnt ? lst[lane] : make_int2(0, 0);
  int2 nxt = 32 + lane < cnt ? lst[32 + lane] : make_int2(0, 0);
  uint32_t k = (uint32_t)__shfl_sync(FULL, cur.x, 0);
  int rep = __shfl_sync(FULL, cur.y, 0);
  for (uint32_t e = 0; e < cnt; ++e) {
    const uint32_t f = e + 1;
    if ((f & 31u) == 0) {
      cur = nxt;
      const uint32_t pn = f + 32 + lane;
      nxt = pn < cnt ? lst[pn] : make_int2(0, 0);
    }
    const uint32_t k_n = (uint32_t)__shfl_sync(FULL, cur.x, f & 31u);
    const int rep_n = __shfl_sync(FULL, cur.y, f & 31u);
    const uint32_t kb = (k - k_lo) / TM_TKB;  // TMEM block within the slice
    while (kb_cur < kb) {
      advance();
      mbar_sleep_wait_at(tfull0 + ts * 8, phase);
      tmem_fence_after();
    }
    acc.run_tm(stage_t + (k % TM_TKB) * 32, rep);
    k = k_n;
    rep = rep_n;
  }
  while (true) {
    advance();
    if (kb_cur >= nkb * (KB / TM_TKB)) break;
    mbar_sleep_wait_at(tfull0 + ts * 8, phase);
  }
  tmem_fence_before();
  asm volatile("bar.sync 1, %0;" ::"n"((CW + 1) * 32) : "memory");

  if (b < nrows) acc.store(out + (uint64_t)b * ld_out, tile_c, ncols, lane, vec_ok != 0);
}

template <class T, bool SPLIT>
cudaError_t launch_tm_impl(const CUtensorMap* tmap, const int2* lists, uint64_t cap,
                           const uint32_t* counts, uint32_t nrows, int32_t col0, int32_t ncols,
                           uint32_t nkb, uint32_t slice_blocks, uint32_t splits,
                           uint64_t slice_stride, T* out, uint64_t ld_out, bool vec_ok,
                           const DevStatus* st, cudaStream_t s) {
  constexpr int CW = kTmemRows, SST = 4;
  auto kern = k_bform_tm<T, CW, SST, SPLIT>;
  const size_t smem = tm_smem_bytes<T, CW, SST>();
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  const uint32_t tiles = (ncols + Geo<T, 8>::TILE_N - 1) / Geo<T, 8>::TILE_N;
  const uint32_t rpc = balanced_rows(nrows, tiles * splits, CW, 1);
  dim3 grid((nrows + rpc - 1) / rpc, tiles, splits);
  kern<<<grid, (CW + 2) * 32, smem, s>>>(*tmap, lists, cap, counts, nrows, rpc, col0, ncols, nkb,
                                         slice_blocks, slice_stride, out, ld_out,
                                         vec_ok ? 1 : 0, st);
  note_launch();
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_tm(const CUtensorMap* tmap, const int2* lists, uint64_t cap,
                      const uint32_t* counts, uint32_t nrows, int32_t col0, int32_t ncols,
                      uint32_t nk, uint32_t* splits, uint64_t slice_stride, T* out,
                      uint64_t ld_out, const DevStatus* st, cudaStream_t s) {
  const uint32_t nkb = (nk + KB - 1) / KB;
  uint32_t want = *splits < 1 ? 1 : *splits;
  if (want > nkb) want = nkb;
  const uint32_t slice_blocks = (nkb + want - 1) / want;
  *splits = (nkb + slice_blocks - 1) / slice_blocks;
  const bool vec_ok = (ld_out * sizeof(T)) % 16 == 0 &&
                      (reinterpret_cast<uintptr_t>(out) % 16) == 0 &&
                      (slice_stride * sizeof(T)) % 16 == 0;
  if (*splits > 1)
    return launch_tm_impl<T, true>(tmap, lists, cap, counts, nrows, col0, ncols, nkb,
                                   slice_blocks, *splits, slice_stride, out, ld_out, vec_ok, st, s);
  return launch_tm_impl<T, false>(tmap, lists, cap, counts, nrows, col0, ncols, nkb, slice_blocks,
                                  1, slice_stride, out, ld_out, vec_ok, st, s);
}

// ---------------------------------------------------------------------------
// k_aform: Case A with the base uniform per warp ("A-form").
//
// The B-form runs Case A on transposed operands, so its lanes are Z rows and
// every zero base X[i,k] leaves a lane idle: at density d1 the FP pipe does at
// most d1 useful work (cfg3 d1 = 0.1: 3-9% of peak). Here a warp owns Z row i
// in the reference's own orientation (kernels.hpp:118-135): it walks row i's
// compacted nonzero bases (k, X[i,k]) -- zero bases are skipped for the whole
// warp, as the reference skips them -- and each lane holds CPL columns j of
// Z[i,:]. The reps Y[k,j] now differ per lane, so the rep loop runs the
// warp-uniform trip count R = max |Y[k,j]| over the CTA's column tile
// (precomputed per (k, tile)), and iteration t adds the base to exactly the
// columns with |Y[k,j]| >= t: one setp.ge.f16x2 tests two columns' fp16 counts
// (exact up to 2048) and sets two predicates for two predicated FADDs. Each
// element still receives its |rep| adds consecutively (iterations 1..|rep|)
// at its k, in k order: the reference's order, bit for bit. The counts arrive
// as fp16 tiles through a TMA ring (2 bytes per element instead of 4).
// Cost ~ R x (CPL/2 setp + CPL FADD) per entry: useful while the zero-base
// waste of the B-form is larger (sparse X).
// ---------------------------------------------------------------------------

template <class T>
struct AformGeo {
  static constexpr int CPL = sizeof(T) == 4 ? 32 : 16;  // columns per lane
  static constexpr int TILE = 32 * CPL;                 // columns per CTA
  static constexpr int NBOX = TILE / 256;               // 256-half TMA boxes per k row
  static constexpr int STAGE_BYTES = KB * TILE * 2;
  static constexpr int NPAIR = CPL / 2;                 // f16x2 count registers per lane
  static constexpr int NGRP = CPL / 8;                  // 128-bit count loads per entry
};

__device__ __forceinline__ uint32_t hadd2_bits(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("add.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

// columns (2p, 2p+1): add b where count >= th (both halves of th equal t)
__device__ __forceinline__ void padd_ge(float& a0, float& a1, uint32_t cnt, uint32_t th, float b) {
  asm("{\n\t.reg .pred p, q;\n\tsetp.ge.f16x2 p|q, %2, %3;\n\t"
      "@p add.rn.f32 %0, %0, %4;\n\t@q add.rn.f32 %1, %1, %4;\n\t}"
      : "+f"(a0), "+f"(a1)
      : "r"(cnt), "r"(th), "f"(b));
}
// add nb (= -base) where count <= thn (= -t): the negative reps
__device__ __forceinline__ void padd_le(float& a0, float& a1, uint32_t cnt, uint32_t thn, float nb) {
  asm("{\n\t.reg .pred p, q;\n\tsetp.le.f16x2 p|q, %2, %3;\n\t"
      "@p add.rn.f32 %0, %0, %4;\n\t@q add.rn.f32 %1, %1, %4;\n\t}"
      : "+f"(a0), "+f"(a1)
      : "r"(cnt), "r"(thn), "f"(nb));
}
__device__ __forceinline__ void padd_ge(double& a0, double& a1, uint32_t cnt, uint32_t th,
                                        double b) {
  asm("{\n\t.reg .pred p, q;\n\tsetp.ge.f16x2 p|q, %2, %3;\n\t"
      "@p add.rn.f64 %0, %0, %4;\n\t@q add.rn.f64 %1, %1, %4;\n\t}"
      : "+d"(a0), "+d"(a1)
      : "r"(cnt), "r"(th), "d"(b));
}
__device__ __forceinline__ void padd_le(double& a0, double& a1, uint32_t cnt, uint32_t thn,
                                        double nb) {
  asm("{\n\t.reg .pred p, q;\n\tsetp.le.f16x2 p|q, %2, %3;\n\t"
      "@p add.rn.f64 %0, %0, %4;\n\t@q add.rn.f64 %1, %1, %4;\n\t}"
      : "+d"(a0), "+d"(a1)
      : "r"(cnt), "r"(thn), "d"(nb));
}

__device__ __forceinline__ float entry_base(int2 e) { return __int_as_float(e.y); }
__device__ __forceinline__ double entry_base(int4 e) { return __hiloint2double(e.w, e.z); }
__device__ __forceinline__ int2 shfl_entry(int2 v, uint32_t src) {
  return make_int2(__shfl_sync(FULL, v.x, src), __shfl_sync(FULL, v.y, src));
}
__device__ __forceinline__ int4 shfl_entry(int4 v, uint32_t src) {
  return make_int4(__shfl_sync(FULL, v.x, src), 0, __shfl_sync(FULL, v.z, src),
                   __shfl_sync(FULL, v.w, src));
}

template <class T, int CW, int STAGES, int MINB>
__global__ void __launch_bounds__((CW + 1) * 32, MINB)
    k_aform(const __grid_constant__ CUtensorMap cmap,
            const typename AEntry<T>::type* __restrict__ lists, uint64_t cap,
            const uint32_t* __restrict__ counts, uint32_t nrows, uint32_t rpc, uint32_t ncols,
            uint32_t nkb, const uint16_t* __restrict__ rmax, uint32_t ntiles,
            T* __restrict__ out, uint64_t ld_out, const uint32_t* __restrict__ row_idx,
            const DevStatus* __restrict__ st) {
  using Ag = AformGeo<T>;
  using E = typename AEntry<T>::type;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + STAGES * Ag::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  const uint32_t ring = smem_u32(base);

  if (status_failed(st)) return;  // validation failed: compute nothing (kernels.hpp:115)

  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  const uint32_t tile = blockIdx.y;
  const int32_t tile_c = (int32_t)(tile * Ag::TILE);

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], CW);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == CW) {
    // ---- TMA producer: fp16 count tiles ----
    if (lane == 0) {
      prefetch_tensormap(&cmap);
      for (uint32_t i = 0; i < nkb; ++i) {
        const uint32_t slot = i % STAGES;
        if (i >= STAGES) mbar_sleep_wait_at(smem_u32(&empty[slot]), ((i / STAGES) - 1) & 1);
        mbar_arrive_expect_tx(&full[slot], (uint32_t)Ag::STAGE_BYTES);
#pragma unroll
        for (int bx = 0; bx < Ag::NBOX; ++bx)
          tma_load_2d(base + slot * Ag::STAGE_BYTES + bx * KB * 512, &cmap, &full[slot],
                      tile_c + bx * 256, (int32_t)(i * KB));
      }
    }
    return;
  }

  // ---- consumers: one Z row per warp ----
  const uint32_t b = warp < rpc ? blockIdx.x * rpc + warp : nrows;
  const uint32_t q = b < nrows ? (row_idx ? row_idx[b] : b) : 0u;  // list / Z row
  const uint32_t cnt = b < nrows ? counts[q] : 0u;
  const E* lst = lists + (uint64_t)q * cap;
  T acc[Ag::CPL];
#pragma unroll
  for (int c = 0; c < Ag::CPL; ++c) acc[c] = T(0);

  const uint32_t full0 = smem_u32(full), empty0 = smem_u32(empty);
  uint32_t kb_cur = 0, slot = 0, phase = 0;
  uint32_t stage_addr = ring + lane * 16;
  auto advance = [&]() {
    __syncwarp();
    if (lane == 0) mbar_arrive_at(empty0 + slot * 8);
    ++kb_cur;
    stage_addr += Ag::STAGE_BYTES;
    if (++slot == STAGES) {
      slot = 0;
      phase ^= 1;
      stage_addr -= STAGES * Ag::STAGE_BYTES;
    }
  };
  const uint16_t* rm_col = rmax + tile;
  mbar_sleep_wait_at(full0, 0);
  E cur = lane < cnt ? lst[lane] : E{};
  E nxt = 32 + lane < cnt ? lst[32 + lane] : E{};
  E ent = shfl_entry(cur, 0);
  uint32_t rm = cnt ? __ldg(rm_col + (uint64_t)(uint32_t)ent.x * ntiles) : 0u;
  for (uint32_t e = 0; e < cnt; ++e) {
    const uint32_t f = e + 1;
    if ((f & 31u) == 0) {
      cur = nxt;
      const uint32_t pn = f + 32 + lane;
      nxt = pn < cnt ? lst[pn] : E{};
    }
    const E ent_n = shfl_entry(cur, f & 31u);
    const uint32_t rm_n = f < cnt ? __ldg(rm_col + (uint64_t)(uint32_t)ent_n.x * ntiles) : 0u;
    const uint32_t k = (uint32_t)ent.x;
    const uint32_t kb = k / KB;
    while (kb_cur < kb) {
      advance();
      mbar_sleep_wait_at(full0 + slot * 8, phase);
    }
    const int R = (int)(rm & 0x7fffu);
    if (R != 0) {
      uint32_t c2[Ag::NPAIR];
#pragma unroll
      for (int g = 0; g < Ag::NGRP; ++g) {
        uint32_t v0, v1, v2, v3;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3)
                     : "r"(stage_addr + g * KB * 512 + (k % KB) * 512));
        c2[4 * g] = v0;
        c2[4 * g + 1] = v1;
        c2[4 * g + 2] = v2;
        c2[4 * g + 3] = v3;
      }
      const T bv = entry_base(ent);
      // thresholds t (and -t) as f16x2, stepped by an exact f16x2 add (t <= 2048
      // is exact in fp16); an I2F.F16 per trip instead was 1-2% slower, and
      // unrolling this loop by 2 or 4 was 4-10% slower (measured)
      constexpr uint32_t kOne2 = 0x3c003c00u, kMinusOne2 = 0xbc00bc00u;
      if ((rm & 0x8000u) == 0) {
        uint32_t th = kOne2;
#pragma unroll 1
        for (int t = 1; t <= R; ++t) {
#pragma unroll
          for (int p = 0; p < Ag::NPAIR; ++p) padd_ge(acc[2 * p], acc[2 * p + 1], c2[p], th, bv);
          th = hadd2_bits(th, kOne2);
        }
      } else {  // the tile row holds negative reps: step = -base there (kernels.hpp:97)
        const T nb = -bv;
        uint32_t th = kOne2, thn = kMinusOne2;
#pragma unroll 1
        for (int t = 1; t <= R; ++t) {
#pragma unroll
          for (int p = 0; p < Ag::NPAIR; ++p) {
            padd_ge(acc[2 * p], acc[2 * p + 1], c2[p], th, bv);
            padd_le(acc[2 * p], acc[2 * p + 1], c2[p], thn, nb);
          }
          th = hadd2_bits(th, kOne2);
          thn = hadd2_bits(thn, kMinusOne2);
        }
      }
    }
    ent = ent_n;
    rm = rm_n;
  }
  while (true) {
    advance();
    if (kb_cur >= nkb) break;
    mbar_sleep_wait_at(full0 + slot * 8, phase);
  }

  if (b < nrows) {
    T* orow = out + (uint64_t)q * ld_out;
#pragma unroll
    for (int g = 0; g < Ag::NGRP; ++g) {
      const uint32_t c0 = (uint32_t)tile_c + g * 256 + 8 * lane;
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (c0 + e < ncols) orow[c0 + e] = acc[8 * g + e];
    }
  }
}

// ---------------------------------------------------------------------------
// k_bform_mr: RW output rows per warp over a DENSE rep tile.
//
// For small reps the per-entry cost of k_bform is the shared-memory read of
// the bases (TILE_N * sizeof(T) bytes per warp per entry, at 128 B/clk/SM),
// not the adds: with |rep| = 1 a 512-column fp32 entry moves 2 KB from smem
// for 16 FADD2. Here each warp owns RW rows, walks k densely, reads the RW
// reps of the current k with one broadcast LDS from a staged dense rep tile,
// and loads the bases once for all RW rows. The rep tile ([k][row] int32,
// built by the prepass) arrives through the same TMA ring as the bases.
// Per element the order is unchanged: k ascending, |rep| sequential adds.
// ---------------------------------------------------------------------------

constexpr int MR_RW = 4;       // rows per warp
// 12 consumer warps + 1 producer: 3 consumers per SM sub-partition and a
// 128-register budget (4 x 16 accumulators + 16 bases); 17 warps cap it at 96.
constexpr int MR_CW = 12;
constexpr int MR_ROWS = MR_RW * MR_CW;  // 48 rows per CTA: a 192-byte int32 rep box row
constexpr int MR_STAGES = 8;

template <class T, int G>
__host__ __device__ constexpr size_t mr_smem_bytes() {
  return 1024 + (size_t)MR_STAGES * (Geo<T, G>::STAGE_BYTES + KB * MR_ROWS * 4) +
         2 * MR_STAGES * sizeof(uint64_t);
}

__device__ __forceinline__ int4 lds128i(uint32_t addr) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr));
  return v;
}

// rmap: dense reps R'[k][row] (int32, rows = B-form rows, inner dimension).
template <class T, int G>
__global__ void __launch_bounds__((MR_CW + 1) * 32, 1)
    k_bform_mr(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap rmap,
               uint32_t nrows, int32_t col0, int32_t ncols, uint32_t nk, uint32_t nkb,
               T* __restrict__ out, uint64_t ld_out, int vec_ok,
               const DevStatus* __restrict__ st) {
  using Gm = Geo<T, G>;
  constexpr int REP_STAGE = KB * MR_ROWS * 4;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* reps = base + MR_STAGES * Gm::STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(reps + MR_STAGES * REP_STAGE);
  uint64_t* empty = full + MR_STAGES;
  const uint32_t ring = smem_u32(base), rring = smem_u32(reps);

  if (status_failed(st)) return;  // validation failed: compute nothing (kernels.hpp:115,144)

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t tile_c = blockIdx.y * Gm::TILE_N;
  const uint32_t row0 = blockIdx.x * MR_ROWS;

  if (threadIdx.x == 0) {
    for (int s = 0; s < MR_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MR_CW);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == MR_CW) {
    // ---- dedicated TMA producer warp: base tile + dense rep tile per stage ----
    if (lane == 0) {
      Pump<T, G, MR_STAGES> pump{&tmap, &rmap, base, reps, full, empty, col0 + tile_c,
                                 (int32_t)row0, nkb, 0, (uint32_t)REP_STAGE, 0};
      prefetch_tensormap(&tmap);
      prefetch_tensormap(&rmap);
      while (true) {
        pump.pump();
        if (pump.next >= nkb) break;
        mbar_sleep_wait_at(smem_u32(&empty[pump.next % MR_STAGES]),
                           ((pump.next / MR_STAGES) - 1) & 1);
      }
    }
    return;
  }

  Acc<T, G> acc[MR_RW];
#pragma unroll
  for (int w = 0; w < MR_RW; ++w) acc[w].zero();

  uint32_t slot = 0, phase = 0;
  for (uint32_t kb = 0; kb < nkb; ++kb) {
    mbar_sleep_wait_at(smem_u32(&full[slot]), phase);
    const uint32_t bstage = ring + slot * Gm::STAGE_BYTES + lane * 16;
    const uint32_t rstage = rring + slot * REP_STAGE + warp * (MR_RW * 4);
    const uint32_t kk_end = nk - kb * KB < (uint32_t)KB ? nk - kb * KB : (uint32_t)KB;
    for (uint32_t kk = 0; kk < kk_end; ++kk) {
      const int4 r = lds128i(rstage + kk * (MR_ROWS * 4));  // this warp's RW reps at k
      if ((r.x | r.y | r.z | r.w) == 0) continue;
      const typename Acc<T, G>::Bases b = Acc<T, G>::load_bases(bstage + kk * BOX_BYTES);
      if (r.x) acc[0].add(b, r.x);
      if (r.y) acc[1].add(b, r.y);
      if (r.z) acc[2].add(b, r.z);
      if (r.w) acc[3].add(b, r.w);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
    if (++slot == MR_STAGES) {
      slot = 0;
      phase ^= 1;
    }
  }

#pragma unroll
  for (int w = 0; w < MR_RW; ++w) {
    const uint32_t row = row0 + warp * MR_RW + w;
    if (row < nrows) acc[w].store(out + (uint64_t)row * ld_out, tile_c, ncols, lane, vec_ok != 0);
  }
}

template <class T, int G, int CW, int STAGES, int MINB>
cudaError_t launch_ring(const CUtensorMap* tmap, const int2* lists, uint64_t cap,
                        const uint32_t* counts, uint32_t nrows, int32_t col0, int32_t ncols,
                        uint32_t nk, uint32_t* splits, uint64_t slice_stride, T* out,
                        uint64_t ld_out, const DevStatus* st, cudaStream_t s) {
  const uint32_t nkb = (nk + KB - 1) / KB;
  uint32_t want = *splits < 1 ? 1 : *splits;
  if (want > nkb) want = nkb;
  auto kern = want > 1 ? k_bform<T, G, CW, STAGES, MINB, true>
                       : k_bform<T, G, CW, STAGES, MINB, false>;
  const size_t smem = ring_smem_bytes<T, G, STAGES>();
  // set on every call: the attribute is per device and costs ~1 us
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  const uint32_t slice_blocks = (nkb + want - 1) / want;
  *splits = (nkb + slice_blocks - 1) / slice_blocks;
  const bool vec_ok = (ld_out * sizeof(T)) % 16 == 0 &&
                      (reinterpret_cast<uintptr_t>(out) % 16) == 0 &&
                      (slice_stride * sizeof(T)) % 16 == 0;
  const uint32_t tiles = (ncols + Geo<T, G>::TILE_N - 1) / Geo<T, G>::TILE_N;
  const uint32_t rpc = balanced_rows(nrows, tiles * *splits, CW, MINB);
  dim3 grid((nrows + rpc - 1) / rpc, tiles, *splits);
  kern<<<grid, (CW + kProdWarps) * 32, smem, s>>>(*tmap, lists, cap, counts, nrows, rpc, col0, ncols, nkb,
                                         slice_blocks, slice_stride, out, ld_out,
                                         vec_ok ? 1 : 0, st);
  note_launch();
  return cudaGetLastError();
}

}  // namespace

int bform_box_bytes() { return BOX_BYTES; }
int bform_kb() { return KB; }

template <class T>
cudaError_t launch_bform(int shape, const CUtensorMap* tmap, const int2* lists, uint64_t cap,
                         const uint32_t* counts, uint32_t nrows, int32_t col0, int32_t ncols,
                         uint32_t nk, uint32_t* splits, uint64_t slice_stride, T* out,
                         uint64_t ld_out, const DevStatus* st, cudaStream_t s) {
  if (shape == kShapeWide)
    // 1024 fp32 / 512 fp64 columns x 16 rows, 16 consumers + producer, 6-stage
    // ring (192 KB), 1 CTA per SM, 83 registers. Measured against 8 rows x 3
    // stages x 2 CTAs per SM (tools/exp_time.py): cfg5 1810 -> 1802 ms, cfg2
    // 0.307 -> 0.285 ms, cfg3 and cfg4 0.3-2% faster -- the deeper ring lets
    // warps drift 5 k blocks apart instead of 2 (consumers had waited on a
    // stage 6.5% of the time, ncu). Before the rep loop and list walk were
    // slimmed (80-83 registers) this shape hit the 96-register cap of 17 warps
    // and spilled.
    return launch_ring<T, AFMM_EXP_WIDE_G, AFMM_EXP_WIDE_CW, AFMM_EXP_WIDE_STAGES, AFMM_EXP_WIDE_MINB>(tmap, lists, cap, counts, nrows, col0, ncols, nk,
                                              splits, slice_stride, out, ld_out, st, s);
  if (shape == kShapeTmem)
    // 1024 fp32 / 512 fp64 columns x 16 rows, bases from tensor memory, 1 CTA per SM
    return launch_tm<T>(tmap, lists, cap, counts, nrows, col0, ncols, nk, splits, slice_stride,
                        out, ld_out, st, s);
  if (shape == kShapeSmall)  // 256 fp32 / 128 fp64 columns x 4 rows, up to 8 CTAs per SM
    return launch_ring<T, 2, 4, 3, 8>(tmap, lists, cap, counts, nrows, col0, ncols, nk, splits,
                                      slice_stride, out, ld_out, st, s);
  return launch_ring<T, 4, 16, 6, 2>(tmap, lists, cap, counts, nrows, col0, ncols, nk, splits,
                                     slice_stride, out, ld_out, st, s);
}

template cudaError_t launch_bform<float>(int, const CUtensorMap*, const int2*, uint64_t,
                                         const uint32_t*, uint32_t, int32_t, int32_t, uint32_t,
                                         uint32_t*, uint64_t, float*, uint64_t, const DevStatus*,
                                         cudaStream_t);
template cudaError_t launch_bform<double>(int, const CUtensorMap*, const int2*, uint64_t,
                                          const uint32_t*, uint32_t, int32_t, int32_t, uint32_t,
                                          uint32_t*, uint64_t, double*, uint64_t,
                                          const DevStatus*, cudaStream_t);

template <class T>
cudaError_t launch_aform(const CUtensorMap* cmap, const typename AEntry<T>::type* lists,
                         uint64_t cap, const uint32_t* counts, uint32_t nrows, uint32_t ncols,
                         uint32_t nk, const uint16_t* rmax, T* out, uint64_t ld_out,
                         const uint32_t* row_idx, const DevStatus* st, cudaStream_t s) {
  using Ag = AformGeo<T>;
  static_assert(Ag::TILE == (int)aform_tile_cols<T>(), "A-form tile width");
  // 16 rows x 12 stages x 1 CTA/SM: 4-5% faster than 8 rows x 6 stages x 2
  // CTAs/SM on cfg3 d1 = 0.1 (tools/exp_time.py --aform)
  constexpr int CW = kAformRows, STAGES = 12, MINB = kAformCtasPerSm;
  auto kern = k_aform<T, CW, STAGES, MINB>;
  const size_t smem = 128 + (size_t)STAGES * Ag::STAGE_BYTES + 2 * STAGES * sizeof(uint64_t);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  const uint32_t nkb = (nk + KB - 1) / KB;
  const uint32_t tiles = (ncols + Ag::TILE - 1) / Ag::TILE;
  const uint32_t rpc = balanced_rows(nrows, tiles, CW, MINB);
  dim3 grid((nrows + rpc - 1) / rpc, tiles);
  kern<<<grid, (CW + 1) * 32, smem, s>>>(*cmap, lists, cap, counts, nrows, rpc, ncols, nkb, rmax,
                                         tiles, out, ld_out, row_idx, st);
  note_launch();
  return cudaGetLastError();
}

template cudaError_t launch_aform<float>(const CUtensorMap*, const int2*, uint64_t,
                                         const uint32_t*, uint32_t, uint32_t, uint32_t,
                                         const uint16_t*, float*, uint64_t, const uint32_t*,
                                         const DevStatus*, cudaStream_t);
template cudaError_t launch_aform<double>(const CUtensorMap*, const int4*, uint64_t,
                                          const uint32_t*, uint32_t, uint32_t, uint32_t,
                                          const uint16_t*, double*, uint64_t, const uint32_t*,
                                          const DevStatus*, cudaStream_t);

int bform_mr_rows() { return MR_ROWS; }

template <class T>
cudaError_t launch_bform_mr(const CUtensorMap* tmap, const CUtensorMap* rmap, uint32_t nrows,
                            int32_t col0, int32_t ncols, uint32_t nk, T* out, uint64_t ld_out,
                            const DevStatus* st, cudaStream_t s) {
  constexpr int G = 4;
  auto kern = k_bform_mr<T, G>;
  const size_t smem = mr_smem_bytes<T, G>();
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  const uint32_t nkb = (nk + KB - 1) / KB;
  const bool vec_ok = (ld_out * sizeof(T)) % 16 == 0 &&
                      (reinterpret_cast<uintptr_t>(out) % 16) == 0;
  dim3 grid((nrows + MR_ROWS - 1) / MR_ROWS, (ncols + Geo<T, G>::TILE_N - 1) / Geo<T, G>::TILE_N);
  kern<<<grid, (MR_CW + 1) * 32, smem, s>>>(*tmap, *rmap, nrows, col0, ncols, nk, nkb, out,
                                            ld_out, vec_ok ? 1 : 0, st);
  note_launch();
  return cudaGetLastError();
}

template cudaError_t launch_bform_mr<float>(const CUtensorMap*, const CUtensorMap*, uint32_t,
                                            int32_t, int32_t, uint32_t, float*, uint64_t,
                                            const DevStatus*, cudaStream_t);
template cudaError_t launch_bform_mr<double>(const CUtensorMap*, const CUtensorMap*, uint32_t,
                                             int32_t, int32_t, uint32_t, double*, uint64_t,
                                             const DevStatus*, cudaStream_t);

}  // namespace afmm_dev
