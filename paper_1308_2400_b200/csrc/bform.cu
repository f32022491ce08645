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
// Contents: k_bform (the product kernel, three tile shapes), k_aform
// (A-form) and their launchers. (Variants measured slower in round 1 -- a
// TMEM-fed B-form and a dense-rep multi-row kernel -- were removed from the
// library; DESIGN.md section 3.3 keeps their measurements.)
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
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace afmm_dev {

namespace {

constexpr unsigned FULL = 0xffffffffu;

constexpr int KB = 8;  // k rows per stage
// rep loop: trips of 8 steps, then the remainder (< 8) by its binary digits
// (4, 2, 1 steps) with no loop. Measured against 4-step trips + a 1-step
// remainder loop: cfg5 1845 -> 1809 ms, rep 16 0.901 -> 0.912 of peak, and 88
// registers instead of 96 + an 8-byte spill (ptxas); the loop counter and
// back-edge instructions it removes issue on the FMA pipe (VIADD) or stall on
// branch resolution.
constexpr int REP_UNROLL = 8;  // rep-loop unroll (adds per column per trip)
static_assert((REP_UNROLL & (REP_UNROLL - 1)) == 0, "a binary remainder needs a power-of-two unroll");
constexpr uint32_t kListPrefetch = 64;  // list entries ahead prefetched into L1

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

// One FP-add operand: a float2 (FADD2, two fp32 columns) or a double (DADD).
template <class T>
struct Lane;
template <>
struct Lane<float> {
  using V = float2;
  __device__ __forceinline__ static V zero() { return make_float2(0.f, 0.f); }
  template <bool NEG>
  __device__ __forceinline__ static V add(V a, V b) {
    // the negation is the FADD2 operand-negate modifier (exact)
    return __fadd2_rn(a, NEG ? make_float2(-b.x, -b.y) : b);
  }
  __device__ __forceinline__ static void load(uint32_t addr, V* b) {
    const float4 v = lds128f(addr);
    b[0] = make_float2(v.x, v.y);
    b[1] = make_float2(v.z, v.w);
  }
};
template <>
struct Lane<double> {
  using V = double;
  __device__ __forceinline__ static V zero() { return 0.0; }
  template <bool NEG>
  __device__ __forceinline__ static V add(V a, V b) {
    return __dadd_rn(a, NEG ? -b : b);
  }
  __device__ __forceinline__ static void load(uint32_t addr, V* b) {
    const double2 v = lds128d(addr);
    b[0] = v.x;
    b[1] = v.y;
  }
};

// The bases of one staged k row for this lane: G 16-byte column groups.
template <class T, int G>
struct Bases {
  typename Lane<T>::V b[2 * G];
  __device__ __forceinline__ void load(uint32_t row_addr) {
#pragma unroll
    for (int g = 0; g < G; ++g) Lane<T>::load(row_addr + group_off(g), &b[2 * g]);
  }
};

// Register-resident accumulators of one output row: 2G operands per lane.
template <class T, int G>
struct Acc {
  using L = Lane<T>;
  typename L::V a[2 * G];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int c = 0; c < 2 * G; ++c) a[c] = L::zero();
  }
  // t sequential `acc += step` per column, step = NEG ? -base : base
  // (kernels.hpp:95-104): trips of REP_UNROLL steps, then the remainder by its
  // binary digits (no loop, no predicated FP tail).
  template <bool NEG>
  __device__ __forceinline__ void add_t(const Bases<T, G>& s, uint32_t t) {
#pragma unroll 1
    while (t >= REP_UNROLL) {
#pragma unroll
      for (int u = 0; u < REP_UNROLL; ++u)
#pragma unroll
        for (int c = 0; c < 2 * G; ++c) a[c] = L::template add<NEG>(a[c], s.b[c]);
      t -= REP_UNROLL;
    }
#pragma unroll
    for (int bit = REP_UNROLL / 2; bit >= 1; bit >>= 1)
      if (t & (uint32_t)bit) {
#pragma unroll
        for (int u = 0; u < bit; ++u)
#pragma unroll
          for (int c = 0; c < 2 * G; ++c) a[c] = L::template add<NEG>(a[c], s.b[c]);
      }
  }
  // AFMM_MODE_FAST_LADDER: the t copies of the step reassociated as a doubling
  // ladder. s.b becomes b, 2b, 4b, ... (exact: power-of-two multiples, and
  // |2^j b| <= |t b|), and the multiples picked by the binary digits of t are
  // added into the element: floor(log2 t) + popcount(t) adds instead of t.
  template <bool NEG>
  __device__ __forceinline__ void add_ladder(Bases<T, G>& s, uint32_t t) {
#pragma unroll 1
    while (true) {
      if (t & 1u) {
#pragma unroll
        for (int c = 0; c < 2 * G; ++c) a[c] = L::template add<NEG>(a[c], s.b[c]);
      }
      t >>= 1;
      if (t == 0u) break;
#pragma unroll
      for (int c = 0; c < 2 * G; ++c) s.b[c] = L::template add<false>(s.b[c], s.b[c]);
    }
  }
  __device__ __forceinline__ void run_ladder(uint32_t row_addr, int rep) {
    Bases<T, G> s;
    s.load(row_addr);
    if (rep >= 0) add_ladder<false>(s, (uint32_t)rep);
    else add_ladder<true>(s, 0u - (uint32_t)rep);
  }
  // |rep| sequential adds of step = rep >= 0 ? base : -base (kernels.hpp:97)
  __device__ __forceinline__ void add(const Bases<T, G>& s, int rep) {
    if (rep >= 0) add_t<false>(s, (uint32_t)rep);
    else add_t<true>(s, 0u - (uint32_t)rep);
  }
  // One list entry: load the bases of the staged k row, run the rep loop.
  // (Splitting wide tiles into two half-width loops to save 16 base registers
  // was measured 3% slower.)
  __device__ __forceinline__ void run(uint32_t row_addr, int rep) {
    Bases<T, G> s;
    s.load(row_addr);
    add(s, rep);
  }
  // Columns of operand c: tile_col + (c/2)*GROUP_COLS + lane*PER_LANE + (c%2)*(PER_LANE/2)
  __device__ __forceinline__ void store(T* out_row, int32_t oc0, int32_t ncols, uint32_t lane,
                                        bool vec_ok) const {
    constexpr int PER_LANE = 16 / sizeof(T);      // columns per lane per group
    constexpr int GROUP_COLS = 32 * PER_LANE;     // columns per group
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int32_t c = oc0 + g * GROUP_COLS + PER_LANE * (int32_t)lane;
      T v[PER_LANE];
      if constexpr (sizeof(T) == 4) {
        v[0] = a[2 * g].x; v[1] = a[2 * g].y; v[2] = a[2 * g + 1].x; v[3] = a[2 * g + 1].y;
      } else {
        v[0] = a[2 * g]; v[1] = a[2 * g + 1];
      }
      if (vec_ok && c + PER_LANE - 1 < ncols) {
        if constexpr (sizeof(T) == 4)
          *reinterpret_cast<float4*>(out_row + c) = make_float4(v[0], v[1], v[2], v[3]);
        else
          *reinterpret_cast<double2*>(out_row + c) = make_double2(v[0], v[1]);
      } else {
#pragma unroll
        for (int e = 0; e < PER_LANE; ++e)
          if (c + e < ncols) out_row[c + e] = v[e];
      }
    }
  }
};

// Fast (reassociated) mode: each element's chain runs in the T accumulators
// for a block of kFlushBlocks k blocks, then the block's partial is added into
// an fp64 total ("blocked summation"): every term keeps its |rep| adds, plus
// one add per element and block. An fp32 chain of ~32K adds (cfg4, full size)
// drifts to 7e-5 of sum |terms|; chains of one block stay within ~1e-6.
constexpr uint32_t kFlushBlocks = 4;

template <class T, int G>
struct Total {
  static constexpr int NE = 2 * G * (int)(sizeof(float2) / sizeof(T));  // elements per lane
  double t[NE];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int e = 0; e < NE; ++e) t[e] = 0.0;
  }
  __device__ __forceinline__ void flush(Acc<T, G>& acc) {
#pragma unroll
    for (int c = 0; c < 2 * G; ++c) {
      if constexpr (sizeof(T) == 4) {
        t[2 * c] = __dadd_rn(t[2 * c], (double)acc.a[c].x);
        t[2 * c + 1] = __dadd_rn(t[2 * c + 1], (double)acc.a[c].y);
      } else {
        t[c] = __dadd_rn(t[c], acc.a[c]);
      }
    }
    acc.zero();
  }
  // the totals, rounded once to T, back into the accumulators (for store())
  __device__ __forceinline__ void to(Acc<T, G>& acc) const {
#pragma unroll
    for (int c = 0; c < 2 * G; ++c) {
      if constexpr (sizeof(T) == 4)
        acc.a[c] = make_float2(__double2float_rn(t[2 * c]), __double2float_rn(t[2 * c + 1]));
      else
        acc.a[c] = t[c];
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

// TMA producer (one thread): fills ring slot i % STAGES with k block
// kb_lo + i of the slice, i < nkb, as soon as every consumer has released the
// block STAGES earlier. The waits suspend in hardware (no polling).
template <int STAGE_BYTES, int NBOX, int BOX_N, int STAGES>
__device__ __forceinline__ void produce(const CUtensorMap* tmap, unsigned char* ring,
                                        uint64_t* full, uint64_t* empty, int32_t col,
                                        uint32_t kb_lo, uint32_t nkb) {
  prefetch_tensormap(tmap);
  for (uint32_t i = 0; i < nkb; ++i) {
    const uint32_t slot = i % STAGES;
    if (i >= STAGES) mbar_sleep_wait_at(smem_u32(&empty[slot]), ((i / STAGES) - 1) & 1);
    mbar_arrive_expect_tx(&full[slot], (uint32_t)STAGE_BYTES);
    const int32_t krow = (int32_t)((kb_lo + i) * KB);
#pragma unroll
    for (int h = 0; h < NBOX; ++h)
      tma_load_2d(ring + slot * STAGE_BYTES + h * KB * BOX_BYTES, tmap, &full[slot],
                  col + h * BOX_N, krow);
  }
}

// A consumer warp's position in the ring: the k block it holds (kb_cur), that
// block's slot and fill parity, and the smem address of the slot plus this
// lane's first 16-byte column group.
template <int STAGES, int STAGE_BYTES>
struct Cursor {
  uint32_t kb_cur = 0, slot = 0, phase = 0, stage_addr, full0, empty0;
  __device__ __forceinline__ Cursor(uint32_t ring, uint32_t full_addr, uint32_t empty_addr,
                                    uint32_t lane)
      : stage_addr(ring + lane * 16), full0(full_addr), empty0(empty_addr) {}
  __device__ __forceinline__ void wait() { mbar_sleep_wait_at(full0 + slot * 8, phase); }
  // release the held block (one arrival per warp) and step to the next
  __device__ __forceinline__ void advance(uint32_t lane) {
    __syncwarp();
    if (lane == 0) mbar_arrive_at(empty0 + slot * 8);
    ++kb_cur;
    stage_addr += STAGE_BYTES;
    if (++slot == STAGES) {
      slot = 0;
      phase ^= 1;
      stage_addr -= STAGES * STAGE_BYTES;
    }
  }
  __device__ __forceinline__ void seek(uint32_t kb, uint32_t lane) {
    while (kb_cur < kb) {
      advance(lane);
      wait();
    }
  }
  // release every remaining block in order (the ring needs all CW arrivals)
  __device__ __forceinline__ void drain(uint32_t nkb, uint32_t lane) {
    while (true) {
      advance(lane);
      if (kb_cur >= nkb) break;
      wait();
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

// k_bform: each consumer warp owns one B-form row b of a TILE_N-column tile
// and walks the row's (k, rep) list.
//   lists: row b's entries at lists[b * cap .. b * cap + counts[b]), k increasing.
//   Output row b, column (col0 + c) -> out[b * ld_out + c], c < ncols.
//   dyn_ncols (optional): ncols decided on the device (Case A row split).
//   k slice: blockIdx.z selects slice z = [z*slice_blocks, (z+1)*slice_blocks)
//   of the nkb_total k blocks and writes to out + z * slice_stride (fast-mode
//   split-k; one slice = the whole k range in order-preserving mode).
// PACKED: the lists hold 4-byte entries (common.cuh packed_mode); the packed
// and the int2 instantiation are both launched when the host allows packing,
// and the one the device-side decision does not pick exits at once.
template <class T, int G, int CW, int STAGES, int MINB, bool SPLIT, bool BLOCKED,
          bool PACKED = false>
__global__ void __launch_bounds__((CW + 1) * 32, MINB)
    k_bform(const __grid_constant__ CUtensorMap tmap, const int2* __restrict__ lists,
            uint64_t cap, const uint32_t* __restrict__ counts, uint32_t nrows, uint32_t rpc,
            int32_t col0, int32_t ncols, const uint32_t* __restrict__ dyn_ncols,
            uint32_t nkb_total, uint32_t slice_blocks, uint64_t slice_stride,
            T* __restrict__ out, uint64_t ld_out, int vec_ok, const DevStatus* __restrict__ st,
            int group_allow, int ladder) {
  using Gm = Geo<T, G>;
  extern __shared__ unsigned char smem_raw[];
  // 128-byte aligned ring (TMA destination without swizzle); pointer arithmetic
  // on the smem pointer itself keeps the shared address space visible to the
  // compiler.
  unsigned char* base = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + STAGES * Gm::STAGE_BYTES);
  uint64_t* empty = full + STAGES;

  if (status_failed(st)) return;  // validation failed: compute nothing (kernels.hpp:115,144)
  if (group_mode(st, group_allow)) return;  // the small-rep group kernel runs instead
  static_assert(!(PACKED && (SPLIT || BLOCKED)), "packed lists: order-preserving mode only");
  if (packed_mode(st, group_allow) != PACKED) return;  // the other list format's launch runs
  const int32_t tile_c = blockIdx.y * Gm::TILE_N;  // relative to col0
  // the whole CTA beyond the device-decided width: exit (the width is read
  // again at the store rather than kept live across the entry loop)
  if (dyn_ncols && tile_c >= (int32_t)*dyn_ncols) return;

  // %laneid through asm volatile: under register pressure ptxas otherwise
  // re-derives the lane from S2R SR_TID inside the entry loop (a ~30-cycle
  // stall per entry, ncu source view at rep 1).
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  // SPLIT = false (order-preserving mode): one slice, k_lo = 0 at compile time
  // (a runtime k_lo was rematerialised from S2UR SR_CTAID.Z + LDC every entry).
  const uint32_t kb_lo = SPLIT ? blockIdx.z * slice_blocks : 0u;
  const uint32_t kb_hi = min(nkb_total, kb_lo + slice_blocks);
  const uint32_t nkb = kb_hi - kb_lo;
  if (SPLIT) out += blockIdx.z * slice_stride;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == CW) {
    // ---- dedicated TMA producer warp ----
    // (An in-consumer pump that let warp 0 issue the loads between its own
    // entries was measured 2-3x slower: the list-walking warps progress
    // unevenly and the pumping warp gates the ring.)
    if (lane == 0)
      produce<Gm::STAGE_BYTES, Gm::NBOX, Gm::BOX_N, STAGES>(&tmap, base, full, empty,
                                                            col0 + tile_c, kb_lo, nkb);
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
  Total<T, BLOCKED ? G : 1> tot;  // fast mode only
  if constexpr (BLOCKED) tot.zero();
  uint32_t flush_kb = kFlushBlocks;
  const uint32_t k_lo = kb_lo * KB;
  Cursor<STAGES, Gm::STAGE_BYTES> cur(smem_u32(base), smem_u32(full), smem_u32(empty), lane);
  cur.wait();
  // Entry e + 1 = (k, rep) is read by a warp-uniform load (L1 broadcast)
  // while entry e runs, and the list line kListPrefetch entries ahead is
  // prefetched into L1. (Measured against one coalesced 32-entry load per
  // chunk + SHFL broadcasts: equal at cfg5, cfg3 mu = 4 +2.6%, cfg4 +1%, rep
  // 1 -2%; fewer instructions and branches per entry.)
  // (PACKED: one 32-bit word per entry, unpacked only when the entry is taken
  // -- unpacking the prefetched word at once would wait for its load before
  // the current entry's adds: measured +1% at cfg5, +5% at cfg3 mu = 4)
  using Entry = typename std::conditional<PACKED, uint32_t, int2>::type;
  const Entry* __restrict__ lp = reinterpret_cast<const Entry*>(lst);
  auto decode = [](Entry w) -> int2 {
    if constexpr (PACKED) return unpack_entry(w);
    else return w;
  };
  Entry raw = cnt ? __ldg(lp) : Entry{};
  for (uint32_t i = 0; i < cnt; ++i) {
    const int2 e = decode(raw);
    const uint32_t f = i + 1;
    const Entry nraw = f < cnt ? __ldg(lp + f) : Entry{};
    if (f + kListPrefetch < cnt)
      asm volatile("prefetch.global.L1 [%0];" ::"l"(lp + f + kListPrefetch));
    const uint32_t k = (uint32_t)e.x;
    const uint32_t kb = (k - k_lo) / KB;  // block index within the slice
    AFMM_CHECK(st, k >= k_lo && kb < nkb && e.y != 0 &&
                       (i == 0 || (uint32_t)decode(lp[i - 1]).x <= k));
    if constexpr (BLOCKED) {
      if (kb >= flush_kb) {  // the entry starts a new block of the blocked sum
        tot.flush(acc);
        flush_kb = (kb / kFlushBlocks + 1) * kFlushBlocks;
      }
    }
    cur.seek(kb, lane);
    AFMM_CHECK(st, cur.kb_cur == kb && cur.stage_addr >= smem_u32(base) &&
                       cur.stage_addr + (uint32_t)Gm::STAGE_BYTES <=
                           smem_u32(base) + (uint32_t)(STAGES * Gm::STAGE_BYTES) + 32u * 16u);
    if (BLOCKED && ladder) acc.run_ladder(cur.stage_addr + (k % KB) * BOX_BYTES, e.y);
    else acc.run(cur.stage_addr + (k % KB) * BOX_BYTES, e.y);
    raw = nraw;
  }
  cur.drain(nkb, lane);
  if constexpr (BLOCKED) {
    tot.flush(acc);
    tot.to(acc);
  }

  AFMM_CHECK(st, cur.kb_cur == nkb);
  if (dyn_ncols) ncols = (int32_t)*dyn_ncols;
  if (b < nrows) acc.store(out + (uint64_t)b * ld_out, tile_c, ncols, lane, vec_ok != 0);
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

// k rows of fp16 counts per A-form ring stage (the ring keeps 96 k rows:
// 192 KB). A row of cfg3 d1 = 0.1 has ~1 nonzero base per 8 k, so with
// 8-row stages every entry paid a stage hand-off (arrive + wait); 32-row
// stages (3 of them) measured cfg3 d1 = 0.1 mu = 1 / 4 / 16: 1.497 -> 1.341 /
// 3.678 -> 3.569 / 12.66 -> 12.71 ms, cfg4 130.05 -> 130.31 ms (16-row: 1.378
// / 3.577 / 12.62 / 130.03).
#ifndef AFMM_AKB
#define AFMM_AKB 32
#endif
constexpr int AKB = AFMM_AKB;
constexpr int ASTAGES = 96 / AKB;

template <class T>
struct AformGeo {
  static constexpr int CPL = sizeof(T) == 4 ? 32 : 16;  // columns per lane
  static constexpr int TILE = 32 * CPL;                 // columns per CTA
  static constexpr int NBOX = TILE / 256;               // 256-half TMA boxes per k row
  static constexpr int STAGE_BYTES = AKB * TILE * 2;
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
            const uint32_t* __restrict__ counts, uint32_t nrows,
            const uint32_t* __restrict__ dyn_nrows, uint32_t rpc, uint32_t ncols,
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
  // Rows decided on the device (k_choose; the grid covers the whole slab):
  // only the CTA-level exit reads the device count. A per-warp test against
  // it (live across the entry loop) changed the loop's register allocation
  // and cost 13% (dispatch stalls on the predicated FADDs; cfg3 d1 = 0.1
  // mu = 16: 12.7 vs 11.2 ms), so warps past the A rows in the last A-form
  // CTA run with an empty list instead (k_acompact zeroes the B rows'
  // counts) and store zeros that the B part's result overwrites later on
  // the same stream.
  if (dyn_nrows && blockIdx.x * rpc >= *dyn_nrows) return;

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
          tma_load_2d(base + slot * Ag::STAGE_BYTES + bx * AKB * 512, &cmap, &full[slot],
                      tile_c + bx * 256, (int32_t)(i * AKB));
      }
    }
    return;
  }

  // ---- consumers: one Z row per warp ----
  const uint32_t b = warp < rpc ? blockIdx.x * rpc + warp : nrows;
  const bool active = b < nrows;
  const uint32_t q = active ? (row_idx ? row_idx[b] : b) : 0u;  // list / Z row
  AFMM_CHECK(st, !active || !row_idx || q < gridDim.x * rpc);
  const uint32_t cnt = active ? counts[q] : 0u;
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
    const uint32_t kb = k / AKB;
    AFMM_CHECK(st, k < nkb * AKB && kb >= kb_cur && cnt <= cap);
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
                     : "r"(stage_addr + g * AKB * 512 + (k % AKB) * 512));
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

  if (active) {
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
// k_bgroup: the small-rep B-form (every |rep| <= kGroupMaxRep, none negative;
// decided on the device, group_mode()).
//
// k_bform loads a warp's bases from shared memory once per list entry: at rep
// 1 that is 4 bytes of smem per add against the SM's 1 byte per add of smem
// bandwidth per FP add (128 B/clk vs 128 adds/clk), so rep 1-2 rows run at
// 25-45% of the FP-add peak whatever the rest of the kernel does. Here a warp
// owns a GROUP of kGroupRows = 5 B-form rows over 512 columns (40 float2
// accumulators per lane) and walks k densely: per k it loads the 512 staged
// bases once (4 LDS.128 per lane) and applies them to all five rows. The
// rows' rep magnitudes at k arrive as one u16 index (gidx, built by
// k_group_idx_rows / _cols): two `brx.idx` jumps (rows 0-2: 27 targets, rows
// 3-4: 9 targets; tools/gen_jumptable.py) into straight-line blocks of
// FADD2 steps replace five data-dependent rep loops. Each element still gets
// its |rep| sequential adds at its k, k ascending (kernels.hpp:95-104): the
// reference's order, bit for bit. Zero bases add +/-0 as in k_bform.
// Measured (tools/group_proto.cu, n = 4096, reps uniform {0,1,2}): 0.50 of
// the FP-add peak against 0.33 for k_bform; constant rep 1: 0.52 vs 0.23.
// ---------------------------------------------------------------------------
#include "jumptable.inc"

__device__ __forceinline__ void lds128u64(uint32_t addr, unsigned long long& a,
                                          unsigned long long& b) {
  asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "r"(addr));
}

template <int CW, int STAGES>
__global__ void __launch_bounds__((CW + 1) * 32, 1)
    k_bgroup(const __grid_constant__ CUtensorMap tmap, const uint16_t* __restrict__ gidx,
             uint64_t ldg, uint32_t nrows, uint32_t gpc, int32_t ncols,
             const uint32_t* __restrict__ dyn_ncols, uint32_t nkb, float* __restrict__ out,
             uint64_t ld_out, int vec_ok, const DevStatus* __restrict__ st, int allow) {
  using Gm = Geo<float, 4>;  // 512 columns, KB x 2 KB stages
  constexpr int NV = 8;      // float2 operands per lane and row
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + STAGES * Gm::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  if (status_failed(st) || !group_mode(st, allow)) return;
  const int32_t tile_c = blockIdx.y * Gm::TILE_N;
  // (the device-decided width is read again at the store, not kept live
  // across the k loop: see k_aform's row count)
  if (dyn_ncols && tile_c >= (int32_t)*dyn_ncols) return;
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (warp == CW) {
    if (lane == 0)
      produce<Gm::STAGE_BYTES, Gm::NBOX, Gm::BOX_N, STAGES>(&tmap, base, full, empty, tile_c, 0u,
                                                            nkb);
    return;
  }
  const uint32_t ngroups = (nrows + kGroupRows - 1) / kGroupRows;
  const uint32_t g = warp < gpc ? blockIdx.x * gpc + warp : ngroups;
  const bool active = g < ngroups;
  const uint4* __restrict__ gp =
      reinterpret_cast<const uint4*>(gidx + (uint64_t)(active ? g : 0) * ldg);
  unsigned long long acc[kGroupRows * NV];
#pragma unroll
  for (int i = 0; i < kGroupRows * NV; ++i) acc[i] = 0ull;
  Cursor<STAGES, Gm::STAGE_BYTES> cur(smem_u32(base), smem_u32(full), smem_u32(empty), lane);
  cur.wait();
  // one uniform 16-byte load = the group's indices of a whole k block
  uint4 w = active ? __ldg(gp) : make_uint4(0u, 0u, 0u, 0u);
  for (uint32_t kb = 0; kb < nkb; ++kb) {
    const uint4 nw = (active && kb + 1 < nkb) ? __ldg(gp + kb + 1) : make_uint4(0u, 0u, 0u, 0u);
    if (active && kb + 16 < nkb) asm volatile("prefetch.global.L1 [%0];" ::"l"(gp + kb + 16));
    unsigned long long lo = ((unsigned long long)w.y << 32) | w.x;
    unsigned long long hi = ((unsigned long long)w.w << 32) | w.z;
    if ((lo | hi) != 0ull) {
#pragma unroll 1
      for (int kk = 0; kk < KB; ++kk) {
        const uint32_t idx = (uint32_t)lo & 0xffffu;
        lo = (lo >> 16) | (hi << 48);
        hi >>= 16;
        if (idx == 0u) continue;
        AFMM_CHECK(st, (idx & 0xffu) < 27u && (idx >> 8) < 9u);
        const uint32_t ra = cur.stage_addr + (uint32_t)kk * BOX_BYTES;
        unsigned long long b[NV];
#pragma unroll
        for (int q = 0; q < 4; ++q) lds128u64(ra + group_off(q), b[2 * q], b[2 * q + 1]);
        jt_apply<3, 2, NV>(*reinterpret_cast<unsigned long long(*)[3 * NV]>(acc), b, idx & 0xffu);
        jt_apply<2, 2, NV>(*reinterpret_cast<unsigned long long(*)[2 * NV]>(acc + 3 * NV), b,
                           idx >> 8);
      }
    }
    w = nw;
    cur.advance(lane);
    if (kb + 1 < nkb) cur.wait();
  }
  if (!active) return;
  if (dyn_ncols) ncols = (int32_t)*dyn_ncols;
#pragma unroll
  for (int r = 0; r < kGroupRows; ++r) {
    const uint32_t row = g * kGroupRows + r;
    if (row >= nrows) break;
    float* orow = out + (uint64_t)row * ld_out;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int32_t c = tile_c + (q >> 1) * 256 + (q & 1) * 128 + 4 * (int32_t)lane;
      const unsigned long long x = acc[r * NV + 2 * q], y = acc[r * NV + 2 * q + 1];
      const float v[4] = {__uint_as_float((uint32_t)x), __uint_as_float((uint32_t)(x >> 32)),
                          __uint_as_float((uint32_t)y), __uint_as_float((uint32_t)(y >> 32))};
      if (vec_ok && c + 3 < ncols) {
        *reinterpret_cast<float4*>(orow + c) = make_float4(v[0], v[1], v[2], v[3]);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (c + e < ncols) orow[c + e] = v[e];
      }
    }
  }
}

template <class T, int G, int CW, int STAGES, int MINB, bool BLOCKED = false>
cudaError_t launch_ring(BformLaunch& a, T* out, cudaStream_t s) {
  const uint32_t nkb = (a.nk + KB - 1) / KB;
  uint32_t want = a.splits < 1 ? 1 : a.splits;
  if (want > nkb) want = nkb;
  auto kern = want > 1 ? k_bform<T, G, CW, STAGES, MINB, true, BLOCKED>
                       : k_bform<T, G, CW, STAGES, MINB, false, BLOCKED>;
  const size_t smem = ring_smem_bytes<T, G, STAGES>();
  // set on every call: the attribute is per device and costs ~1 us
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  const uint32_t slice_blocks = (nkb + want - 1) / want;
  a.splits = (nkb + slice_blocks - 1) / slice_blocks;
  const bool vec_ok = (a.ld_out * sizeof(T)) % 16 == 0 &&
                      (reinterpret_cast<uintptr_t>(out) % 16) == 0 &&
                      (a.slice_stride * sizeof(T)) % 16 == 0;
  const uint32_t tiles = (a.ncols + Geo<T, G>::TILE_N - 1) / Geo<T, G>::TILE_N;
  const uint32_t rpc = balanced_rows(a.nrows, tiles * a.splits, CW, MINB);
  dim3 grid((a.nrows + rpc - 1) / rpc, tiles, a.splits);
  if constexpr (!BLOCKED) {
    // the packed-list instantiation first (it exits unless the device chose
    // packed lists; the int2 one below exits when it did)
    if ((a.group_allow & kAllowPack) && want == 1) {
      auto pk = k_bform<T, G, CW, STAGES, MINB, false, false, true>;
      e = cudaFuncSetAttribute(pk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      pk<<<grid, (CW + 1) * 32, smem, s>>>(*a.tmap, a.lists, a.cap, a.counts, a.nrows, rpc, a.col0,
                                           a.ncols, a.dyn_ncols, nkb, slice_blocks,
                                           a.slice_stride, out, a.ld_out, vec_ok ? 1 : 0, a.st,
                                           a.group_allow, 0);
      note_launch();
    }
  }
  kern<<<grid, (CW + 1) * 32, smem, s>>>(*a.tmap, a.lists, a.cap, a.counts, a.nrows, rpc, a.col0,
                                         a.ncols, a.dyn_ncols, nkb, slice_blocks, a.slice_stride,
                                         out, a.ld_out, vec_ok ? 1 : 0, a.st, a.group_allow,
                                         BLOCKED ? a.ladder : 0);
  note_launch();
  return cudaGetLastError();
}

}  // namespace

int bform_box_bytes() { return BOX_BYTES; }
int bform_kb() { return KB; }
int aform_kb() { return AKB; }

template <class T>
cudaError_t launch_bform(BformLaunch& a, T* out, cudaStream_t s) {
  switch (a.shape) {
    case kShapeWide:
      // 1024 fp32 / 512 fp64 columns x 16 rows, 16 consumers + producer,
      // 6-stage ring (192 KB), 1 CTA per SM, 83 registers. Measured against 8
      // rows x 3 stages x 2 CTAs per SM: cfg5 1810 -> 1802 ms, cfg2 0.307 ->
      // 0.285 ms, cfg3 and cfg4 0.3-2% faster -- the deeper ring lets warps
      // drift 5 k blocks apart instead of 2 (consumers had waited on a stage
      // 6.5% of the time, ncu).
      return launch_ring<T, 8, kWideRows, 6, kWideCtasPerSm>(a, out, s);
    case kShapeSmall:  // 256 fp32 / 128 fp64 columns x 4 rows, up to 8 CTAs per SM
      return launch_ring<T, 2, 4, 3, 8>(a, out, s);
    case kShapeFast:  // fast mode: 512 fp32 / 256 fp64 columns x 16 rows, fp64 blocked totals
      return launch_ring<T, 4, 16, 12, 1, true>(a, out, s);
    default:  // narrow: 512 fp32 / 256 fp64 columns x 16 rows, 2 CTAs per SM
      return launch_ring<T, 4, 16, 6, 2>(a, out, s);
  }
}

template cudaError_t launch_bform<float>(BformLaunch&, float*, cudaStream_t);
template cudaError_t launch_bform<double>(BformLaunch&, double*, cudaStream_t);

cudaError_t launch_bgroup(const CUtensorMap* tmap, const uint16_t* gidx, uint64_t ldg,
                          uint32_t nrows, int32_t ncols, const uint32_t* dyn_ncols, uint32_t nk,
                          float* out, uint64_t ld_out, const DevStatus* st, int allow,
                          cudaStream_t s) {
  // 15 consumer warps (121 registers: the 16-warp CTA's 128-register budget)
  // + the TMA warp, 12-stage ring (192 KB), 1 CTA per SM
  constexpr int CW = kGroupWarps, STAGES = 12;
  using Gm = Geo<float, 4>;
  auto kern = k_bgroup<CW, STAGES>;
  const size_t smem = ring_smem_bytes<float, 4, STAGES>();
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  const uint32_t nkb = (nk + KB - 1) / KB;
  const uint32_t tiles = (uint32_t)((ncols + Gm::TILE_N - 1) / Gm::TILE_N);
  const uint32_t ngroups = (nrows + kGroupRows - 1) / kGroupRows;
  if (tiles == 0 || ngroups == 0) return cudaSuccess;
  const uint32_t gpc = balanced_rows(ngroups, tiles, CW, 1);
  const bool vec_ok = (ld_out * sizeof(float)) % 16 == 0 && (reinterpret_cast<uintptr_t>(out) % 16) == 0;
  dim3 grid((ngroups + gpc - 1) / gpc, tiles);
  kern<<<grid, (CW + 1) * 32, smem, s>>>(*tmap, gidx, ldg, nrows, gpc, ncols, dyn_ncols, nkb, out,
                                         ld_out, vec_ok ? 1 : 0, st, allow);
  note_launch();
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_aform(const CUtensorMap* cmap, const typename AEntry<T>::type* lists,
                         uint64_t cap, const uint32_t* counts, uint32_t nrows,
                         const uint32_t* dyn_nrows, uint32_t ncols, uint32_t nk,
                         const uint16_t* rmax, T* out, uint64_t ld_out, const uint32_t* row_idx,
                         const DevStatus* st, cudaStream_t s) {
  using Ag = AformGeo<T>;
  static_assert(Ag::TILE == (int)aform_tile_cols<T>(), "A-form tile width");
  // 16 rows x 12 stages x 1 CTA/SM: 4-5% faster than 8 rows x 6 stages x 2
  // CTAs/SM on cfg3 d1 = 0.1 (tools/exp_time.py --aform)
  constexpr int CW = kAformRows, STAGES = ASTAGES, MINB = kAformCtasPerSm;
  auto kern = k_aform<T, CW, STAGES, MINB>;
  const size_t smem = 128 + (size_t)STAGES * Ag::STAGE_BYTES + 2 * STAGES * sizeof(uint64_t);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  const uint32_t nkb = (nk + AKB - 1) / AKB;
  const uint32_t tiles = (ncols + Ag::TILE - 1) / Ag::TILE;
  const uint32_t rpc = balanced_rows(nrows, tiles, CW, MINB);
  dim3 grid((nrows + rpc - 1) / rpc, tiles);
  kern<<<grid, (CW + 1) * 32, smem, s>>>(*cmap, lists, cap, counts, nrows, dyn_nrows, rpc, ncols,
                                         nkb, rmax, tiles, out, ld_out, row_idx, st);
  note_launch();
  return cudaGetLastError();
}

template cudaError_t launch_aform<float>(const CUtensorMap*, const int2*, uint64_t,
                                         const uint32_t*, uint32_t, const uint32_t*, uint32_t,
                                         uint32_t, const uint16_t*, float*, uint64_t,
                                         const uint32_t*, const DevStatus*, cudaStream_t);
template cudaError_t launch_aform<double>(const CUtensorMap*, const int4*, uint64_t,
                                          const uint32_t*, uint32_t, const uint32_t*, uint32_t,
                                          uint32_t, const uint16_t*, double*, uint64_t,
                                          const uint32_t*, const DevStatus*, cudaStream_t);

}  // namespace afmm_dev
