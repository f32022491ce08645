// generate.cu -- device-side seeded generation: the
// reference's afmm::generate (/root/reference/proj/include/afmm/random.hpp:
// 111-129) on the GPU, bit-identical, written straight into device memory.
//
// The reference walks the n^2 entries in row-major order with ONE
// std::mt19937_64 stream: each entry draws a Bernoulli variate
// (uniform01 >= density -> zero), and a nonzero entry then draws its value
// from the same stream (IntegerValued: 1 + uniform_below(2 mu' - 1), a
// rejection loop; RealValued: low + (high - low) * uniform01). Which draw
// belongs to which entry is data dependent, so the device pipeline is:
//
//   k_mt_jump       the stream's start offsets: CTA c of a chunk generates
//                   the stretch [c L, (c+1) L) of the chunk, and its start
//                   window comes from a radix-4 tree of jump-aheads (the
//                   window at k + J is a GF(2) convolution of the words after
//                   k with x^J mod phi, mt64jump.h) -- log4(CTAs) levels.
//   k_mt_gen        the raw 64-bit stream, one CTA per stretch: MT19937-64's
//                   recurrence w[k + 312] = f(w[k], w[k + 1], w[k + 156])
//                   makes 156 words computable at once, so a twist is two
//                   parallel half-steps over a 624-word smem ring; tempered
//                   outputs are stored in stream order.
//   k_gen_reduce    every draw is a transition of a two-state automaton
//                   (B: the next draw is an entry's Bernoulli variate, V: a
//                   value variate); per block of draws the composed
//                   transition for both entry states plus the number of
//                   B draws (= entries started), reduced by a warp/block scan
//                   (the composition is associative, not commutative).
//   k_gen_scan      one CTA: exclusive scan of the block transitions from the
//                   chunk's carry (state, entries) -> each block's entry
//                   state and first entry index; the carry moves on.
//   k_gen_write     each block re-derives its draws' states and writes the
//                   value of every nonzero entry at its accepted value draw
//                   (the output was zeroed: zero entries need no store).
//
// Chunks of draws repeat until n^2 entries are complete; each entry gets
// exactly the draws the reference gives it, so the matrix is bit-identical
// (tests/test_generate_gpu.py against the oracle's restatement, itself pinned
// to the reference by tests/test_oracle.py).
#include "common.cuh"
#include "kernels.h"

namespace afmm_dev {

namespace {

constexpr int MT_N = 312, MT_M = 156;
constexpr uint64_t MT_A = 0xB5026F5AA96619E9ull;
constexpr uint64_t MT_UPPER = 0xFFFFFFFF80000000ull, MT_LOWER = 0x7FFFFFFFull;
constexpr int GEN_THREADS = 256, GEN_PER_THREAD = 16;
constexpr int GEN_BLOCK = GEN_THREADS * GEN_PER_THREAD;  // draws per scan block

__device__ __forceinline__ uint64_t mt_mix(uint64_t a, uint64_t b, uint64_t c) {
  const uint64_t x = (a & MT_UPPER) | (b & MT_LOWER);
  return c ^ (x >> 1) ^ ((x & 1ull) ? MT_A : 0ull);
}

__device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

// The raw stream, one CTA per stretch of `twists` x 312 outputs: CTA c starts
// from windows[c] (the window at output offset c * twists * 312, placed there
// by k_mt_jump) and stores its outputs in stream order; the last CTA leaves
// the window that follows the chunk in *end_window. Ring slot of stream word
// k: k % 624; the current generation sits at one half while the next one is
// built in the other: w[k + 312] = f(w[k], w[k + 1], w[k + 156]) makes 156
// words computable at once, so a twist is two parallel half-steps.
__global__ void __launch_bounds__(MT_M) k_mt_gen(const uint64_t* __restrict__ windows,
                                                uint64_t* __restrict__ out, uint32_t twists,
                                                uint64_t* __restrict__ end_window) {
  __shared__ uint64_t ring[2 * MT_N];
  const uint32_t i = threadIdx.x;  // 0..155
  const uint64_t* w0 = windows + (uint64_t)blockIdx.x * MT_N;
  ring[i] = w0[i];
  ring[i + MT_M] = w0[i + MT_M];
  __syncthreads();
  uint64_t* o = out + (uint64_t)blockIdx.x * twists * MT_N;
  uint32_t cur = 0;  // ring offset of the current generation
  for (uint32_t t = 0; t < twists; ++t, o += MT_N) {
    const uint32_t nxt = cur ^ MT_N;
    o[i] = mt_temper(ring[cur + i]);
    o[i + MT_M] = mt_temper(ring[cur + i + MT_M]);
    // first half: w'[i] = f(w[i], w[i+1], w[i+156]) -- all old words
    ring[nxt + i] = mt_mix(ring[cur + i], ring[cur + i + 1], ring[cur + i + MT_M]);
    __syncthreads();
    // second half: w'[i+156] = f(w[i+156], w[i+157], w'[i]); w[312] is w'[0]
    const uint32_t j = i + MT_M;
    const uint64_t b = j + 1 < MT_N ? ring[cur + j + 1] : ring[nxt];
    ring[nxt + j] = mt_mix(ring[cur + j], b, ring[nxt + i]);
    __syncthreads();
    cur = nxt;
  }
  if (end_window && blockIdx.x == gridDim.x - 1) {
    end_window[i] = ring[cur + i];
    end_window[i + MT_M] = ring[cur + i + MT_M];
  }
}

// Jump-ahead (mt64jump.h): the window at offset k + J is the XOR of the
// windows at offsets k + i over the set coefficients c_i of x^J mod phi. One
// CTA per jump of the tree level with stride S (radix 4): block t moves
// windows[t / 3] by (t % 3 + 1) * S stretches with polys[t % 3]. The CTA
// generates the kD + 311 words after its source window into shared memory
// (64 twists), then each warp takes every 32nd coefficient word and, for each
// set bit i, XORs words i .. i + 311 into its lanes' accumulators (lane l
// holds w = l + 32 r); the warps' partial windows are XOR-reduced at the end.
constexpr int JUMP_THREADS = 1024;
constexpr int JUMP_TWISTS = 64;  // 65 x 312 = 20280 >= kD + 311 words
constexpr size_t kJumpSmem = (size_t)(JUMP_TWISTS + 1) * MT_N * sizeof(uint64_t);

__global__ void __launch_bounds__(JUMP_THREADS, 1)
    k_mt_jump(uint64_t* __restrict__ windows, const uint64_t* __restrict__ polys,
              uint32_t stride, uint32_t count) {
  extern __shared__ uint64_t v[];
  const uint32_t src = blockIdx.x / 3, a = blockIdx.x % 3 + 1;
  const uint32_t dst = src + a * stride;
  if (dst >= count) return;  // the whole CTA: no barrier is skipped by part of it
  const uint64_t* __restrict__ poly = polys + (a - 1) * MT_N;
  const uint32_t tid = threadIdx.x;
  if (tid < MT_N) v[tid] = windows[(uint64_t)src * MT_N + tid];
  __syncthreads();
  for (int t = 0; t < JUMP_TWISTS; ++t) {
    uint64_t* g = v + t * MT_N;
    if (tid < MT_M) g[MT_N + tid] = mt_mix(g[tid], g[tid + 1], g[tid + MT_M]);
    __syncthreads();
    if (tid < MT_M) {
      const uint32_t j = tid + MT_M;
      g[MT_N + j] = mt_mix(g[j], g[j + 1], g[MT_N + tid]);
    }
    __syncthreads();
  }
  const uint32_t lane = tid & 31, warp = tid >> 5;
  uint64_t acc[10];
#pragma unroll
  for (int r = 0; r < 10; ++r) acc[r] = 0;
  for (uint32_t q = warp; q < MT_N; q += 32) {
    uint64_t m = __ldg(poly + q);
    while (m) {
      const uint32_t b = __ffsll((long long)m) - 1;
      m &= m - 1;
      const uint64_t* p = v + q * 64 + b + lane;
#pragma unroll
      for (int r = 0; r < 9; ++r) acc[r] ^= p[32 * r];
      if (lane < MT_N - 288) acc[9] ^= p[288];
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t w = lane + 32 * r;
    if (w < MT_N) v[warp * MT_N + w] = acc[r];
  }
  __syncthreads();
  if (tid < MT_N) {
    uint64_t x = 0;
#pragma unroll 8
    for (int wp = 0; wp < JUMP_THREADS / 32; ++wp) x ^= v[wp * MT_N + tid];
    windows[(uint64_t)dst * MT_N + tid] = x;
  }
}

// One draw as an automaton transition (random.hpp:92-104, 118-127).
struct GenParams {
  double density, low, high;
  uint64_t range, limit;  // IntegerValued: 2 mu' - 1 and the rejection limit
  int integer;
};

// Composed transitions of a run of draws for both entry states: exit state
// (bit 0: entering in B, bit 1: entering in V) and B draws seen (= entries
// started) for each.
struct Seg {
  uint32_t exits;
  uint32_t cb, cv;
};

__device__ __forceinline__ double uniform01(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }

__device__ __forceinline__ Seg draw_seg(uint64_t x, const GenParams& p) {
  Seg s;
  const uint32_t from_b = uniform01(x) >= p.density ? 0u : 1u;  // nonzero -> a value follows
  const uint32_t from_v = (p.integer && x >= p.limit) ? 1u : 0u;  // rejected -> draw again
  s.exits = from_b | (from_v << 1);
  s.cb = 1u;
  s.cv = 0u;
  return s;
}

// a then b
__device__ __forceinline__ Seg compose(const Seg& a, const Seg& b) {
  Seg r;
  const uint32_t mb = a.exits & 1u, mv = (a.exits >> 1) & 1u;
  r.exits = ((b.exits >> mb) & 1u) | (((b.exits >> mv) & 1u) << 1);
  r.cb = a.cb + (mb ? b.cv : b.cb);
  r.cv = a.cv + (mv ? b.cv : b.cb);
  return r;
}

__device__ __forceinline__ Seg identity_seg() {
  Seg s;
  s.exits = 2u;  // B -> B, V -> V
  s.cb = s.cv = 0u;
  return s;
}

__device__ __forceinline__ Seg shfl_up_seg(const Seg& s, int d) {
  Seg r;
  r.exits = __shfl_up_sync(0xffffffffu, s.exits, d);
  r.cb = __shfl_up_sync(0xffffffffu, s.cb, d);
  r.cv = __shfl_up_sync(0xffffffffu, s.cv, d);
  return r;
}

// Inclusive block scan of the threads' segments in thread order; returns this
// thread's EXCLUSIVE prefix and (via *total) the block's composition.
__device__ Seg block_exclusive(const Seg& mine, Seg* total) {
  __shared__ Seg warp_tot[GEN_THREADS / 32];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  Seg inc = mine;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const Seg up = shfl_up_seg(inc, d);
    if ((int)lane >= d) inc = compose(up, inc);
  }
  if (lane == 31) warp_tot[wid] = inc;
  __syncthreads();
  Seg before = identity_seg();
  for (uint32_t w = 0; w < wid; ++w) before = compose(before, warp_tot[w]);
  Seg t = identity_seg();
  for (uint32_t w = 0; w < GEN_THREADS / 32; ++w) t = compose(t, warp_tot[w]);
  *total = t;
  const Seg up = shfl_up_seg(inc, 1);
  return compose(before, lane ? up : identity_seg());
}

__device__ __forceinline__ Seg thread_seg(const uint64_t* __restrict__ draws, uint64_t base,
                                          uint64_t ndraws, const GenParams& p, uint64_t* x) {
  Seg s = identity_seg();
#pragma unroll
  for (int e = 0; e < GEN_PER_THREAD; ++e) {
    const uint64_t k = base + e;
    x[e] = k < ndraws ? draws[k] : 0ull;
    if (k < ndraws) s = compose(s, draw_seg(x[e], p));
  }
  return s;
}

__global__ void __launch_bounds__(GEN_THREADS)
    k_gen_reduce(const uint64_t* __restrict__ draws, uint64_t ndraws, GenParams p,
                 Seg* __restrict__ block_segs) {
  uint64_t x[GEN_PER_THREAD];
  const uint64_t base = (uint64_t)blockIdx.x * GEN_BLOCK + threadIdx.x * GEN_PER_THREAD;
  const Seg mine = thread_seg(draws, base, ndraws, p, x);
  Seg total;
  block_exclusive(mine, &total);
  if (threadIdx.x == 0) block_segs[blockIdx.x] = total;
}

// The chunk's carry in: the automaton state and the entries started so far.
struct GenCarry {
  uint32_t state;  // 0 = B, 1 = V
  uint32_t pad;
  unsigned long long entries;
};

// One CTA: each block's entry state and first entry index, then the carry.
__global__ void __launch_bounds__(GEN_THREADS)
    k_gen_scan(const Seg* __restrict__ block_segs, uint32_t nblocks, GenCarry* carry,
               uint32_t* __restrict__ block_state, unsigned long long* __restrict__ block_entries) {
  const uint32_t per = (nblocks + GEN_THREADS - 1) / GEN_THREADS;
  const uint32_t b0 = min(threadIdx.x * per, nblocks), b1 = min(b0 + per, nblocks);
  Seg mine = identity_seg();
  for (uint32_t b = b0; b < b1; ++b) mine = compose(mine, block_segs[b]);
  Seg total;
  const Seg before = block_exclusive(mine, &total);
  const GenCarry c = *carry;
  uint32_t s = c.state;
  unsigned long long ent = c.entries + (s ? before.cv : before.cb);
  s = (before.exits >> s) & 1u;
  for (uint32_t b = b0; b < b1; ++b) {
    block_state[b] = s;
    block_entries[b] = ent;
    const Seg& g = block_segs[b];
    ent += s ? g.cv : g.cb;
    s = (g.exits >> s) & 1u;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    GenCarry o;
    o.state = (total.exits >> c.state) & 1u;
    o.pad = 0;
    o.entries = c.entries + (c.state ? total.cv : total.cb);
    *carry = o;
  }
}

template <class T>
__global__ void __launch_bounds__(GEN_THREADS)
    k_gen_write(const uint64_t* __restrict__ draws, uint64_t ndraws, GenParams p,
                const uint32_t* __restrict__ block_state,
                const unsigned long long* __restrict__ block_entries, uint64_t n, T* __restrict__ out,
                uint64_t ld) {
  uint64_t x[GEN_PER_THREAD];
  const uint64_t base = (uint64_t)blockIdx.x * GEN_BLOCK + threadIdx.x * GEN_PER_THREAD;
  const Seg mine = thread_seg(draws, base, ndraws, p, x);
  Seg total;
  const Seg before = block_exclusive(mine, &total);
  uint32_t s = block_state[blockIdx.x];
  unsigned long long ent = block_entries[blockIdx.x] + (s ? before.cv : before.cb);
  s = (before.exits >> s) & 1u;
  const unsigned long long nn = (unsigned long long)n * n;
#pragma unroll
  for (int e = 0; e < GEN_PER_THREAD; ++e) {
    if (base + e >= ndraws) break;
    const Seg d = draw_seg(x[e], p);
    if (s == 1u && !((d.exits >> 1) & 1u)) {
      // an accepted value draw: the value of entry ent - 1 (random.hpp:121-126)
      const unsigned long long idx = ent - 1;
      if (idx < nn) {
        double v;
        if (p.integer) v = (double)(1ull + x[e] % p.range);
        else v = p.low + (p.high - p.low) * uniform01(x[e]);
        out[(idx / n) * ld + idx % n] = (T)v;
      }
    }
    ent += s ? d.cv : d.cb;
    s = (d.exits >> s) & 1u;
  }
}

}  // namespace

size_t gen_block_count(uint64_t ndraws) { return (ndraws + GEN_BLOCK - 1) / GEN_BLOCK; }
size_t gen_scratch_bytes(uint64_t ndraws) {
  const size_t nb = gen_block_count(ndraws);
  return nb * (sizeof(Seg) + sizeof(uint32_t) + sizeof(unsigned long long)) + 64;
}
size_t gen_carry_bytes() { return sizeof(GenCarry); }

// One chunk: `ctas` stretches of `twists` x 312 draws of the stream, the
// first starting at windows[0]; the jump tree fills windows[1 .. ctas) (levels
// of stride 1, 4, 16, ...; polys: 3 x 312 words per level), the generators
// write the draws and the window after the chunk to end_window; then the
// entries the draws complete are written to out. carry: device GenCarry,
// updated; scratch: gen_scratch_bytes(ctas * twists * 312).
template <class T>
cudaError_t launch_generate_chunk(const GenSpecDev& spec, uint64_t* windows,
                                  const uint64_t* polys, uint32_t ctas, uint32_t twists,
                                  uint64_t* end_window, uint64_t* draws, void* scratch, void* carry,
                                  T* out, uint64_t ld, cudaStream_t s) {
  const uint64_t ndraws = (uint64_t)ctas * twists * MT_N;
  if (ctas > 1) {
    static bool attr = false;  // idempotent; a race only repeats the call
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(k_mt_jump, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)kJumpSmem);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    uint32_t level = 0;
    for (uint64_t stride = 1; stride < ctas; stride *= 4, ++level) {
      const uint32_t jumps = (uint32_t)std::min<uint64_t>(stride, ctas) * 3;
      k_mt_jump<<<jumps, JUMP_THREADS, kJumpSmem, s>>>(windows, polys + (size_t)level * 3 * MT_N,
                                                       (uint32_t)stride, ctas);
      note_launch();
    }
  }
  k_mt_gen<<<ctas, MT_M, 0, s>>>(windows, draws, twists, end_window);
  note_launch();
  GenParams p;
  p.density = spec.density;
  p.low = spec.low;
  p.high = spec.high;
  p.integer = spec.integer;
  p.range = spec.range;
  p.limit = spec.limit;
  const uint32_t nb = (uint32_t)gen_block_count(ndraws);
  Seg* segs = static_cast<Seg*>(scratch);
  uint32_t* bstate = reinterpret_cast<uint32_t*>(segs + nb);
  unsigned long long* bent =
      reinterpret_cast<unsigned long long*>(((reinterpret_cast<uintptr_t>(bstate + nb) + 15) & ~uintptr_t(15)));
  k_gen_reduce<<<nb, GEN_THREADS, 0, s>>>(draws, ndraws, p, segs);
  note_launch();
  k_gen_scan<<<1, GEN_THREADS, 0, s>>>(segs, nb, static_cast<GenCarry*>(carry), bstate, bent);
  note_launch();
  k_gen_write<T><<<nb, GEN_THREADS, 0, s>>>(draws, ndraws, p, bstate, bent, spec.n, out, ld);
  note_launch();
  return cudaGetLastError();
}

template cudaError_t launch_generate_chunk<double>(const GenSpecDev&, uint64_t*, const uint64_t*,
                                                   uint32_t, uint32_t, uint64_t*, uint64_t*, void*,
                                                   void*, double*, uint64_t, cudaStream_t);
template cudaError_t launch_generate_chunk<float>(const GenSpecDev&, uint64_t*, const uint64_t*,
                                                  uint32_t, uint32_t, uint64_t*, uint64_t*, void*,
                                                  void*, float*, uint64_t, cudaStream_t);

}  // namespace afmm_dev
