// runtime.cu -- host runtime behind the C ABI (include/afmm_b200.h).
//
// Owns contexts (device + stream + grow-only workspace), builds the TMA
// tensor maps, sequences prepass -> repeated-addition kernel(s) -> epilogue on
// one stream, replays repeated device calls as CUDA graphs, shards the
// reference-facing call over several devices, and maps device-side
// validation results to the reference's error contract (kernels.hpp:15-43,
// matrix.hpp:25-36, 54-57). No element of the product is computed on the
// host and there is no CPU fallback: the Case A kernel choice is made on the
// device (k_choose), so no call waits on the host between its kernels.
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cinttypes>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <new>
#include <thread>
#include <vector>

#include "../../include/afmm_b200.h"
#include "kernels.h"
#include "mt64jump.h"

using afmm_dev::DevStatus;

namespace afmm_dev {
static std::atomic<uint64_t> g_launches{0};
// Launch errors (a bad configuration, too much shared memory) are recorded
// right after each launch: the runtime's last-error state does not survive a
// later successful call -- a cudaFuncSetAttribute resets it (measured: a
// k_choose launch failure was wiped by the next kernel's attribute call and
// the product returned untouched output) -- so checking once at the end of
// the enqueue is not enough. Per host thread (the multi-device shards enqueue
// from their own threads).
static thread_local cudaError_t t_launch_err = cudaSuccess;
void note_launch() {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess && t_launch_err == cudaSuccess) t_launch_err = e;
}
// The first launch error since the last call (and clear it).
cudaError_t take_launch_error() {
  const cudaError_t e = t_launch_err;
  t_launch_err = cudaSuccess;
  return e;
}
}  // namespace afmm_dev

namespace {

constexpr uint64_t kNone = ~0ull;

// AFMM_BFORM forces one repeated-addition kernel shape or Case A form (all are
// bit-identical; tests/test_gpu_parity.py runs each). Default: automatic (the
// shape from the problem size, the Case A form from the device-side model).
enum Variant {
  kAuto = -1,
  kNarrow = 0,  // 512 fp32 / 256 fp64 columns, 2 CTAs per SM
  kWide = 1,    // 1024 / 512 columns, 1 CTA per SM
  kSmall = 2,   // 256 / 128 columns x 4 rows
  kAForm = 8,   // Case A: every row in the A-form
  kHybrid = 9,  // Case A: the best A-form / B-form row split, forced
};

int variant_from_env() {
  const char* v = std::getenv("AFMM_BFORM");
  if (!v) return kAuto;
  static const struct {
    const char* name;
    int variant;
  } names[] = {{"ring", kNarrow}, {"narrow", kNarrow}, {"wide", kWide},
               {"small", kSmall}, {"aform", kAForm},    {"hybrid", kHybrid}};
  for (const auto& e : names)
    if (std::strcmp(v, e.name) == 0) return e.variant;
  return kAuto;
}

// AFMM_BFORM=nogroup: automatic choices, but never the small-rep group kernel
// (k_bgroup) -- for comparisons; a forced k_bform shape also excludes it.
bool group_off_from_env() {
  const char* v = std::getenv("AFMM_BFORM");
  return v && std::strcmp(v, "nogroup") == 0;
}

// AFMM_BFORM=nopack: automatic choices, but the rep lists stay int2 {k, rep}
// (never the packed 4-byte entries) -- for comparisons.
bool pack_off_from_env() {
  const char* v = std::getenv("AFMM_BFORM");
  return v && std::strcmp(v, "nopack") == 0;
}

inline uint64_t round_up(uint64_t v, uint64_t m) { return (v + m - 1) / m * m; }

int sm_count(int device) {
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess ||
      sms <= 0) {
    cudaGetLastError();
    sms = 148;
  }
  return sms;
}

// Guard bands of the checked build: every workspace allocation is framed by
// kGuard bytes of a known pattern, verified after each product (an
// out-of-bounds write by a library kernel into a neighbouring allocation).
#ifdef AFMM_CHECKED
constexpr size_t kGuard = 4096;
#else
constexpr size_t kGuard = 0;
#endif
constexpr unsigned char kGuardByte = 0xA5;

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  uint64_t* gen = nullptr;  // the owning context's buffer generation (bumped on reallocation)
  // grow-only; contents are not preserved
  cudaError_t ensure(size_t want) {
    if (want <= bytes) return cudaSuccess;
    if (gen) ++*gen;  // captured graphs hold the old addresses
    release();
    want = std::max<size_t>(want, 256);
    void* raw = nullptr;
    cudaError_t e = cudaMalloc(&raw, want + 2 * kGuard);
    if (e != cudaSuccess) return e;
    if (kGuard) {
      e = cudaMemset(raw, kGuardByte, kGuard);
      if (e == cudaSuccess) e = cudaMemset(static_cast<char*>(raw) + kGuard + want, kGuardByte, kGuard);
      if (e != cudaSuccess) {
        cudaFree(raw);
        return e;
      }
    }
    p = static_cast<char*>(raw) + kGuard;
    bytes = want;
    return cudaSuccess;
  }
  void release() {
    if (p) cudaFree(static_cast<char*>(p) - kGuard);  // implicit device sync
    p = nullptr;
    bytes = 0;
  }
#ifdef AFMM_CHECKED
  // checked build: are both guard bands intact?
  bool guards_intact() const {
    if (!kGuard || !p) return true;
    std::vector<unsigned char> g(2 * kGuard);
    if (cudaMemcpy(g.data(), static_cast<char*>(p) - kGuard, kGuard, cudaMemcpyDeviceToHost) !=
            cudaSuccess ||
        cudaMemcpy(g.data() + kGuard, static_cast<char*>(p) + bytes, kGuard,
                   cudaMemcpyDeviceToHost) != cudaSuccess)
      return false;
    for (unsigned char b : g)
      if (b != kGuardByte) return false;
    return true;
  }
#endif

  template <class U>
  U* as() const {
    return static_cast<U*>(p);
  }
};

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

template <class T>
bool make_tmap(CUtensorMap* map, const T* base, uint64_t rows, uint64_t cols, uint64_t ld) {
  auto fn = get_encode_fn();
  if (!fn) return false;
  const cuuint64_t gdim[2] = {cols, rows};
  const cuuint64_t gstride[1] = {ld * sizeof(T)};
  const cuuint32_t box[2] = {(cuuint32_t)(afmm_dev::bform_box_bytes() / sizeof(T)),
                             (cuuint32_t)afmm_dev::bform_kb()};
  const cuuint32_t estride[2] = {1, 1};
  const CUtensorMapDataType dt =
      sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  CUresult r = fn(map, dt, 2, const_cast<T*>(base), gdim, gstride, box, estride,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// fp16 rep counts for k_aform: box = 256 columns x KB rows, out-of-range
// columns read as 0 (no adds).
bool make_count_tmap(CUtensorMap* map, const __half* cnt, uint64_t rows, uint64_t cols,
                     uint64_t ldc) {
  auto fn = get_encode_fn();
  if (!fn) return false;
  const cuuint64_t gdim[2] = {cols, rows};
  const cuuint64_t gstride[1] = {ldc * sizeof(__half)};
  const cuuint32_t box[2] = {256, (cuuint32_t)afmm_dev::aform_kb()};
  const cuuint32_t estride[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(cnt), gdim,
                  gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// One product call, as enqueued (kept for error decoding and the
// list-overflow re-run).
struct Call {
  int which = 0, dtype = 0, mode = 0, split_k = 0;
  const void* lhs = nullptr;
  const void* rhs = nullptr;
  uint64_t n = 0, ld = 0;
  void* out = nullptr;
  uint64_t ld_out = 0, r0 = 0, r1 = 0;
  bool prevalidated = false;  // multi-device: validation and the per-k vector done already
  bool have_counts = false;   // multi-device Case A: fp16 counts and statistics done already
  bool check_finite = true;   // false: AFMM_FLAG_KERNEL_SEMANTICS (no DenseMatrix ctor check)
  // prevalidated calls: the rep statistics of the whole operands (DevStatus
  // rep_max / rep_neg, merged over the shards) for the group-kernel choice
  uint32_t rep_max = 0, rep_neg = 0;
};


// Pageable host buffers (a std::vector-backed DenseMatrix, a numpy array): a
// plain cudaMemcpy2DAsync stages them through the driver's own bounce buffer
// on the calling thread at ~12 GB/s (measured: cfg5 with pageable operands
// 2058 ms against 1842 ms with page-locked ones; 1894 ms through this
// pipeline, cfg4 195 -> 157 ms, n = 4096 23.5 -> 12.8 ms). The stager runs the same
// copy as a pipeline: kWorkers host threads each pack their chunks of rows
// into their own page-locked slots (two per worker, so the memcpy of one
// chunk overlaps the DMA of the previous one) and issue the DMAs on their own
// streams. Only large copies come here; small ones keep the plain call.
struct HostStager {
  static constexpr int kMaxWorkers = 8, kSlots = 2;
  static constexpr size_t kSlotBytes = 8u << 20;
  static constexpr size_t kMinBytes = 16u << 20;  // below this the plain copy is as fast
  int workers = 6;
  int device = -1;
  void* slot[kMaxWorkers][kSlots] = {};
  cudaEvent_t ev[kMaxWorkers][kSlots] = {};
  cudaStream_t st[kMaxWorkers] = {};
  cudaEvent_t done[kMaxWorkers] = {};

  // (AFMM_STAGE_WORKERS is read on every call, so a test can vary it)
  cudaError_t ensure(int dev) {
    if (device != dev && device >= 0) release();
    // 4 -> 6 workers: cfg5 1910 -> 1894 ms, 8 no faster (profiles/r02/pageable);
    // at most half the host's hardware threads
    const unsigned hw = std::thread::hardware_concurrency();
    int want = hw == 0 ? 6 : (int)std::min<unsigned>(6u, std::max<unsigned>(2u, hw / 2));
    if (const char* v = std::getenv("AFMM_STAGE_WORKERS")) {
      const int w = std::atoi(v);
      if (w >= 1 && w <= kMaxWorkers) want = w;
    }
    for (int w = 0; w < want; ++w) {
      if (st[w]) continue;
      cudaError_t e = cudaStreamCreateWithFlags(&st[w], cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&done[w], cudaEventDisableTiming);
      for (int k = 0; k < kSlots && e == cudaSuccess; ++k) {
        e = cudaHostAlloc(&slot[w][k], kSlotBytes, cudaHostAllocDefault);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev[w][k], cudaEventDisableTiming);
      }
      if (e != cudaSuccess) {
        release();
        return e;
      }
    }
    workers = want;
    device = dev;
    return cudaSuccess;
  }
  void release() {
    for (int w = 0; w < kMaxWorkers; ++w) {
      for (int k = 0; k < kSlots; ++k) {
        if (slot[w][k]) cudaFreeHost(slot[w][k]);
        if (ev[w][k]) cudaEventDestroy(ev[w][k]);
        slot[w][k] = nullptr;
        ev[w][k] = nullptr;
      }
      if (st[w]) cudaStreamDestroy(st[w]);
      if (done[w]) cudaEventDestroy(done[w]);
      st[w] = nullptr;
      done[w] = nullptr;
    }
    device = -1;
  }
  // Is p ordinary pageable host memory (not page-locked, not managed)?
  static bool pageable(const void* p) {
    cudaPointerAttributes attr{};
    const cudaError_t e = cudaPointerGetAttributes(&attr, p);
    cudaGetLastError();
    return e == cudaSuccess && attr.type == cudaMemoryTypeUnregistered;
  }
  static bool wants(const void* host, size_t width, size_t height) {
    return width > 0 && width <= kSlotBytes && width * height >= kMinBytes && pageable(host);
  }
  // `height` rows of `width` bytes between a pageable host matrix and device
  // memory. Host to device: returns once every DMA is enqueued; `join` (the
  // compute stream) waits for them on the device. Device to host: the caller
  // has synchronised the producer of `src`; returns when `dst` is complete.
  cudaError_t copy(bool h2d, void* dst, size_t dpitch, const void* src, size_t spitch,
                   size_t width, size_t height, cudaStream_t join) {
    const size_t rpc = std::max<size_t>(1, kSlotBytes / width);
    const size_t nchunks = (height + rpc - 1) / rpc;
    const int W = (int)std::min<size_t>((size_t)workers, nchunks);
    std::vector<cudaError_t> status((size_t)W, cudaSuccess);
    auto pack = [&](char* to, size_t tpitch, const char* from, size_t fpitch, size_t rows) {
      if (tpitch == width && fpitch == width) {
        std::memcpy(to, from, rows * width);
      } else {
        for (size_t r = 0; r < rows; ++r) std::memcpy(to + r * tpitch, from + r * fpitch, width);
      }
    };
    auto work = [&](int w) {
      cudaError_t e = cudaSetDevice(device);
      auto rows_of = [&](size_t i) { return std::min(rpc, height - i * rpc); };
      if (h2d) {
        size_t j = 0;
        for (size_t i = (size_t)w; i < nchunks && e == cudaSuccess; i += (size_t)W, ++j) {
          const int k = (int)(j % kSlots);
          // the slot's last DMA, of this copy or of the previous one (an event
          // never recorded is complete)
          e = cudaEventSynchronize(ev[w][k]);
          if (e != cudaSuccess) break;
          const size_t rows = rows_of(i);
          pack(static_cast<char*>(slot[w][k]), width, static_cast<const char*>(src) + i * rpc * spitch,
               spitch, rows);
          e = cudaMemcpy2DAsync(static_cast<char*>(dst) + i * rpc * dpitch, dpitch, slot[w][k], width,
                                width, rows, cudaMemcpyHostToDevice, st[w]);
          if (e == cudaSuccess) e = cudaEventRecord(ev[w][k], st[w]);
        }
        if (e == cudaSuccess) e = cudaEventRecord(done[w], st[w]);
      } else {
        const size_t mine = nchunks > (size_t)w ? (nchunks - (size_t)w + (size_t)W - 1) / (size_t)W : 0;
        auto issue = [&](size_t j) {
          const size_t i = (size_t)w + j * (size_t)W;
          const int k = (int)(j % kSlots);
          cudaError_t ie = cudaMemcpy2DAsync(slot[w][k], width,
                                             static_cast<const char*>(src) + i * rpc * spitch, spitch,
                                             width, rows_of(i), cudaMemcpyDeviceToHost, st[w]);
          if (ie == cudaSuccess) ie = cudaEventRecord(ev[w][k], st[w]);
          return ie;
        };
        if (mine > 0) e = issue(0);
        for (size_t j = 0; j < mine && e == cudaSuccess; ++j) {
          if (j + 1 < mine) e = issue(j + 1);  // its slot was emptied one iteration ago
          if (e == cudaSuccess) e = cudaEventSynchronize(ev[w][j % kSlots]);
          if (e != cudaSuccess) break;
          const size_t i = (size_t)w + j * (size_t)W;
          pack(static_cast<char*>(dst) + i * rpc * dpitch, dpitch,
               static_cast<const char*>(slot[w][j % kSlots]), width, rows_of(i));
        }
      }
      status[(size_t)w] = e;
    };
    std::vector<std::thread> threads;
    for (int w = 1; w < W; ++w) {
      try {
        threads.emplace_back(work, w);
      } catch (...) {  // no thread to be had: this worker's chunks on the calling thread
        work(w);
      }
    }
    work(0);
    for (auto& t : threads) t.join();
    cudaSetDevice(device);
    for (cudaError_t e : status)
      if (e != cudaSuccess) return e;
    if (h2d)
      for (int w = 0; w < W; ++w) {
        const cudaError_t e = cudaStreamWaitEvent(join, done[w], 0);
        if (e != cudaSuccess) return e;
      }
    return cudaSuccess;
  }
};

}  // namespace

struct afmm_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  // workspace
  DevBuf status, vec_k, work, lists, counts, base_copy, xt, zt, part, cnt16, rmax, fstats;
  DevBuf alists, acounts, ridx, plan, scratch;  // A-form lists / counts, Case A choice
  DevBuf gidx;  // dense group index of the small-rep group kernel (k_bgroup)
  // host-buffer API staging
  DevBuf hx, hy, hz;
  HostStager stager;  // pageable host operands / result (created on first use)
  DevBuf gen_state, gen_draws, gen_scratch, gen_carry, gen_polys;  // seeded generation (generate.cu)
  DevStatus* status_host = nullptr;           // pinned
  unsigned long long* stats_host = nullptr;   // pinned, 4 words (multi-device Case A statistics)
  Call last;            // the last enqueued product
  bool pending = false;
  uint64_t cap_need = 0;  // list capacity demanded by an overflowing product (re-run)
  int variant = kAuto;
  bool group_off = false;  // AFMM_BFORM=nogroup
  bool pack_off = false;   // AFMM_BFORM=nopack
  // kernel(s) of the last call: Case A 0 B-form, 1 A-form, 2 split; + 4 when
  // the B-form part ran the small-rep group kernel (Case B: 0 or 4)
  int last_form = 0;
  // optional phase timing: ev[0] start, ev[1] before compute, ev[2] after compute, ev[3] end
  bool timing = false;
  bool timed_last = false;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};  // direct calls
  cudaEvent_t* rec_ev = ev;  // where mark() records: ev, or a graph's own events while capturing
  cudaEvent_t last_ev[4] = {nullptr, nullptr, nullptr, nullptr};  // the last product's events
  // Under stream capture (graph_call) a plain record only orders the capture
  // and is never replayed; an external record becomes an event-record node, so
  // replays are timed like direct calls. Outside a capture the external flag
  // is rejected (cudaErrorIllegalState, measured), and the captured graph gets
  // its own events.
  bool capturing = false;
  void mark(int i) {
    if (!timing) return;
    if (capturing) cudaEventRecordWithFlags(rec_ev[i], stream, cudaEventRecordExternal);
    else cudaEventRecord(rec_ev[i], stream);
  }
  // CUDA-graph replay of repeated identical device-API calls (graph_call)
  struct GraphKey {
    int which = -1, dtype = 0, mode = 0, split_k = 0, variant = 0, timing = 0, check = 1;
    const void* lhs = nullptr;
    const void* rhs = nullptr;
    void* out = nullptr;
    uint64_t n = 0, ld = 0, ld_out = 0, r0 = 0, r1 = 0;
    cudaStream_t user = nullptr;
    bool operator==(const GraphKey& o) const {
      return which == o.which && dtype == o.dtype && mode == o.mode && split_k == o.split_k &&
             check == o.check &&
             variant == o.variant && timing == o.timing && lhs == o.lhs && rhs == o.rhs &&
             out == o.out && n == o.n && ld == o.ld && ld_out == o.ld_out && r0 == o.r0 &&
             r1 == o.r1 && user == o.user;
    }
  };
  struct GraphEntry {
    GraphKey key;
    cudaGraphExec_t exec = nullptr;
    uint64_t gen = 0, launches = 0;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};  // timing graphs only
    void release() {
      if (exec) cudaGraphExecDestroy(exec);
      exec = nullptr;
      for (cudaEvent_t& e : ev)
        if (e) cudaEventDestroy(e);
    }
  };
  uint64_t buf_gen = 0;
  bool graphs = true;  // AFMM_GRAPHS=0 disables
  GraphKey seen;       // the previous call: the second identical call is captured
  std::vector<GraphEntry> graph_cache;
  cudaStream_t gstream = nullptr;  // capturable stream (the legacy default stream is not)
  cudaEvent_t join_in = nullptr, join_out = nullptr;
  // reference-facing (host buffer) call timing
  cudaEvent_t hev[4] = {nullptr, nullptr, nullptr, nullptr};
  const void* peer_checked = nullptr;  // the last `out` checked for peer access
};

namespace {

std::vector<DevBuf*> all_bufs(afmm_context* c) {
  return {&c->status, &c->vec_k, &c->work,    &c->lists,  &c->counts, &c->base_copy,
          &c->xt,     &c->zt,    &c->part,    &c->cnt16,  &c->rmax,   &c->fstats,
          &c->alists, &c->acounts, &c->ridx,  &c->plan,   &c->scratch, &c->hx,
          &c->hy,     &c->hz,      &c->gidx,   &c->gen_state, &c->gen_draws,
          &c->gen_scratch, &c->gen_carry, &c->gen_polys};
}

void set_error(afmm_error* err, int kind, int operand, uint64_t row, uint64_t col, double value,
               const char* msg) {
  if (!err) return;
  err->kind = kind;
  err->operand = operand;
  err->row = row;
  err->col = col;
  err->value = value;
  std::snprintf(err->message, sizeof err->message, "%s", msg);
}

void clear_error(afmm_error* err) {
  if (!err) return;
  std::memset(err, 0, sizeof *err);
}

afmm_status cuda_fail(afmm_error* err, cudaError_t e, const char* what) {
  char buf[256];
  std::snprintf(buf, sizeof buf, "%s: CUDA error %s (%s)", what, cudaGetErrorName(e),
                cudaGetErrorString(e));
  set_error(err, AFMM_ERRKIND_OTHER, 0, 0, 0, 0.0, buf);
  if (e == cudaErrorMemoryAllocation) return AFMM_ERR_OUT_OF_MEMORY;
  return AFMM_ERR_CUDA;
}

const char* case_name(int which) { return which == AFMM_CASE_A ? "afmm_case_a" : "afmm_case_b"; }

// kernels.hpp:15-21 and matrix.hpp:54-57
afmm_status check_dims(int which, uint64_t n_lhs, uint64_t n_rhs, afmm_error* err) {
  if (n_lhs != n_rhs) {
    char buf[256];
    std::snprintf(buf, sizeof buf, "%s: dimension mismatch %" PRIu64 " vs %" PRIu64,
                  case_name(which), n_lhs, n_rhs);
    set_error(err, AFMM_ERRKIND_SHAPE, 0, 0, 0, 0.0, buf);
    return AFMM_ERR_SHAPE;
  }
  if (n_lhs == 0) {
    set_error(err, AFMM_ERRKIND_EMPTY, 0, 0, 0, 0.0, "DenseMatrix: dimension must be >= 1");
    return AFMM_ERR_INVALID_ARGUMENT;
  }
  if (n_lhs > (1ull << 31) - 1) {
    set_error(err, AFMM_ERRKIND_OTHER, 0, 0, 0, 0.0, "afmm: n exceeds the device index range");
    return AFMM_ERR_UNSUPPORTED;
  }
  return AFMM_OK;
}

// The reassociated modes (AFMM_MODE_FAST, AFMM_MODE_FAST_LADDER) share the
// blocked-sum kernel shape, the k slices and the B-form-only Case A.
inline bool is_fast(int mode) { return mode != AFMM_MODE_ORDER_PRESERVING; }

afmm_status check_options(const afmm_options* o, afmm_error* err) {
  if (!o) return AFMM_OK;
  if (o->mode != AFMM_MODE_ORDER_PRESERVING && o->mode != AFMM_MODE_FAST &&
      o->mode != AFMM_MODE_FAST_LADDER) {
    set_error(err, AFMM_ERRKIND_OTHER, 0, 0, 0, 0.0, "afmm: options.mode must be 0, 1 or 2");
    return AFMM_ERR_INVALID_ARGUMENT;
  }
  if (o->split_k < 0 || o->num_devices < 0 || (o->flags & ~AFMM_FLAG_KERNEL_SEMANTICS) ||
      (o->partition != AFMM_PARTITION_WORK && o->partition != AFMM_PARTITION_ROWS)) {
    set_error(err, AFMM_ERRKIND_OTHER, 0, 0, 0, 0.0,
              "afmm: invalid options (split_k, num_devices or partition)");
    return AFMM_ERR_INVALID_ARGUMENT;
  }
  return AFMM_OK;
}

// Reads element (row, col) of an operand (only on the error path).
using ValueReader = std::function<double(int operand, uint64_t row, uint64_t col)>;

double read_device_element(const void* base, int dtype, uint64_t ld, uint64_t row, uint64_t col) {
  if (dtype == AFMM_F64) {
    double v = 0.0;
    cudaMemcpy(&v, static_cast<const double*>(base) + row * ld + col, sizeof v,
               cudaMemcpyDeviceToHost);
    return v;
  }
  float v = 0.f;
  cudaMemcpy(&v, static_cast<const float*>(base) + row * ld + col, sizeof v,
             cudaMemcpyDeviceToHost);
  return (double)v;
}

// Merge the device status of another shard (first offenders by index, counts summed).
void merge_status(DevStatus* into, const DevStatus& s) {
  into->nonfinite_lhs_inv = std::max(into->nonfinite_lhs_inv, s.nonfinite_lhs_inv);
  into->nonfinite_rhs_inv = std::max(into->nonfinite_rhs_inv, s.nonfinite_rhs_inv);
  into->rep_bad_inv = std::max(into->rep_bad_inv, s.rep_bad_inv);
  into->list_need = std::max(into->list_need, s.list_need);
  into->rep_nan_inv = std::max(into->rep_nan_inv, s.rep_nan_inv);
  into->rep_max = std::max(into->rep_max, s.rep_max);
  into->rep_neg |= s.rep_neg;
  into->check_violations += s.check_violations;
  into->additions += s.additions;
  into->zero_skips += s.zero_skips;
}

// Translate a device status into status / counts / error (the reference's
// exception precedence: non-finite elements at DenseMatrix construction,
// then the rep operand's first offender, kernels.hpp:25-43).
afmm_status decode_status(const DevStatus& s, int which, uint64_t n, const ValueReader& rd,
                          afmm_op_counts* counts, afmm_error* err) {
  const int rep_operand = which == AFMM_CASE_A ? 1 : 0;  // rhs for A, lhs for B
  const char* where = case_name(which);
  const char* opname = rep_operand ? "rhs" : "lhs";
  char buf[256];
  // offenders are stored inverted (0 = none); see DevStatus
  auto key = [](unsigned long long inv) { return inv ? ~inv : kNone; };
  const uint64_t nf_lhs = key(s.nonfinite_lhs_inv), nf_rhs = key(s.nonfinite_rhs_inv);
  const uint64_t rep_bad = key(s.rep_bad_inv);
  if (nf_lhs != kNone || nf_rhs != kNone) {
    const int operand = nf_lhs != kNone ? 0 : 1;
    const uint64_t lin = operand == 0 ? nf_lhs : nf_rhs;
    set_error(err, AFMM_ERRKIND_NON_FINITE, operand, lin / n, lin % n, rd(operand, lin / n, lin % n),
              "DenseMatrix: non-finite element");
    return AFMM_ERR_DOMAIN;
  }
  if (rep_bad != kNone) {
    const uint64_t lin = rep_bad >> 2;
    const int kind = (int)(rep_bad & 3);
    const uint64_t i = lin / n, j = lin % n;
    const double v = rd(rep_operand, i, j);
    if (kind == 1) {
      // std::to_string(double) is "%f" (kernels.hpp:32-34)
      std::snprintf(buf, sizeof buf, "%s: %s[%" PRIu64 "][%" PRIu64 "] = %f is not integer-valued",
                    where, opname, i, j, v);
      set_error(err, AFMM_ERRKIND_NOT_INTEGER, rep_operand, i, j, v, buf);
    } else {
      std::snprintf(buf, sizeof buf,
                    "%s: %s[%" PRIu64 "][%" PRIu64 "] exceeds the exact integer range", where,
                    opname, i, j);
      set_error(err, AFMM_ERRKIND_OUT_OF_RANGE, rep_operand, i, j, v, buf);
    }
    return AFMM_ERR_DOMAIN;
  }
  if (s.rep_nan_inv) {
    // the reference's check passes a NaN rep (both of its tests compare
    // false), then llround(NaN) asks for ~2^63 sequential adds: it never
    // finishes, so this is the one input we reject where it does not
    const uint64_t lin = ~s.rep_nan_inv, i = lin / n, j = lin % n;
    std::snprintf(buf, sizeof buf,
                  "%s: %s[%" PRIu64 "][%" PRIu64 "] is NaN (the reference would repeat "
                  "llround(NaN) ~2^63 times)",
                  where, opname, i, j);
    set_error(err, AFMM_ERRKIND_REP_NAN, rep_operand, i, j, rd(rep_operand, i, j), buf);
    return AFMM_ERR_UNSUPPORTED;
  }
  if (counts) {
    counts->additions = s.additions;
    counts->multiplications = 0;
    counts->zero_skips = s.zero_skips;
  }
  clear_error(err);
  return AFMM_OK;
}

#define CK(expr, what)                              \
  do {                                              \
    cudaError_t _e = (expr);                        \
    if (_e != cudaSuccess) return cuda_fail(err, _e, what); \
  } while (0)

// B-form tile shape for a problem of `nrows` B-form rows and `ncols` base
// columns: the widest shape whose grid still fills the GPU (per-entry
// overhead is amortised over more adds in wider tiles; small problems need the
// parallelism of narrow/small tiles). CTA slots per GPU: wide 1/SM, narrow
// 2/SM, small 8/SM.
int pick_shape(int variant, uint64_t nrows, uint64_t ncols, size_t elem, int sms) {
  switch (variant) {
    case kNarrow: return afmm_dev::kShapeNarrow;
    case kWide: return afmm_dev::kShapeWide;
    case kSmall: return afmm_dev::kShapeSmall;
    default: break;
  }
  const uint64_t cbytes = ncols * elem;
  const uint64_t wide_ctas =
      (nrows + afmm_dev::kWideRows - 1) / afmm_dev::kWideRows * ((cbytes + 4095) / 4096);
  const uint64_t narrow_ctas = (nrows + 15) / 16 * ((cbytes + 2047) / 2048);
  const uint64_t wide_slots = (uint64_t)sms * afmm_dev::kWideCtasPerSm;
  // (launch_ring trims the rows per CTA so a partial last wave costs little;
  // wide tiles need about one wave of CTAs: at n = 1024 fp64 the 128 wide
  // CTAs, trimmed to 148 of 14 rows, run 7% faster than 256 narrow ones)
  if (4 * wide_ctas >= 3 * wide_slots) return afmm_dev::kShapeWide;
  if (narrow_ctas < (uint64_t)sms) return afmm_dev::kShapeSmall;
  return afmm_dev::kShapeNarrow;
}

// Geometry of a B-form shape: (columns per tile in bytes, rows per CTA, CTAs per SM)
struct ShapeGeo {
  uint32_t tile_bytes, rows_per_cta, ctas_per_sm;
};
ShapeGeo shape_geo(int shape) {
  switch (shape) {
    case afmm_dev::kShapeWide: return {4096, afmm_dev::kWideRows, afmm_dev::kWideCtasPerSm};
    case afmm_dev::kShapeSmall: return {1024, 4, 8};
    case afmm_dev::kShapeFast: return {2048, 16, 1};
    default: return {2048, 16, 2};
  }
}

// The Case A cost model for this problem (costmodel.h) with the B-form
// geometry of `shape`; the statistics are filled in on the device.
afmm_dev::CaseAModel case_a_model(size_t elem, uint64_t n, int sms, int shape) {
  afmm_dev::CaseAModel md;
  const ShapeGeo g = shape_geo(shape);
  md.elem = (uint32_t)elem;
  md.n = n;
  md.sms = (uint32_t)sms;
  md.b_tile = (uint32_t)(g.tile_bytes / elem);
  md.b_warps_per_cta = g.rows_per_cta;
  md.b_ctas_per_sm = g.ctas_per_sm;
  // cycles per rep step per list entry and B tile: 2 pipe cycles per FADD2 /
  // DADD warp instruction, 2 instructions per 16-byte column group (G =
  // tile_bytes / 512 groups per lane): 32 cycles for the wide tile
  md.b_step = 4.0 * (double)(g.tile_bytes / 512);
  const double scale = (double)g.tile_bytes / 4096.0;  // fitted on the wide shape
  md.b_entry = 56.0 * (scale < 1.0 ? 1.0 : scale);
  md.b_entry_small = 100.0 * (scale < 1.0 ? 1.0 : scale);
  md.a_tile = afmm_dev::aform_tile_cols<float>() * 4 / (uint32_t)elem;
  md.a_rows_per_cta = afmm_dev::kAformRows;
  md.a_ctas_per_sm = afmm_dev::kAformCtasPerSm;
  return md;
}

// The repeated-addition kernel over B-form rows [0, nrows) (their lists are
// in c->lists / c->counts) and base columns [0, ncols) of the base matrix
// (kb_rows x b_cols, leading dimension ldb). dyn_ncols: ncols decided on the
// device (a Case A split); the grid covers ncols.
template <class T>
afmm_status launch_compute(afmm_context* c, const Call& call, int shape, const T* base,
                           uint64_t kb_rows, uint64_t b_cols, uint64_t ldb, uint32_t nrows,
                           int32_t ncols, const uint32_t* dyn_ncols, T* out, uint64_t ld_out,
                           DevStatus* st, int group_allow, afmm_error* err) {
  // reassociated mode: the blocked-sum kernel (bform.cu kShapeFast), k slices
  // on top when the tile grid is small
  if (is_fast(call.mode)) shape = afmm_dev::kShapeFast;
  const ShapeGeo g = shape_geo(shape);
  const uint64_t cbytes = (uint64_t)ncols * sizeof(T);
  const uint64_t ctas = (nrows + g.rows_per_cta - 1) / g.rows_per_cta *
                        ((cbytes + g.tile_bytes - 1) / g.tile_bytes);
  const uint64_t slots = (uint64_t)sm_count(c->device) * g.ctas_per_sm;
  // Fast mode (reassociated): split the k range into slices when the tile grid
  // alone cannot fill 2 waves, then add the slice partials in a fixed order.
  // Each slice is still the exact repeated-addition chain.
  const uint64_t nkb = (kb_rows + afmm_dev::bform_kb() - 1) / afmm_dev::bform_kb();
  uint32_t splits = 1;
  if (is_fast(call.mode)) {
    uint64_t want = (2 * slots + ctas - 1) / std::max<uint64_t>(ctas, 1);
    want = std::min<uint64_t>(want, std::max<uint64_t>(nkb / 4, 1));
    want = std::min<uint64_t>(want, 32);
    if (call.split_k > 0) want = std::min<uint64_t>(want, (uint64_t)call.split_k);
    splits = (uint32_t)std::max<uint64_t>(1, want);
  }
  CUtensorMap tmap;
  if (!make_tmap<T>(&tmap, base, kb_rows, b_cols, ldb)) {
    set_error(err, AFMM_ERRKIND_OTHER, 0, 0, 0, 0.0, "afmm: cuTensorMapEncodeTiled failed");
    return AFMM_ERR_CUDA;
  }
  afmm_dev::BformLaunch a;
  a.shape = shape;
  a.tmap = &tmap;
  a.lists = c->lists.as<int2>();
  a.cap = std::max<uint64_t>(call.n, c->cap_need);
  a.counts = c->counts.as<uint32_t>();
  a.nrows = nrows;
  a.col0 = 0;
  a.ncols = ncols;
  a.dyn_ncols = dyn_ncols;
  a.nk = (uint32_t)kb_rows;
  a.st = st;
  a.group_allow = group_allow;
  a.ladder = call.mode == AFMM_MODE_FAST_LADDER ? 1 : 0;
  if (splits > 1) {
    const uint64_t ldp = round_up((uint64_t)ncols, 32);
    const uint64_t stride = (uint64_t)nrows * ldp;
    CK(c->part.ensure(stride * splits * sizeof(T)), "workspace");
    a.splits = splits;
    a.slice_stride = stride;
    a.ld_out = ldp;
    CK(afmm_dev::launch_bform<T>(a, c->part.as<T>(), c->stream), "bform");
    afmm_dev::launch_reduce_slices<T>(c->part.as<T>(), stride, ldp, a.splits, nrows,
                                      (uint32_t)ncols, out, ld_out, st, dyn_ncols, c->stream);
    return AFMM_OK;
  }
  a.splits = 1;
  a.ld_out = ld_out;
  CK(afmm_dev::launch_bform<T>(a, out, c->stream), "bform");
  return AFMM_OK;
}

// The host's half of the small-rep group-kernel decision (group_mode() on the
// device completes it from the validated rep statistics): fp32, the
// order-preserving mode, and no forced k_bform shape.
int group_allow(const afmm_context* c, const Call& call) {
  if (call.dtype != AFMM_F32 || is_fast(call.mode) || c->group_off) return 0;
  return (c->variant == kAuto || c->variant == kAForm || c->variant == kHybrid) ? 1 : 0;
}

// The host's half of the packed-list decision (packed_mode() on the device
// completes it: every |rep| <= 127): the order-preserving mode, k < 2^24, and
// a problem whose lists are worth halving (below n = 2048 the second, exiting
// launch costs more than the bytes save). AFMM_BFORM=nopack keeps int2 lists.
int pack_allow(const afmm_context* c, const Call& call) {
  if (is_fast(call.mode) || c->pack_off || call.n < 2048 || call.n >= (1ull << 24)) return 0;
  return afmm_dev::kAllowPack;
}

// Group index row length: k rounded up to whole ring stages.
uint64_t group_ldg(uint64_t n) { return round_up(n, (uint64_t)afmm_dev::bform_kb()); }

// The small-rep group kernel over the same B-form operands as launch_compute
// (it exits on the device unless group mode was chosen, k_bform the reverse).
template <class T>
afmm_status launch_group_compute(afmm_context* c, const T* base, uint64_t kb_rows, uint64_t b_cols,
                                 uint64_t ldb, uint32_t nrows, int32_t ncols,
                                 const uint32_t* dyn_ncols, T* out, uint64_t ld_out,
                                 DevStatus* st, int allow, afmm_error* err) {
  if constexpr (sizeof(T) != 4) {
    return AFMM_OK;  // fp32 only (group_allow is 0 for fp64)
  } else {
    CUtensorMap tmap;
    if (!make_tmap<T>(&tmap, base, kb_rows, b_cols, ldb)) {
      set_error(err, AFMM_ERRKIND_OTHER, 0, 0, 0, 0.0, "afmm: cuTensorMapEncodeTiled failed");
      return AFMM_ERR_CUDA;
    }
    CK(afmm_dev::launch_bgroup(&tmap, c->gidx.as<uint16_t>(), group_ldg(kb_rows), nrows, ncols,
                               dyn_ncols, (uint32_t)kb_rows, out, ld_out, st, allow, c->stream),
       "bgroup");
    return AFMM_OK;
  }
}

// Case A kernel-choice variant code for k_choose
int choose_variant(int variant) {
  if (variant == kAForm) return afmm_dev::kChooseAForm;
  if (variant == kHybrid) return afmm_dev::kChooseSplit;
  return afmm_dev::kChooseAuto;
}

// Enqueue the whole device pipeline for Z rows [r0, r1). Pointers are device
// memory with leading dimension ld (lhs, rhs) and ld_out (out). Nothing waits
// on the host.
template <class T>
afmm_status enqueue_product(afmm_context* c, const Call& call, afmm_error* err) {
  cudaStream_t s = c->stream;
  const T* lhs = static_cast<const T*>(call.lhs);
  const T* rhs = static_cast<const T*>(call.rhs);
  T* out = static_cast<T*>(call.out);
  const uint64_t n = call.n, ld = call.ld, ld_out = call.ld_out, r0 = call.r0, r1 = call.r1;
  const uint64_t rows = r1 - r0;
  const uint32_t n32 = (uint32_t)n;
  const uint64_t cap = std::max<uint64_t>(n, c->cap_need);
  const int sms = sm_count(c->device);
  CK(c->status.ensure(sizeof(DevStatus)), "workspace");
  CK(c->vec_k.ensure(n * 8), "workspace");
  DevStatus* st = c->status.as<DevStatus>();
  c->timed_last = c->timing;
  for (int i = 0; i < 4; ++i) c->last_ev[i] = c->rec_ev[i];
  c->mark(0);
  afmm_dev::take_launch_error();  // (a stale one belongs to no product)
  CK(cudaMemsetAsync(st, 0, sizeof(DevStatus), s), "memset");
  const int gallow = group_allow(c, call);
  // the bits the kernels combine with the validated rep statistics: the group
  // kernel (gallow) and packed 4-byte list entries
  const int allow = gallow | pack_allow(c, call);
  if (call.prevalidated && allow) {
    // the shards' merged rep statistics (k_scan_stats does not run here);
    // both fields are < 256, so a one-byte memset of the low byte sets them
    CK(cudaMemsetAsync(&st->rep_max, (int)std::min<uint32_t>(call.rep_max, 255u), 1, s), "memset");
    CK(cudaMemsetAsync(&st->rep_neg, call.rep_neg ? 1 : 0, 1, s), "memset");
  }

  // validation (kernels.hpp:115 / :144) + DenseMatrix finite check (matrix.hpp:31-35)
  // + the per-k vector of the work formulas, one pass over both operands
  auto* nnz = c->vec_k.as<uint32_t>();
  auto* rsum = c->vec_k.as<unsigned long long>();
  // Case A: the device-side A-form / B-form choice (k_choose) for n >= 1024 or
  // when forced by AFMM_BFORM=aform|hybrid. (Fast mode keeps the B-form: its
  // blocked fp64 totals bound the fp32 chain error, DESIGN 3.2; the A-form's
  // chains are the order-preserving ones, and on sparse rows of n = 8192 they
  // drift to 2.6e-5 of sum |terms|.)
  const bool choose = call.which == AFMM_CASE_A && rows > 0 && !is_fast(call.mode) &&
                      (c->variant == kAForm || c->variant == kHybrid ||
                       (c->variant == kAuto && n >= 1024));
  // its statistics come out of the validation pass; the A-form's fp16 counts
  // are then built after the choice, only when some row takes the A-form
  const bool stats_in_scan = choose && !call.have_counts && !call.prevalidated;
  if (choose) CK(c->fstats.ensure(4 * sizeof(unsigned long long)), "workspace");
  if (stats_in_scan)
    CK(cudaMemsetAsync(c->fstats.p, 0, 4 * sizeof(unsigned long long), s), "memset");
  if (!call.prevalidated)
    afmm_dev::launch_scan_stats<T>(lhs, rhs, ld, n32, call.which == AFMM_CASE_B ? 1 : 0, 0, n32, 0,
                                   n32, st, nnz, rsum, s, call.check_finite ? 1 : 0,
                                   stats_in_scan ? c->fstats.as<unsigned long long>() : nullptr);

  if (call.which == AFMM_CASE_B) {
    // rep = X[i,k] (lhs), bases = Y[k,:] (rhs): B-form directly.
    const int shape = pick_shape(c->variant, rows, n, sizeof(T), sms);
    CK(c->lists.ensure(std::max<uint64_t>(rows, 1) * cap * sizeof(int2)), "workspace");
    CK(c->counts.ensure(std::max<uint64_t>(rows, 1) * 4), "workspace");
    afmm_dev::launch_rows<T>(lhs, ld, n32, 1, nnz, nullptr, (uint32_t)r0, (uint32_t)r1,
                             (uint32_t)r0, (uint32_t)r1, c->lists.as<int2>(), cap,
                             c->counts.as<uint32_t>(), nullptr, st, s, nullptr, allow);
    if (gallow && rows > 0) {
      const uint64_t ldg = group_ldg(n), ngroups = (rows + afmm_dev::kGroupRows - 1) / afmm_dev::kGroupRows;
      CK(c->gidx.ensure(ngroups * ldg * sizeof(uint16_t)), "workspace");
      afmm_dev::launch_group_idx<T>(lhs, ld, n32, 1, (uint32_t)r0, (uint32_t)rows,
                                    c->gidx.as<uint16_t>(), ldg, st, gallow, s);
    }
    const T* base = rhs;
    uint64_t ldb = ld;
    if ((ld * sizeof(T)) % 16 != 0 || reinterpret_cast<uintptr_t>(rhs) % 16 != 0) {
      ldb = round_up(n, 32);
      CK(c->base_copy.ensure(n * ldb * sizeof(T)), "workspace");
      CK(cudaMemcpy2DAsync(c->base_copy.p, ldb * sizeof(T), rhs, ld * sizeof(T), n * sizeof(T), n,
                           cudaMemcpyDeviceToDevice, s),
         "copy");
      base = c->base_copy.as<T>();
    }
    c->mark(1);
    if (rows > 0) {
      afmm_status cs = launch_compute<T>(c, call, shape, base, n, n, ldb, (uint32_t)rows,
                                         (int32_t)n, nullptr, out, ld_out, st, allow, err);
      if (cs != AFMM_OK) return cs;
      if (gallow) {
        cs = launch_group_compute<T>(c, base, n, n, ldb, (uint32_t)rows, (int32_t)n, nullptr, out,
                                     ld_out, st, gallow, err);
        if (cs != AFMM_OK) return cs;
      }
    }
    c->mark(2);
    c->last_form = 0;  // (+ 4 from the status when k_bgroup ran)
  } else {
    // Case A: the B-form on transposed operands, the A-form (base uniform per
    // warp), or the slab's rows split between them. For n >= 1024 (or when
    // forced by AFMM_BFORM=aform|hybrid) k_choose decides on the device from
    // the prepass statistics; every kernel of both forms is enqueued and reads
    // its row count from the plan (a form with no rows exits at once).
    using E = typename afmm_dev::AEntry<T>::type;
    const uint32_t tc = afmm_dev::aform_tile_cols<T>();
    const uint64_t ntiles = (n + tc - 1) / tc, ldc = round_up(n, 64);
    // B part: B-form rows = Z columns j (rep list = column j of Y), B-form
    // columns = the slab's B rows (bases X[i,k], gathered through ridx)
    const int shape = pick_shape(c->variant, n, std::max<uint64_t>(rows, 1), sizeof(T), sms);
    if (choose) CK(c->acounts.ensure(rows * 4), "workspace");
    afmm_dev::launch_rows<T>(lhs, ld, n32, 0, nullptr, rsum, (uint32_t)r0, (uint32_t)r1,
                             (uint32_t)r0, (uint32_t)r1, nullptr, 0, nullptr, nullptr, st, s,
                             choose ? c->acounts.as<uint32_t>() : nullptr);
    const uint32_t* plan = nullptr;
    const uint32_t* ridx = nullptr;
    if (choose) {
      CK(c->cnt16.ensure(n * ldc * sizeof(__half)), "workspace");
      CK(c->rmax.ensure(n * ntiles * sizeof(uint16_t)), "workspace");
      CK(c->plan.ensure(4 * sizeof(uint32_t)), "workspace");
      CK(c->ridx.ensure(rows * 4), "workspace");
      CK(c->scratch.ensure(afmm_dev::choose_scratch_bytes(n)), "workspace");
      CK(c->alists.ensure(rows * n * sizeof(E)), "workspace");
      auto* fs = c->fstats.as<unsigned long long>();
      if (!call.have_counts && !stats_in_scan) {
        CK(cudaMemsetAsync(fs, 0, 4 * sizeof(unsigned long long), s), "memset");
        afmm_dev::launch_counts_f16<T>(rhs, ld, n32, tc, c->cnt16.as<__half>(), ldc,
                                       c->rmax.as<uint16_t>(), fs, s);
      }
      afmm_dev::CaseAModel md = case_a_model(sizeof(T), n, sms, shape);
      md.group_allow = gallow;
      CK(afmm_dev::launch_choose(md, (uint32_t)rows, choose_variant(c->variant),
                                 c->acounts.as<uint32_t>(), fs, c->scratch.as<uint32_t>(),
                                 c->plan.as<uint32_t>(), c->ridx.as<uint32_t>(), st, s),
         "choose");
      plan = c->plan.as<uint32_t>();
      ridx = c->ridx.as<uint32_t>();
      if (stats_in_scan)  // the A-form's counts, only when it got rows (plan[0])
        afmm_dev::launch_counts_f16<T>(rhs, ld, n32, tc, c->cnt16.as<__half>(), ldc,
                                       c->rmax.as<uint16_t>(), nullptr, s, plan);
      // the A rows' compacted nonzero bases (k, X[i,k])
      afmm_dev::launch_acompact<T>(lhs, ld, n32, (uint32_t)r0, (uint32_t)rows, plan, ridx,
                                   c->alists.as<E>(), n, c->acounts.as<uint32_t>(), s);
    }
    const uint64_t lds = round_up(std::max<uint64_t>(rows, 1), 32);
    CK(c->xt.ensure(n * lds * sizeof(T)), "workspace");
    CK(c->zt.ensure(n * lds * sizeof(T)), "workspace");
    CK(c->lists.ensure(n * cap * sizeof(int2)), "workspace");
    CK(c->counts.ensure(n * 4), "workspace");
    if (rows > 0) {
      afmm_dev::launch_transpose_compact<T>(rhs, ld, n32, c->lists.as<int2>(), cap,
                                            c->counts.as<uint32_t>(), st,
                                            plan ? plan + 1 : nullptr, s, allow);
      if (gallow) {
        const uint64_t ldg = group_ldg(n), ngroups = (n + afmm_dev::kGroupRows - 1) / afmm_dev::kGroupRows;
        CK(c->gidx.ensure(ngroups * ldg * sizeof(uint16_t)), "workspace");
        afmm_dev::launch_group_idx<T>(rhs, ld, n32, 0, 0, n32, c->gidx.as<uint16_t>(), ldg, st,
                                      gallow, s, plan ? plan + 1 : nullptr);
      }
      afmm_dev::launch_transpose<T>(lhs + r0 * ld, ld, (uint32_t)rows, n32, c->xt.as<T>(), lds, s,
                                    ridx, nullptr, nullptr, plan, plan ? 1 : 0);
    }
    c->mark(1);
    if (choose) {
      // A-form: the reference's own orientation, zero bases skipped per warp
      CUtensorMap cmap;
      if (!make_count_tmap(&cmap, c->cnt16.as<__half>(), n, n, ldc)) {
        set_error(err, AFMM_ERRKIND_OTHER, 0, 0, 0, 0.0, "afmm: cuTensorMapEncodeTiled failed");
        return AFMM_ERR_CUDA;
      }
      CK(afmm_dev::launch_aform<T>(&cmap, c->alists.as<E>(), n, c->acounts.as<uint32_t>(),
                                   (uint32_t)rows, plan, n32, n32, c->rmax.as<uint16_t>(), out,
                                   ld_out, ridx, st, s),
         "aform");
    }
    if (rows > 0) {
      // B-form: Case A as Case B on transposed operands, Z^T = (Y^T) (x) (X^T)
      afmm_status cs = launch_compute<T>(c, call, shape, c->xt.as<T>(), n, rows, lds, n32,
                                         (int32_t)rows, plan ? plan + 1 : nullptr, c->zt.as<T>(),
                                         lds, st, allow, err);
      if (cs != AFMM_OK) return cs;
      if (gallow) {
        cs = launch_group_compute<T>(c, c->xt.as<T>(), n, rows, lds, n32, (int32_t)rows,
                                     plan ? plan + 1 : nullptr, c->zt.as<T>(), lds, st, gallow,
                                     err);
        if (cs != AFMM_OK) return cs;
      }
    }
    c->mark(2);
    if (rows > 0)
      afmm_dev::launch_transpose<T>(c->zt.as<T>(), lds, n32, (uint32_t)rows, out, ld_out, s,
                                    nullptr, ridx, st, plan, plan ? 2 : 0);
  }
  c->mark(3);
  CK(cudaGetLastError(), "launch");
  CK(afmm_dev::take_launch_error(), "launch");
  CK(cudaMemcpyAsync(c->status_host, st, sizeof(DevStatus), cudaMemcpyDeviceToHost, s),
     "status readback");
  c->last = call;
  c->pending = true;
  return AFMM_OK;
}

afmm_status enqueue_call(afmm_context* c, const Call& call, afmm_error* err) {
  return call.dtype == AFMM_F64 ? enqueue_product<double>(c, call, err)
                                : enqueue_product<float>(c, call, err);
}

ValueReader device_reader(const Call& call) {
  return [call](int operand, uint64_t row, uint64_t col) {
    return read_device_element(operand == 0 ? call.lhs : call.rhs, call.dtype, call.ld, row, col);
  };
}

// Wait for the pending product and decode it. A product whose rep lists did
// not fit (reps beyond an entry's range, split into several entries) is
// re-run once with the capacity it reported.
afmm_status finish_locked(afmm_context* c, afmm_op_counts* counts, afmm_error* err) {
  if (!c->pending) {
    clear_error(err);
    return AFMM_OK;
  }
  c->pending = false;
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cuda_fail(err, e, "afmm: device execution");
  const DevStatus s = *c->status_host;
  if (s.form_rows) c->last_form = s.a_rows == 0 ? 0 : (s.a_rows == s.form_rows ? 1 : 2);
  else c->last_form = 0;
  // the B-form part ran the small-rep group kernel (group_mode on the device)
  const bool b_part = c->last_form != 1 && c->last.r1 > c->last.r0;
  if (b_part && group_allow(c, c->last) && s.rep_max <= afmm_dev::kGroupMaxRep && s.rep_neg == 0)
    c->last_form |= 4;
#ifdef AFMM_CHECKED
  {
    int bad_guards = 0;
    for (DevBuf* b : all_bufs(c)) bad_guards += b->guards_intact() ? 0 : 1;
    if (s.check_violations || bad_guards) {
      char buf[256];
      std::snprintf(buf, sizeof buf,
                    "afmm (checked build): %llu device bound-check violations, %d workspace "
                    "guard bands overwritten",
                    (unsigned long long)s.check_violations, bad_guards);
      set_error(err, AFMM_ERRKIND_OTHER, 0, 0, 0, 0.0, buf);
      return AFMM_ERR_CUDA;
    }
  }
#endif
  const afmm_status st = decode_status(s, c->last.which, c->last.n, device_reader(c->last),
                                       counts, err);
  if (st != AFMM_OK || s.list_need == 0) return st;
  // list overflow (validation passed): re-run with the capacity it needs
  if (s.list_need > (1ull << 40) / std::max<uint64_t>(c->last.n, 1)) {
    set_error(err, AFMM_ERRKIND_OTHER, 0, 0, 0, 0.0,
              "afmm: reps this large need rep lists beyond device memory");
    return AFMM_ERR_OUT_OF_MEMORY;
  }
  c->cap_need = s.list_need;
  const Call again = c->last;
  afmm_status r = enqueue_call(c, again, err);
  c->cap_need = 0;
  if (r != AFMM_OK) return r;
  return finish_locked(c, counts, err);
}

// Device-API calls that repeat with the same pointers, sizes and options (a
// serving loop, a benchmark step) replay a CUDA graph of the whole pipeline:
// the first call runs normally, the second identical call is captured (on the
// context's own capturable stream, joined to the caller's stream by events --
// the legacy default stream cannot be captured), later ones replay it, which
// removes the host enqueue of ~10 launches per call and the GPU gaps between
// them (small problems are launch bound). Every call is capturable: the Case
// A form is chosen on the device. A workspace reallocation invalidates the
// cache; a failed capture falls back to the direct path for good
// (AFMM_GRAPHS=0 disables the mechanism).
afmm_status graph_call(afmm_context* c, const Call& call, afmm_error* err) {
  auto direct = [&]() { return enqueue_call(c, call, err); };
  if (!c->graphs) return direct();
  afmm_context::GraphKey key;
  key.which = call.which;
  key.dtype = call.dtype;
  key.mode = call.mode;
  key.split_k = call.split_k;
  key.check = call.check_finite ? 1 : 0;
  key.variant = c->variant + (c->group_off ? 100 : 0);
  key.timing = c->timing ? 1 : 0;
  key.lhs = call.lhs;
  key.rhs = call.rhs;
  key.out = call.out;
  key.n = call.n;
  key.ld = call.ld;
  key.ld_out = call.ld_out;
  key.r0 = call.r0;
  key.r1 = call.r1;
  key.user = c->stream;
  auto& cache = c->graph_cache;
  for (size_t i = 0; i < cache.size();) {  // entries captured before a reallocation
    if (cache[i].gen != c->buf_gen) {
      cache[i].release();
      cache.erase(cache.begin() + i);
    } else {
      ++i;
    }
  }
  afmm_context::GraphEntry* hit = nullptr;
  for (auto& ge : cache)
    if (ge.key == key) hit = &ge;
  const cudaStream_t user = c->stream;
  auto join_and_launch = [&](const afmm_context::GraphEntry& ge) -> cudaError_t {
    cudaError_t e = cudaEventRecord(c->join_in, user);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c->gstream, c->join_in, 0);
    if (e == cudaSuccess) e = cudaGraphLaunch(ge.exec, c->gstream);
    if (e == cudaSuccess) e = cudaEventRecord(c->join_out, c->gstream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(user, c->join_out, 0);
    return e;
  };
  if (hit) {
    CK(join_and_launch(*hit), "afmm: graph launch");
    for (uint64_t i = 0; i < hit->launches; ++i) afmm_dev::note_launch();
    c->timed_last = c->timing;
    for (int i = 0; i < 4; ++i) c->last_ev[i] = hit->ev[i];
    c->last = call;
    c->pending = true;
    return AFMM_OK;
  }
  if (!(key == c->seen)) {
    c->seen = key;
    return direct();
  }
  // second identical call: capture it
  if (!c->gstream) {
    if (cudaStreamCreateWithFlags(&c->gstream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->join_in, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->join_out, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      c->graphs = false;
      return direct();
    }
  }
  afmm_context::GraphEntry ge;
  for (int i = 0; key.timing && i < 4; ++i)
    if (cudaEventCreate(&ge.ev[i]) != cudaSuccess) {
      cudaGetLastError();
      ge.release();
      return direct();
    }
  const uint64_t launches0 = afmm_dev::g_launches.load();
  c->stream = c->gstream;
  if (cudaStreamBeginCapture(c->gstream, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
    cudaGetLastError();
    c->stream = user;
    c->graphs = false;
    ge.release();
    return direct();
  }
  if (key.timing) c->rec_ev = ge.ev;
  c->capturing = true;
  const afmm_status st = direct();
  c->capturing = false;
  c->rec_ev = c->ev;
  cudaGraph_t graph = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(c->gstream, &graph);
  c->stream = user;
  const bool ok = st == AFMM_OK && ec == cudaSuccess && graph &&
                  cudaGraphInstantiate(&ge.exec, graph, 0) == cudaSuccess;
  if (graph) cudaGraphDestroy(graph);
  if (!ok) {  // fall back to direct calls for the life of the context
    cudaGetLastError();
    ge.release();
    c->graphs = false;
    c->pending = false;
    if (st != AFMM_OK) return st;
    return direct();
  }
  ge.key = key;
  ge.gen = c->buf_gen;
  ge.launches = afmm_dev::g_launches.load() - launches0;
  if (cache.size() >= 8) {
    cache.front().release();
    cache.erase(cache.begin());
  }
  cache.push_back(ge);
  CK(join_and_launch(cache.back()), "afmm: graph launch");
  return AFMM_OK;  // the captured call left the host state of this product
}

// Default contexts of the reference-facing calls: one per (device, shard
// slot) -- a device listed twice in options->devices gets two contexts.
constexpr int kMaxDevices = 64, kMaxSlots = 8;
std::mutex g_default_mu;
afmm_context* g_default[kMaxDevices][kMaxSlots] = {};

afmm_status default_context(int device, int slot, afmm_context** out, afmm_error* err) {
  if (device < 0) {
    cudaError_t e = cudaGetDevice(&device);
    if (e != cudaSuccess) return cuda_fail(err, e, "afmm: no CUDA device");
  }
  if (device >= kMaxDevices || slot >= kMaxSlots) {
    set_error(err, AFMM_ERRKIND_OTHER, 0, 0, 0, 0.0, "afmm: device ordinal out of range");
    return AFMM_ERR_INVALID_ARGUMENT;
  }
  std::lock_guard<std::mutex> g(g_default_mu);
  if (!g_default[device][slot]) {
    afmm_context* c = nullptr;
    afmm_status s = afmm_context_create(device, &c);
    if (s != AFMM_OK) {
      set_error(err, AFMM_ERRKIND_OTHER, 0, 0, 0, 0.0, "afmm: cannot create a CUDA context");
      return s;
    }
    g_default[device][slot] = c;
  }
  *out = g_default[device][slot];
  return AFMM_OK;
}

afmm_status enable_timing_locked(afmm_context* c, int32_t enable) {
  if (enable && !c->ev[0]) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(c->device);
    for (cudaEvent_t& e : c->ev)
      if (cudaEventCreate(&e) != cudaSuccess) {
        cudaSetDevice(prev);
        return AFMM_ERR_CUDA;
      }
    cudaSetDevice(prev);
  }
  c->timing = enable != 0;
  return AFMM_OK;
}

// Is `p` page-locked host memory mapped into the device address space? Then
// the kernels can store Z rows straight into it (zero-copy).
template <class T>
T* mapped_pointer(T* p) {
  cudaPointerAttributes attr{};
  T* d = nullptr;
  if (cudaPointerGetAttributes(&attr, p) == cudaSuccess && attr.type == cudaMemoryTypeHost &&
      attr.devicePointer)
    d = static_cast<T*>(attr.devicePointer);
  cudaGetLastError();  // a pageable pointer is not an error here
  return d;
}

ValueReader host_reader(const void* lhs, const void* rhs, int dtype, uint64_t n) {
  return [=](int operand, uint64_t row, uint64_t col) {
    const void* b = operand == 0 ? lhs : rhs;
    return dtype == AFMM_F64 ? static_cast<const double*>(b)[row * n + col]
                             : (double)static_cast<const float*>(b)[row * n + col];
  };
}

afmm_status ensure_host_events(afmm_context* c) {
  for (cudaEvent_t& e : c->hev)
    if (!e && cudaEventCreate(&e) != cudaSuccess) return AFMM_ERR_CUDA;
  return AFMM_OK;
}

// The reference-facing call on one device: host buffers in, host buffer out.
template <class T>
afmm_status host_product_one(int which, const T* lhs, const T* rhs, uint64_t n, T* out,
                             const afmm_options* opt, afmm_op_counts* counts, afmm_error* err) {
  afmm_context* c = nullptr;
  int device = opt ? opt->device : -1;
  if (opt && opt->num_devices == 1 && opt->devices) device = opt->devices[0];
  afmm_status st = default_context(device, 0, &c, err);
  if (st != AFMM_OK) return st;
  std::lock_guard<std::mutex> g(c->mu);
  CK(cudaSetDevice(c->device), "afmm: cudaSetDevice");
  const uint64_t ld = round_up(n, 32);
  const size_t mat = n * ld * sizeof(T);
  const int mode = opt ? opt->mode : AFMM_MODE_ORDER_PRESERVING;
  afmm_timing* timing = opt ? opt->timing : nullptr;
  if (timing && ensure_host_events(c) != AFMM_OK) return cuda_fail(err, cudaErrorUnknown, "events");
  const bool time_it = timing != nullptr;
  const bool kernel_timing = c->timing;
  if (time_it) CK(enable_timing_locked(c, 1) == AFMM_OK ? cudaSuccess : cudaErrorUnknown,
                  "afmm: timing events");
  // Zero-copy result: when `out` is page-locked host memory (mapped into the
  // device address space) and the only kernel writing Z is k_bform (Case B,
  // order-preserving), the kernel stores Z rows straight into `out` over PCIe
  // as its CTAs finish, so the 1 GiB D2H of cfg5 overlaps the compute instead
  // of following it. k_bform returns before writing when validation failed,
  // so `out` stays untouched on error, as with the staged copy.
  T* zdev = which == AFMM_CASE_B && mode == AFMM_MODE_ORDER_PRESERVING ? mapped_pointer(out)
                                                                         : nullptr;
  CK(c->hx.ensure(mat), "afmm: device allocation");
  CK(c->hy.ensure(mat), "afmm: device allocation");
  if (!zdev) CK(c->hz.ensure(mat), "afmm: device allocation");
  cudaStream_t s = c->stream;
  if (time_it) CK(cudaEventRecord(c->hev[0], s), "event");
  // pageable operands / result: the staged pipeline (HostStager); page-locked
  // or small ones: one plain asynchronous copy each
  auto to_device = [&](void* dst, const T* src) -> cudaError_t {
    // (no page-locked memory for the slots: the plain copy still works)
    if (HostStager::wants(src, n * sizeof(T), n) && c->stager.ensure(c->device) == cudaSuccess)
      return c->stager.copy(true, dst, ld * sizeof(T), src, n * sizeof(T), n * sizeof(T), n, s);
    cudaGetLastError();
    return cudaMemcpy2DAsync(dst, ld * sizeof(T), src, n * sizeof(T), n * sizeof(T), n,
                             cudaMemcpyHostToDevice, s);
  };
  CK(to_device(c->hx.p, lhs), "afmm: H2D");
  CK(to_device(c->hy.p, rhs), "afmm: H2D");
  Call call;
  call.which = which;
  call.dtype = sizeof(T) == 8 ? AFMM_F64 : AFMM_F32;
  call.mode = mode;
  call.split_k = opt ? opt->split_k : 0;
  call.check_finite = !(opt && (opt->flags & AFMM_FLAG_KERNEL_SEMANTICS));
  call.lhs = c->hx.p;
  call.rhs = c->hy.p;
  call.n = n;
  call.ld = ld;
  call.out = zdev ? static_cast<void*>(zdev) : c->hz.p;
  call.ld_out = zdev ? n : ld;
  call.r0 = 0;
  call.r1 = n;
  st = enqueue_call(c, call, err);
  if (st == AFMM_OK) st = finish_locked(c, counts, err);
  if (st == AFMM_OK && !zdev) {
    // (finish_locked has synchronised the stream: Z is complete on the device)
    if (HostStager::wants(out, n * sizeof(T), n) && c->stager.ensure(c->device) == cudaSuccess) {
      CK(c->stager.copy(false, out, n * sizeof(T), c->hz.p, ld * sizeof(T), n * sizeof(T), n, s),
         "afmm: D2H");
    } else {
      CK(cudaMemcpy2DAsync(out, n * sizeof(T), c->hz.p, ld * sizeof(T), n * sizeof(T), n,
                           cudaMemcpyDeviceToHost, s),
         "afmm: D2H");
    }
  }
  if (time_it) CK(cudaEventRecord(c->hev[1], s), "event");
  if (st == AFMM_OK) CK(cudaStreamSynchronize(s), "afmm: D2H");
  if (time_it) {
    float total = -1.f, compute = -1.f;
    if (st == AFMM_OK) {
      cudaEventElapsedTime(&total, c->hev[0], c->hev[1]);
      cudaEventElapsedTime(&compute, c->last_ev[1], c->last_ev[2]);
    }
    timing->total_ms = total;
    timing->compute_ms = compute;
    timing->devices = 1;
    timing->form = c->last_form;
    if (!kernel_timing) enable_timing_locked(c, 0);
  }
  return st;
}

// A reusable barrier for the shard threads of a multi-device call.
class Barrier {
 public:
  explicit Barrier(int n) : n_(n) {}
  void wait() {
    std::unique_lock<std::mutex> l(m_);
    const uint64_t gen = gen_;
    if (++count_ == n_) {
      count_ = 0;
      ++gen_;
      cv_.notify_all();
    } else {
      cv_.wait(l, [&] { return gen_ != gen; });
    }
  }

 private:
  std::mutex m_;
  std::condition_variable cv_;
  int n_, count_ = 0;
  uint64_t gen_ = 0;
};

// Enable peer access from `device` to `peer` once per pair (NVLink): the
// kernels may then store Z rows into another GPU's memory, and peer copies
// go device to device. Returns whether access is possible.
bool ensure_peer_access(int device, int peer) {
  if (device == peer) return true;
  static std::mutex mu;
  static std::vector<std::pair<std::pair<int, int>, bool>> known;
  std::lock_guard<std::mutex> g(mu);
  for (const auto& k : known)
    if (k.first == std::make_pair(device, peer)) return k.second;
  int can = 0;
  cudaDeviceCanAccessPeer(&can, device, peer);
  bool ok = false;
  if (can) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    const cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    ok = e == cudaSuccess || e == cudaErrorPeerAccessAlreadyEnabled;
    cudaGetLastError();
    cudaSetDevice(prev);
  }
  known.push_back({{device, peer}, ok});
  return ok;
}

// Per-row predicted kernel time for the row partition (afmm_row_cost_device
// and the multi-device call): Case B W_i; Case A the cheaper of the row's
// A-form cost and its share of a B-form tile (costmodel.h).
void row_costs(int which, size_t elem, uint64_t n, int sms, const uint64_t* work,
               const uint32_t* nnz_row, const unsigned long long* fstats, uint64_t* cost,
               bool group = false) {
  if (which == AFMM_CASE_B) {
    std::memcpy(cost, work, n * sizeof(uint64_t));
    return;
  }
  const int shape = pick_shape(kAuto, n, n, elem, sms);
  afmm_dev::CaseAModel md = case_a_model(elem, n, sms, shape);
  md.nnz_y = fstats[0];
  md.trip_sum = fstats[1];
  md.rep_sum = fstats[3];
  md.group = group;
  const bool a_ok = fstats[2] == 0;
  const double per_row_b = md.per_tile() / (double)md.tile_rows();
  const double per_base = md.per_base();
  for (uint64_t i = 0; i < n; ++i) {
    const double a = a_ok ? per_base * (double)nnz_row[i] : per_row_b;
    cost[i] = (uint64_t)std::llround(std::min(a, per_row_b) + 1.0);
  }
}

// Modeled kernel time of Case A slabs (rows [r0, r1) of a product whose
// rows have nnz[i] nonzero bases): the device-side choice (k_choose) run on
// the host -- pure B-form, pure A-form or the best split, whichever the model
// picks -- with the slab's own wave quantisation.
class SlabModel {
 public:
  SlabModel(const afmm_dev::CaseAModel& md, const uint32_t* nnz, bool a_ok)
      : md_(md), nnz_(nnz), a_ok_(a_ok), cnt_(md.n + 2), cum_c_(md.n + 3), cum_s_(md.n + 3) {}
  double time(uint64_t r0, uint64_t r1) {
    const uint64_t rows = r1 > r0 ? r1 - r0 : 0, n = md_.n;
    if (rows == 0) return 0.0;
    if (!a_ok_) return md_.cost_b((rows + md_.tile_rows() - 1) / md_.tile_rows());
    std::fill(cnt_.begin(), cnt_.end(), 0u);
    for (uint64_t i = r0; i < r1; ++i) ++cnt_[std::min<uint64_t>(nnz_[i], n)];
    cum_c_[0] = 0;
    cum_s_[0] = 0.0;
    for (uint64_t v = 0; v <= n + 1; ++v) {
      cum_c_[v + 1] = cum_c_[v] + cnt_[v];
      cum_s_[v + 1] = cum_s_[v] + (double)v * cnt_[v];
    }
    auto pre = [&](uint64_t m) {
      // largest v with cum_c[v] <= m: the m sparsest rows take every row of
      // value < v and (m - cum_c[v]) rows of value v
      const uint64_t v =
          (uint64_t)(std::upper_bound(cum_c_.begin(), cum_c_.begin() + n + 2, m) - cum_c_.begin()) - 1;
      return cum_s_[v] + (double)v * (double)(m - cum_c_[v]);
    };
    double t = 0.0;
    afmm_dev::choose_aform_rows(md_, rows, afmm_dev::kChooseAuto, pre, &t);
    return t;
  }

 private:
  const afmm_dev::CaseAModel& md_;
  const uint32_t* nnz_;
  bool a_ok_;
  std::vector<uint32_t> cnt_;
  std::vector<uint64_t> cum_c_;
  std::vector<double> cum_s_;
};

// Case A row cuts by modeled slab time: start from the cut of the additive
// per-row costs (row_costs), then move each boundary between neighbours to
// balance their modeled times (a few sweeps of bisection; the model's
// tile and wave quantisation make the slab time non-additive).
void partition_case_a(const afmm_dev::CaseAModel& md, const uint32_t* nnz, bool a_ok,
                      const uint64_t* add_cost, uint32_t parts, uint64_t* cuts, double* times) {
  const uint64_t n = md.n;
  afmm_partition_rows(add_cost, n, parts, cuts);
  SlabModel sm(md, nnz, a_ok);
  std::vector<double> t(parts);
  for (uint32_t p = 0; p < parts; ++p) t[p] = sm.time(cuts[p], cuts[p + 1]);
  for (int sweep = 0; sweep < 8 && parts > 1; ++sweep) {
    bool moved = false;
    for (uint32_t p = 0; p + 1 < parts; ++p) {
      // boundary b = cuts[p + 1] in [cuts[p], cuts[p + 2]]: find the b where
      // time(left) crosses time(right) (left grows, right shrinks with b)
      uint64_t lo = cuts[p], hi = cuts[p + 2];
      const double before = std::max(t[p], t[p + 1]);
      while (hi - lo > 1) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (sm.time(cuts[p], mid) <= sm.time(mid, cuts[p + 2])) lo = mid;
        else hi = mid;
      }
      // accept a lower pair maximum, or the same maximum with the pair closer
      // together (a B-form slab's time is flat within a tile: its neighbour
      // can take rows up to that level at no cost)
      uint64_t best_b = cuts[p + 1];
      double best = before, gap = std::fabs(t[p] - t[p + 1]);
      for (uint64_t b : {lo, hi}) {
        const double tl = sm.time(cuts[p], b), tr = sm.time(b, cuts[p + 2]);
        const double mx = std::max(tl, tr), g = std::fabs(tl - tr);
        if (mx < best * (1.0 - 1e-9) || (mx <= best * (1.0 + 1e-12) && g < gap * (1.0 - 1e-9))) {
          best = mx;
          gap = g;
          best_b = b;
        }
      }
      if (best_b != cuts[p + 1]) {
        cuts[p + 1] = best_b;
        t[p] = sm.time(cuts[p], best_b);
        t[p + 1] = sm.time(best_b, cuts[p + 2]);
        moved = true;
      }
    }
    if (!moved) break;
  }
  if (times)
    for (uint32_t p = 0; p < parts; ++p) times[p] = t[p];
}

// Row cuts for `parts` devices from the full operands' statistics.
void partition_from_stats(int which, size_t elem, uint64_t n, int sms, const uint64_t* work,
                          const uint32_t* nnz_row, const unsigned long long* fstats,
                          uint32_t parts, uint64_t* cuts, bool group = false) {
  std::vector<uint64_t> cost(n);
  row_costs(which, elem, n, sms, work, nnz_row, fstats, cost.data(), group);
  if (which == AFMM_CASE_B) {
    afmm_partition_rows(cost.data(), n, parts, cuts);
    return;
  }
  afmm_dev::CaseAModel md = case_a_model(elem, n, sms, pick_shape(kAuto, n, n, elem, sms));
  md.nnz_y = fstats[0];
  md.trip_sum = fstats[1];
  md.rep_sum = fstats[3];
  md.group = group;
  partition_case_a(md, nnz_row, fstats[2] == 0, cost.data(), parts, cuts, nullptr);
}

// The reference-facing call sharded over several devices (one process):
//   A  each shard copies an equal row chunk of X and Y to its device (its own
//      host thread: pageable copies run in parallel) and validates it,
//      computing the per-k vector of its Y rows;
//   B  each shard completes Y and the per-k vector from its peers (NVLink peer
//      copies), computes W_i (and, Case A, the nonzero bases per row and the
//      statistics of Y) for its chunk rows, and reads them back;
//   -  the statuses merge (first offender of the whole operands); the cuts
//      balance the predicted time;
//   C  each shard copies the X rows of its cut that it lacks from their owners
//      and runs the product on its rows; its Z rows go straight into `out`
//      (zero-copy Case B) or are copied back.
template <class T>
afmm_status host_product_multi(int which, const T* lhs, const T* rhs, uint64_t n, T* out,
                               const afmm_options* opt, afmm_op_counts* counts,
                               afmm_error* err) {
  const int G = opt->num_devices;
  std::vector<int> devs(G);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return cuda_fail(err, cudaErrorNoDevice, "afmm: no CUDA device");
  for (int g = 0; g < G; ++g) {
    devs[g] = opt->devices ? opt->devices[g] : g;
    if (devs[g] < 0 || devs[g] >= ndev) {
      set_error(err, AFMM_ERRKIND_OTHER, 0, 0, 0, 0.0, "afmm: options.devices holds an invalid ordinal");
      return AFMM_ERR_INVALID_ARGUMENT;
    }
  }
  std::vector<afmm_context*> ctx(G);
  for (int g = 0; g < G; ++g) {
    int slot = 0;
    for (int h = 0; h < g; ++h) slot += devs[h] == devs[g];
    afmm_status st = default_context(devs[g], slot, &ctx[g], err);
    if (st != AFMM_OK) return st;
  }
  // lock the contexts in address order (no lock-order inversion between callers)
  std::vector<afmm_context*> order(ctx);
  std::sort(order.begin(), order.end());
  std::vector<std::unique_lock<std::mutex>> locks;
  for (afmm_context* c : order) locks.emplace_back(c->mu);
  // peer access between the devices (NVLink)
  for (int a : devs)
    for (int b : devs) ensure_peer_access(a, b);
  const int dtype = sizeof(T) == 8 ? AFMM_F64 : AFMM_F32;
  const int mode = opt->mode;
  const bool check_finite = !(opt->flags & AFMM_FLAG_KERNEL_SEMANTICS);
  const uint64_t ld = round_up(n, 32);
  const size_t row_bytes = ld * sizeof(T), mat = n * row_bytes;
  T* zmapped = which == AFMM_CASE_B && mode == AFMM_MODE_ORDER_PRESERVING ? mapped_pointer(out)
                                                                            : nullptr;
  std::vector<uint64_t> e(G + 1), cuts(G + 1);
  for (int g = 0; g <= G; ++g) e[g] = n * (uint64_t)g / (uint64_t)G;
  std::vector<uint64_t> work(n, 0);
  std::vector<uint32_t> nnz_row(which == AFMM_CASE_A ? n : 0, 0);
  std::vector<DevStatus> stat(G);
  std::vector<afmm_status> rc(G, AFMM_OK);
  std::vector<afmm_error> errs(G);
  std::vector<afmm_op_counts> cnt(G);
  std::vector<cudaEvent_t> ev_a(G, nullptr);
  std::vector<float> total_ms(G, -1.f), compute_ms(G, -1.f);
  unsigned long long fstats[4] = {0, 0, 0, 0};
  uint32_t rep_max = 0, rep_neg = 0;  // merged rep statistics (group-kernel choice)
  Barrier bar(G);
  bool failed = false;  // set by shard 0 between the barriers
  const int sms = sm_count(devs[0]);
  afmm_timing* timing = opt->timing;

  auto shard = [&](int g) {
    afmm_context* c = ctx[g];
    afmm_error* er = &errs[g];
    auto fail = [&](cudaError_t ce, const char* what) {
      rc[g] = cuda_fail(er, ce, what);
    };
    cudaSetDevice(c->device);
    cudaStream_t s = c->stream;
    const uint64_t a0 = e[g], a1 = e[g + 1];
    // ---- A: chunk copies + validation ----
    cudaError_t ce = cudaSuccess;
    if (ce == cudaSuccess) ce = c->hx.ensure(mat);
    if (ce == cudaSuccess) ce = c->hy.ensure(mat);
    if (ce == cudaSuccess && !zmapped) ce = c->hz.ensure(mat);
    if (ce == cudaSuccess) ce = c->status.ensure(sizeof(DevStatus));
    if (ce == cudaSuccess) ce = c->vec_k.ensure(n * 8);
    if (ce == cudaSuccess) ce = c->work.ensure(n * 8);
    if (ce == cudaSuccess && which == AFMM_CASE_A) ce = c->acounts.ensure(n * 4);
    if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&ev_a[g], cudaEventDisableTiming);
    if (ce == cudaSuccess && timing && ensure_host_events(c) != AFMM_OK) ce = cudaErrorUnknown;
    if (ce == cudaSuccess && timing) ce = cudaEventRecord(c->hev[0], s);
    auto* st = c->status.as<DevStatus>();
    if (ce == cudaSuccess && a1 > a0) {
      ce = cudaMemcpy2DAsync(c->hx.as<char>() + a0 * row_bytes, row_bytes, lhs + a0 * n,
                             n * sizeof(T), n * sizeof(T), a1 - a0, cudaMemcpyHostToDevice, s);
      if (ce == cudaSuccess)
        ce = cudaMemcpy2DAsync(c->hy.as<char>() + a0 * row_bytes, row_bytes, rhs + a0 * n,
                               n * sizeof(T), n * sizeof(T), a1 - a0, cudaMemcpyHostToDevice, s);
    }
    if (ce == cudaSuccess) ce = cudaMemsetAsync(st, 0, sizeof(DevStatus), s);
    if (ce == cudaSuccess)
      afmm_dev::launch_scan_stats<T>(c->hx.as<T>(), c->hy.as<T>(), ld, (uint32_t)n,
                                     which == AFMM_CASE_B ? 1 : 0, (uint32_t)a0, (uint32_t)a1,
                                     (uint32_t)a0, (uint32_t)a1, st, c->vec_k.as<uint32_t>(),
                                     c->vec_k.as<unsigned long long>(), s, check_finite ? 1 : 0);
    if (ce == cudaSuccess) ce = afmm_dev::take_launch_error();
    if (ce == cudaSuccess) ce = cudaEventRecord(ev_a[g], s);
    if (ce != cudaSuccess) fail(ce, "afmm: shard setup");
    bar.wait();  // every chunk's copy and scan is enqueued (events recorded)
    // ---- B: complete Y and the per-k vector, W_i of the chunk ----
    const size_t vk = which == AFMM_CASE_B ? sizeof(uint32_t) : sizeof(unsigned long long);
    for (int h = 0; h < G && rc[g] == AFMM_OK; ++h) {
      if (h == g || e[h + 1] == e[h]) continue;
      afmm_context* p = ctx[h];
      if (rc[h] != AFMM_OK) continue;
      ce = cudaStreamWaitEvent(s, ev_a[h], 0);
      if (ce == cudaSuccess)
        ce = cudaMemcpyPeerAsync(c->hy.as<char>() + e[h] * row_bytes, c->device,
                                 p->hy.as<char>() + e[h] * row_bytes, p->device,
                                 (e[h + 1] - e[h]) * row_bytes, s);
      if (ce == cudaSuccess)
        ce = cudaMemcpyPeerAsync(c->vec_k.as<char>() + e[h] * vk, c->device,
                                 p->vec_k.as<char>() + e[h] * vk, p->device,
                                 (e[h + 1] - e[h]) * vk, s);
      if (ce != cudaSuccess) fail(ce, "afmm: peer copy");
    }
    if (rc[g] == AFMM_OK) {
      afmm_dev::launch_rows<T>(c->hx.as<T>(), ld, (uint32_t)n, which == AFMM_CASE_B ? 1 : 0,
                               c->vec_k.as<uint32_t>(), c->vec_k.as<unsigned long long>(),
                               (uint32_t)a0, (uint32_t)a1, (uint32_t)a0, (uint32_t)a1, nullptr, 0,
                               nullptr, c->work.as<unsigned long long>(), st, s,
                               which == AFMM_CASE_A ? c->acounts.as<uint32_t>() + 0 : nullptr);
      ce = cudaSuccess;
      if (which == AFMM_CASE_A) {
        // A-form counts / statistics of the (now complete) Y, used by the
        // partition here and by this shard's product in C
        const uint32_t tc = afmm_dev::aform_tile_cols<T>();
        const uint64_t ntiles = (n + tc - 1) / tc, ldc = round_up(n, 64);
        ce = c->cnt16.ensure(n * ldc * sizeof(__half));
        if (ce == cudaSuccess) ce = c->rmax.ensure(n * ntiles * sizeof(uint16_t));
        if (ce == cudaSuccess) ce = c->fstats.ensure(4 * sizeof(unsigned long long));
        if (ce == cudaSuccess)
          ce = cudaMemsetAsync(c->fstats.p, 0, 4 * sizeof(unsigned long long), s);
        if (ce == cudaSuccess)
          afmm_dev::launch_counts_f16<T>(c->hy.as<T>(), ld, (uint32_t)n, tc,
                                         c->cnt16.as<__half>(), ldc, c->rmax.as<uint16_t>(),
                                         c->fstats.as<unsigned long long>(), s);
        // nnz_row of the chunk rows (slab-relative index = i - a0)
        if (ce == cudaSuccess && a1 > a0)
          ce = cudaMemcpyAsync(nnz_row.data() + a0, c->acounts.p, (a1 - a0) * 4,
                               cudaMemcpyDeviceToHost, s);
        if (ce == cudaSuccess && g == 0)
          ce = cudaMemcpyAsync(c->stats_host, c->fstats.p, 4 * sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, s);
      }
      if (ce == cudaSuccess) ce = afmm_dev::take_launch_error();
      if (ce == cudaSuccess && a1 > a0)
        ce = cudaMemcpyAsync(work.data() + a0, c->work.as<uint64_t>() + a0, (a1 - a0) * 8,
                             cudaMemcpyDeviceToHost, s);
      if (ce == cudaSuccess)
        ce = cudaMemcpyAsync(c->status_host, st, sizeof(DevStatus), cudaMemcpyDeviceToHost, s);
      if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
      if (ce != cudaSuccess) fail(ce, "afmm: shard statistics");
      else stat[g] = *c->status_host;
    }
    bar.wait();
    if (g == 0) {
      // ---- merge the statuses; cut the rows ----
      for (int h = 0; h < G; ++h)
        if (rc[h] != AFMM_OK) {
          failed = true;
          if (err) *err = errs[h];
          rc[0] = rc[h];
          break;
        }
      if (!failed) {
        DevStatus all{};
        for (int h = 0; h < G; ++h) merge_status(&all, stat[h]);
        rep_max = all.rep_max;
        rep_neg = all.rep_neg;
        const afmm_status dst =
            decode_status(all, which, n, host_reader(lhs, rhs, dtype, n), nullptr, err);
        if (dst != AFMM_OK) {
          failed = true;
          rc[0] = dst;
        }
      }
      if (!failed) {
        if (which == AFMM_CASE_A) std::memcpy(fstats, ctx[0]->stats_host, sizeof fstats);
        if (opt->partition == AFMM_PARTITION_ROWS) {
          cuts = e;
        } else {
          // the B part's kernel as the shards will choose it (group_mode)
          Call probe;
          probe.dtype = dtype;
          probe.mode = mode;
          const bool grp = group_allow(ctx[0], probe) && rep_max <= afmm_dev::kGroupMaxRep &&
                           rep_neg == 0;
          partition_from_stats(which, sizeof(T), n, sms, work.data(),
                               which == AFMM_CASE_A ? nnz_row.data() : nullptr, fstats,
                               (uint32_t)G, cuts.data(), grp);
        }
      }
    }
    bar.wait();
    if (failed) return;
    // ---- C: the rows of the cut this shard lacks, then its product ----
    const uint64_t r0 = cuts[g], r1 = cuts[g + 1];
    for (int h = 0; h < G; ++h) {
      if (h == g) continue;
      const uint64_t lo = std::max(r0, e[h]), hi = std::min(r1, e[h + 1]);
      if (hi <= lo) continue;
      ce = cudaMemcpyPeerAsync(c->hx.as<char>() + lo * row_bytes, c->device,
                               ctx[h]->hx.as<char>() + lo * row_bytes, ctx[h]->device,
                               (hi - lo) * row_bytes, s);
      if (ce != cudaSuccess) {
        fail(ce, "afmm: peer copy");
        return;
      }
    }
    Call call;
    call.which = which;
    call.dtype = dtype;
    call.mode = mode;
    call.split_k = opt->split_k;
    call.check_finite = check_finite;
    call.lhs = c->hx.p;
    call.rhs = c->hy.p;
    call.n = n;
    call.ld = ld;
    call.out = zmapped ? static_cast<void*>(zmapped + r0 * n) : c->hz.p;
    call.ld_out = zmapped ? n : ld;
    call.r0 = r0;
    call.r1 = r1;
    call.prevalidated = true;
    call.rep_max = rep_max;
    call.rep_neg = rep_neg;
    call.have_counts = which == AFMM_CASE_A;
    const bool kernel_timing = c->timing;
    if (timing) enable_timing_locked(c, 1);
    afmm_status st2 = enqueue_call(c, call, er);
    if (st2 == AFMM_OK) st2 = finish_locked(c, &cnt[g], er);
    if (st2 == AFMM_OK && !zmapped && r1 > r0) {
      ce = cudaMemcpy2DAsync(out + r0 * n, n * sizeof(T), c->hz.p, row_bytes, n * sizeof(T),
                             r1 - r0, cudaMemcpyDeviceToHost, s);
      if (ce == cudaSuccess && timing) ce = cudaEventRecord(c->hev[1], s);
      if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
      if (ce != cudaSuccess) st2 = cuda_fail(er, ce, "afmm: D2H");
    } else if (st2 == AFMM_OK && timing) {
      cudaEventRecord(c->hev[1], s);
      cudaStreamSynchronize(s);
    }
    if (timing && st2 == AFMM_OK) {
      cudaEventElapsedTime(&total_ms[g], c->hev[0], c->hev[1]);
      cudaEventElapsedTime(&compute_ms[g], c->last_ev[1], c->last_ev[2]);
    }
    if (timing && !kernel_timing) enable_timing_locked(c, 0);
    rc[g] = st2;
  };

  std::vector<std::thread> threads;
  for (int g = 1; g < G; ++g) threads.emplace_back(shard, g);
  shard(0);
  for (auto& t : threads) t.join();
  for (int g = 0; g < G; ++g) {
    if (ev_a[g]) {
      cudaSetDevice(ctx[g]->device);
      cudaEventDestroy(ev_a[g]);
    }
  }
  if (failed) return rc[0];
  for (int g = 0; g < G; ++g)
    if (rc[g] != AFMM_OK) {
      if (err) *err = errs[g];
      return rc[g];
    }
  if (counts) {
    *counts = afmm_op_counts{0, 0, 0};
    for (int g = 0; g < G; ++g) {
      counts->additions += cnt[g].additions;
      counts->zero_skips += cnt[g].zero_skips;
    }
  }
  if (timing) {
    timing->total_ms = *std::max_element(total_ms.begin(), total_ms.end());
    timing->compute_ms = *std::max_element(compute_ms.begin(), compute_ms.end());
    timing->devices = G;
    timing->form = ctx[0]->last_form;
  }
  clear_error(err);
  return AFMM_OK;
}

template <class T>
afmm_status host_product(int which, const T* lhs, uint64_t n_lhs, const T* rhs, uint64_t n_rhs,
                         T* out, const afmm_options* opt, afmm_op_counts* counts,
                         afmm_error* err) {
  clear_error(err);
  afmm_status st = check_dims(which, n_lhs, n_rhs, err);
  if (st != AFMM_OK) return st;
  st = check_options(opt, err);
  if (st != AFMM_OK) return st;
  if (!lhs || !rhs || !out) {
    set_error(err, AFMM_ERRKIND_OTHER, 0, 0, 0, 0.0, "afmm: null pointer argument");
    return AFMM_ERR_INVALID_ARGUMENT;
  }
  if (opt && opt->num_devices > 1)
    return host_product_multi<T>(which, lhs, rhs, n_lhs, out, opt, counts, err);
  return host_product_one<T>(which, lhs, rhs, n_lhs, out, opt, counts, err);
}

template <class F>
afmm_status guarded(F f) {
  try {
    return f();
  } catch (const std::bad_alloc&) {
    return AFMM_ERR_OUT_OF_MEMORY;
  } catch (...) {
    return AFMM_ERR_CUDA;
  }
}

}  // namespace

// ---- seeded generation (random.hpp:60-129) ----------------------------------

// validate() of random.hpp:60-79: the same checks, order and messages
// (std::invalid_argument).
afmm_status check_gen_spec(const afmm_generator_spec* sp, afmm_error* err) {
  auto bad = [&](const char* m) {
    set_error(err, AFMM_ERRKIND_OTHER, 0, 0, 0, 0.0, m);
    return AFMM_ERR_INVALID_ARGUMENT;
  };
  if (!sp) return bad("afmm: null generator spec");
  if (sp->n == 0) return bad("GeneratorSpec: n must be >= 1");
  if (!(sp->density >= 0.0 && sp->density <= 1.0))
    return bad("GeneratorSpec: density must be in [0, 1]");
  if (!(sp->mu_prime > 0.0)) return bad("GeneratorSpec: mu_prime must be positive");
  if (sp->role == AFMM_ROLE_INTEGER) {
    if (std::fabs(sp->mu_prime - std::round(sp->mu_prime)) > 1e-9 || sp->mu_prime < 1.0)
      return bad("GeneratorSpec: IntegerValued role requires integer mu_prime >= 1");
  } else if (sp->role == AFMM_ROLE_REAL) {
    if (!(std::isfinite(sp->value_low) && std::isfinite(sp->value_high)) ||
        sp->value_low > sp->value_high)
      return bad("GeneratorSpec: invalid value bounds");
  } else {
    return bad("afmm: unknown generator role");
  }
  if (sp->n > 0x7fffffffull) {
    set_error(err, AFMM_ERRKIND_OTHER, 0, 0, 0, 0.0, "afmm: n beyond 2^31 - 1");
    return AFMM_ERR_UNSUPPORTED;
  }
  return AFMM_OK;
}

// The jump polynomials of the generation tree: per level l (stride 4^l
// stretches of L = kGenTwistsPerCta x 312 draws), x^(a 4^l L) mod phi for
// a = 1, 2, 3 (mt64jump.h); computed once per process (~30 ms of host time).
const std::vector<uint64_t>& gen_jump_polys() {
  static const std::vector<uint64_t> table = [] {
    const auto& f = mt64jump::field();
    std::vector<uint64_t> t;
    if (!f.ok) return t;  // cannot happen for MT19937-64; reported by the caller
    mt64jump::Poly p = f.xpow((uint64_t)afmm_dev::kGenTwistsPerCta * mt64jump::kN);
    for (uint32_t l = 0; l < afmm_dev::kGenLevels; ++l) {
      const mt64jump::Poly p2 = f.mulmod(p, p), p3 = f.mulmod(p2, p);
      t.insert(t.end(), p.begin(), p.end());
      t.insert(t.end(), p2.begin(), p2.end());
      t.insert(t.end(), p3.begin(), p3.end());
      p = f.mulmod(p2, p2);
    }
    return t;
  }();
  return table;
}

// afmm::generate (random.hpp:111-129) into device memory on the context's
// stream: chunks of the MT19937-64 stream until every entry is complete
// (generate.cu). A chunk is up to kGenMaxCtas stretches of L draws generated
// in parallel from jump-ahead start windows; one host round trip per chunk
// (the carry decides whether another chunk is needed); a chunk holds up to
// 3.3e8 draws, so a matrix up to n ~ 13000 is one chunk.
template <class T>
afmm_status generate_locked(afmm_context* c, const afmm_generator_spec& sp, uint64_t seed, T* out,
                            uint64_t ld, afmm_error* err) {
  cudaStream_t s = c->stream;
  const uint64_t n = sp.n, nn = n * n;
  afmm_dev::take_launch_error();
  CK(cudaMemset2DAsync(out, ld * sizeof(T), 0, n * sizeof(T), n, s), "memset");
  if (sp.density == 0.0) {  // every Bernoulli draw says zero (uniform01 >= 0)
    CK(cudaStreamSynchronize(s), "generate");
    return AFMM_OK;
  }
  const std::vector<uint64_t>& polys = gen_jump_polys();
  if (polys.empty()) {
    set_error(err, AFMM_ERRKIND_OTHER, 0, 0, 0, 0.0, "afmm: MT19937-64 jump table unavailable");
    return AFMM_ERR_CUDA;
  }
  uint64_t win[mt64jump::kN];  // std::mt19937_64(seed) after its first twist
  mt64jump::seed_window(seed, win);
  afmm_dev::GenSpecDev g;
  g.n = n;
  g.density = sp.density;
  g.low = sp.value_low;
  g.high = sp.value_high;
  g.integer = sp.role == AFMM_ROLE_INTEGER ? 1 : 0;
  if (g.integer) {
    g.range = 2 * (uint64_t)std::llround(sp.mu_prime) - 1;
    g.limit = UINT64_MAX - UINT64_MAX % g.range;  // random.hpp:97-99
  }
  // draws still needed: one per entry + one per nonzero entry (+ the
  // astronomically rare rejections), 1% slack; whole stretches, except that a
  // one-stretch chunk stops at the twist that covers it
  constexpr uint64_t kL = (uint64_t)afmm_dev::kGenTwistsPerCta * mt64jump::kN;
  auto shape_for = [&](uint64_t entries, uint32_t* ctas, uint32_t* twists) {
    const double rem = entries < nn ? (double)(nn - entries) : 0.0;
    const uint64_t need = (uint64_t)std::ceil(rem * (1.0 + sp.density) * 1.01) + mt64jump::kN;
    const uint64_t k = (need + kL - 1) / kL;
    *ctas = (uint32_t)std::min<uint64_t>(k, afmm_dev::kGenMaxCtas);
    *twists = *ctas > 1 ? afmm_dev::kGenTwistsPerCta
                        : (uint32_t)std::min<uint64_t>((need + mt64jump::kN - 1) / mt64jump::kN,
                                                       afmm_dev::kGenTwistsPerCta);
  };
  uint32_t ctas0, tw0;
  shape_for(0, &ctas0, &tw0);
  const uint64_t cap = (uint64_t)ctas0 * tw0 * mt64jump::kN;
  const size_t wbytes = (size_t)mt64jump::kN * sizeof(uint64_t);
  CK(c->gen_state.ensure(wbytes * (afmm_dev::kGenMaxCtas + 1)), "workspace");
  CK(c->gen_polys.ensure(polys.size() * sizeof(uint64_t)), "workspace");
  CK(c->gen_draws.ensure(cap * 8), "workspace");
  CK(c->gen_scratch.ensure(afmm_dev::gen_scratch_bytes(cap)), "workspace");
  CK(c->gen_carry.ensure(afmm_dev::gen_carry_bytes()), "workspace");
  uint64_t* windows = c->gen_state.as<uint64_t>();
  uint64_t* end_window = windows + (size_t)afmm_dev::kGenMaxCtas * mt64jump::kN;
  CK(cudaMemcpyAsync(c->gen_polys.p, polys.data(), polys.size() * sizeof(uint64_t),
                     cudaMemcpyHostToDevice, s),
     "copy");
  CK(cudaMemcpyAsync(windows, win, wbytes, cudaMemcpyHostToDevice, s), "copy");
  CK(cudaMemsetAsync(c->gen_carry.p, 0, afmm_dev::gen_carry_bytes(), s), "memset");
  uint64_t entries = 0;
  uint32_t state = 0;
  for (bool first = true;; first = false) {
    uint32_t ctas, tw;
    shape_for(entries, &ctas, &tw);
    if (!first)  // the next chunk starts where the last one ended
      CK(cudaMemcpyAsync(windows, end_window, wbytes, cudaMemcpyDeviceToDevice, s), "copy");
    CK(afmm_dev::launch_generate_chunk<T>(g, windows, c->gen_polys.as<uint64_t>(), ctas, tw,
                                          end_window, c->gen_draws.as<uint64_t>(),
                                          c->gen_scratch.p, c->gen_carry.p, out, ld, s),
       "generate");
    CK(afmm_dev::take_launch_error(), "generate");
    CK(cudaMemcpyAsync(c->stats_host, c->gen_carry.p, afmm_dev::gen_carry_bytes(),
                       cudaMemcpyDeviceToHost, s),
       "carry readback");
    CK(cudaStreamSynchronize(s), "generate");
    state = (uint32_t)(c->stats_host[0] & 0xffffffffull);
    entries = c->stats_host[1];
    // every entry started, and the last one's value drawn
    if (entries > nn || (entries == nn && state == 0)) break;
  }
  return AFMM_OK;
}

template <class T>
afmm_status generate_host(const afmm_generator_spec* spec, uint64_t seed, T* out,
                          const afmm_options* opt, afmm_error* err) {
  clear_error(err);
  afmm_status st = check_gen_spec(spec, err);
  if (st != AFMM_OK) return st;
  if (!out) {
    set_error(err, AFMM_ERRKIND_OTHER, 0, 0, 0, 0.0, "afmm: null output");
    return AFMM_ERR_INVALID_ARGUMENT;
  }
  return guarded([&]() -> afmm_status {
    afmm_context* c = nullptr;
    afmm_status s0 = default_context(opt ? opt->device : -1, 0, &c, err);
    if (s0 != AFMM_OK) return s0;
    std::lock_guard<std::mutex> g(c->mu);
    CK(cudaSetDevice(c->device), "afmm: cudaSetDevice");
    if (c->pending) {
      afmm_status prev = finish_locked(c, nullptr, err);
      if (prev != AFMM_OK) return prev;
    }
    const uint64_t n = spec->n;
    CK(c->hz.ensure(n * n * sizeof(T)), "workspace");
    afmm_status r = generate_locked<T>(c, *spec, seed, c->hz.as<T>(), n, err);
    if (r != AFMM_OK) return r;
    if (HostStager::wants(out, n * sizeof(T), n) && c->stager.ensure(c->device) == cudaSuccess) {
      // pageable result: the staged pipeline (its threads also spread the first
      // touch of a fresh array)
      CK(cudaStreamSynchronize(c->stream), "generate");
      CK(c->stager.copy(false, out, n * sizeof(T), c->hz.p, n * sizeof(T), n * sizeof(T), n,
                        c->stream),
         "result copy");
    } else {
      CK(cudaMemcpyAsync(out, c->hz.p, n * n * sizeof(T), cudaMemcpyDeviceToHost, c->stream),
         "result copy");
      CK(cudaStreamSynchronize(c->stream), "result copy");
    }
    clear_error(err);
    return AFMM_OK;
  });
}

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------

extern "C" {

afmm_status afmm_case_a_f64(const double* lhs, uint64_t n_lhs, const double* rhs, uint64_t n_rhs,
                            double* out, const afmm_options* options, afmm_op_counts* counts,
                            afmm_error* error) {
  return guarded([&] {
    return host_product<double>(AFMM_CASE_A, lhs, n_lhs, rhs, n_rhs, out, options, counts, error);
  });
}

afmm_status afmm_case_b_f64(const double* lhs, uint64_t n_lhs, const double* rhs, uint64_t n_rhs,
                            double* out, const afmm_options* options, afmm_op_counts* counts,
                            afmm_error* error) {
  return guarded([&] {
    return host_product<double>(AFMM_CASE_B, lhs, n_lhs, rhs, n_rhs, out, options, counts, error);
  });
}

afmm_status afmm_case_a_f32(const float* lhs, uint64_t n_lhs, const float* rhs, uint64_t n_rhs,
                            float* out, const afmm_options* options, afmm_op_counts* counts,
                            afmm_error* error) {
  return guarded([&] {
    return host_product<float>(AFMM_CASE_A, lhs, n_lhs, rhs, n_rhs, out, options, counts, error);
  });
}

afmm_status afmm_case_b_f32(const float* lhs, uint64_t n_lhs, const float* rhs, uint64_t n_rhs,
                            float* out, const afmm_options* options, afmm_op_counts* counts,
                            afmm_error* error) {
  return guarded([&] {
    return host_product<float>(AFMM_CASE_B, lhs, n_lhs, rhs, n_rhs, out, options, counts, error);
  });
}

afmm_status afmm_context_create(int32_t device, afmm_context** ctx) {
  if (!ctx) return AFMM_ERR_INVALID_ARGUMENT;
  *ctx = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) return AFMM_ERR_CUDA;
  if (device < 0 && cudaGetDevice(&device) != cudaSuccess) return AFMM_ERR_CUDA;
  if (device >= count) return AFMM_ERR_INVALID_ARGUMENT;
  auto* c = new (std::nothrow) afmm_context;
  if (!c) return AFMM_ERR_OUT_OF_MEMORY;
  c->device = device;
  c->variant = variant_from_env();
  c->group_off = group_off_from_env();
  c->pack_off = pack_off_from_env();
  {
    const char* gv = std::getenv("AFMM_GRAPHS");
    c->graphs = !(gv && std::strcmp(gv, "0") == 0);
  }
  for (DevBuf* b : all_bufs(c)) b->gen = &c->buf_gen;
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaHostAlloc(reinterpret_cast<void**>(&c->status_host), sizeof(DevStatus),
                    cudaHostAllocDefault) != cudaSuccess ||
      cudaHostAlloc(reinterpret_cast<void**>(&c->stats_host), 4 * sizeof(unsigned long long),
                    cudaHostAllocDefault) != cudaSuccess) {
    if (c->status_host) cudaFreeHost(c->status_host);
    delete c;
    cudaSetDevice(prev);
    return AFMM_ERR_CUDA;
  }
  cudaSetDevice(prev);
  *ctx = c;
  return AFMM_OK;
}

void afmm_context_destroy(afmm_context* c) {
  if (!c) return;
  {
    std::lock_guard<std::mutex> g(c->mu);
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    if (c->gstream) cudaStreamSynchronize(c->gstream);
    for (auto& ge : c->graph_cache) ge.release();
    c->graph_cache.clear();
    if (c->gstream) cudaStreamDestroy(c->gstream);
    if (c->join_in) cudaEventDestroy(c->join_in);
    if (c->join_out) cudaEventDestroy(c->join_out);
    for (DevBuf* b : all_bufs(c)) b->release();
    if (c->status_host) cudaFreeHost(c->status_host);
    if (c->stats_host) cudaFreeHost(c->stats_host);
    c->stager.release();
    for (cudaEvent_t& e : c->ev)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t& e : c->hev)
      if (e) cudaEventDestroy(e);
  }
  delete c;
}

// Switching streams first drains a pending asynchronous product on the old
// stream (its status readback was queued there), so afmm_context_finish()
// still reports that product.
afmm_status afmm_context_set_stream(afmm_context* c, void* stream) {
  if (!c) return AFMM_ERR_INVALID_ARGUMENT;
  std::lock_guard<std::mutex> g(c->mu);
  if (c->pending) {
    cudaSetDevice(c->device);
    if (cudaStreamSynchronize(c->stream) != cudaSuccess) return AFMM_ERR_CUDA;
  }
  c->stream = static_cast<cudaStream_t>(stream);
  return AFMM_OK;
}

afmm_status afmm_product_device(afmm_context* c, int32_t which_case, int32_t dtype,
                                const void* lhs, const void* rhs, uint64_t n, uint64_t ld,
                                void* out, uint64_t ld_out, uint64_t row_begin, uint64_t row_end,
                                const afmm_options* options, int32_t sync,
                                afmm_op_counts* counts, afmm_error* err) {
  clear_error(err);
  if (!c || (which_case != AFMM_CASE_A && which_case != AFMM_CASE_B) ||
      (dtype != AFMM_F64 && dtype != AFMM_F32)) {
    set_error(err, AFMM_ERRKIND_OTHER, 0, 0, 0, 0.0, "afmm: invalid context/case/dtype");
    return AFMM_ERR_INVALID_ARGUMENT;
  }
  afmm_status st = check_dims(which_case, n, n, err);
  if (st != AFMM_OK) return st;
  st = check_options(options, err);
  if (st != AFMM_OK) return st;
  if (ld < n || ld_out < n || row_begin > row_end || row_end > n || !lhs || !rhs ||
      (!out && row_end > row_begin)) {
    set_error(err, AFMM_ERRKIND_OTHER, 0, 0, 0, 0.0, "afmm: invalid leading dimension / rows");
    return AFMM_ERR_INVALID_ARGUMENT;
  }
  return guarded([&]() -> afmm_status {
    std::lock_guard<std::mutex> g(c->mu);
    CK(cudaSetDevice(c->device), "afmm: cudaSetDevice");
    if (c->pending) {
      // a previous asynchronous product was never finished: report its
      // outcome instead of starting new work on top of it
      afmm_status prev = finish_locked(c, nullptr, err);
      if (prev != AFMM_OK) return prev;
    }
    if (out && out != c->peer_checked) {
      // `out` in another GPU's memory (a row shard storing into the device
      // that gathers Z): enable peer access so the kernels' stores go over NVLink
      cudaPointerAttributes attr{};
      if (cudaPointerGetAttributes(&attr, out) == cudaSuccess &&
          attr.type == cudaMemoryTypeDevice && attr.device != c->device)
        ensure_peer_access(c->device, attr.device);
      cudaGetLastError();
      c->peer_checked = out;
    }
    Call call;
    call.which = which_case;
    call.dtype = dtype;
    call.mode = options ? options->mode : AFMM_MODE_ORDER_PRESERVING;
    call.split_k = options ? options->split_k : 0;
    call.check_finite = !(options && (options->flags & AFMM_FLAG_KERNEL_SEMANTICS));
    call.lhs = lhs;
    call.rhs = rhs;
    call.n = n;
    call.ld = ld;
    call.out = out;
    call.ld_out = ld_out;
    call.r0 = row_begin;
    call.r1 = row_end;
    afmm_status s2 = graph_call(c, call, err);
    if (s2 != AFMM_OK) return s2;
    if (sync) return finish_locked(c, counts, err);
    return AFMM_OK;
  });
}

afmm_status afmm_context_finish(afmm_context* c, afmm_op_counts* counts, afmm_error* err) {
  if (!c) return AFMM_ERR_INVALID_ARGUMENT;
  std::lock_guard<std::mutex> g(c->mu);
  CK(cudaSetDevice(c->device), "afmm: cudaSetDevice");
  return guarded([&] { return finish_locked(c, counts, err); });
}

afmm_status afmm_context_enable_timing(afmm_context* c, int32_t enable) {
  if (!c) return AFMM_ERR_INVALID_ARGUMENT;
  std::lock_guard<std::mutex> g(c->mu);
  return enable_timing_locked(c, enable);
}

afmm_status afmm_context_last_timing(afmm_context* c, float* prepass_ms, float* compute_ms,
                                     float* epilogue_ms) {
  if (!c) return AFMM_ERR_INVALID_ARGUMENT;
  std::lock_guard<std::mutex> g(c->mu);
  float v[3] = {-1.f, -1.f, -1.f};
  if (c->timed_last && !c->pending) {
    for (int i = 0; i < 3; ++i)
      if (cudaEventElapsedTime(&v[i], c->last_ev[i], c->last_ev[i + 1]) != cudaSuccess)
        v[i] = -1.f;
  }
  if (prepass_ms) *prepass_ms = v[0];
  if (compute_ms) *compute_ms = v[1];
  if (epilogue_ms) *epilogue_ms = v[2];
  return AFMM_OK;
}

int32_t afmm_context_last_form(afmm_context* c) {
  if (!c) return -1;
  std::lock_guard<std::mutex> g(c->mu);
  return c->last_form;
}

}  // extern "C"

namespace {

// Statistics of the full operands on one context: W_i (work), and for Case A
// the nonzero bases per row and the statistics of Y. Host arrays out.
template <class T>
afmm_status row_stats(afmm_context* c, int which, const T* lhs, const T* rhs, uint64_t n,
                      uint64_t ld, uint64_t* work_host, std::vector<uint32_t>* nnz_row,
                      unsigned long long* fstats, afmm_error* err) {
  afmm_dev::take_launch_error();
  CK(c->vec_k.ensure(n * 8), "workspace");
  CK(c->work.ensure(n * 8), "workspace");
  CK(c->status.ensure(sizeof(DevStatus)), "workspace");
  cudaStream_t s = c->stream;
  auto* work = c->work.as<unsigned long long>();
  DevStatus* dst = c->status.as<DevStatus>();
  CK(cudaMemsetAsync(dst, 0, sizeof(DevStatus), s), "memset");
  const int cb = which == AFMM_CASE_B ? 1 : 0;
  const uint32_t n32 = (uint32_t)n;
  afmm_dev::launch_scan_stats<T>(lhs, rhs, ld, n32, cb, 0, 0, 0, n32, dst, c->vec_k.as<uint32_t>(),
                                 c->vec_k.as<unsigned long long>(), s);
  if (nnz_row) CK(c->acounts.ensure(n * 4), "workspace");
  afmm_dev::launch_rows<T>(lhs, ld, n32, cb, c->vec_k.as<uint32_t>(),
                           c->vec_k.as<unsigned long long>(), 0, n32, nnz_row ? 0 : n32,
                           nnz_row ? n32 : n32, nullptr, 0, nullptr, work, dst, s,
                           nnz_row ? c->acounts.as<uint32_t>() : nullptr);
  CK(cudaMemcpyAsync(work_host, work, n * 8, cudaMemcpyDeviceToHost, s), "work readback");
  if (nnz_row) {
    const uint32_t tc = afmm_dev::aform_tile_cols<T>();
    const uint64_t ntiles = (n + tc - 1) / tc, ldc = round_up(n, 64);
    CK(c->cnt16.ensure(n * ldc * sizeof(__half)), "workspace");
    CK(c->rmax.ensure(n * ntiles * sizeof(uint16_t)), "workspace");
    CK(c->fstats.ensure(4 * sizeof(unsigned long long)), "workspace");
    CK(cudaMemsetAsync(c->fstats.p, 0, 4 * sizeof(unsigned long long), s), "memset");
    afmm_dev::launch_counts_f16<T>(rhs, ld, n32, tc, c->cnt16.as<__half>(), ldc,
                                   c->rmax.as<uint16_t>(), c->fstats.as<unsigned long long>(), s);
    nnz_row->resize(n);
    CK(cudaMemcpyAsync(nnz_row->data(), c->acounts.p, n * 4, cudaMemcpyDeviceToHost, s),
       "readback");
    CK(cudaMemcpyAsync(c->stats_host, c->fstats.p, 4 * 8, cudaMemcpyDeviceToHost, s), "readback");
  }
  CK(afmm_dev::take_launch_error(), "launch");
  CK(cudaStreamSynchronize(s), "work readback");
  if (fstats && nnz_row) std::memcpy(fstats, c->stats_host, 4 * 8);
  return AFMM_OK;
}

// What a row query returns: W_i, the per-row cost, or the row cuts.
enum RowQuery { kQueryWork, kQueryCost, kQueryCuts };

afmm_status row_query(afmm_context* c, int32_t which, int32_t dtype, const void* lhs,
                      const void* rhs, uint64_t n, uint64_t ld, uint64_t* out, RowQuery q,
                      uint32_t parts, afmm_error* err) {
  clear_error(err);
  if (!c || !out || (dtype != AFMM_F64 && dtype != AFMM_F32) ||
      (which != AFMM_CASE_A && which != AFMM_CASE_B) || !lhs || !rhs ||
      (q == kQueryCuts && parts == 0))
    return AFMM_ERR_INVALID_ARGUMENT;
  afmm_status st = check_dims(which, n, n, err);
  if (st != AFMM_OK) return st;
  if (ld < n) return AFMM_ERR_INVALID_ARGUMENT;
  return guarded([&]() -> afmm_status {
    std::lock_guard<std::mutex> g(c->mu);
    CK(cudaSetDevice(c->device), "afmm: cudaSetDevice");
    const bool case_a_model = q != kQueryWork && which == AFMM_CASE_A;
    std::vector<uint32_t> nnz;
    unsigned long long fstats[4] = {0, 0, 0, 0};
    std::vector<uint64_t> work(q == kQueryWork ? 0 : n);
    uint64_t* w = q == kQueryWork ? out : work.data();
    afmm_status r =
        dtype == AFMM_F64
            ? row_stats<double>(c, which, static_cast<const double*>(lhs),
                                static_cast<const double*>(rhs), n, ld, w,
                                case_a_model ? &nnz : nullptr, fstats, err)
            : row_stats<float>(c, which, static_cast<const float*>(lhs),
                               static_cast<const float*>(rhs), n, ld, w,
                               case_a_model ? &nnz : nullptr, fstats, err);
    if (r != AFMM_OK || q == kQueryWork) return r;
    const size_t elem = dtype == AFMM_F64 ? 8 : 4;
    const int sms = sm_count(c->device);
    if (q == kQueryCost)
      row_costs(which, elem, n, sms, w, case_a_model ? nnz.data() : nullptr, fstats, out);
    else
      partition_from_stats(which, elem, n, sms, w, case_a_model ? nnz.data() : nullptr, fstats,
                           parts, out);
    return AFMM_OK;
  });
}

}  // namespace

extern "C" {

afmm_status afmm_row_work_device(afmm_context* c, int32_t which_case, int32_t dtype,
                                 const void* lhs, const void* rhs, uint64_t n, uint64_t ld,
                                 uint64_t* work_host, afmm_error* err) {
  return row_query(c, which_case, dtype, lhs, rhs, n, ld, work_host, kQueryWork, 0, err);
}

afmm_status afmm_row_cost_device(afmm_context* c, int32_t which_case, int32_t dtype,
                                 const void* lhs, const void* rhs, uint64_t n, uint64_t ld,
                                 uint64_t* cost, afmm_error* err) {
  return row_query(c, which_case, dtype, lhs, rhs, n, ld, cost, kQueryCost, 0, err);
}

afmm_status afmm_partition_device(afmm_context* c, int32_t which_case, int32_t dtype,
                                  const void* lhs, const void* rhs, uint64_t n, uint64_t ld,
                                  uint32_t parts, uint64_t* cuts, afmm_error* err) {
  return row_query(c, which_case, dtype, lhs, rhs, n, ld, cuts, kQueryCuts, parts, err);
}

afmm_status afmm_model_partition_case_a(int32_t dtype, uint64_t n, int32_t sms,
                                        const uint64_t* stats, const uint32_t* nnz_row,
                                        uint32_t parts, uint64_t* cuts, double* slab_cycles) {
  if (!stats || !nnz_row || !cuts || parts == 0 || n == 0 ||
      (dtype != AFMM_F64 && dtype != AFMM_F32))
    return AFMM_ERR_INVALID_ARGUMENT;
  return guarded([&]() -> afmm_status {
    const size_t elem = dtype == AFMM_F64 ? 8 : 4;
    const int s = sms > 0 ? sms : 148;
    const unsigned long long fs[4] = {stats[0], stats[1], stats[2], stats[3]};
    std::vector<uint64_t> cost(n);
    row_costs(AFMM_CASE_A, elem, n, s, nullptr, nnz_row, fs, cost.data());
    afmm_dev::CaseAModel md = case_a_model(elem, n, s, pick_shape(kAuto, n, n, elem, s));
    md.nnz_y = fs[0];
    md.trip_sum = fs[1];
    md.rep_sum = fs[3];
    partition_case_a(md, nnz_row, fs[2] == 0, cost.data(), parts, cuts, slab_cycles);
    return AFMM_OK;
  });
}

afmm_status afmm_model_slab_time_case_a(int32_t dtype, uint64_t n, int32_t sms,
                                        const uint64_t* stats, const uint32_t* nnz_row,
                                        uint64_t row_begin, uint64_t row_end, double* cycles) {
  if (!stats || !nnz_row || !cycles || n == 0 || row_begin > row_end || row_end > n ||
      (dtype != AFMM_F64 && dtype != AFMM_F32))
    return AFMM_ERR_INVALID_ARGUMENT;
  return guarded([&]() -> afmm_status {
    const size_t elem = dtype == AFMM_F64 ? 8 : 4;
    const int s = sms > 0 ? sms : 148;
    afmm_dev::CaseAModel md = case_a_model(elem, n, s, pick_shape(kAuto, n, n, elem, s));
    md.nnz_y = stats[0];
    md.trip_sum = stats[1];
    md.rep_sum = stats[3];
    SlabModel sm(md, nnz_row, stats[2] == 0);
    *cycles = sm.time(row_begin, row_end);
    return AFMM_OK;
  });
}

afmm_status afmm_partition_rows(const uint64_t* work, uint64_t n, uint32_t parts, uint64_t* cuts) {
  if (!work || !cuts || parts == 0) return AFMM_ERR_INVALID_ARGUMENT;
  // Prefix sums in 128-bit-safe form: total may exceed 2^64 only for absurd
  // reps; saturate.
  unsigned __int128 total = 0;
  for (uint64_t i = 0; i < n; ++i) total += work[i];
  cuts[0] = 0;
  unsigned __int128 acc = 0;
  uint64_t i = 0;
  for (uint32_t p = 1; p < parts; ++p) {
    // smallest row index whose prefix reaches p/parts of the total, rounding
    // to the nearer boundary
    const unsigned __int128 target = total * p / parts;
    while (i < n && acc + work[i] <= target) acc += work[i++];
    if (i < n && acc < target) {
      const unsigned __int128 over = acc + work[i] - target, under = target - acc;
      if (over < under) acc += work[i++];
    }
    cuts[p] = std::max<uint64_t>(i, cuts[p - 1]);
  }
  cuts[parts] = n;
  return AFMM_OK;
}

afmm_status afmm_generate_f64(const afmm_generator_spec* spec, uint64_t seed, double* out,
                              const afmm_options* options, afmm_error* err) {
  return generate_host<double>(spec, seed, out, options, err);
}

afmm_status afmm_generate_f32(const afmm_generator_spec* spec, uint64_t seed, float* out,
                              const afmm_options* options, afmm_error* err) {
  return generate_host<float>(spec, seed, out, options, err);
}

afmm_status afmm_generate_device(afmm_context* c, const afmm_generator_spec* spec, uint64_t seed,
                                 int32_t dtype, void* out, uint64_t ld, afmm_error* err) {
  clear_error(err);
  afmm_status st = check_gen_spec(spec, err);
  if (st != AFMM_OK) return st;
  if (!c || !out || ld < spec->n || (dtype != AFMM_F64 && dtype != AFMM_F32)) {
    set_error(err, AFMM_ERRKIND_OTHER, 0, 0, 0, 0.0, "afmm: invalid context/output/dtype");
    return AFMM_ERR_INVALID_ARGUMENT;
  }
  return guarded([&]() -> afmm_status {
    std::lock_guard<std::mutex> g(c->mu);
    CK(cudaSetDevice(c->device), "afmm: cudaSetDevice");
    if (c->pending) {
      afmm_status prev = finish_locked(c, nullptr, err);
      if (prev != AFMM_OK) return prev;
    }
    return dtype == AFMM_F64
               ? generate_locked<double>(c, *spec, seed, static_cast<double*>(out), ld, err)
               : generate_locked<float>(c, *spec, seed, static_cast<float*>(out), ld, err);
  });
}

afmm_status afmm_fp_add_peak(int32_t device, int32_t dtype, double* adds_per_second,
                             double* sm_clock_mhz) {
  int prev = 0;
  if (cudaGetDevice(&prev) != cudaSuccess) return AFMM_ERR_CUDA;
  if (device >= 0 && cudaSetDevice(device) != cudaSuccess) return AFMM_ERR_CUDA;
  cudaError_t e = afmm_dev::run_peak(dtype, adds_per_second, sm_clock_mhz);
  cudaSetDevice(prev);
  return e == cudaSuccess ? AFMM_OK : AFMM_ERR_CUDA;
}

}  // extern "C"

// ---- peer-memory output -----------------------------------------------------

namespace {
std::mutex g_ipc_mu;
std::vector<std::pair<void*, void*>> g_ipc_open;  // (pointer handed out, mapped base)
}  // namespace

extern "C" {

afmm_status afmm_ipc_export(const void* dev_ptr, afmm_ipc_handle* handle, afmm_error* err) {
  clear_error(err);
  if (!dev_ptr || !handle) return AFMM_ERR_INVALID_ARGUMENT;
  static PFN_cuMemGetAddressRange_v3020 range_fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      range_fn = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(p);
  });
  CUdeviceptr base = 0;
  size_t size = 0;
  if (!range_fn || range_fn(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS) {
    set_error(err, AFMM_ERRKIND_OTHER, 0, 0, 0, 0.0,
              "afmm: cuMemGetAddressRange failed (not a device allocation)");
    return AFMM_ERR_INVALID_ARGUMENT;
  }
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return cuda_fail(err, e, "afmm: cudaIpcGetMemHandle");
  static_assert(sizeof(h) <= sizeof(handle->bytes), "IPC handle size");
  std::memset(handle->bytes, 0, sizeof(handle->bytes));
  std::memcpy(handle->bytes, &h, sizeof(h));
  handle->offset = reinterpret_cast<CUdeviceptr>(dev_ptr) - base;
  return AFMM_OK;
}

afmm_status afmm_ipc_open(int32_t device, const afmm_ipc_handle* handle, void** dev_ptr,
                          afmm_error* err) {
  clear_error(err);
  if (!handle || !dev_ptr) return AFMM_ERR_INVALID_ARGUMENT;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(err, e, "afmm: cudaSetDevice");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle->bytes, sizeof(h));
  void* base = nullptr;
  e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
  cudaSetDevice(prev);
  if (e != cudaSuccess) return cuda_fail(err, e, "afmm: cudaIpcOpenMemHandle");
  *dev_ptr = static_cast<char*>(base) + handle->offset;
  std::lock_guard<std::mutex> g(g_ipc_mu);
  g_ipc_open.emplace_back(*dev_ptr, base);
  return AFMM_OK;
}

afmm_status afmm_ipc_close(void* dev_ptr) {
  void* base = nullptr;
  {
    std::lock_guard<std::mutex> g(g_ipc_mu);
    for (size_t i = 0; i < g_ipc_open.size(); ++i)
      if (g_ipc_open[i].first == dev_ptr) {
        base = g_ipc_open[i].second;
        g_ipc_open.erase(g_ipc_open.begin() + i);
        break;
      }
  }
  if (!base) return AFMM_ERR_INVALID_ARGUMENT;
  return cudaIpcCloseMemHandle(base) == cudaSuccess ? AFMM_OK : AFMM_ERR_CUDA;
}

uint64_t afmm_kernel_launch_count(void) {
  return afmm_dev::g_launches.load(std::memory_order_relaxed);
}

const char* afmm_status_string(afmm_status s) {
  switch (s) {
    case AFMM_OK: return "ok";
    case AFMM_ERR_SHAPE: return "shape_error";
    case AFMM_ERR_DOMAIN: return "domain_error";
    case AFMM_ERR_INVALID_ARGUMENT: return "invalid_argument";
    case AFMM_ERR_CUDA: return "cuda_error";
    case AFMM_ERR_UNSUPPORTED: return "unsupported";
    case AFMM_ERR_OUT_OF_MEMORY: return "out_of_memory";
  }
  return "unknown";
}

int32_t afmm_abi_version(void) { return AFMM_B200_ABI_VERSION; }

}  // extern "C"
