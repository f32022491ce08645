/*
 * afmm_b200.h -- C ABI of the B200-native AFMM product (libafmm_b200.so).
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/proj/include/afmm/kernels.hpp):
 *
 *   afmm_case_a_f64  replaces afmm::afmm_case_a(const DenseMatrix&, const DenseMatrix&)
 *                    kernels.hpp:113-136 (real lhs bases, integer rhs reps)
 *   afmm_case_b_f64  replaces afmm::afmm_case_b(...)      kernels.hpp:142-165
 *                    (integer lhs reps, real rhs bases)
 *   afmm_case_{a,b}_f32  the same contract on fp32 storage (the reference is
 *                    fp64-only, proj/README.md:91; BASELINE configs 3-5 are fp32)
 *
 * Plain pointers and sizes only. Inputs are caller-owned row-major n x n
 * host arrays, element (i,j) at p[i*n+j] (matrix.hpp:41-46); the product is
 * written to a caller-owned n x n host array; counts are the reference's
 * OpCounts (op_counts.hpp:17-23). The C ABI cannot throw, so it returns an
 * afmm_status plus an afmm_error naming the first offender; the C++ wrapper
 * include/afmm_b200/kernels.hpp rethrows the reference's exception types
 * with the reference's message text (kernels.hpp:17-19, 32-39; matrix.hpp:55).
 *
 * All compute runs on sm_100a CUDA kernels. There is no CPU fallback: without
 * a usable B200 every compute entry returns AFMM_ERR_CUDA.
 */
#ifndef AFMM_B200_H
#define AFMM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AFMM_B200_ABI_VERSION 2

typedef enum {
  AFMM_OK = 0,
  AFMM_ERR_SHAPE = 1,            /* afmm::shape_error (dimension mismatch)               */
  AFMM_ERR_DOMAIN = 2,           /* std::domain_error (rep not integer / out of range / non-finite) */
  AFMM_ERR_INVALID_ARGUMENT = 3, /* std::invalid_argument (n == 0, bad option)          */
  AFMM_ERR_CUDA = 4,             /* CUDA runtime / driver failure, no device            */
  AFMM_ERR_UNSUPPORTED = 5,      /* n beyond 2^31 - 1; a NaN rep (AFMM_FLAG_KERNEL_SEMANTICS) */
  AFMM_ERR_OUT_OF_MEMORY = 6
} afmm_status;

typedef enum { AFMM_CASE_A = 0, AFMM_CASE_B = 1 } afmm_case;
typedef enum { AFMM_F64 = 0, AFMM_F32 = 1 } afmm_dtype;

typedef enum {
  /* Bit-exact with the reference: every Z element receives its terms in
   * increasing k, each as |rep| sequential `acc += step` (kernels.hpp:95-104). */
  AFMM_MODE_ORDER_PRESERVING = 0,
  /* Same additions, reassociated (split-k partial sums combined in a fixed
   * order). Within 1e-12 (f64) / 1e-5 (f32) of the reference, normalised by
   * sum_k |X[i,k]|*|Y[k,j]|. */
  AFMM_MODE_FAST = 1,
  /* AFMM_MODE_FAST plus a reassociation inside each term: the |rep| copies of
   * a base are summed as a doubling ladder (b, b+b, (b+b)+(b+b), ... are exact
   * power-of-two multiples; the ones selected by the binary digits of |rep|
   * are added into the element), i.e. floor(log2 |rep|) + popcount(|rep|)
   * additions per term instead of |rep|, still no multiplication. Same
   * tolerance as AFMM_MODE_FAST (fewer roundings per term). op_counts keep
   * the reference's tallies (sum of |rep|: the additions the product stands
   * for), not the fewer additions the device performed. */
  AFMM_MODE_FAST_LADDER = 2
} afmm_mode;

/* op_counts.hpp:17-23 */
typedef struct {
  uint64_t additions;
  uint64_t multiplications; /* always 0: the device path never multiplies an element */
  uint64_t zero_skips;
} afmm_op_counts;

typedef enum {
  AFMM_ERRKIND_NONE = 0,
  AFMM_ERRKIND_NOT_INTEGER = 1,   /* kernels.hpp:31-34 */
  AFMM_ERRKIND_OUT_OF_RANGE = 2,  /* kernels.hpp:36-39 */
  AFMM_ERRKIND_NON_FINITE = 3,    /* matrix.hpp:31-35 (DenseMatrix ctor) */
  AFMM_ERRKIND_SHAPE = 4,         /* kernels.hpp:15-21 */
  AFMM_ERRKIND_EMPTY = 5,         /* matrix.hpp:54-57 */
  AFMM_ERRKIND_REP_TOO_LARGE = 6, /* unused since ABI 2: every |rep| <= 2^53 is accepted */
  AFMM_ERRKIND_REP_NAN = 8,       /* a NaN rep under AFMM_FLAG_KERNEL_SEMANTICS */
  AFMM_ERRKIND_OTHER = 7
} afmm_error_kind;

typedef struct {
  int32_t kind;      /* afmm_error_kind */
  int32_t operand;   /* 0 = lhs, 1 = rhs */
  uint64_t row;      /* first offender in row-major order */
  uint64_t col;
  double value;      /* the offending element, widened to double */
  char message[256]; /* the exact text the reference's exception would carry */
} afmm_error;

/* Device-measured phases of one reference-facing call (CUDA events on the
 * call's streams; with several devices, the slowest device's figures). */
typedef struct {
  float total_ms;    /* first host->device copy to the last device->host byte */
  float compute_ms;  /* the repeated-addition kernel(s) */
  int32_t devices;   /* devices the call ran on */
  int32_t form;      /* kernel form of device 0 (afmm_context_last_form codes) */
} afmm_timing;

/* The operands are already-constructed matrices (the C++ wrapper's
 * DenseMatrix arguments), so only the kernel's own checks apply
 * (kernels.hpp:25-43): a non-finite BASE is computed with (inf / NaN
 * propagate through the adds exactly as in the reference), an infinite rep
 * "exceeds the exact integer range", and a NaN rep -- which the reference's
 * check lets through and then repeats llround(NaN) ~ 2^63 times, i.e. never
 * finishes -- is rejected with AFMM_ERR_UNSUPPORTED. Without the flag the
 * arrays are taken as the values a DenseMatrix is constructed from, and any
 * non-finite element is the constructor's "DenseMatrix: non-finite element"
 * (matrix.hpp:31-35). */
#define AFMM_FLAG_KERNEL_SEMANTICS 1

typedef enum {
  /* contiguous Z row ranges of equal predicted kernel time: W_i (exact
   * additions) for Case B, the Case A cost model (A-form / B-form) for Case A */
  AFMM_PARTITION_WORK = 0,
  AFMM_PARTITION_ROWS = 1 /* equal row counts */
} afmm_partition;

typedef struct {
  int32_t mode;         /* afmm_mode; anything else is AFMM_ERR_INVALID_ARGUMENT */
  int32_t device;       /* CUDA device ordinal; -1 = current (num_devices <= 1) */
  int32_t split_k;      /* fast mode: upper bound on k slices (0 = automatic) */
  int32_t num_devices;  /* G > 1: rows of Z sharded over G devices (0 or 1: one device) */
  const int32_t* devices; /* G ordinals (NULL = 0..G-1); a device may repeat (two shards) */
  int32_t partition;    /* afmm_partition */
  int32_t flags;        /* AFMM_FLAG_* */
  afmm_timing* timing;  /* optional out: device-measured phases of this call */
} afmm_options;

/* ---- reference-facing entry points (host buffers) ------------------------
 * One call = one product, host buffers in and out; `options` may be NULL
 * (order-preserving, current device). With options->num_devices = G > 1 the
 * rows of Z are sharded over G devices in one process (row i of Z depends only
 * on row i of X and all of Y, kernels.hpp:119,148): each device receives an
 * equal share of X's and Y's rows over PCIe, Y is completed over NVLink
 * (peer copies), the prepass statistics choose work-balanced row cuts, each
 * device copies the X rows of its cut it lacks from its peers and computes its
 * Z rows, which go straight to `out`. Validation covers the whole operands
 * before any Z element is written; results are bit-identical for every G. */

afmm_status afmm_case_a_f64(const double* lhs, uint64_t n_lhs, const double* rhs, uint64_t n_rhs,
                            double* out, const afmm_options* options, afmm_op_counts* counts,
                            afmm_error* error);
afmm_status afmm_case_b_f64(const double* lhs, uint64_t n_lhs, const double* rhs, uint64_t n_rhs,
                            double* out, const afmm_options* options, afmm_op_counts* counts,
                            afmm_error* error);
afmm_status afmm_case_a_f32(const float* lhs, uint64_t n_lhs, const float* rhs, uint64_t n_rhs,
                            float* out, const afmm_options* options, afmm_op_counts* counts,
                            afmm_error* error);
afmm_status afmm_case_b_f32(const float* lhs, uint64_t n_lhs, const float* rhs, uint64_t n_rhs,
                            float* out, const afmm_options* options, afmm_op_counts* counts,
                            afmm_error* error);

/* ---- device-resident entry points ----------------------------------------
 * An afmm_context owns a CUDA stream binding and a grow-only workspace on one
 * device. Calls on one context are serialised internally; distinct contexts
 * may be used concurrently. */
typedef struct afmm_context afmm_context;

afmm_status afmm_context_create(int32_t device, afmm_context** ctx);
void afmm_context_destroy(afmm_context* ctx);
/* Enqueue work on `stream` (a cudaStream_t; NULL = the legacy default stream). */
afmm_status afmm_context_set_stream(afmm_context* ctx, void* stream);

/* Z rows [row_begin, row_end) of lhs * rhs, all pointers device memory.
 * lhs/rhs are n x n with leading dimension `ld` (elements); `out` receives
 * (row_end - row_begin) rows with leading dimension `ld_out`, row r of the
 * slab holding Z row row_begin + r. Validation of the whole rep operand is
 * done on the device before any product element is computed.
 * When `sync` is nonzero the call waits for completion and fills counts /
 * error; when zero it only enqueues, and afmm_context_finish() later returns
 * the status, counts and error of the last enqueued call. */
afmm_status afmm_product_device(afmm_context* ctx, int32_t which_case, int32_t dtype,
                                const void* lhs, const void* rhs, uint64_t n, uint64_t ld,
                                void* out, uint64_t ld_out, uint64_t row_begin, uint64_t row_end,
                                const afmm_options* options, int32_t sync,
                                afmm_op_counts* counts, afmm_error* error);
afmm_status afmm_context_finish(afmm_context* ctx, afmm_op_counts* counts, afmm_error* error);

/* Record CUDA events around the phases of each product on the context's
 * stream (prepass, repeated-addition kernel, epilogue). After
 * afmm_context_finish(), afmm_context_last_timing() returns the milliseconds
 * of the last product's phases; -1 when timing is off. */
afmm_status afmm_context_enable_timing(afmm_context* ctx, int32_t enable);
afmm_status afmm_context_last_timing(afmm_context* ctx, float* prepass_ms, float* compute_ms,
                                     float* epilogue_ms);

/* Repeated-addition kernel of the context's last product: 0 = B-form
 * (k_bform: rep uniform per warp; Case B directly, Case A on transposed
 * operands), 1 = A-form (k_aform: Case A with the base uniform per warp,
 * zero bases skipped), 2 = split (Case A: the sparsest rows in the A-form,
 * the rest in the B-form); + 4 when the B-form part ran the small-rep group
 * kernel (k_bgroup: fp32, order-preserving, every rep in 0..2; chosen on the
 * device), i.e. 4 = Case B or Case A B-form, 6 = split. */
int32_t afmm_context_last_form(afmm_context* ctx);

/* Per-row work W_i (exact additions of Z row i) for the row partition:
 * Case A  W_i = sum_{k: X[i,k] != 0} sum_j |llround Y[k,j]|
 * Case B  W_i = sum_k |llround X[i,k]| * nnz(Y[k,:])
 * (closed forms of kernels.hpp:119-134 / :148-163). Written to the host
 * array work[n]. Device pointers as in afmm_product_device. */
afmm_status afmm_row_work_device(afmm_context* ctx, int32_t which_case, int32_t dtype,
                                 const void* lhs, const void* rhs, uint64_t n, uint64_t ld,
                                 uint64_t* work, afmm_error* error);

/* Predicted kernel time of each row (arbitrary units, for the row partition):
 * Case B: W_i (the B-form's time is proportional to the additions); Case A:
 * the cost model's time of the row in the cheaper of the A-form (proportional
 * to its nonzero bases) and the B-form (a per-row share of a tile), so that
 * rows of very different densities balance (afmm_partition_rows). Written to
 * the host array cost[n]. */
afmm_status afmm_row_cost_device(afmm_context* ctx, int32_t which_case, int32_t dtype,
                                 const void* lhs, const void* rhs, uint64_t n, uint64_t ld,
                                 uint64_t* cost, afmm_error* error);

/* Row cuts for `parts` devices from the operands' statistics (computed on
 * the context's device): Case B equal W_i; Case A equal modeled kernel time,
 * the device-side A-form / B-form choice evaluated per slab (tile and wave
 * quantisation included). cuts[parts + 1] as in afmm_partition_rows. */
afmm_status afmm_partition_device(afmm_context* ctx, int32_t which_case, int32_t dtype,
                                  const void* lhs, const void* rhs, uint64_t n, uint64_t ld,
                                  uint32_t parts, uint64_t* cuts, afmm_error* error);

/* The same Case A cut from given statistics, on the host (no device): stats =
 * {nonzero reps of Y, sum over (k, A-form tile) of the tile's max |rep|, reps
 * beyond 2048, sum of |rep|}, nnz_row[n] = nonzero bases of each row of X;
 * sms = SM count (0 = 148). slab_cycles[parts] (optional) receives each
 * slab's modeled time. */
afmm_status afmm_model_partition_case_a(int32_t dtype, uint64_t n, int32_t sms,
                                        const uint64_t* stats, const uint32_t* nnz_row,
                                        uint32_t parts, uint64_t* cuts, double* slab_cycles);

/* The modeled kernel time (cycles) of the Case A slab [row_begin, row_end)
 * under the same statistics: the device-side choice evaluated on the host. */
afmm_status afmm_model_slab_time_case_a(int32_t dtype, uint64_t n, int32_t sms,
                                        const uint64_t* stats, const uint32_t* nnz_row,
                                        uint64_t row_begin, uint64_t row_end, double* cycles);

/* Cut n rows into `parts` contiguous ranges of (as near as possible) equal
 * total work: cuts[0] = 0, cuts[parts] = n, range p = [cuts[p], cuts[p+1]).
 * Pure host function (no device needed). */
afmm_status afmm_partition_rows(const uint64_t* work, uint64_t n, uint32_t parts, uint64_t* cuts);

/* ---- peer-memory output (multi-GPU row sharding) -----------
 * A row-sharded product can write its Z slab straight into rank 0's result
 * over NVLink instead of gathering the slabs afterwards: rank 0 exports the
 * device buffer holding Z, every other rank opens the handle (CUDA IPC; peer
 * access is enabled on open) and passes the opened pointer, advanced to its
 * first row, as `out` of afmm_product_device. The repeated-addition kernels
 * then store their Z tiles to the peer GPU as they finish, overlapping the
 * transfer with the compute. Completion: each rank finishes its own product
 * (sync = 1 or afmm_context_finish), then the ranks meet at a host barrier.
 * `offset` is the byte offset of dev_ptr inside its allocation. */
typedef struct afmm_ipc_handle {
  uint8_t bytes[64];
  uint64_t offset;
} afmm_ipc_handle;

afmm_status afmm_ipc_export(const void* dev_ptr, afmm_ipc_handle* handle, afmm_error* error);
/* Opens a handle exported by another process on `device`; *dev_ptr is the
 * exported pointer as seen from this process. */
afmm_status afmm_ipc_open(int32_t device, const afmm_ipc_handle* handle, void** dev_ptr,
                          afmm_error* error);
afmm_status afmm_ipc_close(void* dev_ptr);

/* ---- seeded generation (random.hpp:111-129) ---------------------------------
 * afmm::generate on the GPU: the same matrix, bit for bit, as the reference's
 * single std::mt19937_64 stream over the n^2 entries in row-major order
 * (Bernoulli(density) per entry, then a value draw for a nonzero entry), for
 * the reference's GeneratorSpec (random.hpp:30-58). An invalid spec returns
 * AFMM_ERR_INVALID_ARGUMENT with the text of random.hpp:60-79. */
typedef enum { AFMM_ROLE_REAL = 0, AFMM_ROLE_INTEGER = 1 } afmm_value_role;
typedef struct {
  uint64_t n;
  double density;     /* probability an entry is nonzero */
  double mu_prime;    /* IntegerValued: values uniform over {1, ..., 2 mu' - 1} */
  int32_t role;       /* afmm_value_role */
  double value_low;   /* RealValued: values low + (high - low) * uniform01 */
  double value_high;
} afmm_generator_spec;

/* Into a caller-owned n x n host array (row-major); the device is
 * options->device (NULL options: the current device). f32 stores the
 * reference's double values rounded to float. */
afmm_status afmm_generate_f64(const afmm_generator_spec* spec, uint64_t seed, double* out,
                              const afmm_options* options, afmm_error* error);
afmm_status afmm_generate_f32(const afmm_generator_spec* spec, uint64_t seed, float* out,
                              const afmm_options* options, afmm_error* error);
/* Into device memory on the context's device and stream (n rows of leading
 * dimension ld): operands for afmm_product_device without a host round trip. */
afmm_status afmm_generate_device(afmm_context* ctx, const afmm_generator_spec* spec,
                                 uint64_t seed, int32_t dtype, void* out, uint64_t ld,
                                 afmm_error* error);

/* ---- roofline ---------------------------------------------------------------
 * Measure the CUDA-core FP-add peak of `device` with a register-resident
 * add-chain microbenchmark (the same instruction mix as the product's inner
 * loop: FADD2 for f32, DADD for f64). Returns additions per second. */
afmm_status afmm_fp_add_peak(int32_t device, int32_t dtype, double* adds_per_second,
                             double* sm_clock_mhz);

/* Number of kernels the library launched on this process since load (the
 * bench's gpu_launches claim). */
uint64_t afmm_kernel_launch_count(void);
const char* afmm_status_string(afmm_status s);
int32_t afmm_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* AFMM_B200_H */
