/*
 * fembatch_b200.h -- C-ABI drop-in boundary of the B200 P1 element-integration
 * engine (libfembatch_b200.so).  Plain pointers and sizes only; no C++ or
 * torch types cross this boundary.
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj):
 *
 *   fb_specialize            <- fembatch::specialize_kernel      include/fembatch/engine.hpp:60-63,
 *                                                                src/engine.cpp:301-337
 *   fb_integrate_mesh        <- pack_geometry + integrate_batches (the composition every
 *                               caller makes: src/bench.cpp:120-164, tests/test_engine.cpp:28-38)
 *                               fused into one kernel: G never reaches HBM
 *   fb_integrate_packed      <- fembatch::integrate_batches      include/fembatch/engine.hpp:65-70,
 *                                                                src/engine.cpp:339-376
 *   fb_pack_geometry         <- fembatch::pack_geometry          include/fembatch/geometry.hpp:91,
 *                                                                src/geometry.cpp:312-351
 *   fb_flop_count            <- fembatch::flop_count             src/engine.cpp:378-387
 *   fb_element_matrix_index  <- fembatch::element_matrix_index   src/engine.cpp:287-299
 *   fb_build_analytic_tensor <- fembatch::build_analytic_tensor  src/forms.cpp:234-246
 *   fb_structured_mesh /     <- structured_simplicial_mesh /     src/geometry.cpp:164-262
 *   fb_jitter_mesh              jitter_mesh (input synthesis)
 *   fb_assembly_* /          <- (no reference counterpart: global sparse assembly is the
 *   fb_assemble                 reference's declared non-goal; it consumes the
 *                               ElementMatrixStore, include/fembatch/engine.hpp:27-43)
 *
 * Errors: every call returns an fb_status code and, when `err` is non-NULL,
 * fills it with the reference's exception text (same wording as the
 * std::invalid_argument / std::runtime_error / std::out_of_range the
 * reference throws) and, for degenerate cells, the lowest offending cell.
 * All argument validation happens before any device work.
 *
 * Threading: every entry point is reentrant.  The library keeps one grow-only
 * workspace and two streams per device, guarded by a per-device mutex, so
 * concurrent calls that target the same device serialise; calls on different
 * devices run concurrently.  No global mutable state is shared with callers.
 */
#ifndef FEMBATCH_B200_H
#define FEMBATCH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FB_ABI_VERSION 1

/* Operators (reference Operator enum, include/fembatch/forms.hpp:12). */
enum fb_operator { FB_LAPLACIAN = 0, FB_ELASTICITY = 1, FB_WEIGHTED_LAPLACIAN = 2 };

/* Precision (reference Precision, include/fembatch/kernel_config.hpp:10). */
enum fb_precision { FB_F32 = 0, FB_F64 = 1 };

/* Arithmetic mode (GPU extension).
 *   FB_STRICT: FP64 geometry with IEEE divisions in the reference's operation
 *              order, no FMA contraction anywhere -> bitwise equal to the
 *              reference engine (pack_geometry + integrate_batches).
 *   FB_FAST:   FMA + one reciprocal of det; within the stated tolerances
 *              (normwise 1e-13 f64, 5e-6 f32), not bitwise. */
enum fb_mode { FB_STRICT = 0, FB_FAST = 1 };

/* Output path (GPU extension).  Element matrices are staged per warp tile in
 * shared memory and leave it by TMA store (TMA: bulk or tensor store, where
 * the staged layout allows it) or by a warp block copy LDS.128 -> STG.128
 * (STAGED); DIRECT stores each lane's matrix from registers.  AUTO picks
 * per layout the faster of TMA and STAGED as measured on B200.
 * All give identical values; a store pointer that is not 16-byte aligned
 * falls back to DIRECT. */
enum fb_store { FB_STORE_AUTO = 0, FB_STORE_STAGED = 1, FB_STORE_DIRECT = 2, FB_STORE_TMA = 3 };

enum fb_status {
  FB_OK = 0,
  FB_ERR_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
  FB_ERR_RUNTIME = 2,          /* reference: std::runtime_error (degenerate cell) */
  FB_ERR_OUT_OF_RANGE = 3,     /* reference: std::out_of_range */
  FB_ERR_CUDA = 4,
  FB_ERR_NO_DEVICE = 5
};

/* Reference KernelConfig (include/fembatch/kernel_config.hpp:23-37) plus the
 * GPU extension fields.  The reference axes are value-neutral on the GPU
 * exactly as on the CPU: element_batch_size fixes the padded store length
 * (num_batches * bs * krows^2 scalars) and the bound/divisibility checks;
 * num_concurrent_elements, interleave_stores and loop_unroll are validated
 * and named in the variant description but never change a value. */
typedef struct fb_kernel_config {
  int32_t element_batch_size;      /* reference default 128 */
  int32_t num_concurrent_elements; /* reference default 1 */
  int32_t interleave_stores;       /* bool */
  int32_t loop_unroll;             /* bool */
  int32_t precision;               /* enum fb_precision */
  int32_t mode;                    /* enum fb_mode (GPU) */
  int32_t store;                   /* enum fb_store (GPU) */
  int32_t reserved;                /* must be 0 */
} fb_kernel_config;

/* Reference Mesh (include/fembatch/geometry.hpp:14-35) as a borrowed view.
 * vertices: num_vertices*dim doubles, vertex-major.
 * cells:    num_elements*(dim+1) int32 vertex ids, element-major.
 * Pointers may be host or device memory (detected per call). */
typedef struct fb_mesh_view {
  int32_t dim;
  int32_t reserved;
  int64_t num_vertices;
  int64_t num_elements;
  const double* vertices;
  const int32_t* cells;
} fb_mesh_view;

typedef struct fb_error {
  int32_t code;        /* enum fb_status */
  int32_t reserved;
  int64_t cell;        /* lowest offending cell for degenerate/out-of-range cells, else -1 */
  char message[256];   /* reference exception text */
} fb_error;

/* A frozen kernel variant: spec + config + K cast to engine precision, with
 * the K structure (P1 sparsity, symmetry, elasticity component blocks)
 * validated once so the launch can pick the sparse kernel. */
typedef struct fb_variant fb_variant;

/* ---- library / devices -------------------------------------------------- */
int fb_abi_version(void);
int fb_device_count(void);
/* Number of CUDA kernels this library has launched so far (all devices). */
int64_t fb_launch_counter(void);
/* Number of per-device kernel setups (dynamic shared-memory opt-in +
 * occupancy query of one kernel instantiation) performed on `device` so far;
 * every device a kernel runs on gets its own (attributes are per device
 * context).  -1 for an id outside [0, 64). */
int64_t fb_kernel_setups(int device);
/* Releases the grow-only staging workspace, streams and pinned status word
 * the library keeps for `device` (-1: every device).  Must not race with a
 * call running on that device (it takes the device's mutex). */
int fb_release_workspace(int device, fb_error* err);

/* Element-range sharding (replaces the reference's worker split,
 * src/engine.cpp:254-281, whose threads take contiguous batch ranges):
 * bounds[0..parts] of the contiguous, tile-aligned slot ranges a device list
 * of `parts` devices integrates (shard g = [bounds[g], bounds[g+1])).  The
 * store is element-major, so the shard outputs are the matching contiguous
 * slices of the single-device store and concatenate to it bitwise. */
int fb_shard_bounds(int64_t num_slots, int parts, int64_t* bounds, fb_error* err);

/* ---- pure host helpers -------------------------------------------------- */
int fb_krows(int op, int dim);
int64_t fb_k_len(int op, int dim);
int64_t fb_flop_count(int op, int dim, int64_t num_elements);
int64_t fb_element_matrix_index(int krows, int element_batch_size,
                                int num_concurrent_elements, int64_t element,
                                int i, int j);
/* num_batches * bs * krows^2 (the reference store length). */
int64_t fb_store_length(int op, int dim, int64_t num_elements, int element_batch_size);
int fb_build_analytic_tensor(int op, int dim, double* k_out, int64_t k_len,
                             fb_error* err);

/* ---- input synthesis (reference mesh generators) ------------------------ */
int fb_structured_mesh_sizes(int dim, int n, int64_t* num_vertices,
                             int64_t* num_elements);
int fb_structured_mesh(int dim, int n, double* vertices, int32_t* cells,
                       fb_error* err);
/* In place: displace interior vertices (reference jitter_mesh semantics,
 * bit-identical for a given seed); rejects tangled results. */
int fb_jitter_mesh(int dim, double* vertices, int64_t num_vertices,
                   const int32_t* cells, int64_t num_elements,
                   double magnitude, uint64_t seed, fb_error* err);

/* ---- variants ------------------------------------------------------------ */
fb_variant* fb_specialize(int op, int dim, const double* k_blocks, int64_t k_len,
                          const fb_kernel_config* config, fb_error* err);
void fb_variant_free(fb_variant* v);
/* "bs128_ce2_is_unroll"-style name (reference engine.cpp:329-335). */
const char* fb_variant_description(const fb_variant* v);
/* Kernel path chosen at specialize time: 0 = sparse+symmetric (P1 structure
 * validated), 1 = sparse, 2 = dense fallback (arbitrary K), 3 = sparse +
 * symmetric + uniform magnitude (K = +-kappa on the P1 pattern, as the
 * reference builds it). */
int fb_variant_path(const fb_variant* v);

/* ---- integration ---------------------------------------------------------
 * out / out_len: the ElementMatrixStore scalars (engine precision), length
 * exactly fb_store_length(); padding slots replicate the last element, as the
 * reference computes them.  coefficients: num_elements*(dim+1) doubles for
 * the weighted form (reference CoefficientField), else NULL.
 *
 * devices/ndev: the job is sharded over these devices by contiguous
 * tile-aligned element ranges (no collectives; outputs concatenate).  Any
 * buffer may be on the host or on any device: each shard device stages its
 * own slice (a device-resident operand on another GPU moves by NVLink peer
 * copy, e.g. all shards gathered into one device's store).  NULL/0 means
 * device 0 (or, for device pointers, the pointers' device).  Host buffers
 * should be pinned for full PCIe bandwidth. */
int fb_integrate_mesh(const fb_variant* v, const fb_mesh_view* mesh,
                      const double* coefficients, void* out, int64_t out_len,
                      const int* devices, int ndev, fb_error* err);

/* G-input path: g = num_batches*bs*dim^2 scalars of engine precision in the
 * reference PackedGeometry layout. */
int fb_integrate_packed(const fb_variant* v, int dim, const void* g,
                        int64_t num_batches, int64_t num_elements,
                        const double* coefficients, void* out, int64_t out_len,
                        const int* devices, int ndev, fb_error* err);

/* GPU pack_geometry: g_out = num_batches*bs*dim^2 scalars (precision). */
int fb_pack_geometry(const fb_mesh_view* mesh, int element_batch_size,
                     int precision, void* g_out, int64_t g_len,
                     const int* devices, int ndev, fb_error* err);

/* ---- device buffers (for callers without their own allocator) ------------
 * fb_device_alloc: `bytes` of device memory on `device` (256-byte aligned,
 * so staged/TMA stores apply), NULL on failure (err filled).  fb_free
 * releases it (NULL is a no-op). */
void* fb_device_alloc(int64_t bytes, int device, fb_error* err);
int fb_free(void* device_ptr, fb_error* err);

/* ---- device-resident asynchronous API ------------------------------------
 * All pointers are device pointers on the current device; the launch is
 * enqueued on `stream` (a cudaStream_t, NULL = legacy default stream) and the
 * call returns without synchronising.  `status` is a device buffer of two
 * int64 words (lowest degenerate cell, lowest cell with an out-of-range
 * vertex id): reset it with fb_status_reset, read it with fb_status_check. */
int fb_integrate_mesh_async(const fb_variant* v, const fb_mesh_view* mesh,
                            const double* coefficients, void* out,
                            int64_t out_len, int64_t* status, void* stream,
                            fb_error* err);
int fb_integrate_packed_async(const fb_variant* v, int dim, const void* g,
                              int64_t num_batches, int64_t num_elements,
                              const double* coefficients, void* out,
                              int64_t out_len, void* stream, fb_error* err);
/* GPU pack_geometry on device buffers (degenerate cells -> status). */
int fb_pack_geometry_async(const fb_mesh_view* mesh, int element_batch_size, int precision,
                           void* g_out, int64_t g_len, int64_t* status, void* stream,
                           fb_error* err);
int fb_status_reset(int64_t* status, void* stream, fb_error* err);
/* Synchronises `stream`, then maps the status words to the reference
 * exception (FB_ERR_RUNTIME "degenerate element: det(J) <= 0 in cell N"). */
int fb_status_check(const int64_t* status, void* stream, fb_error* err);

/* ---- global assembly (beyond the reference) -----------
 * CSR matrix of the global operator from an ElementMatrixStore.
 *   dof(v, c) = v*nc + c, nc = dim for elasticity, 1 otherwise (component c
 *   of the store's local index i = a + c*(dim+1)).
 *   Pattern: row (v, c) holds every dof of every vertex sharing an element
 *   with v (v included), columns ascending; explicit zeros are kept
 *   (elasticity's off-diagonal component blocks).
 *   Values: A[r][s] = sum over elements e in ASCENDING order of the store
 *   entries mapping to (r, s), in engine precision from +0 -- bitwise the
 *   serial loop "for e: for (i, j): A[dof_i][dof_j] += Ae(i, j)".
 * The plan (pattern + vertex->element incidence lists) is built once per
 * mesh (GPU or host, see fb_assembly_create); fb_assemble* run one
 * deterministic gather kernel (no atomics).  Only the real elements
 * (0 .. num_elements-1) of the store are read; padding slots are ignored. */
typedef struct fb_assembly fb_assembly;

/* cells: host or device pointer (num_elements*(dim+1) int32).  Device
 * connectivity builds the plan on that GPU; host connectivity of >= 65,536
 * elements is uploaded and planned on the current GPU, smaller meshes (or
 * any, with FB_PLAN_HOST set in the environment, or without a GPU) on the
 * host (multithreaded); all give the same plan.  Errors: out-of-range vertex id
 * or a repeated vertex within a cell (FB_ERR_INVALID_ARGUMENT, err->cell =
 * the lowest such cell), vertex degree > 255. */
fb_assembly* fb_assembly_create(int op, int dim, const int32_t* cells, int64_t num_elements,
                                int64_t num_vertices, fb_error* err);
void fb_assembly_free(fb_assembly* a);
int64_t fb_assembly_rows(const fb_assembly* a);
int64_t fb_assembly_nnz(const fb_assembly* a);
/* Host copies: row_ptr[rows+1] (int64), col_idx[nnz] (int32). */
int fb_assembly_pattern(const fb_assembly* a, int64_t* row_ptr, int64_t row_ptr_len,
                        int32_t* col_idx, int64_t nnz, fb_error* err);
/* flags: FB_ASSEMBLE_SYMMETRIC = the caller promises every element matrix
 * in the store is bitwise symmetric (true of fb_integrate_mesh output of a
 * variant whose fb_variant_path is 0 or 3); the kernel then reads each
 * needed row as the contiguous column.
 * FB_ASSEMBLE_BLOCK_DIAGONAL (elasticity; ignored for one-component forms) =
 * the caller promises every element matrix is zero off the component
 * diagonal and its nc diagonal blocks are bitwise equal (true of
 * fb_integrate_mesh / fb_integrate_packed output of any variant whose
 * fb_variant_path is not 2: SURVEY 8a row A9); only block (0,0) is read,
 * 1/nc^2 of the store.  Values are identical either way when the promise
 * holds. */
enum fb_assemble_flags { FB_ASSEMBLE_SYMMETRIC = 1, FB_ASSEMBLE_BLOCK_DIAGONAL = 2 };
/* values[nnz] (engine precision of v).  store/values: host or device
 * pointers (host data is staged through the device of `device`). */
int fb_assemble(const fb_assembly* a, const fb_variant* v, const void* store, int64_t store_len,
                void* values, int64_t nnz, int flags, int device, fb_error* err);
/* Device pointers on the current device; enqueued on `stream`. */
int fb_assemble_async(const fb_assembly* a, const fb_variant* v, const void* store,
                      int64_t store_len, void* values, int64_t nnz, int flags, void* stream,
                      fb_error* err);
/* Assembly straight from packed geometry (the fb_integrate_batches input:
 * g = num_elements*dim^2 scalars in engine precision, PackedGeometry layout;
 * coeffs = num_elements*(dim+1) doubles for the weighted Laplacian, else
 * NULL): each incidence's element-matrix row is recomputed in registers, the
 * element-matrix store is never written.  values are bitwise those of
 * fb_integrate_batches(g) followed by fb_assemble.  Needs a variant whose K
 * has the P1 pattern (fb_variant_path != 2).  Device pointers on the current
 * device; enqueued on `stream`. */
int fb_assemble_packed_async(const fb_assembly* a, const fb_variant* v, const void* g, int64_t g_len,
                             const double* coeffs, int64_t coeffs_len, void* values, int64_t nnz,
                             void* stream, fb_error* err);
/* Synchronous form: g, coeffs, values host or device pointers (host data is
 * staged through the device of `device`, or of the device-resident input). */
int fb_assemble_packed(const fb_assembly* a, const fb_variant* v, const void* g, int64_t g_len,
                       const double* coeffs, int64_t coeffs_len, void* values, int64_t nnz, int device,
                       fb_error* err);

#ifdef __cplusplus
}
#endif

#endif /* FEMBATCH_B200_H */
