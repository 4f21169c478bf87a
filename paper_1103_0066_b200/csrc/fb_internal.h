// fb_internal.h -- interface between the C-ABI host layer (fb_capi.cpp) and
// the sm_100a kernels (fb_kernels_*.cu).  Not installed; not part of the ABI.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace fbk {

// CTA shape of the dense fallback and pack_geometry kernels (one slot per
// thread); the sparse kernel uses persistent 128-thread CTAs (fb_kernels.cuh).
constexpr int kThreads = 288;
constexpr int kTile = 288;  // element slots per CTA tile

enum Op { kLaplacian = 0, kElasticity = 1, kWeighted = 2,
          kPack = 3 };  // kPack: the sparse kernel emitting G itself (GPU pack_geometry)
enum Mode { kStrict = 0, kFast = 1 };
// kSparseSym: K validated to the P1 zero pattern, symmetric, and (elasticity)
//             equal component-diagonal blocks -> nb(nb+1)/2 contractions.
// kSparse:    P1 pattern, no symmetry shortcut (also used for packed G).
// kDense:     arbitrary K, every dim^2 term, K read from device memory.
// kUniformSym: kSparseSym and every nonzero entry is +-kappa_c with the P1
//             gradient sign pattern (true of the reference's K): products
//             g*kappa are shared between terms.
enum Path { kSparseSym = 0, kSparse = 1, kDense = 2, kUniformSym = 3 };

struct LaunchArgs {
  const double* vtx = nullptr;     // full vertex array (device)
  const int32_t* cells = nullptr;  // base-adjusted: cells + e*(dim+1) valid for touched e
  const double* coeffs = nullptr;  // base-adjusted like cells (weighted form)
  const void* g_in = nullptr;      // packed G, local slot-major (G-input path)
  void* out = nullptr;             // local store (slot-major, krows^2 per slot)
  const void* kdense = nullptr;    // dense path: K in engine precision (device)
  long long* status = nullptr;     // [0] lowest degenerate cell, [1] lowest bad-index cell
  int64_t nv = 0;                  // vertices
  int64_t ne = 0;                  // real elements in the WHOLE mesh (padding clamp)
  int64_t nloc = 0;                // slots handled by this launch
  int64_t slot0 = 0;               // global slot index of local slot 0
  int cells_aligned16 = 0;
  int vtx_aligned16 = 0;
};

struct LaunchSpec {
  int op = 0, dim = 2, prec = 1, mode = 0, path = 0;
  int from_g = 0;   // 1 = G-input path
  int staged = 3;   // 0 = direct per-lane stores, 1 = smem staging + LDS/STG block copy,
                    // 2 = smem staging + TMA store where the layout allows (else 1),
                    // 3 = auto (per layout: the faster of 1 and 2, measured)
};

// Sparse K values in engine precision, layout [((a*nb + b)*ncoef + c)*dim^2 + t]
// for the (a, b) Laplacian-like block (component-0 block for elasticity).
// Passed by value as a kernel parameter (constant bank, broadcast, reentrant).
constexpr int kMaxKParamBytes = 16 * 4 * 9 * 8;  // 3D weighted f64 = 4608 B
struct KParamBlob {
  alignas(16) unsigned char bytes[kMaxKParamBytes];
};

// Per (precision, dim) translation units.
cudaError_t launch_integrate_f32_2d(const LaunchSpec&, const LaunchArgs&, const KParamBlob&, cudaStream_t);
cudaError_t launch_integrate_f32_3d(const LaunchSpec&, const LaunchArgs&, const KParamBlob&, cudaStream_t);
cudaError_t launch_integrate_f64_2d(const LaunchSpec&, const LaunchArgs&, const KParamBlob&, cudaStream_t);
cudaError_t launch_integrate_f64_3d(const LaunchSpec&, const LaunchArgs&, const KParamBlob&, cudaStream_t);
cudaError_t launch_pack(int dim, int prec, const LaunchArgs&, cudaStream_t);

// Global assembly (fb_assemble.cu): the device half of an fb_assembly plan.
// Vertices are taken in groups of 32 (one warp); a group's incidence lists
// are stored sliced (SELL-32): incidence k of vertex 32g + l at
// goff[g] + 32k + l, k < (goff[g+1] - goff[g]) / 32, packed (e << 2 | a)
// ascending in e, padding 0xffffffff; spos at the same index packs the
// neighbour slot of each of the element's nb local vertices (one byte each)
// in v's sorted neighbour list [nbr_ptr[v], nbr_ptr[v+1]).  Row (v, ci)
// starts at value index nbr_ptr[v]*nc^2 + ci*deg*nc; neighbour slot k,
// component cj at + k*nc + cj.
struct AsmArgs {
  const int64_t* goff = nullptr;    // ngroups + 1
  const uint32_t* spk = nullptr;    // sliced incidences
  const uint32_t* spos = nullptr;   // sliced neighbour slots
  const int64_t* nbr_ptr = nullptr; // nv + 1
  const void* store = nullptr;      // element matrices, e*krows^2 + i + j*krows
  void* values = nullptr;           // CSR values (engine precision)
  int64_t nv = 0;
  int sym = 0;                      // element matrices bitwise symmetric: read columns
  int diag = 0;                     // elasticity: block-diagonal element matrices with equal
                                    // diagonal blocks (read block (0,0) only)
  // G-input assembly (fb_assemble_g.cu): element rows recomputed from the
  // packed geometry (PackedGeometry layout) instead of read from a store
  const void* g_in = nullptr;
  const double* coeffs = nullptr;   // weighted form: ne*(dim+1) nodal coefficients
  int64_t g_len = 0;                // scalars readable at g_in (16-byte aligned)
};
cudaError_t launch_assemble(int dim, int nc, int prec, const AsmArgs&, cudaStream_t);
cudaError_t launch_assemble_g(const LaunchSpec& s, const AsmArgs&, const KParamBlob&, cudaStream_t);

// The same plan built on the GPU from device-resident connectivity
// (fb_plan.cu); arrays are stream-ordered allocations the caller frees with
// cudaFree.  bad[0] = lowest cell with an out-of-range id, bad[1] = lowest
// cell with a repeated vertex, bad[2] = lowest vertex of degree > 255 (-1 =
// none); on bad[0|1] nothing is allocated, on bad[2] only the offsets.
struct PlanDevice {
  int64_t* goff = nullptr;
  uint32_t* spk = nullptr;
  uint32_t* spos = nullptr;
  int64_t* nbr_ptr = nullptr;
  int32_t* nbr = nullptr;
  int64_t total_nbr = 0, total_sell = 0;
};
cudaError_t build_plan_device(int dim, int64_t ne, int64_t nv, const int32_t* cells, cudaStream_t st,
                              PlanDevice* out, int64_t* bad);

inline cudaError_t launch_integrate(const LaunchSpec& s, const LaunchArgs& a,
                                    const KParamBlob& k, cudaStream_t st)
{
  if (s.prec == 0)
    return s.dim == 2 ? launch_integrate_f32_2d(s, a, k, st) : launch_integrate_f32_3d(s, a, k, st);
  return s.dim == 2 ? launch_integrate_f64_2d(s, a, k, st) : launch_integrate_f64_3d(s, a, k, st);
}

#ifdef __CUDACC__
__host__ __device__
#endif
inline int64_t num_tiles(int64_t nloc) { return (nloc + kTile - 1) / kTile; }

}  // namespace fbk
