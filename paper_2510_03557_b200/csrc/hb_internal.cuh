// hb_internal.cuh -- internal (non-ABI) entry points shared by the translation
// units: mesh build, list sweep into a receiver CSR, pair-engine pieces.
#pragma once
#include "hb_pairs.cuh"

namespace hb {

struct ListGeom {
  int64_t nb[3];
  int periodic[3];
  double L, reach;
  int64_t active_depth;
};

struct ListArgsDev {
  int64_t n_leaves;
  const int64_t *leaf_bin, *leaf_level, *bin_ptr, *bin_ids;
  const double *leaf_lo, *leaf_hi;
  const uint8_t* ghost_only;
  ListGeom g;
};

int build_mesh(const HbMeshArgs* a, Arena& ws, cudaStream_t st, HbError* err);
// ordered list as a receiver CSR: ent_ptr (n_leaves+1), partner, code|fwd<<8
int assemble_csr(const ListArgsDev& d, int64_t capacity, int32_t* ent_src, int32_t* ent_code,
                 int64_t* ent_ptr, int64_t* total_host, Arena& ws, cudaStream_t st, HbError* err);

// fused SPH passes (hb_sph.cu): pass 0 = neighbour count + density,
// pass 1 = CRK moments + hydro force; gas tiling, gas records P0..P2
struct SphArgs {
  const Tiling* T;
  const int64_t* n_tiles_dev;
  const int64_t* ent_ptr;
  const int32_t* ent_src;
  const int32_t* ent_code;
  const float4 *P0, *P1, *P2, *P3;
  Rows rows;
  const int8_t* pshift;
  double L, reach;
  float band;  // relative band of r^2 around a threshold decided in float64
  double alpha, beta;
  double *ncount, *rho, *moments, *hydro;
  // pass C (gradients): A, B, fallback of the CRK solve; gradA (n,3), gradB (n,9)
  const double *crk_A, *crk_B;
  const uint8_t* crk_fallback;
  double *gradA, *gradB;
  unsigned long long* err_key;
  const uint8_t* skip_leaf;
  int skip_tiles;  // pass B: skip tiles without an owned member
};
int pack_sph(const Tiling& T, const int64_t* ntd, Rows rows, const int8_t* pshift,
             double L, float4* P0, float4* P1, float4* P2, float4* P3, int layout,
             cudaStream_t st, HbError* err, const double* rho = nullptr,
             const double* u = nullptr, double gamma = 0.0);
int launch_sph(int pass, const SphArgs& s, cudaStream_t st, HbError* err);

// bin-level short-range gravity (hb_grav2.cu)
// bin at which the two-launch bin gravity splits (HbStepArgs.grav_half_event):
// 4/5 of the bins go first, so the rows that drain after the step are a fifth
// of the gravity output, while the first part's copy (4/5 of it) still fits
// under the last fifth of the kernel behind the SPH outputs' copy
__host__ __device__ inline int64_t grav_split_bin(int64_t nbins) { return nbins * 4 / 5; }

struct GravBinArgs {
  int64_t n, nbins;
  const int64_t *bin_ptr, *leaf_start, *leaf_end;
  ListGeom geom;
  Rows rows;
  const int8_t* pshift;
  double L, r_s, r_cut, eps;
  double* out;
  unsigned long long* err_key;
  int* overflow_host;
  const uint8_t* ghost = nullptr;  // owned_targets: skip tiles without an owned row
  cudaEvent_t t0 = nullptr, t1 = nullptr;  // optional: recorded around the pair kernel
  // optional: run the pair kernel in two launches split at bin nbins / 2 and
  // record split_event between them (rows of bins < nbins / 2 are then final
  // up to the caller's ghost-row zeroing, done by `between` when set)
  cudaEvent_t split_event = nullptr;
  int (*between)(void* ctx) = nullptr;
  void* between_ctx = nullptr;
  // count instead of sum: exact in-r_cut source counts per row into
  // (int64_t*)out (HB_PASS_COUNT_ONLY)
  bool count_only = false;
  // 0: prepare (segments, stencil, tiling, records) and launch; 1: prepare
  // only; 2: launch only, on what a phase-1 call with the same arena offset
  // prepared (the step prepares gravity while pass B waits for its inputs)
  int phase = 0;
  // optional: the step's bin segments and 27-stencil (bin_stencil_csr),
  // reused instead of recomputed
  const int64_t *pre_seg_s = nullptr, *pre_seg_e = nullptr, *pre_st_ptr = nullptr;
  const int32_t *pre_st_src = nullptr, *pre_st_code = nullptr;
};
int gravity_bins(const GravBinArgs& g, Arena& ws, cudaStream_t st, HbError* err);
// hb_crk_solve over a row list (rows[0, *n_rows), device count); other rows get
// the non-gas result (A = 1, B = 0, no fallback)
int crk_solve_rows(int64_t n, const double* moments, int64_t stride, const uint8_t* species,
                   double cond_limit, double* A, double* B, uint8_t* fallback,
                   const int32_t* rows, const int64_t* n_rows, cudaStream_t st, HbError* err);
// bins as segments: row range per bin and the 27-bin stencil as a receiver CSR
int bin_stencil_csr(int64_t nbins, const int64_t* bin_ptr, const int64_t* leaf_start,
                    const int64_t* leaf_end, const ListGeom& g, int64_t* seg_s, int64_t* seg_e,
                    int64_t* st_ptr, int32_t* st_src, int32_t* st_code, cudaStream_t st,
                    HbError* err);

}  // namespace hb
