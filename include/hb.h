/*
 * hb.h -- C ABI of the B200-native short-range particle-particle engine.
 *
 * Plain pointers and sizes only (no torch or CUDA types): every array argument
 * is a DEVICE pointer unless marked "host"; `stream` is a cudaStream_t passed
 * as void* (NULL = legacy default stream).  Every entry point returns an
 * HbStatus and fills HbError.  Caller owns all memory; work buffers come from a
 * caller-provided arena whose size the matching *_workspace() query returns.
 *
 * Each entry point replaces one reference function of the hydrobox hot path
 * (hb/ = /root/reference/pkg/src/hydrobox/); the python binding a maintainer
 * would add is shown in INTEGRATION.md.
 */
#ifndef HB_H_
#define HB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HB_ABI_VERSION 5

/* status codes; map onto hb/errors.py */
enum HbStatus {
  HB_OK = 0,
  HB_NONFINITE = 1, /* KernelEvalError "non-finite partial in leaf pair (a, b)" hb/lane.py:106-107 */
  HB_OVERFLOW = 2,  /* KernelEvalError "accumulator overflow ..."            hb/lane.py:108,197-198 */
  HB_CONTRACT = 3,  /* HydroboxError: argument contract violated            hb/lane.py:137-144 */
  HB_CUDA = 4       /* CUDA runtime failure                                            */
};

typedef struct HbError {
  int32_t status;
  int32_t cuda_err;
  int64_t leaf_a; /* first failing leaf pair, as the reference's counters[6..7] */
  int64_t leaf_b;
  char msg[224];
} HbError;

int hb_abi_version(void);
/* number of kernels this library has launched in the process (bench accounting) */
int64_t hb_launch_count(void);
/* SM count and compute capability of the current device (host outputs). */
int hb_device_query(int* sm_count, int* cc_major, int* cc_minor);

/* ---------------------------------------------------------------------------
 * Chaining-mesh bins + k-d leaves.  Replaces build_mesh_and_leaves
 * (hb/cmtree.py:125-196): flat bin key of binning_pos = pos + shift*L
 * (hb/particles.py:131-133), stable bin sort, per-bin recursive median split
 * along the longest axis with stable tie-break (hb/cmtree.py:110-122), tight
 * leaf AABBs, ghost-only flags.  Output `perm` is the reorder the caller
 * applies to its particle set (row k of the new order = old row perm[k]).
 * Leaves are numbered bin-ascending then depth-first, so bin_ptr is the CSR
 * bin -> leaves and the leaf ids of a bin are contiguous (bin_ids = arange).
 * ------------------------------------------------------------------------- */
typedef struct HbMeshArgs {
  int64_t n;
  const double* pos;         /* (n,3) canonical wrapped positions               */
  const int8_t* image_shift; /* (n,3) periodic image of ghost copies            */
  const uint8_t* ghost;      /* (n)                                             */
  double side_length;        /* L                                               */
  double lo[3];              /* host: mesh bounds_lo                            */
  double width[3];           /* host: realised bin widths extent/nb             */
  int64_t nb[3];             /* host: bins per axis                             */
  int64_t max_leaf_size;
  int64_t leaf_cap;          /* capacity of the leaf arrays below               */
  /* outputs */
  int64_t* perm;             /* (n)                                             */
  int64_t* leaf_start;       /* (leaf_cap)                                      */
  int64_t* leaf_end;         /* (leaf_cap)                                      */
  double* leaf_lo;           /* (leaf_cap,3)                                    */
  double* leaf_hi;           /* (leaf_cap,3)                                    */
  uint8_t* leaf_ghost_only;  /* (leaf_cap)                                      */
  int64_t* leaf_bin;         /* (leaf_cap)                                      */
  int64_t* bin_ptr;          /* (nbins+1)                                       */
  int64_t* n_leaves_dev;     /* device scalar                                   */
  int64_t* n_leaves_host;    /* host scalar or NULL (NULL: no host sync)        */
  int64_t* max_bin_leaves_host; /* host scalar or NULL                          */
  int64_t* max_bin_count_host;  /* host scalar or NULL: most particles in a bin  */
} HbMeshArgs;

size_t hb_build_mesh_workspace(int64_t n, const int64_t nb[3], int64_t max_leaf_size);
/* upper bound of the leaf count for n particles in nbins bins */
int64_t hb_leaf_capacity(int64_t n, int64_t nbins, int64_t max_leaf_size);
int hb_build_mesh(const HbMeshArgs* args, void* ws, size_t ws_bytes, void* stream, HbError* err);

/* Gather rows by perm for a column block of `width` bytes per row (used to
 * apply the build permutation to particle fields on device;
 * hb/particles.py:115-127).  inv_remap: optional int64 column remapped through
 * the inverse permutation (ghost_src), -1 preserved. */
int hb_permute_rows(int64_t n, const int64_t* perm, const void* src, void* dst,
                    int64_t row_bytes, void* stream, HbError* err);
int hb_remap_through_inverse(int64_t n, const int64_t* perm, int64_t* values,
                             int64_t* scratch, void* stream, HbError* err);

/* Grow leaf AABBs to cover current member positions (hb/cmtree.py:199-207). */
int hb_grow_aabbs(int64_t n_leaves, const int64_t* leaf_start, const int64_t* leaf_end,
                  const double* pos, const int8_t* image_shift, double side_length,
                  double* leaf_lo, double* leaf_hi, void* stream, HbError* err);

/* ---------------------------------------------------------------------------
 * Leaf-pair interaction lists.  Replaces assemble_interaction_lists +
 * _assemble_core (hb/cmtree.py:210-337): 27-stencil sweep per active leaf
 * (level >= active_depth and not ghost-only), periodic wrap on full-box axes
 * with image shift, duplicate (bin, shift) suppression, per-axis AABB gap
 * <= reach in exact float64, output lexsorted by (a, b, sx, sy, sz).
 * Call with out_* == NULL to count; then again with capacity >= count.
 * ------------------------------------------------------------------------- */
typedef struct HbListArgs {
  int64_t n_leaves;
  const int64_t* leaf_bin;
  const double* leaf_lo;           /* (n_leaves,3) */
  const double* leaf_hi;
  const int64_t* leaf_level;       /* may be NULL: all level 0 */
  const uint8_t* leaf_ghost_only;
  const int64_t* bin_ptr;          /* (nbins+1) CSR bin -> positions in bin_ids */
  const int64_t* bin_ids;          /* leaf ids; NULL = identity                 */
  int64_t nb[3];                   /* host */
  uint8_t periodic[3];             /* host */
  double side_length;
  double reach;
  int64_t active_depth;
  int64_t capacity;
  int64_t* out_a;                  /* (capacity) or NULL to count */
  int64_t* out_b;
  int8_t* out_shift;               /* (capacity,3) */
  int64_t* count_host;             /* host: number of entries */
} HbListArgs;

size_t hb_assemble_lists_workspace(int64_t n_leaves, int64_t capacity);
int hb_assemble_lists(const HbListArgs* args, void* ws, size_t ws_bytes, void* stream,
                      HbError* err);

/* ---------------------------------------------------------------------------
 * Pair evaluation over a leaf-pair list.  Replaces eval_pairs_core
 * (hb/kernels.py:281-392) with the same argument meaning: kernel id,
 * float64 state matrix (n,12) in the column layout of hb/particles.py:46-54,
 * per-particle image shift, aux columns, list (a, b, shift), leaf ranges,
 * params, L, lane half-width W2 (accepted; affects only the FLOP-proxy
 * counters), reach, include_self, mirror, channel signs, mirror map, scales,
 * deterministic flag.  Outputs are ACCUMULATED into caller-zeroed out_flt
 * (relaxed) or out_int (deterministic, int64 quanta of the per-pair FP32
 * contribution); counters[8] (host) as hb/kernels.py:46-58.
 * Execution: list entries grouped by receiver leaf (CSR, stable), each
 * receiver leaf cut into <=32-particle tiles, one warp per target tile,
 * FP32 leaf-relative coordinates, gather accumulation (no atomics).
 * ------------------------------------------------------------------------- */
typedef struct HbEvalArgs {
  int32_t kid;
  int32_t nchan;
  int64_t n;
  const double* state;        /* (n,12)                                  */
  const int8_t* pshift;       /* (n,3) or NULL (zeros)                   */
  const double* aux;          /* (n,naux) or NULL                        */
  int32_t naux;
  int32_t W2;
  int64_t n_pairs;
  const int64_t* pair_a;
  const int64_t* pair_b;
  const int8_t* pair_shift;   /* (n_pairs,3)                             */
  int64_t n_leaves;
  const int64_t* leaf_start;
  const int64_t* leaf_end;
  double params[4];           /* host                                    */
  double side_length;
  double reach;
  int32_t include_self;
  int32_t mirror;
  int64_t chan_sign[10];      /* host                                    */
  int64_t mirror_map[10];     /* host                                    */
  double scales[10];          /* host                                    */
  int32_t deterministic;
  int32_t exact_counters;     /* 1: pairs_in_reach over all species, as the
                                 reference counts it (an extra counting pass
                                 for the gas-only SPH kernels)            */
  int64_t* out_int;           /* (n,nchan) device                        */
  double* out_flt;            /* (n,nchan) device                        */
  int64_t counters[8];        /* host out                                */
} HbEvalArgs;

size_t hb_eval_pairs_workspace(const HbEvalArgs* args);
int hb_eval_pairs(HbEvalArgs* args, void* ws, size_t ws_bytes, void* stream, HbError* err);

/* ---------------------------------------------------------------------------
 * CRK linear correction coefficients from the 10 accumulated moments
 * (hb/hydro.py:115-150): per gas row with m0 > 0, 2-norm condition number of
 * m2 (symmetric: |lambda|max/|lambda|min) < cond_limit, B = m2^-1 m1 by
 * partially pivoted elimination, A = 1/(m0 - B.m1) with the |d| > 1e-300
 * guard, fallback A = 1/m0, B = 0.  Float64.
 * ------------------------------------------------------------------------- */
/* assign_timestep_levels (hb/hydro.py:277-317) on the device: per-row
 * levels (uint8) from the gas CFL / dark-matter acceleration timestep,
 * leaf levels (int64) = max over members, all leaves set to the overall
 * maximum when `flat`.  dev_max: 3 device int64 of scratch; max_host[3] <-
 * (max row level, max leaf level, max level over non-ghost-only leaves).  The
 * caller raises StiffStateError when max_host[0] > n_levels - 1 (the row
 * levels are then clamped to 255).  One stream sync.  Replaces the numpy body
 * of assign_timestep_levels. */
int hb_timestep_levels(int64_t n, const double* vel, const double* internal_energy,
                       const double* smoothing, const double* accel, const uint8_t* species,
                       double cfl, double softening, double eos_gamma, double dt_pm,
                       int64_t n_leaves, const int64_t* leaf_start, const int64_t* leaf_end,
                       const uint8_t* leaf_ghost_only, int32_t flat, uint8_t* level,
                       int64_t* leaf_level, int64_t* dev_max, int64_t* max_host, void* stream,
                       HbError* err);

int hb_crk_solve(int64_t n, const double* moments, int64_t stride, const uint8_t* species,
                 double cond_limit, double* A, double* B, uint8_t* fallback, void* stream,
                 HbError* err);

/* ---------------------------------------------------------------------------
 * Resident force evaluation: the s = 0 boundary of subcycle_pm_step
 * (hb/stepper.py:113-179) with the reference's ordered, single-count pair
 * semantics: build_mesh_and_leaves -> assemble_interaction_lists
 * -> neighbour count -> compute_density (+ alias sync) -> refresh_eos_columns ->
 * CRK moments + solve -> short-range gravity -> hydro force, all on device.
 * Particle fields are read from *_in and written reordered (leaf order, as
 * the reference reorders its ParticleSet in place) to the output fields.
 * ------------------------------------------------------------------------- */
#define HB_PASS_NCOUNT 1
#define HB_PASS_DENSITY 2
#define HB_PASS_CRK 4
#define HB_PASS_GRAVITY 8
#define HB_PASS_HYDRO 16
#define HB_PASS_ALL 31
/* Untimed accounting pass (bench.py's roofline): with HB_PASS_GRAVITY, the
 * gravity pass counts instead of summing forces -- grav[0..n) viewed as
 * int64 receives, per row, the exact number of sources j != i within r_cut
 * (float64 re-check of every FP32 decision near the threshold, as the
 * reference's r2 <= reach2 test, hb/kernels.py:357-359). */
#define HB_PASS_COUNT_ONLY 32
/* Optional, with HB_PASS_CRK: the CRK coefficient gradients gradA / gradB
 * (the north star's "A, B, gradA, gradB"; not in the reference, whose
 * compute_crk_coefficients stops at A, B -- hb/hydro.py:99-150).  One more
 * gas pass after the CRK solve (gradient moments + a float64 per-row solve)
 * into HbStepArgs.crk_gradA / crk_gradB. */
#define HB_PASS_CRK_GRAD 64

typedef struct HbStepArgs {
  int64_t n;
  /* inputs (n rows, ParticleSet layout) */
  const double* pos_in; const double* vel_in; const double* mass_in;
  const double* smoothing_in; const double* internal_energy_in; const double* density_in;
  const uint8_t* species_in; const uint8_t* ghost_in; const int8_t* image_shift_in;
  const int64_t* global_id_in; const int64_t* ghost_src_in; /* ghost_src may be NULL */
  /* reordered outputs (may not alias the inputs) */
  double* pos; double* vel; double* mass; double* smoothing; double* internal_energy;
  double* density; uint8_t* species; uint8_t* ghost; int8_t* image_shift; int64_t* global_id;
  int64_t* ghost_src;
  /* mesh (host scalars) */
  double side_length; double lo[3]; double width[3]; int64_t nb[3]; uint8_t periodic[3];
  int64_t max_leaf_size;
  /* physics (host scalars) */
  double reach;      /* list reach = max(r_cut, 2 h_max)                       */
  double h_max;      /* max smoothing length (kernel supports 2 h_max)        */
  double h_min;      /* min gas smoothing length (sizes the float64 re-check band) */
  double r_s, r_cut, softening, eos_gamma, visc_alpha, visc_beta;
  int32_t passes;    /* HB_PASS_* mask                                        */
  int32_t timing;    /* 1: fill ms_phase with per-phase device times          */
  int32_t gravity_mode; /* 0 auto (= 4 when every bin fits the tiler, else 1),
                           1 leaf tiles + leaf list, 4 bin tiles + 27-bin
                           stencil (k_gravity, soft-bits table).  2 and 3
                           (round 1's half-warp and r/t-table variants) were
                           removed and return HB_CONTRACT                     */
  int32_t ghost_density; /* 1: ghost-only leaves are density receivers too, so
                            ghost rows near the rank face get fresh rho, P, c_s
                            (multi-rank; fixes SURVEY.md finding 4); gravity,
                            CRK and hydro still skip ghost-only receivers     */
  int32_t owned_targets; /* 1: gravity and pass B (CRK + hydro) skip target
                            tiles without an owned row (ghost == 0); rows of
                            skipped tiles read 0.  For rank sets whose ghost
                            outputs are discarded (multi-rank).  Pass A still
                            serves every row (ghost densities).             */
  int64_t list_capacity; /* entries the workspace was sized for              */
  /* optional cudaEvent_t handles (void*, NULL = unused) for overlapping host
     copies with the step: the step waits on fields_ready before it first reads
     any input field other than pos / image_shift / ghost (the mesh build only
     needs those), and records sph_done once ncount, density, CRK and hydro
     outputs are final (gravity still running).  With late_fields set as well,
     fields_ready covers only mass / smoothing / species; vel, density,
     internal_energy, global_id and ghost_src are first read after the step
     waits on late_fields, which happens after SPH pass A and before the EOS */
  void* fields_ready_event;
  void* sph_done_event;
  void* late_fields_event;
  /* outputs (device, leaf order) */
  int64_t* perm;        /* (n) row k = input row perm[k]                    */
  double* ncount;       /* (n)                                                */
  double* grav;         /* (n,3) m_i a_i short-range gravity                  */
  double* hydro;        /* (n,5) fx fy fz m du/dt (edot_i) edot_j             */
  double* crk_moments;  /* (n,10), or NULL: the moments then live inside the
                           workspace (over scratch that is dead by pass B) and
                           crk_moments_out says where; valid until the
                           workspace is reused                               */
  double* crk_A;        /* (n)                                                */
  double* crk_B;        /* (n,3)                                              */
  uint8_t* crk_fallback;/* (n)                                                */
  /* host outputs */
  int64_t n_leaves, n_entries, list_capacity_needed;
  float ms_phase[8];    /* build, list, tiling, sph A (count+density+eos),
                           sph B (crk+hydro+solve), gravity, tail, total */
  void* status_out;     /* optional pinned host uint64_t[3] (zeroed by the caller):
                           when non-NULL (and timing == 0) the step does NOT
                           synchronise at its end; the error key and overflow
                           flags are copied there asynchronously and the
                           caller decodes them with hb_force_step_check()
                           once the stream has completed                      */
  float ms_kernel[4];   /* timing=1: event-timed single-kernel spans on the step
                           stream: gravity pair kernel, SPH pass A kernel, SPH
                           pass B kernel, 0 (reserved) -- roofline inputs     */
  double* crk_moments_out; /* out: where the (n,10) moments were written     */
  void* grav_half_event;   /* optional cudaEvent_t: bin gravity runs in two
                              launches split at bin 4 nb/5 and records this
                              event between them; rows [0, grav_split_row)
                              of `grav` are final from then on (the rest at
                              the end of the step), so their copy-out can
                              overlap the second launch                       */
  int64_t grav_split_row;  /* out (host, set before the call returns)         */
  double* crk_gradA;  /* HB_PASS_CRK_GRAD: (n,3) d A / d x_i, or NULL          */
  double* crk_gradB;  /* HB_PASS_CRK_GRAD: (n,3,3) d B_a / d x_g, or NULL      */
  void* last_fields_event; /* optional, with late_fields_event, for sets with
                              no ghost rows (ghost == 0, ghost_src < 0
                              everywhere): late_fields then covers only vel and
                              internal_energy; density, global_id and ghost_src
                              are first read after the step waits on this one,
                              which happens after SPH pass B (the non-gas rows'
                              density and the ids are outputs only)           */
} HbStepArgs;

size_t hb_force_step_workspace(int64_t n, const int64_t nb[3], int64_t max_leaf_size,
                               int64_t list_capacity);
/* The same for steps restricted to `passes` (e.g. HB_PASS_GRAVITY: no room
 * for workspace-resident CRK moments). */
size_t hb_force_step_workspace_passes(int64_t n, const int64_t nb[3], int64_t max_leaf_size,
                                      int64_t list_capacity, int32_t passes);
int hb_force_step(HbStepArgs* args, void* ws, size_t ws_bytes, void* stream, HbError* err);
/* Decode a deferred status (HbStepArgs.status_out) after the step's stream has
 * completed: the status the synchronous call would have returned. */
int hb_force_step_check(const void* status, HbError* err);

/* ---------------------------------------------------------------------------
 * Overload-shell exchange (multi-GPU ranks).  Distributed build_overload /
 * refresh_overload (hb/domain.py:88-189): cuboid ranks of grid g (x-major ids),
 * ghost copy of an owned particle for every (rank r, image s) with pos + s L
 * strictly inside r's bounds widened by w (except its owned copy), owned copy
 * to its (new) owner; DriftError flag for > 1 domain hop.  periodic_unsplit:
 * axes with g = 1 stay periodic in the rank mesh (no self-image ghosts there).
 * stay != NULL: rows that remain owned here are flagged (mode 0) and not
 * emitted, so only shell ghosts and migrants cross the exchange; their number
 * is accumulated into counts[n_ranks * 28 + 1] (counts has n_ranks*28 + 2
 * entries: slots, drift word, staying rows).  Records are
 * hb_halo_record_bytes() wide; slots = dest * 28 + code (27 = owned).
 * hb_halo_select: mode 0 counts per slot, mode 1 emits rows/slots at `fill`
 * offsets.  hb_halo_unpack orders owned rows by global_id then ghosts by
 * (global_id, shift) (hb/domain.py:135-138) into SoA rank fields; key_bits
 * >= bit_length(27 * max_global_id + 26) (0: keep record order).
 * ------------------------------------------------------------------------- */
int64_t hb_halo_record_bytes(void);
int hb_halo_select(int64_t n, const double* pos, const uint8_t* ghost, const int32_t g[3],
                   double side_length, double overload_width, int32_t self,
                   int32_t periodic_unsplit, int32_t mode, uint64_t* counts, uint64_t* fill,
                   int64_t* out_row, int32_t* out_slot, int32_t* drift_flag, uint8_t* stay,
                   void* stream, HbError* err);
int hb_halo_pack(int64_t m, const int64_t* rows, const int32_t* slots, const double* pos,
                 const double* vel, const double* mass, const double* smoothing,
                 const double* internal_energy, const double* density, const uint8_t* species,
                 const int64_t* global_id, const int32_t g[3], double side_length, int32_t self,
                 void* out, void* stream, HbError* err);
size_t hb_halo_unpack_workspace(int64_t m);
int hb_halo_unpack(int64_t m, const void* recs, int32_t key_bits, int64_t row0, double* pos,
                   double* vel, double* mass, double* smoothing, double* internal_energy,
                   double* density, uint8_t* species, uint8_t* ghost, int8_t* image_shift,
                   int64_t* global_id, int64_t* ghost_src, void* ws, size_t ws_bytes,
                   void* stream, HbError* err);
int hb_halo_resolve_sources(int64_t n_owned, int64_t m, const int64_t* global_id,
                            int64_t* ghost_src, void* stream, HbError* err);
/* Fused exchange halves (one C call each; the per-call host round trips, not
 * the data, dominate the exchange at 1-4 M rows per rank).  HbFieldSet: the
 * SoA rank fields (all device pointers).
 * hb_halo_pack_all: select (count) -> counts to counts_host (one stream sync)
 * -> device scan -> select (emit) -> pack.  The source may hold ghost rows
 * (only ghost == 0 rows are sources).  Returns HB_OVERFLOW, with counts_host
 * filled, when the records exceed cap (caller grows rows/slots/send, retries).
 * hb_halo_unpack_keep: dst rows [0, n_stay) = the stay-flagged src rows in
 * row order, then the m received records from row n_stay as hb_halo_unpack. */
typedef struct HbFieldSet {
  double *pos, *vel, *mass, *smoothing, *internal_energy, *density;
  uint8_t *species, *ghost;
  int8_t* image_shift;
  int64_t *global_id, *ghost_src;
} HbFieldSet;
size_t hb_halo_pack_all_workspace(int32_t n_ranks);
int hb_halo_pack_all(int64_t n, const HbFieldSet* src, const int32_t g[3], double side_length,
                     double overload_width, int32_t self, int32_t periodic_unsplit,
                     uint64_t* counts, uint64_t* counts_host, uint8_t* stay, int64_t cap,
                     int64_t* rows, int32_t* slots, void* send, void* ws, size_t ws_bytes,
                     void* stream, HbError* err);
size_t hb_halo_unpack_keep_workspace(int64_t n_src, int64_t m);
int hb_halo_unpack_keep(int64_t m, const void* recs, int32_t key_bits, int64_t n_src,
                        const HbFieldSet* src, const uint8_t* stay, int64_t n_stay,
                        const HbFieldSet* dst, void* ws, size_t ws_bytes, void* stream,
                        HbError* err);
/* ---------------------------------------------------------------------------
 * Particle-mesh long-range gravity (hb/gravity.py:58-245).
 * Grids are float64 row-major (n, n, n); spectra half-complex (n, n, n/2+1)
 * interleaved (re, im) float64, as cuFFT / torch.fft produce them.
 * hb_pm_deposit: CIC mass deposition onto cell centres (periodic), then divided
 *   by cell_volume (pass spacing ** 3 as the caller computes it).
 * hb_pm_spectral: phi_k = -four_pi_g rho_k D(k) (phi_0 = 0) and the three
 *   force spectra -i k_d phi_k; phi_k may be NULL.
 * hb_pm_interp: CIC gather of n_fields (1..3) grids at the positions into
 *   out (np, n_fields). */
int hb_pm_deposit(int64_t np, const double* pos, const double* mass, int64_t grid_n,
                  double spacing, double cell_volume, double* rho, void* stream, HbError* err);
int hb_pm_spectral(int64_t grid_n, double side_length, double four_pi_g, const void* rho_k,
                   const double* influence, void* fx_k, void* fy_k, void* fz_k, void* phi_k,
                   void* stream, HbError* err);
int hb_pm_interp(int64_t np, const double* pos, int32_t n_fields, const double* f0,
                 const double* f1, const double* f2, int64_t grid_n, double spacing,
                 double* out, void* stream, HbError* err);
/* ---------------------------------------------------------------------------
 * In-situ cluster finding (hb/insitu.py:25-142).
 * hb_fof_scan: radius-wide cell grid (lo, inv_w, ncell as _grid_geometry),
 *   27-stencil sweep over binpos (n,3) with the reference's float64 edge test
 *   from the lower row's side.  mode 0: FOF union into parent (init arange,
 *   flattened on return: root = smallest row of the component); 1: counts[i]
 *   += neighbours within r (self included); 2: union of core-core edges;
 *   3: border_key[i] = min(border_key[i], core_label[j]) over core neighbours
 *   j of non-core i.  Unused arrays may be NULL.
 * hb_uf_union_edges: union of the m edges (a[k], b[k]) into parent (n) and
 *   flatten (global-id stitching of rank components).
 * hb_crc32c: CRC32C (Castagnoli) of a HOST buffer, running value in/out. */
size_t hb_fof_workspace(int64_t n, const int64_t ncell[3]);
int hb_fof_scan(int64_t n, const double* binpos, const double lo[3], const double inv_w[3],
                const int64_t ncell[3], double side_length, int32_t periodic, double r2max,
                int32_t mode, int64_t* parent, const uint8_t* core, int64_t* counts,
                int64_t* border_key, const int64_t* core_label, void* ws, size_t ws_bytes,
                void* stream, HbError* err);
int hb_uf_union_edges(int64_t m, const int64_t* a, const int64_t* b, int64_t n, int64_t* parent,
                      void* stream, HbError* err);
uint32_t hb_crc32c(const void* data, size_t nbytes, uint32_t value);
/* CRC32C of a DEVICE buffer (HCKP checkpoint codec, hb/tiered_io.py:80-142):
 * parallel per-chunk CRCs folded with GF(2) zero-shift operators; writes the
 * standard CRC32C to *out_host and synchronises the stream. */
size_t hb_crc32c_device_workspace(int64_t nbytes);
int hb_crc32c_device(const void* data, int64_t nbytes, uint32_t* out_host, void* ws,
                     size_t ws_bytes, void* stream, HbError* err);
/* Row indices of the nonzero flags in row order (a device compaction whose
 * size the caller already knows -- no host sync). */
size_t hb_flag_indices_workspace(int64_t n);
int hb_flag_indices(int64_t n, const uint8_t* flags, int64_t* idx, void* ws, size_t ws_bytes,
                    void* stream, HbError* err);

#ifdef __cplusplus
}
#endif
#endif /* HB_H_ */
