// hb_step.cu -- device-resident force evaluation (hb_force_step, include/hb.h).
//
// One call = the s = 0 boundary of subcycle_pm_step (hb/stepper.py:113-179)
// with ordered single-count pair semantics: mesh build + reorder, list sweep
// straight into a receiver CSR (the list is born grouped by receiver), two
// tilings shared by all passes (gas-only for the SPH kernels, all species for
// gravity), then ncount -> density (+EOS) -> CRK moments + solve -> gravity ->
// hydro with the lean pair kernels.  Host syncs: the leaf count and the list
// entry count (both needed to size launches); everything else is stream-ordered.
#include "hb_internal.cuh"

namespace hb {


// density write-back for gas rows of active leaves (hb/hydro.py:73-80), then
// EOS columns for every row (hb/hydro.py:48-57)
__global__ void k_density_update(int64_t n_leaves, const int64_t* leaf_start,
                                 const int64_t* leaf_end, const uint8_t* ghost_only,
                                 const uint8_t* species, const double* rho_new, double* density) {
  int64_t leaf = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (leaf >= n_leaves || ghost_only[leaf]) return;
  for (int64_t r = leaf_start[leaf] + lane; r < leaf_end[leaf]; r += 32)
    if (species[r] == 1) density[r] = rho_new[r];
}
__global__ void k_alias_sync(int64_t n, const int64_t* ghost_src, double* density) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && ghost_src[i] >= 0) density[i] = density[ghost_src[i]];
}
__global__ void k_zero_ghost_rows(int64_t n_leaves, const int64_t* leaf_start,
                                  const int64_t* leaf_end, const uint8_t* ghost_only,
                                  double* ncount, double* moments, double* hydro, double* grav) {
  int64_t leaf = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (leaf >= n_leaves || !ghost_only[leaf]) return;
  for (int64_t r = leaf_start[leaf] + lane; r < leaf_end[leaf]; r += 32) {
    if (ncount) ncount[r] = 0.0;
    if (moments) for (int c = 0; c < 10; ++c) moments[r * 10 + c] = 0.0;
    if (hydro) for (int c = 0; c < 5; ++c) hydro[r * 5 + c] = 0.0;
    if (grav) for (int c = 0; c < 3; ++c) grav[r * 3 + c] = 0.0;
  }
}

__global__ void k_gather_inverse(int64_t n, const int64_t* perm, int64_t* inv) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) inv[perm[k]] = k;
}
__global__ void k_ghost_src(int64_t n, const int64_t* perm, const int64_t* inv,
                            const int64_t* src_in, int64_t* src_out) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  int64_t g = src_in[perm[k]];
  src_out[k] = g >= 0 ? inv[g] : -1;
}


// mesh order <- input order for every field (hb/particles.py:135-154 reorder):
// each row reads its source row once.  The gathered leaf-order SoA fields are
// both the step's outputs and the rows every later kernel reads (Rows); no
// (n,12) state matrix is built.
struct FieldIn {
  const double *pos, *vel, *mass, *h, *u, *rho;
  const uint8_t *species, *ghost;
  const int8_t* shift;
  const int64_t* gid;
};
struct FieldOut {
  double *pos, *vel, *mass, *h, *u, *rho;
  uint8_t *species, *ghost;
  int8_t* shift;
  int64_t* gid;
};
// late half of a split gather (HbStepArgs.late_fields_event): the fields SPH
// pass A does not read.  PART 0: all of them; PART 1: vel, internal energy
// (pass B needs them); PART 2: density of the non-gas rows (gas rows hold pass
// A's) and global id (HbStepArgs.last_fields_event: needed only by the outputs)
template <int PART>
__global__ void k_gather_late(int64_t n, const int64_t* perm, FieldIn in, FieldOut out) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  int64_t r = perm[k];
  if (PART != 2) {
#pragma unroll
    for (int d = 0; d < 3; ++d) out.vel[3 * k + d] = in.vel[3 * r + d];
    out.u[k] = in.u[r];
  }
  if (PART != 1) {
    out.gid[k] = in.gid[r];
    if (PART == 0 || out.species[k] != 1)   // gas rows get pass A's density
      out.rho[k] = in.rho[r];
  }
}

// LATE = true: skip the late fields (vel, u, density, ids), which pass A does
// not read (pass B's records compute P and c_s from the SoA density and
// internal energy)
// h_lim: the h_max the step's reach, bin width and culls were sized from
// (HbStepArgs.h_max).  A gas row above it would silently lose the pairs
// between 2 h_max and 2 h_i, so it raises HB_CONTRACT (error key code 3)
// instead (the reference recomputes smoothing.max() per call, hb/hydro.py:67).
constexpr int kGatherBlock = 256;
template <bool LATE>
__global__ void __launch_bounds__(kGatherBlock)
k_gather_fields(int64_t n, const int64_t* perm, FieldIn in, FieldOut out, double h_lim,
               unsigned long long* err_key, int no_ghosts) {
  int64_t k = (int64_t)blockIdx.x * kGatherBlock + threadIdx.x;
  if (k >= n) return;
  int64_t r = perm[k];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    out.pos[3 * k + d] = in.pos[3 * r + d];
    if (!LATE) out.vel[3 * k + d] = in.vel[3 * r + d];
    out.shift[3 * k + d] = in.shift[3 * r + d];
  }
  double h = in.h[r];
  uint8_t sp = in.species[r], gh = in.ghost[r];
  out.mass[k] = in.mass[r]; out.h[k] = h;
  out.species[k] = sp; out.ghost[k] = gh;
  // HbStepArgs.last_fields_event is for sets without ghost rows (ghost rows
  // would need their input density before pass B)
  if (no_ghosts && gh != 0) atomicMin(err_key, 7ull);
  if (sp == 1 && !(h <= h_lim)) atomicMin(err_key, 3ull);
  if (!LATE) {
    out.rho[k] = in.rho[r];
    out.u[k] = in.u[r];
    out.gid[k] = in.gid[r];
  }
}

struct StepWs {
  // mesh
  int64_t *leaf_start, *leaf_end, *leaf_bin, *bin_ptr, *n_leaves_dev;
  double *leaf_lo, *leaf_hi;
  uint8_t* ghost_only;
  // list csr
  int64_t* ent_ptr;
  int32_t *ent_src, *ent_code;
  // engine
  Tiling Tg, Ta;
  int64_t *ntg, *nta;
  double *rho_new, *inv_tmp;
  float4 *P0, *P1, *P2;
  unsigned long long* err_key;
  int64_t* inv;
  uint8_t* no_ghost;
  int64_t *seg_s, *seg_e, *st_ptr;
  int32_t *st_src, *st_code;
};

static void carve_step(Arena& ws, int64_t n, int64_t nbins, int64_t cap, int64_t lcap, StepWs& w) {
  w.leaf_start = ws.take<int64_t>(cap); w.leaf_end = ws.take<int64_t>(cap);
  w.leaf_bin = ws.take<int64_t>(cap); w.bin_ptr = ws.take<int64_t>(nbins + 1);
  w.n_leaves_dev = ws.take<int64_t>(1);
  w.leaf_lo = ws.take<double>(3 * cap); w.leaf_hi = ws.take<double>(3 * cap);
  w.ghost_only = ws.take<uint8_t>(cap);
  w.ent_ptr = ws.take<int64_t>(cap + 1);
  w.ent_src = ws.take<int32_t>(lcap + 1); w.ent_code = ws.take<int32_t>(lcap + 1);
  carve_tiling(ws, n, cap > nbins ? cap : nbins, w.Tg);
  carve_tiling(ws, n, cap, w.Ta);
  w.ntg = ws.take<int64_t>(1); w.nta = ws.take<int64_t>(2);
  w.rho_new = ws.take<double>(n + 1);
  w.P0 = ws.take<float4>(n + 1); w.P1 = ws.take<float4>(n + 1); w.P2 = ws.take<float4>(n + 1);
  w.err_key = ws.take<unsigned long long>(1);
  w.inv = ws.take<int64_t>(n + 1);
  w.no_ghost = ws.take<uint8_t>(cap + 1);
  w.seg_s = ws.take<int64_t>(nbins + 1); w.seg_e = ws.take<int64_t>(nbins + 1);
  w.st_ptr = ws.take<int64_t>(nbins + 1);
  w.st_src = ws.take<int32_t>(nbins * 27 + 1); w.st_code = ws.take<int32_t>(nbins * 27 + 1);
}

constexpr bool kGravityBinsDefault = true;

// rows of bins < half: leaf_start of the first leaf at or after bin `half`
__global__ void k_split_row(const int64_t* bin_ptr, const int64_t* leaf_start, int64_t half,
                            int64_t n_leaves, int64_t n, int64_t* out) {
  if (threadIdx.x || blockIdx.x) return;
  int64_t l = bin_ptr[half];
  *out = l < n_leaves ? leaf_start[l] : n;
}

// error key (min over the step): leaf * 4 + code; code 1 non-finite partial,
// 2 accumulator overflow, 3 gas smoothing length above the step's h_max
static int step_key_error(unsigned long long ek, HbError* err) {
  if (err) { err->leaf_a = -1; err->leaf_b = -1; }
  if (ek == 7)
    return set_err(err, HB_CONTRACT, "last_fields_event given for a set with ghost rows");
  if (ek % 4 == 3)
    return set_err(err, HB_CONTRACT, "gas smoothing length exceeds the step's h_max");
  return set_err(err, (ek % 4) == 1 ? HB_NONFINITE : HB_OVERFLOW,
                 (ek % 4) == 1 ? "non-finite partial" : "accumulator overflow");
}

struct GhostZeroCtx {  // zeroes the gravity rows of ghost-only leaves (between halves)
  int64_t nl;
  const int64_t *leaf_start, *leaf_end;
  const uint8_t* ghost_only;
  double* grav;
  cudaStream_t st;
};
static int zero_grav_ghost_rows(void* p) {
  GhostZeroCtx* c = (GhostZeroCtx*)p;
  HbError* err = nullptr;
  k_zero_ghost_rows<<<grid_for(c->nl * 32, 256), 256, 0, c->st>>>(
      c->nl, c->leaf_start, c->leaf_end, c->ghost_only, nullptr, nullptr, nullptr, c->grav);
  HB_LAUNCH_CHECK();
  return HB_OK;
}

struct PhaseTimer {
  bool on;
  cudaStream_t st;
  cudaEvent_t ev[9];
  cudaEvent_t kv[6];  // start/stop of gravity, SPH pass A, SPH pass B kernels
  int k = 0;
  PhaseTimer(bool on_, cudaStream_t s) : on(on_), st(s) {
    if (on) {
      for (int i = 0; i < 9; ++i) cudaEventCreate(&ev[i]);
      for (int i = 0; i < 6; ++i) cudaEventCreate(&kv[i]);
    }
  }
  ~PhaseTimer() {
    if (on) {
      for (int i = 0; i < 9; ++i) cudaEventDestroy(ev[i]);
      for (int i = 0; i < 6; ++i) cudaEventDestroy(kv[i]);
    }
  }
  void mark(int i) { if (on) cudaEventRecord(ev[i], st); }
  void kmark(int i) { if (on) cudaEventRecord(kv[i], st); }
};

int force_step(HbStepArgs* a, Arena& ws, cudaStream_t st, HbError* err) {
  int64_t n = a->n;
  int64_t nbins = a->nb[0] * a->nb[1] * a->nb[2];
  int64_t cap = hb_leaf_capacity(n, nbins, a->max_leaf_size);
  StepWs w;
  carve_step(ws, n, nbins, cap, a->list_capacity, w);
  // nested arenas (mesh build, list csr, tilings) reuse the space after the carve.
  // With crk_moments == NULL the moments live there too, past the scratch the
  // bin gravity needs after pass B; only scratch that is dead before pass B
  // (mesh build, list csr, SPH tiling) overlaps them.  Saves 48 of the 80 B
  // per row the caller's buffer would cost (2x512^3 then fits one GPU).
  size_t mom_end = 0;
  double* mom = a->crk_moments;
  a->crk_moments_out = nullptr;
  if (a->passes & (HB_PASS_CRK | HB_PASS_HYDRO)) {  // gravity-only steps keep no moments
    Arena g = ws;
    g.dry = true;
    GravBinArgs gd = {};
    gd.n = n; gd.nbins = nbins;
    gravity_bins(gd, g, st, err);
    Arena mm = ws;
    mm.used = g.used;
    double* p = mm.take<double>(n * 10 + 1);
    mom_end = mm.used;
    if (!mom) mom = p;
  }
  a->crk_moments_out = mom;
  HbMeshArgs m = {};
  m.n = n; m.pos = a->pos_in; m.image_shift = a->image_shift_in; m.ghost = a->ghost_in;
  m.side_length = a->side_length;
  for (int d = 0; d < 3; ++d) { m.lo[d] = a->lo[d]; m.width[d] = a->width[d]; m.nb[d] = a->nb[d]; }
  m.max_leaf_size = a->max_leaf_size; m.leaf_cap = cap;
  m.perm = a->perm; m.leaf_start = w.leaf_start; m.leaf_end = w.leaf_end; m.leaf_lo = w.leaf_lo;
  m.leaf_hi = w.leaf_hi; m.leaf_ghost_only = w.ghost_only; m.leaf_bin = w.leaf_bin;
  m.bin_ptr = w.bin_ptr; m.n_leaves_dev = w.n_leaves_dev;
  int64_t nl = 0, max_bin_count = 0;
  m.n_leaves_host = &nl;
  m.max_bin_count_host = &max_bin_count;
  ListArgsDev ld;
  if (ws.dry) {
    size_t mx = ws.used;
    Arena s1 = ws; build_mesh(&m, s1, st, err); if (s1.used > mx) mx = s1.used;
    ld.n_leaves = cap;
    Arena s2 = ws; assemble_csr(ld, a->list_capacity, nullptr, nullptr, nullptr, nullptr, s2, st, err);
    if (s2.used > mx) mx = s2.used;
    Arena s3 = ws;
    build_tiling(w.Tg, cap, nullptr, nullptr, Rows{}, nullptr, 0.0, 1, nullptr, s3, st, err);
    if (s3.used > mx) mx = s3.used;
    GravBinArgs gb = {};
    gb.n = n; gb.nbins = nbins;
    Arena s4 = ws; gravity_bins(gb, s4, st, err); if (s4.used > mx) mx = s4.used;
    if (mom_end > mx) mx = mom_end;
    ws.used = mx;
    return HB_OK;
  }
  if (!ws.ok() || mom_end > ws.cap) return set_err(err, HB_CONTRACT, "workspace too small (step)");
  if (a->gravity_mode == 2 || a->gravity_mode == 3)
    return set_err(err, HB_CONTRACT, "gravity_mode 2 / 3 (half-warp, r/t tables) were removed");
  if (n <= 0) return HB_OK;
  if (n >= (1LL << 31)) return set_err(err, HB_CONTRACT, "too many rows for one rank");
  PhaseTimer tm(a->timing != 0, st);
  tm.mark(0);
  // 1. mesh + reorder
  {
    Arena s = ws;
    int rc = build_mesh(&m, s, st, err);
    if (rc) return rc;
  }
  a->n_leaves = nl;
  a->grav_split_row = n;
  if (a->grav_half_event) {  // rows of bins < nbins/2, final after the first gravity half
    // scratch: the 256-B arena slot of err_key has room after its 8 bytes
    int64_t* split_dev = (int64_t*)(w.err_key + 1);
    k_split_row<<<1, 32, 0, st>>>(w.bin_ptr, w.leaf_start, grav_split_bin(nbins), nl, n,
                                  split_dev);
    HB_LAUNCH_CHECK();
    HB_CUDA_TRY(cudaMemcpyAsync(&a->grav_split_row, split_dev, sizeof(int64_t),
                                cudaMemcpyDeviceToHost, st));
    HB_CUDA_TRY(cudaStreamSynchronize(st));
  }
  if (a->fields_ready_event)
    HB_CUDA_TRY(cudaStreamWaitEvent(st, (cudaEvent_t)a->fields_ready_event, 0));
  bool late_split = a->late_fields_event != nullptr;
  // four upload groups (include/hb.h): density / ids / ghost sources last
  bool last_split = late_split && a->last_fields_event != nullptr;
  // SPH passes size every cull from h_max; gravity-only steps read no h
  double h_lim = (a->passes & ~HB_PASS_GRAVITY) ? a->h_max * (1.0 + 1e-12) : INFINITY;
  HB_CUDA_TRY(cudaMemsetAsync(w.err_key, 0xff, sizeof(unsigned long long), st));
  // every kernel after the gather reads the leaf-order output fields
  Rows rows;
  rows.pos = a->pos; rows.vel = a->vel; rows.mass = a->mass; rows.h = a->smoothing;
  rows.rho = a->density; rows.u = a->internal_energy; rows.sp = a->species;
  rows.gamma = a->eos_gamma;
  {
    unsigned g1 = grid_for(n, 256);
    FieldIn fi = {a->pos_in, a->vel_in, a->mass_in, a->smoothing_in, a->internal_energy_in,
                  a->density_in, a->species_in, a->ghost_in, a->image_shift_in, a->global_id_in};
    FieldOut fo = {a->pos, a->vel, a->mass, a->smoothing, a->internal_energy, a->density,
                   a->species, a->ghost, a->image_shift, a->global_id};
    if (late_split) {
      k_gather_fields<true><<<grid_for(n, kGatherBlock), kGatherBlock, 0, st>>>(
          n, a->perm, fi, fo, h_lim, w.err_key, last_split ? 1 : 0);
    } else {
      k_gather_fields<false><<<grid_for(n, kGatherBlock), kGatherBlock, 0, st>>>(
          n, a->perm, fi, fo, h_lim, w.err_key, 0);
      if (a->ghost_src_in && a->ghost_src) {
        k_gather_inverse<<<g1, 256, 0, st>>>(n, a->perm, w.inv);
        k_ghost_src<<<g1, 256, 0, st>>>(n, a->perm, w.inv, a->ghost_src_in, a->ghost_src);
        HB_COUNT_LAUNCH(2);
      }
    }
    HB_LAUNCH_CHECK();
  }
  // the late fields (split gather): waited for and gathered after pass A
  auto gather_late = [&]() -> int {
    if (!late_split) return HB_OK;
    late_split = false;
    HB_CUDA_TRY(cudaStreamWaitEvent(st, (cudaEvent_t)a->late_fields_event, 0));
    unsigned g1 = grid_for(n, 256);
    FieldIn fi = {a->pos_in, a->vel_in, a->mass_in, a->smoothing_in, a->internal_energy_in,
                  a->density_in, a->species_in, a->ghost_in, a->image_shift_in, a->global_id_in};
    FieldOut fo = {a->pos, a->vel, a->mass, a->smoothing, a->internal_energy, a->density,
                   a->species, a->ghost, a->image_shift, a->global_id};
    if (last_split) {
      k_gather_late<1><<<g1, 256, 0, st>>>(n, a->perm, fi, fo);
      HB_LAUNCH_CHECK();
      return HB_OK;
    }
    k_gather_late<0><<<g1, 256, 0, st>>>(n, a->perm, fi, fo);
    if (a->ghost_src_in && a->ghost_src) {
      k_gather_inverse<<<g1, 256, 0, st>>>(n, a->perm, w.inv);
      k_ghost_src<<<g1, 256, 0, st>>>(n, a->perm, w.inv, a->ghost_src_in, a->ghost_src);
      HB_COUNT_LAUNCH(2);
    }
    HB_LAUNCH_CHECK();
    return HB_OK;
  };
  // the last fields (density of non-gas rows, ids, ghost sources): outputs only
  auto gather_last = [&]() -> int {
    if (!last_split) return HB_OK;
    last_split = false;
    HB_CUDA_TRY(cudaStreamWaitEvent(st, (cudaEvent_t)a->last_fields_event, 0));
    unsigned g1 = grid_for(n, 256);
    FieldIn fi = {a->pos_in, a->vel_in, a->mass_in, a->smoothing_in, a->internal_energy_in,
                  a->density_in, a->species_in, a->ghost_in, a->image_shift_in, a->global_id_in};
    FieldOut fo = {a->pos, a->vel, a->mass, a->smoothing, a->internal_energy, a->density,
                   a->species, a->ghost, a->image_shift, a->global_id};
    k_gather_late<2><<<g1, 256, 0, st>>>(n, a->perm, fi, fo);
    if (a->ghost_src_in && a->ghost_src) {
      k_gather_inverse<<<g1, 256, 0, st>>>(n, a->perm, w.inv);
      k_ghost_src<<<g1, 256, 0, st>>>(n, a->perm, w.inv, a->ghost_src_in, a->ghost_src);
      HB_COUNT_LAUNCH(2);
    }
    HB_LAUNCH_CHECK();
    return HB_OK;
  };
  tm.mark(1);
  // 2. ordered list as a receiver CSR
  ld.n_leaves = nl; ld.leaf_bin = w.leaf_bin; ld.leaf_level = nullptr; ld.bin_ptr = w.bin_ptr;
  ld.bin_ids = nullptr; ld.leaf_lo = w.leaf_lo; ld.leaf_hi = w.leaf_hi; ld.ghost_only = w.ghost_only;
  if (a->ghost_density) {  // every leaf receives (ghost-only ones feed fresh ghost densities)
    HB_CUDA_TRY(cudaMemsetAsync(w.no_ghost, 0, nl + 1, st));
    ld.ghost_only = w.no_ghost;
  }
  for (int d = 0; d < 3; ++d) { ld.g.nb[d] = a->nb[d]; ld.g.periodic[d] = a->periodic[d]; }
  ld.g.L = a->side_length; ld.g.reach = a->reach; ld.g.active_depth = 0;
  {
    Arena s = ws;
    int64_t total = 0;
    int rc = assemble_csr(ld, a->list_capacity, w.ent_src, w.ent_code, w.ent_ptr, &total, s, st, err);
    a->n_entries = total;
    a->list_capacity_needed = total;
    if (rc) return rc;
  }
  tm.mark(2);
  // 3. tilings over the gathered leaf-order fields
  w.Tg.n_leaves = nl; w.Ta.n_leaves = nl;
  // gravity over bin segments (half-warp tiles) or leaf tiles; bins beyond the
  // block tiler's capacity force the leaf path
  bool use_leaf_gravity = a->gravity_mode == 1 || max_bin_count > 2048 ||
                          (a->gravity_mode == 0 && !kGravityBinsDefault);
  // SPH passes over bin segments too (fuller gas tiles); the leaf list stays the
  // reference's product and the fallback when a bin outgrows the tiler
  bool sph_bins = a->gravity_mode != 1 && max_bin_count <= 2048;
  // bin segments evaluate every row; the reference's receivers are the
  // non-ghost-only leaves, so their ghost-only rows read zero (hb/cmtree.py:318)
  bool zero_ghost = sph_bins || !use_leaf_gravity;
  bool zero_ghost_sph = zero_ghost;
  auto zero_rows = [&](double* nc, double* mo, double* hy, double* gr) -> int {
    k_zero_ghost_rows<<<grid_for(nl * 32, 256), 256, 0, st>>>(nl, w.leaf_start, w.leaf_end,
                                                               w.ghost_only, nc, mo, hy, gr);
    HB_LAUNCH_CHECK();
    return HB_OK;
  };
  int64_t n_seg = sph_bins ? nbins : nl;
  const int64_t* seg_s = w.leaf_start;
  const int64_t* seg_e = w.leaf_end;
  if (sph_bins) {
    int rcb = bin_stencil_csr(nbins, w.bin_ptr, w.leaf_start, w.leaf_end, ld.g, w.seg_s, w.seg_e,
                              w.st_ptr, w.st_src, w.st_code, st, err);
    if (rcb) return rcb;
    seg_s = w.seg_s;
    seg_e = w.seg_e;
  }
  {
    Arena s = ws;
    int rc = build_tiling(w.Tg, n_seg, seg_s, seg_e, rows, a->image_shift, a->side_length, 1,
                          w.ntg, s, st, err, a->owned_targets ? a->ghost : nullptr);
    if (rc) return rc;
    if ((a->passes & HB_PASS_GRAVITY) && use_leaf_gravity) {
      Arena s2 = ws;
      rc = build_tiling(w.Ta, nl, w.leaf_start, w.leaf_end, rows, a->image_shift,
                        a->side_length, 0, w.nta, s2, st, err);
      if (rc) return rc;
    }
  }
  EvalDev d = {};
  d.ent_ptr = w.ent_ptr; d.ent_src = w.ent_src; d.ent_code = w.ent_code;
  d.P0 = w.P0; d.P1 = w.P1; d.P2 = w.P2; d.rows = rows; d.pshift = a->image_shift;
  d.L = a->side_length; d.include_self = 1; d.write_out = 1; d.err_key = w.err_key;
  d.in_count = nullptr; d.out_int = nullptr;
  double sph_reach = 2.0 * a->h_max;
  auto setup = [&](int kid, double reach, double p0, double p1, int nchan, const Tiling& T,
                   double* out) {
    d.T = T;
    d.reach = reach;
    d.pp.p0 = (float)p0; d.pp.p1 = (float)p1;
    d.pp.inv_rs = p0 != 0.0 ? (float)(1.0 / p0) : 0.0f;
    d.pp.reach2 = (float)(reach * reach);
    d.cull_reach = (float)(reach * (1.0 + 1e-4)) + 1e-30f;
    d.nchan = nchan;
    d.out_flt = out;
    (void)kid;
  };
  int rc = HB_OK;
  int64_t tcap = w.Tg.n_tiles_cap;
  tm.mark(3);
  // geometry-derived band: FP32 r^2 error <= ~6 * 2^-24 * bin width * r; decide
  // in float64 within 64x that of a threshold (exact counts, hb/kernels.py:191,357)
  double wmax = fmax(a->width[0], fmax(a->width[1], a->width[2]));
  double rmin = fmax(fmin(a->reach, 2.0 * a->h_min), 1e-300);
  float band = (float)fmax(64.0 * 5.9604644775390625e-08 * wmax / rmin, 9.5367431640625e-07);
  SphArgs sa{};
  sa.T = &w.Tg; sa.n_tiles_dev = w.ntg;
  sa.ent_ptr = sph_bins ? w.st_ptr : w.ent_ptr;
  sa.ent_src = sph_bins ? w.st_src : w.ent_src;
  sa.ent_code = sph_bins ? w.st_code : w.ent_code;
  sa.P0 = w.P0; sa.P1 = w.P1; sa.P2 = w.P2; sa.P3 = nullptr; sa.rows = rows;
  sa.pshift = a->image_shift; sa.L = a->side_length; sa.reach = sph_reach; sa.band = band;
  sa.alpha = a->visc_alpha; sa.beta = a->visc_beta; sa.err_key = w.err_key;
  sa.ncount = a->ncount; sa.rho = w.rho_new; sa.moments = mom; sa.hydro = a->hydro;
  sa.skip_leaf = (a->ghost_density && !sph_bins) ? w.ghost_only : nullptr;
  sa.skip_tiles = a->owned_targets ? 1 : 0;
  d.skip_leaf = a->ghost_density ? w.ghost_only : nullptr;
  // 4. pass A: neighbour count + density (hb/hydro.py:223-227, 60-84), EOS (48-57)
  if (a->passes & (HB_PASS_NCOUNT | HB_PASS_DENSITY)) {
    HB_CUDA_TRY(cudaMemsetAsync(a->ncount, 0, n * sizeof(double), st));
    HB_CUDA_TRY(cudaMemsetAsync(w.rho_new, 0, n * sizeof(double), st));
    rc = pack_sph(w.Tg, w.ntg, rows, a->image_shift, a->side_length, w.P0, w.P1, w.P2, nullptr, 0, st,
                  err);
    if (rc) return rc;
    tm.kmark(2);
    rc = launch_sph(0, sa, st, err);
    tm.kmark(3);
    if (rc) return rc;
  }
  // bin gravity's preparation (segments, stencil, all-species tiling, records)
  // needs only positions and masses: it runs here, where a host-buffer step
  // would otherwise wait for the late input group (vel, internal energy)
  bool bin_gravity = (a->passes & HB_PASS_GRAVITY) && !use_leaf_gravity;
  auto gravity_args = [&]() {
    GravBinArgs gb;
    gb.n = n; gb.nbins = nbins; gb.bin_ptr = w.bin_ptr; gb.leaf_start = w.leaf_start;
    gb.leaf_end = w.leaf_end; gb.geom = ld.g; gb.rows = rows; gb.pshift = a->image_shift;
    gb.L = a->side_length; gb.r_s = a->r_s; gb.r_cut = a->r_cut; gb.eps = a->softening;
    gb.out = a->grav; gb.err_key = w.err_key; gb.overflow_host = nullptr;
    gb.ghost = a->owned_targets ? a->ghost : nullptr;
    gb.count_only = (a->passes & HB_PASS_COUNT_ONLY) != 0;
    if (sph_bins) {  // the SPH tiling's bin segments and stencil are the same arrays
      gb.pre_seg_s = w.seg_s; gb.pre_seg_e = w.seg_e; gb.pre_st_ptr = w.st_ptr;
      gb.pre_st_src = w.st_src; gb.pre_st_code = w.st_code;
    }
    return gb;
  };
  bool gravity_prepared = false;
  if (bin_gravity) {
    GravBinArgs gb = gravity_args();
    gb.phase = 1;
    Arena s = ws;
    rc = gravity_bins(gb, s, st, err);
    if (rc) return rc;
    gravity_prepared = true;
  }
  rc = gather_late();  // before pass B and the ghost alias sync read them
  if (rc) return rc;
  if (a->passes & HB_PASS_DENSITY) {
    k_density_update<<<grid_for(nl * 32, 256), 256, 0, st>>>(
        nl, w.leaf_start, w.leaf_end, a->ghost_density ? w.no_ghost : w.ghost_only, a->species,
        w.rho_new, a->density);
    if (a->ghost_src_in && a->ghost_src && !last_split) {
      k_alias_sync<<<grid_for(n, 256), 256, 0, st>>>(n, a->ghost_src, a->density);
      HB_COUNT_LAUNCH(1);
    }
    HB_LAUNCH_CHECK();
    // the EOS (P, c_s; hb/hydro.py:48-57) is evaluated where pass B's records
    // are packed, from the leaf-order density and internal energy
  }
  tm.mark(4);
  // 5. pass B: CRK moments (+ 3x3 solve, hb/hydro.py:99-150) + hydro force (hb/kernels.py:222-258)
  if (a->passes & (HB_PASS_CRK | HB_PASS_HYDRO)) {
    HB_CUDA_TRY(cudaMemsetAsync(mom, 0, n * 10 * sizeof(double), st));
    HB_CUDA_TRY(cudaMemsetAsync(a->hydro, 0, n * 5 * sizeof(double), st));
    rc = pack_sph(w.Tg, w.ntg, rows, a->image_shift, a->side_length, w.P0, w.P1, w.P2, nullptr, 1, st,
                  err, a->density, a->internal_energy, a->eos_gamma);
    if (rc) return rc;
    tm.kmark(4);
    rc = launch_sph(1, sa, st, err);
    tm.kmark(5);
    if (rc) return rc;
    if (zero_ghost) {  // before the solve: zero moments give A = 1, B = 0 as in the reference
      rc = zero_rows(a->ghost_density ? nullptr : a->ncount, mom, a->hydro, nullptr);
      if (rc) return rc;
      zero_ghost_sph = false;
    }
    // the SPH tiling lists every gas row once: tperm[0, sel_off[n_seg])
    rc = crk_solve_rows(n, mom, 10, a->species, 1e8, a->crk_A, a->crk_B, a->crk_fallback,
                        w.Tg.tperm, w.Tg.sel_off + n_seg, st, err);
    if (rc) return rc;
    // 6. optional pass C: gradA / gradB (HB_PASS_CRK_GRAD), on the solved A, B
    if ((a->passes & HB_PASS_CRK_GRAD) && a->crk_gradA && a->crk_gradB) {
      HB_CUDA_TRY(cudaMemsetAsync(a->crk_gradA, 0, n * 3 * sizeof(double), st));
      HB_CUDA_TRY(cudaMemsetAsync(a->crk_gradB, 0, n * 9 * sizeof(double), st));
      rc = pack_sph(w.Tg, w.ntg, rows, a->image_shift, a->side_length, w.P0, w.P1, w.P2,
                    nullptr, 2, st, err, a->density, a->internal_energy, a->eos_gamma);
      if (rc) return rc;
      sa.crk_A = a->crk_A; sa.crk_B = a->crk_B; sa.crk_fallback = a->crk_fallback;
      sa.gradA = a->crk_gradA; sa.gradB = a->crk_gradB;
      rc = launch_sph(2, sa, st, err);
      if (rc) return rc;
    }
  }
  if (zero_ghost_sph && !a->ghost_density && (a->passes & HB_PASS_NCOUNT)) {
    rc = zero_rows(a->ncount, nullptr, nullptr, nullptr);
    if (rc) return rc;
  }
  rc = gather_last();  // before sph_done: the density output includes the non-gas rows
  if (rc) return rc;
  // the SPH outputs are final here (ghost rows included): copies may start
  if (a->sph_done_event) HB_CUDA_TRY(cudaEventRecord((cudaEvent_t)a->sph_done_event, st));
  tm.mark(5);
  // 7. short-range gravity (hb/kernels.py:152-163): bin segments (hb_grav2.cu,
  // prepared after pass A above) unless a bin outgrows the block tiler, then
  // leaf tiles.  (Running it on a second stream concurrently with the SPH
  // chain was measured: the two throughput-bound grids time-slice the SMs --
  // whichever has dispatch priority starves the other -- so the step time did
  // not change.)
  if (bin_gravity) {
    HB_CUDA_TRY(cudaMemsetAsync(a->grav, 0, n * 3 * sizeof(double), st));
    GravBinArgs gb = gravity_args();
    gb.phase = gravity_prepared ? 2 : 0;
    gb.t0 = tm.on ? tm.kv[0] : nullptr;
    gb.t1 = tm.on ? tm.kv[1] : nullptr;
    GhostZeroCtx zc = {nl, w.leaf_start, w.leaf_end, w.ghost_only, a->grav, st};
    if (a->grav_half_event && !gb.count_only) {
      gb.split_event = (cudaEvent_t)a->grav_half_event;
      if (zero_ghost) { gb.between = zero_grav_ghost_rows; gb.between_ctx = &zc; }
    }
    Arena s = ws;
    rc = gravity_bins(gb, s, st, err);
    if (rc) return rc;
  }
  if ((a->passes & HB_PASS_GRAVITY) && !bin_gravity) {
    HB_CUDA_TRY(cudaMemsetAsync(a->grav, 0, n * 3 * sizeof(double), st));
    {
      rc = pack_records(KID_GRAVITY, w.Ta, w.nta, rows, a->image_shift, nullptr, 0,
                        a->side_length, w.P0, w.P1, w.P2, st, err);
      if (rc) return rc;
      setup(KID_GRAVITY, a->r_cut, a->r_s, a->softening * a->softening, 3, w.Ta, a->grav);
      if (a->passes & HB_PASS_COUNT_ONLY) {  // exact in-r_cut counts (see hb.h)
        EvalDev c = d;
        c.include_self = 0; c.nchan = 1; c.scale[0] = 1.0f;
        c.out_int = (int64_t*)a->grav;
        c.in_count = (unsigned long long*)w.nta + 1;
        HB_CUDA_TRY(cudaMemsetAsync(a->grav, 0, n * sizeof(int64_t), st));
        rc = launch_pairs(KID_COUNTING, true, false, c, w.Ta.n_tiles_cap, w.nta, st, err);
        if (rc) return rc;
      } else {
      GravTab gt;
      const float4* gtab = gravity_table_device(
          a->r_s, a->r_cut, a->softening, &gt,
          st, err);
      if (!gtab) return err ? err->status : HB_CUDA;
      tm.kmark(0);
      rc = launch_gravity_fast(d, gtab, gt, w.Ta.n_tiles_cap, w.nta, st, err);
      tm.kmark(1);
      if (rc) return rc;
      }
    }
  }
  tm.mark(6);
  // no split (leaf gravity runs as one launch and never records
  // grav_half_event): every row is final at the end
  if (a->grav_half_event && !bin_gravity) {
    a->grav_split_row = 0;
  }
  if (zero_ghost && (a->passes & HB_PASS_GRAVITY) && !(a->passes & HB_PASS_COUNT_ONLY)) {
    rc = zero_rows(nullptr, nullptr, nullptr, a->grav);
    if (rc) return rc;
  }
  tm.mark(7);
  if (a->status_out && !tm.on) {
    // deferred status: the error key and overflow flags land in the caller's
    // pinned words; no end-of-step sync, so the caller can queue its
    // device-to-host copies behind sph_done_event / the step stream right away
    uint64_t* so = (uint64_t*)a->status_out;
    HB_CUDA_TRY(cudaMemcpyAsync(&so[0], w.err_key, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    HB_CUDA_TRY(cudaMemcpyAsync(&so[1], w.Tg.overflow, sizeof(int), cudaMemcpyDeviceToHost, st));
    if (use_leaf_gravity)
      HB_CUDA_TRY(cudaMemcpyAsync(&so[2], w.Ta.overflow, sizeof(int), cudaMemcpyDeviceToHost, st));
    return HB_OK;
  }
  unsigned long long ek = 0;
  int ovf = 0, ovf2 = 0;
  HB_CUDA_TRY(cudaMemcpyAsync(&ek, w.err_key, sizeof(ek), cudaMemcpyDeviceToHost, st));
  HB_CUDA_TRY(cudaMemcpyAsync(&ovf, w.Tg.overflow, sizeof(int), cudaMemcpyDeviceToHost, st));
  if (use_leaf_gravity)
    HB_CUDA_TRY(cudaMemcpyAsync(&ovf2, w.Ta.overflow, sizeof(int), cudaMemcpyDeviceToHost, st));
  HB_CUDA_TRY(cudaStreamSynchronize(st));
  if (tm.on) {
    for (int i = 0; i < 7; ++i) cudaEventElapsedTime(&a->ms_phase[i], tm.ev[i], tm.ev[i + 1]);
    cudaEventElapsedTime(&a->ms_phase[7], tm.ev[0], tm.ev[7]);
    for (int i = 0; i < 4; ++i) a->ms_kernel[i] = 0.f;
    if (a->passes & HB_PASS_GRAVITY) cudaEventElapsedTime(&a->ms_kernel[0], tm.kv[0], tm.kv[1]);
    if (a->passes & (HB_PASS_NCOUNT | HB_PASS_DENSITY))
      cudaEventElapsedTime(&a->ms_kernel[1], tm.kv[2], tm.kv[3]);
    if (a->passes & (HB_PASS_CRK | HB_PASS_HYDRO))
      cudaEventElapsedTime(&a->ms_kernel[2], tm.kv[4], tm.kv[5]);
  }
  if (ovf || ovf2) return set_err(err, HB_CONTRACT, "leaf exceeds the tiling capacity (2048 members)");
  if (ek != ~0ull) return step_key_error(ek, err);
  return HB_OK;
}

}  // namespace hb

using namespace hb;

extern "C" size_t hb_force_step_workspace_passes(int64_t n, const int64_t nb[3],
                                                 int64_t max_leaf_size, int64_t list_capacity,
                                                 int32_t passes) {
  HbStepArgs a = {};
  a.passes = passes;
  a.n = n;
  for (int d = 0; d < 3; ++d) a.nb[d] = nb[d];
  a.max_leaf_size = max_leaf_size;
  a.list_capacity = list_capacity;
  Arena ws;
  ws.dry = true;
  force_step(&a, ws, nullptr, nullptr);
  return ws.used + 4096;
}

extern "C" size_t hb_force_step_workspace(int64_t n, const int64_t nb[3], int64_t max_leaf_size,
                                          int64_t list_capacity) {
  return hb_force_step_workspace_passes(n, nb, max_leaf_size, list_capacity, HB_PASS_ALL);
}

extern "C" int hb_force_step_check(const void* status, HbError* err) {
  if (err) *err = HbError{};
  const uint64_t* so = (const uint64_t*)status;
  if ((uint32_t)so[1] || (uint32_t)so[2])
    return set_err(err, HB_CONTRACT, "leaf exceeds the tiling capacity (2048 members)");
  uint64_t ek = so[0];
  if (ek != ~0ull) return step_key_error(ek, err);
  return HB_OK;
}

extern "C" int hb_force_step(HbStepArgs* a, void* wsp, size_t ws_bytes, void* stream, HbError* err) {
  if (err) *err = HbError{};
  Arena ws;
  ws.base = (char*)wsp; ws.cap = ws_bytes;
  return force_step(a, ws, (cudaStream_t)stream, err);
}
