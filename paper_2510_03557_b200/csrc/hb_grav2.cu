// hb_grav2.cu -- short-range gravity over chaining-mesh BINS (the resident
// step's gravity driver; the pair kernel k_gravity is in hb_pairs.cu).
//
// Segments are bins, not leaves: a bin (~2x the leaf size in near-uniform
// boxes) splits into 32-particle k-d tiles with far less rounding waste, and
// the candidate sources are the 27 stencil bins (with periodic shifts and
// duplicate suppression exactly as the list sweep, hb/cmtree.py:218-245) -- a
// superset of the leaf-pair list; pairs beyond r_cut contribute nothing
// (hb/kernels.py:152-163).
// (Round 2 removed the half-warp variant k_gravity2 -- two 16-target tiles per
// warp with the r/t-indexed table -- and the within-tile k-d reordering: both
// measured slower than k_gravity on 32-target tiles with the soft table,
// including for dark-matter-only sets: 245.6 vs 187.6 ms at 512^3.)
#include "hb_internal.cuh"

namespace hb {

constexpr int kG2Warps = 8;
// rows of bin b: [leaf_start[first leaf], leaf_end[last leaf]) (leaves of a bin are contiguous)
__global__ void k_bin_segments(int64_t nbins, const int64_t* bin_ptr, const int64_t* leaf_start,
                               const int64_t* leaf_end, int64_t* seg_start, int64_t* seg_end) {
  int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nbins) return;
  int64_t l0 = bin_ptr[b], l1 = bin_ptr[b + 1];
  int64_t s = l0 < l1 ? leaf_start[l0] : 0;
  seg_start[b] = s;
  seg_end[b] = l0 < l1 ? leaf_end[l1 - 1] : s;
}

// 27-stencil of every bin: neighbour bin (or -1: off-mesh / duplicate) and shift code
__global__ void k_bin_stencil(int64_t nbins, ListGeom g, int32_t* src, int32_t* code) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nbins * 27) return;
  int64_t b = t / 27;
  int o = (int)(t % 27);
  int64_t bz = b % g.nb[2], by = (b / g.nb[2]) % g.nb[1], bx = b / (g.nb[1] * g.nb[2]);
  auto cell = [&](int oo, int64_t& flat, int& cd) -> bool {
    int64_t c[3] = {bx + oo / 9 - 1, by + (oo / 3) % 3 - 1, bz + oo % 3 - 1};
    int s[3] = {0, 0, 0};
    for (int d = 0; d < 3; ++d) {
      if (g.periodic[d]) {
        if (c[d] < 0) { c[d] += g.nb[d]; s[d] = -1; }
        else if (c[d] >= g.nb[d]) { c[d] -= g.nb[d]; s[d] = 1; }
      } else if (c[d] < 0 || c[d] >= g.nb[d]) {
        return false;
      }
    }
    flat = (c[0] * g.nb[1] + c[1]) * g.nb[2] + c[2];
    cd = (s[0] + 1) * 9 + (s[1] + 1) * 3 + (s[2] + 1);
    return true;
  };
  int64_t flat;
  int cd;
  bool ok = cell(o, flat, cd);
  // duplicates (the same cell and shift reached twice) need an axis with
  // fewer than 3 bins; otherwise the 27 offsets are distinct
  bool dup_possible = g.nb[0] < 3 || g.nb[1] < 3 || g.nb[2] < 3;
  for (int o2 = 0; o2 < o && ok && dup_possible; ++o2) {
    int64_t f2;
    int c2;
    if (cell(o2, f2, c2) && f2 == flat && c2 == cd) ok = false;
  }
  src[t] = ok ? (int32_t)flat : -1;
  code[t] = ok ? cd : 13;
}

__global__ void k_stride_ptr(int64_t n, int64_t stride, int64_t* ptr) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= n) ptr[i] = i * stride;
}

int bin_stencil_csr(int64_t nbins, const int64_t* bin_ptr, const int64_t* leaf_start,
                    const int64_t* leaf_end, const ListGeom& g, int64_t* seg_s, int64_t* seg_e,
                    int64_t* st_ptr, int32_t* st_src, int32_t* st_code, cudaStream_t st,
                    HbError* err) {
  k_bin_segments<<<grid_for(nbins, 256), 256, 0, st>>>(nbins, bin_ptr, leaf_start, leaf_end,
                                                       seg_s, seg_e);
  HB_LAUNCH_CHECK();
  k_bin_stencil<<<grid_for(nbins * 27, 256), 256, 0, st>>>(nbins, g, st_src, st_code);
  HB_LAUNCH_CHECK();
  k_stride_ptr<<<grid_for(nbins + 1, 256), 256, 0, st>>>(nbins, 27, st_ptr);
  HB_LAUNCH_CHECK();
  return HB_OK;
}

// k_gravity (hb_pairs.cu) on 32-target bin tiles with the 27-bin stencil as its
// entry list (one broadcast stage read per pair)
int gravity_bins(const GravBinArgs& g, Arena& ws, cudaStream_t st, HbError* err) {
  int64_t nbins = g.nbins;
  Tiling T;
  carve_tiling(ws, g.n, nbins, T, 32, 0);
  int64_t* st_ptr = ws.take<int64_t>(nbins + 1);
  int64_t* seg_s = ws.take<int64_t>(nbins + 1);
  int64_t* seg_e = ws.take<int64_t>(nbins + 1);
  int32_t* st_src = ws.take<int32_t>(nbins * 27 + 1);
  int32_t* st_code = ws.take<int32_t>(nbins * 27 + 1);
  int64_t* ntd = ws.take<int64_t>(2);
  float4* P0 = ws.take<float4>(g.n + 1);
  unsigned long long* ctr = ws.take<unsigned long long>(2);  // persistent-grid tile counters
  if (ws.dry) {
    Arena s = ws;
    build_tiling(T, nbins, nullptr, nullptr, Rows{}, nullptr, 0.0, 0, nullptr, s, st, err);
    ws.used = s.used;
    return HB_OK;
  }
  if (!ws.ok()) return set_err(err, HB_CONTRACT, "workspace too small (gravity bins)");
  int rc = HB_OK;
  bool reuse = g.pre_seg_s && g.pre_seg_e && g.pre_st_ptr && g.pre_st_src && g.pre_st_code;
  const int64_t* segs = reuse ? g.pre_seg_s : seg_s;
  const int64_t* sege = reuse ? g.pre_seg_e : seg_e;
  const int64_t* sptr = reuse ? g.pre_st_ptr : st_ptr;
  const int32_t* ssrc = reuse ? g.pre_st_src : st_src;
  const int32_t* scode = reuse ? g.pre_st_code : st_code;
  if (g.phase != 2) {
    if (!reuse) {
      k_bin_segments<<<grid_for(nbins, 256), 256, 0, st>>>(nbins, g.bin_ptr, g.leaf_start,
                                                           g.leaf_end, seg_s, seg_e);
      HB_LAUNCH_CHECK();
      k_bin_stencil<<<grid_for(nbins * 27, 256), 256, 0, st>>>(nbins, g.geom, st_src, st_code);
      HB_LAUNCH_CHECK();
    }
    {
      Arena s = ws;
      rc = build_tiling(T, nbins, segs, sege, g.rows, g.pshift, g.L, 0, ntd, s, st, err,
                        g.ghost);
      if (rc) return rc;
    }
    rc = pack_records(KID_GRAVITY, T, ntd, g.rows, g.pshift, nullptr, 0, g.L, P0, nullptr,
                      nullptr, st, err);
    if (rc) return rc;
  }
  GravTab gt;
  const float4* tab = gravity_table_device(g.r_s, g.r_cut, g.eps, &gt, st, err);
  if (!tab) return err ? err->status : HB_CUDA;
  if (g.phase != 2) {
    if (!reuse) {
      k_stride_ptr<<<grid_for(nbins + 1, 256), 256, 0, st>>>(nbins, 27, st_ptr);
      HB_LAUNCH_CHECK();
    }
  }
  if (g.phase == 1) return HB_OK;
  if (g.count_only) {  // k_eval<KID_COUNTING>, float64 band re-check, no self pair
    EvalDev e = {};
    e.T = T; e.ent_ptr = sptr; e.ent_src = ssrc; e.ent_code = scode; e.P0 = P0;
    e.rows = g.rows; e.pshift = g.pshift;
    e.L = g.L; e.reach = g.r_cut;
    e.pp.reach2 = (float)(g.r_cut * g.r_cut);
    e.cull_reach = (float)(g.r_cut * (1.0 + 1e-4)) + 1e-30f;
    e.include_self = 0; e.nchan = 1; e.scale[0] = 1.0f;
    e.out_int = (int64_t*)g.out; e.write_out = 1; e.err_key = g.err_key;
    e.in_count = (unsigned long long*)ntd + 1;  // unused (no counted-entry flags)
    e.skip_tiles = g.ghost ? 1 : 0;
    HB_CUDA_TRY(cudaMemsetAsync(g.out, 0, g.n * sizeof(int64_t), st));
    return launch_pairs(KID_COUNTING, true, false, e, T.n_tiles_cap, ntd, st, err);
  }
  {
    EvalDev e = {};
    e.T = T; e.ent_ptr = sptr; e.ent_src = ssrc; e.ent_code = scode; e.P0 = P0;
    e.L = g.L; e.reach = g.r_cut;
    e.pp.p0 = (float)g.r_s; e.pp.p1 = (float)(g.eps * g.eps);
    e.cull_reach = (float)(g.r_cut * (1.0 + 1e-4)) + 1e-30f;
    e.nchan = 3; e.out_flt = g.out; e.write_out = 1; e.err_key = g.err_key;
    e.skip_leaf = nullptr;
    e.skip_tiles = g.ghost ? 1 : 0;
    if (g.t0) HB_CUDA_TRY(cudaEventRecord(g.t0, st));
    int rc2;
    if (g.split_event) {  // tiles of bins < grav_split_bin, then the rest (tile_ptr is per bin)
      const int64_t* mid = T.tile_ptr + grav_split_bin(nbins);
      rc2 = launch_gravity_fast(e, tab, gt, T.n_tiles_cap, mid, st, err, nullptr, ctr);
      if (rc2) return rc2;
      if (g.between) {
        rc2 = g.between(g.between_ctx);
        if (rc2) return rc2;
      }
      HB_CUDA_TRY(cudaEventRecord(g.split_event, st));
      rc2 = launch_gravity_fast(e, tab, gt, T.n_tiles_cap, ntd, st, err, mid, ctr + 1);
    } else {
      rc2 = launch_gravity_fast(e, tab, gt, T.n_tiles_cap, ntd, st, err, nullptr, ctr);
    }
    if (g.t1) HB_CUDA_TRY(cudaEventRecord(g.t1, st));
    return rc2;
  }
}

}  // namespace hb
