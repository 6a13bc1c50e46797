// hb_grav2.cu -- short-range gravity over chaining-mesh BINS with half-warp tiles.
//
// Same physics and S(t) table as k_gravity (hb_pairs.cu; hb/kernels.py:152-163,
// S(x) hb/kernels.py:96-99).  Differences, both to cut wasted lane-pair slots:
//  * segments are bins, not leaves: a bin (~2x the leaf size in near-uniform
//    boxes) splits into tiles with far less rounding waste, and the candidate
//    sources are the 27 stencil bins (with periodic shifts and duplicate
//    suppression exactly as the list sweep, hb/cmtree.py:218-245) -- a superset
//    of the leaf-pair list; pairs beyond r_cut contribute nothing;
//  * a warp owns TWO 16-target tiles of one bin (lanes 0-15, 16-31).  Every
//    source is culled against each half's box and staged into that half's list;
//    the flush reads stage[q][half] -- two addresses 16 B apart, one shared-
//    memory wavefront -- so each half only evaluates sources near its own box.
#include "hb_internal.cuh"

namespace hb {

constexpr int kG2Warps = 8;
// within-tile k-d levels for the bin-gravity tiles (2: 4 groups of <= 8 lanes).
// It only served the table gather's bank conflicts; with the conflict-free
// 8-copy table (hb_pairs.cu) k_gravity runs the same without it (10.036 ms
// both at c2) and the step saves the 0.21 ms pass, so the default is 0.
// HB_GRAV_TILE_LEVELS overrides for A/B measurement.
static int tile_order_levels() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HB_GRAV_TILE_LEVELS");
    v = e ? atoi(e) : 0;
  }
  return v;
}
constexpr int kG2Stage = 96;

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
  for (int o2 = 0; o2 < o && ok; ++o2) {
    int64_t f2;
    int c2;
    if (cell(o2, f2, c2) && f2 == flat && c2 == cd) ok = false;
  }
  src[t] = ok ? (int32_t)flat : -1;
  code[t] = ok ? cd : 13;
}

struct G2Dev {
  Tiling T;                 // bin segments, tile_max 16, even tile counts
  const int32_t* st_src;    // (nbins*27)
  const int32_t* st_code;
  const float4* P0;         // (x, y, z, m) bin frame
  double L;
  float cull_reach, eps2, tab_scale;
  int tab_last;
  double* out;              // (n,3) m_i a_i
  unsigned long long* err_key;
};

template <bool TVAR>
__global__ void __launch_bounds__(kG2Warps * 32)
k_gravity2(G2Dev a, const float4* __restrict__ table, const int64_t* n_tiles_dev) {
  __shared__ float4 s_tab[kGravTableRMax];
  __shared__ float4 s_stage[kG2Warps][kG2Stage][2];
  for (int k = threadIdx.x; k <= a.tab_last; k += blockDim.x) s_tab[k] = table[k];
  __syncthreads();
  int wid = threadIdx.x >> 5, lane = threadIdx.x & 31, half = lane >> 4, hl = lane & 15;
  int64_t tp = (int64_t)blockIdx.x * kG2Warps + wid;
  int64_t ntiles = *n_tiles_dev;
  if (2 * tp >= ntiles) return;
  const Tiling& T = a.T;
  int64_t t0 = 2 * tp, tme = t0 + half;
  int A = T.tile_leaf[t0];
  int n_t = T.tile_n[tme];
  bool live = hl < n_t;
  int k_i = T.tile_start[tme] + (live ? hl : 0);
  float4 ti = n_t > 0 ? a.P0[k_i] : make_float4(0.f, 0.f, 0.f, 0.f);
  float4 lo0 = T.tile_lo[t0], hi0 = T.tile_hi[t0], lo1 = T.tile_lo[t0 + 1], hi1 = T.tile_hi[t0 + 1];
  float4 ulo = make_float4(fminf(lo0.x, lo1.x), fminf(lo0.y, lo1.y), fminf(lo0.z, lo1.z), 0.f);
  float4 uhi = make_float4(fmaxf(hi0.x, hi1.x), fmaxf(hi0.y, hi1.y), fmaxf(hi0.z, hi1.z), 0.f);
  float R2 = a.cull_reach * a.cull_reach;
  float ax = 0.f, ay = 0.f, az = 0.f;
  double oA[3] = {T.origin[3 * A], T.origin[3 * A + 1], T.origin[3 * A + 2]};
  float4(*stage)[2] = s_stage[wid];
  int c0 = 0, c1 = 0;
  auto flush = [&]() {
    int cm = max(c0, c1);
    // pad the shorter half with massless sources (contribute exactly 0)
    for (int q = (half ? c1 : c0) + hl; q < cm; q += 16) stage[q][half] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncwarp();
#pragma unroll 4
    for (int q = 0; q < cm; ++q) {
      float4 s = stage[q][half];
      float dx = ti.x - s.x, dy = ti.y - s.y, dz = ti.z - s.z;
      float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
      float soft = r2 + a.eps2;
      float ri = rsqrt_ftz(soft);
      float rr = TVAR ? soft * ri : r2 * rsqrt_ftz(fmaxf(r2, 1e-30f));
      float fm = fmaf(rr, a.tab_scale, 12582912.0f);
      int k = min(__float_as_int(fm) - 0x4B400000, a.tab_last);
      float u = fmaf(rr, a.tab_scale, 12582912.0f - fm);
      float4 c = s_tab[k];
      float S = fmaf(fmaf(fmaf(c.w, u, c.z), u, c.y), u, c.x);
      float w = (S * (ri * ri)) * (ri * s.w);
      ax = fmaf(w, dx, ax);
      ay = fmaf(w, dy, ay);
      az = fmaf(w, dz, az);
    }
    __syncwarp();
    c0 = 0;
    c1 = 0;
  };
  for (int o = 0; o < 27; ++o) {
    int B = a.st_src[27 * (int64_t)A + o];
    if (B < 0) continue;
    int code = a.st_code[27 * (int64_t)A + o];
    int sh0 = code / 9 - 1, sh1 = (code / 3) % 3 - 1, sh2 = code % 3 - 1;
    float D0 = (float)((oA[0] - T.origin[3 * B]) - (double)sh0 * a.L);
    float D1 = (float)((oA[1] - T.origin[3 * B + 1]) - (double)sh1 * a.L);
    float D2 = (float)((oA[2] - T.origin[3 * B + 2]) - (double)sh2 * a.L);
    int64_t u0 = T.tile_ptr[B], u1 = T.tile_ptr[B + 1];  // even count: tile pairs
    for (int64_t ub = u0; ub < u1; ub += 64) {
      int64_t up = ub + 2 * lane;  // lane tests source tile pair (up, up+1)
      bool pass = false;
      if (up < u1) {
        float4 la = T.tile_lo[up], ha = T.tile_hi[up], lb = T.tile_lo[up + 1], hb = T.tile_hi[up + 1];
        float lx = fminf(la.x, lb.x) - D0, ly = fminf(la.y, lb.y) - D1, lz = fminf(la.z, lb.z) - D2;
        float hx = fmaxf(ha.x, hb.x) - D0, hy = fmaxf(ha.y, hb.y) - D1, hz = fmaxf(ha.z, hb.z) - D2;
        float gx = fmaxf(fmaxf(lx - uhi.x, ulo.x - hx), 0.0f);
        float gy = fmaxf(fmaxf(ly - uhi.y, ulo.y - hy), 0.0f);
        float gz = fmaxf(fmaxf(lz - uhi.z, ulo.z - hz), 0.0f);
        pass = fmaf(gz, gz, fmaf(gy, gy, gx * gx)) <= R2;
      }
      unsigned tm = __ballot_sync(0xffffffffu, pass);
      while (tm) {
        int j = __ffs(tm) - 1;
        tm &= tm - 1;
        int64_t uu = ub + 2 * j + half;  // lanes 0-15: first tile of the pair, 16-31: second
        int n_u = T.tile_n[uu];
        bool ok0 = false, ok1 = false;
        float4 sj = make_float4(0.f, 0.f, 0.f, 0.f);
        if (hl < n_u) {
          sj = a.P0[T.tile_start[uu] + hl];
          sj.x -= D0; sj.y -= D1; sj.z -= D2;
          ok0 = box_gap2(sj.x, sj.y, sj.z, lo0, hi0) <= R2;
          ok1 = box_gap2(sj.x, sj.y, sj.z, lo1, hi1) <= R2;
        }
        unsigned m0 = __ballot_sync(0xffffffffu, ok0), m1 = __ballot_sync(0xffffffffu, ok1);
        if (max(c0, c1) + 32 > kG2Stage) flush();
        unsigned lt = lanemask_lt();
        if (ok0) stage[c0 + __popc(m0 & lt)][0] = sj;
        if (ok1) stage[c1 + __popc(m1 & lt)][1] = sj;
        c0 += __popc(m0);
        c1 += __popc(m1);
      }
    }
  }
  flush();
  bool bad = !(isfinite(ax) && isfinite(ay) && isfinite(az));
  if (__ballot_sync(0xffffffffu, live && bad)) {
    if (lane == 0) atomicMin(a.err_key, (unsigned long long)(A * 4 + 1));
    return;
  }
  if (live) {
    int64_t row = T.tperm[k_i];
    double mi = -(double)ti.w;
    a.out[row * 3 + 0] += mi * (double)ax;
    a.out[row * 3 + 1] += mi * (double)ay;
    a.out[row * 3 + 2] += mi * (double)az;
  }
}

// Warp per tile: reorder the tile's members (P0 and tperm together) into a
// `levels`-deep median k-d order (each segment split on its longest axis,
// stable by position; first part (sz + 1) / 2).  With 2 levels every 8-lane
// phase of a warp holds a compact group of <= 8 targets, so the GT_SOFT rows
// one phase gathers for a source are closer together.  Measured: k_gravity
// 10.47 -> 10.25 ms at c2 (bank conflicts -4%: even a compact group spans
// several octaves of soft for a near source).
// Internal order only: it changes FP32 summation order, not the pairs.
constexpr int kTOWarps = 8;
__global__ void __launch_bounds__(kTOWarps * 32)
k_tile_order(const int64_t* n_tiles_dev, Tiling T, float4* P0, int levels) {
  __shared__ float4 s_p[kTOWarps][32];
  __shared__ int s_r[kTOWarps][32];
  int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t t = (int64_t)blockIdx.x * kTOWarps + wid;
  if (t >= *n_tiles_dev) return;
  int n = T.tile_n[t];
  if (n <= 8) return;
  int64_t s0 = T.tile_start[t];
  bool live = lane < n;
  float4* sp = s_p[wid];
  int* sr = s_r[wid];
  if (live) {
    sp[lane] = P0[s0 + lane];
    sr[lane] = T.tperm[s0 + lane];
  }
  __syncwarp();
  for (int lvl = 0; lvl < levels; ++lvl) {
    float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
    int r = 0, np = lane;
    if (live) {
      int off = 0, sz = n;
      for (int l = 0; l < lvl; ++l) {
        int h = (sz + 1) >> 1;
        if (lane - off >= h) { off += h; sz -= h; } else { sz = h; }
      }
      float lx = INFINITY, ly = INFINITY, lz = INFINITY;
      float hx = -INFINITY, hy = -INFINITY, hz = -INFINITY;
      for (int j = off; j < off + sz; ++j) {
        float4 q = sp[j];
        lx = fminf(lx, q.x); ly = fminf(ly, q.y); lz = fminf(lz, q.z);
        hx = fmaxf(hx, q.x); hy = fmaxf(hy, q.y); hz = fmaxf(hz, q.z);
      }
      float ex = hx - lx, ey = hy - ly, ez = hz - lz;
      int ax = (ex >= ey && ex >= ez) ? 0 : (ey >= ez ? 1 : 2);
      p = sp[lane];
      r = sr[lane];
      unsigned key = sortable_key(ax == 0 ? p.x : ax == 1 ? p.y : p.z);
      int rank = 0;
      for (int j = off; j < off + sz; ++j) {
        float4 q = sp[j];
        unsigned kj = sortable_key(ax == 0 ? q.x : ax == 1 ? q.y : q.z);
        rank += (kj < key || (kj == key && j < lane)) ? 1 : 0;
      }
      np = off + rank;
    }
    __syncwarp();
    if (live) { sp[np] = p; sr[np] = r; }
    __syncwarp();
  }
  if (live) {
    P0[s0 + lane] = sp[lane];
    T.tperm[s0 + lane] = sr[lane];
  }
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

// half_warp = true: k_gravity2 (two 16-target tiles per warp, per-half stages);
// false: k_gravity (hb_pairs.cu) on 32-target bin tiles with the 27-bin stencil
// as its entry list (one broadcast stage read per pair)
int gravity_bins(const GravBinArgs& g, Arena& ws, cudaStream_t st, HbError* err) {
  int64_t nbins = g.nbins;
  Tiling T;
  carve_tiling(ws, g.n, nbins, T, g.half_warp ? 16 : 32, g.half_warp ? 1 : 0);
  int64_t* st_ptr = ws.take<int64_t>(nbins + 1);
  int64_t* seg_s = ws.take<int64_t>(nbins + 1);
  int64_t* seg_e = ws.take<int64_t>(nbins + 1);
  int32_t* st_src = ws.take<int32_t>(nbins * 27 + 1);
  int32_t* st_code = ws.take<int32_t>(nbins * 27 + 1);
  int64_t* ntd = ws.take<int64_t>(2);
  float4* P0 = ws.take<float4>(g.n + 1);
  if (ws.dry) {
    Arena s = ws;
    build_tiling(T, nbins, nullptr, nullptr, nullptr, nullptr, 0.0, 0, nullptr, s, st, err);
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
      rc = build_tiling(T, nbins, segs, sege, g.state, g.pshift, g.L, 0, ntd, s, st, err,
                        g.ghost);
      if (rc) return rc;
    }
    rc = pack_records(KID_GRAVITY, T, ntd, g.state, g.pshift, nullptr, 0, g.L, P0, nullptr,
                      nullptr, st, err);
    if (rc) return rc;
  }
  GravTab gt;
  // k_gravity2 only has the r / t tables
  int kind = g.half_warp ? (g.eps <= 0.05 * g.r_s ? GT_T : GT_R) : g.table_kind;
  const float4* tab = gravity_table_device(g.r_s, g.r_cut, g.eps, kind, &gt, st, err);
  if (!tab) return err ? err->status : HB_CUDA;
  if (!g.half_warp && g.phase != 2) {
    if (tile_order_levels() > 0) {
      k_tile_order<<<grid_for(T.n_tiles_cap, kTOWarps), kTOWarps * 32, 0, st>>>(
          ntd, T, P0, tile_order_levels());
      HB_LAUNCH_CHECK();
    }
    if (!reuse) {
      k_stride_ptr<<<grid_for(nbins + 1, 256), 256, 0, st>>>(nbins, 27, st_ptr);
      HB_LAUNCH_CHECK();
    }
  }
  if (g.phase == 1) return HB_OK;
  if (g.count_only) {  // k_eval<KID_COUNTING>, float64 band re-check, no self pair
    EvalDev e = {};
    e.T = T; e.ent_ptr = sptr; e.ent_src = ssrc; e.ent_code = scode; e.P0 = P0;
    e.state = g.state; e.pshift = g.pshift;
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
  if (!g.half_warp) {
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
    if (g.split_event) {  // tiles of bins < nbins/2, then the rest (tile_ptr is per bin)
      const int64_t* mid = T.tile_ptr + grav_split_bin(nbins);
      rc2 = launch_gravity_fast(e, tab, gt, T.n_tiles_cap, mid, st, err);
      if (rc2) return rc2;
      if (g.between) {
        rc2 = g.between(g.between_ctx);
        if (rc2) return rc2;
      }
      HB_CUDA_TRY(cudaEventRecord(g.split_event, st));
      rc2 = launch_gravity_fast(e, tab, gt, T.n_tiles_cap, ntd, st, err, mid);
    } else {
      rc2 = launch_gravity_fast(e, tab, gt, T.n_tiles_cap, ntd, st, err);
    }
    if (g.t1) HB_CUDA_TRY(cudaEventRecord(g.t1, st));
    return rc2;
  }
  G2Dev d;
  d.T = T; d.st_src = ssrc; d.st_code = scode; d.P0 = P0; d.L = g.L;
  d.cull_reach = (float)(g.r_cut * (1.0 + 1e-4)) + 1e-30f;
  d.eps2 = (float)(g.eps * g.eps);
  d.tab_scale = gt.scale; d.tab_last = (int)gt.last;
  d.out = g.out; d.err_key = g.err_key;
  unsigned grid = grid_for((T.n_tiles_cap + 1) / 2, kG2Warps);
  if (g.t0) HB_CUDA_TRY(cudaEventRecord(g.t0, st));
  if (kind == GT_T) k_gravity2<true><<<grid, kG2Warps * 32, 0, st>>>(d, tab, ntd);
  else k_gravity2<false><<<grid, kG2Warps * 32, 0, st>>>(d, tab, ntd);
  HB_LAUNCH_CHECK();
  if (g.t1) HB_CUDA_TRY(cudaEventRecord(g.t1, st));
  if (g.overflow_host) {
    int ovf = 0;
    HB_CUDA_TRY(cudaMemcpyAsync(&ovf, T.overflow, sizeof(int), cudaMemcpyDeviceToHost, st));
    HB_CUDA_TRY(cudaStreamSynchronize(st));
    *g.overflow_host = ovf;
  }
  return HB_OK;
}

}  // namespace hb
