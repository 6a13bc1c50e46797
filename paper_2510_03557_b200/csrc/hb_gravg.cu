// hb_gravg.cu -- grouped-target short-range gravity (the resident step's
// gravity pair kernel; the one-list k_gravity in hb_pairs.cu is its A/B twin).
//
// Same pair function, table and source culling as k_gravity (hb_pairs.cu: the
// erfc-split S(r / r_s) (r^2 + eps^2)^-3/2 of hb/kernels.py:152-163 from a
// cubic-per-interval table in the float bits of soft), but the warp's 32
// targets are split into G spatially compact groups of 32 / G lanes and every
// group gets its own source list:
//
// * a one-list warp evaluates every staged source against all 32 targets, and
//   the staged set is the target tile's box (+) the r_cut ball: for a 32-particle
//   tile (a 2.5 d cube at r_cut = 5 d) 1324 d^3 of sources, 40% of them in
//   support;
// * with G = 4 groups (two median splits of the tile: 1.26 x 1.26 x 2.5 d boxes)
//   a group's list is its box (+) the ball, 1003 d^3; a warp step reads one
//   source per group (G distinct 16-B words in one shared-memory wavefront:
//   the lists sit at offsets that differ mod 8 float4s, so no bank conflict),
//   so a tile takes ~max over groups of the list length steps instead of the
//   union's -- ~24% fewer lane-pair slots for the same per-slot cost
//   (4 table wavefronts + 1 source wavefront + 18 instructions).
//
// Lists are drained in steps of 8 sources (the 8-source pipelined table
// gather of k_gravity) when an append could overflow one of them: min over
// groups of the list lengths, rounded down to 8, or the forced amount rounded
// up; lists shorter than the drained count are padded with a mass-0 source far
// away (soft ~ 3e30: the zero table row, an exact 0 contribution); the rest
// moves to the list's front.  Deterministic: the order of every target's sum
// is fixed by the tile, entry and list order.
#include <mutex>

#include "hb_internal.cuh"

namespace hb {

template <int G>
struct GravGroups {
  static constexpr int LPG = 32 / G;  // lanes per group
  // list capacity in float4s, == 8 / G (mod 8): the G list heads then fall in
  // distinct 16-B bank groups at every step
  static constexpr int CAP = G == 2 ? 92 : (G == 4 ? 58 : 41);
  // entries held between drains: a final drain rounds up to 8 and stays <= CAP
  static constexpr int USE = CAP - 7;
  static constexpr int PER_WARP = G * CAP + 2 * G;  // lists + group boxes
};

__device__ __forceinline__ unsigned and_or_g(unsigned a, unsigned b, unsigned c) {
  unsigned d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// n (a multiple of 8) steps over the lane's group list src[0, n): the k_gravity
// batch body (FP32x2 soft / in-interval variable / accumulation, 8 table rows
// requested before the first is used)
template <int JB, int REP>
__device__ __forceinline__ void grav_steps(const float4* src, int n, float4 ti, float2 eps2x2,
                                           const float4* s_tab, const GravTab& gt, float2& rx,
                                           float2& ry, float2& rz) {
  constexpr int B = 8;
  const unsigned lowmask = (1u << (23 - JB)) - 1u, one_bits = 0x3F800000u;
  for (int q0 = 0; q0 < n; q0 += B) {
    float2 bx[B / 2], by[B / 2], bz[B / 2], bu[B / 2];
    float bm[B];
    float4 bc[B];
#pragma unroll
    for (int p = 0; p < B / 2; ++p) {
      float4 s0 = src[q0 + 2 * p], s1 = src[q0 + 2 * p + 1];
      bx[p] = make_float2(ti.x - s0.x, ti.x - s1.x);
      by[p] = make_float2(ti.y - s0.y, ti.y - s1.y);
      bz[p] = make_float2(ti.z - s0.z, ti.z - s1.z);
      bm[2 * p] = s0.w; bm[2 * p + 1] = s1.w;
      float2 soft = __ffma2_rn(bz[p], bz[p], __ffma2_rn(by[p], by[p], __ffma2_rn(bx[p], bx[p], eps2x2)));
      unsigned b0 = __float_as_uint(soft.x), b1 = __float_as_uint(soft.y);
      unsigned k0 = min((b0 >> (23 - JB)) - gt.base, gt.last);
      unsigned k1 = min((b1 >> (23 - JB)) - gt.base, gt.last);
      float2 um = make_float2(__uint_as_float(and_or_g(b0, lowmask, one_bits)),
                              __uint_as_float(and_or_g(b1, lowmask, one_bits)));
      bu[p] = __fadd2_rn(um, make_float2(-1.0f, -1.0f));
      bc[2 * p] = s_tab[k0 * REP];
      bc[2 * p + 1] = s_tab[k1 * REP];
    }
    float2 fx = make_float2(0.0f, 0.0f), fy = fx, fz = fx;
#pragma unroll
    for (int p = 0; p < B / 2; ++p) {
      float4 c0 = bc[2 * p], c1 = bc[2 * p + 1];
      float u0 = bu[p].x, u1 = bu[p].y;
      float2 w = make_float2(fmaf(fmaf(fmaf(c0.w, u0, c0.z), u0, c0.y), u0, c0.x) * bm[2 * p],
                             fmaf(fmaf(fmaf(c1.w, u1, c1.z), u1, c1.y), u1, c1.x) * bm[2 * p + 1]);
      fx = __ffma2_rn(w, bx[p], fx);
      fy = __ffma2_rn(w, by[p], fy);
      fz = __ffma2_rn(w, bz[p], fz);
    }
    rx = __fadd2_rn(rx, fx); ry = __fadd2_rn(ry, fy); rz = __fadd2_rn(rz, fz);
  }
}

template <int JB, int REP, int G>
__device__ __forceinline__ void grav_tile_grp(const EvalDev& a, const float4* s_tab,
                                              const GravTab& gt, float4* ws, int64_t t,
                                              int lane) {
  using GG = GravGroups<G>;
  constexpr int LPG = GG::LPG, CAP = GG::CAP, USE = GG::USE;
  const unsigned FULL = 0xffffffffu;
  const Tiling& T = a.T;
  int A = T.tile_leaf[t];
  if (a.skip_leaf && a.skip_leaf[A]) return;
  if (a.skip_tiles && T.tile_skip[t]) return;
  int64_t e0 = a.ent_ptr[A], e1 = a.ent_ptr[A + 1];
  if (e0 == e1) return;
  int n_t = T.tile_n[t];
  int live = lane < n_t;
  int k_i = T.tile_start[t] + (live ? lane : 0);
  float4 ti = a.P0[k_i];
  float4 tlo = T.tile_lo[t], thi = T.tile_hi[t];
  float4* glo = ws + G * CAP;
  float4* ghi = glo + G;

  // ---- targets into G groups: log2(G) median splits along the longest axis
  // of each segment's live box (rank by coordinate, ties by lane), targets
  // moved through shared memory so that lane == position after each level
#pragma unroll
  for (int S = 32; S > LPG; S >>= 1) {
    float lx = live ? ti.x : INFINITY, ly = live ? ti.y : INFINITY, lz = live ? ti.z : INFINITY;
    float hx = live ? ti.x : -INFINITY, hy = live ? ti.y : -INFINITY, hz = live ? ti.z : -INFINITY;
#pragma unroll
    for (int o = S / 2; o; o >>= 1) {
      lx = fminf(lx, __shfl_xor_sync(FULL, lx, o)); hx = fmaxf(hx, __shfl_xor_sync(FULL, hx, o));
      ly = fminf(ly, __shfl_xor_sync(FULL, ly, o)); hy = fmaxf(hy, __shfl_xor_sync(FULL, hy, o));
      lz = fminf(lz, __shfl_xor_sync(FULL, lz, o)); hz = fmaxf(hz, __shfl_xor_sync(FULL, hz, o));
    }
    float ex = hx - lx, ey = hy - ly, ez = hz - lz;
    float key = (ex >= ey && ex >= ez) ? ti.x : (ey >= ez ? ti.y : ti.z);
    if (!live) key = INFINITY;
    int seg0 = lane & ~(S - 1);
    int r = 0;
#pragma unroll
    for (int k = 0; k < S; ++k) {
      float kk = __shfl_sync(FULL, key, seg0 + k);
      r += (kk < key) || (kk == key && seg0 + k < lane);
    }
    __syncwarp();
    ws[seg0 + r] = ti;
    ws[32 + seg0 + r] = make_float4(__int_as_float(k_i), __int_as_float(live), 0.0f, 0.0f);
    __syncwarp();
    ti = ws[lane];
    float4 x = ws[32 + lane];
    k_i = __float_as_int(x.x);
    live = __float_as_int(x.y);
    __syncwarp();
  }
  {  // group boxes (empty group: lo = +inf, hi = -inf: no source passes)
    float lx = live ? ti.x : INFINITY, ly = live ? ti.y : INFINITY, lz = live ? ti.z : INFINITY;
    float hx = live ? ti.x : -INFINITY, hy = live ? ti.y : -INFINITY, hz = live ? ti.z : -INFINITY;
#pragma unroll
    for (int o = LPG / 2; o; o >>= 1) {
      lx = fminf(lx, __shfl_xor_sync(FULL, lx, o)); hx = fmaxf(hx, __shfl_xor_sync(FULL, hx, o));
      ly = fminf(ly, __shfl_xor_sync(FULL, ly, o)); hy = fmaxf(hy, __shfl_xor_sync(FULL, hy, o));
      lz = fminf(lz, __shfl_xor_sync(FULL, lz, o)); hz = fmaxf(hz, __shfl_xor_sync(FULL, hz, o));
    }
    if ((lane & (LPG - 1)) == 0) {
      glo[lane / LPG] = make_float4(lx, ly, lz, 0.0f);
      ghi[lane / LPG] = make_float4(hx, hy, hz, 0.0f);
    }
    __syncwarp();
  }

  float R2 = a.cull_reach * a.cull_reach;
  float2 eps2x2 = make_float2(a.pp.p1, a.pp.p1);
  float2 rx = make_float2(0.0f, 0.0f), ry = rx, rz = rx;
  const float4* my_list = ws + (lane / LPG) * CAP;
  int cnt[G];
#pragma unroll
  for (int g = 0; g < G; ++g) cnt[g] = 0;
  // drain n (multiple of 8) steps: pad short lists, run, move the rest down
  auto drain = [&](int n) {
#pragma unroll
    for (int g = 0; g < G; ++g)
      for (int i = cnt[g] + lane; i < n; i += 32)
        ws[g * CAP + i] = make_float4(1e15f, 1e15f, 1e15f, 0.0f);
    __syncwarp();
    grav_steps<JB, REP>(my_list, n, ti, eps2x2, s_tab, gt, rx, ry, rz);
    __syncwarp();
#pragma unroll
    for (int g = 0; g < G; ++g) {
      int rest = cnt[g] - n;
      for (int i0 = 0; i0 < rest; i0 += 32) {
        float4 v;
        if (i0 + lane < rest) v = ws[g * CAP + n + i0 + lane];
        __syncwarp();
        if (i0 + lane < rest) ws[g * CAP + i0 + lane] = v;
        __syncwarp();
      }
      cnt[g] = rest > 0 ? rest : 0;
    }
  };

  const double* oA = T.origin + 3 * A;
  for (int64_t e = e0; e < e1; ++e) {
    int Bsrc = a.ent_src[e];
    if (Bsrc < 0) continue;  // bin stencil: off-mesh / duplicate cell
    int code = a.ent_code[e] & 31;
    int sh0 = code / 9 - 1, sh1 = (code / 3) % 3 - 1, sh2 = code % 3 - 1;
    float D0 = (float)((oA[0] - T.origin[3 * Bsrc]) - (double)sh0 * a.L);
    float D1 = (float)((oA[1] - T.origin[3 * Bsrc + 1]) - (double)sh1 * a.L);
    float D2 = (float)((oA[2] - T.origin[3 * Bsrc + 2]) - (double)sh2 * a.L);
    int64_t u0 = T.tile_ptr[Bsrc], u1 = T.tile_ptr[Bsrc + 1];
    for (int64_t ub = u0; ub < u1; ub += 32) {
      int64_t u = ub + lane;
      bool pass = false;
      int my_start = 0, my_n = 0;
      if (u < u1) {
        float4 lo = T.tile_lo[u], hi = T.tile_hi[u];
        my_n = T.tile_n[u];
        my_start = __float_as_int(hi.w);
        float gx = fmaxf(fmaxf((lo.x - D0) - thi.x, tlo.x - (hi.x - D0)), 0.0f);
        float gy = fmaxf(fmaxf((lo.y - D1) - thi.y, tlo.y - (hi.y - D1)), 0.0f);
        float gz = fmaxf(fmaxf((lo.z - D2) - thi.z, tlo.z - (hi.z - D2)), 0.0f);
        pass = fmaf(gz, gz, fmaf(gy, gy, gx * gx)) <= R2;
      }
      unsigned tm = __ballot_sync(FULL, pass);
      while (tm) {
        int j = __ffs(tm) - 1;
        tm &= tm - 1;
        int n_u = __shfl_sync(FULL, my_n, j);
        int s_u = __shfl_sync(FULL, my_start, j);
        bool has = lane < n_u;
        float4 sj = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        if (has) {
          sj = a.P0[s_u + lane];
          sj.x -= D0; sj.y -= D1; sj.z -= D2;
        }
        unsigned m[G];
        int over = 0, mx = 0;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          m[g] = __ballot_sync(FULL, has && box_gap2(sj.x, sj.y, sj.z, glo[g], ghi[g]) <= R2);
          int c = cnt[g] + __popc(m[g]);
          over |= c > USE;
          mx = max(mx, c);
        }
        if (over) {
          int mn = cnt[0];
#pragma unroll
          for (int g = 1; g < G; ++g) mn = min(mn, cnt[g]);
          drain(max(mn & ~7, (mx - USE + 7) & ~7));
        }
        unsigned lt = lanemask_lt();
#pragma unroll
        for (int g = 0; g < G; ++g) {
          if ((m[g] >> lane) & 1u) ws[g * CAP + cnt[g] + __popc(m[g] & lt)] = sj;
          cnt[g] += __popc(m[g]);
        }
      }
    }
  }
  {
    int mx = 0;
#pragma unroll
    for (int g = 0; g < G; ++g) mx = max(mx, cnt[g]);
    __syncwarp();
    if (mx) drain((mx + 7) & ~7);
  }
  float ax = rx.x + rx.y, ay = ry.x + ry.y, az = rz.x + rz.y;
  bool bad = !(isfinite(ax) && isfinite(ay) && isfinite(az));
  unsigned bm = __ballot_sync(FULL, live && bad);
  if (bm) {
    if (lane == 0) atomicMin(a.err_key, (unsigned long long)(e0 * 4 + 1));
    return;
  }
  if (live && a.write_out) {
    int64_t row = T.tperm[k_i];
    double mi = -(double)ti.w;
    a.out_flt[row * 3 + 0] += mi * (double)ax;
    a.out_flt[row * 3 + 1] += mi * (double)ay;
    a.out_flt[row * 3 + 2] += mi * (double)az;
  }
}

template <int JB, int REP, int G, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1)
k_gravity_grp(EvalDev a, const float4* __restrict__ table, GravTab gt, const int64_t* n_tiles_dev,
              const int64_t* t_begin_dev) {
  extern __shared__ float4 smem[];  // table (gt.rows * REP), then per-warp lists + boxes
  int64_t t0 = (int64_t)blockIdx.x * WARPS + (t_begin_dev ? *t_begin_dev : 0);
  int64_t t_end = *n_tiles_dev;
  if (t0 >= t_end) return;
  for (int k = threadIdx.x; k < gt.rows * REP; k += blockDim.x) smem[k] = table[k / REP];
  __syncthreads();
  int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t t = t0 + wid;
  float4* ws = smem + gt.rows * REP + wid * GravGroups<G>::PER_WARP;
  if (t < t_end)
    grav_tile_grp<JB, REP, G>(a, smem + (lane & (REP - 1)), gt, ws, t, lane);
}

template <int JB, int G, int WARPS>
static int launch_grp(const EvalDev& d, const float4* table, const GravTab& gt, int64_t tcap,
                      const int64_t* ntd, const int64_t* t_begin, cudaStream_t st, HbError* err) {
  constexpr int REP = 8;
  size_t sm = ((size_t)gt.rows * REP + (size_t)WARPS * GravGroups<G>::PER_WARP) * sizeof(float4);
  static std::mutex mu;
  static size_t set_for[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    if (dev >= 0 && dev < 64 && sm > set_for[dev]) {
      HB_CUDA_TRY(cudaFuncSetAttribute(k_gravity_grp<JB, REP, G, WARPS>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      set_for[dev] = sm;
    }
  }
  unsigned grid = grid_for(tcap, WARPS), blk = WARPS * 32;
  k_gravity_grp<JB, REP, G, WARPS><<<grid, blk, sm, st>>>(d, table, gt, ntd, t_begin);
  HB_LAUNCH_CHECK();
  return HB_OK;
}

// G target groups per warp (2, 4 or 8); 0 = not handled here
int launch_gravity_groups(int G, const EvalDev& d, const float4* table, const GravTab& gt,
                          int64_t tcap, const int64_t* ntd, cudaStream_t st, HbError* err,
                          const int64_t* t_begin) {
  if (gt.jbits == 4) {
    if (G == 2) return launch_grp<4, 2, 32>(d, table, gt, tcap, ntd, t_begin, st, err);
    if (G == 4) return launch_grp<4, 4, 32>(d, table, gt, tcap, ntd, t_begin, st, err);
    if (G == 8) return launch_grp<4, 8, 24>(d, table, gt, tcap, ntd, t_begin, st, err);
  } else {
    if (G == 2) return launch_grp<5, 2, 32>(d, table, gt, tcap, ntd, t_begin, st, err);
    if (G == 4) return launch_grp<5, 4, 32>(d, table, gt, tcap, ntd, t_begin, st, err);
    if (G == 8) return launch_grp<5, 8, 24>(d, table, gt, tcap, ntd, t_begin, st, err);
  }
  return set_err(err, HB_CONTRACT, "gravity target groups must be 2, 4 or 8");
}

}  // namespace hb
