// hb_sph.cu -- fused SPH passes of the resident force step.
//
//   pass A: neighbour count (hb/kernels.py:187-192) + summation density
//           (hb/kernels.py:170-186); both need only positions, masses and h_i.
//   pass B: CRK moments (hb/kernels.py:193-221) + hydro force with Monaghan
//           viscosity (hb/kernels.py:222-258); both need the post-density
//           state (rho, P, c_s), so they run after pass A and share one sweep.
//
// Work shape: one warp per gas target tile (<= 32 targets, lane = target),
// sources culled per tile then per source against the target tile box and
// staged in shared memory (as in hb_pairs.cu).  SPH supports (2h ~ 2.6 d) are
// small next to a tile, so most staged sources are out of support for most
// lanes.  Instead of evaluating every staged source on every lane, a cheap
// r^2 sweep builds a per-lane bitmask of in-support sources, then each lane
// walks only its own bits (divergent shared-memory reads, dense arithmetic).
// Gather formulation: every ordered pair accumulates on its receiving lane,
// no atomics, fixed order -> run-to-run deterministic.
#include "hb_internal.cuh"

namespace hb {

constexpr int kSphWarps = 4;
constexpr int kStageA = 256;  // pass A staged sources per warp (8 mask words per lane)

struct SphDev {
  Tiling T;
  const int64_t* ent_ptr;
  const int32_t* ent_src;
  const int32_t* ent_code;
  const float4 *P0, *P1, *P2, *P3;  // layouts: k_pack_sph
  Rows rows;                   // exact predicate re-checks (float64 rows)
  const int8_t* pshift;
  double L, reach;
  float reach2, band, alpha, beta;
  double *ncount, *rho, *moments, *hydro;
  const double *crk_A, *crk_B;
  const uint8_t* crk_fallback;
  double *gradA, *gradB;
  unsigned long long* err_key;
  const uint8_t* skip_leaf;  // pass B: ghost-only receivers to skip (or null)
  int skip_tiles;            // pass B: skip tiles without an owned member
};

__device__ __forceinline__ double exact_r2_rows(const Rows& st, const int8_t* ps, double L,
                                                int64_t i, int64_t j, int code) {
  int s[3] = {code / 9 - 1, (code / 3) % 3 - 1, code % 3 - 1};
  double r2 = 0.0;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    int64_t pi = ps ? ps[3 * i + d] : 0, pj = ps ? ps[3 * j + d] : 0;
    double dx = __dadd_rn(__dsub_rn(st.x(i, d), st.x(j, d)),
                          __dmul_rn((double)(pi - pj - s[d]), L));
    r2 = d == 0 ? __dmul_rn(dx, dx) : __dadd_rn(r2, __dmul_rn(dx, dx));
  }
  return r2;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// staging shared by both passes: walks the receiver's entries, culls source
// tiles and sources against the target box, calls consume() when the stage
// would overflow and at the end.  (A two-phase variant -- tile candidates
// collected into a per-warp list, then drained with the next tile's records
// prefetched into registers -- measured slower at c2: pass A 1.535 -> 1.563
// ms, pass B 2.84 -> 2.97 ms with spills at pass B's register budget.  A
// bulk-async variant -- each passing source tile's record runs requested with
// cp.async.bulk into a per-warp mbarrier ring, all of a cull batch's passing
// tiles in flight at once -- measured slower too: pass A 1.466 -> 1.558 ms,
// pass B 2.730 -> 2.959 ms (2 slots, 160-source stages to keep 4 CTAs / SM);
// commit 54c0e54, profiles/ab_r02.md.)
template <int NP, bool HYDRO, int CAP, class Consume>
__device__ __forceinline__ void sph_sweep(const SphDev& a, int A, int64_t e0, int64_t e1,
                                          float4 tlo, float4 thi, float hmax_t, float Rcap,
                                          float4 (*stage)[NP], int2* meta, int& cnt,
                                          Consume consume) {
  const Tiling& T = a.T;
  int lane = threadIdx.x & 31;
  double oA0 = T.origin[3 * A], oA1 = T.origin[3 * A + 1], oA2 = T.origin[3 * A + 2];
  float Rt = fminf(Rcap, 2.0f * hmax_t * 1.0001f);
  // pass B: support radius^2 of the pair (i, j) is 4 max(h_i, h_j)^2 (h_j:
  // the source record's P0.w)
  float Rt2 = Rt * Rt, Rcap2 = Rcap * Rcap;
  for (int64_t e = e0; e < e1; ++e) {
    int B = a.ent_src[e];
    if (B < 0) continue;  // bin stencil: off-mesh / duplicate cell
    int cw = a.ent_code[e];
    int code = cw & 31;
    int sh0 = code / 9 - 1, sh1 = (code / 3) % 3 - 1, sh2 = code % 3 - 1;
    float D0 = (float)((oA0 - T.origin[3 * B]) - (double)sh0 * a.L);
    float D1 = (float)((oA1 - T.origin[3 * B + 1]) - (double)sh1 * a.L);
    float D2 = (float)((oA2 - T.origin[3 * B + 2]) - (double)sh2 * a.L);
    int64_t u0 = T.tile_ptr[B], u1 = T.tile_ptr[B + 1];
    for (int64_t ub = u0; ub < u1; ub += 32) {
      int64_t u = ub + lane;
      bool pass = false;
      int my_start = 0, my_n = 0;
      if (u < u1) {
        float4 lo = T.tile_lo[u], hi = T.tile_hi[u];
        my_n = T.tile_n[u];
        my_start = __float_as_int(hi.w);  // emit_tile_box: first record index
        float R = HYDRO ? fminf(Rcap, 2.0f * fmaxf(hmax_t, lo.w) * 1.0001f) : Rt;
        float gx = fmaxf(fmaxf((lo.x - D0) - thi.x, tlo.x - (hi.x - D0)), 0.0f);
        float gy = fmaxf(fmaxf((lo.y - D1) - thi.y, tlo.y - (hi.y - D1)), 0.0f);
        float gz = fmaxf(fmaxf((lo.z - D2) - thi.z, tlo.z - (hi.z - D2)), 0.0f);
        pass = fmaf(gz, gz, fmaf(gy, gy, gx * gx)) <= R * R;
      }
      unsigned tm = __ballot_sync(0xffffffffu, pass);
      while (tm) {
        int j = __ffs(tm) - 1;
        tm &= tm - 1;
        int n_u = __shfl_sync(0xffffffffu, my_n, j);
        int k_j = __shfl_sync(0xffffffffu, my_start, j) + lane;
        bool ok = false;
        float4 sj[NP];
        if (lane < n_u) {
          sj[0] = a.P0[k_j];
          if (NP > 1) sj[1] = a.P1[k_j];
          if (NP > 2) sj[2] = a.P2[k_j];
          sj[0].x -= D0; sj[0].y -= D1; sj[0].z -= D2;
          float R2 = HYDRO ? fminf(Rcap2, fmaxf(Rt2, 4.0008f * sj[0].w * sj[0].w)) : Rt2;
          float gx = fmaxf(fmaxf(tlo.x - sj[0].x, sj[0].x - thi.x), 0.0f);
          float gy = fmaxf(fmaxf(tlo.y - sj[0].y, sj[0].y - thi.y), 0.0f);
          float gz = fmaxf(fmaxf(tlo.z - sj[0].z, sj[0].z - thi.z), 0.0f);
          ok = fmaf(gz, gz, fmaf(gy, gy, gx * gx)) <= R2;
        }
        unsigned sm = __ballot_sync(0xffffffffu, ok);
        if (cnt + 32 > CAP) consume();
        if (ok) {
          int slot = cnt + __popc(sm & lanemask_lt());
#pragma unroll
          for (int p = 0; p < NP; ++p) stage[slot][p] = sj[p];
          meta[slot] = make_int2(k_j, cw);
        }
        cnt += __popc(sm);
      }
    }
  }
  consume();
}

// per-lane in-support bitmask over the stage, stored word-major in shared
// memory (mask[w][lane], conflict-free); threshold on r^2 per lane (and per
// source h_j for hydro's 2 max(h_i, h_j) support)
// The last word is padded with far sources (r^2 ~ 3e36 beyond any threshold)
// so every word is a fully unrolled 32-source sweep with constant shifts.
template <int NP, bool HYDRO>
__device__ __forceinline__ unsigned build_masks(float4 (*stage)[NP], int cnt, float4 ti0,
                                                float hi, float thr_i, float reach2c,
                                                unsigned (*mask)[32]) {
  int lane = threadIdx.x & 31;
  int nw = (cnt + 31) >> 5;
  if (cnt + lane < nw * 32) stage[cnt + lane][0] = make_float4(1e18f, 1e18f, 1e18f, 0.0f);
  __syncwarp();
  unsigned nz = 0u;  // non-empty words of this lane
  for (int w = 0; w < nw; ++w) {
    unsigned bits = 0u;
    // two sources per step in packed FP32x2 (same rounding as the scalar form)
#pragma unroll
    for (int b = 0; b < 32; b += 2) {
      float4 s = stage[w * 32 + b][0], t = stage[w * 32 + b + 1][0];
      float2 dx = make_float2(ti0.x - s.x, ti0.x - t.x);
      float2 dy = make_float2(ti0.y - s.y, ti0.y - t.y);
      float2 dz = make_float2(ti0.z - s.z, ti0.z - t.z);
      float2 r2 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
      float2 thr = make_float2(thr_i, thr_i);  // pass B: thr_i = 4 h_i^2 (1 + 2e-4), s.w = h_j
      if (HYDRO) {
        float2 hj = make_float2(s.w, t.w);
        float2 t4 = __fmul2_rn(__fmul2_rn(make_float2(4.0008f, 4.0008f), hj), hj);
        thr = make_float2(fminf(reach2c, fmaxf(thr_i, t4.x)), fminf(reach2c, fmaxf(thr_i, t4.y)));
      }
      bits |= (r2.x <= thr.x ? 1u : 0u) << b;
      bits |= (r2.y <= thr.y ? 1u : 0u) << (b + 1);
    }
    mask[w][lane] = bits;
    nz |= (bits != 0u ? 1u : 0u) << w;
  }
  __syncwarp();
  return nz;
}

// ---------------------------------------------------------------- pass A
// 7 CTAs / SM (the shared-memory limit; 72 registers, small spills): 1.413 ->
// 1.342 ms at c2, 89.6 -> 84.9 ms at c4 against 6 CTAs at 80 registers (8 CTAs
// with 224-source stages at 64 registers spill: 1.49 ms, 94.0 ms)
template <int STG = kStageA, int MINB = 7>
__global__ void __launch_bounds__(kSphWarps * 32, MINB)
k_sph_density(SphDev a, const int64_t* n_tiles_dev) {
  __shared__ float4 s_stage[kSphWarps][STG][1];
  __shared__ int2 s_meta[kSphWarps][STG];
  __shared__ unsigned s_mask[kSphWarps][STG / 32][32];
  int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t t = (int64_t)blockIdx.x * kSphWarps + wid;
  if (t >= *n_tiles_dev) return;
  const Tiling& T = a.T;
  int A = T.tile_leaf[t];
  int64_t e0 = a.ent_ptr[A], e1 = a.ent_ptr[A + 1];
  if (e0 == e1) return;
  int n_t = T.tile_n[t];
  bool live = lane < n_t;
  int k_i = T.tile_start[t] + (live ? lane : 0);
  int64_t row_i = T.tperm[k_i];
  float4 ti0 = a.P0[k_i];
  float h = a.P1[k_i].w;
  float hinv = h > 0.0f ? 1.0f / h : 0.0f;
  double h64 = a.rows.hh(row_i);
  double thr4_64 = __dmul_rn(__dmul_rn(4.0, h64), h64);   // (4 h) h as hb/kernels.py:191
  float thr4 = (float)thr4_64;
  float thr4b = thr4 * a.band;
  float thr_mask = fminf(a.reach2, thr4) * (1.0f + 2.0f * a.band);
  float4 tlo = a.T.tile_lo[t], thi = a.T.tile_hi[t];
  float rho = 0.0f;
  unsigned count = 0;
  int cnt = 0;
  float4(*stage)[1] = s_stage[wid];
  int2* meta = s_meta[wid];
  unsigned(*mask)[32] = s_mask[wid];
  auto consume = [&]() {
    __syncwarp();
    unsigned nz = build_masks<1, false>(stage, cnt, ti0, h, live ? thr_mask : -1.0f, 0.0f, mask);
    // the two pairs of a walk iteration (walk_masks2; the second may be absent,
    // onb = false) in packed FP32x2 arithmetic (FFMA2 / FMUL2 / FADD2: one
    // issue slot for both pairs).  Per pair: r^2 = (dx dx + dy dy) + dz dz; 4 h_i^2
    // <= reach^2 = (2 h_max)^2 exactly, so the count predicate r^2 <= 4 h_i^2
    // implies the reach test, and W(r, h_i) vanishes past 2 h_i: only the count
    // needs the float64 decision near its threshold.  q = r^2 rsqrt(r^2) / h_i
    // (MUFU.RSQ, no IEEE sqrt fix-up).  Same rounding order as the scalar
    // form it replaced (density and counts unchanged bitwise; 1.462 -> 1.445
    // ms at c2)
    auto pair2 = [&](int qa, int qb, bool onb) {
      float4 sa = stage[qa][0], sb = stage[qb][0];
      float2 dx = make_float2(ti0.x - sa.x, ti0.x - sb.x);
      float2 dy = make_float2(ti0.y - sa.y, ti0.y - sb.y);
      float2 dz = make_float2(ti0.z - sa.z, ti0.z - sb.z);
      float2 r2 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
      bool ca = r2.x <= thr4, cb = r2.y <= thr4;
      if (fabsf(r2.x - thr4) <= thr4b) {  // exact float64 decision, reference expression
        int2 mt = meta[qa];
        ca = exact_r2_rows(a.rows, a.pshift, a.L, row_i, T.tperm[mt.x], mt.y & 31) <= thr4_64;
      }
      if (onb && fabsf(r2.y - thr4) <= thr4b) {
        int2 mt = meta[qb];
        cb = exact_r2_rows(a.rows, a.pshift, a.L, row_i, T.tperm[mt.x], mt.y & 31) <= thr4_64;
      }
      float2 rs = make_float2(rsqrt_ftz(fmaxf(r2.x, 1e-30f)), rsqrt_ftz(fmaxf(r2.y, 1e-30f)));
      float2 qq = __fmul2_rn(__fmul2_rn(r2, rs), make_float2(hinv, hinv));
      count += (ca ? 1u : 0u) + ((onb && cb) ? 1u : 0u);
      // w_body: t = max(2 - q, 0) zeroes the outer branch past q = 2
      float2 t = __ffma2_rn(qq, make_float2(-1.0f, -1.0f), make_float2(2.0f, 2.0f));
      t = make_float2(fmaxf(t.x, 0.0f), fmaxf(t.y, 0.0f));
      float2 outer = __fmul2_rn(__fmul2_rn(__fmul2_rn(make_float2(0.25f, 0.25f), t), t), t);
      float2 inner = __ffma2_rn(__fmul2_rn(qq, qq),
                                __ffma2_rn(make_float2(0.75f, 0.75f), qq,
                                           make_float2(-1.5f, -1.5f)),
                                make_float2(1.0f, 1.0f));
      float2 wv = make_float2(qq.x < 1.0f ? inner.x : outer.x, qq.y < 1.0f ? inner.y : outer.y);
      float2 ww = __fmul2_rn(make_float2(sa.w, sb.w), wv);
      rho += ww.x + (onb ? ww.y : 0.0f);
    };
    walk_masks2(mask, nz, [&](int q1, int q2) { pair2(q1, q2 >= 0 ? q2 : q1, q2 >= 0); });
    __syncwarp();
    cnt = 0;
  };
  // cull radius from the tile's largest h (emit_tile_box: tile_lo.w), not this
  // lane's: every lane culls sources for the whole tile
  sph_sweep<1, false, STG>(a, A, e0, e1, tlo, thi, tlo.w, a.reach * 1.0001f, stage, meta,
                               cnt, consume);
  if (live) {
    float norm3 = h > 0.0f ? kSigma * hinv * hinv * hinv : 0.0f;
    a.ncount[row_i] += (double)count;
    a.rho[row_i] += (double)(norm3 * rho);
  }
}

// ---------------------------------------------------------------- pass B
// records (k_pack_sph layout 1): P0 = (x, y, z, h), P1 = (vx, vy, vz, m),
// P2 = (P/rho^2, c_s, rho, sigma/h^5).  1/q = h r^-1 reuses the rsqrt the
// separation needs: a pair issues 5 MUFU (rsqrt, 1/h_j, 1/rho_j and the two of
// the viscosity term, evaluated for every pair and selected).  (A fourth record with 1/h_j and
// m_j/rho_j precomputed, and 160-source stages to stay at 4 CTAs / SM, measured
// 3.32 vs 2.83 ms at c2: staging and flush count outweigh the two MUFU.)
// Two pairs per walk iteration at 4 CTAs / SM (127 registers, no spills).
constexpr int kStageB = 192;
// (5 CTAs / SM at 96 registers spills and measured 2.41 -> 2.62 ms at c2)
__global__ void __launch_bounds__(kSphWarps * 32, 4)
k_sph_force(SphDev a, const int64_t* n_tiles_dev) {
  __shared__ float4 s_stage[kSphWarps][kStageB][3];
  __shared__ int2 s_meta[kSphWarps][kStageB];
  __shared__ unsigned s_mask[kSphWarps][kStageB / 32][32];
  int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t t = (int64_t)blockIdx.x * kSphWarps + wid;
  if (t >= *n_tiles_dev) return;
  const Tiling& T = a.T;
  int A = T.tile_leaf[t];
  if (a.skip_leaf && a.skip_leaf[A]) return;
  if (a.skip_tiles && T.tile_skip[t]) return;
  int64_t e0 = a.ent_ptr[A], e1 = a.ent_ptr[A + 1];
  if (e0 == e1) return;
  int n_t = T.tile_n[t];
  bool live = lane < n_t;
  int k_i = T.tile_start[t] + (live ? lane : 0);
  float4 ti0 = a.P0[k_i], ti1 = a.P1[k_i], ti2 = a.P2[k_i];
  float hi = ti0.w;
  float hinv = hi > 0.0f ? 1.0f / hi : 0.0f;
  float thr_i = 4.0008f * hi * hi;
  float reach2c = a.reach2 * (1.0f + 2.0f * a.band);
  float4 tlo = a.T.tile_lo[t], thi = a.T.tile_hi[t];
  float mo[10];
#pragma unroll
  for (int c = 0; c < 10; ++c) mo[c] = 0.0f;
  float fx = 0.f, fy = 0.f, fz = 0.f, ei = 0.f, ej = 0.f;
  int cnt = 0;
  float4(*stage)[3] = s_stage[wid];
  int2* meta = s_meta[wid];
  unsigned(*mask)[32] = s_mask[wid];
  auto consume = [&]() {
    __syncwarp();
    unsigned nz = build_masks<3, true>(stage, cnt, ti0, hi, live ? thr_i : -1.0f,
                                       live ? reach2c : -1.0f, mask);
    // the two pairs of a walk iteration (walk_masks2; the second may be absent,
    // onb = false) evaluated together in packed FP32x2 arithmetic (FFMA2 /
    // FMUL2 / FADD2: one issue slot for both pairs); the viscosity branch
    // (approaching pairs) is a select, and the accumulators stay scalar, pair a
    // then pair b.  Against one scalar pair per call: 261 -> 209 instructions
    // per walk iteration, pass B 2.728 -> 2.439 ms at c2, 173.2 -> 154.1 ms at c4.
    auto pair2 = [&](int qa, int qb, bool onb) {
      const float2 one = make_float2(1.0f, 1.0f), half = make_float2(0.5f, 0.5f);
      float4 a0 = stage[qa][0], a1 = stage[qa][1], a2 = stage[qa][2];
      float4 b0 = stage[qb][0], b1 = stage[qb][1], b2 = stage[qb][2];
      float2 dx = make_float2(ti0.x - a0.x, ti0.x - b0.x);
      float2 dy = make_float2(ti0.y - a0.y, ti0.y - b0.y);
      float2 dz = make_float2(ti0.z - a0.z, ti0.z - b0.z);
      float2 r2 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
      bool va = r2.x <= a.reach2, vb = onb && r2.y <= a.reach2;
      if (!(va || vb)) return;
      float2 rinv = make_float2(rsqrt_ftz(fmaxf(r2.x, 1e-30f)), rsqrt_ftz(fmaxf(r2.y, 1e-30f)));
      float2 r = __fmul2_rn(r2, rinv);
      float2 hj = make_float2(a0.w, b0.w);
      float2 qi = __fmul2_rn(r, make_float2(hinv, hinv));
      float2 qj = __fmul2_rn(r, make_float2(rcp_approx(a0.w), rcp_approx(b0.w)));
      // u = max(2 - q, 0): the outer branch vanishes past q = 2 by itself
      float2 ui = __ffma2_rn(qi, make_float2(-1.0f, -1.0f), make_float2(2.0f, 2.0f));
      float2 uj = __ffma2_rn(qj, make_float2(-1.0f, -1.0f), make_float2(2.0f, 2.0f));
      ui = make_float2(fmaxf(ui.x, 0.0f), fmaxf(ui.y, 0.0f));
      uj = make_float2(fmaxf(uj.x, 0.0f), fmaxf(uj.y, 0.0f));
      float2 ui2 = __fmul2_rn(ui, ui), uj2 = __fmul2_rn(uj, uj);
      float2 w_in = __ffma2_rn(__fmul2_rn(qi, qi),
                               __ffma2_rn(make_float2(0.75f, 0.75f), qi, make_float2(-1.5f, -1.5f)),
                               one);
      float2 w_out = __fmul2_rn(__fmul2_rn(make_float2(0.25f, 0.25f), ui2), ui);
      float2 c3 = make_float2(-3.0f, -3.0f), c225 = make_float2(2.25f, 2.25f),
             c075 = make_float2(-0.75f, -0.75f);
      float2 gi_in = __ffma2_rn(c225, qi, c3), gj_in = __ffma2_rn(c225, qj, c3);
      float2 gi_out = __fmul2_rn(__fmul2_rn(c075, ui2), __fmul2_rn(make_float2(hi, hi), rinv));
      float2 gj_out = __fmul2_rn(__fmul2_rn(c075, uj2), __fmul2_rn(hj, rinv));
      float2 wi = make_float2(qi.x < 1.0f ? w_in.x : w_out.x, qi.y < 1.0f ? w_in.y : w_out.y);
      float2 gi = make_float2(qi.x < 1.0f ? gi_in.x : gi_out.x, qi.y < 1.0f ? gi_in.y : gi_out.y);
      float2 gj = make_float2(qj.x < 1.0f ? gj_in.x : gj_out.x, qj.y < 1.0f ? gj_in.y : gj_out.y);
      // CRK moments: w = V_j W(r, h_i) (hb/kernels.py:205-220)
      float2 vj = make_float2(a2.z > 0.0f ? a1.w * rcp_approx(a2.z) : 0.0f,
                              b2.z > 0.0f ? b1.w * rcp_approx(b2.z) : 0.0f);
      float2 wk = __fmul2_rn(vj, wi);
      wk = make_float2(va ? wk.x : 0.0f, vb ? wk.y : 0.0f);
      float2 wx = __fmul2_rn(wk, dx), wy = __fmul2_rn(wk, dy), wz = __fmul2_rn(wk, dz);
      mo[0] += wk.x; mo[0] += wk.y;
      mo[1] -= wx.x; mo[1] -= wx.y; mo[2] -= wy.x; mo[2] -= wy.y; mo[3] -= wz.x; mo[3] -= wz.y;
      mo[4] = fmaf(wx.y, dx.y, fmaf(wx.x, dx.x, mo[4]));
      mo[5] = fmaf(wx.y, dy.y, fmaf(wx.x, dy.x, mo[5]));
      mo[6] = fmaf(wx.y, dz.y, fmaf(wx.x, dz.x, mo[6]));
      mo[7] = fmaf(wy.y, dy.y, fmaf(wy.x, dy.x, mo[7]));
      mo[8] = fmaf(wy.y, dz.y, fmaf(wy.x, dz.x, mo[8]));
      mo[9] = fmaf(wz.y, dz.y, fmaf(wz.x, dz.x, mo[9]));
      // hydro (hb/kernels.py:227-258), m_i factored out
      float2 gw = __fmul2_rn(half, __ffma2_rn(gi, make_float2(ti2.w, ti2.w),
                                              __fmul2_rn(gj, make_float2(a2.w, b2.w))));
      float2 vx = make_float2(ti1.x - a1.x, ti1.x - b1.x);
      float2 vy = make_float2(ti1.y - a1.y, ti1.y - b1.y);
      float2 vz = make_float2(ti1.z - a1.z, ti1.z - b1.z);
      float2 vdotr = __ffma2_rn(vz, dz, __ffma2_rn(vy, dy, __fmul2_rn(vx, dx)));
      float2 hbar = __fmul2_rn(half, __fadd2_rn(make_float2(hi, hi), hj));
      float2 cbar = __fmul2_rn(half, __fadd2_rn(make_float2(ti2.y, ti2.y), make_float2(a2.y, b2.y)));
      float2 rhobar = __fmul2_rn(half, __fadd2_rn(make_float2(ti2.z, ti2.z), make_float2(a2.z, b2.z)));
      float2 den = __ffma2_rn(__fmul2_rn(make_float2(0.01f, 0.01f), hbar), hbar, r2);
      float2 mu = __fmul2_rn(__fmul2_rn(hbar, vdotr),
                             make_float2(rcp_approx(den.x), rcp_approx(den.y)));
      float2 acm = __fmul2_rn(__fmul2_rn(make_float2(a.alpha, a.alpha), cbar), mu);
      float2 vis = __fmul2_rn(__ffma2_rn(__fmul2_rn(make_float2(a.beta, a.beta), mu), mu,
                                         make_float2(-acm.x, -acm.y)),
                              make_float2(rcp_approx(rhobar.x), rcp_approx(rhobar.y)));
      float2 visc = make_float2(vdotr.x < 0.0f ? vis.x : 0.0f, vdotr.y < 0.0f ? vis.y : 0.0f);
      float2 mjg = __fmul2_rn(make_float2(a1.w, b1.w), gw);
      mjg = make_float2(va ? mjg.x : 0.0f, vb ? mjg.y : 0.0f);
      float2 w = __fmul2_rn(__fadd2_rn(__fadd2_rn(make_float2(ti2.x, ti2.x), make_float2(a2.x, b2.x)),
                                       visc), mjg);
      fx = fmaf(-w.y, dx.y, fmaf(-w.x, dx.x, fx));
      fy = fmaf(-w.y, dy.y, fmaf(-w.x, dy.x, fy));
      fz = fmaf(-w.y, dz.y, fmaf(-w.x, dz.x, fz));
      float2 work = __fmul2_rn(vdotr, mjg);
      float2 hv = __fmul2_rn(half, visc);
      float2 pi_ = __fadd2_rn(make_float2(ti2.x, ti2.x), hv);
      float2 pj_ = __fadd2_rn(make_float2(a2.x, b2.x), hv);
      ei = fmaf(pi_.y, work.y, fmaf(pi_.x, work.x, ei));
      ej = fmaf(pj_.y, work.y, fmaf(pj_.x, work.x, ej));
    };
    walk_masks2(mask, nz, [&](int q1, int q2) { pair2(q1, q2 >= 0 ? q2 : q1, q2 >= 0); });
    __syncwarp();
    cnt = 0;
  };
  sph_sweep<3, true, kStageB>(a, A, e0, e1, tlo, thi, tlo.w, a.reach * 1.0001f, stage, meta,
                              cnt, consume);
  bool bad = !(isfinite(fx) && isfinite(fy) && isfinite(fz) && isfinite(ei) && isfinite(mo[0]));
  if (__ballot_sync(0xffffffffu, live && bad)) {
    if (lane == 0) atomicMin(a.err_key, (unsigned long long)(e0 * 4 + 1));
    return;
  }
  if (live) {
    int64_t row = T.tperm[k_i];
    double norm3 = hi > 0.0f ? (double)kSigma * (double)hinv * (double)hinv * (double)hinv : 0.0;
    for (int c = 0; c < 10; ++c) a.moments[row * 10 + c] += norm3 * (double)mo[c];
    double mi = (double)ti1.w;
    a.hydro[row * 5 + 0] += mi * (double)fx;
    a.hydro[row * 5 + 1] += mi * (double)fy;
    a.hydro[row * 5 + 2] += mi * (double)fz;
    a.hydro[row * 5 + 3] += mi * (double)ei;
    a.hydro[row * 5 + 4] += mi * (double)ej;
  }
}

// ---------------------------------------------------------------- pass C
// gradA / gradB of the CRK coefficients (north star; the reference computes
// only A and B, hb/hydro.py:99-150).  With G = V_j (dW/dr)/r at h_i and
// dr = x_i - x_j, the gradient moments are sum G dr (3), sum G dr dr (6) and
// sum G dr dr dr (10) over gas-gas pairs within 2 h_i -- the compat path's
// KID_CRK_GRAD1/2 channels (hb_pairs.cuh).  The epilogue solves, in float64
// per target lane, from the pass-B moments and the CRK solve's A, B:
//   d_g m0 = S1_g;  d_g m1_a = -S2_ag - delta_ag m0;
//   d_g m2_ab = S3_abg - delta_ag m1_b - delta_bg m1_a;
//   d_g B = m2^-1 (d_g m1 - d_g m2 B);  d_g A = -A^2 (d_g m0 - d_g B.m1 - B.d_g m1);
//   fallback rows (A = 1/m0, B = 0): d_g A = -d_g m0 / m0^2, d_g B = 0
// (hydro.crk_gradients_from_moments is the same algebra on the compat path).
__device__ __forceinline__ void crk_grad_solve(const double* mom, double A, const double* B,
                                               bool fb, const double* S1, const double* S2v,
                                               const double* S3v, double* dA, double* dB) {
  double m0 = mom[0];
  double m1[3] = {mom[1], mom[2], mom[3]};
  for (int k = 0; k < 3; ++k) dA[k] = 0.0;
  for (int k = 0; k < 9; ++k) dB[k] = 0.0;
  if (!(m0 > 0.0)) return;
  if (fb) {
    for (int g = 0; g < 3; ++g) dA[g] = -S1[g] / (m0 * m0);
    return;
  }
  // symmetric tensors from the packed channels
  const int i2[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};
  double S2[3][3];
  for (int a = 0; a < 3; ++a) for (int b = 0; b < 3; ++b) S2[a][b] = S2v[i2[a][b]];
  // S3 channel order (KID_CRK_GRAD2): xxx xxy xxz xyy xyz xzz yyy yyz yzz zzz
  auto s3 = [&](int a, int b, int c) -> double {
    int n[3] = {0, 0, 0};
    n[a]++; n[b]++; n[c]++;
    int x = n[0], y = n[1];
    if (x == 3) return S3v[0];
    if (x == 2) return y == 1 ? S3v[1] : S3v[2];
    if (x == 1) return y == 2 ? S3v[3] : (y == 1 ? S3v[4] : S3v[5]);
    return y == 3 ? S3v[6] : (y == 2 ? S3v[7] : (y == 1 ? S3v[8] : S3v[9]));
  };
  double dm1[3][3], rhs[3][3];
  for (int a = 0; a < 3; ++a)
    for (int g = 0; g < 3; ++g) dm1[a][g] = -S2[a][g] - (a == g ? m0 : 0.0);
  for (int a = 0; a < 3; ++a)
    for (int g = 0; g < 3; ++g) {
      double t = dm1[a][g];
      for (int b = 0; b < 3; ++b) {
        double dm2 = s3(a, b, g) - (a == g ? m1[b] : 0.0) - (b == g ? m1[a] : 0.0);
        t -= dm2 * B[b];
      }
      rhs[a][g] = t;
    }
  // m2 dB = rhs (Gaussian elimination with partial pivoting, 3 right-hand sides)
  double m[3][6] = {{mom[4], mom[5], mom[6]}, {mom[5], mom[7], mom[8]}, {mom[6], mom[8], mom[9]}};
  for (int r = 0; r < 3; ++r) for (int g = 0; g < 3; ++g) m[r][3 + g] = rhs[r][g];
  for (int c = 0; c < 3; ++c) {
    int piv = c;
    for (int r = c + 1; r < 3; ++r) if (fabs(m[r][c]) > fabs(m[piv][c])) piv = r;
    if (piv != c) for (int k = 0; k < 6; ++k) { double t = m[c][k]; m[c][k] = m[piv][k]; m[piv][k] = t; }
    for (int r = c + 1; r < 3; ++r) {
      double f = m[r][c] / m[c][c];
      for (int k = c; k < 6; ++k) m[r][k] -= f * m[c][k];
    }
  }
  double X[3][3];
  for (int g = 0; g < 3; ++g)
    for (int r = 2; r >= 0; --r) {
      double t = m[r][3 + g];
      for (int k = r + 1; k < 3; ++k) t -= m[r][k] * X[k][g];
      X[r][g] = t / m[r][r];
    }
  for (int a = 0; a < 3; ++a) for (int g = 0; g < 3; ++g) dB[3 * a + g] = X[a][g];
  for (int g = 0; g < 3; ++g) {
    double dD = S1[g];
    for (int a = 0; a < 3; ++a) dD -= X[a][g] * m1[a] + B[a] * dm1[a][g];
    dA[g] = -(A * A) * dD;
  }
}

__global__ void __launch_bounds__(kSphWarps * 32, 4)
k_sph_grad(SphDev a, const int64_t* n_tiles_dev) {
  __shared__ float4 s_stage[kSphWarps][kStageA][1];
  __shared__ int2 s_meta[kSphWarps][kStageA];
  __shared__ unsigned s_mask[kSphWarps][kStageA / 32][32];
  int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t t = (int64_t)blockIdx.x * kSphWarps + wid;
  if (t >= *n_tiles_dev) return;
  const Tiling& T = a.T;
  int A = T.tile_leaf[t];
  if (a.skip_leaf && a.skip_leaf[A]) return;
  if (a.skip_tiles && T.tile_skip[t]) return;
  int64_t e0 = a.ent_ptr[A], e1 = a.ent_ptr[A + 1];
  if (e0 == e1) return;
  int n_t = T.tile_n[t];
  bool live = lane < n_t;
  int k_i = T.tile_start[t] + (live ? lane : 0);
  float4 ti0 = a.P0[k_i];
  float h = a.P1[k_i].w;
  float hinv = h > 0.0f ? 1.0f / h : 0.0f;
  float thr_mask = fminf(a.reach2, 4.0f * h * h) * (1.0f + 2.0f * a.band);
  float4 tlo = a.T.tile_lo[t], thi = a.T.tile_hi[t];
  float g1[9], g2[10];
#pragma unroll
  for (int c = 0; c < 9; ++c) g1[c] = 0.0f;
#pragma unroll
  for (int c = 0; c < 10; ++c) g2[c] = 0.0f;
  int cnt = 0;
  float4(*stage)[1] = s_stage[wid];
  int2* meta = s_meta[wid];
  unsigned(*mask)[32] = s_mask[wid];
  auto consume = [&]() {
    __syncwarp();
    unsigned nz = build_masks<1, false>(stage, cnt, ti0, h, live ? thr_mask : -1.0f, 0.0f, mask);
    walk_masks(mask, nz, [&](int q) {
      float4 s = stage[q][0];
      float dx = ti0.x - s.x, dy = ti0.y - s.y, dz = ti0.z - s.z;
      float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
      float rinv = rsqrt_ftz(fmaxf(r2, 1e-30f));
      float qq = r2 * rinv * hinv;
      float u = 2.0f - qq;
      float gw = qq < 1.0f ? fmaf(2.25f, qq, -3.0f)
                           : (qq < 2.0f ? -0.75f * u * u * (h * rinv) : 0.0f);
      float g = s.w * gw;
      float gx = g * dx, gy = g * dy, gz = g * dz;
      g1[0] += gx; g1[1] += gy; g1[2] += gz;
      g1[3] = fmaf(gx, dx, g1[3]); g1[4] = fmaf(gx, dy, g1[4]); g1[5] = fmaf(gx, dz, g1[5]);
      g1[6] = fmaf(gy, dy, g1[6]); g1[7] = fmaf(gy, dz, g1[7]); g1[8] = fmaf(gz, dz, g1[8]);
      float gxx = gx * dx, gyy = gy * dy, gzz = gz * dz, gxy = gx * dy;
      g2[0] = fmaf(gxx, dx, g2[0]); g2[1] = fmaf(gxx, dy, g2[1]); g2[2] = fmaf(gxx, dz, g2[2]);
      g2[3] = fmaf(gyy, dx, g2[3]); g2[4] = fmaf(gxy, dz, g2[4]); g2[5] = fmaf(gzz, dx, g2[5]);
      g2[6] = fmaf(gyy, dy, g2[6]); g2[7] = fmaf(gyy, dz, g2[7]); g2[8] = fmaf(gzz, dy, g2[8]);
      g2[9] = fmaf(gzz, dz, g2[9]);
    });
    __syncwarp();
    cnt = 0;
  };
  sph_sweep<1, false, kStageA>(a, A, e0, e1, tlo, thi, tlo.w, a.reach * 1.0001f, stage, meta,
                               cnt, consume);
  bool bad = !(isfinite(g1[0]) && isfinite(g1[3]) && isfinite(g2[0]) && isfinite(g2[9]));
  if (__ballot_sync(0xffffffffu, live && bad)) {
    if (lane == 0) atomicMin(a.err_key, (unsigned long long)(e0 * 4 + 1));
    return;
  }
  if (!live) return;
  int64_t row = T.tperm[k_i];
  double norm5 = h > 0.0f ? (double)kSigma * pow((double)hinv, 5.0) : 0.0;
  double S1[3], S2[6], S3[10];
  for (int c = 0; c < 3; ++c) S1[c] = norm5 * (double)g1[c];
  for (int c = 0; c < 6; ++c) S2[c] = norm5 * (double)g1[3 + c];
  for (int c = 0; c < 10; ++c) S3[c] = norm5 * (double)g2[c];
  double Bi[3] = {a.crk_B[3 * row], a.crk_B[3 * row + 1], a.crk_B[3 * row + 2]};
  double dA[3], dB[9];
  crk_grad_solve(a.moments + row * 10, a.crk_A[row], Bi, a.crk_fallback[row] != 0, S1, S2, S3,
                 dA, dB);
  for (int c = 0; c < 3; ++c) a.gradA[row * 3 + c] = dA[c];
  for (int c = 0; c < 9; ++c) a.gradB[row * 9 + c] = dB[c];
}

// gas records for both passes
// layout 0 (pass A): P0 = (x, y, z, m), P1 = (.., .., .., h)
// layout 2 (pass C): P0 = (x, y, z, V = m/rho), P1 = (.., .., .., h)
// layout 1 (pass B): P0 = (x, y, z, h), P1 = (vx, vy, vz, m),
//                    P2 = (P/rho^2, c_s, rho, sigma/h^5)
// rho_f / u_f (optional, leaf-order SoA density and internal energy): rho, P
// and c_s come from them with the EOS of hb/hydro.py:48-57 evaluated here
// (P = ((gamma - 1) rho) u, c_s = sqrt(max((gamma (gamma - 1)) u, 0))), so the
// step needs no separate EOS pass
__global__ void k_pack_sph(int64_t tcap, const int64_t* n_tiles_dev, const Tiling T,
                           Rows rows, const int8_t* pshift, double L, float4* P0,
                           float4* P1, float4* P2, float4* P3, int layout, const double* rho_f,
                           const double* u_f, double gamma) {
  int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (t >= *n_tiles_dev || lane >= T.tile_n[t]) return;
  int leaf = T.tile_leaf[t];
  int64_t k = T.tile_start[t] + lane;
  int64_t r = T.tperm[k];
  float c[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double v = __dadd_rn(rows.x(r, d), __dmul_rn((double)(pshift ? pshift[3 * r + d] : 0), L));
    c[d] = (float)(v - T.origin[3 * leaf + d]);
  }
  double h = rows.hh(r), m = rows.m(r);
  if (layout == 0) {
    P0[k] = make_float4(c[0], c[1], c[2], (float)m);
    P1[k] = make_float4(0.f, 0.f, 0.f, (float)h);
    return;
  }
  double rho = rho_f ? rho_f[r] : rows.dens(r);
  if (layout == 2) {
    P0[k] = make_float4(c[0], c[1], c[2], rho > 0 ? (float)(m / rho) : 0.0f);
    P1[k] = make_float4(0.f, 0.f, 0.f, (float)h);
    return;
  }
  double P, cs;
  if (rho_f && u_f) {
    double gm1 = gamma - 1.0, u = u_f[r];
    P = gm1 * rho * u;
    cs = sqrt(fmax(gamma * gm1 * u, 0.0));
  } else {
    P = rows.pres(r);
    cs = rows.snd(r);
  }
  double norm5 = h > 0 ? 0.31830988618379067 / (h * h * h * h * h) : 0.0;
  double fpart = rho > 0 ? P / (rho * rho) : 0.0;
  P0[k] = make_float4(c[0], c[1], c[2], (float)h);
  P1[k] = make_float4((float)rows.v(r, 0), (float)rows.v(r, 1), (float)rows.v(r, 2), (float)m);
  P2[k] = make_float4((float)fpart, (float)cs, (float)rho, (float)norm5);
}

int pack_sph(const Tiling& T, const int64_t* ntd, Rows rows, const int8_t* pshift,
             double L, float4* P0, float4* P1, float4* P2, float4* P3, int layout,
             cudaStream_t st, HbError* err, const double* rho, const double* u, double gamma) {
  k_pack_sph<<<grid_for(T.n_tiles_cap * 32, 256), 256, 0, st>>>(
      T.n_tiles_cap, ntd, T, rows, pshift, L, P0, P1, P2, P3, layout, rho, u, gamma);
  HB_LAUNCH_CHECK();
  return HB_OK;
}

int launch_sph(int pass, const SphArgs& s, cudaStream_t st, HbError* err) {
  SphDev a;
  a.T = *s.T; a.ent_ptr = s.ent_ptr; a.ent_src = s.ent_src; a.ent_code = s.ent_code;
  a.P0 = s.P0; a.P1 = s.P1; a.P2 = s.P2; a.P3 = s.P3; a.rows = s.rows; a.pshift = s.pshift;
  a.L = s.L; a.reach = s.reach; a.reach2 = (float)(s.reach * s.reach); a.band = s.band;
  a.alpha = (float)s.alpha; a.beta = (float)s.beta;
  a.ncount = s.ncount; a.rho = s.rho; a.moments = s.moments; a.hydro = s.hydro;
  a.crk_A = s.crk_A; a.crk_B = s.crk_B; a.crk_fallback = s.crk_fallback;
  a.gradA = s.gradA; a.gradB = s.gradB;
  a.err_key = s.err_key;
  a.skip_leaf = s.skip_leaf;
  a.skip_tiles = s.skip_tiles;
  unsigned grid = grid_for(s.T->n_tiles_cap, kSphWarps);
  if (pass == 0) k_sph_density<><<<grid, kSphWarps * 32, 0, st>>>(a, s.n_tiles_dev);
  else if (pass == 1) k_sph_force<<<grid, kSphWarps * 32, 0, st>>>(a, s.n_tiles_dev);
  else k_sph_grad<<<grid, kSphWarps * 32, 0, st>>>(a, s.n_tiles_dev);
  HB_LAUNCH_CHECK();
  return HB_OK;
}

}  // namespace hb
