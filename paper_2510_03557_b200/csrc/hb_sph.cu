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
constexpr int kStageB = 192;  // pass B (3 records per source)

struct SphDev {
  Tiling T;
  const int64_t* ent_ptr;
  const int32_t* ent_src;
  const int32_t* ent_code;
  const float4 *P0, *P1, *P2;  // (x,y,z,m) (vx,vy,vz,h) (P/rho^2, c_s, rho, sigma/h^5)
  const double* state;         // exact predicate re-checks (float64 rows)
  const int8_t* pshift;
  double L, reach;
  float reach2, band, alpha, beta;
  double *ncount, *rho, *moments, *hydro;
  unsigned long long* err_key;
  const uint8_t* skip_leaf;  // pass B: ghost-only receivers to skip (or null)
  int skip_tiles;            // pass B: skip tiles without an owned member
};

__device__ __forceinline__ double exact_r2_rows(const double* st, const int8_t* ps, double L,
                                                int64_t i, int64_t j, int code) {
  int s[3] = {code / 9 - 1, (code / 3) % 3 - 1, code % 3 - 1};
  double r2 = 0.0;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    int64_t pi = ps ? ps[3 * i + d] : 0, pj = ps ? ps[3 * j + d] : 0;
    double dx = __dadd_rn(__dsub_rn(st[i * NCOL + d], st[j * NCOL + d]),
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
// would overflow and at the end.
template <int NP, bool HYDRO, int CAP, class Consume>
__device__ __forceinline__ void sph_sweep(const SphDev& a, int A, int64_t e0, int64_t e1,
                                          float4 tlo, float4 thi, float hmax_t, float Rcap,
                                          float4 (*stage)[NP], int2* meta, int& cnt,
                                          Consume consume) {
  const Tiling& T = a.T;
  int lane = threadIdx.x & 31;
  double oA0 = T.origin[3 * A], oA1 = T.origin[3 * A + 1], oA2 = T.origin[3 * A + 2];
  float Rt = fminf(Rcap, 2.0f * hmax_t * 1.0001f);
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
      if (u < u1) {
        float4 lo = T.tile_lo[u], hi = T.tile_hi[u];
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
        int64_t uu = ub + j;
        int n_u = T.tile_n[uu];
        int k_j = T.tile_start[uu] + lane;
        bool ok = false;
        float4 sj[NP];
        if (lane < n_u) {
          sj[0] = a.P0[k_j];
          if (NP > 1) sj[1] = a.P1[k_j];
          if (NP > 2) sj[2] = a.P2[k_j];
          sj[0].x -= D0; sj[0].y -= D1; sj[0].z -= D2;
          float R = HYDRO ? fminf(Rcap, 2.0f * fmaxf(hmax_t, sj[0].w) * 1.0001f) : Rt;
          float gx = fmaxf(fmaxf(tlo.x - sj[0].x, sj[0].x - thi.x), 0.0f);
          float gy = fmaxf(fmaxf(tlo.y - sj[0].y, sj[0].y - thi.y), 0.0f);
          float gz = fmaxf(fmaxf(tlo.z - sj[0].z, sj[0].z - thi.z), 0.0f);
          ok = fmaf(gz, gz, fmaf(gy, gy, gx * gx)) <= R * R;
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
#pragma unroll
    for (int b = 0; b < 32; ++b) {
      float4 s = stage[w * 32 + b][0];
      float dx = ti0.x - s.x, dy = ti0.y - s.y, dz = ti0.z - s.z;
      float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
      float thr = thr_i;
      if (HYDRO) {
        float hm = fmaxf(hi, s.w);
        thr = fminf(reach2c, 4.0f * hm * hm * 1.0002f);
      }
      bits |= (r2 <= thr ? 1u : 0u) << b;
    }
    mask[w][lane] = bits;
    nz |= (bits != 0u ? 1u : 0u) << w;
  }
  __syncwarp();
  return nz;
}

// ---------------------------------------------------------------- pass A
__global__ void __launch_bounds__(kSphWarps * 32, 6)
k_sph_density(SphDev a, const int64_t* n_tiles_dev) {
  __shared__ float4 s_stage[kSphWarps][kStageA][1];
  __shared__ int2 s_meta[kSphWarps][kStageA];
  __shared__ unsigned s_mask[kSphWarps][kStageA / 32][32];
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
  double h64 = a.state[row_i * NCOL + C_H];
  double thr4_64 = __dmul_rn(__dmul_rn(4.0, h64), h64);   // (4 h) h as hb/kernels.py:191
  double reach2_64 = __dmul_rn(a.reach, a.reach);
  float thr4 = (float)thr4_64;
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
    walk_masks(mask, nz, [&](int q) {
      float4 s = stage[q][0];
      float dx = ti0.x - s.x, dy = ti0.y - s.y, dz = ti0.z - s.z;
      float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
      bool in = r2 <= a.reach2, c4 = r2 <= thr4;
      bool near_r = fabsf(r2 - a.reach2) <= a.reach2 * a.band;
      bool near_h = fabsf(r2 - thr4) <= thr4 * a.band;
      if (near_r || near_h) {  // exact float64 decision, reference expression
        int2 mt = meta[q];
        double e2 = exact_r2_rows(a.state, a.pshift, a.L, row_i, T.tperm[mt.x], mt.y & 31);
        in = e2 <= reach2_64;
        c4 = e2 <= thr4_64;
      }
      if (in) {
        count += c4 ? 1u : 0u;
        float qq = r2 * rsqrt_ftz(fmaxf(r2, 1e-30f)) * hinv;  // MUFU.RSQ, no IEEE sqrt fix-up
        rho = fmaf(s.w, w_body(qq), rho);
      }
    });
    __syncwarp();
    cnt = 0;
  };
  // cull radius from the tile's largest h (k_tile_boxes: tile_lo.w), not this
  // lane's: every lane culls sources for the whole tile
  sph_sweep<1, false, kStageA>(a, A, e0, e1, tlo, thi, tlo.w, a.reach * 1.0001f, stage, meta,
                               cnt,
                               consume);
  if (live) {
    float norm3 = h > 0.0f ? kSigma * hinv * hinv * hinv : 0.0f;
    a.ncount[row_i] += (double)count;
    a.rho[row_i] += (double)(norm3 * rho);
  }
}

// ---------------------------------------------------------------- pass B
// 5 CTAs / SM (<= 102 registers, no spills): 2.90 -> 2.82 ms at c2 vs the
// compiler's 113-register choice (4 CTAs)
__global__ void __launch_bounds__(kSphWarps * 32, 5)
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
  // records: P0 = (x, y, z, h), P1 = (vx, vy, vz, m), P2 = (P/rho^2, c_s, rho, sigma/h^5)
  float4 ti0 = a.P0[k_i], ti1 = a.P1[k_i], ti2 = a.P2[k_i];
  float hi = ti0.w;
  float hinv = hi > 0.0f ? 1.0f / hi : 0.0f;
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
    unsigned nz =
        build_masks<3, true>(stage, cnt, ti0, live ? hi : -1.0f, 0.0f, live ? reach2c : -1.0f, mask);
    walk_masks(mask, nz, [&](int q) {
      float4 s0 = stage[q][0], s1 = stage[q][1], s2 = stage[q][2];
      float dx = ti0.x - s0.x, dy = ti0.y - s0.y, dz = ti0.z - s0.z;
      float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
      if (!(r2 <= a.reach2)) return;
      float rinv = rsqrt_ftz(fmaxf(r2, 1e-30f));
      float r = r2 * rinv;
      // CRK moments: w = V_j W(r, h_i) (hb/kernels.py:205-220)
      float qi = r * hinv;
      float mj = s1.w;
      float vj = s2.z > 0.0f ? mj * rcp_approx(s2.z) : 0.0f;
      float wk = vj * w_body(qi);
      float wx = wk * dx, wy = wk * dy, wz = wk * dz;
      mo[0] += wk;
      mo[1] -= wx; mo[2] -= wy; mo[3] -= wz;
      mo[4] = fmaf(wx, dx, mo[4]); mo[5] = fmaf(wx, dy, mo[5]); mo[6] = fmaf(wx, dz, mo[6]);
      mo[7] = fmaf(wy, dy, mo[7]); mo[8] = fmaf(wy, dz, mo[8]); mo[9] = fmaf(wz, dz, mo[9]);
      // hydro (hb/kernels.py:227-258), m_i factored out
      float hj = s0.w;
      float qj = r * rcp_approx(hj);
      float gw = 0.5f * (gradw_body(qi) * ti2.w + gradw_body(qj) * s2.w);
      float vx = ti1.x - s1.x, vy = ti1.y - s1.y, vz = ti1.z - s1.z;
      float vdotr = fmaf(vz, dz, fmaf(vy, dy, vx * dx));
      float visc = 0.0f;
      if (vdotr < 0.0f) {
        float hbar = 0.5f * (hi + hj);
        float cbar = 0.5f * (ti2.y + s2.y);
        float rhobar = 0.5f * (ti2.z + s2.z);
        float mu = hbar * vdotr * rcp_approx(fmaf(0.01f * hbar, hbar, r2));
        visc = fmaf(a.beta * mu, mu, -(a.alpha * cbar * mu)) * rcp_approx(rhobar);
      }
      float w = mj * (ti2.x + s2.x + visc) * gw;
      fx = fmaf(-w, dx, fx); fy = fmaf(-w, dy, fy); fz = fmaf(-w, dz, fz);
      float work = mj * vdotr * gw;
      ei = fmaf(fmaf(0.5f, visc, ti2.x), work, ei);
      ej = fmaf(fmaf(0.5f, visc, s2.x), work, ej);
    });
    __syncwarp();
    cnt = 0;
  };
  sph_sweep<3, true, kStageB>(a, A, e0, e1, tlo, thi, tlo.w, a.reach * 1.0001f, stage, meta,
                              cnt,
                              consume);
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

// gas records for both passes
// layout 0 (pass A): P0 = (x, y, z, m), P1 = (.., .., .., h)
// layout 1 (pass B): P0 = (x, y, z, h), P1 = (vx, vy, vz, m), P2 = (P/rho^2, c_s, rho, sigma/h^5)
__global__ void k_pack_sph(int64_t tcap, const int64_t* n_tiles_dev, const Tiling T,
                           const double* state, const int8_t* pshift, double L, float4* P0,
                           float4* P1, float4* P2, int layout) {
  int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (t >= *n_tiles_dev || lane >= T.tile_n[t]) return;
  int leaf = T.tile_leaf[t];
  int64_t k = T.tile_start[t] + lane;
  int64_t r = T.tperm[k];
  const double* st = state + r * NCOL;
  float c[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double v = __dadd_rn(st[d], __dmul_rn((double)(pshift ? pshift[3 * r + d] : 0), L));
    c[d] = (float)(v - T.origin[3 * leaf + d]);
  }
  double h = st[C_H], rho = st[C_RHO];
  double norm5 = h > 0 ? 0.31830988618379067 / (h * h * h * h * h) : 0.0;
  double fpart = rho > 0 ? st[C_P] / (rho * rho) : 0.0;
  if (layout == 0) {
    P0[k] = make_float4(c[0], c[1], c[2], (float)st[C_M]);
    P1[k] = make_float4(0.f, 0.f, 0.f, (float)h);
  } else {
    P0[k] = make_float4(c[0], c[1], c[2], (float)h);
    P1[k] = make_float4((float)st[C_VX], (float)st[C_VY], (float)st[C_VZ], (float)st[C_M]);
    P2[k] = make_float4((float)fpart, (float)st[C_CS], (float)rho, (float)norm5);
  }
}

int pack_sph(const Tiling& T, const int64_t* ntd, const double* state, const int8_t* pshift,
             double L, float4* P0, float4* P1, float4* P2, int layout, cudaStream_t st,
             HbError* err) {
  k_pack_sph<<<grid_for(T.n_tiles_cap * 32, 256), 256, 0, st>>>(T.n_tiles_cap, ntd, T, state,
                                                                pshift, L, P0, P1, P2, layout);
  HB_LAUNCH_CHECK();
  return HB_OK;
}

int launch_sph(int pass, const SphArgs& s, cudaStream_t st, HbError* err) {
  SphDev a;
  a.T = *s.T; a.ent_ptr = s.ent_ptr; a.ent_src = s.ent_src; a.ent_code = s.ent_code;
  a.P0 = s.P0; a.P1 = s.P1; a.P2 = s.P2; a.state = s.state; a.pshift = s.pshift;
  a.L = s.L; a.reach = s.reach; a.reach2 = (float)(s.reach * s.reach); a.band = s.band;
  a.alpha = (float)s.alpha; a.beta = (float)s.beta;
  a.ncount = s.ncount; a.rho = s.rho; a.moments = s.moments; a.hydro = s.hydro;
  a.err_key = s.err_key;
  a.skip_leaf = s.skip_leaf;
  a.skip_tiles = s.skip_tiles;
  unsigned grid = grid_for(s.T->n_tiles_cap, kSphWarps);
  if (pass == 0) k_sph_density<<<grid, kSphWarps * 32, 0, st>>>(a, s.n_tiles_dev);
  else k_sph_force<<<grid, kSphWarps * 32, 0, st>>>(a, s.n_tiles_dev);
  HB_LAUNCH_CHECK();
  return HB_OK;
}

}  // namespace hb
