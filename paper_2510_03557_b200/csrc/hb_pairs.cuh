// hb_pairs.cuh -- pair-kernel physics on FP32 leaf-relative coordinates.
//
// Each policy restates one branch of _pair_phi (hb/kernels.py:143-278) with
// its _fill_partials pieces (hb/kernels.py:102-140), as a per-ordered-pair
// function over packed per-particle float4 records.  Operation counts follow
// the FP32 pipe, not the reference's float64; tolerances are stated in tests.
#pragma once
#include "hb_common.cuh"

namespace hb {
struct Tiling;
}

namespace hb {

enum {
  KID_COUNTING = 0, KID_GRAVITY = 1, KID_GRAV_POT = 2, KID_DENSITY = 3, KID_CRK_MOMENTS = 4,
  KID_HYDRO_FORCE = 5, KID_NEIGHBOR_COUNT = 6, KID_STUB_ZERO = 7, KID_CRK_INTERP = 8,
  KID_CRK_GRAD1 = 9, KID_CRK_GRAD2 = 10
};
enum { C_X = 0, C_Y, C_Z, C_VX, C_VY, C_VZ, C_M, C_H, C_RHO, C_P, C_CS, C_SP, NCOL };

constexpr float kSigma = 0.318309886183790671f;  // 1/pi (hb/kernels.py:63)

// walk this lane's set bits across all words; body(q) per in-support source.
// The warp loops max-over-lanes(total bits) times: balanced over the stage.
// nz = this lane's bitmask of non-empty words (from the mask build), so moving
// to the next word is one predicated step (ffs), never a divergent scan.
template <class Body>
__device__ __forceinline__ void walk_masks(const unsigned (*mask)[32], unsigned nz, Body body) {
  int lane = threadIdx.x & 31;
  int wi = 0;
  unsigned m = 0u;
  while (true) {
    if (m == 0u && nz != 0u) {
      wi = __ffs(nz) - 1;
      nz &= nz - 1;
      m = mask[wi][lane];
    }
    bool has = m != 0u;
    if (!__any_sync(0xffffffffu, has)) break;
    if (has) {
      int q = wi * 32 + __ffs(m) - 1;
      m &= m - 1;
      body(q);
    }
  }
}
// walk_masks taking two set bits of the current word per iteration (the
// second may be absent: q2 = -1), so two independent pair chains are in
// flight per lane
template <class Body2>
__device__ __forceinline__ void walk_masks2(const unsigned (*mask)[32], unsigned nz, Body2 body) {
  int lane = threadIdx.x & 31;
  int wi = 0;
  unsigned m = 0u;
  while (true) {
    if (m == 0u && nz != 0u) {
      wi = __ffs(nz) - 1;
      nz &= nz - 1;
      m = mask[wi][lane];
    }
    bool has = m != 0u;
    if (!__any_sync(0xffffffffu, has)) break;
    if (has) {
      int q1 = wi * 32 + __ffs(m) - 1;
      m &= m - 1;
      int q2 = m ? wi * 32 + __ffs(m) - 1 : -1;
      m &= m - 1;
      body(q1, q2);
    }
  }
}
// MUFU.RSQ without the denormal fix-up rsqrtf() wraps around it (inputs here
// are >= 1e-30, normal in FP32)
__device__ __forceinline__ float rsqrt_ftz(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

struct PairParams {
  float p0, p1;        // kernel params (rs, eps2) or (alpha, beta)
  float inv_rs;
  float reach2;        // reach^2 in FP32
};

// cubic spline body: W(q) h^3/sigma, q < 2 (hb/kernels.py:71-81)
__device__ __forceinline__ float w_body(float q) {
  float t = 2.0f - q;
  float outer = 0.25f * t * t * t;
  float inner = fmaf(q * q, fmaf(0.75f, q, -1.5f), 1.0f);
  return q < 1.0f ? inner : (q < 2.0f ? outer : 0.0f);
}

// (dW/dr)/r * h^5/sigma for the cubic spline (hb/kernels.py:83-93); finite at 0
__device__ __forceinline__ float gradw_body(float q) {
  float t = 2.0f - q;
  float rq;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rq) : "f"(fmaxf(q, 1e-30f)));
  float outer = -0.75f * t * t * rq;
  float inner = fmaf(2.25f, q, -3.0f);
  return q < 1.0f ? inner : (q < 2.0f ? outer : 0.0f);
}

// S(x) = erfc(x) + 2x/sqrt(pi) exp(-x^2) (hb/kernels.py:96-99)
__device__ __forceinline__ float grav_s(float x) {
  return erfcf(x) + 1.1283791670955126f * x * __expf(-x * x);
}

// Policies: NP = float4 records per particle, NC channels, SEL = 1 gas-only.
// pair(): returns phi for target i (ti) and source j (sj) given dx = x_i - x_j.
template <int KID> struct Pol;

template <> struct Pol<KID_COUNTING> {
  static constexpr int NP = 1, NC = 1, SEL = 0;
  static constexpr bool HVAR = false;
  __device__ static void pair(const float4*, const float4*, float, float, float, float,
                              const PairParams&, float* phi) { phi[0] = 1.0f; }
};
template <> struct Pol<KID_STUB_ZERO> {
  static constexpr int NP = 1, NC = 1, SEL = 0;
  static constexpr bool HVAR = false;
  __device__ static void pair(const float4*, const float4*, float, float, float, float,
                              const PairParams&, float* phi) { phi[0] = 0.0f; }
};
// gravity: record P0 = (x, y, z, m)
template <> struct Pol<KID_GRAVITY> {
  static constexpr int NP = 1, NC = 3, SEL = 0;
  static constexpr bool HVAR = false;
  __device__ static void pair(const float4* ti, const float4* sj, float dx, float dy, float dz,
                              float r2, const PairParams& pp, float* phi) {
    float soft = r2 + pp.p1;
    float rinv = rsqrtf(soft);
    float r = r2 > 0.0f ? r2 * rsqrtf(r2) : 0.0f;
    float s = grav_s(r * pp.inv_rs) * (rinv * rinv * rinv);
    float w = (ti[0].w * sj[0].w) * s;
    phi[0] = -(w * dx); phi[1] = -(w * dy); phi[2] = -(w * dz);
  }
};
template <> struct Pol<KID_GRAV_POT> {
  static constexpr int NP = 1, NC = 1, SEL = 0;
  static constexpr bool HVAR = false;
  __device__ static void pair(const float4* ti, const float4* sj, float, float, float, float r2,
                              const PairParams& pp, float* phi) {
    float r = r2 > 0.0f ? r2 * rsqrtf(r2) : 0.0f;
    phi[0] = -(ti[0].w * sj[0].w) * erfcf(r * pp.inv_rs) * rsqrtf(r2 + pp.p1);
  }
};
// density: target P0 = (x,y,z,h), P1.x = sigma/h^3 ; source P0.w = m ... both share layout:
// P0 = (x, y, z, m), P1 = (h, sigma/h^3, 1/h, 0)
template <> struct Pol<KID_DENSITY> {
  static constexpr int NP = 2, NC = 1, SEL = 1;
  static constexpr bool HVAR = true;
  __device__ static void pair(const float4* ti, const float4* sj, float, float, float, float r2,
                              const PairParams&, float* phi) {
    float q = sqrtf(r2) * ti[1].z;
    phi[0] = sj[0].w * (ti[1].y * w_body(q));
  }
};
template <> struct Pol<KID_NEIGHBOR_COUNT> {
  static constexpr int NP = 2, NC = 1, SEL = 1;
  static constexpr bool HVAR = true;
  __device__ static void pair(const float4* ti, const float4*, float, float, float, float r2,
                              const PairParams&, float* phi) {
    float h = ti[1].x;
    phi[0] = r2 <= 4.0f * h * h ? 1.0f : 0.0f;  // exact predicate re-checked in float64 near the edge
  }
};
// CRK moments: source P0.w = V = m/rho (hb/kernels.py:119-121)
template <> struct Pol<KID_CRK_MOMENTS> {
  static constexpr int NP = 2, NC = 10, SEL = 1;
  static constexpr bool HVAR = true;
  __device__ static void pair(const float4* ti, const float4* sj, float dx, float dy, float dz,
                              float r2, const PairParams&, float* phi) {
    float q = sqrtf(r2) * ti[1].z;
    float w = sj[0].w * (ti[1].y * w_body(q));
    phi[0] = w;
    phi[1] = -(w * dx); phi[2] = -(w * dy); phi[3] = -(w * dz);
    float wx = w * dx, wy = w * dy;
    phi[4] = wx * dx; phi[5] = wx * dy; phi[6] = wx * dz;
    phi[7] = wy * dy; phi[8] = wy * dz; phi[9] = (w * dz) * dz;
  }
};
// CRK gradient moments (north star's gradA / gradB; not in the reference):
// G = V_j (dW/dr)/r (h_i) = V_j sigma/h_i^5 gradw(q); dr = x_i - x_j.
// GRAD1: sum G dr (3), sum G dr dr (xx xy xz yy yz zz);  GRAD2: sum G dr dr dr
// (xxx xxy xxz xyy xyz xzz yyy yyz yzz zzz).  P1.w = sigma/h^5 of the target.
template <> struct Pol<KID_CRK_GRAD1> {
  static constexpr int NP = 2, NC = 9, SEL = 1;
  static constexpr bool HVAR = true;
  __device__ static void pair(const float4* ti, const float4* sj, float dx, float dy, float dz,
                              float r2, const PairParams&, float* phi) {
    float q = sqrtf(r2) * ti[1].z;
    float g = sj[0].w * (ti[1].w * gradw_body(q));
    float gx = g * dx, gy = g * dy, gz = g * dz;
    phi[0] = gx; phi[1] = gy; phi[2] = gz;
    phi[3] = gx * dx; phi[4] = gx * dy; phi[5] = gx * dz;
    phi[6] = gy * dy; phi[7] = gy * dz; phi[8] = gz * dz;
  }
};
template <> struct Pol<KID_CRK_GRAD2> {
  static constexpr int NP = 2, NC = 10, SEL = 1;
  static constexpr bool HVAR = true;
  __device__ static void pair(const float4* ti, const float4* sj, float dx, float dy, float dz,
                              float r2, const PairParams&, float* phi) {
    float q = sqrtf(r2) * ti[1].z;
    float g = sj[0].w * (ti[1].w * gradw_body(q));
    float gxx = g * dx * dx, gyy = g * dy * dy, gzz = g * dz * dz, gxy = g * dx * dy;
    phi[0] = gxx * dx; phi[1] = gxx * dy; phi[2] = gxx * dz;
    phi[3] = gyy * dx; phi[4] = gxy * dz; phi[5] = gzz * dx;
    phi[6] = gyy * dy; phi[7] = gyy * dz; phi[8] = gzz * dy; phi[9] = gzz * dz;
  }
};
// hydro: P0 = (x,y,z,m), P1 = (vx,vy,vz,h), P2 = (P/rho^2, c_s, rho, sigma/h^5)
template <> struct Pol<KID_HYDRO_FORCE> {
  static constexpr int NP = 3, NC = 5, SEL = 1;
  static constexpr bool HVAR = true;
  __device__ static void pair(const float4* ti, const float4* sj, float dx, float dy, float dz,
                              float r2, const PairParams& pp, float* phi) {
    float r = sqrtf(r2);
    float hi = ti[1].w, hj = sj[1].w;
    float gi = gradw_body(r * __frcp_rn(hi)) * ti[2].w;
    float gj = gradw_body(r * __frcp_rn(hj)) * sj[2].w;
    float gw = 0.5f * (gi + gj);
    float vx = ti[1].x - sj[1].x, vy = ti[1].y - sj[1].y, vz = ti[1].z - sj[1].z;
    float vdotr = fmaf(vz, dz, fmaf(vy, dy, vx * dx));
    float visc = 0.0f;
    if (vdotr < 0.0f) {
      float hbar = 0.5f * (hi + hj);
      float cbar = 0.5f * (ti[2].y + sj[2].y);
      float rhobar = 0.5f * (ti[2].z + sj[2].z);
      float mu = hbar * vdotr / fmaf(0.01f * hbar, hbar, r2);
      visc = fmaf(pp.p1 * mu, mu, -(pp.p0 * cbar * mu)) / rhobar;
    }
    float mm = ti[0].w * sj[0].w;
    float w = mm * (ti[2].x + sj[2].x + visc) * gw;
    bool z = gw == 0.0f;
    phi[0] = z ? 0.0f : -(w * dx);
    phi[1] = z ? 0.0f : -(w * dy);
    phi[2] = z ? 0.0f : -(w * dz);
    float work = mm * vdotr * gw;
    phi[3] = z ? 0.0f : fmaf(0.5f, visc, ti[2].x) * work;
    phi[4] = z ? 0.0f : fmaf(0.5f, visc, sj[2].x) * work;
  }
};
// corrected interpolation: target P1 = (h, sigma/h^3, 1/h, A), P2 = (Bx, By, Bz, 0);
// source P0.w = V = m/rho, P1.x... source F in P2.w  (aux columns [F, A, Bx, By, Bz])
template <> struct Pol<KID_CRK_INTERP> {
  static constexpr int NP = 3, NC = 1, SEL = 1;
  static constexpr bool HVAR = true;
  __device__ static void pair(const float4* ti, const float4* sj, float dx, float dy, float dz,
                              float r2, const PairParams&, float* phi) {
    float q = sqrtf(r2) * ti[1].z;
    float wk = ti[1].y * w_body(q);
    float corr = ti[1].w * fmaf(ti[2].z, dz, fmaf(ti[2].y, dy, fmaf(ti[2].x, dx, 1.0f)));
    phi[0] = sj[0].w * sj[2].w * corr * wk;
  }
};

constexpr int kTileMax = 32;

// squared distance from a point to an axis-aligned box (0 inside)
__device__ __forceinline__ float box_gap2(float x, float y, float z, float4 lo, float4 hi) {
  float gx = fmaxf(fmaxf(lo.x - x, x - hi.x), 0.0f);
  float gy = fmaxf(fmaxf(lo.y - y, y - hi.y), 0.0f);
  float gz = fmaxf(fmaxf(lo.z - z, z - hi.z), 0.0f);
  return fmaf(gz, gz, fmaf(gy, gy, gx * gx));
}



// Per-leaf tiling of the selected particles (all, or gas only) into spatially
// compact tiles of <= 32 (one warp each); internal order = tile order.
struct Tiling {
  int64_t n_leaves, n_tiles_cap;
  int tile_max = 32;    // members per tile
  int even = 0;         // 1: even tile count per segment (half-warp tile pairs)
  int64_t* sel_cnt;     // (n_leaves+1)
  int64_t* sel_off;     // (n_leaves+1)
  int64_t* tile_cnt;    // (n_leaves+1)
  int64_t* tile_ptr;    // (n_leaves+1)  CSR leaf -> tiles
  int32_t* tperm;       // (n) internal -> state row
  int32_t* tile_start;  // (cap) internal index
  int32_t* tile_n;
  int32_t* tile_leaf;
  float4* tile_lo;      // w = hmax
  float4* tile_hi;
  double* origin;       // (n_leaves,3)
  int* overflow;        // device flag: a leaf exceeded kTileBuildCap
  uint8_t* tile_skip;   // (cap) 1: no owned member (set when built with a ghost array)
};

// Everything one pair-kernel launch reads.
// Row source of the tiling, packing and exact-recheck kernels: the (n,12)
// float64 state matrix the compat API is handed (hb/particles.py:135-154), or
// the resident step's leaf-order SoA fields -- the step keeps no state matrix
// (SURVEY.md 8a row a2); P and c_s then come from density and internal energy
// with the EOS of hb/hydro.py:48-57.  The branch on `st` is warp-uniform.
struct Rows {
  const double* st = nullptr;
  const double *pos = nullptr, *vel = nullptr, *mass = nullptr, *h = nullptr, *rho = nullptr,
               *u = nullptr;
  const uint8_t* sp = nullptr;
  double gamma = 0.0;
  __host__ __device__ static Rows state(const double* s) { Rows r; r.st = s; return r; }
  __device__ __forceinline__ double x(int64_t r, int d) const {
    return st ? st[r * NCOL + d] : pos[3 * r + d];
  }
  __device__ __forceinline__ double v(int64_t r, int d) const {
    return st ? st[r * NCOL + C_VX + d] : vel[3 * r + d];
  }
  __device__ __forceinline__ double m(int64_t r) const { return st ? st[r * NCOL + C_M] : mass[r]; }
  __device__ __forceinline__ double hh(int64_t r) const { return st ? st[r * NCOL + C_H] : h[r]; }
  __device__ __forceinline__ double dens(int64_t r) const {
    return st ? st[r * NCOL + C_RHO] : rho[r];
  }
  __device__ __forceinline__ double pres(int64_t r) const {
    return st ? st[r * NCOL + C_P] : (gamma - 1.0) * rho[r] * u[r];
  }
  __device__ __forceinline__ double snd(int64_t r) const {
    return st ? st[r * NCOL + C_CS] : sqrt(fmax(gamma * (gamma - 1.0) * u[r], 0.0));
  }
  __device__ __forceinline__ bool gas(int64_t r) const {
    return st ? st[r * NCOL + C_SP] == 1.0 : sp[r] == 1;
  }
};

struct EvalDev {
  Tiling T;
  const int64_t* ent_ptr;  // (n_leaves+1)
  const int32_t* ent_src;
  const int32_t* ent_code;  // shift code | fwd << 8 | scatter-eligible << 9
  const float4 *P0, *P1, *P2;
  Rows rows;
  const int8_t* pshift;
  double L, reach;
  PairParams pp;
  float cull_reach;
  int include_self;
  int nchan;
  float scale[10];
  int scatter;               // deterministic mirror: scatter chan_sign * q[mirror_map] to partners
  int csign[10], mmap[10];
  double* out_flt;
  int64_t* out_int;
  int write_out;
  const uint8_t* skip_leaf;  // receivers to skip (ghost-only leaves), or null
  int skip_tiles;            // 1: skip tiles with T.tile_skip set (owned_targets)
  unsigned long long* in_count;
  unsigned long long* err_key;  // min (entry*4 + kind)
};

// ---- internal driver pieces shared by hb_eval_pairs and hb_force_step ----
int64_t tile_capacity(int64_t n, int64_t n_leaves);
void carve_tiling(Arena& ws, int64_t n, int64_t n_leaves, Tiling& T, int tile_max = 32,
                  int even = 0);
__host__ __device__ inline int tiles_for(int m, int tile_max, int even) {
  return even ? 2 * ((m + 2 * tile_max - 1) / (2 * tile_max)) : (m + tile_max - 1) / tile_max;
}
int build_tiling(Tiling& T, int64_t n_leaves, const int64_t* leaf_start, const int64_t* leaf_end,
                 Rows rows, const int8_t* pshift, double L, int sel,
                 int64_t* n_tiles_dev, Arena& ws, cudaStream_t st, HbError* err,
                 const uint8_t* ghost = nullptr);
int pack_records(int kid, const Tiling& T, const int64_t* n_tiles_dev, Rows rows,
                 const int8_t* pshift, const double* aux, int naux, double L, float4* P0,
                 float4* P1, float4* P2, cudaStream_t st, HbError* err);
// lean: resident hot path (no exact counters / per-entry error attribution)
int launch_pairs(int kid, bool det, bool lean, const EvalDev& d, int64_t tile_cap,
                 const int64_t* n_tiles_dev, cudaStream_t st, HbError* err);
int kid_selects_gas(int kid);
// resident fast gravity: table of G(soft) = S(sqrt(soft - eps^2)/r_s) soft^-3/2,
// cubic per interval of soft, 2^jbits intervals per octave (indexed by the
// float bits of soft)
constexpr int kGravSoftBitsMax = 5;
// 32 intervals per octave (cubic fit error ~2e-8 relative; 16 per octave leave
// ~3e-7, which near-cancelling dark-matter lattices amplify past the 1e-5
// relative gate).  The twice larger table runs in 16-warp CTAs so residency
// stays at 32 warps per SM: 10.13 vs 10.04 ms at c2 (HB_GRAV_JBITS=4 selects
// the coarser table).
constexpr int kGravSoftBitsDefault = 5;
constexpr int kGravSoftOctaves = 40;
constexpr int kGravTableMax = (kGravSoftOctaves + 1) * (1 << kGravSoftBitsMax) + 2;
struct GravTab {
  int rows;        // rows to stage in shared memory (the last one is zero)
  unsigned base;   // (bits of the lowest soft) >> (23 - jbits)
  unsigned last;   // zero row index
  int jbits;       // log2(intervals per octave), 4 or 5
};
// host: fill host_out (kGravTableMax rows) and gt; returns rows or -1 (unrepresentable)
int gravity_table(double r_s, double r_cut, double eps, float4* host_out, GravTab* gt);
// cached device copy (library-owned, per device); nullptr + err on failure
const float4* gravity_table_device(double r_s, double r_cut, double eps, GravTab* gt,
                                   cudaStream_t st, HbError* err);
// tiles [*t_begin (0 if null), *ntd)
// ctr (optional): a device counter the launch zeroes and the persistent grid
// hands tiles out from (one per concurrent launch)
int launch_gravity_fast(const EvalDev& d, const float4* table, const GravTab& gt, int64_t tcap,
                        const int64_t* ntd, cudaStream_t st, HbError* err,
                        const int64_t* t_begin = nullptr, unsigned long long* ctr = nullptr);

}  // namespace hb
