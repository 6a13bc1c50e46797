// hb_pairs.cu -- the leaf-pair evaluation engine (replaces eval_pairs_core,
// hb/kernels.py:281-392, behind hb_eval_pairs in include/hb.h).
//
// Layout (all device-resident, built per call from the reference-order state):
//   * the list is expanded (mirror mode: + reversed entries, so every ordered
//     pair is gathered on its receiving side -- no scatter, no atomics) and
//     grouped by receiver leaf with a stable radix sort (deterministic order);
//   * every leaf's selected particles (all, or gas only for the SPH kernels
//     whose phi vanishes off gas-gas pairs, hb/kernels.py:171,188,194,223,260)
//     are cut into spatially compact tiles of <= 32 by proportional median
//     splits: the receiving tile maps onto one warp, lane = target;
//   * coordinates are FP32 relative to a per-leaf float64 origin; the
//     separation of a listed image is dx = x_i - (x_j - D) with
//     D = f32(o_A - o_B - s L)  ==  (pos_i - pos_j) + tau L  of hb/kernels.py:346-355;
//   * per entry, source tiles are culled against the target tile box, then
//     per source; survivors are staged in shared memory and broadcast;
//   * integer outputs (counting, neighbour counts, pairs_in_reach) decide the
//     reach / 4h^2 predicates in float64 with the reference's exact expression
//     whenever the FP32 r^2 falls within 2^-12 of the threshold.
#include <mutex>

#include "hb_pairs.cuh"

namespace hb {

constexpr int kTileBuildBlock = 256;
constexpr int kTileBuildCap = 2048;  // selected members per leaf held in shared memory
constexpr int kTileWarpCapBlock = 384;  // leaves up to this many go to the warp kernel
constexpr int kEvalWarps = 4;
constexpr int kStage = 64;           // staged sources per warp



// ---------------------------------------------------------------- tiling
// Segment origins on a global grid of q = 2^(ilogb(L) - 23): the difference of
// two origins minus a periodic shift s L (L a multiple of q, as for L = 1) is a
// multiple of q below 2 L, so the per-entry FP32 offset D = (o_A - o_B) - s L
// the interaction kernels apply to a whole source segment is exact.  A rounded
// D would move every source of that segment by up to half an ulp of D
// together -- a coherent error, unlike the independent per-record roundings;
// it was the largest FP32 error term of the lattice gravity.
__device__ __forceinline__ double grid_origin(double o, double L) {
  if (!(L > 0.0) || !isfinite(L)) return o;
  double q = ldexp(1.0, ilogb(L) - 23);
  return rint(o / q) * q;
}

__global__ void k_tile_count(int64_t n_leaves, const int64_t* leaf_start, const int64_t* leaf_end,
                             Rows rows, int sel, int64_t* sel_cnt, int64_t* tile_cnt,
                             int tile_max, int even) {
  int64_t leaf = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (leaf >= n_leaves) return;
  int64_t s = leaf_start[leaf], e = leaf_end[leaf];
  int c = 0;
  for (int64_t r = s + lane; r < e; r += 32) c += (sel == 0 || rows.gas(r));
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) {
    sel_cnt[leaf] = c;
    tile_cnt[leaf] = tiles_for(c, tile_max, even);
  }
}

__device__ __forceinline__ double bin_coord(double p, int8_t s, double L) {
  return __dadd_rn(p, __dmul_rn((double)s, L));
}

// a tile's box (FP32, segment frame, exactly as the members' coordinates
// were computed for the splits) with the members' largest h in lo.w and the
// first record index in hi.w, and its owned-target skip flag: emitted by the
// builders as each tile is cut (no separate pass over the state rows).
// Called by one full warp; lanes < m hold members (c = frame coordinates, r =
// state row).
__device__ __forceinline__ void emit_tile_box(Tiling& T, int64_t t, int start, int m, bool have,
                                              float cx, float cy, float cz, int64_t r,
                                              const Rows& rows, const uint8_t* ghost) {
  float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  float hm = 0.0f;
  bool own = false;
  if (have) {
    lo[0] = hi[0] = cx; lo[1] = hi[1] = cy; lo[2] = hi[2] = cz;
    hm = (float)rows.hh(r);
    own = ghost && ghost[r] == 0;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      lo[d] = fminf(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
      hi[d] = fmaxf(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
    }
    hm = fmaxf(hm, __shfl_xor_sync(0xffffffffu, hm, o));
  }
  unsigned ob = __ballot_sync(0xffffffffu, own);
  if ((threadIdx.x & 31) == 0) {
    T.tile_lo[t] = make_float4(lo[0], lo[1], lo[2], hm);
    // .w carries the tile's first record index (int bits): the culling loops
    // read it with the box, so a passing tile needs no dependent load of
    // tile_start before its records
    T.tile_hi[t] = make_float4(hi[0], hi[1], hi[2], __int_as_float(start));
    T.tile_skip[t] = (ghost && ob == 0u) ? 1 : 0;
  }
}

__global__ void __launch_bounds__(kTileBuildBlock)
k_tile_build(Tiling T, const int64_t* leaf_start, const int64_t* leaf_end, Rows rows,
             const int8_t* pshift, double L, int sel, const uint8_t* ghost) {
  __shared__ int32_t s_row[kTileBuildCap];
  __shared__ int32_t s_tmp[kTileBuildCap];
  __shared__ float s_c[3][kTileBuildCap];
  __shared__ int32_t s_flag_scan[kTileBuildBlock];
  __shared__ double red[2][3][kTileBuildBlock / 32];
  __shared__ double org[3];
  __shared__ int stk_a[64], stk_m[64], stk_k[64];
  __shared__ int sp_sh, tile_j;
  __shared__ float seg_ext[3][2][kTileBuildBlock / 32];
  int64_t leaf = blockIdx.x;
  int64_t s = leaf_start[leaf], e = leaf_end[leaf];
  int m_sel = (int)T.sel_cnt[leaf];
  if (m_sel == 0) {
    if (threadIdx.x < 3) T.origin[3 * leaf + threadIdx.x] = 0.0;
    return;
  }
  if (m_sel <= kTileWarpCapBlock) return;  // k_tile_build_warp's leaves
  if (m_sel > kTileBuildCap) {
    if (threadIdx.x == 0) atomicExch(T.overflow, 1);
    return;
  }
  // 1. compact selected rows in row order
  int base = 0;
  for (int64_t r0 = s; r0 < e; r0 += blockDim.x) {
    int64_t r = r0 + threadIdx.x;
    int f = r < e && (sel == 0 || rows.gas(r));
    // block exclusive scan of f
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned b = __ballot_sync(0xffffffffu, f);
    int wpre = __popc(b & lanemask_lt());
    if (lane == 0) s_flag_scan[wid] = __popc(b);
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      int c = s_flag_scan[w];
      if (w < wid) before += c;
      total += c;
    }
    if (f) s_row[base + before + wpre] = (int32_t)r;
    base += total;
    __syncthreads();
  }
  // 2. origin = midpoint of the selected binning positions (float64)
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int k = threadIdx.x; k < m_sel; k += blockDim.x) {
    int64_t r = s_row[k];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      double v = bin_coord(rows.x(r, d), pshift ? pshift[3 * r + d] : (int8_t)0, L);
      mn[d] = fmin(mn[d], v); mx[d] = fmax(mx[d], v);
    }
  }
#pragma unroll
  for (int d = 0; d < 3; ++d)
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      mn[d] = fmin(mn[d], __shfl_xor_sync(0xffffffffu, mn[d], o));
      mx[d] = fmax(mx[d], __shfl_xor_sync(0xffffffffu, mx[d], o));
    }
  {
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0)
      for (int d = 0; d < 3; ++d) { red[0][d][wid] = mn[d]; red[1][d][wid] = mx[d]; }
    __syncthreads();
    if (threadIdx.x < 3) {
      int d = threadIdx.x;
      double a = red[0][d][0], b = red[1][d][0];
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { a = fmin(a, red[0][d][w]); b = fmax(b, red[1][d][w]); }
      org[d] = grid_origin(0.5 * (a + b), L);
      T.origin[3 * leaf + d] = org[d];
    }
    __syncthreads();
  }
  for (int k = threadIdx.x; k < m_sel; k += blockDim.x) {
    int64_t r = s_row[k];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      double v = bin_coord(rows.x(r, d), pshift ? pshift[3 * r + d] : (int8_t)0, L);
      s_c[d][k] = (float)(v - org[d]);
    }
  }
  int ntiles = tiles_for(m_sel, T.tile_max, T.even);
  if (threadIdx.x == 0) { sp_sh = 1; stk_a[0] = 0; stk_m[0] = m_sel; stk_k[0] = ntiles; tile_j = 0; }
  __syncthreads();
  // 3. proportional median splits into ntiles tiles of <= 32 (DFS left-first)
  while (true) {
    int sp = sp_sh;
    if (sp == 0) break;
    int a0 = stk_a[sp - 1], m = stk_m[sp - 1], kk = stk_k[sp - 1];
    __syncthreads();
    if (kk == 1) {
      int64_t t = T.tile_ptr[leaf] + tile_j;
      if (threadIdx.x < 32) {
        bool have = (int)threadIdx.x < m;
        int k = a0 + (have ? (int)threadIdx.x : 0);
        emit_tile_box(T, t, (int)(T.sel_off[leaf] + a0), m, have, s_c[0][k], s_c[1][k],
                      s_c[2][k], s_row[k], rows, ghost);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        T.tile_start[t] = (int32_t)(T.sel_off[leaf] + a0);
        T.tile_n[t] = m;
        T.tile_leaf[t] = (int32_t)leaf;
        tile_j += 1;
        sp_sh = sp - 1;
      }
      __syncthreads();
      continue;
    }
    // longest axis of this segment (FP32)
    float lo3[3] = {INFINITY, INFINITY, INFINITY}, hi3[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int k = threadIdx.x; k < m; k += blockDim.x)
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        float v = s_c[d][a0 + k];
        lo3[d] = fminf(lo3[d], v); hi3[d] = fmaxf(hi3[d], v);
      }
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        lo3[d] = fminf(lo3[d], __shfl_xor_sync(0xffffffffu, lo3[d], o));
        hi3[d] = fmaxf(hi3[d], __shfl_xor_sync(0xffffffffu, hi3[d], o));
      }
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane == 0)
      for (int d = 0; d < 3; ++d) { seg_ext[d][0][wid] = lo3[d]; seg_ext[d][1][wid] = hi3[d]; }
    __syncthreads();
    float ex[3];
    for (int d = 0; d < 3; ++d) {
      float a = seg_ext[d][0][0], b = seg_ext[d][1][0];
      for (int w = 1; w < nw; ++w) { a = fminf(a, seg_ext[d][0][w]); b = fmaxf(b, seg_ext[d][1][w]); }
      ex[d] = b - a;
    }
    int axis = ex[1] > ex[0] ? 1 : 0;
    if (ex[2] > ex[axis]) axis = 2;
    // rank sort of the segment by (coord, position): deterministic
    for (int k = threadIdx.x; k < m; k += blockDim.x) {
      float v = s_c[axis][a0 + k];
      int rank = 0;
      for (int q = 0; q < m; ++q) {
        float w = s_c[axis][a0 + q];
        rank += (w < v) || (w == v && q < k);
      }
      s_tmp[a0 + rank] = a0 + k;  // source slot
    }
    __syncthreads();
    // apply the permutation to rows and coords (via registers)
    int32_t rr[kTileBuildCap / kTileBuildBlock];
    float cc[3][kTileBuildCap / kTileBuildBlock];
    int nloc = 0;
    for (int k = threadIdx.x; k < m; k += blockDim.x, ++nloc) {
      int src = s_tmp[a0 + k];
      rr[nloc] = s_row[src];
      for (int d = 0; d < 3; ++d) cc[d][nloc] = s_c[d][src];
    }
    __syncthreads();
    nloc = 0;
    for (int k = threadIdx.x; k < m; k += blockDim.x, ++nloc) {
      s_row[a0 + k] = rr[nloc];
      for (int d = 0; d < 3; ++d) s_c[d][a0 + k] = cc[d][nloc];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int k1 = (kk + 1) / 2, k2 = kk - k1;
      int left = (int)(((int64_t)m * k1 + kk - 1) / kk);
      stk_a[sp - 1] = a0 + left; stk_m[sp - 1] = m - left; stk_k[sp - 1] = k2;
      stk_a[sp] = a0; stk_m[sp] = left; stk_k[sp] = k1;
      sp_sh = sp + 1;
    }
    __syncthreads();
  }
  // 4. internal order -> state rows
  int64_t so = T.sel_off[leaf];
  for (int k = threadIdx.x; k < m_sel; k += blockDim.x) T.tperm[so + k] = s_row[k];
}

// Same tiling as k_tile_build, one WARP per leaf (leaves with <= 256 selected
// members -- the common case -- without block barriers); larger leaves are
// left to k_tile_build (flagged by big != 0).
// members per warp-built segment (larger segments: the block kernel).  384:
// 71 registers / 30 KB per 4-warp block; 512 (96 registers, 40 KB) took
// 645 us for the two c2 tilings, 384 takes 554 us, and 320 is equal at c2 but
// sends more of c3's clustered bins to the slower block kernel
constexpr int kTileWarpCap = 384;
constexpr int kTileWarps = 4;
__global__ void __launch_bounds__(kTileWarps * 32)
k_tile_build_warp(Tiling T, const int64_t* leaf_start, const int64_t* leaf_end,
                  Rows rows, const int8_t* pshift, double L, int sel, int nl,
                  const uint8_t* ghost) {
  __shared__ int32_t s_row[kTileWarps][kTileWarpCap];
  __shared__ int32_t s_tmp[kTileWarps][kTileWarpCap];
  __shared__ float s_c[kTileWarps][3][kTileWarpCap];
  int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t leaf = (int64_t)blockIdx.x * kTileWarps + wid;
  if (leaf >= nl) return;
  int m_sel = (int)T.sel_cnt[leaf];
  if (m_sel > kTileWarpCap) return;  // handled by the block kernel
  if (m_sel == 0) {
    if (lane < 3) T.origin[3 * leaf + lane] = 0.0;
    return;
  }
  int32_t* row = s_row[wid];
  int32_t* tmp = s_tmp[wid];
  float (*cc)[kTileWarpCap] = s_c[wid];
  int64_t s = leaf_start[leaf], e = leaf_end[leaf];
  int base = 0;
  for (int64_t r0 = s; r0 < e; r0 += 32) {
    int64_t r = r0 + lane;
    bool f = r < e && (sel == 0 || rows.gas(r));
    unsigned b = __ballot_sync(0xffffffffu, f);
    if (f) row[base + __popc(b & lanemask_lt())] = (int32_t)r;
    base += __popc(b);
  }
  __syncwarp();
  constexpr int J = kTileWarpCap / 32;  // members per lane in the split loop
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int k = lane; k < m_sel; k += 32) {
    int64_t r = row[k];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      double v = bin_coord(rows.x(r, d), pshift ? pshift[3 * r + d] : (int8_t)0, L);
      mn[d] = fmin(mn[d], v); mx[d] = fmax(mx[d], v);
    }
  }
  double org[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      mn[d] = fmin(mn[d], __shfl_xor_sync(0xffffffffu, mn[d], o));
      mx[d] = fmax(mx[d], __shfl_xor_sync(0xffffffffu, mx[d], o));
    }
    org[d] = grid_origin(0.5 * (mn[d] + mx[d]), L);
  }
  if (lane < 3) T.origin[3 * leaf + lane] = org[lane];
  for (int k = lane; k < m_sel; k += 32) {  // second pass (L1-hot): leaf-frame FP32
    int64_t r = row[k];
#pragma unroll
    for (int d = 0; d < 3; ++d)
      cc[d][k] = (float)(bin_coord(rows.x(r, d), pshift ? pshift[3 * r + d] : (int8_t)0, L) -
                         org[d]);
  }
  __syncwarp();
  // proportional median splits into ceil(m/32) tiles (DFS left-first).  The
  // coordinates stay put; each split permutes the member order `ord` (kept in
  // the row buffer's twin) with a stable median partition: the `left` smallest
  // (key, position) members go first, in position order.  K = the left-th
  // smallest key by radix descent (32 warp-reduced counting passes over
  // register-held keys), ties at K by position: O(m) per level.
  int32_t* ord = tmp;
  for (int k = lane; k < m_sel; k += 32) ord[k] = k;
  __syncwarp();
  int stk_a[24], stk_m[24], stk_k[24];  // warp-uniform stack
  int sp = 1, tile_j = 0;
  stk_a[0] = 0; stk_m[0] = m_sel; stk_k[0] = tiles_for(m_sel, T.tile_max, T.even);
  int64_t tbase = T.tile_ptr[leaf], so = T.sel_off[leaf];
  unsigned lt = lanemask_lt();
  while (sp) {
    --sp;
    int a0 = stk_a[sp], m = stk_m[sp], kk = stk_k[sp];
    if (kk == 1) {
      int64_t t = tbase + tile_j;
      {
        bool have = lane < m;
        int id = have ? ord[a0 + lane] : 0;
        emit_tile_box(T, t, (int)(so + a0), m, have, cc[0][id], cc[1][id], cc[2][id], row[id],
                      rows, ghost);
      }
      if (lane == 0) {
        T.tile_start[t] = (int32_t)(so + a0);
        T.tile_n[t] = m;
        T.tile_leaf[t] = (int32_t)leaf;
      }
      ++tile_j;
      continue;
    }
    int id[J];
    float lo3[3] = {INFINITY, INFINITY, INFINITY}, hi3[3] = {-INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int jj = 0; jj < J; ++jj) {
      int k = 32 * jj + lane;
      id[jj] = k < m ? ord[a0 + k] : 0;
      if (32 * jj >= m) continue;
      if (k < m)
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          float x = cc[d][id[jj]];
          lo3[d] = fminf(lo3[d], x); hi3[d] = fmaxf(hi3[d], x);
        }
    }
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        lo3[d] = fminf(lo3[d], __shfl_xor_sync(0xffffffffu, lo3[d], o));
        hi3[d] = fmaxf(hi3[d], __shfl_xor_sync(0xffffffffu, hi3[d], o));
      }
    float ex0 = hi3[0] - lo3[0], ex1 = hi3[1] - lo3[1], ex2 = hi3[2] - lo3[2];
    int axis = ex1 > ex0 ? 1 : 0;
    if (ex2 > (axis ? ex1 : ex0)) axis = 2;
    int k1 = (kk + 1) / 2, k2 = kk - k1;
    int left = (int)(((int64_t)m * k1 + kk - 1) / kk);
    const int nj = (m + 31) >> 5;  // warp-uniform: slots in use
    // 16-bit keys: the coordinate along the split axis quantised over the
    // segment's extent (monotone; ties -- also merged neighbours -- are split
    // by position, so the left part still holds exactly `left` members):
    // at most 16 descent passes instead of 32 for sign-straddling floats
    float qlo = axis == 0 ? lo3[0] : axis == 1 ? lo3[1] : lo3[2];
    float qex = axis == 0 ? ex0 : axis == 1 ? ex1 : ex2;
    float qsc = qex > 0.0f ? 65535.0f / qex : 0.0f;
    unsigned key[J];
    unsigned kmin = 0xffffffffu, kmax = 0u;
#pragma unroll
    for (int jj = 0; jj < J; ++jj) {
      bool v = 32 * jj + lane < m;
      float qv = fminf(fmaxf((cc[axis][id[jj]] - qlo) * qsc, 0.0f), 65535.0f);
      key[jj] = v ? (qv == qv ? (unsigned)qv : 65535u) : 0xffffffffu;
      if (v) { kmin = min(kmin, key[jj]); kmax = max(kmax, key[jj]); }
    }
    kmin = __reduce_min_sync(0xffffffffu, kmin);
    kmax = __reduce_max_sync(0xffffffffu, kmax);
    // bits above the highest one where kmin and kmax differ are common to all
    int top = 31 - __clz(kmin ^ kmax | 1u);
    unsigned K = top >= 31 ? 0u : (kmin >> (top + 1)) << (top + 1);
    // radix-4 descent: three candidates per pass, their counts packed in
    // 10-bit fields of one warp reduction (counts <= 384), so half the passes
    // of the binary descent -- the same K (two binary steps pick the largest
    // of K, K+1, K+2, K+3 (x 2^(b-1)) whose count stays below `left`)
    int b = top;
    if ((top + 1) & 1) {  // odd number of bits: one binary step first
      unsigned cand = K | (1u << b);
      int c = 0;
#pragma unroll
      for (int jj = 0; jj < J; ++jj)
        if (jj < nj) c += key[jj] < cand ? 1 : 0;  // padding keys are 0xffffffff
      if (__reduce_add_sync(0xffffffffu, c) < left) K = cand;
      --b;
    }
    for (; b >= 1; b -= 2) {
      unsigned c1 = K | (1u << (b - 1)), c2 = K | (2u << (b - 1)), c3 = K | (3u << (b - 1));
      int c = 0;
#pragma unroll
      for (int jj = 0; jj < J; ++jj)
        if (jj < nj) {
          unsigned kj = key[jj];
          c += (kj < c1 ? 1 : 0) + (kj < c2 ? 1 << 10 : 0) + (kj < c3 ? 1 << 20 : 0);
        }
      int tot = __reduce_add_sync(0xffffffffu, c);
      int n1 = tot & 1023, n2 = (tot >> 10) & 1023, n3 = (tot >> 20) & 1023;
      K = n3 < left ? c3 : (n2 < left ? c2 : (n1 < left ? c1 : K));
    }
    int c_lt = 0;
#pragma unroll
    for (int jj = 0; jj < J; ++jj)
      if (jj < nj) c_lt += key[jj] < K ? 1 : 0;
    int need_eq = left - __reduce_add_sync(0xffffffffu, c_lt);
    int eq_seen = 0, nl_run = 0, nr_run = 0;
    __syncwarp();
#pragma unroll
    for (int jj = 0; jj < J; ++jj) {
      if (jj < nj) {
        bool valid = 32 * jj + lane < m;
        bool eq = valid && key[jj] == K;
        unsigned be = __ballot_sync(0xffffffffu, eq);
        bool isl = valid && (key[jj] < K || (eq && eq_seen + __popc(be & lt) < need_eq));
        eq_seen += __popc(be);
        unsigned bl = __ballot_sync(0xffffffffu, isl), bv = __ballot_sync(0xffffffffu, valid);
        if (isl) ord[a0 + nl_run + __popc(bl & lt)] = id[jj];
        else if (valid) ord[a0 + left + nr_run + __popc(bv & ~bl & lt)] = id[jj];
        nl_run += __popc(bl);
        nr_run += __popc(bv & ~bl);
      }
    }
    __syncwarp();
    stk_a[sp] = a0 + left; stk_m[sp] = m - left; stk_k[sp] = k2; ++sp;   // right (popped last)
    stk_a[sp] = a0; stk_m[sp] = left; stk_k[sp] = k1; ++sp;              // left first
  }
  for (int k = lane; k < m_sel; k += 32) T.tperm[so + k] = row[ord[k]];
}

// ---------------------------------------------------------------- packing
__global__ void k_pack(int kid, int64_t n_tiles_cap, const int64_t* n_tiles_dev, const Tiling T,
                       Rows rows, const int8_t* pshift, const double* aux, int naux,
                       double L, float4* P0, float4* P1, float4* P2) {
  int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (t >= *n_tiles_dev) return;
  if (lane >= T.tile_n[t]) return;
  int leaf = T.tile_leaf[t];
  int64_t k = T.tile_start[t] + lane;
  int64_t r = T.tperm[k];
  float c[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double v = bin_coord(rows.x(r, d), pshift ? pshift[3 * r + d] : (int8_t)0, L);
    c[d] = (float)(v - T.origin[3 * leaf + d]);
  }
  double m = rows.m(r);
  if (kid == KID_GRAVITY || kid == KID_GRAV_POT || kid == KID_COUNTING ||
      kid == KID_STUB_ZERO) {  // position + mass records only
    P0[k] = make_float4(c[0], c[1], c[2], (float)m);
    return;
  }
  double h = rows.hh(r), rho = rows.dens(r);
  double sig = 0.31830988618379067;
  double norm3 = h > 0 ? sig / (h * h * h) : 0.0;
  double hinv = h > 0 ? 1.0 / h : 0.0;
  double vol = rho > 0 ? m / rho : 0.0;
  switch (kid) {
    case KID_DENSITY:
    case KID_NEIGHBOR_COUNT:
      P0[k] = make_float4(c[0], c[1], c[2], (float)m);
      P1[k] = make_float4((float)h, (float)norm3, (float)hinv, 0.0f);
      break;
    case KID_CRK_MOMENTS:
    case KID_CRK_GRAD1:
    case KID_CRK_GRAD2: {
      double n5 = h > 0 ? sig / (h * h * h * h * h) : 0.0;
      P0[k] = make_float4(c[0], c[1], c[2], (float)vol);
      P1[k] = make_float4((float)h, (float)norm3, (float)hinv, (float)n5);
      break;
    }
    case KID_HYDRO_FORCE: {
      double fpart = rho > 0 ? rows.pres(r) / (rho * rho) : 0.0;
      double norm5 = h > 0 ? sig / (h * h * h * h * h) : 0.0;
      P0[k] = make_float4(c[0], c[1], c[2], (float)m);
      P1[k] = make_float4((float)rows.v(r, 0), (float)rows.v(r, 1), (float)rows.v(r, 2), (float)h);
      P2[k] = make_float4((float)fpart, (float)rows.snd(r), (float)rho, (float)norm5);
      break;
    }
    case KID_CRK_INTERP: {
      const double* ax = aux + r * naux;
      P0[k] = make_float4(c[0], c[1], c[2], (float)vol);
      P1[k] = make_float4((float)h, (float)norm3, (float)hinv, (float)ax[1]);
      P2[k] = make_float4((float)ax[2], (float)ax[3], (float)ax[4], (float)ax[0]);
      break;
    }
    default:
      P0[k] = make_float4(c[0], c[1], c[2], (float)m);
  }
}

// ---------------------------------------------------------------- entry CSR
__global__ void k_expand(int64_t n_pairs, int mirror, const int64_t* pa, const int64_t* pb,
                         const int8_t* ps, const int64_t* rev_off, uint64_t* keys, uint32_t* vals,
                         int32_t* e_src, int32_t* e_code, int32_t* e_orig) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_pairs) return;
  int64_t a = pa[i], b = pb[i];
  int sx = ps[3 * i], sy = ps[3 * i + 1], sz = ps[3 * i + 2];
  int code = (sx + 1) * 9 + (sy + 1) * 3 + (sz + 1);
  keys[i] = (uint64_t)a; vals[i] = (uint32_t)i;
  // mirror 2 (deterministic): no reversed entries; partners of a != b or
  // shifted entries receive the mirrored quanta by scatter (bit 9)
  int scat = (mirror == 2 && (a != b || code != 13)) ? (1 << 9) : 0;
  e_src[i] = (int32_t)b; e_code[i] = code | (1 << 8) | scat; e_orig[i] = (int32_t)i;
  if (mirror == 1 && (a != b || code != 13)) {
    int64_t j = n_pairs + rev_off[i];
    keys[j] = (uint64_t)b; vals[j] = (uint32_t)j;
    e_src[j] = (int32_t)a; e_code[j] = 26 - code; e_orig[j] = (int32_t)i;
  }
}
__global__ void k_rev_flags(int64_t n_pairs, const int64_t* pa, const int64_t* pb,
                            const int8_t* ps, int64_t* flag) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_pairs) return;
  bool shifted = ps[3 * i] != 0 || ps[3 * i + 1] != 0 || ps[3 * i + 2] != 0;
  flag[i] = (pa[i] != pb[i] || shifted) ? 1 : 0;
}
__global__ void k_recv_hist(int64_t E, const uint64_t* keys_sorted, int64_t* cnt) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= E) return;
  atomicAdd((unsigned long long*)&cnt[keys_sorted[i]], 1ull);
}
__global__ void k_gather_entries(int64_t E, const uint32_t* vals, const int32_t* src,
                                 const int32_t* code, const int32_t* orig, int32_t* o_src,
                                 int32_t* o_code, int32_t* o_orig) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= E) return;
  uint32_t v = vals[i];
  o_src[i] = src[v]; o_code[i] = code[v]; o_orig[i] = orig[v];
}

// FLOP-proxy counters of the lane-split schedule (hb/kernels.py:319-343)
__global__ void k_sched_counters(int64_t n_pairs, const int64_t* pa, const int64_t* pb,
                                 const int64_t* ls, const int64_t* le, int W2,
                                 unsigned long long* cnt) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long f = 0, g = 0;
  if (i < n_pairs) {
    int64_t na = le[pa[i]] - ls[pa[i]], nb = le[pb[i]] - ls[pb[i]];
    int64_t nit = (na + W2 - 1) / W2, njt = (nb + W2 - 1) / W2;
    f = (unsigned long long)nit;
    g = (unsigned long long)(nit * njt);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    f += __shfl_xor_sync(0xffffffffu, f, o);
    g += __shfl_xor_sync(0xffffffffu, g, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&cnt[0], f);
    atomicAdd(&cnt[1], g);
  }
}

// ---------------------------------------------------------------- the gather kernel



// exact float64 separation of rows i, j for image code (hb/kernels.py:346-356)
__device__ __forceinline__ double exact_r2(const EvalDev& a, int64_t i, int64_t j, int code) {
  int s[3] = {code / 9 - 1, (code / 3) % 3 - 1, code % 3 - 1};
  double r2 = 0.0;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    int64_t pi = a.pshift ? a.pshift[3 * i + d] : 0, pj = a.pshift ? a.pshift[3 * j + d] : 0;
    int64_t tau = pi - pj - s[d];
    double dx = __dadd_rn(__dsub_rn(a.rows.x(i, d), a.rows.x(j, d)),
                          __dmul_rn((double)tau, a.L));
    r2 = d == 0 ? __dmul_rn(dx, dx) : __dadd_rn(r2, __dmul_rn(dx, dx));
  }
  return r2;
}

// LEAN (resident hot path): no float64 reach recheck (only the integer kernel
// keeps it), no index-based self test (r = 0 terms vanish or are included by
// the kernel's own definition), no pairs_in_reach tally, staged sources are
// flushed only when the stage fills, finiteness checked once at the end.
template <int KID, bool DET, bool LEAN>
__global__ void __launch_bounds__(kEvalWarps * 32) k_eval(EvalDev a, int64_t n_tiles_cap,
                                                          const int64_t* n_tiles_dev) {
  using P = Pol<KID>;
  constexpr int NP = P::NP, NC = P::NC;
  __shared__ float4 s_rec[kEvalWarps][kStage][NP];
  __shared__ int2 s_meta[kEvalWarps][kStage];
  int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t t = (int64_t)blockIdx.x * kEvalWarps + wid;
  if (t >= *n_tiles_dev) return;
  const Tiling& T = a.T;
  int A = T.tile_leaf[t];
  int64_t e0 = a.ent_ptr[A], e1 = a.ent_ptr[A + 1];
  if (e0 == e1) return;
  int n_t = T.tile_n[t];
  bool live = lane < n_t;
  int k_i = T.tile_start[t] + (live ? lane : 0);
  int64_t row_i = T.tperm[k_i];
  float4 ti[NP];
  ti[0] = a.P0[k_i];
  if (NP > 1) ti[1] = a.P1[k_i];
  if (NP > 2) ti[2] = a.P2[k_i];
  float4 tlo = T.tile_lo[t], thi = T.tile_hi[t];
  float hmax_t = tlo.w;
  float Rt = a.cull_reach;
  if (P::HVAR && KID != KID_HYDRO_FORCE) Rt = fminf(Rt, 2.0f * hmax_t * 1.0001f);
  float acc[NC];
  long long iacc[DET ? NC : 1];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = 0.0f;
#pragma unroll
  for (int c = 0; c < (DET ? NC : 1); ++c) iacc[c] = 0;
  unsigned long long nin = 0;
  double oA[3] = {T.origin[3 * A], T.origin[3 * A + 1], T.origin[3 * A + 2]};
  float thr_n = 0.0f;
  double thr_n64 = 0.0;
  if (KID == KID_NEIGHBOR_COUNT) {
    double h = a.rows.hh(row_i);
    thr_n64 = __dmul_rn(__dmul_rn(4.0, h), h);
    thr_n = (float)thr_n64;
  }
  double reach2_64 = __dmul_rn(a.reach, a.reach);
  int bad = 0;
  int cnt = 0;
  // evaluate the staged sources against this lane's target
  auto flush = [&]() {
    __syncwarp();
    for (int q = 0; q < cnt; ++q) {
      const float4* rec = s_rec[wid][q];
      int2 meta = s_meta[wid][q];
      float dx = ti[0].x - rec[0].x, dy = ti[0].y - rec[0].y, dz = ti[0].z - rec[0].z;
      float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
      bool in = r2 <= a.pp.reach2;
      int64_t row_j = -1;
      if ((!LEAN || KID == KID_NEIGHBOR_COUNT) && live &&
          fabsf(r2 - a.pp.reach2) <= a.pp.reach2 * 2.44140625e-4f) {
        row_j = T.tperm[meta.x];
        in = exact_r2(a, row_i, row_j, meta.y & 31) <= reach2_64;
      }
      if (!LEAN && !a.include_self && meta.x == k_i && (meta.y & 31) == 13) in = false;
      long long qv[DET ? NC : 1];
#pragma unroll
      for (int c = 0; c < (DET ? NC : 1); ++c) qv[c] = 0;
      if (in) {
        if (!LEAN && live && ((meta.y >> 8) & 1)) nin += 1;
        float phi[NC];
        if (KID == KID_NEIGHBOR_COUNT) {
          bool c4 = r2 <= thr_n;
          if (live && fabsf(r2 - thr_n) <= thr_n * 2.44140625e-4f) {
            if (row_j < 0) row_j = T.tperm[meta.x];
            c4 = exact_r2(a, row_i, row_j, meta.y & 31) <= thr_n64;
          }
          phi[0] = c4 ? 1.0f : 0.0f;
        } else {
          P::pair(ti, rec, dx, dy, dz, r2, a.pp, phi);
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          if (DET) {
            float v = phi[c] * a.scale[c];
            if (!(fabsf(v) <= 7.2057594e16f)) bad |= (v == v && fabsf(v) != INFINITY) ? 2 : 1;
            else qv[c] = __float2ll_rn(v);
            iacc[c] += qv[c];
          } else {
            acc[c] += phi[c];
          }
        }
      }
      // deterministic mirror: the partner row gets chan_sign * q[mirror_map]
      // summed over this warp's live targets, one integer atomic per channel
      // (integer sums are order-independent: still run-to-run deterministic)
      if (DET && !LEAN && a.scatter && ((meta.y >> 9) & 1)) {
        int64_t prow = T.tperm[meta.x];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          long long m = 0;
          if (live && c < a.nchan) {
            int mc = a.mmap[c];
#pragma unroll
            for (int k = 0; k < NC; ++k)
              if (k == mc) m = (long long)a.csign[c] * qv[k];
          }
#pragma unroll
          for (int o = 16; o; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
          if (lane == 0 && m != 0 && c < a.nchan && a.write_out)
            atomicAdd((unsigned long long*)&a.out_int[prow * a.nchan + c], (unsigned long long)m);
        }
      }
    }
    __syncwarp();
    cnt = 0;
  };
  for (int64_t e = e0; e < e1; ++e) {
    int B = a.ent_src[e];
    int cw = a.ent_code[e];
    int code = cw & 31;
    double oB[3] = {T.origin[3 * B], T.origin[3 * B + 1], T.origin[3 * B + 2]};
    int sh[3] = {code / 9 - 1, (code / 3) % 3 - 1, code % 3 - 1};
    float D[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) D[d] = (float)((oA[d] - oB[d]) - (double)sh[d] * a.L);
    int64_t u0 = T.tile_ptr[B], u1 = T.tile_ptr[B + 1];
    for (int64_t ub = u0; ub < u1; ub += 32) {
      int64_t u = ub + lane;
      bool pass = false;
      if (u < u1) {
        float4 lo = T.tile_lo[u], hi = T.tile_hi[u];
        float R = Rt;
        if (KID == KID_HYDRO_FORCE) R = fminf(a.cull_reach, 2.0f * fmaxf(hmax_t, lo.w) * 1.0001f);
        float gx = fmaxf(fmaxf((lo.x - D[0]) - thi.x, tlo.x - (hi.x - D[0])), 0.0f);
        float gy = fmaxf(fmaxf((lo.y - D[1]) - thi.y, tlo.y - (hi.y - D[1])), 0.0f);
        float gz = fmaxf(fmaxf((lo.z - D[2]) - thi.z, tlo.z - (hi.z - D[2])), 0.0f);
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
          sj[0].x -= D[0]; sj[0].y -= D[1]; sj[0].z -= D[2];
          float R = Rt;
          if (KID == KID_HYDRO_FORCE) R = fminf(a.cull_reach, 2.0f * fmaxf(hmax_t, sj[1].w) * 1.0001f);
          ok = box_gap2(sj[0].x, sj[0].y, sj[0].z, tlo, thi) <= R * R;
        }
        unsigned sm = __ballot_sync(0xffffffffu, ok);
        if (cnt + __popc(sm) > kStage) flush();
        if (ok) {
          int slot = cnt + __popc(sm & lanemask_lt());
#pragma unroll
          for (int p = 0; p < NP; ++p) s_rec[wid][slot][p] = sj[p];
          s_meta[wid][slot] = make_int2(k_j, cw);
        }
        cnt += __popc(sm);
      }
    }
    if (!LEAN) {
      flush();  // per entry: keeps error attribution per leaf pair
      if (!DET) {
#pragma unroll
        for (int c = 0; c < NC; ++c) if (!isfinite(acc[c])) bad |= 1;
      }
      unsigned bm = __ballot_sync(0xffffffffu, live && bad);
      if (bm) {
        int kind = __shfl_sync(0xffffffffu, bad, __ffs(bm) - 1);
        if (lane == 0) atomicMin(a.err_key, (unsigned long long)(e * 4 + ((kind & 1) ? 1 : 2)));
        return;
      }
    }
  }
  if (LEAN) {
    flush();
    if (!DET) {
#pragma unroll
      for (int c = 0; c < NC; ++c) if (!isfinite(acc[c])) bad |= 1;
    }
    unsigned bm = __ballot_sync(0xffffffffu, live && bad);
    if (bm) {
      int kind = __shfl_sync(0xffffffffu, bad, __ffs(bm) - 1);
      if (lane == 0) atomicMin(a.err_key, (unsigned long long)(e0 * 4 + ((kind & 1) ? 1 : 2)));
      return;
    }
  }
  if (live && a.write_out) {
    if (DET && !LEAN && a.scatter) {  // partners' scatter lands in these rows concurrently
#pragma unroll
      for (int c = 0; c < NC; ++c)
        if (c < a.nchan && iacc[c] != 0)
          atomicAdd((unsigned long long*)&a.out_int[row_i * a.nchan + c],
                    (unsigned long long)iacc[c]);
    } else if (DET) {
#pragma unroll
      for (int c = 0; c < NC; ++c)
        if (c < a.nchan) a.out_int[row_i * a.nchan + c] += iacc[c];
    } else {
#pragma unroll
      for (int c = 0; c < NC; ++c)
        if (c < a.nchan) a.out_flt[row_i * a.nchan + c] += (double)acc[c];
    }
  }
  if (!LEAN) {
#pragma unroll
    for (int o = 16; o; o >>= 1) nin += __shfl_xor_sync(0xffffffffu, nin, o);
    if (lane == 0 && nin) atomicAdd(a.in_count, nin);
  }
}

// ---------------------------------------------------------------- fast gravity
// Resident-path short-range gravity.  Same tiling, culling and staging as
// k_eval<KID_GRAVITY> (per entry: lane-parallel source-tile box cull, then a
// per-source cull against the target tile box; survivors staged in shared
// memory and broadcast to the 32 target lanes), but the pair function comes
// from a cubic-per-interval table in shared memory and m_i is applied once
// per target.  The table (host fit in float64 at Chebyshev nodes) is indexed
// by the float bits of soft = r^2 + eps^2 (2^JB intervals per octave: index =
// bits >> (23 - JB), in-interval variable = the low 23 - JB mantissa bits as a
// float in [1, 1 + 2^-JB) minus 1) and stores G(soft) = S(sqrt(soft - eps^2) /
// r_s) * soft^{-3/2}.  Sources go in pairs through Blackwell's packed FP32x2
// instructions: per two sources 6 FADD (dx) + 3 FFMA2 (soft) + 2 LEA.HI + 2
// VIMNMX + 2 LOP3 + FADD2 + 2 LEA + 2 LDS + 6 FFMA + 2 FMUL (cubic, m_j) + 3
// FFMA2 (accumulate), no MUFU: 18 SASS instructions per source in the
// 8-source batch loop against 22 scalar (c2: 10.06 -> 9.70 ms).  Fit error ~2e-8
// relative (JB = 5, default) / ~3e-7 (JB = 4).  (Round 1's r- and t-indexed S
// tables -- one or two MUFU and 27 instructions per pair -- were removed.)
// Rows past r_cut (to the end of the interval holding r_cut) carry the smooth
// continuation (|S| <= S(r_cut/r_s) < 1e-5 by the ForceSplit guard); the next
// row is zero.  The resident step launches a persistent grid (2 CTAs per SM)
// whose warps take tiles from a device counter: a one-tile-per-warp grid
// keeps each CTA's slots (and its 66 KB table) until its slowest warp ends,
// and a static-stride persistent grid (round 1) idled warps at the tail;
// with the counter k_gravity went 9.69 -> 9.03 ms at c2, 596 -> 556 ms at c4.
constexpr int kGravWarps = 8;
constexpr int kGravStage = 128;

// (a & b) | c as one LOP3 (ptxas splits it in two when b and c are both
// immediates; here they are loop-invariant registers)
__device__ __forceinline__ unsigned and_or(unsigned a, unsigned b, unsigned c) {
  unsigned d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// 16-B shared-memory load from a 32-bit shared-window byte address
__device__ __forceinline__ float4 lds128(unsigned addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
// s_tab: the table's base (row r, copy j at float4 8 r + j).  A lane reads
// copy lane & 7 of its row through a 32-bit shared-window byte address: row
// offset + this lane's copy offset, clamped to this lane's copy of the zero
// row (soft past r_cut, or below the table, whose index wraps to the top).
// (Measured against the float4-indexed gather: 9.03 -> 8.87 ms at c2, same
// instruction count.  Predicating the out-of-range gathers off cut the
// shared-memory wavefronts 19% but added 10% instructions: 8.96 ms.)
template <int JB, int REP, int kGravBatch>
__device__ __forceinline__ void grav_tile(const EvalDev& a, const float4* s_tab, const GravTab& gt,
                                          float4* stage, int64_t t, int lane) {
  const Tiling& T = a.T;
  int A = T.tile_leaf[t];
  if (a.skip_leaf && a.skip_leaf[A]) return;
  if (a.skip_tiles && T.tile_skip[t]) return;  // owned_targets: no owned member
  int64_t e0 = a.ent_ptr[A], e1 = a.ent_ptr[A + 1];
  if (e0 == e1) return;
  int n_t = T.tile_n[t];
  bool live = lane < n_t;
  int k_i = T.tile_start[t] + (live ? lane : 0);
  float4 ti = a.P0[k_i];
  float4 tlo = T.tile_lo[t], thi = T.tile_hi[t];
  float R2 = a.cull_reach * a.cull_reach;
  float eps2 = a.pp.p1;
  // shared-memory byte addresses: this lane's copy of row 0 and of the zero row
  const unsigned tab_s = (unsigned)__cvta_generic_to_shared(s_tab);
  const unsigned lane_a = tab_s + (((unsigned)lane & (REP - 1)) << 4);
  const unsigned zero_a = lane_a + ((gt.last * REP) << 4);
  float2 eps2x2 = make_float2(eps2, eps2);
  const unsigned lowmask = (1u << (23 - JB)) - 1u, one_bits = 0x3F800000u;
  // even / odd-source running sums (packed pairs), fed with fresh FP32x2
  // partial sums of each 8-source batch: a running sum takes one rounding per
  // batch instead of one per source (the lattice gravity's relative error,
  // dark matter 512^3 median 8.7e-6 -> 6.3e-6 for 3% of the kernel)
  float2 rx = make_float2(0.0f, 0.0f), ry = rx, rz = rx;
  const double* oA = T.origin + 3 * A;  // re-read per entry (L1): 6 registers fewer
  int cnt = 0;
  auto flush = [&]() {
    __syncwarp();
    int q0 = 0;
    {
      // batches of kGravBatch sources: every table row is requested before the
      // first one is used, so the gathers' latency overlaps within the warp
      // (the unrolled per-pair loop stalled on each row: short scoreboard).
      // The order within each accumulator is fixed (deterministic).
      for (; q0 + kGravBatch <= cnt; q0 += kGravBatch) {
        // sources in pairs: soft, u - 1 and the accumulation run as packed
        // FP32x2 instructions (FFMA2 / FADD2, one issue slot for two lanes'
        // worth of a pair of sources); dx, the table index and the cubic stay
        // scalar, their results landing in the pair registers
        float2 bx[kGravBatch / 2], by[kGravBatch / 2], bz[kGravBatch / 2], bu[kGravBatch / 2];
        float bm[kGravBatch];
        float4 bc[kGravBatch];
#pragma unroll
        for (int p = 0; p < kGravBatch / 2; ++p) {
          float4 s0 = stage[q0 + 2 * p], s1 = stage[q0 + 2 * p + 1];
          bx[p] = make_float2(ti.x - s0.x, ti.x - s1.x);
          by[p] = make_float2(ti.y - s0.y, ti.y - s1.y);
          bz[p] = make_float2(ti.z - s0.z, ti.z - s1.z);
          bm[2 * p] = s0.w; bm[2 * p + 1] = s1.w;
          float2 soft = __ffma2_rn(bz[p], bz[p], __ffma2_rn(by[p], by[p], __ffma2_rn(bx[p], bx[p], eps2x2)));
          unsigned b0 = __float_as_uint(soft.x), b1 = __float_as_uint(soft.y);
          unsigned r0 = (b0 >> (23 - JB)) - gt.base, r1 = (b1 >> (23 - JB)) - gt.base;
          float2 um = make_float2(__uint_as_float(and_or(b0, lowmask, one_bits)),
                                  __uint_as_float(and_or(b1, lowmask, one_bits)));
          bu[p] = __fadd2_rn(um, make_float2(-1.0f, -1.0f));
          bc[2 * p] = lds128(min(r0 * (REP * 16) + lane_a, zero_a));
          bc[2 * p + 1] = lds128(min(r1 * (REP * 16) + lane_a, zero_a));
        }
        float2 fx = make_float2(0.0f, 0.0f), fy = fx, fz = fx;
#pragma unroll
        for (int p = 0; p < kGravBatch / 2; ++p) {
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
    float tx = 0.0f, ty = 0.0f, tz = 0.0f;
#pragma unroll 4
    for (int q = q0; q < cnt; ++q) {
      float4 s = stage[q];
      float dx = ti.x - s.x, dy = ti.y - s.y, dz = ti.z - s.z;
      float soft = fmaf(dz, dz, fmaf(dy, dy, fmaf(dx, dx, eps2)));
      unsigned bits = __float_as_uint(soft);
      unsigned k = min(((bits >> (23 - JB)) - gt.base) * (REP * 16) + lane_a, zero_a);
      float u = __uint_as_float((bits & ((1u << (23 - JB)) - 1u)) | 0x3F800000u) - 1.0f;
      float4 c = lds128(k);
      float w = fmaf(fmaf(fmaf(c.w, u, c.z), u, c.y), u, c.x) * s.w;
      tx = fmaf(w, dx, tx);
      ty = fmaf(w, dy, ty);
      tz = fmaf(w, dz, tz);
    }
    rx.x += tx; ry.x += ty; rz.x += tz;
    __syncwarp();
    cnt = 0;
  };
  for (int64_t e = e0; e < e1; ++e) {
    int B = a.ent_src[e];
    if (B < 0) continue;  // bin stencil: off-mesh / duplicate cell
    int code = a.ent_code[e] & 31;
    int sh0 = code / 9 - 1, sh1 = (code / 3) % 3 - 1, sh2 = code % 3 - 1;
    float D0 = (float)((oA[0] - T.origin[3 * B]) - (double)sh0 * a.L);
    float D1 = (float)((oA[1] - T.origin[3 * B + 1]) - (double)sh1 * a.L);
    float D2 = (float)((oA[2] - T.origin[3 * B + 2]) - (double)sh2 * a.L);
    int64_t u0 = T.tile_ptr[B], u1 = T.tile_ptr[B + 1];
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
      unsigned tm = __ballot_sync(0xffffffffu, pass);
      while (tm) {
        int j = __ffs(tm) - 1;
        tm &= tm - 1;
        int n_u = __shfl_sync(0xffffffffu, my_n, j);
        int s_u = __shfl_sync(0xffffffffu, my_start, j);
        bool ok = false;
        float4 sj;
        if (lane < n_u) {
          sj = a.P0[s_u + lane];
          sj.x -= D0; sj.y -= D1; sj.z -= D2;
          ok = box_gap2(sj.x, sj.y, sj.z, tlo, thi) <= R2;
        }
        unsigned sm = __ballot_sync(0xffffffffu, ok);
        if (cnt + 32 > kGravStage) flush();
        if (ok) stage[cnt + __popc(sm & lanemask_lt())] = sj;
        cnt += __popc(sm);
      }
    }
  }
  flush();
  float ax = rx.x + rx.y, ay = ry.x + ry.y, az = rz.x + rz.y;
  bool bad = !(isfinite(ax) && isfinite(ay) && isfinite(az));
  unsigned bm = __ballot_sync(0xffffffffu, live && bad);
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

// REP = 8: the table is held as 8 interleaved copies (row r of copy j at
// float4 index 8 r + j) and lane l reads copy l & 7.  A 16-B gather is served
// in quarter-warp phases of 8 consecutive lanes; with the copies every lane of
// a phase owns one 16-B bank group whatever row it reads, so the gather takes
// the minimum 4 wavefronts instead of 4 + bank conflicts (5.9 measured).
template <int JB, int REP, int NB, int MINB = 4, int WARPS = kGravWarps>
__global__ void __launch_bounds__(WARPS * 32, MINB)
k_gravity(EvalDev a, const float4* __restrict__ table, GravTab gt, const int64_t* n_tiles_dev,
          const int64_t* t_begin_dev, unsigned long long* ctr) {
  extern __shared__ float4 s_tab[];  // gt.rows * REP
  __shared__ float4 s_src[WARPS][kGravStage];
  int64_t tb = t_begin_dev ? *t_begin_dev : 0;
  int64_t t_end = *n_tiles_dev;
  int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (ctr) {
    // persistent: the grid is the resident CTAs; each warp takes the next
    // tile from a counter (zeroed by the launcher), so warps never wait for
    // their CTA's slowest tile and the table is staged once per CTA
    if ((int64_t)blockIdx.x * WARPS + tb >= t_end) return;
    for (int k = threadIdx.x; k < gt.rows * REP; k += blockDim.x) s_tab[k] = table[k / REP];
    __syncthreads();
    while (true) {
      unsigned long long u = 0;
      if (lane == 0) u = atomicAdd(ctr, 1ull);
      int64_t t = tb + (int64_t)__shfl_sync(0xffffffffu, u, 0);
      if (t >= t_end) break;
      grav_tile<JB, REP, NB>(a, s_tab, gt, s_src[wid], t, lane);
      __syncwarp();
    }
    return;
  }
  // the grid covers the tiling's capacity; a range launch (t_begin_dev, a
  // bin-range end in n_tiles_dev) leaves whole CTAs past its end: they leave
  // before loading the 66 KB table
  int64_t t0 = (int64_t)blockIdx.x * WARPS + tb;
  if (t0 >= t_end) return;
  for (int k = threadIdx.x; k < gt.rows * REP; k += blockDim.x) s_tab[k] = table[k / REP];
  __syncthreads();
  int64_t t = t0 + wid;
  if (t < t_end)
    grav_tile<JB, REP, NB>(a, s_tab, gt, s_src[wid], t, lane);
}

template <int JB, int NB, int REP = 8, int MINB = 4, int WARPS = kGravWarps>
static int launch_gravity_kind(const EvalDev& d, const float4* table, const GravTab& gt,
                               int64_t tcap, const int64_t* ntd,
                               const int64_t* t_begin, cudaStream_t st, HbError* err,
                               unsigned long long* ctr) {
  size_t sm = (size_t)gt.rows * REP * sizeof(float4);
  // static staging + dynamic table may pass the 48 KB default: raise the
  // per-kernel limit whenever the table grows (per device and instantiation)
  static std::mutex mu;
  static size_t set_for[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    if (dev >= 0 && dev < 64 && sm > set_for[dev]) {
      HB_CUDA_TRY(cudaFuncSetAttribute(k_gravity<JB, REP, NB, MINB, WARPS>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      set_for[dev] = sm;
    }
  }
  unsigned grid = grid_for(tcap, WARPS), blk = WARPS * 32;
  if (ctr) {  // persistent: MINB resident CTAs per SM
    static int sms[64] = {};
    if (dev >= 0 && dev < 64 && !sms[dev])
      HB_CUDA_TRY(cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev));
    unsigned cap = (unsigned)MINB * (unsigned)(dev >= 0 && dev < 64 ? sms[dev] : 148);
    grid = grid < cap ? grid : cap;
    HB_CUDA_TRY(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), st));
  }
  k_gravity<JB, REP, NB, MINB, WARPS><<<grid, blk, sm, st>>>(d, table, gt, ntd, t_begin, ctr);
  return HB_OK;
}

int launch_gravity_fast(const EvalDev& d, const float4* table, const GravTab& gt, int64_t tcap,
                        const int64_t* ntd, cudaStream_t st, HbError* err,
                        const int64_t* t_begin, unsigned long long* ctr) {
  static int persist = -1;
  if (persist < 0) {  // HB_GRAV_PERSIST: 1 = persistent grid with a tile counter (when given one)
    const char* e = getenv("HB_GRAV_PERSIST");
    persist = e ? atoi(e) != 0 : 1;
  }
  if (!persist) ctr = nullptr;
  // batches of 8 sources per pipelined table gather (1 / 2 / 4: 10.31 / 10.17 /
  // 10.15 ms against 10.04 ms at c2 in round 1); 8 interleaved table copies.
  // The 32-per-octave table (default) is twice the 8-copy footprint (~70 KB):
  // 16-warp CTAs keep 2 x 16 = 32 resident warps per SM, as 4 x 8 for JB = 4.
  // (Round 1's fewer-copy / higher-occupancy variants were all slower and are
  // gone.)
  int rc = gt.jbits == 4
               ? launch_gravity_kind<4, 8>(d, table, gt, tcap, ntd, t_begin, st, err, ctr)
               : launch_gravity_kind<5, 8, 8, 2, 16>(d, table, gt, tcap, ntd, t_begin, st, err, ctr);
  if (rc) return rc;
  HB_LAUNCH_CHECK();
  return HB_OK;
}

// cubic through f at the 4 Chebyshev nodes of [lo, hi]: coefficients in u
static float4 cheb_cubic(double lo, double hi, double (*f)(double, const double*),
                         const double* prm) {
  double m[4][5];
  for (int i = 0; i < 4; ++i) {
    double x = 0.5 * (lo + hi) + 0.5 * (hi - lo) * cos(M_PI * (i + 0.5) / 4);
    double p = 1.0;
    for (int j = 0; j < 4; ++j) { m[i][j] = p; p *= x; }
    m[i][4] = f(x, prm);
  }
  for (int c = 0; c < 4; ++c) {  // Gauss-Jordan on the 4x4 Vandermonde
    int piv = c;
    for (int r = c + 1; r < 4; ++r) if (fabs(m[r][c]) > fabs(m[piv][c])) piv = r;
    for (int j = 0; j < 5; ++j) { double tmp = m[c][j]; m[c][j] = m[piv][j]; m[piv][j] = tmp; }
    for (int r = 0; r < 4; ++r) {
      if (r == c) continue;
      double q = m[r][c] / m[c][c];
      for (int j = c; j < 5; ++j) m[r][j] -= q * m[c][j];
    }
  }
  return make_float4((float)(m[0][4] / m[0][0]), (float)(m[1][4] / m[1][1]),
                     (float)(m[2][4] / m[2][2]), (float)(m[3][4] / m[3][3]));
}

static double split_s(double x) { return erfc(x) + 1.1283791670955126 * x * exp(-x * x); }
static unsigned f2u(float f) { unsigned u; memcpy(&u, &f, 4); return u; }
static float u2f(unsigned u) { float f; memcpy(&f, &u, 4); return f; }
// prm: r_s, eps, x0, scale.  u in [0, 2^-jb) is the in-interval mantissa
// offset, soft = x0 + scale * u (x0 = interval start, scale = 2^exponent).
static double tab_fn(double u, const double* p) {
  double rs = p[0], eps = p[1], x0 = p[2], sc = p[3];
  double soft = x0 + sc * u;
  return split_s(sqrt(fmax(soft - eps * eps, 0.0)) / rs) * pow(soft, -1.5);
}

int gravity_table(double r_s, double r_cut, double eps, float4* host_out, GravTab* gt) {
  static int jb = 0;
  if (!jb) {  // HB_GRAV_JBITS: 5 (default) or 4 intervals-per-octave bits
    const char* e = getenv("HB_GRAV_JBITS");
    jb = e ? (atoi(e) == 4 ? 4 : 5) : kGravSoftBitsDefault;
  }
  gt->jbits = jb;
  const int sh = 23 - jb;
  float scut = (float)(r_cut * r_cut + eps * eps);
  // lowest row: eps^2, floored so the table spans <= kGravSoftOctaves octaves
  // (soft below the floor -- only r < 2^-20 r_cut at eps = 0 -- reads zero)
  double fl = fmax(eps * eps, ldexp((double)scut, -kGravSoftOctaves + 1));
  float smin = (float)fl;
  unsigned base = f2u(smin) >> sh;
  unsigned kc = f2u(scut) >> sh;
  unsigned rows = kc - base + 1;
  if (rows + 1 > (unsigned)kGravTableMax) return -1;
  for (unsigned k = 0; k < rows; ++k) {
    unsigned b = (base + k) << sh;
    float f0 = u2f(b);
    int e = 0;
    frexp((double)f0, &e);
    double prm[4] = {r_s, eps, (double)f0, ldexp(1.0, e - 1)};
    host_out[k] = cheb_cubic(0.0, ldexp(1.0, -jb), tab_fn, prm);
    if (!(isfinite(host_out[k].x) && isfinite(host_out[k].y) && isfinite(host_out[k].z) &&
          isfinite(host_out[k].w)))
      return -1;
  }
  host_out[rows] = make_float4(0.f, 0.f, 0.f, 0.f);
  gt->base = base; gt->last = rows; gt->rows = (int)rows + 1;
  return gt->rows;
}

// Device copy of the table, cached per device and re-uploaded only when the
// parameters change.  A per-step upload from pageable host memory would be
// host-synchronous (and on the legacy stream wait for all device work),
// which serialised the gravity chain behind the concurrent SPH chain.
const float4* gravity_table_device(double r_s, double r_cut, double eps, GravTab* gt,
                                   cudaStream_t st, HbError* err) {
  struct Slot {
    bool ok = false;
    double r_s, r_cut, eps;
    GravTab gt;
    float4* dev = nullptr;
    float4* host = nullptr;
    uint64_t used = 0;
  };
  // a few tables per device, keyed by their parameters: kernels on other
  // streams may still read a cached table, so a live entry is never
  // rewritten; evicting the least recently used one (rare: > kSlots distinct
  // parameter sets) first waits for the device to go idle
  constexpr int kSlots = 8;
  static Slot slots[64][kSlots];
  static uint64_t tick = 0;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
    set_err(err, HB_CUDA, "no CUDA device for the gravity table");
    return nullptr;
  }
  Slot* victim = &slots[dev][0];
  for (int k = 0; k < kSlots; ++k) {
    Slot& c = slots[dev][k];
    if (c.ok && c.r_s == r_s && c.r_cut == r_cut && c.eps == eps) {
      c.used = ++tick;
      *gt = c.gt;
      return c.dev;
    }
    if (!c.ok) { if (victim->ok) victim = &c; }
    else if (victim->ok && c.used < victim->used) victim = &c;
  }
  Slot& sl = *victim;
  if (sl.ok && cudaDeviceSynchronize() != cudaSuccess) {
    set_err(err, HB_CUDA, "gravity table eviction: device error");
    return nullptr;
  }
  sl.ok = false;
  if (!sl.dev && (cudaMalloc(&sl.dev, kGravTableMax * sizeof(float4)) != cudaSuccess ||
                  cudaMallocHost(&sl.host, kGravTableMax * sizeof(float4)) != cudaSuccess)) {
    set_err(err, HB_CUDA, "gravity table allocation failed");
    return nullptr;
  }
  if (gravity_table(r_s, r_cut, eps, sl.host, gt) < 0) {
    set_err(err, HB_CONTRACT, "gravity table: r_cut / softening not representable");
    return nullptr;
  }
  // the pinned staging buffer is reused on the next parameter change: finish the copy
  if (cudaMemcpyAsync(sl.dev, sl.host, gt->rows * sizeof(float4), cudaMemcpyHostToDevice, st) !=
          cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess) {
    set_err(err, HB_CUDA, "gravity table upload failed");
    return nullptr;
  }
  sl.used = ++tick;
  sl.ok = true; sl.r_s = r_s; sl.r_cut = r_cut; sl.eps = eps; sl.gt = *gt;
  return sl.dev;
}


// ---------------------------------------------------------------- driver pieces
int64_t tile_capacity(int64_t n, int64_t n_leaves) { return n / 8 + 2 * n_leaves + 2; }

void carve_tiling(Arena& ws, int64_t n, int64_t nl, Tiling& T, int tile_max, int even) {
  int64_t tc = tile_capacity(n, nl);
  T.n_leaves = nl; T.n_tiles_cap = tc;
  T.tile_max = tile_max; T.even = even;
  T.sel_cnt = ws.take<int64_t>(nl + 1); T.sel_off = ws.take<int64_t>(nl + 1);
  T.tile_cnt = ws.take<int64_t>(nl + 1); T.tile_ptr = ws.take<int64_t>(nl + 1);
  T.tperm = ws.take<int32_t>(n + 1);
  T.tile_start = ws.take<int32_t>(tc); T.tile_n = ws.take<int32_t>(tc);
  T.tile_leaf = ws.take<int32_t>(tc);
  T.tile_lo = ws.take<float4>(tc); T.tile_hi = ws.take<float4>(tc);
  T.origin = ws.take<double>(3 * nl + 3);
  T.overflow = ws.take<int>(1);
  T.tile_skip = ws.take<uint8_t>(tc);
}

int kid_selects_gas(int kid) {
  return kid == KID_DENSITY || kid == KID_NEIGHBOR_COUNT || kid == KID_CRK_MOMENTS ||
         kid == KID_HYDRO_FORCE || kid == KID_CRK_INTERP || kid == KID_CRK_GRAD1 ||
         kid == KID_CRK_GRAD2;
}

int build_tiling(Tiling& T, int64_t nl, const int64_t* leaf_start, const int64_t* leaf_end,
                 Rows rows, const int8_t* pshift, double L, int sel,
                 int64_t* n_tiles_dev, Arena& ws, cudaStream_t st, HbError* err,
                 const uint8_t* ghost) {
  if (ws.dry) {
    Arena s = ws;
    exclusive_scan_i64(nullptr, nullptr, nl, nullptr, s, st, err);
    ws.used = s.used;
    return HB_OK;
  }
  HB_CUDA_TRY(cudaMemsetAsync(T.overflow, 0, sizeof(int), st));
  k_tile_count<<<grid_for(nl * 32, 256), 256, 0, st>>>(nl, leaf_start, leaf_end, rows, sel,
                                                       T.sel_cnt, T.tile_cnt, T.tile_max, T.even);
  HB_LAUNCH_CHECK();
  {
    Arena s = ws;
    int rc = exclusive_scan_i64(T.sel_cnt, T.sel_off, nl, T.sel_off + nl, s, st, err);
    if (rc) return rc;
    Arena s2 = ws;
    rc = exclusive_scan_i64(T.tile_cnt, T.tile_ptr, nl, n_tiles_dev, s2, st, err);
    if (rc) return rc;
    HB_CUDA_TRY(cudaMemcpyAsync(T.tile_ptr + nl, n_tiles_dev, sizeof(int64_t),
                                cudaMemcpyDeviceToDevice, st));
  }
  // the builders emit each tile's box as they cut it (emit_tile_box)
  k_tile_build_warp<<<grid_for(nl, kTileWarps), kTileWarps * 32, 0, st>>>(
      T, leaf_start, leaf_end, rows, pshift, L, sel, (int)nl, ghost);
  HB_LAUNCH_CHECK();
  k_tile_build<<<(unsigned)nl, kTileBuildBlock, 0, st>>>(T, leaf_start, leaf_end, rows, pshift,
                                                         L, sel, ghost);
  HB_LAUNCH_CHECK();
  return HB_OK;
}

int pack_records(int kid, const Tiling& T, const int64_t* n_tiles_dev, Rows rows,
                 const int8_t* pshift, const double* aux, int naux, double L, float4* P0,
                 float4* P1, float4* P2, cudaStream_t st, HbError* err) {
  int64_t tcap = T.n_tiles_cap;
  k_pack<<<grid_for(tcap * 32, 256), 256, 0, st>>>(kid, tcap, n_tiles_dev, T, rows, pshift, aux,
                                                   naux, L, P0, P1, P2);
  HB_LAUNCH_CHECK();
  return HB_OK;
}

template <int KID>
static void launch_kid(const EvalDev& d, int64_t tcap, const int64_t* ntd, bool det, bool lean,
                       cudaStream_t st) {
  unsigned grid = grid_for(tcap, kEvalWarps);
  if (lean) {
    if (det) k_eval<KID, true, true><<<grid, kEvalWarps * 32, 0, st>>>(d, tcap, ntd);
    else k_eval<KID, false, true><<<grid, kEvalWarps * 32, 0, st>>>(d, tcap, ntd);
  } else {
    if (det) k_eval<KID, true, false><<<grid, kEvalWarps * 32, 0, st>>>(d, tcap, ntd);
    else k_eval<KID, false, false><<<grid, kEvalWarps * 32, 0, st>>>(d, tcap, ntd);
  }
}

int launch_pairs(int kid, bool det, bool lean, const EvalDev& d, int64_t tcap,
                 const int64_t* ntd, cudaStream_t st, HbError* err) {
  switch (kid) {
    case KID_COUNTING: launch_kid<KID_COUNTING>(d, tcap, ntd, det, lean, st); break;
    case KID_GRAVITY: launch_kid<KID_GRAVITY>(d, tcap, ntd, det, lean, st); break;
    case KID_GRAV_POT: launch_kid<KID_GRAV_POT>(d, tcap, ntd, det, lean, st); break;
    case KID_DENSITY: launch_kid<KID_DENSITY>(d, tcap, ntd, det, lean, st); break;
    case KID_CRK_MOMENTS: launch_kid<KID_CRK_MOMENTS>(d, tcap, ntd, det, lean, st); break;
    case KID_HYDRO_FORCE: launch_kid<KID_HYDRO_FORCE>(d, tcap, ntd, det, lean, st); break;
    case KID_NEIGHBOR_COUNT: launch_kid<KID_NEIGHBOR_COUNT>(d, tcap, ntd, det, lean, st); break;
    case KID_STUB_ZERO: launch_kid<KID_STUB_ZERO>(d, tcap, ntd, det, lean, st); break;
    case KID_CRK_INTERP: launch_kid<KID_CRK_INTERP>(d, tcap, ntd, det, lean, st); break;
    case KID_CRK_GRAD1: launch_kid<KID_CRK_GRAD1>(d, tcap, ntd, det, lean, st); break;
    case KID_CRK_GRAD2: launch_kid<KID_CRK_GRAD2>(d, tcap, ntd, det, lean, st); break;
    default: return set_err(err, HB_CONTRACT, "unknown kernel id");
  }
  HB_LAUNCH_CHECK();
  return HB_OK;
}

// ---------------------------------------------------------------- hb_eval_pairs driver
struct EvalWs {
  Tiling T;
  uint64_t* keys; uint32_t* vals;
  int32_t *e_src, *e_code, *e_orig, *s_src, *s_code, *s_orig;
  int64_t *rev_flag, *rev_off, *ent_cnt, *ent_ptr, *n_tiles_dev, *tot;
  float4 *P0, *P1, *P2;
  unsigned long long* dev_cnt;  // [0]=f [1]=g [2]=in_count [3]=err_key [4]=scratch
};

static void carve_eval(Arena& ws, const HbEvalArgs* a, EvalWs& w, int64_t E) {
  int64_t n = a->n, nl = a->n_leaves;
  carve_tiling(ws, n, nl, w.T);
  w.keys = ws.take<uint64_t>(E + 1); w.vals = ws.take<uint32_t>(E + 1);
  w.e_src = ws.take<int32_t>(E + 1); w.e_code = ws.take<int32_t>(E + 1); w.e_orig = ws.take<int32_t>(E + 1);
  w.s_src = ws.take<int32_t>(E + 1); w.s_code = ws.take<int32_t>(E + 1); w.s_orig = ws.take<int32_t>(E + 1);
  w.rev_flag = ws.take<int64_t>(a->n_pairs + 1); w.rev_off = ws.take<int64_t>(a->n_pairs + 1);
  w.ent_cnt = ws.take<int64_t>(nl + 1); w.ent_ptr = ws.take<int64_t>(nl + 1);
  w.n_tiles_dev = ws.take<int64_t>(1); w.tot = ws.take<int64_t>(1);
  w.P0 = ws.take<float4>(n + 1); w.P1 = ws.take<float4>(n + 1); w.P2 = ws.take<float4>(n + 1);
  w.dev_cnt = ws.take<unsigned long long>(5);
}

int eval_pairs(HbEvalArgs* a, Arena& ws, cudaStream_t st, HbError* err) {
  int64_t E = a->n_pairs * (a->mirror ? 2 : 1);
  EvalWs w;
  carve_eval(ws, a, w, E);
  if (ws.dry) {
    Arena s1 = ws, s2 = ws, s3 = ws, s4 = ws;
    radix_sort_u64_u32(w.keys, w.vals, E, 40, s1, st, err);
    exclusive_scan_i64(nullptr, nullptr, a->n_leaves + 1, nullptr, s2, st, err);
    exclusive_scan_i64(nullptr, nullptr, a->n_pairs + 1, nullptr, s3, st, err);
    build_tiling(w.T, a->n_leaves, nullptr, nullptr, Rows{}, nullptr, 0.0, 0, nullptr, s4, st, err);
    size_t mx = s1.used;
    if (s2.used > mx) mx = s2.used;
    if (s3.used > mx) mx = s3.used;
    if (s4.used > mx) mx = s4.used;
    ws.used = mx;
    return HB_OK;
  }
  if (!ws.ok()) return set_err(err, HB_CONTRACT, "workspace too small (eval)");
  for (int k = 0; k < 8; ++k) a->counters[k] = 0;
  if (a->nchan < 1 || a->nchan > 10) return set_err(err, HB_CONTRACT, "nchan must be 1..10");
  if (a->n <= 0 || a->n_pairs <= 0 || a->n_leaves <= 0) return HB_OK;
  if (a->n >= (1LL << 31)) return set_err(err, HB_CONTRACT, "too many rows for one evaluation");
  int sel = kid_selects_gas(a->kid);
  int64_t nl = a->n_leaves;
  // receiver CSR (stable: deterministic accumulation order)
  int64_t n_rev = 0;
  // mirror: relaxed -> receiver expansion (every ordered pair gathered on its
  // receiver, fixed order); deterministic -> each listed pair evaluated once and
  // the partner gets chan_sign * q[mirror_map] by integer scatter, so the two
  // sides' quanta cancel exactly as in hb/kernels.py:378-382
  int mm = a->mirror ? (a->deterministic ? 2 : 1) : 0;
  if (mm == 1) {
    k_rev_flags<<<grid_for(a->n_pairs, 256), 256, 0, st>>>(a->n_pairs, a->pair_a, a->pair_b,
                                                           a->pair_shift, w.rev_flag);
    HB_LAUNCH_CHECK();
    Arena s = ws;
    int rc = exclusive_scan_i64(w.rev_flag, w.rev_off, a->n_pairs, w.tot, s, st, err);
    if (rc) return rc;
    HB_CUDA_TRY(cudaMemcpyAsync(&n_rev, w.tot, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    HB_CUDA_TRY(cudaStreamSynchronize(st));
  }
  int64_t En = a->n_pairs + n_rev;
  k_expand<<<grid_for(a->n_pairs, 256), 256, 0, st>>>(a->n_pairs, mm, a->pair_a, a->pair_b,
                                                      a->pair_shift, w.rev_off, w.keys, w.vals,
                                                      w.e_src, w.e_code, w.e_orig);
  HB_LAUNCH_CHECK();
  {
    int bits = 1;
    while ((1LL << bits) < nl) ++bits;
    Arena s = ws;
    int rc = radix_sort_u64_u32(w.keys, w.vals, En, bits, s, st, err);
    if (rc) return rc;
  }
  HB_CUDA_TRY(cudaMemsetAsync(w.ent_cnt, 0, (nl + 1) * sizeof(int64_t), st));
  k_recv_hist<<<grid_for(En, 256), 256, 0, st>>>(En, w.keys, w.ent_cnt);
  HB_LAUNCH_CHECK();
  {
    Arena s = ws;
    int rc = exclusive_scan_i64(w.ent_cnt, w.ent_ptr, nl + 1, nullptr, s, st, err);
    if (rc) return rc;
  }
  k_gather_entries<<<grid_for(En, 256), 256, 0, st>>>(En, w.vals, w.e_src, w.e_code, w.e_orig,
                                                      w.s_src, w.s_code, w.s_orig);
  HB_LAUNCH_CHECK();
  Tiling& T = w.T;
  int rc0 = build_tiling(T, nl, a->leaf_start, a->leaf_end, Rows::state(a->state), a->pshift, a->side_length,
                         sel, w.n_tiles_dev, ws, st, err);
  if (rc0) return rc0;
  rc0 = pack_records(a->kid, T, w.n_tiles_dev, Rows::state(a->state), a->pshift, a->aux, a->naux,
                     a->side_length, w.P0, w.P1, w.P2, st, err);
  if (rc0) return rc0;
  int64_t tcap = T.n_tiles_cap;
  HB_CUDA_TRY(cudaMemsetAsync(w.dev_cnt, 0, 3 * sizeof(unsigned long long), st));
  HB_CUDA_TRY(cudaMemsetAsync(w.dev_cnt + 3, 0xff, sizeof(unsigned long long), st));
  k_sched_counters<<<grid_for(a->n_pairs, 256), 256, 0, st>>>(a->n_pairs, a->pair_a, a->pair_b,
                                                              a->leaf_start, a->leaf_end, a->W2,
                                                              w.dev_cnt);
  HB_LAUNCH_CHECK();
  EvalDev d = {};
  d.T = T; d.ent_ptr = w.ent_ptr; d.ent_src = w.s_src; d.ent_code = w.s_code;
  d.P0 = w.P0; d.P1 = w.P1; d.P2 = w.P2; d.rows = Rows::state(a->state); d.pshift = a->pshift;
  d.L = a->side_length; d.reach = a->reach;
  d.pp.p0 = (float)a->params[0]; d.pp.p1 = (float)a->params[1];
  d.pp.inv_rs = a->params[0] != 0.0 ? (float)(1.0 / a->params[0]) : 0.0f;
  d.pp.reach2 = (float)(a->reach * a->reach);
  d.cull_reach = (float)(a->reach * (1.0 + 1e-4)) + 1e-30f;
  d.include_self = a->include_self; d.nchan = a->nchan;
  for (int c = 0; c < 10; ++c) d.scale[c] = (float)a->scales[c];
  d.scatter = mm == 2;
  for (int c = 0; c < 10; ++c) {
    d.csign[c] = (int)a->chan_sign[c];
    d.mmap[c] = (a->mirror_map[c] >= 0 && a->mirror_map[c] < 10) ? (int)a->mirror_map[c] : c;
  }
  d.out_flt = a->out_flt; d.out_int = a->out_int; d.write_out = 1; d.skip_leaf = nullptr;
  d.in_count = w.dev_cnt + 2; d.err_key = w.dev_cnt + 3;
  int rc = launch_pairs(a->kid, a->deterministic != 0, false, d, tcap, w.n_tiles_dev, st, err);
  if (rc) return rc;
  if (a->exact_counters && sel) {
    // the reference counts pairs in reach over every species (hb/kernels.py:356-359)
    HB_CUDA_TRY(cudaMemsetAsync(w.dev_cnt + 2, 0, sizeof(unsigned long long), st));
    rc = build_tiling(T, nl, a->leaf_start, a->leaf_end, Rows::state(a->state), a->pshift, a->side_length, 0,
                      w.n_tiles_dev, ws, st, err);
    if (rc) return rc;
    rc = pack_records(KID_COUNTING, T, w.n_tiles_dev, Rows::state(a->state), a->pshift, nullptr, 0,
                      a->side_length, w.P0, w.P1, w.P2, st, err);
    if (rc) return rc;
    EvalDev c = d;
    c.T = T;
    c.write_out = 0;
    c.err_key = w.dev_cnt + 4;
    rc = launch_pairs(KID_COUNTING, false, false, c, tcap, w.n_tiles_dev, st, err);
    if (rc) return rc;
  }
  unsigned long long hc[4];
  int ovf = 0;
  HB_CUDA_TRY(cudaMemcpyAsync(hc, w.dev_cnt, sizeof(hc), cudaMemcpyDeviceToHost, st));
  HB_CUDA_TRY(cudaMemcpyAsync(&ovf, T.overflow, sizeof(int), cudaMemcpyDeviceToHost, st));
  HB_CUDA_TRY(cudaStreamSynchronize(st));
  if (ovf) return set_err(err, HB_CONTRACT, "leaf exceeds the tiling capacity (2048 members)");
  int64_t W2 = a->W2;
  a->counters[0] = (int64_t)hc[0];
  a->counters[1] = (int64_t)hc[1];
  a->counters[2] = (int64_t)hc[1] * W2;
  a->counters[3] = (int64_t)hc[1] * W2 * W2;
  a->counters[4] = (int64_t)hc[2];
  if (hc[3] != ~0ull) {
    int64_t e = (int64_t)(hc[3] / 4);
    int kind = (int)(hc[3] % 4);
    int32_t orig = 0;
    HB_CUDA_TRY(cudaMemcpy(&orig, w.s_orig + e, sizeof(int32_t), cudaMemcpyDeviceToHost));
    int64_t la = 0, lb = 0;
    HB_CUDA_TRY(cudaMemcpy(&la, a->pair_a + orig, sizeof(int64_t), cudaMemcpyDeviceToHost));
    HB_CUDA_TRY(cudaMemcpy(&lb, a->pair_b + orig, sizeof(int64_t), cudaMemcpyDeviceToHost));
    a->counters[5] = kind; a->counters[6] = la; a->counters[7] = lb;
    if (err) { err->leaf_a = la; err->leaf_b = lb; }
    return set_err(err, kind == 1 ? HB_NONFINITE : HB_OVERFLOW,
                   kind == 1 ? "non-finite partial" : "accumulator overflow");
  }
  return HB_OK;
}

}  // namespace hb

using namespace hb;

extern "C" size_t hb_eval_pairs_workspace(const HbEvalArgs* a) {
  Arena ws;
  ws.dry = true;
  HbEvalArgs c = *a;
  eval_pairs(&c, ws, nullptr, nullptr);
  return ws.used + 1024;
}

extern "C" int hb_eval_pairs(HbEvalArgs* a, void* wsp, size_t ws_bytes, void* stream, HbError* err) {
  if (err) *err = HbError{};
  Arena ws;
  ws.base = (char*)wsp; ws.cap = ws_bytes;
  return eval_pairs(a, ws, (cudaStream_t)stream, err);
}
