// hb_mesh.cu -- chaining-mesh bins, k-d leaves, AABBs and leaf-pair lists.
//
// Bit-exact restatement on the GPU of hb/cmtree.py:110-337 (hb/ =
// /root/reference/pkg/src/hydrobox/):
//   * flat bin key of binning_pos = pos + shift*L, trunc((bp-lo)/width) clipped
//     (hb/cmtree.py:152-154; hb/particles.py:131-133) -- float64, no FMA;
//   * stable sort by key (radix, hb_sort.cu) == np.argsort(kind="stable");
//   * per bin: recursive split at mid=(n+1)//2 of a STABLE sort along the
//     longest AABB axis (first max on ties) -- hb/cmtree.py:110-122.  Leaf
//     sizes depend on n only, so leaf counts/offsets are known before the
//     split; one CTA per bin performs the data-dependent sorts in shared
//     memory (stable merge sort by rank-in-sibling-run binary search);
//   * leaf AABBs by min/max, ghost_only by count (hb/cmtree.py:184-188);
//   * lists: 27-stencil sweep, periodic wrap with image shift on full-box
//     axes, duplicate (bin,shift) suppression, per-axis gap test, ordered by
//     (a, b, sx, sy, sz) (hb/cmtree.py:210-337).
#include "hb_internal.cuh"

namespace hb {

// ------------------------------------------------------------------ bin keys
struct BinGeom {
  double L, lo[3], width[3];
  int64_t nb[3];
};

__device__ __forceinline__ double binning_coord(double p, int8_t s, double L) {
  return dadd(p, dmul((double)s, L));  // two roundings, as numpy does
}

__device__ __forceinline__ int64_t bin_cell(double bp, double lo, double width, int64_t nb) {
  double u = ddiv(dsub(bp, lo), width);
  if (!(u >= 0.0)) return 0;                 // trunc toward zero then clip at 0
  if (u >= (double)nb) return nb - 1;
  int64_t c = (int64_t)u;
  return c > nb - 1 ? nb - 1 : c;
}

__global__ void k_bin_keys(int64_t n, const double* __restrict__ pos,
                           const int8_t* __restrict__ shift, BinGeom g, double* bx, double* by,
                           double* bz, uint64_t* keys, uint32_t* vals,
                           unsigned long long* bin_cnt) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool live = i < n;
  uint64_t flat = 0;
  if (live) {
    double p0 = binning_coord(pos[3 * i], shift[3 * i], g.L);
    double p1 = binning_coord(pos[3 * i + 1], shift[3 * i + 1], g.L);
    double p2 = binning_coord(pos[3 * i + 2], shift[3 * i + 2], g.L);
    bx[i] = p0; by[i] = p1; bz[i] = p2;
    int64_t c0 = bin_cell(p0, g.lo[0], g.width[0], g.nb[0]);
    int64_t c1 = bin_cell(p1, g.lo[1], g.width[1], g.nb[1]);
    int64_t c2 = bin_cell(p2, g.lo[2], g.width[2], g.nb[2]);
    flat = (uint64_t)((c0 * g.nb[1] + c1) * g.nb[2] + c2);
    keys[i] = flat;
    vals[i] = (uint32_t)i;
  }
  // warp-aggregated histogram (coherent inputs hit the same bin)
  unsigned live_mask = __ballot_sync(0xffffffffu, live);
  if (!live) return;
  unsigned peers = __match_any_sync(live_mask, flat);
  if (__popc(peers & lanemask_lt()) == 0) atomicAdd(&bin_cnt[flat], (unsigned long long)__popc(peers));
}

// leaves produced by the recursive split of n members (depends on n only)
__host__ __device__ inline int64_t leaves_for(int64_t n, int64_t max_leaf) {
  if (n == 0) return 0;
  if (n <= max_leaf) return 1;
  // at depth d sizes are floor/ceil(n/2^d); count leaves by explicit stack
  int64_t stack[128];
  int sp = 0;
  int64_t cnt = 0;
  stack[sp++] = n;
  while (sp) {
    int64_t m = stack[--sp];
    if (m <= max_leaf) { ++cnt; continue; }
    int64_t mid = (m + 1) / 2;
    stack[sp++] = m - mid;
    stack[sp++] = mid;
  }
  return cnt;
}

__global__ void k_leaf_counts(int64_t nbins, const unsigned long long* bin_cnt, int64_t max_leaf,
                              int64_t* bin_cnt64, int64_t* leaf_cnt) {
  int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nbins) return;
  int64_t c = (int64_t)bin_cnt[b];
  bin_cnt64[b] = c;
  leaf_cnt[b] = leaves_for(c, max_leaf);
}

// ------------------------------------------------------------------ k-d split
constexpr int kKdBlock = 256;
// members held in shared memory (larger bins use global scratch).  768 (18 KB)
// lets 8 CTAs share an SM; 1792 (43 KB, 5 CTAs) was 15% slower at c2
// (k_kd_split 247 -> 215 us), bins there hold ~270 members
constexpr int kKdSmemCap = 768;

// stable merge sort of (key, idx)[0,m): after return data is in (key, idx)
__device__ void block_stable_sort(double* key, uint32_t* idx, double* tk, uint32_t* ti, int m) {
  double *ka = key, *kb = tk;
  uint32_t *ia = idx, *ib = ti;
  for (int w = 1; w < m; w <<= 1) {
    for (int p = threadIdx.x; p < m; p += blockDim.x) {
      int base = (p / (2 * w)) * (2 * w);
      int mid = min(base + w, m), end = min(base + 2 * w, m);
      double kp = ka[p];
      int dest;
      if (p < mid) {  // left run: count right keys strictly less
        int lo = mid, hi = end;
        while (lo < hi) {
          int md = (lo + hi) >> 1;
          if (ka[md] < kp) lo = md + 1; else hi = md;
        }
        dest = base + (p - base) + (lo - mid);
      } else {        // right run: count left keys <= (stability)
        int lo = base, hi = mid;
        while (lo < hi) {
          int md = (lo + hi) >> 1;
          if (ka[md] <= kp) lo = md + 1; else hi = md;
        }
        dest = base + (p - mid) + (lo - base);
      }
      kb[dest] = kp;
      ib[dest] = ia[p];
    }
    __syncthreads();
    double* t = ka; ka = kb; kb = t;
    uint32_t* u = ia; ia = ib; ib = u;
  }
  if (ia != idx) {
    for (int p = threadIdx.x; p < m; p += blockDim.x) { key[p] = ka[p]; idx[p] = ia[p]; }
    __syncthreads();
  }
}

__device__ void block_minmax3(const uint32_t* idx, int m, const double* bx, const double* by,
                              const double* bz, double* out /*[6]: min3, max3*/, double* red) {
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int p = threadIdx.x; p < m; p += blockDim.x) {
    uint32_t i = idx[p];
    double v[3] = {bx[i], by[i], bz[i]};
#pragma unroll
    for (int d = 0; d < 3; ++d) { mn[d] = fmin(mn[d], v[d]); mx[d] = fmax(mx[d], v[d]); }
  }
#pragma unroll
  for (int d = 0; d < 3; ++d) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      mn[d] = fmin(mn[d], __shfl_xor_sync(0xffffffffu, mn[d], o));
      mx[d] = fmax(mx[d], __shfl_xor_sync(0xffffffffu, mx[d], o));
    }
  }
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0)
    for (int d = 0; d < 3; ++d) { red[wid * 6 + d] = mn[d]; red[wid * 6 + 3 + d] = mx[d]; }
  __syncthreads();
  if (threadIdx.x < 6) {
    int d = threadIdx.x;
    double v = red[d];
    for (int w = 1; w < nw; ++w) v = d < 3 ? fmin(v, red[w * 6 + d]) : fmax(v, red[w * 6 + d]);
    out[d] = v;
  }
  __syncthreads();
}

struct KdArgs {
  const int64_t* bin_start;  // (nbins+1)
  const int64_t* leaf_off;   // (nbins+1)
  const uint32_t* sorted_vals;
  const double *bx, *by, *bz;
  int64_t max_leaf;
  // global scratch for oversized bins, indexed by bin_start
  double *g_key, *g_tkey;
  uint32_t *g_idx, *g_tidx;
  int64_t* perm;
  int64_t *leaf_start, *leaf_end, *leaf_bin;
};

__global__ void __launch_bounds__(kKdBlock) k_kd_split(KdArgs a) {
  __shared__ double s_key[kKdSmemCap], s_tkey[kKdSmemCap];
  __shared__ uint32_t s_idx[kKdSmemCap], s_tidx[kKdSmemCap];
  __shared__ double red[(kKdBlock / 32) * 6];
  __shared__ double ext[6];
  __shared__ int64_t stack_s[128], stack_n[128];
  __shared__ int sp_sh;
  __shared__ int64_t leaf_j;
  int64_t b = blockIdx.x;
  int64_t s0 = a.bin_start[b];
  int64_t nb = a.bin_start[b + 1] - s0;
  if (nb == 0) return;
  int64_t l0 = a.leaf_off[b];
  if (nb <= a.max_leaf) {
    for (int64_t k = threadIdx.x; k < nb; k += blockDim.x) a.perm[s0 + k] = a.sorted_vals[s0 + k];
    if (threadIdx.x == 0) { a.leaf_start[l0] = s0; a.leaf_end[l0] = s0 + nb; a.leaf_bin[l0] = b; }
    return;
  }
  bool in_smem = nb <= kKdSmemCap;
  double* key = in_smem ? s_key : a.g_key + s0;
  double* tkey = in_smem ? s_tkey : a.g_tkey + s0;
  uint32_t* idx = in_smem ? s_idx : a.g_idx + s0;
  uint32_t* tidx = in_smem ? s_tidx : a.g_tidx + s0;
  for (int64_t k = threadIdx.x; k < nb; k += blockDim.x) idx[k] = a.sorted_vals[s0 + k];
  if (threadIdx.x == 0) {
    sp_sh = 1; stack_s[0] = 0; stack_n[0] = nb; leaf_j = 0;
  }
  __syncthreads();
  while (true) {
    int sp = sp_sh;
    if (sp == 0) break;
    int64_t ss = stack_s[sp - 1], sn = stack_n[sp - 1];
    __syncthreads();
    if (sn <= a.max_leaf) {
      if (threadIdx.x == 0) {
        int64_t j = l0 + leaf_j;
        a.leaf_start[j] = s0 + ss; a.leaf_end[j] = s0 + ss + sn; a.leaf_bin[j] = b;
        leaf_j += 1;
        sp_sh = sp - 1;
      }
      __syncthreads();
      continue;
    }
    block_minmax3(idx + ss, (int)sn, a.bx, a.by, a.bz, ext, red);
    double e0 = ext[3] - ext[0], e1 = ext[4] - ext[1], e2 = ext[5] - ext[2];
    int axis = 0;  // np.argmax: first maximum
    double best = e0;
    if (e1 > best) { axis = 1; best = e1; }
    if (e2 > best) axis = 2;
    const double* src = axis == 0 ? a.bx : (axis == 1 ? a.by : a.bz);
    for (int64_t k = threadIdx.x; k < sn; k += blockDim.x) key[ss + k] = src[idx[ss + k]];
    __syncthreads();
    block_stable_sort(key + ss, idx + ss, tkey + ss, tidx + ss, (int)sn);
    if (threadIdx.x == 0) {
      int64_t mid = (sn + 1) / 2;
      // replace top with right child, push left child (processed first: DFS left-first)
      stack_s[sp - 1] = ss + mid; stack_n[sp - 1] = sn - mid;
      stack_s[sp] = ss; stack_n[sp] = mid;
      sp_sh = sp + 1;
    }
    __syncthreads();
  }
  for (int64_t k = threadIdx.x; k < nb; k += blockDim.x) a.perm[s0 + k] = idx[k];
}

// ------------------------------------------------------------------ leaf boxes
__global__ void k_leaf_boxes(int64_t n_leaves_cap, const int64_t* n_leaves_dev,
                             const int64_t* leaf_start, const int64_t* leaf_end,
                             const int64_t* perm, const double* bx, const double* by,
                             const double* bz, const uint8_t* ghost, double* leaf_lo,
                             double* leaf_hi, uint8_t* ghost_only) {
  int64_t leaf = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (leaf >= *n_leaves_dev) return;
  int64_t s = leaf_start[leaf], e = leaf_end[leaf];
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  int gcount = 0;
  for (int64_t k = s + lane; k < e; k += 32) {
    int64_t i = perm[k];
    double v[3] = {bx[i], by[i], bz[i]};
#pragma unroll
    for (int d = 0; d < 3; ++d) { mn[d] = fmin(mn[d], v[d]); mx[d] = fmax(mx[d], v[d]); }
    gcount += ghost[i] != 0;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      mn[d] = fmin(mn[d], __shfl_xor_sync(0xffffffffu, mn[d], o));
      mx[d] = fmax(mx[d], __shfl_xor_sync(0xffffffffu, mx[d], o));
    }
    gcount += __shfl_xor_sync(0xffffffffu, gcount, o);
  }
  if (lane == 0) {
    for (int d = 0; d < 3; ++d) { leaf_lo[3 * leaf + d] = mn[d]; leaf_hi[3 * leaf + d] = mx[d]; }
    ghost_only[leaf] = gcount == (int)(e - s);
  }
}

__global__ void k_max_bin_leaves(int64_t nbins, const int64_t* leaf_cnt, unsigned long long* mx) {
  int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long v = b < nbins ? (unsigned long long)leaf_cnt[b] : 0ull;
#pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0 && v) atomicMax(mx, v);
}

struct MeshWs {
  double *bx, *by, *bz;
  uint64_t* keys;
  uint32_t* vals;
  unsigned long long* bin_cnt;
  int64_t *bin_cnt64, *bin_start, *leaf_cnt;
  double *g_key, *g_tkey;
  uint32_t *g_idx, *g_tidx;
  unsigned long long* maxbl;
  unsigned long long* maxbc;
};

static void carve_mesh(Arena& ws, int64_t n, int64_t nbins, MeshWs& m) {
  m.bx = ws.take<double>(n); m.by = ws.take<double>(n); m.bz = ws.take<double>(n);
  m.keys = ws.take<uint64_t>(n); m.vals = ws.take<uint32_t>(n);
  m.bin_cnt = ws.take<unsigned long long>(nbins);
  m.bin_cnt64 = ws.take<int64_t>(nbins + 1);
  m.bin_start = ws.take<int64_t>(nbins + 1);
  m.leaf_cnt = ws.take<int64_t>(nbins + 1);
  m.g_key = ws.take<double>(n); m.g_tkey = ws.take<double>(n);
  m.g_idx = ws.take<uint32_t>(n); m.g_tidx = ws.take<uint32_t>(n);
  m.maxbl = ws.take<unsigned long long>(1);
  m.maxbc = ws.take<unsigned long long>(1);
}

static int bit_length(uint64_t v) { int b = 0; while (v) { ++b; v >>= 1; } return b; }

int build_mesh(const HbMeshArgs* a, Arena& ws, cudaStream_t st, HbError* err) {
  int64_t n = a->n;
  int64_t nbins = a->nb[0] * a->nb[1] * a->nb[2];
  MeshWs m;
  carve_mesh(ws, n, nbins, m);
  if (ws.dry) {
    Arena sub = ws;
    int rc = radix_sort_u64_u32(m.keys, m.vals, n, bit_length((uint64_t)(nbins - 1)), sub, st, err);
    if (rc) return rc;
    Arena sub2 = ws;
    rc = exclusive_scan_i64(nullptr, nullptr, nbins + 1, nullptr, sub2, st, err);
    ws.used = sub.used > sub2.used ? sub.used : sub2.used;
    return HB_OK;
  }
  if (!ws.ok()) return set_err(err, HB_CONTRACT, "workspace too small (mesh)");
  if (n >= (int64_t)0xffffffffLL) return set_err(err, HB_CONTRACT, "too many particles for one mesh");
  int64_t cap = hb_leaf_capacity(n, nbins, a->max_leaf_size);
  if (a->leaf_cap < cap) return set_err(err, HB_CONTRACT, "leaf_cap below hb_leaf_capacity()");
  BinGeom g;
  g.L = a->side_length;
  for (int d = 0; d < 3; ++d) { g.lo[d] = a->lo[d]; g.width[d] = a->width[d]; g.nb[d] = a->nb[d]; }
  HB_CUDA_TRY(cudaMemsetAsync(m.bin_cnt, 0, nbins * sizeof(unsigned long long), st));
  HB_CUDA_TRY(cudaMemsetAsync(m.maxbl, 0, sizeof(unsigned long long), st));
  HB_CUDA_TRY(cudaMemsetAsync(m.maxbc, 0, sizeof(unsigned long long), st));
  if (n > 0) {
    k_bin_keys<<<grid_for(n, 256), 256, 0, st>>>(n, a->pos, a->image_shift, g, m.bx, m.by, m.bz,
                                                  m.keys, m.vals, m.bin_cnt);
    HB_LAUNCH_CHECK();
  }
  {
    Arena sub = ws;
    int rc = radix_sort_u64_u32(m.keys, m.vals, n, bit_length((uint64_t)(nbins - 1)), sub, st, err);
    if (rc) return rc;
  }
  k_leaf_counts<<<grid_for(nbins, 256), 256, 0, st>>>(nbins, m.bin_cnt, a->max_leaf_size,
                                                      m.bin_cnt64, m.leaf_cnt);
  HB_LAUNCH_CHECK();
  {
    Arena sub = ws;
    int rc = exclusive_scan_i64(m.bin_cnt64, m.bin_start, nbins, m.bin_start + nbins, sub, st, err);
    if (rc) return rc;
    Arena sub2 = ws;
    rc = exclusive_scan_i64(m.leaf_cnt, a->bin_ptr, nbins, a->bin_ptr + nbins, sub2, st, err);
    if (rc) return rc;
  }
  HB_CUDA_TRY(cudaMemcpyAsync(a->n_leaves_dev, a->bin_ptr + nbins, sizeof(int64_t),
                              cudaMemcpyDeviceToDevice, st));
  k_max_bin_leaves<<<grid_for(nbins, 256), 256, 0, st>>>(nbins, m.leaf_cnt, m.maxbl);
  HB_LAUNCH_CHECK();
  k_max_bin_leaves<<<grid_for(nbins, 256), 256, 0, st>>>(nbins, m.bin_cnt64, m.maxbc);
  HB_LAUNCH_CHECK();
  KdArgs k;
  k.bin_start = m.bin_start; k.leaf_off = a->bin_ptr; k.sorted_vals = m.vals;
  k.bx = m.bx; k.by = m.by; k.bz = m.bz; k.max_leaf = a->max_leaf_size;
  k.g_key = m.g_key; k.g_tkey = m.g_tkey; k.g_idx = m.g_idx; k.g_tidx = m.g_tidx;
  k.perm = a->perm; k.leaf_start = a->leaf_start; k.leaf_end = a->leaf_end; k.leaf_bin = a->leaf_bin;
  k_kd_split<<<(unsigned)nbins, kKdBlock, 0, st>>>(k);
  HB_LAUNCH_CHECK();
  k_leaf_boxes<<<grid_for(cap * 32, 256), 256, 0, st>>>(cap, a->n_leaves_dev, a->leaf_start,
                                                         a->leaf_end, a->perm, m.bx, m.by, m.bz,
                                                         a->ghost, a->leaf_lo, a->leaf_hi,
                                                         a->leaf_ghost_only);
  HB_LAUNCH_CHECK();
  if (a->n_leaves_host || a->max_bin_leaves_host || a->max_bin_count_host) {
    unsigned long long mbl = 0, mbc = 0;
    HB_CUDA_TRY(cudaMemcpyAsync(&mbl, m.maxbl, sizeof(mbl), cudaMemcpyDeviceToHost, st));
    HB_CUDA_TRY(cudaMemcpyAsync(&mbc, m.maxbc, sizeof(mbc), cudaMemcpyDeviceToHost, st));
    int64_t nl = 0;
    HB_CUDA_TRY(cudaMemcpyAsync(&nl, a->n_leaves_dev, sizeof(nl), cudaMemcpyDeviceToHost, st));
    HB_CUDA_TRY(cudaStreamSynchronize(st));
    if (a->n_leaves_host) *a->n_leaves_host = nl;
    if (a->max_bin_leaves_host) *a->max_bin_leaves_host = (int64_t)mbl;
    if (a->max_bin_count_host) *a->max_bin_count_host = (int64_t)mbc;
  }
  return HB_OK;
}

// ------------------------------------------------------------------ permutation helpers
__global__ void k_permute_rows(int64_t n, const int64_t* perm, const char* src, char* dst,
                               int64_t row_bytes) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row_bytes % 8 == 0) {
    int64_t w = row_bytes / 8;
    if (t >= n * w) return;
    int64_t r = t / w, c = t % w;
    reinterpret_cast<uint64_t*>(dst)[r * w + c] = reinterpret_cast<const uint64_t*>(src)[perm[r] * w + c];
  } else {
    if (t >= n * row_bytes) return;
    int64_t r = t / row_bytes, c = t % row_bytes;
    dst[r * row_bytes + c] = src[perm[r] * row_bytes + c];
  }
}

__global__ void k_inverse(int64_t n, const int64_t* perm, int64_t* inv) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) inv[perm[k]] = k;
}
__global__ void k_remap(int64_t n, const int64_t* inv, int64_t* v) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n && v[k] >= 0) v[k] = inv[v[k]];
}

// ------------------------------------------------------------------ grow AABBs
__global__ void k_grow(int64_t n_leaves, const int64_t* leaf_start, const int64_t* leaf_end,
                       const double* pos, const int8_t* shift, double L, double* leaf_lo,
                       double* leaf_hi) {
  int64_t leaf = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (leaf >= n_leaves) return;
  int64_t s = leaf_start[leaf], e = leaf_end[leaf];
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t k = s + lane; k < e; k += 32) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      double v = binning_coord(pos[3 * k + d], shift ? shift[3 * k + d] : (int8_t)0, L);
      mn[d] = fmin(mn[d], v); mx[d] = fmax(mx[d], v);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1)
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      mn[d] = fmin(mn[d], __shfl_xor_sync(0xffffffffu, mn[d], o));
      mx[d] = fmax(mx[d], __shfl_xor_sync(0xffffffffu, mx[d], o));
    }
  if (lane == 0 && e > s)
    for (int d = 0; d < 3; ++d) {
      leaf_lo[3 * leaf + d] = fmin(leaf_lo[3 * leaf + d], mn[d]);
      leaf_hi[3 * leaf + d] = fmax(leaf_hi[3 * leaf + d], mx[d]);
    }
}

// ------------------------------------------------------------------ lists


// stencil cell o (0..26) of bin (bx,by,bz): returns false if off-mesh; flat bin, shift code
__device__ __forceinline__ bool stencil_cell(const ListGeom& g, int64_t bx, int64_t by, int64_t bz,
                                             int o, int64_t& flat, int& code, int s[3]) {
  int64_t c[3] = {bx + o / 9 - 1, by + (o / 3) % 3 - 1, bz + o % 3 - 1};
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    s[d] = 0;
    if (g.periodic[d]) {
      if (c[d] < 0) { c[d] += g.nb[d]; s[d] = -1; }
      else if (c[d] >= g.nb[d]) { c[d] -= g.nb[d]; s[d] = 1; }
    } else if (c[d] < 0 || c[d] >= g.nb[d]) {
      return false;
    }
  }
  flat = (c[0] * g.nb[1] + c[1]) * g.nb[2] + c[2];
  code = (s[0] + 1) * 9 + (s[1] + 1) * 3 + (s[2] + 1);
  return true;
}

__device__ __forceinline__ bool gap_ok(const double* lo_a, const double* hi_a, const double* lo_b,
                                       const double* hi_b, const int s[3], double L, double reach) {
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double sh = dmul((double)s[d], L);
    double g1 = dsub(lo_a[d], dadd(hi_b[d], sh));
    double g2 = dsub(dadd(lo_b[d], sh), hi_a[d]);
    double gmax = g1 > g2 ? g1 : g2;  // python max(): first on ties
    if (gmax > reach) return false;
  }
  return true;
}



// one warp per receiving leaf, lane o < 27 owns stencil cell o; duplicate
// (bin, shift) cells (tiny periodic meshes) keep the lowest offset, as the
// reference's sequential sweep does (hb/cmtree.py:218-245)
template <bool EMIT>
__global__ void k_list_sweep(ListArgsDev a, int64_t* cnt, const int64_t* off, int64_t* tmp_b,
                             int32_t* tmp_code) {
  int64_t leaf = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (leaf >= a.n_leaves) return;
  bool active = !a.ghost_only[leaf] && (a.leaf_level ? a.leaf_level[leaf] : 0) >= a.g.active_depth;
  if (!active) {
    if (!EMIT && lane == 0) cnt[leaf] = 0;
    return;
  }
  int64_t bf = a.leaf_bin[leaf];
  int64_t bz = bf % a.g.nb[2], by = (bf / a.g.nb[2]) % a.g.nb[1], bx = bf / (a.g.nb[1] * a.g.nb[2]);
  int64_t flat = 0;
  int code = 0, s[3] = {0, 0, 0};
  bool valid = lane < 27 && stencil_cell(a.g, bx, by, bz, lane, flat, code, s);
  long long key = valid ? (long long)(flat * 27 + code) : -1 - lane;
  unsigned peers = __match_any_sync(0xffffffffu, key);
  valid = valid && (__ffs(peers) - 1 == lane);
  double lo_a[3], hi_a[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) { lo_a[d] = a.leaf_lo[3 * leaf + d]; hi_a[d] = a.leaf_hi[3 * leaf + d]; }
  int64_t p0 = valid ? a.bin_ptr[flat] : 0, p1 = valid ? a.bin_ptr[flat + 1] : 0;
  int mine = 0;
  for (int64_t p = p0; p < p1; ++p) {
    int64_t b = a.bin_ids ? a.bin_ids[p] : p;
    double lo_b[3], hi_b[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) { lo_b[d] = a.leaf_lo[3 * b + d]; hi_b[d] = a.leaf_hi[3 * b + d]; }
    mine += gap_ok(lo_a, hi_a, lo_b, hi_b, s, a.g.L, a.g.reach);
  }
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (!EMIT) {
    if (lane == 31) cnt[leaf] = incl;
    return;
  }
  int64_t slot = off[leaf] + incl - mine;
  for (int64_t p = p0; p < p1; ++p) {
    int64_t b = a.bin_ids ? a.bin_ids[p] : p;
    double lo_b[3], hi_b[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) { lo_b[d] = a.leaf_lo[3 * b + d]; hi_b[d] = a.leaf_hi[3 * b + d]; }
    if (gap_ok(lo_a, hi_a, lo_b, hi_b, s, a.g.L, a.g.reach)) {
      tmp_b[slot] = b;
      tmp_code[slot] = code;
      ++slot;
    }
  }
}

// order each receiver's entries by (b, code); keys are unique per receiver
__global__ void k_list_order(int64_t n_leaves, const int64_t* cnt, const int64_t* off,
                             const int64_t* tmp_b, const int32_t* tmp_code, int64_t* out_a,
                             int64_t* out_b, int8_t* out_s) {
  int64_t leaf = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (leaf >= n_leaves) return;
  int64_t m = cnt[leaf], o = off[leaf];
  for (int64_t e = lane; e < m; e += 32) {
    int64_t ke = tmp_b[o + e] * 27 + tmp_code[o + e];
    int64_t rank = 0;
    for (int64_t f = 0; f < m; ++f) rank += (tmp_b[o + f] * 27 + tmp_code[o + f]) < ke;
    int code = tmp_code[o + e];
    out_a[o + rank] = leaf;
    out_b[o + rank] = tmp_b[o + e];
    out_s[3 * (o + rank)] = (int8_t)(code / 9 - 1);
    out_s[3 * (o + rank) + 1] = (int8_t)((code / 3) % 3 - 1);
    out_s[3 * (o + rank) + 2] = (int8_t)(code % 3 - 1);
  }
}

// receiver-CSR output for the resident step: entries already grouped by
// receiver (leaf order), partner as int32, code | fwd<<8 as the pair engine reads
__global__ void k_list_order_csr(int64_t n_leaves, const int64_t* cnt, const int64_t* off,
                                 const int64_t* tmp_b, const int32_t* tmp_code, int32_t* ent_src,
                                 int32_t* ent_code) {
  int64_t leaf = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (leaf >= n_leaves) return;
  int64_t m = cnt[leaf], o = off[leaf];
  for (int64_t e = lane; e < m; e += 32) {
    int64_t ke = tmp_b[o + e] * 27 + tmp_code[o + e];
    int64_t rank = 0;
    for (int64_t f = 0; f < m; ++f) rank += (tmp_b[o + f] * 27 + tmp_code[o + f]) < ke;
    ent_src[o + rank] = (int32_t)tmp_b[o + e];
    ent_code[o + rank] = tmp_code[o + e] | (1 << 8);
  }
}

int assemble_csr(const ListArgsDev& d, int64_t capacity, int32_t* ent_src, int32_t* ent_code,
                 int64_t* ent_ptr, int64_t* total_host, Arena& ws, cudaStream_t st, HbError* err) {
  int64_t nl = d.n_leaves;
  int64_t* cnt = ws.take<int64_t>(nl + 1);
  int64_t* tmp_b = ws.take<int64_t>(capacity > 0 ? capacity : 1);
  int32_t* tmp_code = ws.take<int32_t>(capacity > 0 ? capacity : 1);
  if (ws.dry) {
    Arena sub = ws;
    exclusive_scan_i64(nullptr, nullptr, nl, nullptr, sub, st, err);
    ws.used = sub.used;
    return HB_OK;
  }
  if (!ws.ok()) return set_err(err, HB_CONTRACT, "workspace too small (list csr)");
  k_list_sweep<false><<<grid_for(nl * 32, 256), 256, 0, st>>>(d, cnt, nullptr, nullptr, nullptr);
  HB_LAUNCH_CHECK();
  {
    Arena sub = ws;
    int rc = exclusive_scan_i64(cnt, ent_ptr, nl, ent_ptr + nl, sub, st, err);
    if (rc) return rc;
  }
  int64_t total = 0;
  HB_CUDA_TRY(cudaMemcpyAsync(&total, ent_ptr + nl, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  HB_CUDA_TRY(cudaStreamSynchronize(st));
  *total_host = total;
  if (total > capacity) return set_err(err, HB_CONTRACT, "list capacity below entry count");
  k_list_sweep<true><<<grid_for(nl * 32, 256), 256, 0, st>>>(d, cnt, ent_ptr, tmp_b, tmp_code);
  HB_LAUNCH_CHECK();
  k_list_order_csr<<<grid_for(nl * 32, 256), 256, 0, st>>>(nl, cnt, ent_ptr, tmp_b, tmp_code,
                                                          ent_src, ent_code);
  HB_LAUNCH_CHECK();
  return HB_OK;
}

int assemble_lists(const HbListArgs* a, Arena& ws, cudaStream_t st, HbError* err) {
  int64_t nl = a->n_leaves;
  int64_t* cnt = ws.take<int64_t>(nl + 1);
  int64_t* off = ws.take<int64_t>(nl + 1);
  int64_t* tot = ws.take<int64_t>(1);
  int64_t* tmp_b = ws.take<int64_t>(a->capacity > 0 ? a->capacity : 1);
  int32_t* tmp_code = ws.take<int32_t>(a->capacity > 0 ? a->capacity : 1);
  if (ws.dry) {
    Arena sub = ws;
    exclusive_scan_i64(cnt, off, nl, tot, sub, st, err);
    ws.used = sub.used;
    return HB_OK;
  }
  if (!ws.ok()) return set_err(err, HB_CONTRACT, "workspace too small (lists)");
  ListArgsDev d;
  d.n_leaves = nl; d.leaf_bin = a->leaf_bin; d.leaf_level = a->leaf_level; d.bin_ptr = a->bin_ptr;
  d.bin_ids = a->bin_ids; d.leaf_lo = a->leaf_lo; d.leaf_hi = a->leaf_hi;
  d.ghost_only = a->leaf_ghost_only;
  for (int k = 0; k < 3; ++k) { d.g.nb[k] = a->nb[k]; d.g.periodic[k] = a->periodic[k]; }
  d.g.L = a->side_length; d.g.reach = a->reach; d.g.active_depth = a->active_depth;
  if (nl == 0) {
    if (a->count_host) *a->count_host = 0;
    return HB_OK;
  }
  k_list_sweep<false><<<grid_for(nl * 32, 256), 256, 0, st>>>(d, cnt, nullptr, nullptr, nullptr);
  HB_LAUNCH_CHECK();
  {
    Arena sub = ws;
    int rc = exclusive_scan_i64(cnt, off, nl, tot, sub, st, err);
    if (rc) return rc;
  }
  int64_t total = 0;
  HB_CUDA_TRY(cudaMemcpyAsync(&total, tot, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  HB_CUDA_TRY(cudaStreamSynchronize(st));
  if (a->count_host) *a->count_host = total;
  if (a->out_a == nullptr) return HB_OK;
  if (total > a->capacity) return set_err(err, HB_CONTRACT, "list capacity below entry count");
  k_list_sweep<true><<<grid_for(nl * 32, 256), 256, 0, st>>>(d, cnt, off, tmp_b, tmp_code);
  HB_LAUNCH_CHECK();
  k_list_order<<<grid_for(nl * 32, 256), 256, 0, st>>>(nl, cnt, off, tmp_b, tmp_code, a->out_a,
                                                        a->out_b, a->out_shift);
  HB_LAUNCH_CHECK();
  return HB_OK;
}

}  // namespace hb

// ------------------------------------------------------------------ C ABI (mesh, lists)
using namespace hb;

extern "C" int64_t hb_leaf_capacity(int64_t n, int64_t nbins, int64_t max_leaf_size) {
  int64_t ml = max_leaf_size < 1 ? 1 : max_leaf_size;
  int64_t nonempty = n < nbins ? n : nbins;
  return nonempty + (2 * n) / ml + 2;
}

extern "C" size_t hb_build_mesh_workspace(int64_t n, const int64_t nb[3], int64_t max_leaf_size) {
  HbMeshArgs a = {};
  a.n = n;
  for (int d = 0; d < 3; ++d) a.nb[d] = nb[d];
  a.max_leaf_size = max_leaf_size;
  Arena ws;
  ws.dry = true;
  build_mesh(&a, ws, nullptr, nullptr);
  return ws.used + 1024;
}

extern "C" int hb_build_mesh(const HbMeshArgs* a, void* wsp, size_t ws_bytes, void* stream,
                             HbError* err) {
  if (err) *err = HbError{};
  Arena ws;
  ws.base = (char*)wsp; ws.cap = ws_bytes;
  return build_mesh(a, ws, (cudaStream_t)stream, err);
}

extern "C" int hb_permute_rows(int64_t n, const int64_t* perm, const void* src, void* dst,
                               int64_t row_bytes, void* stream, HbError* err) {
  if (err) *err = HbError{};
  if (n <= 0) return HB_OK;
  int64_t units = row_bytes % 8 == 0 ? n * (row_bytes / 8) : n * row_bytes;
  k_permute_rows<<<grid_for(units, 256), 256, 0, (cudaStream_t)stream>>>(
      n, perm, (const char*)src, (char*)dst, row_bytes);
  HB_LAUNCH_CHECK();
  return HB_OK;
}

extern "C" int hb_remap_through_inverse(int64_t n, const int64_t* perm, int64_t* values,
                                        int64_t* scratch, void* stream, HbError* err) {
  if (err) *err = HbError{};
  if (n <= 0) return HB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  k_inverse<<<grid_for(n, 256), 256, 0, st>>>(n, perm, scratch);
  HB_LAUNCH_CHECK();
  k_remap<<<grid_for(n, 256), 256, 0, st>>>(n, scratch, values);
  HB_LAUNCH_CHECK();
  return HB_OK;
}

extern "C" int hb_grow_aabbs(int64_t n_leaves, const int64_t* leaf_start, const int64_t* leaf_end,
                             const double* pos, const int8_t* image_shift, double side_length,
                             double* leaf_lo, double* leaf_hi, void* stream, HbError* err) {
  if (err) *err = HbError{};
  if (n_leaves <= 0) return HB_OK;
  k_grow<<<grid_for(n_leaves * 32, 256), 256, 0, (cudaStream_t)stream>>>(
      n_leaves, leaf_start, leaf_end, pos, image_shift, side_length, leaf_lo, leaf_hi);
  HB_LAUNCH_CHECK();
  return HB_OK;
}

extern "C" size_t hb_assemble_lists_workspace(int64_t n_leaves, int64_t capacity) {
  HbListArgs a = {};
  a.n_leaves = n_leaves;
  a.capacity = capacity;
  Arena ws;
  ws.dry = true;
  assemble_lists(&a, ws, nullptr, nullptr);
  return ws.used + 1024;
}

extern "C" int hb_assemble_lists(const HbListArgs* a, void* wsp, size_t ws_bytes, void* stream,
                                 HbError* err) {
  if (err) *err = HbError{};
  Arena ws;
  ws.base = (char*)wsp; ws.cap = ws_bytes;
  return assemble_lists(a, ws, (cudaStream_t)stream, err);
}
