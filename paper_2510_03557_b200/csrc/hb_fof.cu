// hb_fof.cu -- in-situ cluster finding on the device (hb/insitu.py:25-142,
// SURVEY.md §8(f) row 3): the radius-wide cell grid, the 27-stencil pair
// sweep and a lock-free union-find.
//
// The sweep restates _pair_scan (hb/insitu.py:67-139) per particle i:
//   cell of i from ((x - lo) * inv_w) truncated and clamped, the 27 stencil
//   cells with a +-L image shift where a periodic axis wraps, and for every
//   member j the edge test  ((xi - (xj + sx))^2 + (..)^2) + (..)^2 <= r^2
//   in float64, evaluated from the LOWER row's side exactly as the reference
//   (unions only for j > i), so every edge decision is bit-identical.
// mode 0: FOF union; 1: neighbour counts (self included); 2: core-core union;
// 3: border attachment (min core label among core neighbours of non-core i).
// Union-find: hook the larger root under the smaller with atomicCAS; the
// final root of a component is its smallest row (order-independent result).
#include "hb_common.cuh"

namespace hb {

struct FofGrid {
  double lo[3], inv_w[3];
  int64_t nc[3];
  double L;
  int periodic;
  double r2max;
};

__device__ __forceinline__ int64_t fof_cell_axis(double x, double lo, double inv_w, int64_t nc) {
  int64_t c = (int64_t)__dmul_rn(__dsub_rn(x, lo), inv_w);  // truncation, as np.int64()
  return c < 0 ? 0 : (c > nc - 1 ? nc - 1 : c);
}

__global__ void k_fof_keys(int64_t n, const double* pos, FofGrid G, uint64_t* keys,
                           uint32_t* vals) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t c[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) c[d] = fof_cell_axis(pos[3 * i + d], G.lo[d], G.inv_w[d], G.nc[d]);
  keys[i] = (uint64_t)((c[0] * G.nc[1] + c[1]) * G.nc[2] + c[2]);
  vals[i] = (uint32_t)i;
}

__global__ void k_fof_cell_ranges(int64_t n, const uint64_t* keys_sorted, int64_t* start,
                                  int64_t* end) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  uint64_t c = keys_sorted[k];
  if (k == 0 || keys_sorted[k - 1] != c) start[c] = k;
  if (k == n - 1 || keys_sorted[k + 1] != c) end[c] = k + 1;
}

__device__ __forceinline__ int64_t uf_find(int64_t* parent, int64_t x) {
  int64_t p = parent[x];
  while (p != x) {
    int64_t gp = parent[p];
    if (gp != p) atomicCAS((unsigned long long*)&parent[x], (unsigned long long)p,
                           (unsigned long long)gp);  // path halving
    x = p;
    p = parent[x];
  }
  return x;
}

__device__ __forceinline__ void uf_union(int64_t* parent, int64_t a, int64_t b) {
  while (true) {
    a = uf_find(parent, a);
    b = uf_find(parent, b);
    if (a == b) return;
    if (a > b) { int64_t t = a; a = b; b = t; }
    // hook root b under the smaller root a; retry if b stopped being a root
    unsigned long long old = atomicCAS((unsigned long long*)&parent[b],
                                       (unsigned long long)b, (unsigned long long)a);
    if (old == (unsigned long long)b) return;
  }
}

__global__ void k_fof_scan(int64_t n, const double* pos, FofGrid G, const uint32_t* order,
                           const int64_t* start, const int64_t* end, int mode, int64_t* parent,
                           const uint8_t* core, int64_t* counts, int64_t* border_key,
                           const int64_t* core_label) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double xi = pos[3 * i], yi = pos[3 * i + 1], zi = pos[3 * i + 2];
  int64_t cc[3] = {fof_cell_axis(xi, G.lo[0], G.inv_w[0], G.nc[0]),
                   fof_cell_axis(yi, G.lo[1], G.inv_w[1], G.nc[1]),
                   fof_cell_axis(zi, G.lo[2], G.inv_w[2], G.nc[2])};
  int64_t cnt = 0;
  int64_t bkey = mode == 3 ? border_key[i] : 0;
  bool core_i = (mode == 2 || mode == 3) ? core[i] != 0 : false;
  if (mode == 2 && !core_i) return;
  if (mode == 3 && core_i) return;
  for (int ox = -1; ox <= 1; ++ox) {
    int64_t gx = cc[0] + ox;
    double sx = 0.0;
    if (G.periodic) {
      if (gx < 0) { gx += G.nc[0]; sx = -G.L; }
      else if (gx >= G.nc[0]) { gx -= G.nc[0]; sx = G.L; }
    } else if (gx < 0 || gx >= G.nc[0]) {
      continue;
    }
    for (int oy = -1; oy <= 1; ++oy) {
      int64_t gy = cc[1] + oy;
      double sy = 0.0;
      if (G.periodic) {
        if (gy < 0) { gy += G.nc[1]; sy = -G.L; }
        else if (gy >= G.nc[1]) { gy -= G.nc[1]; sy = G.L; }
      } else if (gy < 0 || gy >= G.nc[1]) {
        continue;
      }
      for (int oz = -1; oz <= 1; ++oz) {
        int64_t gz = cc[2] + oz;
        double sz = 0.0;
        if (G.periodic) {
          if (gz < 0) { gz += G.nc[2]; sz = -G.L; }
          else if (gz >= G.nc[2]) { gz -= G.nc[2]; sz = G.L; }
        } else if (gz < 0 || gz >= G.nc[2]) {
          continue;
        }
        int64_t flat = (gx * G.nc[1] + gy) * G.nc[2] + gz;
        int64_t k0 = start[flat], k1 = end[flat];
        for (int64_t k = k0; k < k1; ++k) {
          int64_t j = order[k];
          if ((mode == 0 || mode == 2) && j <= i) continue;
          double dx = __dsub_rn(xi, __dadd_rn(pos[3 * j], sx));
          double dy = __dsub_rn(yi, __dadd_rn(pos[3 * j + 1], sy));
          double dz = __dsub_rn(zi, __dadd_rn(pos[3 * j + 2], sz));
          double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
          if (r2 > G.r2max) continue;
          if (mode == 0) {
            uf_union(parent, i, j);
          } else if (mode == 1) {
            ++cnt;
          } else if (mode == 2) {
            if (core[j]) uf_union(parent, i, j);
          } else if (core[j]) {
            int64_t lab = core_label[j];
            if (lab < bkey) bkey = lab;
          }
        }
      }
    }
  }
  if (mode == 1) counts[i] += cnt;
  if (mode == 3) border_key[i] = bkey;
}

__global__ void k_uf_edges(int64_t m, const int64_t* a, const int64_t* b, int64_t* parent) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < m) uf_union(parent, a[k], b[k]);
}

__global__ void k_fof_flatten(int64_t n, int64_t* parent) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t r = i;
  while (parent[r] != r) r = parent[r];
  parent[i] = r;
}

// CRC32C (Castagnoli, reflected 0x82F63B78), slice-by-8 host tables
static uint32_t g_crc_tab[8][256];
static void crc_init() {
  static bool done = false;
  if (done) return;
  for (uint32_t i = 0; i < 256; ++i) {
    uint32_t c = i;
    for (int k = 0; k < 8; ++k) c = (c >> 1) ^ ((c & 1u) ? 0x82F63B78u : 0u);
    g_crc_tab[0][i] = c;
  }
  for (uint32_t i = 0; i < 256; ++i)
    for (int t = 1; t < 8; ++t)
      g_crc_tab[t][i] = (g_crc_tab[t - 1][i] >> 8) ^ g_crc_tab[0][g_crc_tab[t - 1][i] & 0xFF];
  done = true;
}

}  // namespace hb

using namespace hb;

extern "C" size_t hb_fof_workspace(int64_t n, const int64_t ncell[3]) {
  Arena ws;
  ws.dry = true;
  int64_t nc = ncell[0] * ncell[1] * ncell[2];
  ws.take<uint64_t>(n + 1);
  ws.take<uint32_t>(n + 1);
  ws.take<int64_t>(nc + 1);
  ws.take<int64_t>(nc + 1);
  radix_sort_u64_u32(nullptr, nullptr, n, 64, ws, nullptr, nullptr);
  return ws.used + 1024;
}

extern "C" int hb_fof_scan(int64_t n, const double* binpos, const double lo[3],
                           const double inv_w[3], const int64_t ncell[3], double side_length,
                           int32_t periodic, double r2max, int32_t mode, int64_t* parent,
                           const uint8_t* core, int64_t* counts, int64_t* border_key,
                           const int64_t* core_label, void* wsp, size_t ws_bytes, void* stream,
                           HbError* err) {
  if (err) *err = HbError{};
  if (mode < 0 || mode > 3) return set_err(err, HB_CONTRACT, "mode must be 0..3");
  if (n <= 0) return HB_OK;
  if (n >= (1LL << 32)) return set_err(err, HB_CONTRACT, "too many rows for one scan");
  cudaStream_t st = (cudaStream_t)stream;
  FofGrid G;
  for (int d = 0; d < 3; ++d) { G.lo[d] = lo[d]; G.inv_w[d] = inv_w[d]; G.nc[d] = ncell[d]; }
  G.L = side_length; G.periodic = periodic; G.r2max = r2max;
  int64_t nc = ncell[0] * ncell[1] * ncell[2];
  Arena ws;
  ws.base = (char*)wsp; ws.cap = ws_bytes;
  uint64_t* keys = ws.take<uint64_t>(n + 1);
  uint32_t* vals = ws.take<uint32_t>(n + 1);
  int64_t* cs = ws.take<int64_t>(nc + 1);
  int64_t* ce = ws.take<int64_t>(nc + 1);
  if (!ws.ok()) return set_err(err, HB_CONTRACT, "workspace too small (fof)");
  k_fof_keys<<<grid_for(n, 256), 256, 0, st>>>(n, binpos, G, keys, vals);
  HB_LAUNCH_CHECK();
  int bits = 1;
  while ((1LL << bits) < nc) ++bits;
  {
    Arena s = ws;
    int rc = radix_sort_u64_u32(keys, vals, n, bits, s, st, err);  // stable: as mergesort
    if (rc) return rc;
  }
  HB_CUDA_TRY(cudaMemsetAsync(cs, 0, (nc + 1) * sizeof(int64_t), st));
  HB_CUDA_TRY(cudaMemsetAsync(ce, 0, (nc + 1) * sizeof(int64_t), st));
  k_fof_cell_ranges<<<grid_for(n, 256), 256, 0, st>>>(n, keys, cs, ce);
  HB_LAUNCH_CHECK();
  k_fof_scan<<<grid_for(n, 128), 128, 0, st>>>(n, binpos, G, vals, cs, ce, mode, parent, core,
                                               counts, border_key, core_label);
  HB_LAUNCH_CHECK();
  if (mode == 0 || mode == 2) {
    k_fof_flatten<<<grid_for(n, 256), 256, 0, st>>>(n, parent);
    HB_LAUNCH_CHECK();
  }
  return HB_OK;
}

extern "C" int hb_uf_union_edges(int64_t m, const int64_t* a, const int64_t* b, int64_t n,
                                 int64_t* parent, void* stream, HbError* err) {
  if (err) *err = HbError{};
  cudaStream_t st = (cudaStream_t)stream;
  if (m > 0) {
    k_uf_edges<<<grid_for(m, 256), 256, 0, st>>>(m, a, b, parent);
    HB_LAUNCH_CHECK();
  }
  if (n > 0) {
    k_fof_flatten<<<grid_for(n, 256), 256, 0, st>>>(n, parent);
    HB_LAUNCH_CHECK();
  }
  return HB_OK;
}

extern "C" uint32_t hb_crc32c(const void* data, size_t nbytes, uint32_t value) {
  crc_init();
  const uint8_t* p = (const uint8_t*)data;
  uint32_t c = value ^ 0xFFFFFFFFu;
  while (nbytes >= 8) {
    uint32_t lo = c ^ ((uint32_t)p[0] | (uint32_t)p[1] << 8 | (uint32_t)p[2] << 16 |
                       (uint32_t)p[3] << 24);
    uint32_t hi = (uint32_t)p[4] | (uint32_t)p[5] << 8 | (uint32_t)p[6] << 16 |
                  (uint32_t)p[7] << 24;
    c = g_crc_tab[7][lo & 0xFF] ^ g_crc_tab[6][(lo >> 8) & 0xFF] ^
        g_crc_tab[5][(lo >> 16) & 0xFF] ^ g_crc_tab[4][lo >> 24] ^ g_crc_tab[3][hi & 0xFF] ^
        g_crc_tab[2][(hi >> 8) & 0xFF] ^ g_crc_tab[1][(hi >> 16) & 0xFF] ^ g_crc_tab[0][hi >> 24];
    p += 8;
    nbytes -= 8;
  }
  while (nbytes--) c = (c >> 8) ^ g_crc_tab[0][(c ^ *p++) & 0xFF];
  return c ^ 0xFFFFFFFFu;
}
