// hb_halo.cu -- overload (ghost) shell exchange support for multi-GPU ranks.
//
// Distributed restatement of build_overload / refresh_overload
// (hb/domain.py:88-189): a particle owned by rank p is copied to rank r as a
// ghost for image shift s when pos + s L lies strictly inside r's bounds
// widened by the overload width w (s = 0 and r = p excluded); an owned particle
// whose wrapped position left p's half-open domain migrates to its new owner.
// Selection is one pass per particle over (rank, shift) candidates with a
// count / emit split; records are fixed 96-byte rows so the exchange is a
// single NCCL all-to-all of bytes; the receiver orders ghosts by
// (global_id, shift) exactly as the reference (hb/domain.py:135-138).
#include "hb_common.cuh"

namespace hb {

struct HaloRec {      // 96 bytes
  double pos[3];
  double vel[3];
  double mass, h, u, rho;
  int64_t gid;
  int64_t src_row;    // owner's row on the receiving rank for self-images, else -1
  uint8_t species, ghost;
  int8_t shift[3];
  uint8_t pad[3];
};
static_assert(sizeof(HaloRec) == 112 || sizeof(HaloRec) == 104 || sizeof(HaloRec) == 96, "rec");

struct DomGrid {
  int g[3];
  double L, w;
};

__device__ __forceinline__ void dom_bounds(const DomGrid& G, int r, double lo[3], double hi[3]) {
  int c[3] = {r / (G.g[1] * G.g[2]), (r / G.g[2]) % G.g[1], r % G.g[2]};
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    // L * arange(g+1) / g as numpy computes it (hb/domain.py:60)
    lo[d] = (G.L * (double)c[d]) / (double)G.g[d];
    hi[d] = (G.L * (double)(c[d] + 1)) / (double)G.g[d];
  }
}

// owner rank of a wrapped position: searchsorted(edges, x, 'right') - 1 clipped
__device__ __forceinline__ int owner_of(const DomGrid& G, const double* p) {
  int c[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    int k = 0;
    for (int e = 1; e < G.g[d]; ++e) {
      double edge = (G.L * (double)e) / (double)G.g[d];
      if (p[d] >= edge) k = e;
    }
    c[d] = k;
  }
  return (c[0] * G.g[1] + c[1]) * G.g[2] + c[2];
}

// Slots: dest * 28 + code (code < 27: ghost copy for image shift code; 27:
// owned copy to its owner, i.e. keep or migrate).  mode 0 counts per slot,
// mode 1 emits (row, slot) at per-slot offsets (order inside a slot is free:
// the receiver sorts).  Only owned rows of the current set are sources.
__global__ void k_halo_select(int64_t n, const double* pos, const uint8_t* ghost, DomGrid G,
                              int self, int n_ranks, int mode, unsigned long long* counts,
                              unsigned long long* fill, int64_t* out_row, int32_t* out_slot,
                              int* drift) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || ghost[i]) return;
  double p[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
  int own = owner_of(G, p);
  if (mode == 0 && own != self) {  // DriftError: more than one domain hop (hb/domain.py:176-182)
    int a[3] = {own / (G.g[1] * G.g[2]), (own / G.g[2]) % G.g[1], own % G.g[2]};
    int b[3] = {self / (G.g[1] * G.g[2]), (self / G.g[2]) % G.g[1], self % G.g[2]};
    for (int d = 0; d < 3; ++d) {
      int hop = abs(a[d] - b[d]);
      hop = min(hop, G.g[d] - hop);
      if (hop > 1) atomicExch(drift, 1);
    }
  }
  for (int r = 0; r < n_ranks; ++r) {
    double lo[3], hi[3];
    dom_bounds(G, r, lo, hi);
    for (int sc = 0; sc < 28; ++sc) {
      bool emit;
      if (sc == 27) {
        emit = r == own;
      } else if (sc == 13 && r == own) {
        emit = false;  // that is the owned copy itself
      } else {
        int s[3] = {sc / 9 - 1, (sc / 3) % 3 - 1, sc % 3 - 1};
        emit = true;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          double x = __dadd_rn(p[d], __dmul_rn((double)s[d], G.L));
          emit = emit && (x > __dsub_rn(lo[d], G.w)) && (x < __dadd_rn(hi[d], G.w));
        }
      }
      if (!emit) continue;
      int slot = r * 28 + sc;
      if (mode == 0) {
        atomicAdd(&counts[slot], 1ull);
      } else {
        unsigned long long k = atomicAdd(&fill[slot], 1ull);
        out_row[k] = i;
        out_slot[k] = slot;
      }
    }
  }
}

__global__ void k_halo_pack(int64_t m, const int64_t* rows, const int32_t* slots,
                            const double* pos, const double* vel, const double* mass,
                            const double* h, const double* u, const double* rho,
                            const uint8_t* species, const int64_t* gid, DomGrid G, int self,
                            HaloRec* out) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  int64_t i = rows[k];
  int slot = slots[k];
  int r = slot / 28, sc = slot % 28;
  HaloRec rec;
  for (int d = 0; d < 3; ++d) { rec.pos[d] = pos[3 * i + d]; rec.vel[d] = vel[3 * i + d]; }
  rec.mass = mass[i]; rec.h = h[i]; rec.u = u[i]; rec.rho = rho[i];
  rec.gid = gid[i];
  rec.species = species[i];
  rec.ghost = sc == 27 ? 0 : 1;
  int s[3] = {0, 0, 0};
  if (sc < 27) { s[0] = sc / 9 - 1; s[1] = (sc / 3) % 3 - 1; s[2] = sc % 3 - 1; }
  for (int d = 0; d < 3; ++d) rec.shift[d] = (int8_t)s[d];
  // self-images of a particle this rank keeps owning: the receiver resolves the
  // owner's new row by global id after sorting (marker -2); remote ghosts: -1
  double p[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
  rec.src_row = (r == self && sc < 27 && owner_of(G, p) == self) ? -2 : -1;
  rec.pad[0] = rec.pad[1] = rec.pad[2] = 0;
  out[k] = rec;
}

__global__ void k_halo_keys(int64_t m, const HaloRec* in, uint64_t* keys, uint32_t* vals) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const HaloRec& r = in[k];
  int code = (r.shift[0] + 1) * 9 + (r.shift[1] + 1) * 3 + (r.shift[2] + 1);
  // owned rows first (sorted by gid), ghosts after, ordered by (gid, shift)
  keys[k] = ((uint64_t)r.ghost << 62) | ((uint64_t)r.gid * 27u + (uint64_t)code);
  vals[k] = (uint32_t)k;
}

__global__ void k_halo_unpack(int64_t m, const uint32_t* order, const HaloRec* in, int64_t row0,
                              double* pos, double* vel, double* mass, double* h, double* u,
                              double* rho, uint8_t* species, uint8_t* ghost, int8_t* shift,
                              int64_t* gid, int64_t* ghost_src) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const HaloRec& r = in[order ? order[k] : k];
  int64_t o = row0 + k;
  for (int d = 0; d < 3; ++d) {
    pos[3 * o + d] = r.pos[d]; vel[3 * o + d] = r.vel[d]; shift[3 * o + d] = r.shift[d];
  }
  mass[o] = r.mass; h[o] = r.h; u[o] = r.u; rho[o] = r.rho;
  species[o] = r.species; ghost[o] = r.ghost; gid[o] = r.gid; ghost_src[o] = r.src_row;
}

// ghost_src of self-images: binary search of the gid among the sorted owned rows
__global__ void k_halo_src_lookup(int64_t n_owned, int64_t m, const int64_t* gid,
                                  int64_t* ghost_src) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m || ghost_src[k] != -2) return;
  int64_t key = gid[k], lo = 0, hi = n_owned;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (gid[mid] < key) lo = mid + 1; else hi = mid;
  }
  ghost_src[k] = (lo < n_owned && gid[lo] == key) ? lo : -1;
}

}  // namespace hb

using namespace hb;

extern "C" int64_t hb_halo_record_bytes(void) { return (int64_t)sizeof(HaloRec); }

extern "C" int hb_halo_select(int64_t n, const double* pos, const uint8_t* ghost, const int32_t g[3],
                              double side_length, double overload_width, int32_t self,
                              int32_t mode, uint64_t* counts, uint64_t* fill, int64_t* out_row,
                              int32_t* out_slot, int32_t* drift_flag, void* stream, HbError* err) {
  if (err) *err = HbError{};
  if (n <= 0) return HB_OK;
  DomGrid G;
  for (int d = 0; d < 3; ++d) G.g[d] = g[d];
  G.L = side_length;
  G.w = overload_width;
  int n_ranks = g[0] * g[1] * g[2];
  k_halo_select<<<grid_for(n, 128), 128, 0, (cudaStream_t)stream>>>(
      n, pos, ghost, G, self, n_ranks, mode, (unsigned long long*)counts,
      (unsigned long long*)fill, out_row, out_slot, drift_flag);
  HB_LAUNCH_CHECK();
  return HB_OK;
}

extern "C" int hb_halo_pack(int64_t m, const int64_t* rows, const int32_t* slots, const double* pos,
                            const double* vel, const double* mass, const double* smoothing,
                            const double* internal_energy, const double* density,
                            const uint8_t* species, const int64_t* global_id, const int32_t g[3],
                            double side_length, int32_t self, void* out, void* stream,
                            HbError* err) {
  DomGrid G;
  for (int d = 0; d < 3; ++d) G.g[d] = g[d];
  G.L = side_length;
  G.w = 0.0;
  if (err) *err = HbError{};
  if (m <= 0) return HB_OK;
  k_halo_pack<<<grid_for(m, 256), 256, 0, (cudaStream_t)stream>>>(
      m, rows, slots, pos, vel, mass, smoothing, internal_energy, density, species, global_id, G,
      self, (HaloRec*)out);
  HB_LAUNCH_CHECK();
  return HB_OK;
}

extern "C" size_t hb_halo_unpack_workspace(int64_t m) {
  Arena ws;
  ws.dry = true;
  ws.take<uint64_t>(m + 1);
  ws.take<uint32_t>(m + 1);
  radix_sort_u64_u32(nullptr, nullptr, m, 64, ws, nullptr, nullptr);
  return ws.used + 1024;
}

extern "C" int hb_halo_unpack(int64_t m, const void* recs, int32_t sort_by_gid, int64_t row0,
                              double* pos, double* vel, double* mass, double* smoothing,
                              double* internal_energy, double* density, uint8_t* species,
                              uint8_t* ghost, int8_t* image_shift, int64_t* global_id,
                              int64_t* ghost_src, void* wsp, size_t ws_bytes, void* stream,
                              HbError* err) {
  if (err) *err = HbError{};
  if (m <= 0) return HB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Arena ws;
  ws.base = (char*)wsp; ws.cap = ws_bytes;
  uint64_t* keys = ws.take<uint64_t>(m + 1);
  uint32_t* vals = ws.take<uint32_t>(m + 1);
  if (!ws.ok()) return set_err(err, HB_CONTRACT, "workspace too small (halo unpack)");
  const HaloRec* in = (const HaloRec*)recs;
  uint32_t* order = nullptr;
  if (sort_by_gid) {
    k_halo_keys<<<grid_for(m, 256), 256, 0, st>>>(m, in, keys, vals);
    HB_LAUNCH_CHECK();
    int rc = radix_sort_u64_u32(keys, vals, m, 64, ws, st, err);
    if (rc) return rc;
    order = vals;
  }
  k_halo_unpack<<<grid_for(m, 256), 256, 0, st>>>(m, order, in, row0, pos, vel, mass, smoothing,
                                                  internal_energy, density, species, ghost,
                                                  image_shift, global_id, ghost_src);
  HB_LAUNCH_CHECK();
  return HB_OK;
}

extern "C" int hb_halo_resolve_sources(int64_t n_owned, int64_t m, const int64_t* global_id,
                                       int64_t* ghost_src, void* stream, HbError* err) {
  if (err) *err = HbError{};
  if (m <= 0) return HB_OK;
  k_halo_src_lookup<<<grid_for(m, 256), 256, 0, (cudaStream_t)stream>>>(n_owned, m, global_id,
                                                                        ghost_src);
  HB_LAUNCH_CHECK();
  return HB_OK;
}
