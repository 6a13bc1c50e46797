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
// The reference tests every (rank, shift) on all three axes; the test is a
// product of per-axis interval tests, so candidates are enumerated per axis
// (<= 4 per axis, usually 1).  Axes with periodic_unsplit (g = 1, kept
// periodic in the rank mesh) take only (cell 0, shift 0).
__device__ __forceinline__ void halo_emit(int mode, int slot, int64_t i,
                                          unsigned long long* counts, unsigned long long* fill,
                                          int64_t* out_row, int32_t* out_slot) {
  if (mode == 0) {
    atomicAdd(&counts[slot], 1ull);
  } else {
    unsigned long long k = atomicAdd(&fill[slot], 1ull);
    out_row[k] = i;
    out_slot[k] = slot;
  }
}

__global__ void k_halo_select(int64_t n, const double* pos, const uint8_t* ghost, DomGrid G,
                              int self, int periodic_unsplit, int mode,
                              unsigned long long* counts, unsigned long long* fill,
                              int64_t* out_row, int32_t* out_slot, int* drift, uint8_t* stay) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool live = i < n && !ghost[i];
  int own_slot = -1;
  double p[3] = {0.0, 0.0, 0.0};
  int own = 0;
  if (live) {
    p[0] = pos[3 * i]; p[1] = pos[3 * i + 1]; p[2] = pos[3 * i + 2];
    own = owner_of(G, p);
    own_slot = own * 28 + 27;
  }
  // stay != null: particles this rank keeps owning are flagged, not exchanged;
  // their number goes to counts[n_ranks * 28 + 1]
  bool emit_owned = live && !(stay && own == self);
  if (stay && mode == 0) {
    bool st = live && own == self;
    if (i < n) stay[i] = st ? 1 : 0;
    unsigned sm = __ballot_sync(0xffffffffu, st);
    if ((threadIdx.x & 31) == 0 && sm)
      atomicAdd(&counts[G.g[0] * G.g[1] * G.g[2] * 28 + 1], (unsigned long long)__popc(sm));
  }
  // owned copies: one per particle, nearly all to the same slot -> warp-aggregated
  {
    unsigned act = __ballot_sync(0xffffffffu, emit_owned);
    if (emit_owned) {
      unsigned peers = __match_any_sync(act, own_slot);
      int leader = __ffs(peers) - 1;
      int rank_in = __popc(peers & lanemask_lt());
      unsigned long long base = 0;
      if ((int)(threadIdx.x & 31) == leader)
        base = atomicAdd(mode == 0 ? &counts[own_slot] : &fill[own_slot],
                         (unsigned long long)__popc(peers));
      base = __shfl_sync(peers, base, leader);
      if (mode == 1) {
        out_row[base + rank_in] = i;
        out_slot[base + rank_in] = own_slot;
      }
    }
  }
  if (!live) return;
  if (mode == 0 && own != self) {  // DriftError: more than one domain hop (hb/domain.py:176-182)
    int a[3] = {own / (G.g[1] * G.g[2]), (own / G.g[2]) % G.g[1], own % G.g[2]};
    int b[3] = {self / (G.g[1] * G.g[2]), (self / G.g[2]) % G.g[1], self % G.g[2]};
    for (int d = 0; d < 3; ++d) {
      int hop = abs(a[d] - b[d]);
      hop = min(hop, G.g[d] - hop);
      if (hop > 1) atomicExch(drift, 1);
    }
  }
  int oc[3] = {own / (G.g[1] * G.g[2]), (own / G.g[2]) % G.g[1], own % G.g[2]};
  {  // interior rows (farther than w, with margin, from every face of the owner
     // cell on the axes that can have images) have no ghost copies: skip the
     // FP64 enumeration.  The margin (1e-9 L) dwarfs its rounding, so the
     // enumeration below could not have found a candidate either.
    bool interior = true;
    double margin = G.w + 1e-9 * G.L;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      if (periodic_unsplit && G.g[d] == 1) continue;
      double lo = (G.L * (double)oc[d]) / (double)G.g[d];
      double hi = (G.L * (double)(oc[d] + 1)) / (double)G.g[d];
      interior = interior && (p[d] - lo > margin) && (hi - p[d] > margin);
    }
    if (interior) return;
  }
  int cand_c[3][6], cand_s[3][6], nc[3];
  for (int d = 0; d < 3; ++d) {
    nc[d] = 0;
    if (periodic_unsplit && G.g[d] == 1) {
      cand_c[d][0] = 0; cand_s[d][0] = 0; nc[d] = 1;
      continue;
    }
    for (int c = 0; c < G.g[d] && nc[d] < 6; ++c) {
      double lo = (G.L * (double)c) / (double)G.g[d];
      double hi = (G.L * (double)(c + 1)) / (double)G.g[d];
      for (int sv = -1; sv <= 1; ++sv) {
        double x = __dadd_rn(p[d], __dmul_rn((double)sv, G.L));
        if (x > __dsub_rn(lo, G.w) && x < __dadd_rn(hi, G.w) && nc[d] < 6) {
          cand_c[d][nc[d]] = c; cand_s[d][nc[d]] = sv; ++nc[d];
        }
      }
    }
  }
  // ghost copies (shell particles only; the owned copy was emitted above)
  for (int a0 = 0; a0 < nc[0]; ++a0)
    for (int a1 = 0; a1 < nc[1]; ++a1)
      for (int a2 = 0; a2 < nc[2]; ++a2) {
        int c0 = cand_c[0][a0], c1 = cand_c[1][a1], c2 = cand_c[2][a2];
        int s0 = cand_s[0][a0], s1 = cand_s[1][a1], s2 = cand_s[2][a2];
        if (s0 == 0 && s1 == 0 && s2 == 0 && c0 == oc[0] && c1 == oc[1] && c2 == oc[2]) continue;
        int r = (c0 * G.g[1] + c1) * G.g[2] + c2;
        halo_emit(mode, r * 28 + (s0 + 1) * 9 + (s1 + 1) * 3 + (s2 + 1), i, counts, fill,
                  out_row, out_slot);
      }
}

// ---- block-aggregated select (hb_halo_pack_all) -------------------------------
// Same selection as k_halo_select, restructured for throughput (it was
// load-latency bound at ~320 GB/s): a block owns kSelRows consecutive rows and
// prefetches the next row's position and ghost flag before working on the
// current one; domain edges come precomputed (identical FP64 expression, no
// division in the kernel); counts go to a shared-memory slot histogram with one
// global atomic per (block, slot).  mode 1 re-walks the block's rows (L1/L2
// resident) after reserving each slot's range with one atomic.
constexpr int kSelBlock = 256;
constexpr int kSelRows = 2048;
constexpr int kSelMaxSlots = 1024;

struct DomEdges {
  double e[3][9];  // e[d][c] = (L * c) / g[d], c = 0..g[d]  (g[d] <= 8)
};

__device__ __forceinline__ int owner_edges(const DomGrid& G, const DomEdges& E, const double* p) {
  int c[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    int k = 0;
    for (int e = 1; e < G.g[d]; ++e)
      if (p[d] >= E.e[d][e]) k = e;
    c[d] = k;
  }
  return (c[0] * G.g[1] + c[1]) * G.g[2] + c[2];
}

// every ghost-copy slot of an owned row at p (owner cell oc), as k_halo_select
template <class F>
__device__ __forceinline__ void for_each_ghost_slot(const DomGrid& G, const DomEdges& E,
                                                    int periodic_unsplit, const double* p,
                                                    const int* oc, F&& f) {
  bool interior = true;
  double margin = G.w + 1e-9 * G.L;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    if (periodic_unsplit && G.g[d] == 1) continue;
    double lo = E.e[d][oc[d]], hi = E.e[d][oc[d] + 1];
    interior = interior && (p[d] - lo > margin) && (hi - p[d] > margin);
  }
  if (interior) return;
  int cand_c[3][6], cand_s[3][6], nc[3];
  for (int d = 0; d < 3; ++d) {
    nc[d] = 0;
    if (periodic_unsplit && G.g[d] == 1) {
      cand_c[d][0] = 0; cand_s[d][0] = 0; nc[d] = 1;
      continue;
    }
    for (int c = 0; c < G.g[d] && nc[d] < 6; ++c) {
      double lo = E.e[d][c], hi = E.e[d][c + 1];
      for (int sv = -1; sv <= 1; ++sv) {
        double x = __dadd_rn(p[d], __dmul_rn((double)sv, G.L));
        if (x > __dsub_rn(lo, G.w) && x < __dadd_rn(hi, G.w) && nc[d] < 6) {
          cand_c[d][nc[d]] = c; cand_s[d][nc[d]] = sv; ++nc[d];
        }
      }
    }
  }
  for (int a0 = 0; a0 < nc[0]; ++a0)
    for (int a1 = 0; a1 < nc[1]; ++a1)
      for (int a2 = 0; a2 < nc[2]; ++a2) {
        int c0 = cand_c[0][a0], c1 = cand_c[1][a1], c2 = cand_c[2][a2];
        int s0 = cand_s[0][a0], s1 = cand_s[1][a1], s2 = cand_s[2][a2];
        if (s0 == 0 && s1 == 0 && s2 == 0 && c0 == oc[0] && c1 == oc[1] && c2 == oc[2]) continue;
        int r = (c0 * G.g[1] + c1) * G.g[2] + c2;
        f(r * 28 + (s0 + 1) * 9 + (s1 + 1) * 3 + (s2 + 1));
      }
}

__global__ void __launch_bounds__(kSelBlock)
k_halo_select_blk(int64_t n, const double* __restrict__ pos, const uint8_t* __restrict__ ghost,
                  DomGrid G, DomEdges E, int self, int periodic_unsplit, int mode, int nslot,
                  unsigned long long* counts, unsigned long long* fill, int64_t* out_row,
                  int32_t* out_slot, int* drift, uint8_t* stay) {
  __shared__ unsigned int hist[kSelMaxSlots];
  __shared__ unsigned long long base[kSelMaxSlots];
  __shared__ unsigned int s_stay;
  for (int t = threadIdx.x; t < nslot; t += blockDim.x) hist[t] = 0;
  if (threadIdx.x == 0) s_stay = 0;
  __syncthreads();
  int64_t r0 = (int64_t)blockIdx.x * kSelRows;
  int64_t r1 = min(n, r0 + (int64_t)kSelRows);
  unsigned my_stay = 0;
  for (int sweep = 0; sweep < (mode == 0 ? 1 : 2); ++sweep) {
    if (sweep == 1) {  // reserve this block's range of every slot
      __syncthreads();
      for (int t = threadIdx.x; t < nslot; t += blockDim.x) {
        unsigned c = hist[t];
        base[t] = c ? atomicAdd(&fill[t], (unsigned long long)c) : 0ull;
        hist[t] = 0;
      }
      __syncthreads();
    }
    auto emit = [&](int slot, int64_t i) {
      unsigned k = atomicAdd(&hist[slot], 1u);
      if (sweep == 1) {
        unsigned long long o = base[slot] + k;
        out_row[o] = i;
        out_slot[o] = slot;
      }
    };
    int64_t i = r0 + threadIdx.x;
    double px = 0.0, py = 0.0, pz = 0.0;
    uint8_t gh = 1;
    if (i < r1) { px = pos[3 * i]; py = pos[3 * i + 1]; pz = pos[3 * i + 2]; gh = ghost[i]; }
    for (; i < r1; i += kSelBlock) {
      int64_t in = i + kSelBlock;
      double nx = 0.0, ny = 0.0, nz = 0.0;
      uint8_t ng = 1;
      if (in < r1) { nx = pos[3 * in]; ny = pos[3 * in + 1]; nz = pos[3 * in + 2]; ng = ghost[in]; }
      bool st = false;
      if (!gh) {
        double p[3] = {px, py, pz};
        int own = owner_edges(G, E, p);
        st = stay && own == self;
        if (!st) emit(own * 28 + 27, i);  // owned copy: migrant (or every row without stay)
        int oc[3] = {own / (G.g[1] * G.g[2]), (own / G.g[2]) % G.g[1], own % G.g[2]};
        if (mode == 0 && own != self) {  // DriftError: more than one domain hop
          int b[3] = {self / (G.g[1] * G.g[2]), (self / G.g[2]) % G.g[1], self % G.g[2]};
          for (int d = 0; d < 3; ++d) {
            int hop = abs(oc[d] - b[d]);
            hop = min(hop, G.g[d] - hop);
            if (hop > 1) atomicExch(drift, 1);
          }
        }
        for_each_ghost_slot(G, E, periodic_unsplit, p, oc, [&](int slot) { emit(slot, i); });
      }
      if (mode == 0 && stay) {
        stay[i] = st ? 1 : 0;
        my_stay += st ? 1u : 0u;
      }
      px = nx; py = ny; pz = nz; gh = ng;
    }
  }
  if (mode != 0) return;
  my_stay = __reduce_add_sync(0xffffffffu, my_stay);
  if ((threadIdx.x & 31) == 0 && my_stay) atomicAdd(&s_stay, my_stay);
  __syncthreads();
  for (int t = threadIdx.x; t < nslot; t += blockDim.x)
    if (hist[t]) atomicAdd(&counts[t], (unsigned long long)hist[t]);
  if (threadIdx.x == 0 && s_stay) atomicAdd(&counts[nslot + 1], (unsigned long long)s_stay);
}

static DomEdges dom_edges(const DomGrid& G) {
  DomEdges E;
  for (int d = 0; d < 3; ++d)
    for (int c = 0; c < 9; ++c) E.e[d][c] = c <= G.g[d] ? (G.L * (double)c) / (double)G.g[d] : 0.0;
  return E;
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

__global__ void k_halo_keys(int64_t m, const HaloRec* in, int key_bits, uint64_t* keys,
                            uint32_t* vals) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const HaloRec& r = in[k];
  int code = (r.shift[0] + 1) * 9 + (r.shift[1] + 1) * 3 + (r.shift[2] + 1);
  // owned rows first (sorted by gid), ghosts after, ordered by (gid, shift)
  keys[k] = ((uint64_t)r.ghost << key_bits) | ((uint64_t)r.gid * 27u + (uint64_t)code);
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

__global__ void k_flag_scan_scatter(int64_t n, const uint8_t* flags, const int64_t* pos,
                                    int64_t* idx) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && flags[i]) idx[pos[i]] = i;
}
__global__ void k_flags_to_i64(int64_t n, const uint8_t* flags, int64_t* out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = flags[i] ? 1 : 0;
}

// kept rows: dst[pos[i]] = src[i] for every flagged row, all fields in one pass
__global__ void k_keep_gather(int64_t n, const uint8_t* flags, const int64_t* pos, HbFieldSet s,
                              HbFieldSet d) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !flags[i]) return;
  int64_t o = pos[i];
  for (int c = 0; c < 3; ++c) {
    d.pos[3 * o + c] = s.pos[3 * i + c];
    d.vel[3 * o + c] = s.vel[3 * i + c];
    d.image_shift[3 * o + c] = s.image_shift[3 * i + c];
  }
  d.mass[o] = s.mass[i]; d.smoothing[o] = s.smoothing[i];
  d.internal_energy[o] = s.internal_energy[i]; d.density[o] = s.density[i];
  d.species[o] = s.species[i]; d.ghost[o] = s.ghost[i];
  d.global_id[o] = s.global_id[i]; d.ghost_src[o] = s.ghost_src[i];
}

}  // namespace hb

using namespace hb;

// owned rows are wrapped into [0, L) before the owner lookup, as
// refresh_overload wraps them (hb/domain.py:175, hb/box.py:40-52: x - L
// floor(x / L), a result of exactly L folded to 0 side, tiny negatives to 0)
__global__ void k_wrap_owned(int64_t n, double* pos, const uint8_t* ghost, double L) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 3 * n || ghost[i / 3]) return;
  double x = pos[i];
  double y = x - L * floor(x / L);
  if (y >= L) y -= L;
  if (y < 0.0) y = 0.0;
  pos[i] = y;
}

extern "C" size_t hb_flag_indices_workspace(int64_t n) {
  Arena ws;
  ws.dry = true;
  ws.take<int64_t>(n + 1);
  exclusive_scan_i64(nullptr, nullptr, n, nullptr, ws, nullptr, nullptr);
  return ws.used + 1024;
}

extern "C" int hb_flag_indices(int64_t n, const uint8_t* flags, int64_t* idx, void* wsp,
                               size_t ws_bytes, void* stream, HbError* err) {
  if (err) *err = HbError{};
  if (n <= 0) return HB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Arena ws;
  ws.base = (char*)wsp; ws.cap = ws_bytes;
  int64_t* pos = ws.take<int64_t>(n + 1);
  if (!ws.ok()) return set_err(err, HB_CONTRACT, "workspace too small (flag indices)");
  k_flags_to_i64<<<grid_for(n, 256), 256, 0, st>>>(n, flags, pos);
  HB_LAUNCH_CHECK();
  int rc = exclusive_scan_i64(pos, pos, n, nullptr, ws, st, err);
  if (rc) return rc;
  k_flag_scan_scatter<<<grid_for(n, 256), 256, 0, st>>>(n, flags, pos, idx);
  HB_LAUNCH_CHECK();
  return HB_OK;
}

extern "C" int64_t hb_halo_record_bytes(void) { return (int64_t)sizeof(HaloRec); }

extern "C" int hb_halo_select(int64_t n, const double* pos, const uint8_t* ghost, const int32_t g[3],
                              double side_length, double overload_width, int32_t self,
                              int32_t periodic_unsplit, int32_t mode, uint64_t* counts,
                              uint64_t* fill, int64_t* out_row, int32_t* out_slot,
                              int32_t* drift_flag, uint8_t* stay, void* stream, HbError* err) {
  if (err) *err = HbError{};
  if (n <= 0) return HB_OK;
  DomGrid G;
  for (int d = 0; d < 3; ++d) G.g[d] = g[d];
  G.L = side_length;
  G.w = overload_width;
  k_halo_select<<<grid_for(n, 128), 128, 0, (cudaStream_t)stream>>>(
      n, pos, ghost, G, self, periodic_unsplit, mode, (unsigned long long*)counts,
      (unsigned long long*)fill, out_row, out_slot, drift_flag, stay);
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

extern "C" int hb_halo_unpack(int64_t m, const void* recs, int32_t key_bits, int64_t row0,
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
  if (key_bits > 0) {  // sort by (ghost flag, global_id * 27 + shift code)
    k_halo_keys<<<grid_for(m, 256), 256, 0, st>>>(m, in, key_bits, keys, vals);
    HB_LAUNCH_CHECK();
    int rc = radix_sort_u64_u32(keys, vals, m, key_bits + 1, ws, st, err);
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

extern "C" size_t hb_halo_pack_all_workspace(int32_t n_ranks) {
  Arena ws;
  ws.dry = true;
  int64_t nslot = (int64_t)n_ranks * 28;
  ws.take<int64_t>(nslot + 1);
  exclusive_scan_i64(nullptr, nullptr, nslot, nullptr, ws, nullptr, nullptr);
  return ws.used + 1024;
}

extern "C" int hb_halo_pack_all(int64_t n, const HbFieldSet* src, const int32_t g[3],
                                double side_length, double overload_width, int32_t self,
                                int32_t periodic_unsplit, uint64_t* counts, uint64_t* counts_host,
                                uint8_t* stay, int64_t cap, int64_t* rows, int32_t* slots,
                                void* send, void* wsp, size_t ws_bytes, void* stream,
                                HbError* err) {
  if (err) *err = HbError{};
  cudaStream_t st = (cudaStream_t)stream;
  DomGrid G;
  for (int d = 0; d < 3; ++d) G.g[d] = g[d];
  G.L = side_length;
  G.w = overload_width;
  int64_t nslot = (int64_t)g[0] * g[1] * g[2] * 28;
  Arena ws;
  ws.base = (char*)wsp; ws.cap = ws_bytes;
  int64_t* fill = ws.take<int64_t>(nslot + 1);
  if (!ws.ok()) return set_err(err, HB_CONTRACT, "workspace too small (halo pack)");
  int* drift = (int*)(counts + nslot);
  HB_CUDA_TRY(cudaMemsetAsync(counts, 0, (nslot + 2) * sizeof(uint64_t), st));
  bool blk = nslot <= kSelMaxSlots && g[0] <= 8 && g[1] <= 8 && g[2] <= 8;
  DomEdges E = dom_edges(G);
  if (n > 0) {
    k_wrap_owned<<<grid_for(3 * n, 256), 256, 0, st>>>(n, src->pos, src->ghost, side_length);
    HB_LAUNCH_CHECK();
  }
  unsigned sel_grid = (unsigned)((n + kSelRows - 1) / kSelRows);
  if (n > 0) {
    if (blk)
      k_halo_select_blk<<<sel_grid, kSelBlock, 0, st>>>(
          n, src->pos, src->ghost, G, E, self, periodic_unsplit, 0, (int)nslot,
          (unsigned long long*)counts, nullptr, nullptr, nullptr, drift, stay);
    else
      k_halo_select<<<grid_for(n, 128), 128, 0, st>>>(
          n, src->pos, src->ghost, G, self, periodic_unsplit, 0, (unsigned long long*)counts,
          nullptr, nullptr, nullptr, drift, stay);
    HB_LAUNCH_CHECK();
  }
  HB_CUDA_TRY(cudaMemcpyAsync(counts_host, counts, (nslot + 2) * sizeof(uint64_t),
                              cudaMemcpyDeviceToHost, st));
  HB_CUDA_TRY(cudaStreamSynchronize(st));
  int64_t m = 0;
  for (int64_t s = 0; s < nslot; ++s) m += (int64_t)counts_host[s];
  if ((counts_host[nslot] & 0xFFFFFFFFull) != 0) return HB_OK;  // drift: caller raises
  if (m > cap) return set_err(err, HB_OVERFLOW, "halo records exceed the buffer capacity");
  if (m == 0) return HB_OK;
  {
    Arena s2 = ws;
    int rc = exclusive_scan_i64((const int64_t*)counts, fill, nslot, nullptr, s2, st, err);
    if (rc) return rc;
  }
  if (blk)
    k_halo_select_blk<<<sel_grid, kSelBlock, 0, st>>>(
        n, src->pos, src->ghost, G, E, self, periodic_unsplit, 1, (int)nslot,
        (unsigned long long*)counts, (unsigned long long*)fill, rows, slots, drift, stay);
  else
    k_halo_select<<<grid_for(n, 128), 128, 0, st>>>(
        n, src->pos, src->ghost, G, self, periodic_unsplit, 1, (unsigned long long*)counts,
        (unsigned long long*)fill, rows, slots, drift, stay);
  HB_LAUNCH_CHECK();
  G.w = 0.0;
  k_halo_pack<<<grid_for(m, 256), 256, 0, st>>>(m, rows, slots, src->pos, src->vel, src->mass,
                                                src->smoothing, src->internal_energy,
                                                src->density, src->species, src->global_id, G,
                                                self, (HaloRec*)send);
  HB_LAUNCH_CHECK();
  return HB_OK;
}

extern "C" size_t hb_halo_unpack_keep_workspace(int64_t n_src, int64_t m) {
  Arena ws;
  ws.dry = true;
  ws.take<int64_t>(n_src + 1);
  exclusive_scan_i64(nullptr, nullptr, n_src, nullptr, ws, nullptr, nullptr);
  size_t a = ws.used;
  Arena w2;
  w2.dry = true;
  w2.take<uint64_t>(m + 1);
  w2.take<uint32_t>(m + 1);
  radix_sort_u64_u32(nullptr, nullptr, m, 64, w2, nullptr, nullptr);
  return (a > w2.used ? a : w2.used) + 1024;
}

extern "C" int hb_halo_unpack_keep(int64_t m, const void* recs, int32_t key_bits, int64_t n_src,
                                   const HbFieldSet* src, const uint8_t* stay, int64_t n_stay,
                                   const HbFieldSet* dst, void* wsp, size_t ws_bytes,
                                   void* stream, HbError* err) {
  if (err) *err = HbError{};
  cudaStream_t st = (cudaStream_t)stream;
  if (n_stay > 0 && n_src > 0) {
    Arena ws;
    ws.base = (char*)wsp; ws.cap = ws_bytes;
    int64_t* pos = ws.take<int64_t>(n_src + 1);
    if (!ws.ok()) return set_err(err, HB_CONTRACT, "workspace too small (halo keep)");
    k_flags_to_i64<<<grid_for(n_src, 256), 256, 0, st>>>(n_src, stay, pos);
    HB_LAUNCH_CHECK();
    int rc = exclusive_scan_i64(pos, pos, n_src, nullptr, ws, st, err);
    if (rc) return rc;
    k_keep_gather<<<grid_for(n_src, 256), 256, 0, st>>>(n_src, stay, pos, *src, *dst);
    HB_LAUNCH_CHECK();
  }
  return hb_halo_unpack(m, recs, key_bits, n_stay, dst->pos, dst->vel, dst->mass, dst->smoothing,
                        dst->internal_energy, dst->density, dst->species, dst->ghost,
                        dst->image_shift, dst->global_id, dst->ghost_src, wsp, ws_bytes, stream,
                        err);
}
