// hb_sort.cu -- device-wide scan and stable LSD radix sort.
//
// The bin sort of the mesh build (hb/cmtree.py:152-159: np.argsort(kind=
// "stable") of the flat bin key) and the receiver grouping of pair lists both
// need a STABLE sort: ties must keep input order, which also makes every FP32
// sum downstream run-to-run deterministic.  8-bit digits, three kernels per
// pass (tile histogram -> digit-major scan -> stable tile scatter).
#include "hb_common.cuh"

namespace hb {

// ------------------------------------------------------------ exclusive scan
constexpr int kScanBlock = 512;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanBlock * kScanItems;

__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t* sh, int64_t* total) {
  // sh: kScanBlock/32 entries
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int64_t w = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < (int)(blockDim.x >> 5)) sh[lane] = w;
  }
  __syncthreads();
  int64_t before = wid ? sh[wid - 1] : 0;
  if (total) *total = sh[(blockDim.x >> 5) - 1];
  int64_t res = before + x - v;
  __syncthreads();
  return res;
}

__global__ void k_scan_tiles(const int64_t* in, int64_t* out, int64_t n, int64_t* tile_sums) {
  __shared__ int64_t sh[kScanBlock / 32];
  int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int64_t v[kScanItems];
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = base + k < n ? in[base + k] : 0;
    s += v[k];
  }
  int64_t tot;
  int64_t ex = block_excl_scan(s, sh, &tot);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k < n) out[base + k] = ex;
    ex += v[k];
  }
  if (threadIdx.x == 0 && tile_sums) tile_sums[blockIdx.x] = tot;
}

__global__ void k_scan_add(int64_t* out, int64_t n, const int64_t* tile_off) {
  int64_t base = (int64_t)blockIdx.x * kScanTile;
  int64_t add = tile_off[blockIdx.x];
  for (int k = threadIdx.x; k < kScanTile; k += blockDim.x)
    if (base + k < n) out[base + k] += add;
}

__global__ void k_scan_total(const int64_t* in_last, const int64_t* ex_last, int64_t* total) {
  *total = *in_last + *ex_last;
}

int exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, int64_t* total_dev,
                       Arena& ws, cudaStream_t st, HbError* err) {
  if (n <= 0) {
    if (total_dev && !ws.dry) HB_CUDA_TRY(cudaMemsetAsync(total_dev, 0, sizeof(int64_t), st));
    return HB_OK;
  }
  int64_t ntiles = (n + kScanTile - 1) / kScanTile;
  int64_t* sums = ws.take<int64_t>(ntiles);
  int64_t* last_in = ws.take<int64_t>(1);
  if (ws.dry) {
    if (ntiles > 1) {
      Arena sub = ws;  // recursive sizing
      exclusive_scan_i64(nullptr, nullptr, ntiles, nullptr, sub, st, err);
      ws.used = sub.used;
    }
    return HB_OK;
  }
  if (!ws.ok()) return set_err(err, HB_CONTRACT, "workspace too small (scan)");
  // keep the last input (in may alias out)
  if (total_dev)
    HB_CUDA_TRY(cudaMemcpyAsync(last_in, in + n - 1, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
  k_scan_tiles<<<(unsigned)ntiles, kScanBlock, 0, st>>>(in, out, n, sums);
  HB_LAUNCH_CHECK();
  if (ntiles > 1) {
    int rc = exclusive_scan_i64(sums, sums, ntiles, nullptr, ws, st, err);
    if (rc) return rc;
    k_scan_add<<<(unsigned)ntiles, 256, 0, st>>>(out, n, sums);
    HB_LAUNCH_CHECK();
  }
  if (total_dev) {
    k_scan_total<<<1, 1, 0, st>>>(last_in, out + n - 1, total_dev);
    HB_LAUNCH_CHECK();
  }
  return HB_OK;
}

// ------------------------------------------------------------ radix sort
constexpr int kRadixBlock = 256;
constexpr int kRadixItems = 4;
constexpr int kRadixTile = kRadixBlock * kRadixItems;  // striped: item k of thread t = k*256+t

__global__ void k_radix_hist(const uint64_t* keys, int64_t n, int shift, int64_t ntiles,
                             int64_t* counts) {
  __shared__ int hist[256];
  hist[threadIdx.x] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * kRadixTile;
#pragma unroll
  for (int k = 0; k < kRadixItems; ++k) {
    int64_t i = base + k * kRadixBlock + threadIdx.x;
    if (i < n) atomicAdd(&hist[(keys[i] >> shift) & 255u], 1);
  }
  __syncthreads();
  counts[(int64_t)threadIdx.x * ntiles + blockIdx.x] = hist[threadIdx.x];
}

__global__ void k_radix_scatter(const uint64_t* keys, const uint32_t* vals, uint64_t* okeys,
                                uint32_t* ovals, int64_t n, int shift, int64_t ntiles,
                                const int64_t* offsets) {
  constexpr int NW = kRadixBlock / 32;
  __shared__ int warp_cnt[NW][256];
  __shared__ int64_t running[256];
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  running[threadIdx.x] = offsets[(int64_t)threadIdx.x * ntiles + blockIdx.x];
  int64_t base = (int64_t)blockIdx.x * kRadixTile;
  for (int k = 0; k < kRadixItems; ++k) {
#pragma unroll
    for (int w = 0; w < NW; ++w) warp_cnt[w][threadIdx.x] = 0;
    __syncthreads();
    int64_t i = base + k * kRadixBlock + threadIdx.x;
    bool live = i < n;
    uint64_t key = live ? keys[i] : 0;
    unsigned d = live ? (unsigned)((key >> shift) & 255u) : 256u + lane;  // dead lanes unique
    unsigned peers = __match_any_sync(0xffffffffu, d);
    int rank = __popc(peers & lanemask_lt());
    if (live && rank == 0) warp_cnt[wid][d] = __popc(peers);
    __syncthreads();
    {  // thread t owns digit t: exclusive prefix over warps
      int64_t r = running[threadIdx.x];
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        int c = warp_cnt[w][threadIdx.x];
        warp_cnt[w][threadIdx.x] = (int)(r - running[threadIdx.x]);
        r += c;
      }
      __syncthreads();
      if (live) {
        int64_t dst = running[d] + warp_cnt[wid][d] + rank;
        okeys[dst] = key;
        ovals[dst] = vals[i];
      }
      __syncthreads();
      running[threadIdx.x] = r;
    }
  }
}

int radix_sort_u64_u32(uint64_t* keys, uint32_t* vals, int64_t n, int bits, Arena& ws,
                       cudaStream_t st, HbError* err) {
  int64_t ntiles = (n + kRadixTile - 1) / kRadixTile;
  if (ntiles < 1) ntiles = 1;
  uint64_t* k2 = ws.take<uint64_t>(n);
  uint32_t* v2 = ws.take<uint32_t>(n);
  int64_t* counts = ws.take<int64_t>(256 * ntiles);
  if (ws.dry) {
    Arena sub = ws;
    exclusive_scan_i64(nullptr, nullptr, 256 * ntiles, nullptr, sub, st, err);
    ws.used = sub.used;
    return HB_OK;
  }
  if (!ws.ok()) return set_err(err, HB_CONTRACT, "workspace too small (radix)");
  if (n <= 1) return HB_OK;
  int passes = (bits + 7) / 8;
  if (passes < 1) passes = 1;
  uint64_t *ka = keys, *kb = k2;
  uint32_t *va = vals, *vb = v2;
  for (int p = 0; p < passes; ++p) {
    int shift = 8 * p;
    k_radix_hist<<<(unsigned)ntiles, kRadixBlock, 0, st>>>(ka, n, shift, ntiles, counts);
    HB_LAUNCH_CHECK();
    Arena sub = ws;
    int rc = exclusive_scan_i64(counts, counts, 256 * ntiles, nullptr, sub, st, err);
    if (rc) return rc;
    k_radix_scatter<<<(unsigned)ntiles, kRadixBlock, 0, st>>>(ka, va, kb, vb, n, shift, ntiles,
                                                              counts);
    HB_LAUNCH_CHECK();
    uint64_t* tk = ka; ka = kb; kb = tk;
    uint32_t* tv = va; va = vb; vb = tv;
  }
  if (ka != keys) {
    HB_CUDA_TRY(cudaMemcpyAsync(keys, ka, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
    HB_CUDA_TRY(cudaMemcpyAsync(vals, va, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
  }
  return HB_OK;
}

}  // namespace hb
