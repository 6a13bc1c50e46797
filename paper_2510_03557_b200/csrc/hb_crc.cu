// hb_crc.cu -- CRC32C (Castagnoli) of device buffers, for the HCKP checkpoint
// codec (hb/tiered_io.py:80-96, hb/crc.py).
//
// CRC is linear over GF(2): for the raw register update R(init, data),
//   R(c, A || B) = Z_|B|(R(c, A)) ^ R(0, B)
// where Z_L is the "shift through L zero bytes" operator, a 32x32 GF(2)
// matrix applied here as 4 byte-indexed tables (4 lookups).  So:
//   1. every thread computes R(0, chunk) of one 1 KiB chunk (slice-by-8 tables
//      in shared memory);
//   2. each block folds its 256 chunk CRCs in order with Z_1KiB (thread 0),
//      the final block's last chunk with Z_tail;
//   3. one thread folds the block CRCs with Z_256KiB (Z for the last block's
//      length) and applies the standard pre/post inversion via Z_total(~0).
// The operators are built on the host by binary powers of the one-byte shift.
#include <cstring>

#include "hb_common.cuh"

namespace hb {

constexpr int kCrcChunk = 1024;   // bytes per thread
constexpr int kCrcBlock = 256;    // chunks per block

struct CrcOps {  // byte tables of Z operators: chunk, last chunk, block, last block
  uint32_t t[4][4][256];
};

__device__ __forceinline__ uint32_t z_apply(const uint32_t (*T)[256], uint32_t v) {
  return T[0][v & 0xFF] ^ T[1][(v >> 8) & 0xFF] ^ T[2][(v >> 16) & 0xFF] ^ T[3][v >> 24];
}

__global__ void __launch_bounds__(kCrcBlock)
k_crc_chunks(const uint8_t* data, int64_t n, const uint32_t* slice8, const CrcOps* ops,
             uint32_t* block_crc) {
  __shared__ uint32_t s_tab[8][256];
  __shared__ uint32_t s_crc[kCrcBlock];
  for (int k = threadIdx.x; k < 8 * 256; k += blockDim.x) s_tab[k >> 8][k & 255] = slice8[k];
  __syncthreads();
  int64_t chunk = (int64_t)blockIdx.x * kCrcBlock + threadIdx.x;
  int64_t b0 = chunk * kCrcChunk;
  uint32_t c = 0;
  if (b0 < n) {
    int64_t len = n - b0 < kCrcChunk ? n - b0 : kCrcChunk;
    const uint8_t* p = data + b0;
    int64_t k = 0;
    if (((uintptr_t)p & 7) == 0) {
      for (; k + 8 <= len; k += 8) {
        uint64_t w = *(const uint64_t*)(p + k);
        uint32_t lo = c ^ (uint32_t)w, hi = (uint32_t)(w >> 32);
        c = s_tab[7][lo & 0xFF] ^ s_tab[6][(lo >> 8) & 0xFF] ^ s_tab[5][(lo >> 16) & 0xFF] ^
            s_tab[4][lo >> 24] ^ s_tab[3][hi & 0xFF] ^ s_tab[2][(hi >> 8) & 0xFF] ^
            s_tab[1][(hi >> 16) & 0xFF] ^ s_tab[0][hi >> 24];
      }
    }
    for (; k < len; ++k) c = (c >> 8) ^ s_tab[0][(c ^ p[k]) & 0xFF];
  }
  s_crc[threadIdx.x] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t first = (int64_t)blockIdx.x * kCrcBlock;
    int64_t n_chunks = (n + kCrcChunk - 1) / kCrcChunk;
    uint32_t acc = 0;
    for (int t = 0; t < kCrcBlock && first + t < n_chunks; ++t) {
      bool tail = first + t == n_chunks - 1 && (n % kCrcChunk) != 0;
      acc = z_apply(ops->t[tail ? 1 : 0], acc) ^ s_crc[t];
    }
    block_crc[blockIdx.x] = acc;
  }
}

__global__ void k_crc_blocks(const uint32_t* block_crc, int64_t n_blocks, const CrcOps* ops,
                             uint32_t z_init, uint32_t* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  uint32_t acc = 0;
  for (int64_t b = 0; b < n_blocks; ++b)
    acc = z_apply(ops->t[b == n_blocks - 1 ? 3 : 2], acc) ^ block_crc[b];
  *out = (z_init ^ acc) ^ 0xFFFFFFFFu;
}

// ---- host: GF(2) operators ----------------------------------------------------
using Mat = uint32_t[32];  // column j = image of bit j

static uint32_t mat_times(const uint32_t* m, uint32_t v) {
  uint32_t s = 0;
  for (int j = 0; v; ++j, v >>= 1)
    if (v & 1) s ^= m[j];
  return s;
}
static void mat_mul(const uint32_t* a, const uint32_t* b, uint32_t* out) {  // out = a * b
  uint32_t tmp[32];
  for (int j = 0; j < 32; ++j) tmp[j] = mat_times(a, b[j]);
  memcpy(out, tmp, sizeof(tmp));
}
// Z_L: shift a raw CRC register through L zero bytes
static void z_operator(uint64_t L, uint32_t* out) {
  uint32_t bit[32], byte8[32];
  bit[0] = 0x82F63B78u;  // one zero bit (reflected polynomial)
  for (int j = 1; j < 32; ++j) bit[j] = 1u << (j - 1);
  mat_mul(bit, bit, byte8);      // 2 bits
  mat_mul(byte8, byte8, byte8);  // 4 bits
  mat_mul(byte8, byte8, byte8);  // 8 bits = one byte
  uint32_t res[32];
  for (int j = 0; j < 32; ++j) res[j] = 1u << j;  // identity
  uint32_t p[32];
  memcpy(p, byte8, sizeof(p));
  while (L) {
    if (L & 1) mat_mul(p, res, res);
    L >>= 1;
    if (L) mat_mul(p, p, p);
  }
  memcpy(out, res, sizeof(res));
}
static void z_tables(uint64_t L, uint32_t (*T)[256]) {
  uint32_t m[32];
  z_operator(L, m);
  for (int b = 0; b < 4; ++b)
    for (int v = 0; v < 256; ++v) T[b][v] = mat_times(m, (uint32_t)v << (8 * b));
}

}  // namespace hb

using namespace hb;

extern "C" size_t hb_crc32c_device_workspace(int64_t nbytes) {
  int64_t n_chunks = (nbytes + kCrcChunk - 1) / kCrcChunk;
  int64_t n_blocks = (n_chunks + kCrcBlock - 1) / kCrcBlock;
  return sizeof(CrcOps) + 8 * 256 * sizeof(uint32_t) + (n_blocks + 2) * sizeof(uint32_t) + 1024;
}

extern "C" int hb_crc32c_device(const void* data, int64_t nbytes, uint32_t* out_host, void* wsp,
                                size_t ws_bytes, void* stream, HbError* err) {
  if (err) *err = HbError{};
  cudaStream_t st = (cudaStream_t)stream;
  if (ws_bytes < hb_crc32c_device_workspace(nbytes))
    return set_err(err, HB_CONTRACT, "workspace too small (crc32c)");
  if (nbytes <= 0) {
    *out_host = 0;
    return HB_OK;
  }
  int64_t n_chunks = (nbytes + kCrcChunk - 1) / kCrcChunk;
  int64_t n_blocks = (n_chunks + kCrcBlock - 1) / kCrcBlock;
  // host staging, per calling thread (the call synchronises before it returns,
  // so one thread's buffers are never read by an earlier call's pending copy)
  thread_local CrcOps ops;
  thread_local uint32_t slice8[8][256];
  thread_local bool slice_ready = false;
  if (!slice_ready) {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c >> 1) ^ ((c & 1u) ? 0x82F63B78u : 0u);
      slice8[0][i] = c;
    }
    for (uint32_t i = 0; i < 256; ++i)
      for (int t = 1; t < 8; ++t) slice8[t][i] = (slice8[t - 1][i] >> 8) ^ slice8[0][slice8[t - 1][i] & 0xFF];
    slice_ready = true;
  }
  int64_t tail = nbytes % kCrcChunk ? nbytes % kCrcChunk : kCrcChunk;
  int64_t last_block = nbytes - (n_blocks - 1) * (int64_t)kCrcChunk * kCrcBlock;
  z_tables(kCrcChunk, ops.t[0]);
  z_tables((uint64_t)tail, ops.t[1]);
  z_tables((uint64_t)kCrcChunk * kCrcBlock, ops.t[2]);
  z_tables((uint64_t)last_block, ops.t[3]);
  uint32_t zt[32];
  z_operator((uint64_t)nbytes, zt);
  uint32_t z_init = mat_times(zt, 0xFFFFFFFFu);
  char* base = (char*)wsp;
  CrcOps* d_ops = (CrcOps*)base;
  uint32_t* d_slice = (uint32_t*)(base + sizeof(CrcOps));
  uint32_t* d_blocks = d_slice + 8 * 256;
  uint32_t* d_out = d_blocks + n_blocks;
  HB_CUDA_TRY(cudaMemcpyAsync(d_ops, &ops, sizeof(ops), cudaMemcpyHostToDevice, st));
  HB_CUDA_TRY(cudaMemcpyAsync(d_slice, slice8, sizeof(slice8), cudaMemcpyHostToDevice, st));
  k_crc_chunks<<<(unsigned)n_blocks, kCrcBlock, 0, st>>>((const uint8_t*)data, nbytes, d_slice,
                                                        d_ops, d_blocks);
  HB_LAUNCH_CHECK();
  k_crc_blocks<<<1, 32, 0, st>>>(d_blocks, n_blocks, d_ops, z_init, d_out);
  HB_LAUNCH_CHECK();
  HB_CUDA_TRY(cudaMemcpyAsync(out_host, d_out, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  HB_CUDA_TRY(cudaStreamSynchronize(st));
  return HB_OK;
}
