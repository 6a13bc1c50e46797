// hb_common.cuh -- shared device helpers for the B200 short-range engine.
//
// Everything here is sm_100a CUDA C++; no library kernels.  The C-ABI lives in
// hb_api.cu and is declared in include/hb.h.
#pragma once
#include <cstdint>
#include <cstddef>
#include <cuda_runtime.h>

#include "../../include/hb.h"

namespace hb {

constexpr int kWarp = 32;

// ---- workspace: bump allocator over one caller-owned device arena -----------
struct Arena {
  char* base = nullptr;
  size_t cap = 0;
  size_t used = 0;
  bool dry = false;  // size query: count bytes, hand out nullptr
  template <class T>
  T* take(size_t count) {
    size_t bytes = (count * sizeof(T) + 255) & ~size_t(255);
    size_t off = used;
    used += bytes;
    if (dry || base == nullptr) return nullptr;
    if (used > cap) return nullptr;
    return reinterpret_cast<T*>(base + off);
  }
  bool ok() const { return dry || used <= cap; }
};

// ---- status plumbing ---------------------------------------------------------
inline int set_err(HbError* e, int status, const char* msg, int cuda_err = 0) {
  if (e) {
    e->status = status;
    e->cuda_err = cuda_err;
    int k = 0;
    for (; msg && msg[k] && k < (int)sizeof(e->msg) - 1; ++k) e->msg[k] = msg[k];
    e->msg[k] = 0;
  }
  return status;
}

#define HB_CUDA_TRY(expr)                                                   \
  do {                                                                      \
    cudaError_t _e = (expr);                                                \
    if (_e != cudaSuccess) return ::hb::set_err(err, HB_CUDA, cudaGetErrorString(_e), (int)_e); \
  } while (0)

extern unsigned long long g_launches;  // kernels launched (hb_crk.cu)
#define HB_COUNT_LAUNCH(k) (::hb::g_launches += (k))
#define HB_LAUNCH_CHECK()                                                   \
  do {                                                                      \
    ::hb::g_launches += 1;                                                  \
    cudaError_t _e = cudaGetLastError();                                    \
    if (_e != cudaSuccess) return ::hb::set_err(err, HB_CUDA, cudaGetErrorString(_e), (int)_e); \
  } while (0)

inline unsigned grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  return (unsigned)(g < 1 ? 1 : g);
}

// ---- exact double arithmetic (no contraction) for reference predicates -------
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// order-preserving map float -> uint (total order; NaN sorts last by sign)
__device__ __forceinline__ unsigned sortable_key(float f) {
  unsigned u = __float_as_uint(f);
  return u ^ ((unsigned)((int)u >> 31) | 0x80000000u);
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---- device-wide primitives (hb_sort.cu) --------------------------------------
// Exclusive scan of n int64 values (in -> out may alias); writes total to *total_dev if given.
int exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, int64_t* total_dev,
                       Arena& ws, cudaStream_t st, HbError* err);
// Stable LSD radix sort of (key, val) by the low `bits` bits of key.  Result in
// keys/vals (the alt buffers are scratch from ws).
int radix_sort_u64_u32(uint64_t* keys, uint32_t* vals, int64_t n, int bits, Arena& ws,
                       cudaStream_t st, HbError* err);

}  // namespace hb
