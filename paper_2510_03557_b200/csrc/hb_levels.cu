// hb_levels.cu -- per-particle timestep levels and leaf levels
// (assign_timestep_levels, hb/hydro.py:277-317), on the device.
//
// Row pass: dt_i from the reference's float64 expressions in its evaluation
// order (numpy evaluates left to right; |v| = sqrt((vx^2 + vy^2) + vz^2) as
// np.linalg.norm's add.reduce over a length-3 row):
//   gas: cs = sqrt(max((gamma (gamma - 1)) u, 0)); speed = (cs + |v|) + 1e-300;
//        dt = (cfl h) / speed                                  (hydro.py:289-293)
//   DM:  dt = cfl sqrt(eps / max(|a|, 1e-300))                 (hydro.py:294-298)
//   level = ceil(log2(dt_pm / dt) - 1e-12) where dt_pm / dt > 1, else 0
// Leaf pass: one warp per leaf, level max over members (np.maximum.reduceat on
// leaf_start); the maxima over all rows, all leaves and the active (not
// ghost-only) leaves land in dev_max[0..2] for the host's StiffStateError test
// and the hierarchy depth.  No contraction: every product and sum is rounded
// as numpy rounds it.
#include "hb_internal.cuh"

namespace hb {

__global__ void k_row_levels(int64_t n, const double* vel, const double* u, const double* h,
                             const double* accel, const uint8_t* species, double cfl, double eps,
                             double gamma, double dt_pm, uint8_t* level, int64_t* dev_max) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int lv = 0;
  if (i < n) {
    double dt;
    if (species[i] == 1) {
      double gm1 = __dsub_rn(gamma, 1.0);
      double cs = sqrt(fmax(__dmul_rn(__dmul_rn(gamma, gm1), u[i]), 0.0));
      const double* v = vel + 3 * i;
      double vn = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(v[0], v[0]), __dmul_rn(v[1], v[1])),
                                 __dmul_rn(v[2], v[2])));
      double speed = __dadd_rn(__dadd_rn(cs, vn), 1e-300);
      dt = __ddiv_rn(__dmul_rn(cfl, h[i]), speed);
    } else {
      const double* a = accel + 3 * i;
      double am = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(a[0], a[0]), __dmul_rn(a[1], a[1])),
                                 __dmul_rn(a[2], a[2])));
      dt = __dmul_rn(cfl, sqrt(__ddiv_rn(eps, fmax(am, 1e-300))));
    }
    double ratio = __ddiv_rn(dt_pm, dt);
    if (ratio > 1.0) lv = (int)ceil(__dsub_rn(log2(ratio), 1e-12));
    level[i] = (uint8_t)min(lv, 255);
  }
  int m = lv;
#pragma unroll
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0) atomicMax((unsigned long long*)&dev_max[0], (unsigned long long)m);
}

__global__ void k_leaf_levels(int64_t n_leaves, const int64_t* leaf_start, const int64_t* leaf_end,
                              const uint8_t* ghost_only, const uint8_t* level, int64_t* leaf_level,
                              int64_t* dev_max) {
  int64_t leaf = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (leaf >= n_leaves) return;
  int m = 0;
  for (int64_t r = leaf_start[leaf] + lane; r < leaf_end[leaf]; r += 32) m = max(m, (int)level[r]);
#pragma unroll
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) {
    leaf_level[leaf] = m;
    if (m > 0) {
      atomicMax((unsigned long long*)&dev_max[1], (unsigned long long)m);
      if (!ghost_only[leaf]) atomicMax((unsigned long long*)&dev_max[2], (unsigned long long)m);
    }
  }
}

__global__ void k_fill_i64(int64_t n, int64_t* out, const int64_t* value) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = *value;
}

}  // namespace hb

using namespace hb;

// dev_max: 3 int64 device words (row max, leaf max, active-leaf max), copied
// to max_host before returning (one stream sync)
extern "C" int hb_timestep_levels(int64_t n, const double* vel, const double* internal_energy,
                                  const double* smoothing, const double* accel,
                                  const uint8_t* species, double cfl, double softening,
                                  double eos_gamma, double dt_pm, int64_t n_leaves,
                                  const int64_t* leaf_start, const int64_t* leaf_end,
                                  const uint8_t* leaf_ghost_only, int32_t flat, uint8_t* level,
                                  int64_t* leaf_level, int64_t* dev_max, int64_t* max_host,
                                  void* stream, HbError* err) {
  if (err) *err = HbError{};
  cudaStream_t st = (cudaStream_t)stream;
  HB_CUDA_TRY(cudaMemsetAsync(dev_max, 0, 3 * sizeof(int64_t), st));
  if (n > 0) {
    k_row_levels<<<grid_for(n, 256), 256, 0, st>>>(n, vel, internal_energy, smoothing, accel,
                                                   species, cfl, softening, eos_gamma, dt_pm,
                                                   level, dev_max);
    HB_LAUNCH_CHECK();
  }
  if (n_leaves > 0) {
    k_leaf_levels<<<grid_for(n_leaves * 32, 256), 256, 0, st>>>(
        n_leaves, leaf_start, leaf_end, leaf_ghost_only, level, leaf_level, dev_max);
    HB_LAUNCH_CHECK();
    if (flat) {  // every leaf at the global deepest level (hydro.py:311-312)
      k_fill_i64<<<grid_for(n_leaves, 256), 256, 0, st>>>(n_leaves, leaf_level, dev_max + 1);
      HB_LAUNCH_CHECK();
    }
  }
  HB_CUDA_TRY(cudaMemcpyAsync(max_host, dev_max, 3 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  HB_CUDA_TRY(cudaStreamSynchronize(st));
  return HB_OK;
}
