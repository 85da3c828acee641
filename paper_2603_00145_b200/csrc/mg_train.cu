// mg_train.cu -- O(N) / O(B) kernels around the pair kernels:
//   forward finish (PSF tap reduction)
//   backward point prep (upstream, d_points)      _kernels.py:131-144
//   backward epilogue chain rule                  render.py:319-340, 207-243
//   transform gradients                           render.py:246-273
//   smooth-L1 loss + gradient                     train.py:108-120
//   fused epilogue + aniso + Adam                 train.py:128-147, 239-271, 457-474
//   progressive lattice upsample                  train.py:157-218
#include "mg_render.cuh"

namespace mg {

static inline unsigned gridn(int64_t n, int t = 256) {
  int64_t b = (n + t - 1) / t;
  int64_t cap = (int64_t)num_sms() * 16;
  if (b > cap) b = cap;
  return (unsigned)(b < 1 ? 1 : b);
}

#define GRID_LOOP(i, n) for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

// ---------------------------------------------------------------------------
// Forward finish: I_b = sum_t w_t I_(b,t); counts summed over taps.
// ---------------------------------------------------------------------------
__global__ void forward_finish_kernel(const float4* __restrict__ out4, const int* __restrict__ cnt,
                                      const int* __restrict__ inv, int64_t b, int ntaps,
                                      const double* __restrict__ tap_w, double* __restrict__ out_i,
                                      float* __restrict__ out_i32, int64_t* __restrict__ out_cnt,
                                      unsigned long long* __restrict__ pair_total) {
  unsigned long long mine = 0;
  GRID_LOOP(pb, b) {
    double acc = 0.0;
    int64_t c = 0;
    for (int t = 0; t < ntaps; ++t) {
      int p = inv[pb * ntaps + t];
      double w = tap_w ? tap_w[t] : 1.0;
      acc += w * (double)out4[p].w;
      c += cnt[p];
    }
    if (out_i) out_i[pb] = acc;
    if (out_i32) out_i32[pb] = (float)acc;
    if (out_cnt) out_cnt[pb] = c;
    mine += (unsigned long long)c;
  }
  if (pair_total) {  // whole-launch pair count (integer: order-independent)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(pair_total, mine);
  }
}

__global__ void gather_batch_kernel(const int64_t* __restrict__ idx, int64_t n, const double* __restrict__ pc,
                                    const int64_t* __restrict__ ps, const float* __restrict__ pt,
                                    double* __restrict__ c, int64_t* __restrict__ s, float* __restrict__ t) {
  GRID_LOOP(i, n) {
    const int64_t j = idx[i];
    c[3 * i + 0] = pc[3 * j + 0];
    c[3 * i + 1] = pc[3 * j + 1];
    c[3 * i + 2] = pc[3 * j + 2];
    s[i] = ps[j];
    t[i] = pt[j];
  }
}

// Upstream per sub-point u_(b,t) = w_t * u_b into the point records; the
// gradient w.r.t. the transformed sub-point is h = -u * H (H from forward).
__global__ void backward_points_kernel(const double* __restrict__ up64, const float* __restrict__ up32,
                                       const int* __restrict__ inv, int64_t b, int ntaps,
                                       const double* __restrict__ tap_w, const float4* __restrict__ out4,
                                       float4* __restrict__ prec, double* __restrict__ dpoints) {
  GRID_LOOP(j, b * ntaps) {
    int64_t pb = j / ntaps;
    int t = (int)(j - pb * ntaps);
    double u = up64 ? up64[pb] : (double)up32[pb];
    double us = u * (tap_w ? tap_w[t] : 1.0);
    int p = inv[j];
    prec[p].w = (float)(us * kWeightScaleD);  // u' = u / kCutScale (FTZ cutoff, mg_common.cuh)
    if (dpoints) {
      float4 H = out4[p];
      dpoints[3 * j + 0] = -us * (double)H.x;
      dpoints[3 * j + 1] = -us * (double)H.y;
      dpoints[3 * j + 2] = -us * (double)H.z;
    }
  }
}

// ---------------------------------------------------------------------------
// Epilogue helpers (float64)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void rot_quat_grad(const double g[9], double w, double x, double y, double z,
                                              double out[4]) {
  // render.py:207-235, g row-major (a, b) -> g[3a+b]
  out[0] = 2.0 * (-z * g[1] + y * g[2] + z * g[3] - x * g[5] - y * g[6] + x * g[7]);
  out[1] = 2.0 * (y * g[1] + z * g[2] + y * g[3] - 2.0 * x * g[4] - w * g[5] + z * g[6] + w * g[7] - 2.0 * x * g[8]);
  out[2] = 2.0 * (-2.0 * y * g[0] + x * g[1] + w * g[2] + x * g[3] + z * g[5] - w * g[6] + z * g[7] - 2.0 * y * g[8]);
  out[3] = 2.0 * (-2.0 * z * g[0] - w * g[1] + x * g[2] + w * g[3] - 2.0 * z * g[4] + y * g[5] + x * g[6] + y * g[7]);
}

__device__ __forceinline__ void quat_rot_d2(double w, double x, double y, double z, double R[9]) {
  R[0] = 1.0 - 2.0 * (y * y + z * z);
  R[1] = 2.0 * (x * y - w * z);
  R[2] = 2.0 * (x * z + w * y);
  R[3] = 2.0 * (x * y + w * z);
  R[4] = 1.0 - 2.0 * (x * x + z * z);
  R[5] = 2.0 * (y * z - w * x);
  R[6] = 2.0 * (x * z - w * y);
  R[7] = 2.0 * (y * z + w * x);
  R[8] = 1.0 - 2.0 * (x * x + y * y);
}

struct GaussGrad {
  double dmu[3], dq[4], ds[3], dl;
};

// Full chain for one Gaussian from the reference-convention accumulators.
__device__ __forceinline__ GaussGrad chain_one(const double dmu[3], const double dab[6], double dalpha, double qw,
                                               double qx, double qy, double qz, const double s_raw[3],
                                               double logit) {
  GaussGrad o;
  double nrm = sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
  double w = qw / nrm, x = qx / nrm, y = qy / nrm, z = qz / nrm;
  double R[9];
  quat_rot_d2(w, x, y, z, R);
  double e[3];
  for (int a = 0; a < 3; ++a) {
    double s = s_raw[a] < -20.0 ? -20.0 : (s_raw[a] > 20.0 ? 20.0 : s_raw[a]);
    e[a] = exp(-2.0 * s);
  }
  double A[9] = {dab[0], dab[1], dab[2], dab[1], dab[3], dab[4], dab[2], dab[4], dab[5]};
  double AR[9];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) AR[3 * a + b] = A[3 * a] * R[b] + A[3 * a + 1] * R[3 + b] + A[3 * a + 2] * R[6 + b];
  for (int k = 0; k < 3; ++k) {
    double de = R[k] * AR[k] + R[3 + k] * AR[3 + k] + R[6 + k] * AR[6 + k];
    o.ds[k] = (fabs(s_raw[k]) > 20.0) ? 0.0 : -2.0 * e[k] * de;
  }
  double grot[9];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) grot[3 * a + b] = 2.0 * AR[3 * a + b] * e[b];
  double dqh[4];
  rot_quat_grad(grot, w, x, y, z, dqh);
  double inner = dqh[0] * w + dqh[1] * x + dqh[2] * y + dqh[3] * z;
  o.dq[0] = (dqh[0] - inner * w) / nrm;
  o.dq[1] = (dqh[1] - inner * x) / nrm;
  o.dq[2] = (dqh[2] - inner * y) / nrm;
  o.dq[3] = (dqh[3] - inner * z) / nrm;
  double alpha = 1.0 / (1.0 + exp(-logit));
  o.dl = dalpha * alpha * (1.0 - alpha);
  o.dmu[0] = dmu[0];
  o.dmu[1] = dmu[1];
  o.dmu[2] = dmu[2];
  return o;
}

// acc10 (kernel convention, sorted order) -> reference accumulators.
__device__ __forceinline__ void acc_to_ref(const float* a, double alpha, double dmu[3], double dab[6], double* dal) {
  *dal = (double)a[0];
  const double sc = alpha / kMScaleD;
  dmu[0] = sc * (double)a[1];
  dmu[1] = sc * (double)a[2];
  dmu[2] = sc * (double)a[3];
  for (int k = 0; k < 6; ++k) dab[k] = -0.5 * alpha * (double)a[4 + k];
}

// Reference block_backward ABI: d_mu/d_abar6/d_alpha are ACCUMULATED into
// (caller-zeroed, render.py:300-302), alpha given as float64.
__global__ void acc_to_ref_kernel(const float* __restrict__ acc10, const int* __restrict__ order, int64_t n,
                                  const double* __restrict__ alpha64, double* __restrict__ d_mu,
                                  double* __restrict__ d_abar6, double* __restrict__ d_alpha) {
  GRID_LOOP(p, n) {
    int64_t i = order[p];
    double dmu[3], dab[6], dal;
    acc_to_ref(acc10 + 10 * p, alpha64[i], dmu, dab, &dal);
    for (int a = 0; a < 3; ++a) d_mu[3 * i + a] += dmu[a];
    for (int k = 0; k < 6; ++k) d_abar6[6 * i + k] += dab[k];
    d_alpha[i] += dal;
  }
}

// Full epilogue to parameter gradients (RenderGradients fields, float64).
__global__ void epilogue_kernel(const float* __restrict__ acc10, const int* __restrict__ order, int64_t n,
                                const float* __restrict__ quat, const float* __restrict__ ls,
                                const float* __restrict__ lg, double* __restrict__ d_pos, double* __restrict__ d_q,
                                double* __restrict__ d_s, double* __restrict__ d_l) {
  GRID_LOOP(p, n) {
    int64_t i = order[p];
    double logit = lg[i];
    double alpha = 1.0 / (1.0 + exp(-logit));
    double dmu[3], dab[6], dal;
    acc_to_ref(acc10 + 10 * p, alpha, dmu, dab, &dal);
    double s[3] = {ls[3 * i], ls[3 * i + 1], ls[3 * i + 2]};
    GaussGrad gg = chain_one(dmu, dab, dal, quat[4 * i], quat[4 * i + 1], quat[4 * i + 2], quat[4 * i + 3], s, logit);
    for (int a = 0; a < 3; ++a) d_pos[3 * i + a] = gg.dmu[a];
    for (int a = 0; a < 4; ++a) d_q[4 * i + a] = gg.dq[a];
    for (int a = 0; a < 3; ++a) d_s[3 * i + a] = gg.ds[a];
    d_l[i] = gg.dl;
  }
}

// Chain rule from float64 reference-convention accumulators (primitive order).
__global__ void epilogue_f64_kernel(const double* __restrict__ d_mu, const double* __restrict__ d_abar6,
                                    const double* __restrict__ d_alpha, const double* __restrict__ quat,
                                    const double* __restrict__ ls, const double* __restrict__ lg, int64_t n,
                                    double* __restrict__ d_pos, double* __restrict__ d_q, double* __restrict__ d_s,
                                    double* __restrict__ d_l) {
  GRID_LOOP(i, n) {
    double s[3] = {ls[3 * i], ls[3 * i + 1], ls[3 * i + 2]};
    GaussGrad gg = chain_one(d_mu + 3 * i, d_abar6 + 6 * i, d_alpha[i], quat[4 * i], quat[4 * i + 1], quat[4 * i + 2],
                             quat[4 * i + 3], s, lg[i]);
    for (int a = 0; a < 3; ++a) d_pos[3 * i + a] = gg.dmu[a];
    for (int a = 0; a < 4; ++a) d_q[4 * i + a] = gg.dq[a];
    for (int a = 0; a < 3; ++a) d_s[3 * i + a] = gg.ds[a];
    d_l[i] = gg.dl;
  }
}

// ---------------------------------------------------------------------------
// Transform gradients: per slice sums of h and h (x) c over sub-points
// (render.py:246-273), then the quaternion chain.
// ---------------------------------------------------------------------------
// Each thread walks a contiguous chunk of sub-points, accumulating in float64
// registers while the slice id is unchanged (the taps of a point, and the
// per-step SSIM slice, are contiguous runs).  Completed runs flush 12 sums
// with global fp64 atomics; the run still open at the end of the chunk is
// first reduced across the warp when all 32 lanes share its slice (the SSIM
// slice range), which removes the same-address atomic contention there.
__global__ void transform_reduce_kernel(const double* __restrict__ dpoints, const double* __restrict__ coords,
                                        const int64_t* __restrict__ sids, int64_t b, int ntaps,
                                        const double* __restrict__ tap_off, const double* __restrict__ dirs, int k,
                                        double* __restrict__ out12) {
  constexpr int CH = 8;
  const int64_t total = b * ntaps;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  const int64_t nloop = (total + CH * nthreads - 1) / (CH * nthreads);
  for (int64_t it = 0; it < nloop; ++it) {
    const int64_t c0 = (it * nthreads + (int64_t)blockIdx.x * blockDim.x + threadIdx.x) * CH;
    const int64_t c1 = min(total, c0 + CH);
    int64_t cur = -1;
    double acc[12];
#pragma unroll
    for (int i = 0; i < 12; ++i) acc[i] = 0.0;
    for (int64_t j = c0; j < c1; ++j) {
      const int64_t pb = j / ntaps;
      const int t = (int)(j - pb * ntaps);
      const int64_t s = sids[pb];
      if (s < 0 || s >= k) continue;
      if (s != cur) {
        if (cur >= 0) {
#pragma unroll
          for (int i = 0; i < 12; ++i)
            if (acc[i] != 0.0) atomicAdd(out12 + 12 * cur + i, acc[i]);
        }
#pragma unroll
        for (int i = 0; i < 12; ++i) acc[i] = 0.0;
        cur = s;
      }
      double c[3] = {coords[3 * pb], coords[3 * pb + 1], coords[3 * pb + 2]};
      if (tap_off) {
        const double o = tap_off[t];
#pragma unroll
        for (int a = 0; a < 3; ++a) c[a] = __dadd_rn(c[a], __dmul_rn(o, dirs[3 * s + a]));
      }
      const double h[3] = {dpoints[3 * j], dpoints[3 * j + 1], dpoints[3 * j + 2]};
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        acc[a] += h[a];
#pragma unroll
        for (int bb = 0; bb < 3; ++bb) acc[3 + 3 * a + bb] += h[a] * c[bb];
      }
    }
    // open run: warp-reduce when the whole warp shares its slice
    const long long key = (long long)cur;
    const unsigned peers = __match_any_sync(MG_FULL, key);
    if (peers == MG_FULL) {
      if (cur >= 0) {
#pragma unroll
        for (int i = 0; i < 12; ++i) {
          double v = acc[i];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(MG_FULL, v, o);
          acc[i] = v;
        }
        if ((threadIdx.x & 31) == 0) {
#pragma unroll
          for (int i = 0; i < 12; ++i)
            if (acc[i] != 0.0) atomicAdd(out12 + 12 * cur + i, acc[i]);
        }
      }
    } else if (cur >= 0) {
#pragma unroll
      for (int i = 0; i < 12; ++i)
        if (acc[i] != 0.0) atomicAdd(out12 + 12 * cur + i, acc[i]);
    }
  }
}

// Deterministic version: block b owns a contiguous range of sub-points, split
// into one contiguous sub-range per warp.  Each warp keeps its own per-slice
// 12-sum table in shared memory; 32 sub-points at a time, the lanes of one
// slice are summed by their lowest lane in lane order (a butterfly when the
// whole warp shares the slice).  The block adds its warps' tables in warp
// order into partials[b]; transform_finish_kernel then reduces the partials
// in a fixed order.  Same result on every run, no fp64 atomics.
__device__ __forceinline__ void transform_contrib(const double* __restrict__ dpoints, const double* __restrict__ coords,
                                                  const int64_t* __restrict__ sids, int ntaps,
                                                  const double* __restrict__ tap_off, const double* __restrict__ dirs,
                                                  int k, int64_t j, int& key, double (&v)[12]) {
  const int64_t pb = j / ntaps;
  const int t = (int)(j - pb * ntaps);
  const int64_t s = sids[pb];
  key = (s < 0 || s >= k) ? -1 : (int)s;
  double c[3] = {coords[3 * pb], coords[3 * pb + 1], coords[3 * pb + 2]};
  if (tap_off && key >= 0) {
    const double o = tap_off[t];
#pragma unroll
    for (int a = 0; a < 3; ++a) c[a] = __dadd_rn(c[a], __dmul_rn(o, dirs[3 * s + a]));
  }
  const double h[3] = {dpoints[3 * j], dpoints[3 * j + 1], dpoints[3 * j + 2]};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    v[a] = h[a];
#pragma unroll
    for (int bb = 0; bb < 3; ++bb) v[3 + 3 * a + bb] = h[a] * c[bb];
  }
}

__global__ void transform_reduce_det_kernel(const double* __restrict__ dpoints, const double* __restrict__ coords,
                                            const int64_t* __restrict__ sids, int64_t b, int ntaps,
                                            const double* __restrict__ tap_off, const double* __restrict__ dirs, int k,
                                            double* __restrict__ partials) {
  extern __shared__ double tr_sh[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int kk = 12 * k;
  double* table = tr_sh + (size_t)warp * kk;
  double* stage = tr_sh + (size_t)nw * kk + (size_t)warp * 32 * 12;
  for (int e = lane; e < kk; e += 32) table[e] = 0.0;
  __syncwarp();
  const int64_t total = b * ntaps;
  const int64_t per_block = (total + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = (int64_t)blockIdx.x * per_block, b1 = min(total, b0 + per_block);
  const int64_t per_warp = (b1 - b0 + nw - 1) / nw;
  const int64_t w0 = b0 + (int64_t)warp * per_warp, w1 = min(b1, w0 + per_warp);
  for (int64_t j0 = w0; j0 < w1; j0 += 32) {
    const int64_t j = j0 + lane;
    int key = -1;
    double v[12];
#pragma unroll
    for (int c = 0; c < 12; ++c) v[c] = 0.0;
    if (j < w1) transform_contrib(dpoints, coords, sids, ntaps, tap_off, dirs, k, j, key, v);
    const unsigned peers = __match_any_sync(MG_FULL, key);
    if (peers == MG_FULL) {
      if (key >= 0) {
#pragma unroll
        for (int c = 0; c < 12; ++c) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v[c] += __shfl_xor_sync(MG_FULL, v[c], o);
        }
        if (lane == 0) {
#pragma unroll
          for (int c = 0; c < 12; ++c) table[12 * key + c] += v[c];
        }
      }
    } else {
#pragma unroll
      for (int c = 0; c < 12; ++c) stage[12 * lane + c] = v[c];
      __syncwarp();
      if (key >= 0 && lane == __ffs(peers) - 1) {
        double acc[12];
#pragma unroll
        for (int c = 0; c < 12; ++c) acc[c] = 0.0;
        for (unsigned m = peers; m; m &= m - 1) {
          const int l = __ffs(m) - 1;
#pragma unroll
          for (int c = 0; c < 12; ++c) acc[c] += stage[12 * l + c];
        }
#pragma unroll
        for (int c = 0; c < 12; ++c) table[12 * key + c] += acc[c];
      }
    }
    __syncwarp();
  }
  __syncthreads();
  for (int e = threadIdx.x; e < kk; e += blockDim.x) {
    double acc = 0.0;
    for (int w = 0; w < nw; ++w) acc += tr_sh[(size_t)w * kk + e];
    partials[(size_t)blockIdx.x * kk + e] = acc;
  }

}

// Quaternion chain of one slice (render.py:246-273): 12 sums -> (d_q, d_t).
__device__ __forceinline__ void transform_chain_slice(const double* a, const double* __restrict__ tq, int64_t s,
                                                      double* __restrict__ out7, int accumulate) {
  double qw = tq[4 * s], qx = tq[4 * s + 1], qy = tq[4 * s + 2], qz = tq[4 * s + 3];
  double nrm = sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
  double w = qw / nrm, x = qx / nrm, y = qy / nrm, z = qz / nrm;
  double dqh[4];
  rot_quat_grad(a + 3, w, x, y, z, dqh);
  double inner = dqh[0] * w + dqh[1] * x + dqh[2] * y + dqh[3] * z;
  double o[7] = {(dqh[0] - inner * w) / nrm, (dqh[1] - inner * x) / nrm, (dqh[2] - inner * y) / nrm,
                 (dqh[3] - inner * z) / nrm, a[0], a[1], a[2]};
  for (int c = 0; c < 7; ++c) out7[7 * s + c] = accumulate ? out7[7 * s + c] + o[c] : o[c];
}

__global__ void transform_chain_kernel(const double* __restrict__ acc12, const double* __restrict__ tq, int k,
                                       double* __restrict__ out7, int accumulate) {
  GRID_LOOP(s, k) transform_chain_slice(acc12 + 12 * s, tq, s, out7, accumulate);
}

// One warp per slice: lanes stride over the block partials, a fixed-order
// butterfly finishes each of the 12 sums, then lane 0 applies the chain.
__global__ void transform_finish_kernel(const double* __restrict__ partials, int nblk, const double* __restrict__ tq,
                                        int k, double* __restrict__ acc12, double* __restrict__ out7,
                                        int accumulate) {
  const int lane = threadIdx.x & 31;
  const int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (s >= k) return;
  const int kk = 12 * k;
  double v[12];
#pragma unroll
  for (int c = 0; c < 12; ++c) v[c] = 0.0;
  for (int blk = lane; blk < nblk; blk += 32) {
    const double* p = partials + (size_t)blk * kk + 12 * s;
#pragma unroll
    for (int c = 0; c < 12; ++c) v[c] += p[c];
  }
#pragma unroll
  for (int c = 0; c < 12; ++c) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[c] += __shfl_xor_sync(MG_FULL, v[c], o);
  }
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < 12; ++c) acc12[12 * s + c] = v[c];
    transform_chain_slice(v, tq, s, out7, accumulate);
  }
}

// ---------------------------------------------------------------------------
// Smooth-L1 (train.py:108-120): mean Huber (delta 1) and its gradient.
// ---------------------------------------------------------------------------
// DIV: the gradient is g / scale (the reference's `g / x.size`) instead of g * scale.
template <typename T, bool DIV>
__global__ void smooth_l1_kernel(const T* __restrict__ pred, const T* __restrict__ target, int64_t b,
                                 double scale, T* __restrict__ up_out, double* __restrict__ loss_acc) {
  double local = 0.0;
  GRID_LOOP(pb, b) {
    double x = (double)pred[pb] - (double)target[pb];
    double ax = fabs(x);
    local += ax < 1.0 ? 0.5 * x * x : ax - 0.5;
    const double g = ax < 1.0 ? x : (x > 0 ? 1.0 : (x < 0 ? -1.0 : 0.0));
    up_out[pb] = (T)(DIV ? g / scale : g * scale);
  }
  if (DIV) local /= scale;
  __shared__ double s_red[32];
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(MG_FULL, local, o);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = local;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? s_red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(MG_FULL, v, o);
    if (threadIdx.x == 0) atomicAdd(loss_acc, DIV ? v : v * scale);
  }
}

// ---------------------------------------------------------------------------
// Fused: epilogue chain + aniso penalty + Adam on the four Gaussian groups.
// Adam in float64 math, float32 state (train.py:251-271); groups share t.
// ---------------------------------------------------------------------------
struct AdamHyper {
  double lr_pos, lr_quat, lr_scale, lr_logit;
  double beta1, beta2, eps;
  double lambda_aniso, lambda_ratio;
  int use_aniso;
  double bc1, bc2;  // filled in-kernel from the device step counter
};

// Adam (train.py:251-271) with the bias corrections as reciprocals computed
// once per block: m/bc1 -> m * (1/bc1), sqrt(v/bc2) -> sqrt(v) * (1/sqrt(bc2)).
// Evaluated in float32 arithmetic (the state is float32; the chain-rule
// gradient arrives in float64 and is rounded once): the float64 version spent
// a quarter of its stall cycles in F2F conversions.
struct AdamF {
  float b1, a1, b2, a2, eps, bc1, bc2;  // bc1 = 1/(1 - b1^t), bc2 = 1/sqrt(1 - b2^t)
};
__device__ __forceinline__ void adam_upd32(float& p, float& m, float& v, double g64, float lr, const AdamF& h) {
  const float g = (float)g64;
  const float mm = fmaf(h.b1, m, h.a1 * g);
  const float vv = fmaf(h.b2, v, h.a2 * g * g);
  m = mm;
  v = vv;
  p -= lr * (mm * h.bc1) / fmaf(sqrtf(vv), h.bc2, h.eps);
}

#ifndef MG_UPD_MINB
#define MG_UPD_MINB 2  // 128 registers, no spills: 111 -> 107 us at 1M Gaussians
#endif
// BY_INV = false: thread p walks the cell-sorted order, i = perm[p] (perm =
// the binning's cell_indices), so parameter and moment rows are gathered.
// BY_INV = true: thread i walks the ORIGINAL order and reads its accumulator
// row p = perm[i] (perm = the inverse permutation): all parameter and moment
// traffic is coalesced and only the 40-byte acc10 row is gathered.  After
// training drift the sorted order is a local shuffle of the original one and
// the gathered walk was latency-bound (C4, 1M Gaussians: 375 us at 10% of
// HBM bandwidth).
template <bool BY_INV>
__global__ void __launch_bounds__(256, MG_UPD_MINB) gauss_update_kernel(const float* __restrict__ acc10,
                                                                        const int* __restrict__ perm, int64_t n,
                                    float* __restrict__ pos, float* __restrict__ quat, float* __restrict__ ls,
                                    float* __restrict__ lg, float* __restrict__ mom_m, float* __restrict__ mom_v,
                                    AdamHyper h, const int* __restrict__ t_dev, double* __restrict__ aniso_acc) {
  double aniso_local = 0.0;
  __shared__ double s_bc[2];
  __shared__ double s_red[8];
  if (threadIdx.x == 0) {  // bias corrections once per block: h.bc1 = 1/bc1, h.bc2 = 1/sqrt(bc2)
    const double t = (double)*t_dev;
    s_bc[0] = 1.0 / (1.0 - pow(h.beta1, t));
    s_bc[1] = 1.0 / sqrt(1.0 - pow(h.beta2, t));
  }
  __syncthreads();
  h.bc1 = s_bc[0];
  h.bc2 = s_bc[1];
  const AdamF af{(float)h.beta1, (float)(1.0 - h.beta1), (float)h.beta2, (float)(1.0 - h.beta2), (float)h.eps,
                 (float)h.bc1, (float)h.bc2};
  const float lr[4] = {(float)h.lr_pos, (float)h.lr_quat, (float)h.lr_scale, (float)h.lr_logit};
  GRID_LOOP(tix, n) {
    const int64_t i = BY_INV ? tix : (int64_t)perm[tix];
    const int64_t p = BY_INV ? (int64_t)perm[tix] : tix;
    // every load of the element is issued before the float64 chain rule;
    // moments are structure-of-arrays [11][n] (coalesced across the warp)
    float mm[11], vv[11];
#pragma unroll
    for (int a = 0; a < 11; ++a) {
      mm[a] = mom_m[(int64_t)a * n + i];
      vv[a] = mom_v[(int64_t)a * n + i];
    }
    const double logit = lg[i];
    double s[3] = {ls[3 * i], ls[3 * i + 1], ls[3 * i + 2]};
    const float q0 = quat[4 * i], q1 = quat[4 * i + 1], q2 = quat[4 * i + 2], q3 = quat[4 * i + 3];
    const double alpha = 1.0 / (1.0 + exp(-logit));
    double dmu[3], dab[6], dal;
    acc_to_ref(acc10 + 10 * p, alpha, dmu, dab, &dal);
    GaussGrad gg = chain_one(dmu, dab, dal, q0, q1, q2, q3, s, logit);
    if (h.use_aniso) {
      // train.py:128-147: ratio = exp(s_max - s_min), first index on ties
      int hi = 0, lo = 0;
      for (int a = 1; a < 3; ++a) {
        if (s[a] > s[hi]) hi = a;
        if (s[a] < s[lo]) lo = a;
      }
      double ratio = exp(s[hi] - s[lo]);
      double excess = ratio - h.lambda_ratio;
      if (excess > 0) {
        aniso_local += excess;
        double c = h.lambda_aniso * ratio / (double)n;
        gg.ds[hi] += c;
        gg.ds[lo] -= c;
      }
    }
    // moment slots: pos(3) quat(4) scale(3) logit(1)
#pragma unroll
    for (int a = 0; a < 3; ++a) adam_upd32(pos[3 * i + a], mm[a], vv[a], gg.dmu[a], lr[0], af);
#pragma unroll
    for (int a = 0; a < 4; ++a) adam_upd32(quat[4 * i + a], mm[3 + a], vv[3 + a], gg.dq[a], lr[1], af);
#pragma unroll
    for (int a = 0; a < 3; ++a) adam_upd32(ls[3 * i + a], mm[7 + a], vv[7 + a], gg.ds[a], lr[2], af);
    adam_upd32(lg[i], mm[10], vv[10], gg.dl, lr[3], af);
#pragma unroll
    for (int a = 0; a < 11; ++a) {
      mom_m[(int64_t)a * n + i] = mm[a];
      mom_v[(int64_t)a * n + i] = vv[a];
    }
  }
  if (aniso_acc && h.use_aniso) {  // one float64 atomic per block (was one per warp: 31k on one address)
    for (int o = 16; o > 0; o >>= 1) aniso_local += __shfl_xor_sync(MG_FULL, aniso_local, o);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = aniso_local;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_red[w];
      if (t != 0.0) atomicAdd(aniso_acc, t / (double)n);
    }
  }
}

__global__ void invert_perm_kernel(const int* __restrict__ perm, int64_t n, int* __restrict__ inv) {
  GRID_LOOP(p, n) inv[perm[p]] = (int)p;
}
void launch_invert_perm(const int* perm, int64_t n, int* inv, cudaStream_t st) {
  if (n > 0) MG_LAUNCH(invert_perm_kernel<<<gridn(n), 256, 0, st>>>(perm, n, inv));
}

// Transform group: quats (K,4) + trans (K,3) fp64, one Adam group.
__global__ void transform_adam_kernel(double* __restrict__ tq, double* __restrict__ tt, const double* __restrict__ g7,
                                      double* __restrict__ m7, double* __restrict__ v7, int k, double lr, double b1,
                                      double b2, double eps, const int* __restrict__ t_dev) {
  const double bc1 = 1.0 - pow(b1, (double)*t_dev), bc2 = 1.0 - pow(b2, (double)*t_dev);
  GRID_LOOP(j, (int64_t)k * 7) {
    int64_t s = j / 7;
    int c = (int)(j - s * 7);
    double g = g7[j];
    double m = b1 * m7[j] + (1.0 - b1) * g;
    double v = b2 * v7[j] + (1.0 - b2) * g * g;
    m7[j] = m;
    v7[j] = v;
    double upd = lr * (m / bc1) / (sqrt(v / bc2) + eps);
    if (c < 4)
      tq[4 * s + c] -= upd;
    else
      tt[3 * s + c - 4] -= upd;
  }
}

// ---------------------------------------------------------------------------
// Progressive upsample (train.py:157-218), lattice-index addressed.
// Input arrays are indexed by the (C-ordered) lattice node id old_id.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void upsample_kernel(const T* __restrict__ q_old, const T* __restrict__ s_old,
                                const T* __restrict__ l_old, const int* __restrict__ node_of_old, int ro,
                                int rn, T* __restrict__ pos, T* __restrict__ q, T* __restrict__ s,
                                T* __restrict__ l) {
  const int64_t nn = (int64_t)rn * rn * rn;
  GRID_LOOP(id, nn) {
    int c3[3] = {(int)(id / ((int64_t)rn * rn)), (int)((id / rn) % rn), (int)(id % rn)};
    double f[3], t[3];
    int base[3];
    for (int a = 0; a < 3; ++a) {
      double fr = ((double)c3[a] + 0.5) * ((double)ro / (double)rn) - 0.5;
      fr = fr < 0.0 ? 0.0 : (fr > ro - 1.0 ? ro - 1.0 : fr);
      f[a] = fr;
      int bs = ro > 1 ? (int)floor(fr) : 0;
      if (ro > 1 && bs > ro - 2) bs = ro - 2;
      base[a] = bs;
      t[a] = fr - bs;
    }
    int ref[3];
    for (int a = 0; a < 3; ++a) ref[a] = min(base[a] + (t[a] >= 0.5 ? 1 : 0), ro - 1);
    int rid = node_of_old[((int64_t)ref[0] * ro + ref[1]) * ro + ref[2]];
    double rq[4] = {q_old[4 * rid], q_old[4 * rid + 1], q_old[4 * rid + 2], q_old[4 * rid + 3]};
    double lo = 0.0, sc[3] = {0, 0, 0}, qs[4] = {0, 0, 0, 0};
    for (int da = 0; da < 2; ++da)
      for (int db = 0; db < 2; ++db)
        for (int dc = 0; dc < 2; ++dc) {
          int ia = min(base[0] + da, ro - 1), ib = min(base[1] + db, ro - 1), ic = min(base[2] + dc, ro - 1);
          double w = (da ? t[0] : 1.0 - t[0]) * (db ? t[1] : 1.0 - t[1]) * (dc ? t[2] : 1.0 - t[2]);
          int src = node_of_old[((int64_t)ia * ro + ib) * ro + ic];
          lo += w * (double)l_old[src];
          for (int a = 0; a < 3; ++a) sc[a] += w * (double)s_old[3 * src + a];
          double qq[4] = {q_old[4 * src], q_old[4 * src + 1], q_old[4 * src + 2], q_old[4 * src + 3]};
          double dot = qq[0] * rq[0] + qq[1] * rq[1] + qq[2] * rq[2] + qq[3] * rq[3];
          double sg = dot < 0.0 ? -1.0 : 1.0;
          for (int a = 0; a < 4; ++a) qs[a] += w * sg * qq[a];
        }
    double nrm = sqrt(qs[0] * qs[0] + qs[1] * qs[1] + qs[2] * qs[2] + qs[3] * qs[3]);
    if (!(nrm > 1e-12)) nrm = 1.0;
    for (int a = 0; a < 4; ++a) q[4 * id + a] = (T)(qs[a] / nrm);
    for (int a = 0; a < 3; ++a) s[3 * id + a] = (T)sc[a];
    l[id] = (T)lo;
    // lattice_node_positions (core.py:304-309): -1 + (c + 0.5) * (2 / r), no FMA contraction
    for (int a = 0; a < 3; ++a) pos[3 * id + a] = (T)__dadd_rn(-1.0, __dmul_rn((double)c3[a] + 0.5, 2.0 / rn));
  }
}

// ---------------------------------------------------------------------------
// Launchers
// ---------------------------------------------------------------------------
void launch_forward_finish(const float4* out4, const int* cnt, const int* inv, int64_t b, int ntaps,
                           const double* tap_w, double* out_i, float* out_i32, int64_t* out_cnt, int64_t* pair_total, cudaStream_t st) {
  if (b > 0)
    MG_LAUNCH(forward_finish_kernel<<<gridn(b), 256, 0, st>>>(out4, cnt, inv, b, ntaps, tap_w, out_i, out_i32, out_cnt,
                                                              (unsigned long long*)pair_total));
}
void launch_gather_batch(const int64_t* idx, int64_t n, const double* pc, const int64_t* ps, const float* pt,
                         double* c, int64_t* s, float* t, cudaStream_t st) {
  if (n > 0) MG_LAUNCH(gather_batch_kernel<<<gridn(n), 256, 0, st>>>(idx, n, pc, ps, pt, c, s, t));
}
void launch_backward_points(const double* up64, const float* up32, const int* inv, int64_t b, int ntaps,
                            const double* tap_w, const float4* out4, float4* prec, double* dpoints, cudaStream_t st) {
  if (b > 0)
    MG_LAUNCH(backward_points_kernel<<<gridn(b * ntaps), 256, 0, st>>>(up64, up32, inv, b, ntaps, tap_w, out4, prec, dpoints));
}
void launch_acc_to_ref(const float* acc10, const int* order, int64_t n, const double* alpha64, double* d_mu,
                       double* d_abar6, double* d_alpha, cudaStream_t st) {
  if (n > 0) MG_LAUNCH(acc_to_ref_kernel<<<gridn(n), 256, 0, st>>>(acc10, order, n, alpha64, d_mu, d_abar6, d_alpha));
}
void launch_epilogue(const float* acc10, const int* order, int64_t n, const float* quat, const float* ls,
                     const float* lg, double* d_pos, double* d_q, double* d_s, double* d_l, cudaStream_t st) {
  if (n > 0) MG_LAUNCH(epilogue_kernel<<<gridn(n), 256, 0, st>>>(acc10, order, n, quat, ls, lg, d_pos, d_q, d_s, d_l));
}
void launch_epilogue_f64(const double* d_mu, const double* d_abar6, const double* d_alpha, const double* quat,
                         const double* ls, const double* lg, int64_t n, double* d_pos, double* d_q, double* d_s,
                         double* d_l, cudaStream_t st) {
  if (n > 0) MG_LAUNCH(epilogue_f64_kernel<<<gridn(n), 256, 0, st>>>(d_mu, d_abar6, d_alpha, quat, ls, lg, n, d_pos, d_q, d_s, d_l));
}
// Deterministic reduction geometry: blocks of kTrWarps warps, at most
// kTrBlocks blocks; the per-warp slice tables must fit in shared memory.
#ifndef MG_TR_BLOCKS
#define MG_TR_BLOCKS 296  // two blocks per SM (smem-bound tables): C4 -28 us, C2 -8 us per step vs 148; 592 slower
#endif
constexpr int kTrWarps = 4, kTrBlocks = MG_TR_BLOCKS;
constexpr size_t kTrSmemMax = 200 * 1024;
static size_t tr_smem(int k) { return sizeof(double) * ((size_t)kTrWarps * 12 * k + (size_t)kTrWarps * 32 * 12); }
static bool tr_deterministic(int k) { return tr_smem(k) <= kTrSmemMax; }

size_t transform_grads_ws_bytes(int64_t k) {
  if (k <= 0 || !tr_deterministic((int)k)) return 256;
  return (((size_t)kTrBlocks * 12 * k * sizeof(double) + 255) & ~(size_t)255) + 256;
}

void launch_transform_grads(const double* dpoints, const double* coords, const int64_t* sids, int64_t b, int ntaps,
                            const double* tap_off, const double* dirs, const double* tq, int k, double* acc12,
                            double* out7, int accumulate, void* ws, cudaStream_t st) {
  if (k <= 0) return;
  if (b > 0 && ws && tr_deterministic(k)) {
    const size_t smem = tr_smem(k);
    static size_t attr = 0;
    if (smem > 48 * 1024 && smem > attr) {
      cudaFuncSetAttribute(transform_reduce_det_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = smem;
    }
    const int64_t total = b * ntaps;
    int64_t blocks = (total + kTrWarps * 32 * 4 - 1) / (kTrWarps * 32 * 4);
    blocks = blocks < 1 ? 1 : (blocks > kTrBlocks ? kTrBlocks : blocks);
    double* partials = (double*)ws;
    MG_LAUNCH(transform_reduce_det_kernel<<<(unsigned)blocks, kTrWarps * 32, smem, st>>>(
        dpoints, coords, sids, b, ntaps, tap_off, dirs, k, partials));
    MG_LAUNCH(transform_finish_kernel<<<(unsigned)((k * 32 + 255) / 256), 256, 0, st>>>(partials, (int)blocks, tq, k,
                                                                                      acc12, out7, accumulate));
    return;
  } else {
    cudaMemsetAsync(acc12, 0, sizeof(double) * 12 * k, st);
    if (b > 0) {
      int64_t chunks = (b * ntaps + 7) / 8;
      MG_LAUNCH(transform_reduce_kernel<<<gridn(chunks, 128), 128, 0, st>>>(dpoints, coords, sids, b, ntaps, tap_off,
                                                                            dirs, k, acc12));
    }
  }
  MG_LAUNCH(transform_chain_kernel<<<gridn(k), 256, 0, st>>>(acc12, tq, k, out7, accumulate));
}
// Standalone aniso_loss_grad (train.py:128-147) in float64: grad (n,3) is
// overwritten, loss_acc += sum(excess) / n.
__global__ void aniso_f64_kernel(const double* __restrict__ ls, int64_t n, double lambda_ratio,
                                 double* __restrict__ grad, double* __restrict__ loss_acc) {
  double local = 0.0;
  GRID_LOOP(i, n) {
    const double s[3] = {ls[3 * i], ls[3 * i + 1], ls[3 * i + 2]};
    int hi = 0, lo = 0;
    for (int a = 1; a < 3; ++a) {
      if (s[a] > s[hi]) hi = a;
      if (s[a] < s[lo]) lo = a;
    }
    const double ratio = exp(s[hi] - s[lo]);
    const double excess = ratio - lambda_ratio;
    double gr[3] = {0.0, 0.0, 0.0};
    if (excess > 0) {
      local += excess;
      const double c = ratio / (double)n;
      gr[hi] += c;
      gr[lo] -= c;
    }
    for (int a = 0; a < 3; ++a) grad[3 * i + a] = gr[a];
  }
  __shared__ double s_red[32];
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(MG_FULL, local, o);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = local;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? s_red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(MG_FULL, v, o);
    if (threadIdx.x == 0 && v != 0.0) atomicAdd(loss_acc, v / (double)n);
  }
}
void launch_aniso_f64(const double* ls, int64_t n, double lambda_ratio, double* grad, double* loss_acc,
                      cudaStream_t st) {
  if (n > 0) MG_LAUNCH(aniso_f64_kernel<<<gridn(n), 256, 0, st>>>(ls, n, lambda_ratio, grad, loss_acc));
}

// AdamState.step on one float64 tensor (train.py:251-271), t = the
// post-increment step count of the group.
__global__ void adam_f64_kernel(double* __restrict__ p, const double* __restrict__ g, double* __restrict__ m,
                                double* __restrict__ v, int64_t n, double lr, double b1, double b2, double eps,
                                double bc1, double bc2) {
  GRID_LOOP(i, n) {
    const double gi = g[i];
    double mi = m[i] * b1;
    mi += (1.0 - b1) * gi;
    double vi = v[i] * b2;
    vi += (1.0 - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    p[i] -= lr * (mi / bc1) / (sqrt(vi / bc2) + eps);
  }
}
void launch_adam_f64(double* p, const double* g, double* m, double* v, int64_t n, int64_t t, double lr, double b1,
                     double b2, double eps, cudaStream_t st) {
  if (n > 0)
    MG_LAUNCH(adam_f64_kernel<<<gridn(n), 256, 0, st>>>(p, g, m, v, n, lr, b1, b2, eps, 1.0 - pow(b1, (double)t),
                                                        1.0 - pow(b2, (double)t)));
}

void launch_smooth_l1(const float* pred, const float* target, int64_t b, double scale, float* up_out,
                      double* loss_acc, cudaStream_t st) {
  if (b > 0) MG_LAUNCH((smooth_l1_kernel<float, false><<<gridn(b), 256, 0, st>>>(pred, target, b, scale, up_out, loss_acc)));
}
void launch_smooth_l1_f64(const double* pred, const double* target, int64_t b, double divisor, double* up_out,
                          double* loss_acc, cudaStream_t st) {
  if (b > 0) MG_LAUNCH((smooth_l1_kernel<double, true><<<gridn(b), 256, 0, st>>>(pred, target, b, divisor, up_out, loss_acc)));
}

__global__ void quat_to_rot_kernel(const double* __restrict__ q, int64_t k, double* __restrict__ rot) {
  GRID_LOOP(s, k) {
    double qw = q[4 * s], qx = q[4 * s + 1], qy = q[4 * s + 2], qz = q[4 * s + 3];
    double nrm = sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
    quat_rot_d2(qw / nrm, qx / nrm, qy / nrm, qz / nrm, rot + 9 * s);
  }
}
void launch_quat_to_rot(const double* q, int64_t k, double* rot, cudaStream_t st) {
  if (k > 0) MG_LAUNCH(quat_to_rot_kernel<<<gridn(k), 256, 0, st>>>(q, k, rot));
}
__global__ void counter_incr_kernel(int* c, int n) {
  if (threadIdx.x < n) c[threadIdx.x] += 1;
}
void launch_counter_incr(int* c, int n, cudaStream_t st) { MG_LAUNCH(counter_incr_kernel<<<1, 32, 0, st>>>(c, n)); }

void launch_gauss_update(const float* acc10, const int* perm, int by_inv, int64_t n, float* pos, float* quat,
                         float* ls, float* lg, float* mom_m, float* mom_v, const double* hyper, int use_aniso,
                         const int* t_dev, double* aniso_acc, cudaStream_t st) {
  AdamHyper h;
  h.lr_pos = hyper[0];
  h.lr_quat = hyper[1];
  h.lr_scale = hyper[2];
  h.lr_logit = hyper[3];
  h.beta1 = hyper[4];
  h.beta2 = hyper[5];
  h.eps = hyper[6];
  h.lambda_aniso = hyper[7];
  h.lambda_ratio = hyper[8];
  h.use_aniso = use_aniso;
  h.bc1 = h.bc2 = 1.0;
  if (n <= 0) return;
  if (by_inv)
    MG_LAUNCH(gauss_update_kernel<true><<<gridn(n), 256, 0, st>>>(acc10, perm, n, pos, quat, ls, lg, mom_m, mom_v, h,
                                                                  t_dev, aniso_acc));
  else
    MG_LAUNCH(gauss_update_kernel<false><<<gridn(n), 256, 0, st>>>(acc10, perm, n, pos, quat, ls, lg, mom_m, mom_v, h,
                                                                   t_dev, aniso_acc));
}
void launch_transform_adam(double* tq, double* tt, const double* g7, double* m7, double* v7, int k, double lr,
                           double b1, double b2, double eps, const int* t_dev, cudaStream_t st) {
  if (k > 0) MG_LAUNCH(transform_adam_kernel<<<gridn((int64_t)k * 7), 256, 0, st>>>(tq, tt, g7, m7, v7, k, lr, b1, b2, eps, t_dev));
}
void launch_upsample(const float* q_old, const float* s_old, const float* l_old, const int* node_of_old, int ro, int rn,
                     float* pos, float* q, float* s, float* l, cudaStream_t st) {
  int64_t nn = (int64_t)rn * rn * rn;
  if (nn > 0) MG_LAUNCH(upsample_kernel<<<gridn(nn), 256, 0, st>>>(q_old, s_old, l_old, node_of_old, ro, rn, pos, q, s, l));
}
void launch_upsample_f64(const double* q_old, const double* s_old, const double* l_old, const int* node_of_old,
                         int ro, int rn, double* pos, double* q, double* s, double* l, cudaStream_t st) {
  int64_t nn = (int64_t)rn * rn * rn;
  if (nn > 0) MG_LAUNCH(upsample_kernel<<<gridn(nn), 256, 0, st>>>(q_old, s_old, l_old, node_of_old, ro, rn, pos, q, s, l));
}

}  // namespace mg
