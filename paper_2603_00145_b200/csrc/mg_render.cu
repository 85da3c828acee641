// mg_render.cu -- Gaussian preprocessing, point binning and the block
// forward / backward pair kernels for sm_100a.
//
// Reference semantics (cited per kernel):
//   activated_parameters   render.py:122-142, core.py:36-67
//   block_forward          _kernels.py:24-70   (+ render.py:161-187)
//   block_backward         _kernels.py:73-144  (+ render.py:276-317)
//
// Candidate rule: Gaussian i is a candidate of point x iff the Chebyshev
// distance between cell(mu_i) and cell(x) is <= r (both clamped cells,
// spatial.py:18-27, _kernels.py:43-58).  The relation is symmetric, which
// lets the backward run Gaussian-major with no atomics.
//
// Layout in HBM (all in cell-sorted order):
//   grec (SoA, 12 floats per Gaussian): A = float4[N] {mu.xyz, alpha} at 0,
//                        B = float4[N] {P'00,P'11,P'22,P'01} at 4N, C = float2[N] {P'02,P'12} at 8N
//                        with P' = -0.5*log2(e) * P  (exp(-m/2) = 2^{d^T P' d})
//   prec[p]              float4 {x, y, z, upstream} of sub-point p (fp32)
//   gstart / pstart      int32 CSR over the G^3 cells
#include "mg_render.cuh"
#include "mg_sort.cuh"

namespace mg {

// ---------------------------------------------------------------------------
// Gaussian keys and activation
// ---------------------------------------------------------------------------
__global__ void gauss_keys_kernel(const float* __restrict__ pos, int64_t n, int g, uint32_t* __restrict__ keys) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int ci = cell_of_d((double)pos[3 * i + 0], g);
    int cj = cell_of_d((double)pos[3 * i + 1], g);
    int ck = cell_of_d((double)pos[3 * i + 2], g);
    keys[i] = (uint32_t)flat_cell(ci, cj, ck, g);
  }
}

// Same key math on float64 positions (the reference drop-in ABI passes f64).
__global__ void gauss_keys_f64_kernel(const double* __restrict__ pos, int64_t n, int g, uint32_t* __restrict__ keys) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int ci = cell_of_d(pos[3 * i + 0], g);
    int cj = cell_of_d(pos[3 * i + 1], g);
    int ck = cell_of_d(pos[3 * i + 2], g);
    keys[i] = (uint32_t)flat_cell(ci, cj, ck, g);
  }
}

// Quaternion -> rotation exactly as core.py:48-67 (w-first), in float64.
__device__ __forceinline__ void quat_rot_d(double w, double x, double y, double z, double R[9]) {
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

// Cutoff box half-extents from Sigma_aa (m <= 64 <=> |d_a| <= 8 sqrt(Sigma_aa)),
// padded by 1% (+1e-6) and rounded up to fp16; cond > 1e4 or non-finite: +inf.
__device__ __forceinline__ uint2 pack_extents(const double (&sig)[3], double cond) {
  unsigned short h[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double e = 8.08 * sqrt(sig[a]) + 1e-6;
    const bool ok = sig[a] > 0.0 && e < 6.0e4 && cond < 1e4;
    h[a] = __half_as_ushort(ok ? __float2half_ru((float)e) : __ushort_as_half((unsigned short)0x7c00));
  }
  return make_uint2((unsigned)h[0] | ((unsigned)h[1] << 16), (unsigned)h[2]);
}

__device__ __forceinline__ void activate_one(const float* pos, const float* quat, const float* ls, const float* lg,
                                             int64_t i, GaussOut rec, int64_t p, int* err) {
  double qw = quat[4 * i], qx = quat[4 * i + 1], qy = quat[4 * i + 2], qz = quat[4 * i + 3];
  double nrm = sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
  if (!(nrm > 1e-12)) {  // core.py:43-44 (DegenerateQuaternion); NaN also flags
    atomicOr(err, MG_ERR_DEGENERATE_QUAT);
    nrm = 1.0;
  }
  double R[9];
  quat_rot_d(qw / nrm, qx / nrm, qy / nrm, qz / nrm, R);
  double e[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double s = (double)ls[3 * i + a];
    s = s < -20.0 ? -20.0 : (s > 20.0 ? 20.0 : s);  // LOG_SCALE_LIMIT clamp, render.py:131
    e[a] = exp(-2.0 * s);
  }
  // P = R diag(e) R^T, scaled by -0.5*log2(e)
  double P[6];
  const int ia[6] = {0, 1, 2, 0, 0, 1}, ib[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    int a = ia[k], b = ib[k];
    P[k] = kMScaleD * (R[3 * a] * e[0] * R[3 * b] + R[3 * a + 1] * e[1] * R[3 * b + 1] + R[3 * a + 2] * e[2] * R[3 * b + 2]);
  }
  double alpha = 1.0 / (1.0 + exp(-(double)lg[i]));  // core.py:21-26
  rec.A[p] = make_float4(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], (float)(alpha * kWeightScaleD));
  rec.B[p] = make_float4((float)P[0], (float)P[1], (float)P[2], (float)P[3]);
  rec.C[p] = make_float2((float)P[4], (float)P[5]);
  // Sigma = R diag(1/e) R^T
  double sig[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) sig[a] = R[3 * a] * R[3 * a] / e[0] + R[3 * a + 1] * R[3 * a + 1] / e[1] + R[3 * a + 2] * R[3 * a + 2] / e[2];
  const double emax = fmax(e[0], fmax(e[1], e[2])), emin = fmin(e[0], fmin(e[1], e[2]));
  rec.E[p] = pack_extents(sig, emax / emin);
}

__global__ void gauss_activate_kernel(const float* __restrict__ pos, const float* __restrict__ quat,
                                      const float* __restrict__ ls, const float* __restrict__ lg,
                                      const int* __restrict__ order, int64_t n, GaussOut grec,
                                      int* __restrict__ err) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = order ? order[p] : p;
    activate_one(pos, quat, ls, lg, i, grec, p, err);
  }
}

// Records straight from precomputed float64 (mu, prec6, alpha) -- the
// reference kernel ABI (_kernels.py:24-27) hands these in already activated.
__global__ void gauss_pack_prepared_kernel(const double* __restrict__ mu, const double* __restrict__ prec6,
                                           const double* __restrict__ alpha, const int* __restrict__ order,
                                           int64_t n, GaussOut grec) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = order[p];
    const double* P = prec6 + 6 * i;
    grec.A[p] = make_float4((float)mu[3 * i], (float)mu[3 * i + 1], (float)mu[3 * i + 2],
                            (float)(alpha[i] * kWeightScaleD));
    grec.B[p] = make_float4((float)(kMScaleD * P[0]), (float)(kMScaleD * P[3]), (float)(kMScaleD * P[5]),
                            (float)(kMScaleD * P[1]));
    grec.C[p] = make_float2((float)(kMScaleD * P[2]), (float)(kMScaleD * P[4]));
    // Sigma_aa = cof_aa(P) / det(P); Sigma_aa * P_aa >= 1 grows with the condition number
    const double c00 = P[3] * P[5] - P[4] * P[4], c11 = P[0] * P[5] - P[2] * P[2], c22 = P[0] * P[3] - P[1] * P[1];
    const double det = P[0] * c00 - P[1] * (P[1] * P[5] - P[4] * P[2]) + P[2] * (P[1] * P[4] - P[3] * P[2]);
    double sig[3] = {c00 / det, c11 / det, c22 / det};
    const double cond = fmax(sig[0] * P[0], fmax(sig[1] * P[3], sig[2] * P[5]));
    grec.E[p] = pack_extents(sig, cond);
  }
}

// ---------------------------------------------------------------------------
// Point preparation: PSF tap expansion, rigid transform (float64, same
// operation order as _kernels.py:33-38), cell key.
// ---------------------------------------------------------------------------
__global__ void points_prepare_kernel(const double* __restrict__ coords, const int64_t* __restrict__ sids64,
                                      const int* __restrict__ sids32, int64_t b, int ntaps,
                                      const double* __restrict__ tap_off, const double* __restrict__ dirs,
                                      const double* __restrict__ rot, const double* __restrict__ trans,
                                      int nslices, int g, uint32_t* __restrict__ keys, float4* __restrict__ xf,
                                      double* __restrict__ xout) {
  const int64_t total = b * ntaps;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < total; j += (int64_t)gridDim.x * blockDim.x) {
    int64_t pb = j / ntaps;
    int t = (int)(j - pb * ntaps);
    int64_t s = sids64 ? sids64[pb] : (sids32 ? sids32[pb] : -1);
    double px = coords[3 * pb], py = coords[3 * pb + 1], pz = coords[3 * pb + 2];
    if (s >= 0 && tap_off) {
      double o = tap_off[t];
      px = __dadd_rn(px, __dmul_rn(o, dirs[3 * s]));
      py = __dadd_rn(py, __dmul_rn(o, dirs[3 * s + 1]));
      pz = __dadd_rn(pz, __dmul_rn(o, dirs[3 * s + 2]));
    }
    double x, y, z;
    if (s >= 0 && s < nslices) {
      const double* R = rot + 9 * s;
      const double* T = trans + 3 * s;
      x = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(R[0], px), __dmul_rn(R[1], py)), __dmul_rn(R[2], pz)), T[0]);
      y = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(R[3], px), __dmul_rn(R[4], py)), __dmul_rn(R[5], pz)), T[1]);
      z = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(R[6], px), __dmul_rn(R[7], py)), __dmul_rn(R[8], pz)), T[2]);
    } else {
      x = px;
      y = py;
      z = pz;
    }
    keys[j] = (uint32_t)flat_cell(cell_of_d(x, g), cell_of_d(y, g), cell_of_d(z, g), g);
    xf[j] = make_float4((float)x, (float)y, (float)z, 0.f);
    if (xout) {
      xout[3 * j] = x;
      xout[3 * j + 1] = y;
      xout[3 * j + 2] = z;
    }
  }
}

// Gather point records into cell order; inv[j] = sorted position of j.
__global__ void points_gather_kernel(const float4* __restrict__ xf, const int* __restrict__ perm, int64_t n,
                                     float4* __restrict__ prec, int* __restrict__ inv) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    int j = perm[p];
    prec[p] = xf[j];
    inv[j] = (int)p;
  }
}

// ---------------------------------------------------------------------------
// Work items: runs of equal cell key chunked into groups of <= Q.
// flag[p] = 1 if p starts an item.
// ---------------------------------------------------------------------------
// dense_min > 0: cells with >= dense_min elements are chunked by 64 instead of q
__global__ void item_flags_kernel(const uint32_t* __restrict__ keys, const int* __restrict__ starts, int64_t n, int q,
                                  int dense_min, int* __restrict__ flags) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t key = keys[p];
    const int s = starts[key];
    const int qq = (dense_min > 0 && starts[key + 1] - s >= dense_min) ? 64 : q;
    flags[p] = ((p - s) % qq) == 0 ? 1 : 0;
  }
}

// Item record {first element, cell, element count, 0}: a warp starts an item
// with ONE load instead of the items -> key -> starts dependency chain.
__global__ void item_compact_kernel(const int* __restrict__ flags, const int* __restrict__ scan,
                                    const uint32_t* __restrict__ keys, const int* __restrict__ starts, int64_t n, int q,
                                    int dense_min, int4* __restrict__ items, int* __restrict__ nitems,
                                    int single_gauss = 0) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    if (flags[p]) {
      const uint32_t key = keys[p];
      const int e = starts[key + 1];
      const int qq = (dense_min > 0 && e - starts[key] >= dense_min) ? 64 : q;
      items[scan[p]] = make_int4((int)p, (int)key, single_gauss ? -1 : min(qq, e - (int)p), 0);
    }
    if (p == n - 1) *nitems = scan[p] + flags[p];
  }
}

// ---------------------------------------------------------------------------
// Segment table: the (2r+1)^2 (clipped) neighbor columns of a cell, each a
// contiguous CSR range over the k-window [klo, khi].  Built 128 columns at a
// time into per-warp shared memory.
// ---------------------------------------------------------------------------
struct Window {
  int ilo, jlo, klo, khi, nj, ncol;
  float inv_nj;  // exact column -> (i, j) split for ncol < 2^22
};

// cell -> (ci, cj, ck) with two float-reciprocal divisions: (n + 0.5) * (1/g)
// is exact after truncation while the quotient's fractional part (>= 0.5/g
// away from an integer) exceeds the float rounding, n * 2^-23 / g: holds for
// every n < 2^21 at g <= 2^10 (host-guarded: larger grids take the integer
// path).  Replaces two integer div/mod sequences per item (~45 instructions).
#ifndef MG_FAST_SPLIT
#define MG_FAST_SPLIT 1
#endif
#ifndef MG_BWD_SMEM_STORE
#define MG_BWD_SMEM_STORE 0  // smem f2 reduction: fewer instructions but 2.27 -> 2.32 ms at C4 (latency)
#endif
__device__ __forceinline__ void split_cell(int cell, int g, int& ci, int& cj, int& ck) {
  if (MG_FAST_SPLIT && g * g * g <= (1 << 21)) {
    const float inv_g = 1.0f / (float)g;
    const int t = (int)(((float)cell + 0.5f) * inv_g);
    ck = cell - t * g;
    ci = (int)(((float)t + 0.5f) * inv_g);
    cj = t - ci * g;
  } else {
    ck = cell % g;
    const int t = cell / g;
    cj = t % g;
    ci = t / g;
  }
}

__device__ __noinline__ Window make_window(int cell, int g, int r) {
  int ci, cj, ck;
  split_cell(cell, g, ci, cj, ck);
  Window w;
  w.ilo = max(ci - r, 0);
  int ihi = min(ci + r, g - 1);
  w.jlo = max(cj - r, 0);
  int jhi = min(cj + r, g - 1);
  w.klo = max(ck - r, 0);
  w.khi = min(ck + r, g - 1);
  w.nj = jhi - w.jlo + 1;
  w.ncol = (ihi - w.ilo + 1) * w.nj;
  w.inv_nj = 1.0f / (float)w.nj;
  return w;
}

// ---------------------------------------------------------------------------
// Cutoff culling for the Gaussian-major backward.  A pair whose Mahalanobis
// form exceeds 64 contributes nothing (_kernels.py:21, 106-110: skipped), and
// {d : d^T P d <= 64} lies inside the axis box |d_a| <= 8 sqrt(Sigma_aa)
// (precomputed per Gaussian with the records, GaussSoA::E).  A
// Gaussian's candidate points therefore only need the cells of that box
// intersected with its Chebyshev window.  The box is padded by 1% (m by 2%),
// far beyond the float32 rounding of m, so every culled pair is one the
// kernel would have flushed to an exact zero: culling drops no contribution
// (the sums differ from the unculled walk only in float32 summation order,
// as the shorter candidate list hands points to different lanes).
// ---------------------------------------------------------------------------
#ifndef MG_BWD_CULL
#define MG_BWD_CULL 1
#endif
struct CellBox {
  int lo[3], hi[3];
};
// MGAUSS_BWD_CULL=0 turns culling off at launch time (A/B and the test that
// checks culling drops no contribution); read at every launch, so a graph
// keeps the value it was captured with.
static inline int bwd_cull_enabled() {
  const char* e = getenv("MGAUSS_BWD_CULL");
  return (e && e[0] == '0') ? 0 : 1;
}

__device__ __forceinline__ CellBox cutoff_box(const float4 A, const uint2 E, int g) {
  const float e[3] = {__half2float(__ushort_as_half((unsigned short)(E.x & 0xffffu))),
                      __half2float(__ushort_as_half((unsigned short)(E.x >> 16))),
                      __half2float(__ushort_as_half((unsigned short)(E.y & 0xffffu)))};
  const float mu[3] = {A.x, A.y, A.z}, hg = 0.5f * (float)g;
  CellBox b;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    // +inf extents clamp to the whole grid; float rounding of the box edges is
    // ~1e-7 relative, far inside the 1% padding
    b.lo[a] = (int)fminf(fmaxf(floorf((mu[a] + 1.0f - e[a]) * hg), 0.0f), (float)(g - 1));
    b.hi[a] = (int)fminf(fmaxf(floorf((mu[a] + 1.0f + e[a]) * hg), 0.0f), (float)(g - 1));
  }
  return b;
}

// Can the box trim the window at all?  Only if some half-extent is below r
// cells: a box reaches floor(frac + e) >= floor(e) cells either side (fp16
// bit patterns of non-negative values order like integers);
// fields whose Gaussians all reach past the window (upsampled levels) then
// skip the out-of-line call.
__device__ __forceinline__ bool may_cull(uint2 E, int g, int r) {
  const unsigned thr = __half_as_ushort(__float2half_ru(2.0f * (float)r / (float)g));
  const unsigned m = min(min(E.x & 0xffffu, E.x >> 16), E.y & 0xffffu);
  return m < thr;
}

// Kept out of line so the item loops' register allocation is unaffected.
__device__ __forceinline__ void cull_window(Window& w, const CellBox& b);
__device__ __noinline__ Window cull_single_window(Window w, const GaussSoA grec, int j, int g) {
  cull_window(w, cutoff_box(grec.A[j], grec.E[j], g));
  return w;
}
// union of the pair's two boxes (even lanes: Gaussian j, odd lanes: j + 1)
__device__ __noinline__ Window cull_pair_window(Window w, const GaussSoA grec, int j, int g, int lane) {
  const int jj = j + (lane & 1);
  CellBox b = cutoff_box(grec.A[jj], grec.E[jj], g);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    b.lo[a] = min(b.lo[a], __shfl_xor_sync(MG_FULL, b.lo[a], 1));
    b.hi[a] = max(b.hi[a], __shfl_xor_sync(MG_FULL, b.hi[a], 1));
  }
  cull_window(w, b);
  return w;
}

// Shrink a window to (its intersection with) a cell box.
__device__ __forceinline__ void cull_window(Window& w, const CellBox& b) {
  const int ihi = min(w.ilo + (int)(((float)w.ncol + 0.5f) * w.inv_nj) - 1, b.hi[0]);
  const int jhi = min(w.jlo + w.nj - 1, b.hi[1]);
  w.ilo = max(w.ilo, b.lo[0]);
  w.jlo = max(w.jlo, b.lo[1]);
  w.klo = max(w.klo, b.lo[2]);
  w.khi = min(w.khi, b.hi[2]);
  w.nj = max(jhi - w.jlo + 1, 0);
  w.ncol = w.nj > 0 && ihi >= w.ilo && w.khi >= w.klo ? (ihi - w.ilo + 1) * w.nj : 0;
  w.inv_nj = 1.0f / (float)max(w.nj, 1);
}

// ---------------------------------------------------------------------------
// Bitmap segment cursor.  For a batch of <= 128 columns the candidate list is
// the concatenation of the non-empty column segments.  Each warp keeps, in
// shared memory, delta[seg] = (segment start element) - (segment start in the
// flattened index) for the compacted non-empty segments, and a bitmap with one
// bit per flattened index that starts a segment, over a window of
// kBmWords*32 indices.  A lane then maps its flattened index v to its element
// with one broadcast LDS + popc + one LDS: no loops, no divergence.
// ---------------------------------------------------------------------------
constexpr int kBmWords = 128;  // window of 4096 flattened indices

struct SegSmem {
  uint32_t bits[kBmWords];  // first: pair items alias this struct (PairSmem) and share the bitmap
  int delta[128];
  __align__(16) float pts[3][8];  // an item's sub-points, coordinate-major (pairs load as 64-bit)
};

// Per-lane copy of its 4 columns' (pre, len, start) for window rebuilds.
struct LaneSegs {
  int pre[4], len[4], st[4];
  int nonempty_before;  // # non-empty segments owned by lower lanes
  int tot;
};

// Column bounds from the global CSR starts (the default source).
struct CsrCols {
  const int* __restrict__ starts;
  __device__ __forceinline__ void bounds(const Window& w, int ii, int jj, int g, int& a, int& b) const {
    const int base = (ii * g + jj) * g;
    a = __ldg(starts + base + w.klo);
    b = __ldg(starts + base + w.khi + 1);
  }
};

template <class Cols>
__device__ __noinline__ LaneSegs build_lane_segs_t(const Window& w, int c0, int g, const Cols& cols, SegSmem& sm,
                                                   int lane) {
  LaneSegs L;
  int sum = 0, ne = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    int col = c0 + lane * 4 + k;
    L.st[k] = 0;
    L.len[k] = 0;
    if (col < w.ncol) {
      const int q = (int)(((float)col + 0.5f) * w.inv_nj);  // == col / nj (exact for small ints)
      int a, b;
      cols.bounds(w, w.ilo + q, w.jlo + (col - q * w.nj), g, a, b);
      L.st[k] = a;
      L.len[k] = b - a;
    }
    sum += L.len[k];
    ne += L.len[k] > 0;
  }
  int tot, netot;
  int off = warp_excl_scan(sum, lane, &tot);
  int nbefore = warp_excl_scan(ne, lane, &netot);
  int e = nbefore;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    L.pre[k] = off;
    if (L.len[k] > 0) sm.delta[e++] = L.st[k] - off;
    off += L.len[k];
  }
  L.nonempty_before = nbefore;
  L.tot = tot;
  return L;
}

__device__ __forceinline__ LaneSegs build_lane_segs(const Window& w, int c0, int g, const int* __restrict__ starts,
                                                    SegSmem& sm, int lane) {
  return build_lane_segs_t(w, c0, g, CsrCols{starts}, sm, lane);
}

// Fill the bitmap for flattened window [w0, w0 + 32*kBmWords); returns the
// number of non-empty segments that start before w0 (the window's seg base).
__device__ __noinline__ int build_window(const LaneSegs& L, int w0, SegSmem& sm, int lane) {
#pragma unroll
  for (int i = 0; i < kBmWords / 32; ++i) sm.bits[lane + 32 * i] = 0u;
  __syncwarp();
  int before = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (L.len[k] > 0) {
      int p = L.pre[k] - w0;
      if (p < 0)
        ++before;
      else if (p < 32 * kBmWords)
        atomicOr(&sm.bits[p >> 5], 1u << (p & 31));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) before += __shfl_xor_sync(MG_FULL, before, o);
  __syncwarp();
  return before;
}

// ---------------------------------------------------------------------------
// Transposed ("reduce-scatter") warp reduction of NV <= 32 per-lane values:
// after it, lane l holds the warp sum of value index (l >> (5 - log2 NV)).
// NV - 1 + (5 - log2 NV) shuffles instead of 5 * NV.
// ---------------------------------------------------------------------------
template <int NV>
__device__ __forceinline__ float transpose_reduce(float (&v)[32], int lane) {
  int nrem = NV;
#pragma unroll
  for (int half = 16; half >= 1; half >>= 1) {
    if (nrem > 1) {
      const bool upper = (lane & half) != 0;
      const int h2 = nrem / 2;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (i < h2) {
          float send = upper ? v[i] : v[i + h2];
          float keep = upper ? v[i + h2] : v[i];
          v[i] = keep + __shfl_xor_sync(MG_FULL, send, half);
        }
      }
      nrem = h2;
    } else {
      v[0] += __shfl_xor_sync(MG_FULL, v[0], half);
    }
  }
  return v[0];
}
template <int NV>
struct RedShift {
  static constexpr int value = NV >= 32 ? 0 : (NV >= 16 ? 1 : (NV >= 8 ? 2 : (NV >= 4 ? 3 : (NV >= 2 ? 4 : 5))));
};

// Write the reduced (I, H) of point q of an item.  comp 0 = I -> .w,
// comps 1..3 = H' -> .xyz (P' scale removed).
__device__ __forceinline__ void write_point_out(float4* __restrict__ out4, int* __restrict__ cnt_out, int p, int comp,
                                                float val, int total) {
  float* o = reinterpret_cast<float*>(out4 + p);
  if (comp == 0) {
    o[3] = val;
    cnt_out[p] = total;
  } else {
    o[comp - 1] = val * (1.0f / kMScale);
  }
}

// ---------------------------------------------------------------------------
// Forward: one warp per (point cell, <= Q sub-points of that cell); lanes
// stride over the flattened candidate Gaussians, two per lane per 64-wide
// window, with the next window's records prefetched while the current one
// is evaluated.  The item's sub-points are warp-uniform and packed two per
// f32x2 register; Gaussian parameters enter FFMA2 as scalar-broadcast
// operands.  Every sub-point of an item shares the exact candidate set, so
// contributor_counts is the item's total candidate count.
// ---------------------------------------------------------------------------
// One CTA per SM: all resident warps take consecutive (neighbouring-cell)
// items, so their candidate windows overlap in L1 (3 CTAs x 8 warps ran
// three unrelated regions per SM: forward 0.584 -> 0.552 ms, backward
// 0.598 -> 0.560 ms at C2).
#ifndef MG_FWD_MINB
#define MG_FWD_MINB 1
#endif
#ifndef MG_BWD_MINB
#define MG_BWD_MINB 1
#endif
#ifndef MG_FWD_QMAX
#define MG_FWD_QMAX 6  // up to 6 sub-points per item: Q=8 spills at 80 registers (C2: 0.618 -> 0.593 ms)
#endif
#ifndef MG_FWD_GPL_Q2
#define MG_FWD_GPL_Q2 2  // candidates per lane per window for 2-point items (2 or 4)
#endif
#ifndef MG_FWD_GPL1_QP
#define MG_FWD_GPL1_QP 4  // items with >= this many point pairs take one candidate per lane per window:
                          // two per lane (two record loads in flight) measured 3% faster up to Q = 6
#endif
#ifndef MG_FWD_SCHED
#define MG_FWD_SCHED 1  // CTA-contiguous item ranges + shared-counter hand-out (0: fixed stride)
#endif
#ifndef MG_FWD_WARPS
#define MG_FWD_WARPS 24
#endif
#ifndef MG_FWD_IPF
#define MG_FWD_IPF 0  // next-item prefetch: was 2% faster at 3 CTAs/SM, is 1.5% slower with the per-CTA hand-out
#endif
#ifndef MG_BWD_IPF
#define MG_BWD_IPF 0  // off: with implicit items the prefetch measured ~2% slower
#endif
#ifndef MG_BWD_PAIR_GPACK
#define MG_BWD_PAIR_GPACK 1  // pair items: Gaussian-packed f32x2 (points broadcast)
#endif
#ifndef MG_BWD_WARPS
#define MG_BWD_WARPS 16
#endif
constexpr int kFwdWarps = MG_FWD_WARPS;

struct GRec {
  float4 A, B;  // {mu, alpha}, {P'00, P'11, P'22, P'01}
  float2 C;     // {P'02, P'12}
};

__device__ __forceinline__ GRec load_rec(const GaussSoA& grec, int gi) {
  GRec r;
  r.A = __ldg(grec.A + gi);
  r.B = __ldg(grec.B + gi);
  r.C = __ldg(grec.C + gi);
  return r;
}

// Record sources of the forward item loops: candidate columns + records from
// global memory (CSR starts, SoA records), or from a block's staged tile.
struct GlobalRecs {
  GaussSoA grec;
  const int* __restrict__ gstart;
  __device__ __forceinline__ LaneSegs segs(const Window& w, int c0, int g, SegSmem& sm, int lane) const {
    return build_lane_segs_t(w, c0, g, CsrCols{gstart}, sm, lane);
  }
  __device__ __forceinline__ GRec rec(int i) const { return load_rec(grec, i); }
};

// cp.async helpers (4/8/16-byte asynchronous global -> shared copies).
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Flattened-window cursor, one candidate per lane per 32-wide window.
struct Cursor1 {
  int sbase;
  __device__ __forceinline__ void next(const SegSmem& sm, int w0, int base, unsigned upto, int lane, int& va,
                                       int& ga) {
    const uint32_t M0 = sm.bits[(base - w0) >> 5];
    va = base + lane;
    const int sega = sbase + __popc(M0 & upto) - 1;
    sbase += __popc(M0);
    ga = va + sm.delta[sega];
  }
};

// Flattened-window cursor: lanes take va = base + lane and vb = va + 32.
struct Cursor2 {
  int sbase;
  __device__ __forceinline__ void next(const SegSmem& sm, int w0, int base, unsigned upto, int lane, int& va, int& vb,
                                       int& ga, int& gb) {
    const int wi = (base - w0) >> 5;
    const uint32_t M0 = sm.bits[wi], M1 = sm.bits[wi + 1];
    va = base + lane;
    vb = va + 32;
    const int p0 = __popc(M0);
    const int sega = sbase + __popc(M0 & upto) - 1;
    const int segb = sbase + p0 + __popc(M1 & upto) - 1;
    sbase += p0 + __popc(M1);
    ga = va + sm.delta[sega];
    gb = vb + sm.delta[segb];
  }
};

// Flattened-window cursor for 128-wide windows: lane owns v_i = base + 32 i +
// lane (i = 0..3), so each warp-wide point load reads 512 contiguous bytes.
struct Cursor4 {
  int sbase;
  __device__ __forceinline__ void next(const SegSmem& sm, int w0, int base, unsigned upto, int lane, int (&v)[4],
                                       int (&e)[4]) {
    const int wi = (base - w0) >> 5;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t M = sm.bits[wi + i];
      v[i] = base + 32 * i + lane;
      e[i] = v[i] + sm.delta[sbase + __popc(M & upto) - 1];
      sbase += __popc(M);
    }
  }
};

template <int QP, bool WITH_H>
__device__ __forceinline__ void fwd_pair_math(const GRec& g, const f2 (&px)[QP], const f2 (&py)[QP],
                                              const f2 (&pz)[QP], f2 (&accI)[QP], f2 (&hx)[QP], f2 (&hy)[QP],
                                              f2 (&hz)[QP]) {
  const float p00 = g.B.x, p11 = g.B.y, p22 = g.B.z, p01 = g.B.w, p02 = g.C.x, p12 = g.C.y;
  const f2 mx = bc2(g.A.x), my = bc2(g.A.y), mz = bc2(g.A.z), al = bc2(g.A.w);
  if (WITH_H) {
#pragma unroll
    for (int q = 0; q < QP; ++q) {
      f2 dx = sub2(px[q], mx), dy = sub2(py[q], my), dz = sub2(pz[q], mz);
      f2 pdx = fma2(bc2(p02), dz, fma2(bc2(p01), dy, mul2(bc2(p00), dx)));
      f2 pdy = fma2(bc2(p12), dz, fma2(bc2(p11), dy, mul2(bc2(p01), dx)));
      f2 pdz = fma2(bc2(p22), dz, fma2(bc2(p12), dy, mul2(bc2(p02), dx)));
      f2 m = fma2(dz, pdz, fma2(dy, pdy, mul2(dx, pdx)));
      f2 wv = mul2(al, gauss_w2(m));
      accI[q] = add2(accI[q], wv);
      hx[q] = fma2(wv, pdx, hx[q]);
      hy[q] = fma2(wv, pdy, hy[q]);
      hz[q] = fma2(wv, pdz, hz[q]);
    }
  } else {
    const float a01 = 2.f * p01, a02 = 2.f * p02, a12 = 2.f * p12;
#pragma unroll
    for (int q = 0; q < QP; ++q) {
      f2 dx = sub2(px[q], mx), dy = sub2(py[q], my), dz = sub2(pz[q], mz);
      f2 t1 = fma2(bc2(a02), dz, fma2(bc2(a01), dy, mul2(bc2(p00), dx)));
      f2 m = mul2(dx, t1);
      f2 t2 = fma2(bc2(a12), dz, mul2(bc2(p11), dy));
      m = fma2(dy, t2, m);
      m = fma2(dz, mul2(bc2(p22), dz), m);
      accI[q] = fma2(al, gauss_w2(m), accI[q]);
    }
  }
}

template <int Q, bool WITH_H, class Src>
__device__ __forceinline__ void fwd_item(const Src& src, int g, int r, const float4* __restrict__ prec, int p0,
                                         int np, int cell, float4* __restrict__ out4, int* __restrict__ cnt_out,
                                         SegSmem& sm, int lane) {
  constexpr int QP = Q / 2;
  // candidates per lane per window: two, so two record loads are in flight
  // per lane (the loop is L1/L2-latency bound), unless QP >= MG_FWD_GPL1_QP.
  constexpr int GPL = QP >= MG_FWD_GPL1_QP ? 1 : (QP == 1 ? MG_FWD_GPL_Q2 : 2);
  constexpr int WIN = 32 * GPL;
  // stage the item's sub-points coordinate-major in shared memory and read
  // them back as 64-bit pairs: the f32x2 operands then sit in aligned
  // register pairs for the whole loop (no re-pairing moves per use)
  if (lane < Q) {
    const float4 a = prec[p0 + min(lane, np - 1)];
    sm.pts[0][lane] = a.x;
    sm.pts[1][lane] = a.y;
    sm.pts[2][lane] = a.z;
  }
  __syncwarp();
  f2 px[QP], py[QP], pz[QP];
#pragma unroll
  for (int q = 0; q < QP; ++q) {
    px[q].v = *reinterpret_cast<const unsigned long long*>(&sm.pts[0][2 * q]);
    py[q].v = *reinterpret_cast<const unsigned long long*>(&sm.pts[1][2 * q]);
    pz[q].v = *reinterpret_cast<const unsigned long long*>(&sm.pts[2][2 * q]);
  }
  __syncwarp();
  f2 accI[QP], hx[QP], hy[QP], hz[QP];
#pragma unroll
  for (int q = 0; q < QP; ++q) accI[q] = hx[q] = hy[q] = hz[q] = bc2(0.f);
  const Window w = make_window(cell, g, r);
  const unsigned upto = 0xffffffffu >> (31 - lane);  // bits 0..lane
  int total = 0;
  for (int c0 = 0; c0 < w.ncol; c0 += 128) {
    const LaneSegs L = src.segs(w, c0, g, sm, lane);
    const int tot = L.tot;
    total += tot;
    for (int w0 = 0; w0 < tot; w0 += 32 * kBmWords) {
      const int sb0 = build_window(L, w0, sm, lane);
      const int wend = min(tot, w0 + 32 * kBmWords);
      // one compact loop: prefetching (register ring, cp.async ring, L1
      // prefetch) all measured slower -- the kernel is L1/issue-bound
      if (GPL == 1) {
        Cursor1 cur{sb0};
        for (int base = w0; base < wend; base += WIN) {
          int va, ga;
          cur.next(sm, w0, base, upto, lane, va, ga);
          if (va < wend) fwd_pair_math<QP, WITH_H>(src.rec(ga), px, py, pz, accI, hx, hy, hz);
        }
      } else if (GPL == 2) {
        Cursor2 cur{sb0};
        for (int base = w0; base < wend; base += WIN) {
          int va, vb, ga, gb;
          cur.next(sm, w0, base, upto, lane, va, vb, ga, gb);
          const GRec ra = src.rec(va < wend ? ga : 0);
          const GRec rb = src.rec(vb < wend ? gb : 0);
          if (va < wend) fwd_pair_math<QP, WITH_H>(ra, px, py, pz, accI, hx, hy, hz);
          if (vb < wend) fwd_pair_math<QP, WITH_H>(rb, px, py, pz, accI, hx, hy, hz);
        }
      } else {  // four candidates per lane (four record loads in flight)
        Cursor4 cur{sb0};
        for (int base = w0; base < wend; base += WIN) {
          int v[4], e[4];
          cur.next(sm, w0, base, upto, lane, v, e);
          GRec rr[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) rr[i] = src.rec(v[i] < wend ? e[i] : 0);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (v[i] < wend) fwd_pair_math<QP, WITH_H>(rr[i], px, py, pz, accI, hx, hy, hz);
        }
      }
      __syncwarp();
    }
  }
  constexpr int NV = Q == 6 ? 32 : 4 * Q;  // 8 or 16 (32 at Q = 6, 8)
  float vals[32];
#pragma unroll
  for (int q = 0; q < QP; ++q) {
    vals[8 * q + 0] = lo(accI[q]);
    vals[8 * q + 1] = lo(hx[q]);
    vals[8 * q + 2] = lo(hy[q]);
    vals[8 * q + 3] = lo(hz[q]);
    vals[8 * q + 4] = hi(accI[q]);
    vals[8 * q + 5] = hi(hx[q]);
    vals[8 * q + 6] = hi(hy[q]);
    vals[8 * q + 7] = hi(hz[q]);
  }
#pragma unroll
  for (int i = NV; i < 32; ++i) vals[i] = 0.f;
  const float red = transpose_reduce<NV>(vals, lane);
  constexpr int SH = RedShift<NV>::value;
  const int idx = lane >> SH;
  const int q = idx >> 2, comp = idx & 3;
  if ((lane & ((1 << SH) - 1)) == 0 && q < np) write_point_out(out4, cnt_out, p0 + q, comp, red, total);
}

// np == 1: the single sub-point is broadcast; each lane packs its TWO
// candidates of the window (va, vb) into the two f32x2 halves.
template <bool WITH_H>
__device__ __forceinline__ void single_math(const GRec& a, const GRec& b, bool hb, f2 X, f2 Y, f2 Z, f2& accI,
                                            f2& hx, f2& hy, f2& hz) {
  const f2 dx = sub2(X, mk2(a.A.x, b.A.x)), dy = sub2(Y, mk2(a.A.y, b.A.y)), dz = sub2(Z, mk2(a.A.z, b.A.z));
  const f2 p00 = mk2(a.B.x, b.B.x), p11 = mk2(a.B.y, b.B.y), p22 = mk2(a.B.z, b.B.z), p01 = mk2(a.B.w, b.B.w),
           p02 = mk2(a.C.x, b.C.x), p12 = mk2(a.C.y, b.C.y);
  const f2 al = mk2(a.A.w, hb ? b.A.w : 0.f);
  if (WITH_H) {
    f2 pdx = fma2(p02, dz, fma2(p01, dy, mul2(p00, dx)));
    f2 pdy = fma2(p12, dz, fma2(p11, dy, mul2(p01, dx)));
    f2 pdz = fma2(p22, dz, fma2(p12, dy, mul2(p02, dx)));
    f2 m = fma2(dz, pdz, fma2(dy, pdy, mul2(dx, pdx)));
    f2 wv = mul2(al, gauss_w2(m));
    accI = add2(accI, wv);
    hx = fma2(wv, pdx, hx);
    hy = fma2(wv, pdy, hy);
    hz = fma2(wv, pdz, hz);
  } else {
    f2 t1 = fma2(add2(p02, p02), dz, fma2(add2(p01, p01), dy, mul2(p00, dx)));
    f2 m = mul2(dx, t1);
    m = fma2(dy, fma2(add2(p12, p12), dz, mul2(p11, dy)), m);
    m = fma2(dz, mul2(p22, dz), m);
    accI = fma2(al, gauss_w2(m), accI);
  }
}

template <bool WITH_H, class Src>
__device__ __forceinline__ void fwd_item_single(const Src& src, int g, int r, const float4* __restrict__ prec,
                                                int p0, int cell, float4* __restrict__ out4,
                                                int* __restrict__ cnt_out, SegSmem& sm, int lane) {
  const float4 pt = prec[p0];
  const f2 X = bc2(pt.x), Y = bc2(pt.y), Z = bc2(pt.z);
  f2 accI = bc2(0.f), hx = accI, hy = accI, hz = accI;
  const Window w = make_window(cell, g, r);
  const unsigned upto = 0xffffffffu >> (31 - lane);
  int total = 0;
  for (int c0 = 0; c0 < w.ncol; c0 += 128) {
    const LaneSegs L = src.segs(w, c0, g, sm, lane);
    const int tot = L.tot;
    total += tot;
    for (int w0 = 0; w0 < tot; w0 += 32 * kBmWords) {
      Cursor2 cur{build_window(L, w0, sm, lane)};
      const int wend = min(tot, w0 + 32 * kBmWords);
      for (int base = w0; base < wend; base += 64) {
        int va, vb, ga, gb;
        cur.next(sm, w0, base, upto, lane, va, vb, ga, gb);
        if (va < wend) {
          const bool hb = vb < wend;
          const GRec ra = src.rec(ga);
          const GRec rb = src.rec(hb ? gb : ga);
          single_math<WITH_H>(ra, rb, hb, X, Y, Z, accI, hx, hy, hz);
        }
      }
      __syncwarp();
    }
  }
  float vals[32];
  vals[0] = lo(accI) + hi(accI);
  vals[1] = lo(hx) + hi(hx);
  vals[2] = lo(hy) + hi(hy);
  vals[3] = lo(hz) + hi(hz);
#pragma unroll
  for (int i = 4; i < 32; ++i) vals[i] = 0.f;
  const float red = transpose_reduce<4>(vals, lane);
  const int comp = lane >> 3;
  if ((lane & 7) == 0) write_point_out(out4, cnt_out, p0, comp, red, total);
}


// Dense cells (>= kFwdDenseMin sub-points, e.g. the per-step SSIM slice plane):
// lanes own sub-points (two per lane, packed), the cell's candidate Gaussians
// stream through warp-uniform (broadcast) loads -- one record fetch serves 64
// pairs instead of 4.
#ifndef MG_FWD_DENSE_MIN
#define MG_FWD_DENSE_MIN 0  // measured slower at C2 (long serial per-item Gaussian stream): off
#endif
constexpr int kFwdDenseMin = MG_FWD_DENSE_MIN;

template <bool WITH_H>
__device__ __forceinline__ void fwd_item_dense(const GaussSoA& grec, const int* __restrict__ gstart, int g, int r,
                                               const float4* __restrict__ prec, int p0, int np, int cell,
                                               float4* __restrict__ out4, int* __restrict__ cnt_out, SegSmem& sm,
                                               int lane) {
  // lane owns points lane (lo half) and lane + 32 (hi half); staged adjacently
  // in shared memory so each coordinate pair reloads as one 64-bit value
  static_assert(sizeof(SegSmem::delta) + sizeof(SegSmem::bits) >= 3 * 64 * sizeof(float), "dense staging");
  float* buf = reinterpret_cast<float*>(sm.bits);  // 3 x 64 floats in bits[] + delta[] (unused on this path)
  {
    const float4 a = prec[p0 + min(lane, np - 1)];
    const float4 b = prec[p0 + min(lane + 32, np - 1)];
    buf[0 * 64 + 2 * lane] = a.x;
    buf[0 * 64 + 2 * lane + 1] = b.x;
    buf[1 * 64 + 2 * lane] = a.y;
    buf[1 * 64 + 2 * lane + 1] = b.y;
    buf[2 * 64 + 2 * lane] = a.z;
    buf[2 * 64 + 2 * lane + 1] = b.z;
  }
  __syncwarp();
  f2 px[1], py[1], pz[1];
  px[0].v = *reinterpret_cast<const unsigned long long*>(buf + 0 * 64 + 2 * lane);
  py[0].v = *reinterpret_cast<const unsigned long long*>(buf + 1 * 64 + 2 * lane);
  pz[0].v = *reinterpret_cast<const unsigned long long*>(buf + 2 * 64 + 2 * lane);
  __syncwarp();
  f2 accI[1], hx[1], hy[1], hz[1];
  accI[0] = hx[0] = hy[0] = hz[0] = bc2(0.f);
  const Window w = make_window(cell, g, r);
  int total = 0;
  for (int col = 0; col < w.ncol; ++col) {
    const int q = (int)(((float)col + 0.5f) * w.inv_nj);
    const int base = ((w.ilo + q) * g + (w.jlo + col - q * w.nj)) * g;
    const int a = __ldg(gstart + base + w.klo), b = __ldg(gstart + base + w.khi + 1);
    total += b - a;
#pragma unroll 2
    for (int gi = a; gi < b; ++gi) fwd_pair_math<1, WITH_H>(load_rec(grec, gi), px, py, pz, accI, hx, hy, hz);
  }
  const float s = 1.0f / kMScale;
  if (lane < np) {
    out4[p0 + lane] = make_float4(lo(hx[0]) * s, lo(hy[0]) * s, lo(hz[0]) * s, lo(accI[0]));
    cnt_out[p0 + lane] = total;
  }
  if (lane + 32 < np) {
    out4[p0 + lane + 32] = make_float4(hi(hx[0]) * s, hi(hy[0]) * s, hi(hz[0]) * s, hi(accI[0]));
    cnt_out[p0 + lane + 32] = total;
  }
}

template <bool WITH_H, class Src>
__device__ __forceinline__ void fwd_dispatch(const Src& src, int g, int r, const float4* __restrict__ prec, int p0,
                                             int np, int cell, float4* __restrict__ out4, int* __restrict__ cnt_out,
                                             SegSmem& sm, int lane) {
  if (MG_FWD_QMAX > 4 && np > 4)
    fwd_item<(MG_FWD_QMAX > 6 ? 8 : (MG_FWD_QMAX > 4 ? 6 : 4)), WITH_H>(src, g, r, prec, p0, np, cell, out4, cnt_out,
                                                                        sm, lane);
  else if (np > 2)
    fwd_item<4, WITH_H>(src, g, r, prec, p0, np, cell, out4, cnt_out, sm, lane);
  else if (np == 2)
    fwd_item<2, WITH_H>(src, g, r, prec, p0, np, cell, out4, cnt_out, sm, lane);
  else
    fwd_item_single<WITH_H>(src, g, r, prec, p0, cell, out4, cnt_out, sm, lane);
}

template <bool WITH_H>
__global__ void __launch_bounds__(kFwdWarps * 32, MG_FWD_MINB) forward_kernel(const GaussSoA grec,
                                                                 const int* __restrict__ gstart, int g, int r,
                                                                 const float4* __restrict__ prec,
                                                                 const uint32_t* __restrict__ pkey,
                                                                 const int* __restrict__ pstart,
                                                                 const int4* __restrict__ items,
                                                                 const int* __restrict__ nitems_dev,
                                                                 float4* __restrict__ out4, int* __restrict__ cnt_out) {
  __shared__ SegSmem s_seg[kFwdWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nitems = *nitems_dev;
#if MG_FWD_SCHED
  // CTA-contiguous item range, items handed to warps by a shared counter:
  // the CTA's warps stay on neighbouring cells (L1 reuse) and balance
  // dynamically (a warp's share is no longer a fixed stride of items)
  __shared__ int s_next;
  if (threadIdx.x == 0) s_next = 0;
  __syncthreads();
  const int per = (nitems + gridDim.x - 1) / gridDim.x;
  const int beg = blockIdx.x * per, end = min(nitems, beg + per);
  auto grab = [&]() {
    int t = 0;
    if (lane == 0) t = atomicAdd(&s_next, 1);
    return beg + __shfl_sync(MG_FULL, t, 0);
  };
  int it = grab();
  int nx = it < end ? grab() : end;
  int4 next = (MG_FWD_IPF && it < end) ? items[it] : make_int4(0, 0, 0, 0);
  while (it < end) {
    const int4 item = MG_FWD_IPF ? next : items[it];  // {first, cell, count, 0}
    if (MG_FWD_IPF && nx < end) next = items[nx];  // loads under this item
    it = nx;
    nx = it < end ? grab() : end;
#else
  const int nw = blockDim.x >> 5;  // kFwdWarps, or 8 for small launches
  const int stride = gridDim.x * nw;
  int it = blockIdx.x * nw + warp;
  int4 next = (MG_FWD_IPF && it < nitems) ? items[it] : make_int4(0, 0, 0, 0);
  for (; it < nitems; it += stride) {
    const int4 item = MG_FWD_IPF ? next : items[it];  // {first, cell, count, 0}
    if (MG_FWD_IPF && it + stride < nitems) next = items[it + stride];  // loads under this item
#endif
    const int p0 = item.x, cell = item.y;
    if (kFwdDenseMin > 0 && item.z > MG_FWD_QMAX) {
      fwd_item_dense<WITH_H>(grec, gstart, g, r, prec, p0, item.z, cell, out4, cnt_out, s_seg[warp], lane);
      continue;
    }
    fwd_dispatch<WITH_H>(GlobalRecs{grec, gstart}, g, r, prec, p0, item.z, cell, out4, cnt_out, s_seg[warp], lane);
  }
}

// ---------------------------------------------------------------------------
// Backward, Gaussian-major: one warp per (Gaussian cell, <= 2 Gaussians of
// that cell); lanes stride over the flattened candidate sub-points, four per
// lane per 128-wide window as two f32x2 pairs (v, v+1) and (v+64, v+65), the
// next window's points prefetched.  Per Gaussian it accumulates
// (register-resident, no atomics):
//   S = sum u*g,  T = sum u*g*(P'd),  A6 = sum u*g*(d d^T)
// and the epilogue forms d_alpha = S, d_mu = alpha*T/kMScale,
// d_abar6 = -0.5*alpha*A6 (_kernels.py:118-141).
// ---------------------------------------------------------------------------
constexpr int kBwdWarps = MG_BWD_WARPS;

struct Pts4 {
  float4 p[4];
};

template <int QG>
struct GaussAcc {
  float mx[QG], my[QG], mz[QG], P[QG][6];  // P: P'00, P'11, P'22, 2P'01, 2P'02, 2P'12
  // S = sum u g, D1 = sum u g d (T = P' D1 is formed at the end), A6 = sum u g d d^T
  f2 S[QG], T[QG][3], A6[QG][6];

  __device__ __forceinline__ void pair(const float4& a, const float4& b) {
    const f2 px = mk2(a.x, b.x), py = mk2(a.y, b.y), pz = mk2(a.z, b.z), u = mk2(a.w, b.w);
#pragma unroll
    for (int k = 0; k < QG; ++k) accum(k, px, py, pz, u);
  }
  // Gaussian k over a point pair with upstream u (f32x2)
  __device__ __forceinline__ void accum(int k, f2 px, f2 py, f2 pz, f2 u) {
    {
      f2 dx = sub2(px, bc2(mx[k])), dy = sub2(py, bc2(my[k])), dz = sub2(pz, bc2(mz[k]));
      // m' = d^T P' d, Horner with doubled off-diagonals (9 FP32 ops)
      f2 t1 = fma2(bc2(P[k][4]), dz, fma2(bc2(P[k][3]), dy, mul2(bc2(P[k][0]), dx)));
      f2 m = mul2(dx, t1);
      m = fma2(dy, fma2(bc2(P[k][5]), dz, mul2(bc2(P[k][1]), dy)), m);
      m = fma2(dz, mul2(bc2(P[k][2]), dz), m);
      f2 ug = mul2(u, gauss_w2(m));
      S[k] = add2(S[k], ug);
      f2 cx = mul2(ug, dx), cy = mul2(ug, dy), cz = mul2(ug, dz);
      T[k][0] = add2(T[k][0], cx);
      T[k][1] = add2(T[k][1], cy);
      T[k][2] = add2(T[k][2], cz);
      A6[k][0] = fma2(cx, dx, A6[k][0]);
      A6[k][1] = fma2(cx, dy, A6[k][1]);
      A6[k][2] = fma2(cx, dz, A6[k][2]);
      A6[k][3] = fma2(cy, dy, A6[k][3]);
      A6[k][4] = fma2(cy, dz, A6[k][4]);
      A6[k][5] = fma2(cz, dz, A6[k][5]);
    }
  }

  __device__ __forceinline__ void load(const GaussSoA& grec, int k, int gi) {
    const float4 A = grec.A[gi], B = grec.B[gi];
    const float2 C = grec.C[gi];
    mx[k] = A.x;
    my[k] = A.y;
    mz[k] = A.z;
    P[k][0] = B.x;
    P[k][1] = B.y;
    P[k][2] = B.z;
    P[k][3] = 2.f * B.w;  // doubling is exact
    P[k][4] = 2.f * C.x;
    P[k][5] = 2.f * C.y;
    S[k] = bc2(0.f);
#pragma unroll
    for (int c = 0; c < 3; ++c) T[k][c] = bc2(0.f);
#pragma unroll
    for (int c = 0; c < 6; ++c) A6[k][c] = bc2(0.f);
  }
  // one 128-wide window: the lane's points v, v+32, v+64, v+96 as two pairs
  __device__ __forceinline__ void quad(const float4 (&q)[4]) {
    pair(q[0], q[1]);
    pair(q[2], q[3]);
  }
  // ragged window: missing points are zero records (zero upstream)
  __device__ __forceinline__ void quad_tail(const float4 (&q)[4], const int (&v)[4], int wend) {
    if (v[0] < wend) pair(q[0], q[1]);
    if (v[2] < wend) pair(q[2], q[3]);
  }

  // lane-local totals of the 10 accumulators of Gaussian k, T = P' D1
  __device__ __forceinline__ void totals(int k, float* v) const {
    v[0] = lo(S[k]) + hi(S[k]);
    const float d1x = lo(T[k][0]) + hi(T[k][0]), d1y = lo(T[k][1]) + hi(T[k][1]), d1z = lo(T[k][2]) + hi(T[k][2]);
    const float h01 = 0.5f * P[k][3], h02 = 0.5f * P[k][4], h12 = 0.5f * P[k][5];
    v[1] = P[k][0] * d1x + h01 * d1y + h02 * d1z;
    v[2] = h01 * d1x + P[k][1] * d1y + h12 * d1z;
    v[3] = h02 * d1x + h12 * d1y + P[k][2] * d1z;
#pragma unroll
    for (int c = 0; c < 6; ++c) v[4 + c] = lo(A6[k][c]) + hi(A6[k][c]);
  }
};

// Candidate-point window loop: lanes stride over the flattened candidate
// points, four per lane per 128-wide window.
template <class Acc>
__device__ __forceinline__ void bwd_window_loop(Acc& acc, const Window& w, int g, const float4* __restrict__ prec,
                                                const int* __restrict__ pstart, SegSmem& sm, int lane) {
  const unsigned upto = 0xffffffffu >> (31 - lane);  // bits 0..lane
  for (int c0 = 0; c0 < w.ncol; c0 += 128) {
    const LaneSegs L = build_lane_segs(w, c0, g, pstart, sm, lane);
    const int tot = L.tot;
    for (int w0 = 0; w0 < tot; w0 += 32 * kBmWords) {
      Cursor4 cur{build_window(L, w0, sm, lane)};
      const int wend = min(tot, w0 + 32 * kBmWords);
      const int nfull = (wend - w0) >> 7;
      int v[4], e[4];
      for (int t = 0; t < nfull; ++t) {
        cur.next(sm, w0, w0 + 128 * t, upto, lane, v, e);
        float4 q[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) q[i] = __ldg(prec + e[i]);
        acc.quad(q);
      }
      const int tb = w0 + (nfull << 7);
      if (tb < wend) {  // ragged tail window
        cur.next(sm, w0, tb, upto, lane, v, e);
        float4 pt[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) pt[i] = v[i] < wend ? __ldg(prec + e[i]) : make_float4(0.f, 0.f, 0.f, 0.f);
        acc.quad_tail(pt, v, wend);
      }
      __syncwarp();
    }
  }
}

template <int QG, class Acc>
__device__ __forceinline__ void bwd_store(const Acc& acc, int g0, int ng, float* __restrict__ acc10, int lane);

template <int QG>
__device__ __forceinline__ void bwd_item(const GaussSoA grec, int g0, int ng, int cell, int g, int r,
                                         const float4* __restrict__ prec, const int* __restrict__ pstart,
                                         float* __restrict__ acc10, SegSmem& sm, int lane, bool cull = false) {
  Window w = make_window(cell, g, r);
  if (MG_BWD_CULL && QG == 1 && cull && may_cull(grec.E[g0], g, r)) w = cull_single_window(w, grec, g0, g);
  GaussAcc<QG> acc;
#pragma unroll
  for (int k = 0; k < QG; ++k) acc.load(grec, k, g0 + min(k, ng - 1));
  bwd_window_loop(acc, w, g, prec, pstart, sm, lane);
  bwd_store<QG>(acc, g0, ng, acc10, lane);
}

// 10 sums per Gaussian (x QG, padded to 16 / 32) -> transposed reduction.
template <int QG, class Acc>
__device__ __forceinline__ void bwd_store(const Acc& acc, int g0, int ng, float* __restrict__ acc10, int lane) {
  constexpr int NV = QG == 1 ? 16 : 32;
  float vals[32];
#pragma unroll
  for (int k = 0; k < QG; ++k) {
    acc.totals(k, vals + 16 * k);
#pragma unroll
    for (int c = 10; c < 16; ++c) vals[16 * k + c] = 0.f;
  }
#pragma unroll
  for (int i = 16 * QG; i < 32; ++i) vals[i] = 0.f;
  const float red = transpose_reduce<NV>(vals, lane);
  constexpr int SH = RedShift<NV>::value;
  const int idx = lane >> SH;
  const int k = idx >> 4, c = idx & 15;
  if ((lane & ((1 << SH) - 1)) == 0 && c < 10 && k < ng) acc10[(int64_t)(g0 + k) * 10 + c] = red;
}


// ---------------------------------------------------------------------------
// Pair items: sorted Gaussians 2j and 2j+1 whose cells lie in one (i, j)
// column at most MG_BWD_PAIR_DMAX k-cells apart share ONE candidate window --
// the union of their (2r+1)^3 neighbourhoods, which differs from each by dk
// k-cells per column.  Every column also records two element thresholds:
// elements before `aend` lie in the A-only cells, elements from `bbeg` on in
// the B-only cells, and the other Gaussian sees those points
// with zero upstream -- so each Gaussian still sums over exactly its own
// candidate set.  Halves the per-item window builds and shares every point
// load and cursor step between two Gaussians.
// ---------------------------------------------------------------------------
// Per-warp shared memory of a pair item; aliases SegSmem (the bitmap is the
// first member of both, so build_window serves either).
struct PairSmem {
  uint32_t bits[kBmWords];
  int4 dt[128];            // per non-empty column segment: {delta, A-only end, B-only start, -} (flattened index)
  __align__(16) float stage[24];  // the pair's 9 parameter pairs (read back as 64-bit)
};
union WarpSmem {
  SegSmem seg;
  PairSmem pair;
};
static_assert(offsetof(SegSmem, bits) == 0 && offsetof(PairSmem, bits) == 0, "bitmap must alias");

struct PairCols {
  const int* __restrict__ starts;
  int kae, kbs;  // A-only cells [klo, kae), B-only cells [kbs, khi]
};

__device__ __noinline__ LaneSegs build_lane_segs_pair(const Window& w, int c0, int g, const PairCols cols,
                                                      PairSmem& ps, int lane) {
  LaneSegs L;
  int2 t[4];
  int sum = 0, ne = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int col = c0 + lane * 4 + k;
    L.st[k] = 0;
    L.len[k] = 0;
    t[k] = make_int2(0, 0);
    if (col < w.ncol) {
      const int q = (int)(((float)col + 0.5f) * w.inv_nj);  // == col / nj
      const int base = ((w.ilo + q) * g + w.jlo + (col - q * w.nj)) * g;
      const int a = __ldg(cols.starts + base + w.klo);
      const int b = __ldg(cols.starts + base + w.khi + 1);
      t[k] = make_int2(__ldg(cols.starts + base + cols.kae), __ldg(cols.starts + base + cols.kbs));
      L.st[k] = a;
      L.len[k] = b - a;
    }
    sum += L.len[k];
    ne += L.len[k] > 0;
  }
  int tot, netot;
  int off = warp_excl_scan(sum, lane, &tot);
  const int nbefore = warp_excl_scan(ne, lane, &netot);
  int e = nbefore;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    L.pre[k] = off;
    if (L.len[k] > 0) {  // {delta, A-only end, B-only start} with thresholds in flattened-index space
      const int d = L.st[k] - off;
      ps.dt[e++] = make_int4(d, t[k].x - d, t[k].y - d, 0);
    }
    off += L.len[k];
  }
  L.nonempty_before = nbefore;
  L.tot = tot;
  return L;
}

#ifndef MG_PAIR_INLINE
#define MG_PAIR_INLINE 1
#endif
// Inlined pair builder: the window arrives as scalars in registers (the
// noinline form took it by reference, i.e. from local memory, reloading six
// fields per column, and rebuilt the global-memory descriptor for every
// load), and the four CSR bounds of a column are int32-indexed from one base.
// Per item ~335 -> ~120 instructions at C4.
__device__ __forceinline__ LaneSegs build_lane_segs_pair_inl(int ilo, int jlo, int nj, int ncol, float inv_nj,
                                                             int klo, int kend, int kae, int kbs, int g,
                                                             const int* __restrict__ starts, PairSmem& ps,
                                                             int lane) {
  LaneSegs L;
  int2 t[4];
  int sum = 0, ne = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int col = lane * 4 + k;
    L.st[k] = 0;
    L.len[k] = 0;
    t[k] = make_int2(0, 0);
    if (col < ncol) {
      const int q = (int)(((float)col + 0.5f) * inv_nj);  // == col / nj
      const int base = ((ilo + q) * g + jlo + (col - q * nj)) * g;
      const int a = __ldg(starts + (base + klo));
      const int b = __ldg(starts + (base + kend));
      t[k] = make_int2(__ldg(starts + (base + kae)), __ldg(starts + (base + kbs)));
      L.st[k] = a;
      L.len[k] = b - a;
    }
    sum += L.len[k];
    ne += L.len[k] > 0;
  }
  int tot, netot;
  int off = warp_excl_scan(sum, lane, &tot);
  const int nbefore = warp_excl_scan(ne, lane, &netot);
  int e = nbefore;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    L.pre[k] = off;
    if (L.len[k] > 0) {
      const int d = L.st[k] - off;
      ps.dt[e++] = make_int4(d, t[k].x - d, t[k].y - d, 0);
    }
    off += L.len[k];
  }
  L.nonempty_before = nbefore;
  L.tot = tot;
  return L;
}

__device__ __forceinline__ int build_window_inl(const LaneSegs& L, int w0, uint32_t* bits, int lane) {
#pragma unroll
  for (int i = 0; i < kBmWords / 32; ++i) bits[lane + 32 * i] = 0u;
  __syncwarp();
  int before = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (L.len[k] > 0) {
      const int p = L.pre[k] - w0;
      if (p < 0)
        ++before;
      else if (p < 32 * kBmWords)
        atomicOr(&bits[p >> 5], 1u << (p & 31));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) before += __shfl_xor_sync(MG_FULL, before, o);
  __syncwarp();
  return before;
}

// Cursor4 that also classifies each candidate against its column's
// thresholds: m bit 0 = B-only cell (not A's), bit 1 = A-only cell (not B's).
struct Cursor4P {
  int sbase;
  __device__ __forceinline__ void next(const PairSmem& ps, int w0, int base, unsigned upto, int lane, int (&v)[4],
                                       int (&e)[4], int (&m)[4]) {
    const int wi = (base - w0) >> 5;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t M = ps.bits[wi + i];
      v[i] = base + 32 * i + lane;
      const int4 d = ps.dt[sbase + __popc(M & upto) - 1];  // one LDS.128: delta + both thresholds
      e[i] = v[i] + d.x;
      m[i] = (v[i] >= d.z ? 1 : 0) | (v[i] < d.y ? 2 : 0);
      sbase += __popc(M);
    }
  }
};

// Gaussian-packed accumulators of a pair item: every f32x2 register holds
// (Gaussian A, Gaussian B), and each candidate point enters as broadcast
// scalars straight from its loaded record (no re-pairing moves), with its own
// upstream per half (the edge masks).  d is formed as mu - x (the broadcast
// operand must be the second source), so D1 is negated in totals().
struct GaussPairAcc {
  f2 mx, my, mz, P[6];  // P: P'00, P'11, P'22, 2P'01, 2P'02, 2P'12
  f2 S, T[3], A6[6];

  // The 9 parameter pairs are staged through shared memory (18 floats, pair
  // interleaved) and read back as 64-bit loads, so they live in aligned
  // register pairs: built with register moves, ptxas re-pairs them before
  // every FFMA2 in the loop.
  __device__ __forceinline__ void load(const GaussSoA& grec, int ja, int jb, float* stage, int lane) {
    if (lane < 2) {
      const int j = lane ? jb : ja;
      const float4 A = grec.A[j], B = grec.B[j];
      const float2 C = grec.C[j];
      stage[0 + lane] = A.x;
      stage[2 + lane] = A.y;
      stage[4 + lane] = A.z;
      stage[6 + lane] = B.x;
      stage[8 + lane] = B.y;
      stage[10 + lane] = B.z;
      stage[12 + lane] = 2.f * B.w;  // doubling is exact
      stage[14 + lane] = 2.f * C.x;
      stage[16 + lane] = 2.f * C.y;
    }
    __syncwarp();
    const unsigned long long* st2 = reinterpret_cast<const unsigned long long*>(stage);
    mx.v = st2[0];
    my.v = st2[1];
    mz.v = st2[2];
#pragma unroll
    for (int c = 0; c < 6; ++c) P[c].v = st2[3 + c];
    __syncwarp();
    S = bc2(0.f);
#pragma unroll
    for (int c = 0; c < 3; ++c) T[c] = bc2(0.f);
#pragma unroll
    for (int c = 0; c < 6; ++c) A6[c] = bc2(0.f);
  }
  // one candidate point p with upstream u = (u seen by A, u seen by B)
  __device__ __forceinline__ void point(const float4& p, f2 u) {
    const f2 dx = sub2(mx, bc2(p.x)), dy = sub2(my, bc2(p.y)), dz = sub2(mz, bc2(p.z));
    f2 t1 = fma2(P[4], dz, fma2(P[3], dy, mul2(P[0], dx)));
    f2 m = mul2(dx, t1);
    m = fma2(dy, fma2(P[5], dz, mul2(P[1], dy)), m);
    m = fma2(dz, mul2(P[2], dz), m);
    const f2 ug = mul2(u, gauss_w2(m));
    S = add2(S, ug);
    const f2 cx = mul2(ug, dx), cy = mul2(ug, dy), cz = mul2(ug, dz);
    T[0] = add2(T[0], cx);
    T[1] = add2(T[1], cy);
    T[2] = add2(T[2], cz);
    A6[0] = fma2(cx, dx, A6[0]);
    A6[1] = fma2(cx, dy, A6[1]);
    A6[2] = fma2(cx, dz, A6[2]);
    A6[3] = fma2(cy, dy, A6[3]);
    A6[4] = fma2(cy, dz, A6[4]);
    A6[5] = fma2(cz, dz, A6[5]);
  }
  __device__ __forceinline__ static float half(f2 v, int k) { return k ? hi(v) : lo(v); }
  // lane-local totals of Gaussian k (0 = A, 1 = B); T = P' D1, D1 = -sum u g (mu - x)
  __device__ __forceinline__ void totals(int k, float* v) const {
    v[0] = half(S, k);
    const float d1x = -half(T[0], k), d1y = -half(T[1], k), d1z = -half(T[2], k);
    const float p00 = half(P[0], k), p11 = half(P[1], k), p22 = half(P[2], k);
    const float h01 = 0.5f * half(P[3], k), h02 = 0.5f * half(P[4], k), h12 = 0.5f * half(P[5], k);
    v[1] = p00 * d1x + h01 * d1y + h02 * d1z;
    v[2] = h01 * d1x + p11 * d1y + h12 * d1z;
    v[3] = h02 * d1x + h12 * d1y + p22 * d1z;
#pragma unroll
    for (int c = 0; c < 6; ++c) v[4 + c] = half(A6[c], k);
  }
};

// Warp reduction of the pair's 10 f32x2 accumulators through the warp's
// (no longer needed) shared memory: every lane stores its 10 packed sums, lane
// c < 10 adds column c over the 32 lanes as 64-bit loads + FADD2 (both
// Gaussians at once, 4 independent chains), T = P' D1 is formed once on
// lanes 1..3.  ~90 instructions where the 20-value shuffle transpose took 165.
__device__ __forceinline__ void bwd_store_pair(const GaussPairAcc& acc, int j, float* __restrict__ acc10,
                                               PairSmem& ps, int lane) {
  static_assert(sizeof(PairSmem) >= 32 * 10 * sizeof(unsigned long long), "pair reduction buffer");
  unsigned long long* red = reinterpret_cast<unsigned long long*>(&ps);
  __syncwarp();  // the window loop's last shared-memory reads are done
  {
    unsigned long long* row = red + lane * 10;
    row[0] = acc.S.v;
    row[1] = acc.T[0].v;
    row[2] = acc.T[1].v;
    row[3] = acc.T[2].v;
#pragma unroll
    for (int c = 0; c < 6; ++c) row[4 + c] = acc.A6[c].v;
  }
  __syncwarp();
  const int c = lane < 10 ? lane : 0;
  f2 s0, s1, s2, s3;
  s0.v = red[0 * 10 + c];
  s1.v = red[1 * 10 + c];
  s2.v = red[2 * 10 + c];
  s3.v = red[3 * 10 + c];
#pragma unroll
  for (int l = 4; l < 32; l += 4) {
    f2 a, b, d, e;
    a.v = red[(l + 0) * 10 + c];
    b.v = red[(l + 1) * 10 + c];
    d.v = red[(l + 2) * 10 + c];
    e.v = red[(l + 3) * 10 + c];
    s0 = add2(s0, a);
    s1 = add2(s1, b);
    s2 = add2(s2, d);
    s3 = add2(s3, e);
  }
  f2 v = add2(add2(s0, s1), add2(s2, s3));
  // D1 = -sum u g (mu - x) on lanes 1..3 -> T = P' D1 (rows of the symmetric P')
  const float lo1 = __shfl_sync(MG_FULL, lo(v), 1), hi1 = __shfl_sync(MG_FULL, hi(v), 1);
  const float lo2 = __shfl_sync(MG_FULL, lo(v), 2), hi2 = __shfl_sync(MG_FULL, hi(v), 2);
  const float lo3 = __shfl_sync(MG_FULL, lo(v), 3), hi3 = __shfl_sync(MG_FULL, hi(v), 3);
  if (lane >= 1 && lane <= 3) {
    const f2 d1x = mk2(-lo1, -hi1), d1y = mk2(-lo2, -hi2), d1z = mk2(-lo3, -hi3);
    const f2 half = bc2(0.5f);
    const f2 h01 = mul2(half, acc.P[3]), h02 = mul2(half, acc.P[4]), h12 = mul2(half, acc.P[5]);
    // row (lane - 1) of P' = [[p00, h01, h02], [h01, p11, h12], [h02, h12, p22]]
    const f2 ra = lane == 1 ? acc.P[0] : (lane == 2 ? h01 : h02);
    const f2 rb = lane == 1 ? h01 : (lane == 2 ? acc.P[1] : h12);
    const f2 rc = lane == 1 ? h02 : (lane == 2 ? h12 : acc.P[2]);
    v = fma2(rc, d1z, fma2(rb, d1y, mul2(ra, d1x)));
  }
  if (lane < 10) {
    acc10[(int64_t)j * 10 + lane] = lo(v);
    acc10[(int64_t)(j + 1) * 10 + lane] = hi(v);
  }
}

__device__ __forceinline__ void pair_masked(GaussPairAcc& acc, const float4& a, const float4& b, int ma, int mb) {
  acc.point(a, mk2((ma & 1) ? 0.f : a.w, (ma & 2) ? 0.f : a.w));
  acc.point(b, mk2((mb & 1) ? 0.f : b.w, (mb & 2) ? 0.f : b.w));
}

// Points a, b (elements ea, eb) into both Gaussians of a pair item.
__device__ __forceinline__ void pair_masked(GaussAcc<2>& acc, const float4& a, const float4& b, int ma, int mb) {
  const f2 px = mk2(a.x, b.x), py = mk2(a.y, b.y), pz = mk2(a.z, b.z);
  const f2 uA = mk2((ma & 1) ? 0.f : a.w, (mb & 1) ? 0.f : b.w);
  const f2 uB = mk2((ma & 2) ? 0.f : a.w, (mb & 2) ? 0.f : b.w);
  acc.accum(0, px, py, pz, uA);
  acc.accum(1, px, py, pz, uB);
}

__device__ __forceinline__ void bwd_pair_item(const GaussSoA grec, int j, int cell_a, int cell_b, int g, int r,
                                              const float4* __restrict__ prec, const int* __restrict__ pstart,
                                              float* __restrict__ acc10, PairSmem& ps, int lane, bool cull) {
  // window first: the out-of-line cull call then has few live registers
  Window w = make_window(cell_a, g, r);
  const int ka = cell_a % g, kb = ka + (cell_b - cell_a);
  w.khi = min(kb + r, g - 1);
  if (MG_BWD_CULL && cull && (may_cull(grec.E[j], g, r) || may_cull(grec.E[j + 1], g, r)))
    w = cull_pair_window(w, grec, j, g, lane);
#if MG_BWD_PAIR_GPACK
  GaussPairAcc acc;
  acc.load(grec, j, j + 1, &ps.stage[0], lane);
#else
  GaussAcc<2> acc;
  acc.load(grec, 0, j);
  acc.load(grec, 1, j + 1);
#endif
  const PairCols cols{pstart, max(kb - r, 0), min(ka + r, g - 1) + 1};
  const unsigned upto = 0xffffffffu >> (31 - lane);
  for (int c0 = 0; c0 < w.ncol; c0 += 128) {
#if MG_PAIR_INLINE
    // r <= 5 windows have <= 121 columns: one table (c0 == 0) per item
    const LaneSegs L = w.ncol <= 128 ? build_lane_segs_pair_inl(w.ilo, w.jlo, w.nj, w.ncol, w.inv_nj, w.klo,
                                                                w.khi + 1, cols.kae, cols.kbs, g, pstart, ps, lane)
                                     : build_lane_segs_pair(w, c0, g, cols, ps, lane);
#else
    const LaneSegs L = build_lane_segs_pair(w, c0, g, cols, ps, lane);
#endif
    const int tot = L.tot;
    for (int w0 = 0; w0 < tot; w0 += 32 * kBmWords) {
#if MG_PAIR_INLINE
      Cursor4P cur{build_window_inl(L, w0, ps.bits, lane)};
#else
      Cursor4P cur{build_window(L, w0, reinterpret_cast<SegSmem&>(ps), lane)};
#endif
      const int wend = min(tot, w0 + 32 * kBmWords);
      const int nfull = (wend - w0) >> 7;
      int v[4], e[4], m[4];
      for (int it = 0; it < nfull; ++it) {
        cur.next(ps, w0, w0 + 128 * it, upto, lane, v, e, m);
        float4 q[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) q[i] = __ldg(prec + e[i]);
        pair_masked(acc, q[0], q[1], m[0], m[1]);
        pair_masked(acc, q[2], q[3], m[2], m[3]);
      }
      const int tb = w0 + (nfull << 7);
      if (tb < wend) {  // ragged tail window: missing points are zero records
        cur.next(ps, w0, tb, upto, lane, v, e, m);
        float4 q[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) q[i] = v[i] < wend ? __ldg(prec + e[i]) : make_float4(0.f, 0.f, 0.f, 0.f);
        if (v[0] < wend) pair_masked(acc, q[0], q[1], m[0], m[1]);
        if (v[2] < wend) pair_masked(acc, q[2], q[3], m[2], m[3]);
      }
      __syncwarp();
    }
  }
#if MG_BWD_PAIR_GPACK && MG_BWD_SMEM_STORE
  bwd_store_pair(acc, j, acc10, ps, lane);
#else
  bwd_store<2>(acc, j, 2, acc10, lane);
#endif
}

#ifndef MG_BWD_PAIR_DMAX
// pair Gaussians up to this many k-cells apart in one column: the union
// window grows by dk cells, still cheaper than two windows.  Training drift
// empties about half the lattice cells within ~200 steps at C4; with dk <= 1
// the backward then slowed 2.13 -> 3.30 ms, with dk <= 4 only to 2.28 ms
// (dk <= 6 and <= 10 measured the same)
#define MG_BWD_PAIR_DMAX 4
#endif
#ifndef MG_BWD_PAIR_MINB
#define MG_BWD_PAIR_MINB 1  // 16 warps x 1 CTA: two Gaussians' accumulators need ~122 registers
#endif
template <bool PAIR>
__global__ void __launch_bounds__(kBwdWarps * 32, PAIR ? MG_BWD_PAIR_MINB : MG_BWD_MINB) backward_kernel(const GaussSoA grec,
                                                                  const uint32_t* __restrict__ gkey,
                                                                  const int* __restrict__ gstart, int g, int r,
                                                                  const float4* __restrict__ prec,
                                                                  const int* __restrict__ pstart,
                                                                  const int4* __restrict__ items,
                                                                  const int* __restrict__ nitems_dev,
                                                                  int n_implicit, float* __restrict__ acc10,
                                                                  int cull) {
  // per warp: SegSmem for single items, PairSmem for pairs (aliased); dynamic,
  // so more than 16 warps fit (static shared memory stops at 48 KB)
  extern __shared__ __align__(16) unsigned char bwd_dyn[];
  WarpSmem* s_ws = reinterpret_cast<WarpSmem*>(bwd_dyn);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;  // kBwdWarps, or 8 for small launches
  // implicit pair items: sorted Gaussians (2j, 2j+1)
  if (PAIR && items == nullptr) {
    const int npairs = (n_implicit + 1) >> 1;
    // strided: CTA-contiguous pair ranges (as the forward uses) were much
    // slower, because a pair's cost follows the local point density; loading
    // the next pair's keys ahead measured 2% slower (registers)
    for (int it = blockIdx.x * nw + warp; it < npairs; it += gridDim.x * nw) {
      const int j = 2 * it;
      const int ca = (int)gkey[j];
      const int cb = j + 1 < n_implicit ? (int)gkey[j + 1] : -1;
      const int dk = cb - ca;  // cells of one column, dk apart (sorted, so dk >= 0 when cb >= 0)
      if (cb >= 0 && dk <= MG_BWD_PAIR_DMAX && ca % g + dk <= g - 1) {
        bwd_pair_item(grec, j, ca, cb, g, r, prec, pstart, acc10, s_ws[warp].pair, lane, cull != 0);
      } else {
        bwd_item<1>(grec, j, 1, ca, g, r, prec, pstart, acc10, s_ws[warp].seg, lane, cull != 0);
        if (cb >= 0) bwd_item<1>(grec, j + 1, 1, cb, g, r, prec, pstart, acc10, s_ws[warp].seg, lane, cull != 0);
      }
    }
    return;
  }
  // item {Gaussian, cell, -1, 0} (staged-path overflow list); items ==
  // nullptr: one item per sorted Gaussian, in cell order, so concurrently
  // running warps share their candidate point windows
  const int nitems = items ? *nitems_dev : n_implicit;
  auto load_item = [&](int j) {
    return items ? items[j] : make_int4(j, (int)gkey[j], -1, 0);
  };
  const int stride = gridDim.x * nw;
  int it = blockIdx.x * nw + warp;
  int4 next = (MG_BWD_IPF && it < nitems) ? load_item(it) : make_int4(0, 0, 0, 0);
  for (; it < nitems; it += stride) {
    const int4 item = MG_BWD_IPF ? next : load_item(it);  // {first, cell, count, 0}
    if (MG_BWD_IPF && it + stride < nitems) next = load_item(it + stride);  // loads under this item
    bwd_item<1>(grec, item.x, 1, item.y, g, r, prec, pstart, acc10, s_ws[warp].seg, lane, cull != 0);
  }
}

// ---------------------------------------------------------------------------
// Staged backward.  A block owns a STRIP of kSbS consecutive Gaussian cells
// (i, j, k0 .. k0+kSbS-1), one warp per cell.  The union of the strip's
// candidate sub-points -- (2r+1)^2 columns x (kSbS + 2r) cells, each column a
// contiguous range of the cell-sorted point records -- is copied into shared
// memory with TMA bulk copies (cp.async.bulk + mbarrier), in rounds of
// "pieces" (column sub-ranges) that fit the buffer.  Every warp then streams
// its own 11x11x11 neighbourhood out of shared memory with the bitmap
// cursor: each staged point is read ~kSbS*11/(kSbS+10) times from SMEM
// instead of once per Gaussian from L2.  Cells with more than 2 Gaussians
// hand their later chunks to the global-memory item kernel (overflow list).
// ---------------------------------------------------------------------------
#ifndef MG_SB_S
#define MG_SB_S 16
#endif
#ifndef MG_SB_CAP
#define MG_SB_CAP 8192
#endif
constexpr int kSbS = MG_SB_S;      // cells per strip == warps per block
constexpr int kSbCap = MG_SB_CAP;  // staged point records (16 B each)
constexpr int kSbPieces = 128;

struct StageSmem {
  uint64_t bar;
  int phase;
  // round builder state (thread 0)
  int bc, bstart, brem, done;
  // current round
  int npieces;
  int pc[kSbPieces];   // column index of piece
  int pga[kSbPieces];  // global start (point index) of piece
  int plen[kSbPieces];
  int pso[kSbPieces];  // smem offset of piece
  // strip columns
  int ncol, ks_lo, ks_hi, ilo, jlo, nj;
  int cst[kSbPieces], clen[kSbPieces];
  float part[kSbS][32];  // per-warp partial sums: Gaussian k value c at [16k + c]
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, int parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Greedy: next round of pieces (thread 0).  Returns bytes to stage.
__device__ int next_round(StageSmem& st) {
  int used = 0, np = 0;
  while (st.bc < st.ncol && np < kSbPieces) {
    if (st.brem == 0) {
      ++st.bc;
      if (st.bc < st.ncol) {
        st.bstart = st.cst[st.bc];
        st.brem = st.clen[st.bc];
      }
      continue;
    }
    const int take = min(st.brem, kSbCap - used);
    if (take == 0) break;
    st.pc[np] = st.bc;
    st.pga[np] = st.bstart;
    st.plen[np] = take;
    st.pso[np] = used;
    ++np;
    used += take;
    st.bstart += take;
    st.brem -= take;
  }
  st.npieces = np;
  st.done = (st.bc >= st.ncol) ? 1 : 0;
  return used * 16;
}

template <int QG>
__device__ __forceinline__ void staged_load_gauss(GaussAcc<QG>& acc, const GaussSoA& grec, int g0, int ng) {
#pragma unroll
  for (int k = 0; k < QG; ++k) {
    const int gi = g0 + min(k, ng - 1);
    const float4 A = grec.A[gi], B = grec.B[gi];
    const float2 C = grec.C[gi];
    acc.mx[k] = A.x;
    acc.my[k] = A.y;
    acc.mz[k] = A.z;
    acc.P[k][0] = B.x;
    acc.P[k][1] = B.y;
    acc.P[k][2] = B.z;
    acc.P[k][3] = 2.f * B.w;
    acc.P[k][4] = 2.f * C.x;
    acc.P[k][5] = 2.f * C.y;
    acc.S[k] = bc2(0.f);
#pragma unroll
    for (int c = 0; c < 3; ++c) acc.T[k][c] = bc2(0.f);
#pragma unroll
    for (int c = 0; c < 6; ++c) acc.A6[k][c] = bc2(0.f);
  }
}

template <int QG>
__device__ __forceinline__ void staged_round(const GaussSoA& grec, int g0, float* __restrict__ part,
                                             const float4* __restrict__ stage, const StageSmem& st,
                                             const int* __restrict__ pstart, int g, int r, int kw, SegSmem& sm,
                                             int lane) {
  GaussAcc<QG> acc;
  staged_load_gauss<QG>(acc, grec, g0, QG);
  // this warp's sub-range [a, b) of every piece, as segments into `stage`
  const int kl = max(kw - r, st.ks_lo), kh = min(kw + r, st.ks_hi);
  int stt[4], ln[4], sum = 0, ne = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int p = lane * 4 + k;
    stt[k] = 0;
    ln[k] = 0;
    if (p < st.npieces) {
      const int c = st.pc[p];
      const int q = (int)(((float)c + 0.5f) / (float)st.nj);
      const int ii = st.ilo + q, jj = st.jlo + (c - q * st.nj);
      const int base = (ii * g + jj) * g;
      const int a = max(__ldg(pstart + base + kl), st.pga[p]);
      const int b = min(__ldg(pstart + base + kh + 1), st.pga[p] + st.plen[p]);
      if (b > a) {
        stt[k] = st.pso[p] + (a - st.pga[p]);
        ln[k] = b - a;
      }
    }
    sum += ln[k];
    ne += ln[k] > 0;
  }
  int tot, netot;
  int off = warp_excl_scan(sum, lane, &tot);
  int e = warp_excl_scan(ne, lane, &netot);
  LaneSegs L;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    L.pre[k] = off;
    L.len[k] = ln[k];
    L.st[k] = stt[k];
    if (ln[k] > 0) sm.delta[e++] = stt[k] - off;
    off += ln[k];
  }
  L.tot = tot;
  const unsigned upto = 0xffffffffu >> (31 - lane);
  for (int w0 = 0; w0 < tot; w0 += 32 * kBmWords) {
    Cursor4 cur{build_window(L, w0, sm, lane)};
    const int wend = min(tot, w0 + 32 * kBmWords);
    for (int base = w0; base < wend; base += 128) {
      int v[4], ei[4];
      cur.next(sm, w0, base, upto, lane, v, ei);
      float4 pt[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) pt[i] = v[i] < wend ? stage[ei[i]] : make_float4(0.f, 0.f, 0.f, 0.f);
      if (v[0] < wend) acc.pair(pt[0], pt[1]);
      if (v[2] < wend) acc.pair(pt[2], pt[3]);
    }
    __syncwarp();
  }
  // lane-reduce this round's sums and add them to the warp's smem partials
  constexpr int NV = QG == 1 ? 16 : 32;
  float vals[32];
#pragma unroll
  for (int k = 0; k < QG; ++k) {
    acc.totals(k, vals + 16 * k);
#pragma unroll
    for (int c = 10; c < 16; ++c) vals[16 * k + c] = 0.f;
  }
#pragma unroll
  for (int i = 16 * QG; i < 32; ++i) vals[i] = 0.f;
  const float red = transpose_reduce<NV>(vals, lane);
  constexpr int SH = RedShift<NV>::value;
  const int idx = lane >> SH;
  if ((lane & ((1 << SH) - 1)) == 0 && (idx & 15) < 10) part[idx] += red;
  __syncwarp();
}

__global__ void __launch_bounds__(kSbS * 32, (16 / kSbS) > 0 ? (16 / kSbS) : 1) backward_staged_kernel(
    const GaussSoA grec, const int* __restrict__ gstart, int g, int r, const float4* __restrict__ prec,
    const int* __restrict__ pstart, const int* __restrict__ strips, const int* __restrict__ nstrips_dev,
    float* __restrict__ acc10) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float4* stage = reinterpret_cast<float4*>(smem_raw);
  SegSmem* segs = reinterpret_cast<SegSmem*>(smem_raw + sizeof(float4) * kSbCap);
  StageSmem& st = *reinterpret_cast<StageSmem*>(smem_raw + sizeof(float4) * kSbCap + sizeof(SegSmem) * kSbS);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&st.bar, 1);
    st.phase = 0;
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const int nstrips = *nstrips_dev;
  const int nkb = (g + kSbS - 1) / kSbS;
  for (int si = blockIdx.x; si < nstrips; si += gridDim.x) {
    const int sk = strips[si];
    const int kb = sk % nkb, col = sk / nkb;
    const int j = col % g, i = col / g;
    const int k0 = kb * kSbS;
    const int kc = min(kSbS, g - k0);
    // strip geometry + per-column window ranges
    if (threadIdx.x == 0) {
      st.ilo = max(i - r, 0);
      st.jlo = max(j - r, 0);
      st.nj = min(j + r, g - 1) - st.jlo + 1;
      st.ncol = (min(i + r, g - 1) - st.ilo + 1) * st.nj;
      st.ks_lo = max(k0 - r, 0);
      st.ks_hi = min(k0 + kc - 1 + r, g - 1);
    }
    __syncthreads();
    for (int c = threadIdx.x; c < st.ncol; c += blockDim.x) {
      const int q = (int)(((float)c + 0.5f) / (float)st.nj);
      const int ii = st.ilo + q, jj = st.jlo + (c - q * st.nj);
      const int base = (ii * g + jj) * g;
      const int a = __ldg(pstart + base + st.ks_lo), b = __ldg(pstart + base + st.ks_hi + 1);
      st.cst[c] = a;
      st.clen[c] = b - a;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      st.bc = 0;
      st.bstart = st.cst[0];
      st.brem = st.clen[0];
      st.done = 0;
    }
    // this warp's cell and its first <= 2 Gaussians (later chunks -> overflow kernel)
    const int kw = k0 + warp;
    const int cell = (i * g + j) * g + kw;
    const int g0 = warp < kc ? __ldg(gstart + cell) : 0;
    const int ngc = warp < kc ? __ldg(gstart + cell + 1) - g0 : 0;
    const int ng = min(ngc, 2);
    float* part = st.part[warp];
    part[lane] = 0.f;
    __syncthreads();
    while (true) {
      if (threadIdx.x == 0) {
        const int bytes = next_round(st);
        fence_proxy_async();
        mbar_arrive_expect(&st.bar, (uint32_t)bytes);
      }
      __syncthreads();
      if (warp == 0) {
        for (int p = lane; p < st.npieces; p += 32)
          bulk_g2s(stage + st.pso[p], prec + st.pga[p], (uint32_t)st.plen[p] * 16u, &st.bar);
      }
      mbar_wait(&st.bar, st.phase);
      if (ng == 2) staged_round<2>(grec, g0, part, stage, st, pstart, g, r, kw, segs[warp], lane);
      if (ng == 1) staged_round<1>(grec, g0, part, stage, st, pstart, g, r, kw, segs[warp], lane);
      const int done = st.done;
      __syncthreads();
      if (threadIdx.x == 0) st.phase ^= 1;
      __syncthreads();
      if (done) break;
    }
    if (lane < 10 * ng) acc10[(int64_t)(g0 + lane / 10) * 10 + lane % 10] = part[(lane / 10) * 16 + lane % 10];
  }
}

// strip flags: strip (i, j, kb) is live if its cells hold at least one Gaussian
__global__ void strip_flags_kernel(const int* __restrict__ starts, int g, int s, int* __restrict__ flags) {
  const int nkb = (g + s - 1) / s;
  const int64_t nstrips = (int64_t)g * g * nkb;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nstrips; t += (int64_t)gridDim.x * blockDim.x) {
    const int kb = (int)(t % nkb);
    const int64_t col = t / nkb;
    const int k0 = kb * s, k1 = min(k0 + s, g);
    flags[t] = starts[col * g + k1] > starts[col * g + k0] ? 1 : 0;
  }
}

__global__ void strip_compact_kernel(const int* __restrict__ flags, const int* __restrict__ scan, int64_t n,
                                     int* __restrict__ out, int* __restrict__ count) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    if (flags[t]) out[scan[t]] = (int)t;
    if (t == n - 1) *count = scan[t] + flags[t];
  }
}

// overflow items: chunk starts p (step 2) of cells with > 2 Gaussians, past the first chunk
__global__ void overflow_flags_kernel(const uint32_t* __restrict__ keys, const int* __restrict__ starts, int64_t n,
                                      int* __restrict__ flags) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int d = (int)(p - starts[keys[p]]);
    flags[p] = d >= 2 ? 1 : 0;
  }
}

// ---------------------------------------------------------------------------
// Host launchers
// ---------------------------------------------------------------------------
static int g_num_sms = 0;
int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

static inline unsigned grid_for(int64_t n, int threads = 256) {
  int64_t b = (n + threads - 1) / threads;
  int64_t cap = (int64_t)num_sms() * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (unsigned)b;
}

void launch_gauss_keys(const float* pos, int64_t n, int g, uint32_t* keys, cudaStream_t st) {
  if (n > 0) MG_LAUNCH(gauss_keys_kernel<<<grid_for(n), 256, 0, st>>>(pos, n, g, keys));
}
void launch_gauss_keys_f64(const double* pos, int64_t n, int g, uint32_t* keys, cudaStream_t st) {
  if (n > 0) MG_LAUNCH(gauss_keys_f64_kernel<<<grid_for(n), 256, 0, st>>>(pos, n, g, keys));
}
void launch_gauss_activate(const float* pos, const float* quat, const float* ls, const float* lg, const int* order,
                           int64_t n, float* grec, int* err, cudaStream_t st) {
  if (n > 0) MG_LAUNCH(gauss_activate_kernel<<<grid_for(n), 256, 0, st>>>(pos, quat, ls, lg, order, n, gauss_out(grec, n), err));
}
void launch_gauss_pack_prepared(const double* mu, const double* prec6, const double* alpha, const int* order,
                                int64_t n, float* grec, cudaStream_t st) {
  if (n > 0) MG_LAUNCH(gauss_pack_prepared_kernel<<<grid_for(n), 256, 0, st>>>(mu, prec6, alpha, order, n, gauss_out(grec, n)));
}
void launch_points_prepare(const double* coords, const int64_t* sids64, const int* sids32, int64_t b, int ntaps,
                           const double* tap_off, const double* dirs, const double* rot, const double* trans,
                           int nslices, int g, uint32_t* keys, float4* xf, double* xout, cudaStream_t st) {
  if (b * ntaps > 0)
    MG_LAUNCH(points_prepare_kernel<<<grid_for(b * ntaps), 256, 0, st>>>(coords, sids64, sids32, b, ntaps, tap_off, dirs, rot,
                                                               trans, nslices, g, keys, xf, xout));
}
void launch_points_gather(const float4* xf, const int* perm, int64_t n, float4* prec, int* inv, cudaStream_t st) {
  if (n > 0) MG_LAUNCH(points_gather_kernel<<<grid_for(n), 256, 0, st>>>(xf, perm, n, prec, inv));
}

int fwd_qmax() { return MG_FWD_QMAX; }
int fwd_dense_min() { return kFwdDenseMin; }

size_t items_workspace_bytes(int64_t n) { return 2 * (((size_t)n * 4 + 255) & ~(size_t)255) + scan_workspace_bytes(n); }

// One pass over cells: each occupied cell appends its ceil(count / q) item
// records with one warp-aggregated atomic per warp.  Item ORDER only affects
// scheduling (every item's arithmetic is self-contained), and cells are
// visited in index order, so neighbouring warps get neighbouring cells (a
// 2 x 2 x 8-cell tiled visiting order measured the same).
__global__ void cell_items_kernel(const int* __restrict__ starts, int g, int q, int dense_min,
                                  int4* __restrict__ items, int* __restrict__ nitems) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t nvisit = (int64_t)g * g * g;
  for (int64_t t0 = (int64_t)blockIdx.x * blockDim.x; t0 < nvisit; t0 += stride) {
    const int64_t t = t0 + threadIdx.x;
    const int64_t c = t < nvisit ? t : -1;
    int s = 0, e = 0;
    if (c >= 0) {
      s = starts[c];
      e = starts[c + 1];
    }
    const int cnt = e - s;
    const int qq = (dense_min > 0 && cnt >= dense_min) ? 64 : q;
    const int m = (cnt + qq - 1) / qq;
    int tot;
    const int off = warp_excl_scan(m, lane, &tot);
    int base = 0;
    if (lane == 0 && tot > 0) base = atomicAdd(nitems, tot);
    base = __shfl_sync(0xffffffffu, base, 0) + off;
    for (int i = 0; i < m; ++i) {
      const int p = s + i * qq;
      items[base + i] = make_int4(p, (int)c, min(qq, e - p), 0);
    }
  }
}

void build_items_cells(const int* starts, int g, int q, int4* items, int* nitems, cudaStream_t st, int dense_min) {
  cudaMemsetAsync(nitems, 0, sizeof(int), st);
  if (g <= 0) return;
  const int64_t ncell = (int64_t)g * g * g;
  int64_t blocks = (ncell + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  MG_LAUNCH(cell_items_kernel<<<(unsigned)blocks, 256, 0, st>>>(starts, g, q, dense_min, items, nitems));
}

void build_items(const uint32_t* keys, const int* starts, int64_t n, int q, int4* items, int* nitems, void* ws,
                 cudaStream_t st, int dense_min) {
  if (n <= 0) {
    cudaMemsetAsync(nitems, 0, sizeof(int), st);
    return;
  }
  int* flags = (int*)ws;
  int* scan = (int*)((char*)ws + (((size_t)n * 4 + 255) & ~(size_t)255));
  void* sws = (char*)ws + 2 * (((size_t)n * 4 + 255) & ~(size_t)255);
  MG_LAUNCH(item_flags_kernel<<<grid_for(n), 256, 0, st>>>(keys, starts, n, q, dense_min, flags));
  excl_scan(flags, scan, n, sws, st);
  MG_LAUNCH(item_compact_kernel<<<grid_for(n), 256, 0, st>>>(flags, scan, keys, starts, n, q, dense_min, items,
                                                             nitems));
}

// Warps per CTA for a persistent pair-kernel launch: the full one-CTA-per-SM
// shape when every SM gets >= 8 items per warp, else 8-warp CTAs (several
// per SM), so small launches (early reconstruction levels) still cover all SMs.
static int block_warps(int full, int64_t items) {
  return items >= (int64_t)num_sms() * full * 8 ? full : 8;
}

template <class K>
static int64_t persistent_blocks(K kernel, int threads, int64_t max_blocks, size_t dyn_smem = 0) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, dyn_smem);
  if (per_sm < 1) per_sm = 1;
  int64_t b = (int64_t)num_sms() * per_sm;
  return b < max_blocks ? b : (max_blocks < 1 ? 1 : max_blocks);
}

void launch_forward(bool with_h, const float* grec_raw, int64_t n_gauss, const int* gstart, int g, int r,
                    const float4* prec,
                    const uint32_t* pkey, const int* pstart, const int4* items, const int* nitems, int64_t max_items,
                    float4* out4, int* cnt, cudaStream_t st) {
  if (max_items <= 0) return;
  const int nw = block_warps(kFwdWarps, max_items / 2);  // ~2+ sub-points per item
  const int64_t want = (max_items + nw - 1) / nw;
  const GaussSoA grec = gauss_soa(grec_raw, n_gauss);
  auto k = with_h ? forward_kernel<true> : forward_kernel<false>;
  const unsigned blocks = (unsigned)persistent_blocks(k, nw * 32, want);
  constexpr size_t smem = 0;
  MG_LAUNCH(k<<<blocks, nw * 32, smem, st>>>(grec, gstart, g, r, prec, pkey, pstart, items, nitems, out4, cnt));
}

static size_t bwd_smem_bytes(int nw) {
  const size_t b = sizeof(WarpSmem) * (size_t)nw;
  static bool done = false;  // opt in above 48 KB once per process
  if (!done) {
    cudaFuncSetAttribute(backward_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(WarpSmem) * kBwdWarps));
    cudaFuncSetAttribute(backward_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(WarpSmem) * kBwdWarps));
    done = true;
  }
  return b;
}

size_t staged_smem_bytes() { return sizeof(float4) * kSbCap + sizeof(SegSmem) * kSbS + sizeof(StageSmem); }

size_t backward_staged_ws_bytes(int64_t n, int g) {
  const int64_t nstrips = (int64_t)g * g * ((g + kSbS - 1) / kSbS);
  const int64_t m = nstrips > n ? nstrips : n;
  const size_t a4 = (((size_t)m * 4) + 255) & ~(size_t)255, a16 = (((size_t)m * 16) + 255) & ~(size_t)255;
  const size_t sw = (scan_workspace_bytes(m) + 255) & ~(size_t)255;
  return 3 * a4 + 512 + sw + a16;
}

// Staged backward: strips for the first <= 2 Gaussians of every cell, the
// global-memory item kernel for the rest (rare at lattice densities).
void launch_backward_staged(const float* grec_raw, int64_t n_gauss, const uint32_t* gkey, const int* gstart, int g,
                            int r, const float4* prec, const int* pstart, float* acc10, void* ws, cudaStream_t st) {
  if (n_gauss <= 0) return;
  const int nkb = (g + kSbS - 1) / kSbS;
  const int64_t nstrips = (int64_t)g * g * nkb;
  const int64_t m = nstrips > n_gauss ? nstrips : n_gauss;
  const size_t al = (((size_t)m * 4) + 255) & ~(size_t)255;
  char* w = (char*)ws;
  int* flags = (int*)w;
  int* scan = (int*)(w + al);
  int* list = (int*)(w + 2 * al);
  int* counts = (int*)(w + 3 * al);
  void* sws = w + 3 * al + 512;
  int4* oitems = (int4*)(w + 3 * al + 512 + ((scan_workspace_bytes(m) + 255) & ~(size_t)255));
  MG_LAUNCH(strip_flags_kernel<<<grid_for(nstrips), 256, 0, st>>>(gstart, g, kSbS, flags));
  excl_scan(flags, scan, nstrips, sws, st);
  MG_LAUNCH(strip_compact_kernel<<<grid_for(nstrips), 256, 0, st>>>(flags, scan, nstrips, list, counts));
  const GaussSoA grec = gauss_soa(grec_raw, n_gauss);
  static bool attr = false;
  const size_t smem = staged_smem_bytes();
  if (!attr) {
    cudaFuncSetAttribute(backward_staged_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, backward_staged_kernel, kSbS * 32, smem);
  int64_t blocks = (int64_t)num_sms() * (per_sm > 0 ? per_sm : 1);
  if (blocks > nstrips) blocks = nstrips;
  MG_LAUNCH(backward_staged_kernel<<<(unsigned)blocks, kSbS * 32, smem, st>>>(grec, gstart, g, r, prec, pstart, list,
                                                                             counts, acc10));
  // overflow chunks (cells with > 2 Gaussians) through the item kernel
  int* oflags = flags;
  int* oscan = scan;
  MG_LAUNCH(overflow_flags_kernel<<<grid_for(n_gauss), 256, 0, st>>>(gkey, gstart, n_gauss, oflags));
  excl_scan(oflags, oscan, n_gauss, sws, st);
  MG_LAUNCH(item_compact_kernel<<<grid_for(n_gauss), 256, 0, st>>>(oflags, oscan, gkey, gstart, n_gauss, 1, 0,
                                                                    oitems, counts + 1, 1));
  const int64_t want = (n_gauss / 2 + kBwdWarps) / kBwdWarps;
  const size_t dsm = bwd_smem_bytes(kBwdWarps);
  MG_LAUNCH(backward_kernel<false><<<(unsigned)persistent_blocks(backward_kernel<false>, kBwdWarps * 32, want, dsm),
                                     kBwdWarps * 32, dsm, st>>>(grec, gkey, gstart, g, r, prec, pstart, oitems,
                                                                counts + 1, 0, acc10, bwd_cull_enabled()));
}

void launch_backward(const float* grec_raw, int64_t n_gauss, const uint32_t* gkey, const int* gstart, int g, int r,
                     const float4* prec, const int* pstart, const int4* items, const int* nitems, int64_t max_items,
                     float* acc10, cudaStream_t st, int pair_mode) {
  if (max_items <= 0) return;
  const GaussSoA grec = gauss_soa(grec_raw, n_gauss);
  const bool pairs = pair_mode > 0 && items == nullptr;
  const int nw = block_warps(kBwdWarps, pairs ? (max_items + 1) / 2 : max_items);
  const int64_t want = (max_items + nw - 1) / nw;
  auto k = pairs ? backward_kernel<true> : backward_kernel<false>;
  const size_t dsm = bwd_smem_bytes(nw);
  MG_LAUNCH(k<<<(unsigned)persistent_blocks(k, nw * 32, want, dsm), nw * 32, dsm, st>>>(
      grec, gkey, gstart, g, r, prec, pstart, items, nitems, (int)n_gauss, acc10, bwd_cull_enabled()));
}

}  // namespace mg
