// mg_strict.cu -- strict float64 instantiation of the reference pair kernels
// (_kernels.py:24-144), selectable for parity runs (render.set_strict_fp64).
//
// The default pair kernels (mg_render.cu) evaluate in float32 with ex2.approx
// on pre-scaled precisions (rel. error ~1e-6).  These kernels evaluate every
// pair in IEEE float64 with the reference's exact operation order and no FMA
// contraction (__dmul_rn / __dadd_rn), so intensities, d_points and the
// per-Gaussian accumulators agree with the reference to ~1e-15 relative and
// the reference's float64 finite-difference gradient checks
// (tests/test_render.py:177-259) hold on the GPU.
//
// Layout: points are transformed (float64) and binned by cell with the same
// counting sort as the fast path.  Forward and d_points are point-major (one
// thread per cell-sorted point walking its (2r+1)^2 CSR columns in the
// reference order); the per-Gaussian accumulators are Gaussian-major (one
// thread per cell-sorted Gaussian walking the sorted points of its window:
// the candidate relation |cell(x) - cell(mu)|_inf <= r is symmetric), so
// there are no atomics and results are run-to-run bit-reproducible.
#include "mg_render.cuh"
#include "mg_sort.cuh"

namespace mg {
namespace {

constexpr double kCut = 64.0;  // EXP_CUTOFF, _kernels.py:21

__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ds(double a, double b) { return __dsub_rn(a, b); }

// _kernels.py:33-48: x = R_s p + t_s (s >= 0), cell key of x.
__global__ void strict_points_kernel(const double* __restrict__ pts, const int64_t* __restrict__ sids, int64_t b,
                                     const double* __restrict__ rot, const double* __restrict__ trans, int64_t k,
                                     int g, double* __restrict__ xt, uint32_t* __restrict__ keys) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < b; i += (int64_t)gridDim.x * blockDim.x) {
    const double px = pts[3 * i], py = pts[3 * i + 1], pz = pts[3 * i + 2];
    const int64_t s = sids ? sids[i] : -1;
    double x = px, y = py, z = pz;
    if (s >= 0 && s < k) {
      const double* R = rot + 9 * s;
      const double* T = trans + 3 * s;
      x = da(da(da(dm(R[0], px), dm(R[1], py)), dm(R[2], pz)), T[0]);
      y = da(da(da(dm(R[3], px), dm(R[4], py)), dm(R[5], pz)), T[1]);
      z = da(da(da(dm(R[6], px), dm(R[7], py)), dm(R[8], pz)), T[2]);
    }
    xt[3 * i] = x;
    xt[3 * i + 1] = y;
    xt[3 * i + 2] = z;
    keys[i] = (uint32_t)flat_cell(cell_of_d(x, g), cell_of_d(y, g), cell_of_d(z, g), g);
  }
}

// cell key of every CSR position (the Gaussian's own cell), int64 CSR.
__global__ void strict_gkeys_kernel(const int64_t* __restrict__ cs, int64_t ncell, uint32_t* __restrict__ gkey) {
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < ncell; c += (int64_t)gridDim.x * blockDim.x)
    for (int64_t p = cs[c]; p < cs[c + 1]; ++p) gkey[p] = (uint32_t)c;
}

// Point-major pass: forward (_kernels.py:50-70) or d_points (_kernels.py:104-144).
template <bool BACKWARD>
__global__ void strict_point_pass_kernel(const double* __restrict__ xt, const uint32_t* __restrict__ pkey,
                                         const int* __restrict__ porder, int64_t b, const double* __restrict__ mu,
                                         const double* __restrict__ p6, const double* __restrict__ alpha,
                                         const int64_t* __restrict__ cs, const int64_t* __restrict__ ci, int g, int r,
                                         const double* __restrict__ up, double* __restrict__ out_i,
                                         int64_t* __restrict__ out_cnt, double* __restrict__ out_dp) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < b; q += (int64_t)gridDim.x * blockDim.x) {
    const int bi = porder[q];
    const double x = xt[3 * bi], y = xt[3 * bi + 1], z = xt[3 * bi + 2];
    const int key = (int)pkey[q];
    const int ck = key % g, cj = (key / g) % g, cii = key / (g * g);
    const int klo = max(ck - r, 0), khi = min(ck + r, g - 1);
    double acc = 0.0, hx = 0.0, hy = 0.0, hz = 0.0;
    int64_t cnt = 0;
    const double u = BACKWARD ? up[bi] : 0.0;
    for (int ii = max(cii - r, 0); ii <= min(cii + r, g - 1); ++ii) {
      for (int jj = max(cj - r, 0); jj <= min(cj + r, g - 1); ++jj) {
        const int64_t base = ((int64_t)ii * g + jj) * g;
        const int64_t p1 = cs[base + khi + 1];
        for (int64_t p = cs[base + klo]; p < p1; ++p) {
          const int64_t i = ci[p];
          const double dx = ds(x, mu[3 * i]), dy = ds(y, mu[3 * i + 1]), dz = ds(z, mu[3 * i + 2]);
          const double* P = p6 + 6 * i;
          if (!BACKWARD) {
            // P00 dx dx + P11 dy dy + P22 dz dz + 2 (P01 dx dy + P02 dx dz + P12 dy dz)
            double m = da(da(dm(dm(P[0], dx), dx), dm(dm(P[3], dy), dy)), dm(dm(P[5], dz), dz));
            const double off = da(da(dm(dm(P[1], dx), dy), dm(dm(P[2], dx), dz)), dm(dm(P[4], dy), dz));
            m = da(m, dm(2.0, off));
            ++cnt;
            if (m <= kCut) acc = da(acc, dm(alpha[i], exp(dm(-0.5, m))));
          } else {
            const double pdx = da(da(dm(P[0], dx), dm(P[1], dy)), dm(P[2], dz));
            const double pdy = da(da(dm(P[1], dx), dm(P[3], dy)), dm(P[4], dz));
            const double pdz = da(da(dm(P[2], dx), dm(P[4], dy)), dm(P[5], dz));
            const double m = da(da(dm(dx, pdx), dm(dy, pdy)), dm(dz, pdz));
            if (m > kCut) continue;
            const double gv = exp(dm(-0.5, m));
            const double coef = dm(dm(u, alpha[i]), gv);
            hx = ds(hx, dm(coef, pdx));
            hy = ds(hy, dm(coef, pdy));
            hz = ds(hz, dm(coef, pdz));
          }
        }
      }
    }
    if (!BACKWARD) {
      out_i[bi] = acc;
      out_cnt[bi] = cnt;
    } else if (out_dp) {
      out_dp[3 * bi] = hx;
      out_dp[3 * bi + 1] = hy;
      out_dp[3 * bi + 2] = hz;
    }
  }
}

// Gaussian-major accumulators (_kernels.py:124-141), ADDED into d_mu, d_abar6, d_alpha.
__global__ void strict_gauss_pass_kernel(const double* __restrict__ xt, const int* __restrict__ porder,
                                         const int* __restrict__ pstart, const double* __restrict__ up,
                                         const double* __restrict__ mu, const double* __restrict__ p6,
                                         const double* __restrict__ alpha, const int64_t* __restrict__ ci,
                                         const uint32_t* __restrict__ gkey, int64_t n, int g, int r,
                                         double* __restrict__ d_mu, double* __restrict__ d_abar6,
                                         double* __restrict__ d_alpha) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = ci[p];
    const int key = (int)gkey[p];
    const int ck = key % g, cj = (key / g) % g, cii = key / (g * g);
    const int klo = max(ck - r, 0), khi = min(ck + r, g - 1);
    const double mx = mu[3 * i], my = mu[3 * i + 1], mz = mu[3 * i + 2];
    double P[6];
#pragma unroll
    for (int a = 0; a < 6; ++a) P[a] = p6[6 * i + a];
    const double al = alpha[i];
    double sa = 0.0, m0 = 0.0, m1 = 0.0, m2 = 0.0, a6[6] = {0, 0, 0, 0, 0, 0};
    for (int ii = max(cii - r, 0); ii <= min(cii + r, g - 1); ++ii) {
      for (int jj = max(cj - r, 0); jj <= min(cj + r, g - 1); ++jj) {
        const int64_t base = ((int64_t)ii * g + jj) * g;
        const int q1 = pstart[base + khi + 1];
        for (int q = pstart[base + klo]; q < q1; ++q) {
          const int bi = porder[q];
          const double dx = ds(xt[3 * bi], mx), dy = ds(xt[3 * bi + 1], my), dz = ds(xt[3 * bi + 2], mz);
          const double pdx = da(da(dm(P[0], dx), dm(P[1], dy)), dm(P[2], dz));
          const double pdy = da(da(dm(P[1], dx), dm(P[3], dy)), dm(P[4], dz));
          const double pdz = da(da(dm(P[2], dx), dm(P[4], dy)), dm(P[5], dz));
          const double m = da(da(dm(dx, pdx), dm(dy, pdy)), dm(dz, pdz));
          if (m > kCut) continue;
          const double u = up[bi];
          const double gv = exp(dm(-0.5, m));
          sa = da(sa, dm(u, gv));
          const double coef = dm(dm(u, al), gv);
          m0 = da(m0, dm(coef, pdx));
          m1 = da(m1, dm(coef, pdy));
          m2 = da(m2, dm(coef, pdz));
          const double w = dm(-0.5, coef);
          a6[0] = da(a6[0], dm(dm(w, dx), dx));
          a6[1] = da(a6[1], dm(dm(w, dx), dy));
          a6[2] = da(a6[2], dm(dm(w, dx), dz));
          a6[3] = da(a6[3], dm(dm(w, dy), dy));
          a6[4] = da(a6[4], dm(dm(w, dy), dz));
          a6[5] = da(a6[5], dm(dm(w, dz), dz));
        }
      }
    }
    d_alpha[i] = da(d_alpha[i], sa);
    d_mu[3 * i] = da(d_mu[3 * i], m0);
    d_mu[3 * i + 1] = da(d_mu[3 * i + 1], m1);
    d_mu[3 * i + 2] = da(d_mu[3 * i + 2], m2);
#pragma unroll
    for (int a = 0; a < 6; ++a) d_abar6[6 * i + a] = da(d_abar6[6 * i + a], a6[a]);
  }
}

inline size_t al256(size_t b) { return (b + 255) & ~(size_t)255; }

unsigned blocks_for(int64_t n, int threads) {
  int64_t bl = (n + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms() * 32;
  if (bl > cap) bl = cap;
  return (unsigned)(bl < 1 ? 1 : bl);
}

}  // namespace

size_t strict_workspace_bytes(int64_t b, int64_t n, int64_t g) {
  const int64_t ncell = g * g * g;
  return al256((size_t)b * 24) + al256((size_t)b * 4) * 3 + al256((size_t)(ncell + 1) * 4) +
         al256((size_t)n * 4) + counting_workspace_bytes(b, ncell) + 2048;
}

// Returns 0, or 1 when the workspace is too small.
int strict_block(const double* points, const int64_t* sids, int64_t b, const double* rot, const double* trans,
                 int64_t k, const double* mu, const double* prec6, const double* alpha, int64_t n, const int64_t* cs,
                 const int64_t* ci, int g, int r, double* out_i, int64_t* out_cnt, double* out_x,
                 const double* upstream, double* d_mu, double* d_abar6, double* d_alpha, double* out_dp, void* ws,
                 size_t wsb, cudaStream_t st) {
  if (wsb < strict_workspace_bytes(b, n, g)) return 1;
  const int64_t ncell = (int64_t)g * g * g;
  char* p = (char*)ws;
  auto take = [&](size_t bytes) {
    char* q = p;
    p += al256(bytes);
    return (void*)q;
  };
  double* xt = out_x ? out_x : (double*)take((size_t)b * 24);
  if (out_x) take((size_t)b * 24);
  uint32_t* keys = (uint32_t*)take((size_t)b * 4);
  uint32_t* pkey = (uint32_t*)take((size_t)b * 4);
  int* porder = (int*)take((size_t)b * 4);
  int* pstart = (int*)take((size_t)(ncell + 1) * 4);
  uint32_t* gkey = (uint32_t*)take((size_t)n * 4);
  void* rest = p;
  if (b > 0) {
    MG_LAUNCH(strict_points_kernel<<<blocks_for(b, 256), 256, 0, st>>>(points, sids, b, rot, trans, k, g, xt, keys));
  }
  counting_sort_pairs(keys, pkey, porder, pstart, b, ncell, rest, st);
  if (b == 0) return 0;
  if (!upstream) {
    MG_LAUNCH(strict_point_pass_kernel<false><<<blocks_for(b, 128), 128, 0, st>>>(
        xt, pkey, porder, b, mu, prec6, alpha, cs, ci, g, r, nullptr, out_i, out_cnt, nullptr));
    return 0;
  }
  if (out_dp)
    MG_LAUNCH(strict_point_pass_kernel<true><<<blocks_for(b, 128), 128, 0, st>>>(
        xt, pkey, porder, b, mu, prec6, alpha, cs, ci, g, r, upstream, nullptr, nullptr, out_dp));
  if (n > 0) {
    MG_LAUNCH(strict_gkeys_kernel<<<blocks_for(ncell, 256), 256, 0, st>>>(cs, ncell, gkey));
    MG_LAUNCH(strict_gauss_pass_kernel<<<blocks_for(n, 128), 128, 0, st>>>(
        xt, porder, pstart, upstream, mu, prec6, alpha, ci, gkey, n, g, r, d_mu, d_abar6, d_alpha));
  }
  return 0;
}

}  // namespace mg
