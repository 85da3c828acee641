// mg_capi.cu -- extern "C" entry points (include/mgauss_b200.h).
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/mgauss_b200.h"
#include "mg_render.cuh"
#include "mg_sort.cuh"

using namespace mg;

namespace {
thread_local char g_err[512] = "";

int fail(const char* msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg);
  return MG_EINVAL;
}

int cuda_status() {
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) {
    snprintf(g_err, sizeof(g_err), "CUDA: %s", cudaGetErrorString(e));
    cudaGetLastError();
    return -(int)e;
  }
  return 0;
}

inline size_t al(size_t b) { return (b + 255) & ~(size_t)255; }

struct Bump {
  char* p;
  size_t left;
  bool ok = true;
  Bump(void* base, size_t n) : p((char*)base), left(n) {}
  template <class T>
  T* take(size_t count) {
    size_t b = al(count * sizeof(T) + (count == 0 ? 1 : 0));
    if (b > left) {
      ok = false;
      return nullptr;
    }
    T* r = (T*)p;
    p += b;
    left -= b;
    return r;
  }
  void* rest() { return p; }
};

inline cudaStream_t S(void* s) { return (cudaStream_t)s; }

int64_t ncell_of(int64_t g) { return g * g * g; }

// ---- small kernels local to the ABI layer ----
__global__ void csr64_to_32_kernel(const int64_t* __restrict__ cs, int64_t ncell1, const int64_t* __restrict__ ci,
                                   int64_t n, int* __restrict__ cs32, int* __restrict__ ci32) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ncell1 || i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < ncell1) cs32[i] = (int)cs[i];
    if (i < n) ci32[i] = (int)ci[i];
  }
}

// gkey[p] = cell c with cs[c] <= p < cs[c+1]  (follows the caller's CSR exactly)
__global__ void keys_from_csr_kernel(const int* __restrict__ cs, int64_t ncell, uint32_t* __restrict__ gkey) {
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < ncell; c += (int64_t)gridDim.x * blockDim.x) {
    for (int p = cs[c]; p < cs[c + 1]; ++p) gkey[p] = (uint32_t)c;
  }
}

__global__ void iota32_kernel(int* __restrict__ v, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (int)i;
}

__global__ void i32_to_i64_kernel(const int* __restrict__ s, int64_t n, int64_t* __restrict__ d) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = s[i];
}

__global__ void activate_f64_kernel(const double* __restrict__ quat, const double* __restrict__ ls,
                                    const double* __restrict__ lg, int64_t n, double* __restrict__ qn,
                                    double* __restrict__ rot, double* __restrict__ inv_var,
                                    double* __restrict__ prec6, double* __restrict__ alpha, int* __restrict__ err) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double q[4] = {quat[4 * i], quat[4 * i + 1], quat[4 * i + 2], quat[4 * i + 3]};
    double nrm = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    if (!(nrm > 1e-12)) {
      atomicOr(err, MG_ERR_DEGENERATE_QUAT);
      nrm = 1.0;
    }
    double w = q[0] / nrm, x = q[1] / nrm, y = q[2] / nrm, z = q[3] / nrm;
    qn[4 * i] = w;
    qn[4 * i + 1] = x;
    qn[4 * i + 2] = y;
    qn[4 * i + 3] = z;
    double R[9] = {1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y),
                   2.0 * (x * y + w * z),       1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x),
                   2.0 * (x * z - w * y),       2.0 * (y * z + w * x),       1.0 - 2.0 * (x * x + y * y)};
    for (int a = 0; a < 9; ++a) rot[9 * i + a] = R[a];
    double e[3];
    for (int a = 0; a < 3; ++a) {
      double s = ls[3 * i + a];
      s = s < -20.0 ? -20.0 : (s > 20.0 ? 20.0 : s);
      e[a] = exp(-2.0 * s);
      inv_var[3 * i + a] = e[a];
    }
    const int ia[6] = {0, 0, 0, 1, 1, 2}, ib[6] = {0, 1, 2, 1, 2, 2};
    for (int k = 0; k < 6; ++k) {
      int a = ia[k], b = ib[k];
      prec6[6 * i + k] = R[3 * a] * e[0] * R[3 * b] + R[3 * a + 1] * e[1] * R[3 * b + 1] + R[3 * a + 2] * e[2] * R[3 * b + 2];
    }
    alpha[i] = 1.0 / (1.0 + exp(-lg[i]));
  }
}

// All-pairs evaluation (_kernels.py:147-162) over fp32 records, smem-tiled.
__global__ void dense_kernel(const double* __restrict__ pts, int64_t b, GaussSoA grec, int64_t n,
                             double* __restrict__ out) {
  __shared__ float4 ta[128], tb[128];
  __shared__ float2 tc[128];
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  float x = 0.f, y = 0.f, z = 0.f;
  if (q < b) {
    x = (float)pts[3 * q];
    y = (float)pts[3 * q + 1];
    z = (float)pts[3 * q + 2];
  }
  float acc = 0.f;
  for (int64_t t0 = 0; t0 < n; t0 += 128) {
    int cnt = (int)min((int64_t)128, n - t0);
    __syncthreads();
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
      ta[i] = grec.A[t0 + i];
      tb[i] = grec.B[t0 + i];
      tc[i] = grec.C[t0 + i];
    }
    __syncthreads();
    for (int i = 0; i < cnt; ++i) {
      float4 A = ta[i], B = tb[i];
      float2 C = tc[i];
      float dx = x - A.x, dy = y - A.y, dz = z - A.z;
      float m = dx * (B.x * dx + 2.f * B.w * dy + 2.f * C.x * dz) + dy * (B.y * dy + 2.f * C.y * dz) + B.z * dz * dz;
      acc += A.w * gauss_w(m);
    }
  }
  if (q < b) out[q] = acc;
}

unsigned grid_of(int64_t n) {
  int64_t b = (n + 255) / 256;
  int64_t cap = (int64_t)num_sms() * 16;
  if (b > cap) b = cap;
  return (unsigned)(b < 1 ? 1 : b);
}

// ---- composite workspace layouts ----
// Binning sorts cell keys with the counting sort (MG_SORT_RADIX=1: stable LSD
// radix sort + CSR build; same output).
#ifndef MG_SORT_RADIX
#define MG_SORT_RADIX 0
#endif

size_t sort_ws(int64_t n, int64_t g) {
  const size_t a = radix_workspace_bytes(n) + csr_workspace_bytes(ncell_of(g));
  const size_t b = counting_workspace_bytes(n, ncell_of(g));
  return (a > b ? a : b) + 512;
}

void sort_cells(const uint32_t* keys, uint32_t* keys_sorted, int* order, int* starts, int64_t n, int64_t g, void* ws,
                cudaStream_t st) {
  if (MG_SORT_RADIX) {
    radix_sort_pairs(keys, keys_sorted, order, n, bits_for(ncell_of(g) - 1), ws, st);
    csr_starts(keys_sorted, n, ncell_of(g), starts, ws, st);
  } else {
    counting_sort_pairs(keys, keys_sorted, order, starts, n, ncell_of(g), ws, st);
  }
}

size_t bin_ws(int64_t n, int64_t g) { return al((size_t)n * 4) + sort_ws(n, g) + 1024; }

size_t points_ws(int64_t ns, int64_t g) {
  return al((size_t)ns * 4) * 2 + al((size_t)ns * 16) + sort_ws(ns, g) + 2048;
}

size_t fwd_ws(int64_t ns) { return al((size_t)ns * 16) + 256 + items_workspace_bytes(ns) + 1024; }

int do_bin(const float* pos32, const double* pos64, int64_t n, int64_t g, uint32_t* keys_sorted, int* order,
           int* starts, void* ws, size_t wsb, cudaStream_t st) {
  Bump b(ws, wsb);
  uint32_t* keys = b.take<uint32_t>(n);
  if (!b.ok) return fail("mg_bin: workspace too small");
  if (pos32)
    launch_gauss_keys(pos32, n, (int)g, keys, st);
  else
    launch_gauss_keys_f64(pos64, n, (int)g, keys, st);
  sort_cells(keys, keys_sorted, order, starts, n, g, b.rest(), st);
  return cuda_status();
}

}  // namespace

namespace mg {
long long& launch_counter() {
  static long long c = 0;
  return c;
}
}  // namespace mg

extern "C" {

int mg_abi_version(void) { return MG_ABI_VERSION; }
long long mg_launch_count(void) { return mg::launch_counter(); }
const char* mg_last_error(void) { return g_err; }
int mg_device_sm_count(void) { return num_sms(); }

int mg_cell_keys_f64(const double* pos, int64_t n, int64_t g, uint32_t* keys, void* stream) {
  if (g < 1 || n < 0) return fail("mg_cell_keys_f64: bad sizes");
  launch_gauss_keys_f64(pos, n, (int)g, keys, S(stream));
  return cuda_status();
}

size_t mg_bin_workspace_bytes(int64_t n, int64_t g) { return bin_ws(n, g); }

int mg_bin_f32(const float* pos, int64_t n, int64_t g, uint32_t* keys_sorted, int32_t* cell_indices,
               int32_t* cell_starts, void* ws, size_t wsb, void* stream) {
  if (g < 1 || n < 0 || ncell_of(g) >= (1ll << 31)) return fail("mg_bin_f32: bad sizes");
  return do_bin(pos, nullptr, n, g, keys_sorted, cell_indices, cell_starts, ws, wsb, S(stream));
}

int mg_bin_f64(const double* pos, int64_t n, int64_t g, uint32_t* keys_sorted, int32_t* cell_indices,
               int32_t* cell_starts, void* ws, size_t wsb, void* stream) {
  if (g < 1 || n < 0 || ncell_of(g) >= (1ll << 31)) return fail("mg_bin_f64: bad sizes");
  return do_bin(nullptr, pos, n, g, keys_sorted, cell_indices, cell_starts, ws, wsb, S(stream));
}

size_t mg_scan_workspace_bytes(int64_t n) { return scan_workspace_bytes(n); }

int mg_excl_scan_i32(const int32_t* in, int32_t* out, int64_t n, void* ws, size_t wsb, void* stream) {
  if (wsb < scan_workspace_bytes(n)) return fail("mg_excl_scan_i32: workspace too small");
  excl_scan(in, out, n, ws, S(stream));
  return cuda_status();
}

int mg_keys_from_csr(const int32_t* cs, int64_t ncell, uint32_t* keys, void* stream) {
  if (ncell > 0) MG_LAUNCH(keys_from_csr_kernel<<<grid_of(ncell), 256, 0, S(stream)>>>(cs, ncell, keys));
  return cuda_status();
}

int mg_i64_to_i32(const int64_t* src, int64_t n, int32_t* dst, void* stream) {
  if (n > 0) MG_LAUNCH(csr64_to_32_kernel<<<grid_of(n), 256, 0, S(stream)>>>(src, n, nullptr, 0, dst, nullptr));
  return cuda_status();
}

int mg_i32_to_i64(const int32_t* src, int64_t n, int64_t* dst, void* stream) {
  if (n > 0) MG_LAUNCH(i32_to_i64_kernel<<<grid_of(n), 256, 0, S(stream)>>>(src, n, dst));
  return cuda_status();
}

int mg_activate(const float* pos, const float* quat, const float* ls, const float* lg, int64_t n,
                const int32_t* cell_indices, void* grec, int32_t* err_flag, void* stream) {
  launch_gauss_activate(pos, quat, ls, lg, cell_indices, n, (float*)grec, err_flag, S(stream));
  return cuda_status();
}

int mg_activate_f64(const double* quat, const double* ls, const double* lg, int64_t n, double* qn, double* rot,
                    double* inv_var, double* prec6, double* alpha, int32_t* err_flag, void* stream) {
  if (n > 0)
    MG_LAUNCH(activate_f64_kernel<<<grid_of(n), 256, 0, S(stream)>>>(quat, ls, lg, n, qn, rot, inv_var, prec6, alpha, err_flag));
  return cuda_status();
}

size_t mg_points_workspace_bytes(int64_t ns, int64_t g) { return points_ws(ns, g); }

int mg_bin_points(const double* coords, const int64_t* sids, int64_t b, int32_t ntaps, const double* tap_off,
                  const double* dirs, const double* rot, const double* trans, int64_t k, int64_t g,
                  uint32_t* pkey_sorted, int32_t* pinv, int32_t* pstart, void* prec, double* transformed, void* ws,
                  size_t wsb, void* stream) {
  if (g < 1 || b < 0 || ntaps < 1) return fail("mg_bin_points: bad sizes");
  if (ntaps > 1 && (!tap_off || !dirs)) return fail("mg_bin_points: PSF taps need offsets and directions");
  cudaStream_t st = S(stream);
  int64_t ns = b * ntaps;
  Bump w(ws, wsb);
  uint32_t* keys = w.take<uint32_t>(ns);
  int* perm = w.take<int>(ns);
  float4* xf = w.take<float4>(ns);
  if (!w.ok) return fail("mg_bin_points: workspace too small");
  launch_points_prepare(coords, sids, nullptr, b, ntaps, ntaps > 1 ? tap_off : nullptr, dirs, rot, trans, (int)k,
                        (int)g, keys, xf, transformed, st);
  sort_cells(keys, pkey_sorted, perm, pstart, ns, g, w.rest(), st);
  launch_points_gather(xf, perm, ns, (float4*)prec, pinv, st);
  return cuda_status();
}

size_t mg_forward_workspace_bytes(int64_t ns) { return fwd_ws(ns); }

int mg_forward(const void* grec, int64_t n_gauss, const int32_t* gstart, int64_t g, int64_t r, const void* prec,
               const uint32_t* pkey_sorted, const int32_t* pstart, int64_t ns, int32_t with_h, void* out4,
               int32_t* counts, void* ws, size_t wsb, void* stream) {
  if (g < 1 || r < 0 || ns < 0) return fail("mg_forward: bad sizes");
  cudaStream_t st = S(stream);
  Bump w(ws, wsb);
  int4* items = w.take<int4>(ns);
  int* nitems = w.take<int>(1);
  if (!w.ok) return fail("mg_forward: workspace too small");
  if (ns == 0) return 0;
  build_items_cells(pstart, (int)g, fwd_qmax(), items, nitems, st, fwd_dense_min());
  launch_forward(with_h != 0, (const float*)grec, n_gauss, gstart, (int)g, (int)r, (const float4*)prec, pkey_sorted,
                 pstart,
                 items, nitems, ns, (float4*)out4, counts, st);
  return cuda_status();
}

int mg_forward_finish(const void* out4, const int32_t* counts, const int32_t* pinv, int64_t b, int32_t ntaps,
                      const double* tap_w, double* intensity, float* intensity_f32, int64_t* counts_out,
                      int64_t* pair_total, void* stream) {
  launch_forward_finish((const float4*)out4, counts, pinv, b, ntaps, ntaps > 1 ? tap_w : nullptr, intensity,
                        intensity_f32, counts_out, pair_total, S(stream));
  return cuda_status();
}

int mg_backward_points(const double* up, const float* up32, int64_t b, int32_t ntaps, const double* tap_w,
                       const int32_t* pinv, const void* out4, void* prec, double* d_points, void* stream) {
  if (!up && !up32) return fail("mg_backward_points: no upstream");
  launch_backward_points(up, up32, pinv, b, ntaps, ntaps > 1 ? tap_w : nullptr, (const float4*)out4, (float4*)prec,
                         d_points, S(stream));
  return cuda_status();
}

size_t mg_backward_workspace_bytes(int64_t n, int64_t g) {
  size_t a = fwd_ws(n), b = backward_staged_ws_bytes(n, (int)g) + 1024;
  return a > b ? a : b;
}

static bool staged_backward_enabled(int64_t r) {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("MGAUSS_STAGED_BWD");
    env = (e && e[0] == '1') ? 1 : 0;
  }
  return env == 1 && (2 * r + 1) * (2 * r + 1) <= 128;
}

// MGAUSS_BWD_PAIRS=0: one item per Gaussian (default: k-adjacent pairs)
static int backward_pair_mode() {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("MGAUSS_BWD_PAIRS");
    env = (e && e[0] == '0') ? 0 : 1;
  }
  return env;
}

int mg_backward(const void* grec, const uint32_t* gkey_sorted, const int32_t* gstart, int64_t n, int64_t g, int64_t r,
                const void* prec, const int32_t* pstart, float* acc10, void* ws, size_t wsb, void* stream) {
  if (g < 1 || r < 0 || n < 0) return fail("mg_backward: bad sizes");
  cudaStream_t st = S(stream);
  if (n == 0) return 0;
  if (staged_backward_enabled(r)) {
    if (wsb < backward_staged_ws_bytes(n, (int)g)) return fail("mg_backward: workspace too small");
    launch_backward_staged((const float*)grec, n, gkey_sorted, gstart, (int)g, (int)r, (const float4*)prec, pstart,
                           acc10, ws, st);
    return cuda_status();
  }
  // one work item per sorted Gaussian (or per k-adjacent Gaussian pair),
  // implicit: no item build, no workspace
  launch_backward((const float*)grec, n, gkey_sorted, gstart, (int)g, (int)r, (const float4*)prec, pstart, nullptr,
                  nullptr, n, acc10, st, backward_pair_mode());
  return cuda_status();
}

int mg_backward_epilogue(const float* acc10, const int32_t* order, int64_t n, const float* quat, const float* ls,
                         const float* lg, double* d_pos, double* d_q, double* d_s, double* d_l, void* stream) {
  launch_epilogue(acc10, order, n, quat, ls, lg, d_pos, d_q, d_s, d_l, S(stream));
  return cuda_status();
}

int mg_epilogue_f64(const double* d_mu, const double* d_abar6, const double* d_alpha, const double* quat,
                    const double* ls, const double* lg, int64_t n, double* d_pos, double* d_q, double* d_s,
                    double* d_l, void* stream) {
  launch_epilogue_f64(d_mu, d_abar6, d_alpha, quat, ls, lg, n, d_pos, d_q, d_s, d_l, S(stream));
  return cuda_status();
}

int mg_pack_records(const double* mu, const double* prec6, const double* alpha, const int32_t* order, int64_t n,
                    void* grec, void* stream) {
  launch_gauss_pack_prepared(mu, prec6, alpha, order, n, (float*)grec, S(stream));
  return cuda_status();
}

int mg_backward_accumulators(const float* acc10, const int32_t* order, int64_t n, const double* alpha, double* d_mu,
                             double* d_abar6, double* d_alpha, void* stream) {
  launch_acc_to_ref(acc10, order, n, alpha, d_mu, d_abar6, d_alpha, S(stream));
  return cuda_status();
}

size_t mg_transform_grads_workspace_bytes(int64_t k) { return transform_grads_ws_bytes(k); }

int mg_transform_grads(const double* d_points, const double* coords, const int64_t* sids, int64_t b, int32_t ntaps,
                       const double* tap_off, const double* dirs, const double* t_quats, int64_t k, double* scratch12,
                       double* out7, int32_t accumulate, void* ws, size_t ws_bytes, void* stream) {
  if (ws && ws_bytes < transform_grads_ws_bytes(k)) return fail("mg_transform_grads: workspace too small");
  launch_transform_grads(d_points, coords, sids, b, ntaps, ntaps > 1 ? tap_off : nullptr, dirs, t_quats, (int)k,
                         scratch12, out7, accumulate, ws, S(stream));
  return cuda_status();
}

size_t mg_volume_workspace_bytes(int64_t nx, int64_t ny, int64_t nz) {
  return volume_workspace_bytes((int)nx, (int)ny, (int)nz);
}

int mg_sample_volume(const void* grec, int64_t n_gauss, const int32_t* gstart, int64_t g, int64_t r, int64_t nx,
                     int64_t ny,
                     int64_t nz, const double* lo, const double* hi, int64_t i0, int64_t i1, const float* residual,
                     float* out, void* ws, size_t wsb, void* stream) {
  if (nx < 1 || ny < 1 || nz < 1 || i0 < 0 || i1 > nx || i1 <= i0 || g < 1 || r < 0)
    return fail("mg_sample_volume: bad sizes");
  if (wsb < volume_workspace_bytes((int)nx, (int)ny, (int)nz)) return fail("mg_sample_volume: workspace too small");
  int dims[3] = {(int)nx, (int)ny, (int)nz};
  launch_sample_volume((const float*)grec, n_gauss, gstart, (int)g, (int)r, dims, lo, hi, (int)i0, (int)i1, residual,
                       out, ws,
                       S(stream));
  return cuda_status();
}

int mg_smooth_l1(const float* pred, const float* target, int64_t b, float* up_out, double* loss_acc, void* stream) {
  return mg_smooth_l1_scaled(pred, target, b, b > 0 ? 1.0 / (double)b : 0.0, up_out, loss_acc, stream);
}

int mg_aniso_loss_grad_f64(const double* log_scales, int64_t n, double lambda_ratio, double* grad,
                           double* loss_acc, void* stream) {
  if (n < 0) return fail("mg_aniso_loss_grad_f64: n < 0");
  launch_aniso_f64(log_scales, n, lambda_ratio, grad, loss_acc, S(stream));
  return cuda_status();
}

int mg_adam_f64(double* param, const double* grad, double* m, double* v, int64_t n, int64_t t, double lr,
                double beta1, double beta2, double eps, void* stream) {
  if (n < 0 || t < 1) return fail("mg_adam_f64: need n >= 0 and t >= 1");
  launch_adam_f64(param, grad, m, v, n, t, lr, beta1, beta2, eps, S(stream));
  return cuda_status();
}

int mg_smooth_l1_scaled(const float* pred, const float* target, int64_t b, double scale, float* up_out,
                        double* loss_acc, void* stream) {
  if (b < 0) return fail("mg_smooth_l1: b < 0");
  launch_smooth_l1(pred, target, b, scale, up_out, loss_acc, S(stream));
  return cuda_status();
}

size_t mg_nrf_backward_workspace_bytes(int64_t b) { return b < 0 ? 0 : nrf_backward_ws_bytes(b); }

int mg_nrf_forward(const float* x, int64_t b, const float* const* w, const float* const* bias, float* pred_add,
                   float* r_out, float* t_out, float* z_out, void* stream) {
  if (b < 0 || !w || !bias) return fail("mg_nrf_forward: bad arguments");
  if (b == 0) return 0;
  launch_nrf_forward(x, b, w, bias, pred_add, r_out, t_out, z_out, S(stream));
  return cuda_status();
}

int mg_nrf_backward(const float* x, int64_t b, const float* const* w, const float* const* bias, const float* up,
                    const float* t, const float* z, float* d_points, float* const* dw, float* const* db, void* ws,
                    size_t wsb, void* stream) {
  if (b < 0 || !w || !bias || !dw || !db) return fail("mg_nrf_backward: bad arguments");
  if (wsb < nrf_backward_ws_bytes(b)) return fail("mg_nrf_backward: workspace too small");
  launch_nrf_backward(x, b, w, bias, up, t, z, d_points, dw, db, ws, S(stream));
  return cuda_status();
}

int mg_nrf_adam(const float* const* grads, float* const* params, float* const* m, float* const* v,
                const int64_t* sizes, int32_t count, double* tstep, double lr, double beta1, double beta2, double eps,
                void* stream) {
  if (count < 0 || count > 10 || !tstep) return fail("mg_nrf_adam: bad arguments");
  if (count == 0) return 0;
  launch_nrf_adam(grads, params, m, v, sizes, count, tstep, lr, beta1, beta2, eps, S(stream));
  return cuda_status();
}

size_t mg_ssim_workspace_bytes(int64_t h, int64_t w) { return ssim_workspace_bytes((int)h, (int)w); }

int mg_ssim_loss_grad(const float* pred, const float* target, int64_t h, int64_t w, double scale, float* up,
                      double* ssim_sum, void* ws, size_t wsb, void* stream) {
  if (h < 11 || w < 11) return fail("mg_ssim_loss_grad: slice smaller than the 11-tap window");
  if (wsb < ssim_workspace_bytes((int)h, (int)w)) return fail("mg_ssim_loss_grad: workspace too small");
  launch_ssim(pred, target, (int)h, (int)w, scale, up, ssim_sum, ws, S(stream));
  return cuda_status();
}

// ---- float64 variants for strict-float64 training ----
int mg_smooth_l1_f64(const double* pred, const double* target, int64_t b, double* up_out, double* loss_acc,
                     void* stream) {
  if (b < 0) return fail("mg_smooth_l1_f64: b < 0");
  launch_smooth_l1_f64(pred, target, b, (double)b, up_out, loss_acc, S(stream));
  return cuda_status();
}

int mg_ssim_loss_grad_f64(const double* pred, const double* target, int64_t h, int64_t w, double scale, double* up,
                          double* ssim_sum, void* ws, size_t wsb, void* stream) {
  if (h < 11 || w < 11) return fail("mg_ssim_loss_grad_f64: slice smaller than the 11-tap window");
  if (wsb < ssim_workspace_bytes((int)h, (int)w)) return fail("mg_ssim_loss_grad_f64: workspace too small");
  launch_ssim_f64(pred, target, (int)h, (int)w, scale, up, ssim_sum, ws, S(stream));
  return cuda_status();
}

int mg_upsample_f64(const double* q_old, const double* s_old, const double* l_old, const int32_t* node_of_old,
                    int64_t ro, int64_t rn, double* pos, double* q, double* s, double* l, void* stream) {
  if (rn < ro || ro < 1) return fail("mg_upsample_f64: bad resolutions");
  launch_upsample_f64(q_old, s_old, l_old, node_of_old, (int)ro, (int)rn, pos, q, s, l, S(stream));
  return cuda_status();
}

size_t mg_nrf_f64_workspace_bytes(int64_t b) { return b < 0 ? 0 : nrf64_workspace_bytes(b); }

int mg_nrf_forward_f64(const double* x, int64_t b, const double* const* w, const double* const* bias,
                       const int32_t* widths, int32_t depth, int32_t bands, double bound, double* r_out, void* ws,
                       size_t wsb, void* stream) {
  if (b < 0 || !w || !bias || !widths) return fail("mg_nrf_forward_f64: bad arguments");
  if (wsb < nrf64_workspace_bytes(b)) return fail("mg_nrf_forward_f64: workspace too small");
  if (b == 0) return 0;
  if (!launch_nrf64_forward(x, b, w, bias, widths, depth, bands, bound, r_out, ws, S(stream)))
    return fail("mg_nrf_forward_f64: unsupported widths (<= 8 layers, widths <= 64, input 3 + 6 bands, output 1)");
  return cuda_status();
}

int mg_nrf_backward_f64(const double* x, int64_t b, const double* const* w, const double* const* bias,
                        const int32_t* widths, int32_t depth, int32_t bands, double bound, const double* upstream,
                        double* d_points, double* const* dw, double* const* db, void* ws, size_t wsb,
                        void* stream) {
  if (b < 0 || !w || !bias || !dw || !db || !widths) return fail("mg_nrf_backward_f64: bad arguments");
  if (wsb < nrf64_workspace_bytes(b)) return fail("mg_nrf_backward_f64: workspace too small");
  if (!launch_nrf64_backward(x, b, w, bias, widths, depth, bands, bound, upstream, d_points, dw, db, ws, S(stream)))
    return fail("mg_nrf_backward_f64: unsupported widths (<= 8 layers, widths <= 64, input 3 + 6 bands, output 1)");
  return cuda_status();
}

int mg_quat_to_rot_f64(const double* q, int64_t k, double* rot, void* stream) {
  launch_quat_to_rot(q, k, rot, S(stream));
  return cuda_status();
}

int mg_gather_batch(const int64_t* idx, int64_t n, const double* pool_coords, const int64_t* pool_sids,
                    const float* pool_target, double* coords, int64_t* sids, float* target, void* stream) {
  if (n < 0) return fail("mg_gather_batch: bad size");
  launch_gather_batch(idx, n, pool_coords, pool_sids, pool_target, coords, sids, target, S(stream));
  return cuda_status();
}

int mg_counter_incr(int32_t* c, int32_t n, void* stream) {
  launch_counter_incr(c, n, S(stream));
  return cuda_status();
}

int mg_gauss_update(const float* acc10, const int32_t* order, int64_t n, float* pos, float* quat, float* ls,
                    float* lg, float* m, float* v, const double* hyper, int32_t use_aniso, const int32_t* t_dev,
                    double* aniso_acc, void* stream) {
  launch_gauss_update(acc10, order, 0, n, pos, quat, ls, lg, m, v, hyper, use_aniso, t_dev, aniso_acc, S(stream));
  return cuda_status();
}

int mg_gauss_update_inv(const float* acc10, const int32_t* inv, int64_t n, float* pos, float* quat, float* ls,
                        float* lg, float* m, float* v, const double* hyper, int32_t use_aniso, const int32_t* t_dev,
                        double* aniso_acc, void* stream) {
  launch_gauss_update(acc10, inv, 1, n, pos, quat, ls, lg, m, v, hyper, use_aniso, t_dev, aniso_acc, S(stream));
  return cuda_status();
}

int mg_invert_permutation(const int32_t* perm, int64_t n, int32_t* inv, void* stream) {
  if (n < 0) return fail("mg_invert_permutation: n < 0");
  launch_invert_perm(perm, n, inv, S(stream));
  return cuda_status();
}

int mg_transform_adam(double* tq, double* tt, const double* g7, double* m7, double* v7, int64_t k, double lr,
                      double b1, double b2, double eps, const int32_t* t_dev, void* stream) {
  launch_transform_adam(tq, tt, g7, m7, v7, (int)k, lr, b1, b2, eps, t_dev, S(stream));
  return cuda_status();
}

int mg_upsample(const float* q_old, const float* s_old, const float* l_old, const int32_t* node_of_old, int64_t ro,
                int64_t rn, float* pos, float* q, float* s, float* l, void* stream) {
  if (rn < ro || ro < 1) return fail("mg_upsample: bad resolutions");
  launch_upsample(q_old, s_old, l_old, node_of_old, (int)ro, (int)rn, pos, q, s, l, S(stream));
  return cuda_status();
}

// ---- drop-in reference kernel ABI ----
size_t mg_block_workspace_bytes(int64_t b, int64_t n, int64_t g) {
  int64_t nc1 = ncell_of(g) + 1;
  return al((size_t)nc1 * 4) * 2 + al((size_t)n * 4) * 2 + al((size_t)n * 48) + al((size_t)b * 4) * 3 +
         al((size_t)b * 16) * 2 + al((size_t)n * 40) + points_ws(b, g) + fwd_ws(b > n ? b : n) +
         backward_staged_ws_bytes(n, (int)g) + 8192;
}

static int block_common(const double* points, const int64_t* sids, int64_t b, const double* rot, const double* trans,
                        int64_t k, const double* mu, const double* prec6, const double* alpha, int64_t n,
                        const int64_t* cs, const int64_t* ci, int64_t g, int64_t r, bool with_h, double* out_i,
                        int64_t* out_cnt, double* out_x, const double* upstream, double* d_mu, double* d_abar6,
                        double* d_alpha, double* out_dp, void* ws, size_t wsb, cudaStream_t st) {
  if (g < 1 || r < 0 || b < 0 || n < 0) return fail("mg_block: bad sizes");
  if (ncell_of(g) >= (1ll << 31)) return fail("mg_block: grid too large");
  int64_t nc1 = ncell_of(g) + 1;
  Bump w(ws, wsb);
  int* gstart = w.take<int>(nc1);
  int* pstart = w.take<int>(nc1);
  int* gorder = w.take<int>(n);
  uint32_t* gkey = w.take<uint32_t>(n);
  float* grec = w.take<float>(12 * n);
  uint32_t* pkey = w.take<uint32_t>(b);
  int* pinv = w.take<int>(b);
  int* cnt = w.take<int>(b);
  float4* prec = w.take<float4>(b);
  float4* out4 = w.take<float4>(b);
  float* acc10 = w.take<float>(10 * n);
  char* rest = (char*)w.rest();
  size_t restb = w.left;
  if (!w.ok || restb < points_ws(b, g)) return fail("mg_block: workspace too small");
  MG_LAUNCH(csr64_to_32_kernel<<<grid_of(nc1 > n ? nc1 : n), 256, 0, st>>>(cs, nc1, ci, n, gstart, gorder));
  MG_LAUNCH(keys_from_csr_kernel<<<grid_of(nc1 - 1), 256, 0, st>>>(gstart, nc1 - 1, gkey));
  launch_gauss_pack_prepared(mu, prec6, alpha, gorder, n, grec, st);
  int rc = mg_bin_points(points, sids, b, 1, nullptr, nullptr, rot, trans, k, g, pkey, pinv, pstart, prec, out_x,
                         rest, restb, st);
  if (rc) return rc;
  if (b == 0) return cuda_status();
  rc = mg_forward(grec, n, gstart, g, r, prec, pkey, pstart, b, with_h ? 1 : 0, out4, cnt, rest, restb, st);
  if (rc) return rc;
  if (!upstream) {
    launch_forward_finish(out4, cnt, pinv, b, 1, nullptr, out_i, nullptr, out_cnt, nullptr, st);
    return cuda_status();
  }
  launch_backward_points(upstream, nullptr, pinv, b, 1, nullptr, out4, prec, out_dp, st);
  rc = mg_backward(grec, gkey, gstart, n, g, r, prec, pstart, acc10, rest, restb, st);
  if (rc) return rc;
  launch_acc_to_ref(acc10, gorder, n, alpha, d_mu, d_abar6, d_alpha, st);
  return cuda_status();
}

int mg_block_forward(const double* points, const int64_t* sids, int64_t b, const double* rot, const double* trans,
                     int64_t k, const double* mu, const double* prec6, const double* alpha, int64_t n,
                     const int64_t* cs, const int64_t* ci, int64_t g, int64_t r, double* out_i, int64_t* out_cnt,
                     double* out_x, void* ws, size_t wsb, void* stream) {
  return block_common(points, sids, b, rot, trans, k, mu, prec6, alpha, n, cs, ci, g, r, false, out_i, out_cnt, out_x,
                      nullptr, nullptr, nullptr, nullptr, nullptr, ws, wsb, S(stream));
}

int mg_block_backward(const double* points, const int64_t* sids, int64_t b, const double* rot, const double* trans,
                      int64_t k, const double* mu, const double* prec6, const double* alpha, int64_t n,
                      const int64_t* cs, const int64_t* ci, int64_t g, int64_t r, const double* upstream,
                      double* d_mu, double* d_abar6, double* d_alpha, double* out_dp, void* ws, size_t wsb,
                      void* stream) {
  if (!upstream) return fail("mg_block_backward: upstream is required");
  return block_common(points, sids, b, rot, trans, k, mu, prec6, alpha, n, cs, ci, g, r, true, nullptr, nullptr,
                      nullptr, upstream, d_mu, d_abar6, d_alpha, out_dp, ws, wsb, S(stream));
}

// ---- tensor-core self-test (mg_nrf_tc.cu) ----
int mg_tc_selftest(const float* A, const float* Bt, float* D, int32_t split, void* stream) {
  launch_tc_selftest(A, Bt, D, split, S(stream));
  return cuda_status();
}

// ---- strict float64 instantiation of the same ABI (mg_strict.cu) ----
size_t mg_block_f64_workspace_bytes(int64_t b, int64_t n, int64_t g) { return strict_workspace_bytes(b, n, g); }

static int strict_common(const double* points, const int64_t* sids, int64_t b, const double* rot, const double* trans,
                         int64_t k, const double* mu, const double* prec6, const double* alpha, int64_t n,
                         const int64_t* cs, const int64_t* ci, int64_t g, int64_t r, double* out_i, int64_t* out_cnt,
                         double* out_x, const double* upstream, double* d_mu, double* d_abar6, double* d_alpha,
                         double* out_dp, void* ws, size_t wsb, cudaStream_t st) {
  if (g < 1 || r < 0 || b < 0 || n < 0) return fail("mg_block_f64: bad sizes");
  if (ncell_of(g) >= (1ll << 31)) return fail("mg_block_f64: grid too large");
  if (strict_block(points, sids, b, rot, trans, k, mu, prec6, alpha, n, cs, ci, (int)g, (int)r, out_i, out_cnt, out_x,
                   upstream, d_mu, d_abar6, d_alpha, out_dp, ws, wsb, st))
    return fail("mg_block_f64: workspace too small");
  return cuda_status();
}

int mg_block_forward_f64(const double* points, const int64_t* sids, int64_t b, const double* rot, const double* trans,
                         int64_t k, const double* mu, const double* prec6, const double* alpha, int64_t n,
                         const int64_t* cs, const int64_t* ci, int64_t g, int64_t r, double* out_i, int64_t* out_cnt,
                         double* out_x, void* ws, size_t wsb, void* stream) {
  if (!out_i || !out_cnt) return fail("mg_block_forward_f64: out_intensity and out_counts are required");
  return strict_common(points, sids, b, rot, trans, k, mu, prec6, alpha, n, cs, ci, g, r, out_i, out_cnt, out_x,
                       nullptr, nullptr, nullptr, nullptr, nullptr, ws, wsb, S(stream));
}

int mg_block_backward_f64(const double* points, const int64_t* sids, int64_t b, const double* rot,
                          const double* trans, int64_t k, const double* mu, const double* prec6, const double* alpha,
                          int64_t n, const int64_t* cs, const int64_t* ci, int64_t g, int64_t r,
                          const double* upstream, double* d_mu, double* d_abar6, double* d_alpha, double* out_dp,
                          void* ws, size_t wsb, void* stream) {
  if (!upstream || !d_mu || !d_abar6 || !d_alpha) return fail("mg_block_backward_f64: upstream and accumulators are required");
  return strict_common(points, sids, b, rot, trans, k, mu, prec6, alpha, n, cs, ci, g, r, nullptr, nullptr, nullptr,
                       upstream, d_mu, d_abar6, d_alpha, out_dp, ws, wsb, S(stream));
}

size_t mg_dense_workspace_bytes(int64_t n) { return al((size_t)n * 48) + al((size_t)n * 4) + 512; }

int mg_dense_forward(const double* points, int64_t b, const double* mu, const double* prec6, const double* alpha,
                     int64_t n, double* out, void* ws, size_t wsb, void* stream) {
  cudaStream_t st = S(stream);
  Bump w(ws, wsb);
  float* grec = w.take<float>(12 * n);
  int* ident = w.take<int>(n);
  if (!w.ok) return fail("mg_dense_forward: workspace too small");
  if (n > 0) {
    MG_LAUNCH(iota32_kernel<<<grid_of(n), 256, 0, st>>>(ident, n));
    launch_gauss_pack_prepared(mu, prec6, alpha, ident, n, grec, st);
  }
  if (b > 0) MG_LAUNCH(dense_kernel<<<(unsigned)((b + 127) / 128), 128, 0, st>>>(points, b, gauss_soa(grec, n), n, out));
  return cuda_status();
}

}  // extern "C"
