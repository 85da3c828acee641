// mg_nrf64.cu -- float64 Neural Residual Field for the strict-float64 training
// path (StrictTrainer, render.set_strict_fp64): the same network and manual
// backward as /root/reference/pkg/src/mgauss/nrf.py:23-182, evaluated in
// float64 like the reference's numpy code, so strict training follows the
// reference's trajectory to rounding level.  Throughput is not the goal here
// (the float32 tensor-core kernels in mg_nrf.cu / mg_nrf_tc.cu are the
// production path); every array is feature-major [feature][point] so a warp's
// loads and stores are coalesced, and every reduction over points has a fixed
// order (warp-strided partial sums + a shuffle tree), so results are
// run-to-run deterministic.
//
// Any reference configuration with widths <= 64 and <= 8 layers (the
// production 39-64-64-64-64-1 and e.g. the acceptance suite's 15-8-8-1).
// Workspace (the reference's `cache`, nrf.py:140-145), doubles, sized for the
// maximum shape:
//   enc  [64][b]        fourier_encode(x)                        (nrf.py:23-36)
//   post [7][64][b]     silu(pre[l])  for the hidden layers      (nrf.py:121-125)
//   pre  [7][64][b]     hidden pre-activations z = h W + b
//   t    [b]            tanh of the output pre-activation        (nrf.py:126)
//   dz   [7][64][b]     d/dz of the hidden layers (backward)     (nrf.py:165-172)
//   dzo  [b]            d/dz of the output layer
#include "mg_render.cuh"

namespace mg {

namespace {
constexpr int kMaxW = 64, kMaxDepth = 8;

// Widths (fan_in of layer 0 = 3 + 6 bands, hidden <= 64, output 1), up to 8
// layers: the reference's ResidualField.create(frequency_bands, hidden)
// (nrf.py:58-83) for any such configuration.
struct Nrf64Params {
  const double* w[kMaxDepth];
  const double* b[kMaxDepth];
  int width[kMaxDepth + 1];
  int depth, bands;
  double bound;
  __host__ __device__ int fan_in(int l) const { return width[l]; }
  __host__ __device__ int fan_out(int l) const { return width[l + 1]; }
};
struct Nrf64Grads {
  double* w[kMaxDepth];
  double* b[kMaxDepth];
};

struct Ws64 {
  double *enc, *post, *pre, *t, *dz, *dzo;
};
__host__ __device__ inline Ws64 carve64(void* ws, int64_t b) {
  double* p = (double*)ws;
  Ws64 w;
  w.enc = p;
  p += (int64_t)kMaxW * b;
  w.post = p;
  p += (int64_t)(kMaxDepth - 1) * kMaxW * b;
  w.pre = p;
  p += (int64_t)(kMaxDepth - 1) * kMaxW * b;
  w.t = p;
  p += b;
  w.dz = p;
  p += (int64_t)(kMaxDepth - 1) * kMaxW * b;
  w.dzo = p;
  return w;
}

__device__ __forceinline__ double sigmoid64(double z) { return 1.0 / (1.0 + exp(-z)); }

// h(l): the input activations of layer l for point p, feature-major.
__device__ __forceinline__ const double* layer_input(const Ws64& W, int l, int64_t b) {
  return l == 0 ? W.enc : W.post + (int64_t)(l - 1) * kMaxW * b;
}

__global__ void __launch_bounds__(128) nrf64_fwd_kernel(const double* __restrict__ x, int64_t b, Nrf64Params P,
                                                        Ws64 W, double* __restrict__ r_out) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < b; p += (int64_t)gridDim.x * blockDim.x) {
    // fourier_encode (nrf.py:23-36): [x, sin(2^k pi x), cos(2^k pi x)]
    double xs[3] = {x[3 * p], x[3 * p + 1], x[3 * p + 2]};
    for (int a = 0; a < 3; ++a) W.enc[(int64_t)a * b + p] = xs[a];
    for (int k = 0; k < P.bands; ++k) {
      const double f = ldexp(3.141592653589793, k);  // (2.0**k) * np.pi, exact
      for (int a = 0; a < 3; ++a) {
        double s, c;
        sincos(xs[a] * f, &s, &c);
        W.enc[(int64_t)(3 + 6 * k + a) * b + p] = s;
        W.enc[(int64_t)(6 + 6 * k + a) * b + p] = c;
      }
    }
    for (int l = 0; l < P.depth; ++l) {
      const double* h = layer_input(W, l, b);
      const int fi = P.fan_in(l), fo = P.fan_out(l);
      for (int j = 0; j < fo; ++j) {
        double z = 0.0;
        for (int i = 0; i < fi; ++i) z = fma(h[(int64_t)i * b + p], P.w[l][i * fo + j], z);
        z += P.b[l][j];
        if (l < P.depth - 1) {
          W.pre[((int64_t)l * kMaxW + j) * b + p] = z;
          W.post[((int64_t)l * kMaxW + j) * b + p] = z * sigmoid64(z);
        } else {
          const double t = tanh(z);
          W.t[p] = t;
          r_out[p] = P.bound * t;
        }
      }
    }
  }
}

__global__ void __launch_bounds__(128) nrf64_bwd_kernel(const double* __restrict__ x, int64_t b, Nrf64Params P,
                                                        Ws64 W, const double* __restrict__ up,
                                                        double* __restrict__ d_points) {
  const int L = P.depth;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < b; p += (int64_t)gridDim.x * blockDim.x) {
    const double t = W.t[p];
    const double dzo = up[p] * P.bound * (1.0 - t * t);  // nrf.py:164
    W.dzo[p] = dzo;
    // last hidden layer (L - 2) from the output layer (fan_out 1)
    if (L >= 2) {
      const int fo = P.fan_out(L - 2);
      for (int i = 0; i < fo; ++i) {
        const double z = W.pre[((int64_t)(L - 2) * kMaxW + i) * b + p], s = sigmoid64(z);
        W.dz[((int64_t)(L - 2) * kMaxW + i) * b + p] = dzo * P.w[L - 1][i] * (s * (1.0 + z * (1.0 - s)));
      }
    }
    for (int l = L - 2; l >= 1; --l) {  // dh = dz W^T, dz_prev = dh * silu'(pre)   (nrf.py:165-172)
      const int fi = P.fan_in(l), fo = P.fan_out(l);
      for (int i = 0; i < fi; ++i) {
        double dh = 0.0;
        for (int j = 0; j < fo; ++j) dh = fma(W.dz[((int64_t)l * kMaxW + j) * b + p], P.w[l][i * fo + j], dh);
        const double z = W.pre[((int64_t)(l - 1) * kMaxW + i) * b + p], s = sigmoid64(z);
        W.dz[((int64_t)(l - 1) * kMaxW + i) * b + p] = dh * (s * (1.0 + z * (1.0 - s)));
      }
    }
    // d_enc = dz0 W0^T, then the encoding Jacobian (nrf.py:174-181)
    const int fi0 = P.fan_in(0), fo0 = P.fan_out(0);
    double dp[3] = {0.0, 0.0, 0.0};
    for (int i = 0; i < fi0; ++i) {
      double dh = 0.0;
      if (L == 1) {
        dh = dzo * P.w[0][i];
      } else {
        for (int j = 0; j < fo0; ++j) dh = fma(W.dz[(int64_t)j * b + p], P.w[0][i * fo0 + j], dh);
      }
      if (i < 3) {
        dp[i] += dh;
      } else {
        const int k = (i - 3) / 6, a = (i - 3) % 6;
        const double f = ldexp(3.141592653589793, k);
        double s, c;
        sincos(f * x[3 * p + (a % 3)], &s, &c);
        if (a < 3)
          dp[a] += f * c * dh;
        else
          dp[a - 3] -= f * s * dh;
      }
    }
    for (int a = 0; a < 3; ++a) d_points[3 * p + a] = dp[a];
  }
}

// dW[l][i][j] = sum_p h_l[i][p] dz_l[j][p];  db[l][j] = sum_p dz_l[j][p].
// One warp per output element (output index = global warp id over all layers).
__global__ void __launch_bounds__(256) nrf64_dw_kernel(int64_t b, Nrf64Params P, Ws64 W, Nrf64Grads G) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t e = warp;
  int l = 0;
  for (; l < P.depth; ++l) {
    const int64_t nl = (int64_t)(P.fan_in(l) + 1) * P.fan_out(l);  // weights + biases of layer l
    if (e < nl) break;
    e -= nl;
  }
  if (l >= P.depth) return;
  const int fi = P.fan_in(l), fo = P.fan_out(l);
  const double* dz = l == P.depth - 1 ? W.dzo : W.dz + (int64_t)l * kMaxW * b;
  const int j = (int)(e % fo);
  const int i = (int)(e / fo);  // i == fi: bias
  const double* dzj = dz + (int64_t)j * b;
  double s = 0.0;
  if (i < fi) {
    const double* h = layer_input(W, l, b) + (int64_t)i * b;
    for (int64_t p = lane; p < b; p += 32) s = fma(h[p], dzj[p], s);
  } else {
    for (int64_t p = lane; p < b; p += 32) s += dzj[p];
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(MG_FULL, s, o);
  if (lane == 0) {
    if (i < fi)
      G.w[l][i * fo + j] = s;
    else
      G.b[l][j] = s;
  }
}

unsigned grid_for(int64_t n, int thr) {
  int64_t g = (n + thr - 1) / thr;
  if (g > 148 * 16) g = 148 * 16;
  return (unsigned)(g < 1 ? 1 : g);
}

bool make_params(Nrf64Params& P, const double* const* w, const double* const* bias, const int* widths, int depth,
                 int bands, double bound) {
  if (depth < 1 || depth > kMaxDepth || bands < 0 || 3 + 6 * bands > kMaxW) return false;
  if (widths[0] != 3 + 6 * bands || widths[depth] != 1) return false;
  for (int l = 0; l <= depth; ++l)
    if (widths[l] < 1 || widths[l] > kMaxW) return false;
  for (int l = 0; l < depth; ++l) P.w[l] = w[l], P.b[l] = bias[l];
  for (int l = 0; l <= depth; ++l) P.width[l] = widths[l];
  P.depth = depth;
  P.bands = bands;
  P.bound = bound;
  return true;
}
}  // namespace

size_t nrf64_workspace_bytes(int64_t b) {
  return (size_t)(kMaxW + 3 * (kMaxDepth - 1) * kMaxW + 2) * (size_t)b * sizeof(double) + 256;
}

bool launch_nrf64_forward(const double* x, int64_t b, const double* const* w, const double* const* bias,
                          const int* widths, int depth, int bands, double bound, double* r, void* ws,
                          cudaStream_t st) {
  Nrf64Params P;
  if (!make_params(P, w, bias, widths, depth, bands, bound)) return false;
  MG_LAUNCH(nrf64_fwd_kernel<<<grid_for(b, 128), 128, 0, st>>>(x, b, P, carve64(ws, b), r));
  return true;
}

bool launch_nrf64_backward(const double* x, int64_t b, const double* const* w, const double* const* bias,
                           const int* widths, int depth, int bands, double bound, const double* up,
                           double* d_points, double* const* dw, double* const* db, void* ws, cudaStream_t st) {
  Nrf64Params P;
  if (!make_params(P, w, bias, widths, depth, bands, bound)) return false;
  Nrf64Grads G;
  for (int l = 0; l < depth; ++l) G.w[l] = dw[l], G.b[l] = db[l];
  const Ws64 W = carve64(ws, b);
  MG_LAUNCH(nrf64_bwd_kernel<<<grid_for(b, 128), 128, 0, st>>>(x, b, P, W, up, d_points));
  int64_t outs = 0;
  for (int l = 0; l < depth; ++l) outs += (int64_t)(widths[l] + 1) * widths[l + 1];
  MG_LAUNCH(nrf64_dw_kernel<<<(unsigned)((outs * 32 + 255) / 256), 256, 0, st>>>(b, P, W, G));
  return true;
}

}  // namespace mg
