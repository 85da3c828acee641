// mg_ssim.cu -- 2D SSIM loss and its analytic gradient for the per-step
// full-slice term (/root/reference/pkg/src/mgauss/ssim.py:21-122; used at
// train.py:407-436).  11-tap Gaussian window (sigma 1.5), valid windows,
// float64 separable correlations; the gradient is pushed back through the
// adjoint (zero-padded full) correlation.
#include "mg_render.cuh"

namespace mg {

constexpr int kWin = 11;
constexpr double kC1 = 0.01 * 0.01, kC2 = 0.03 * 0.03;

__constant__ double c_w[kWin];

#define GL(i, n) for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

// pass 1: horizontal valid correlation of the 5 moment fields, (H, Wv, 5)
template <typename T>
__global__ void ssim_h_kernel(const T* __restrict__ pred, const T* __restrict__ tgt, int H, int W,
                              double* __restrict__ h5) {
  const int Wv = W - kWin + 1;
  GL(e, (int64_t)H * Wv) {
    int y = (int)(e / Wv), x = (int)(e % Wv);
    double s[5] = {0, 0, 0, 0, 0};
    for (int j = 0; j < kWin; ++j) {
      double p = pred[(int64_t)y * W + x + j], t = tgt[(int64_t)y * W + x + j], w = c_w[j];
      s[0] += w * p;
      s[1] += w * t;
      s[2] += w * p * p;
      s[3] += w * t * t;
      s[4] += w * p * t;
    }
    for (int f = 0; f < 5; ++f) h5[e * 5 + f] = s[f];
  }
}

// pass 2: vertical -> ssim map, coefficient fields (g_mu, g_sqr, g_cross), loss sum
__global__ void ssim_v_kernel(const double* __restrict__ h5, int H, int W, double* __restrict__ g3,
                              double* __restrict__ ssim_sum) {
  const int Wv = W - kWin + 1, Hv = H - kWin + 1;
  const double u = -1.0 / ((double)Hv * Wv);
  double local = 0.0;
  GL(e, (int64_t)Hv * Wv) {
    int y = (int)(e / Wv), x = (int)(e % Wv);
    double m[5] = {0, 0, 0, 0, 0};
    for (int i = 0; i < kWin; ++i) {
      const double* r = h5 + ((int64_t)(y + i) * Wv + x) * 5;
      for (int f = 0; f < 5; ++f) m[f] += c_w[i] * r[f];
    }
    double mp = m[0], mt = m[1];
    double vp = m[2] - mp * mp, vt = m[3] - mt * mt, cv = m[4] - mp * mt;
    double a1 = 2.0 * mp * mt + kC1, a2 = 2.0 * cv + kC2;
    double b1 = mp * mp + mt * mt + kC1, b2 = vp + vt + kC2;
    double den = b1 * b2;
    double s = (a1 * a2) / den;
    local += s;
    double da1 = a2 / den, da2 = a1 / den, db1 = -s / b1, db2 = -s / b2;
    g3[e * 3 + 0] = u * (2.0 * mt * da1 + 2.0 * mp * db1 - 2.0 * mt * da2 - 2.0 * mp * db2);
    g3[e * 3 + 1] = u * db2;
    g3[e * 3 + 2] = u * 2.0 * da2;
  }
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(MG_FULL, local, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(ssim_sum, local);
}

// pass 3: adjoint horizontal (full), (Hv, W, 3)
__global__ void ssim_ah_kernel(const double* __restrict__ g3, int H, int W, double* __restrict__ a3) {
  const int Wv = W - kWin + 1, Hv = H - kWin + 1;
  GL(e, (int64_t)Hv * W) {
    int y = (int)(e / W), x = (int)(e % W);
    double s[3] = {0, 0, 0};
    for (int j = 0; j < kWin; ++j) {
      int xs = x - j;
      if (xs < 0 || xs >= Wv) continue;
      const double* r = g3 + ((int64_t)y * Wv + xs) * 3;
      for (int f = 0; f < 3; ++f) s[f] += c_w[j] * r[f];
    }
    for (int f = 0; f < 3; ++f) a3[e * 3 + f] = s[f];
  }
}

// pass 4: adjoint vertical + combine -> upstream[y*W + x] = scale * dloss/dpred
template <typename T>
__global__ void ssim_av_kernel(const double* __restrict__ a3, const T* __restrict__ pred,
                               const T* __restrict__ tgt, int H, int W, double scale, T* __restrict__ up) {
  const int Hv = H - kWin + 1;
  GL(e, (int64_t)H * W) {
    int y = (int)(e / W), x = (int)(e % W);
    double s[3] = {0, 0, 0};
    for (int i = 0; i < kWin; ++i) {
      int ys = y - i;
      if (ys < 0 || ys >= Hv) continue;
      const double* r = a3 + ((int64_t)ys * W + x) * 3;
      for (int f = 0; f < 3; ++f) s[f] += c_w[i] * r[f];
    }
    double gr = s[0] + s[1] * 2.0 * (double)pred[e] + s[2] * (double)tgt[e];
    up[e] = (T)(scale * gr);
  }
}

static bool g_w_init = false;

size_t ssim_workspace_bytes(int H, int W) {
  size_t a = (size_t)H * (W - kWin + 1) * 5 * 8;
  size_t b = (size_t)(H - kWin + 1) * (W - kWin + 1) * 3 * 8;
  size_t c = (size_t)(H - kWin + 1) * W * 3 * 8;
  return ((a + 255) & ~(size_t)255) + ((b + 255) & ~(size_t)255) + ((c + 255) & ~(size_t)255) + 256;
}

static unsigned gs(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b > 4096) b = 4096;
  return (unsigned)(b < 1 ? 1 : b);
}

template <typename T>
static void launch_ssim_t(const T* pred, const T* tgt, int H, int W, double scale, T* up, double* ssim_sum,
                          void* ws, cudaStream_t st) {
  if (!g_w_init) {
    double w[kWin], s = 0.0;
    for (int i = 0; i < kWin; ++i) {
      double o = i - (kWin - 1) / 2.0;
      w[i] = exp(-(o * o) / (2.0 * 1.5 * 1.5));
      s += w[i];
    }
    for (int i = 0; i < kWin; ++i) w[i] /= s;
    cudaMemcpyToSymbol(c_w, w, sizeof(w));
    g_w_init = true;
  }
  const int Wv = W - kWin + 1, Hv = H - kWin + 1;
  char* p = (char*)ws;
  double* h5 = (double*)p;
  p += (((size_t)H * Wv * 5 * 8 + 255) & ~(size_t)255);
  double* g3 = (double*)p;
  p += (((size_t)Hv * Wv * 3 * 8 + 255) & ~(size_t)255);
  double* a3 = (double*)p;
  MG_LAUNCH(ssim_h_kernel<<<gs((int64_t)H * Wv), 256, 0, st>>>(pred, tgt, H, W, h5));
  MG_LAUNCH(ssim_v_kernel<<<gs((int64_t)Hv * Wv), 256, 0, st>>>(h5, H, W, g3, ssim_sum));
  MG_LAUNCH(ssim_ah_kernel<<<gs((int64_t)Hv * W), 256, 0, st>>>(g3, H, W, a3));
  MG_LAUNCH(ssim_av_kernel<<<gs((int64_t)H * W), 256, 0, st>>>(a3, pred, tgt, H, W, scale, up));
}

void launch_ssim(const float* pred, const float* tgt, int H, int W, double scale, float* up, double* ssim_sum,
                 void* ws, cudaStream_t st) {
  launch_ssim_t(pred, tgt, H, W, scale, up, ssim_sum, ws, st);
}

// float64 prediction / target / gradient (strict-float64 training)
void launch_ssim_f64(const double* pred, const double* tgt, int H, int W, double scale, double* up,
                     double* ssim_sum, void* ws, cudaStream_t st) {
  launch_ssim_t(pred, tgt, H, W, scale, up, ssim_sum, ws, st);
}

}  // namespace mg
