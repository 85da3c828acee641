// mg_nrf.cu -- fused residual field (NRF) for the training step: the
// reference's r(x) = 0.1 tanh(MLP(enc(x))) (/root/reference/pkg/src/mgauss/
// nrf.py:23-182) with widths 39-64-64-64-64-1, SiLU hidden activations and 6
// Fourier bands, in four launches instead of ~45 small torch kernels:
//
//   nrf_fwd_kernel   encode + 4 hidden layers + output, one 64-point tile per
//                    CTA iteration; layer GEMMs on shared-memory tiles with
//                    f32x2 FFMA2 (4 outputs x 4 points per thread); writes r
//                    (optionally added into the prediction), tanh(.) and the
//                    pre-activations z (point-major) for the backward
//   nrf_bwd_kernel   output/hidden deltas down to the encoding and d_points
//                    (through the sin/cos features), writing the per-layer
//                    deltas point-major
//   nrf_dw_kernel    dW_l = A_l^T dZ_l and db_l over point chunks, one partial
//                    per CTA (A_l = enc or SiLU(z_{l-1}), staged point-major
//                    in shared memory)
//   nrf_reduce_kernel  fixed-order sum of the partials -> deterministic grads
//
// Everything is float32 like the torch path it replaces (nrf.py host mirror).
#include <stdlib.h>

#include "mg_render.cuh"

namespace mg {

constexpr int kNE = 39;       // 3 + 6 * bands
constexpr int kNH = 64;       // hidden width
constexpr int kNBands = 6;
constexpr int kNT = 64;       // points per tile
constexpr int kNThr = 256;    // threads per CTA (4 outputs x 4 points each for a 64 x 64 tile)
#ifndef MG_NRF_CHUNK
#define MG_NRF_CHUNK 128
#endif
constexpr int kNChunk = MG_NRF_CHUNK;  // points per dW staging chunk (double-buffered: 2 x 2 x chunk x 256 B smem)
// the largest float32 not above 0.1 (0.1f itself is 0.1000000015): |r| <= 0.1 then holds exactly, as
// nrf.py:126 guarantees in float64 (relative change 6e-8)
constexpr float kNOutBound = 0.099999994f;
#ifndef MG_NRF_UNROLL
#define MG_NRF_UNROLL 8  // k-loop unroll of the tile GEMMs (4: fwd 0.181 ms, 8: 0.173 ms, 16: 0.176 ms at 131k points)
#endif
constexpr int kNUnroll = MG_NRF_UNROLL;

// parameter block in shared memory (floats)
constexpr int oW0 = 0;
constexpr int oW1 = oW0 + kNE * kNH;
constexpr int oW2 = oW1 + kNH * kNH;
constexpr int oW3 = oW2 + kNH * kNH;
constexpr int oW4 = oW3 + kNH * kNH;
constexpr int oB0 = oW4 + kNH;
constexpr int oB4 = oB0 + 4 * kNH;
constexpr int kNParams = oB4 + 1;                    // 15105
constexpr int kNParamsPad = (kNParams + 3) & ~3;

struct NrfParams {
  const float* w[5];
  const float* b[5];
};
struct NrfGrads {
  float* w[5];
  float* b[5];
};

__device__ __forceinline__ void nrf_load_params(float* s, const NrfParams& P) {
  const int t = threadIdx.x, n = blockDim.x;
  for (int i = t; i < kNE * kNH; i += n) s[oW0 + i] = P.w[0][i];
  for (int l = 1; l <= 3; ++l)
    for (int i = t; i < kNH * kNH; i += n) s[oW1 + (l - 1) * kNH * kNH + i] = P.w[l][i];
  for (int i = t; i < kNH; i += n) s[oW4 + i] = P.w[4][i];
  for (int l = 0; l < 4; ++l)
    for (int i = t; i < kNH; i += n) s[oB0 + l * kNH + i] = P.b[l][i];
  if (t == 0) s[oB4] = P.b[4][0];
}

// Fourier feature f of point x (nrf.py:23-36 column order: x, then per band
// sin(xyz), cos(xyz)); frequency 2^band * pi in float32 like the torch mirror.
__device__ __forceinline__ float nrf_enc(const float* x, int f) {
  if (f < 3) return x[f];
  const int g = f - 3, band = g / 6, w = g - 6 * band, c = w % 3;
  const float s = x[c] * ldexpf(3.14159265358979323846f, band);
  return w < 3 ? sinf(s) : cosf(s);
}

// MUFU ex2 + rcp (a few ulp; the torch mirror agrees to ~1e-7 relative)
__device__ __forceinline__ float nrf_sigmoid(float z) { return __frcp_rn(1.0f + __expf(-z)); }
__device__ __forceinline__ float nrf_silu(float z) { return z * nrf_sigmoid(z); }
__device__ __forceinline__ float nrf_dsilu(float z) {
  const float s = nrf_sigmoid(z);
  return s * (1.0f + z * (1.0f - s));
}
// silu'(z), with silu(z) = z s as a by-product
__device__ __forceinline__ float nrf_dsilu_h(float z, float& h) {
  const float s = nrf_sigmoid(z);
  h = z * s;
  return s * (1.0f + z * (1.0f - s));
}

// acc[jj][q] += sum_k W[k][4jb + jj] * A[k][4pb + 2q .. +1]: A feature-major
// [K][kNT], W row-major [K][kNH] (one layer of the forward).
template <int K>
__device__ __forceinline__ void nrf_gemm_fwd(const float* A, const float* W, int pb, int jb, f2 (&acc)[4][2]) {
#pragma unroll
  for (int jj = 0; jj < 4; ++jj) acc[jj][0] = acc[jj][1] = bc2(0.f);
#pragma unroll kNUnroll
  for (int k = 0; k < K; ++k) {
    const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(A + k * kNT + 4 * pb);
    const float4 w = *reinterpret_cast<const float4*>(W + k * kNH + 4 * jb);
    const f2 a0{a.x}, a1{a.y};
    acc[0][0] = fma2(bc2(w.x), a0, acc[0][0]);
    acc[0][1] = fma2(bc2(w.x), a1, acc[0][1]);
    acc[1][0] = fma2(bc2(w.y), a0, acc[1][0]);
    acc[1][1] = fma2(bc2(w.y), a1, acc[1][1]);
    acc[2][0] = fma2(bc2(w.z), a0, acc[2][0]);
    acc[2][1] = fma2(bc2(w.z), a1, acc[2][1]);
    acc[3][0] = fma2(bc2(w.w), a0, acc[3][0]);
    acc[3][1] = fma2(bc2(w.w), a1, acc[3][1]);
  }
}

// acc[ii][q] += sum_k W[4ib + ii][k] * D[k][4pb + 2q .. +1]: D feature-major
// [kNH][kNT] deltas of layer l, W = W_l (in x out), i.e. D back through W^T.
__device__ __forceinline__ void nrf_gemm_bwd(const float* D, const float* W, int nrows, int pb, int ib,
                                             f2 (&acc)[4][2]) {
#pragma unroll
  for (int ii = 0; ii < 4; ++ii) acc[ii][0] = acc[ii][1] = bc2(0.f);
  const float* w0 = W + min(4 * ib + 0, nrows - 1) * kNH;
  const float* w1 = W + min(4 * ib + 1, nrows - 1) * kNH;
  const float* w2 = W + min(4 * ib + 2, nrows - 1) * kNH;
  const float* w3 = W + min(4 * ib + 3, nrows - 1) * kNH;
#pragma unroll kNUnroll
  for (int k = 0; k < kNH; ++k) {
    const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(D + k * kNT + 4 * pb);
    const f2 a0{a.x}, a1{a.y};
    const float v0 = w0[k], v1 = w1[k], v2 = w2[k], v3 = w3[k];
    acc[0][0] = fma2(bc2(v0), a0, acc[0][0]);
    acc[0][1] = fma2(bc2(v0), a1, acc[0][1]);
    acc[1][0] = fma2(bc2(v1), a0, acc[1][0]);
    acc[1][1] = fma2(bc2(v1), a1, acc[1][1]);
    acc[2][0] = fma2(bc2(v2), a0, acc[2][0]);
    acc[2][1] = fma2(bc2(v2), a1, acc[2][1]);
    acc[3][0] = fma2(bc2(v3), a0, acc[3][0]);
    acc[3][1] = fma2(bc2(v3), a1, acc[3][1]);
  }
}

__device__ __forceinline__ float acc_at(const f2 (&acc)[4][2], int r, int s) {
  return (s & 1) ? hi(acc[r][s >> 1]) : lo(acc[r][s >> 1]);
}

struct NrfFwdSmem {
  float prm[kNParamsPad];
  float enc[kNE][kNT];   // feature-major
  float h[2][kNH][kNT];  // ping-pong activations, feature-major
  float red[4][kNT];
};

// z_out (optional): 4 x b x 64 pre-activations, point-major (row per point).
__global__ void __launch_bounds__(kNThr) nrf_fwd_kernel(const float* __restrict__ x, int64_t b, NrfParams P,
                                                        float* __restrict__ pred_add, float* __restrict__ r_out,
                                                        float* __restrict__ t_out, float* __restrict__ z_out) {
  extern __shared__ __align__(16) unsigned char nrf_dyn[];
  NrfFwdSmem& sm = *reinterpret_cast<NrfFwdSmem*>(nrf_dyn);
  nrf_load_params(sm.prm, P);
  const int tid = threadIdx.x, pb = tid & 15, jb = tid >> 4;
  const int64_t ntiles = (b + kNT - 1) / kNT;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t p0 = tile * kNT;
    __syncthreads();  // previous tile's readers are done (and the parameters are loaded)
    for (int e = tid; e < kNE * kNT; e += kNThr) {
      const int f = e / kNT, p = e - f * kNT;
      float xv[3] = {0.f, 0.f, 0.f};
      if (p0 + p < b) {
        xv[0] = x[(p0 + p) * 3 + 0];
        xv[1] = x[(p0 + p) * 3 + 1];
        xv[2] = x[(p0 + p) * 3 + 2];
      }
      sm.enc[f][p] = nrf_enc(xv, f);
    }
    __syncthreads();
    f2 acc[4][2];
#pragma unroll 1
    for (int l = 0; l < 4; ++l) {
      if (l == 0)
        nrf_gemm_fwd<kNE>(&sm.enc[0][0], sm.prm + oW0, pb, jb, acc);
      else
        nrf_gemm_fwd<kNH>(&sm.h[(l - 1) & 1][0][0], sm.prm + oW1 + (l - 1) * kNH * kNH, pb, jb, acc);
      float z[4][4];
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const float bj = sm.prm[oB0 + l * kNH + 4 * jb + jj];
#pragma unroll
        for (int s = 0; s < 4; ++s) z[jj][s] = acc_at(acc, jj, s) + bj;
      }
      if (z_out) {
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const int64_t p = p0 + 4 * pb + s;
          if (p < b)
            *reinterpret_cast<float4*>(z_out + ((int64_t)l * b + p) * kNH + 4 * jb) =
                make_float4(z[0][s], z[1][s], z[2][s], z[3][s]);
        }
      }
#pragma unroll
      for (int jj = 0; jj < 4; ++jj)
        *reinterpret_cast<float4*>(&sm.h[l & 1][4 * jb + jj][4 * pb]) =
            make_float4(nrf_silu(z[jj][0]), nrf_silu(z[jj][1]), nrf_silu(z[jj][2]), nrf_silu(z[jj][3]));
      __syncthreads();
    }
    {  // output layer 64 -> 1 (h3 in h[1]), four partial sums per point
      const int p = tid & (kNT - 1), part = tid >> 6;
      float s = 0.f;
#pragma unroll
      for (int j = part * 16; j < part * 16 + 16; ++j) s = fmaf(sm.prm[oW4 + j], sm.h[1][j][p], s);
      sm.red[part][p] = s;
    }
    __syncthreads();
    if (tid < kNT && p0 + tid < b) {
      const float z4 = sm.prm[oB4] + ((sm.red[0][tid] + sm.red[1][tid]) + (sm.red[2][tid] + sm.red[3][tid]));
      const float t = tanhf(z4);
      const float r = kNOutBound * t;
      if (t_out) t_out[p0 + tid] = t;
      if (r_out) r_out[p0 + tid] = r;
      if (pred_add) pred_add[p0 + tid] += r;
    }
  }
}

struct NrfBwdSmem {
  float prm[kNParamsPad];
  float d[2][kNH][kNT];  // ping-pong deltas, feature-major
  float denc[kNE + 1][kNT];
  float d4[kNT];
  float xs[kNT][3];
};

// dz: 4 x b x 64 layer deltas (point-major), d4: b output deltas, dp: b x 3.
__global__ void __launch_bounds__(kNThr) nrf_bwd_kernel(const float* __restrict__ x, int64_t b, NrfParams P,
                                                        const float* __restrict__ up, const float* __restrict__ tin,
                                                        const float* __restrict__ z, float* __restrict__ dz,
                                                        float* __restrict__ d4g, float* __restrict__ dp,
                                                        float* __restrict__ hout, float* __restrict__ encout) {
  extern __shared__ __align__(16) unsigned char nrf_dyn[];
  NrfBwdSmem& sm = *reinterpret_cast<NrfBwdSmem*>(nrf_dyn);
  nrf_load_params(sm.prm, P);
  const int tid = threadIdx.x, pb = tid & 15, jb = tid >> 4;
  const int64_t ntiles = (b + kNT - 1) / kNT;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t p0 = tile * kNT;
    __syncthreads();
    if (tid < kNT) {
      const int64_t p = p0 + tid;
      float d = 0.f;
      if (p < b) {
        const float t = tin[p];
        d = up[p] * kNOutBound * (1.0f - t * t);
        d4g[p] = d;
        sm.xs[tid][0] = x[p * 3 + 0];
        sm.xs[tid][1] = x[p * 3 + 1];
        sm.xs[tid][2] = x[p * 3 + 2];
      } else {
        sm.xs[tid][0] = sm.xs[tid][1] = sm.xs[tid][2] = 0.f;
      }
      sm.d4[tid] = d;
    }
    __syncthreads();
    // layer 3: dz3 = d4 * W4 * silu'(z3)
    {
      float dv[4][4];
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const int64_t p = p0 + 4 * pb + s;
        float4 zz = make_float4(0.f, 0.f, 0.f, 0.f);
        if (p < b) zz = *reinterpret_cast<const float4*>(z + ((int64_t)3 * b + p) * kNH + 4 * jb);
        const float d = sm.d4[4 * pb + s];
        float4 hh;
        dv[0][s] = d * sm.prm[oW4 + 4 * jb + 0] * nrf_dsilu_h(zz.x, hh.x);
        dv[1][s] = d * sm.prm[oW4 + 4 * jb + 1] * nrf_dsilu_h(zz.y, hh.y);
        dv[2][s] = d * sm.prm[oW4 + 4 * jb + 2] * nrf_dsilu_h(zz.z, hh.z);
        dv[3][s] = d * sm.prm[oW4 + 4 * jb + 3] * nrf_dsilu_h(zz.w, hh.w);
        if (p < b) {
          *reinterpret_cast<float4*>(dz + ((int64_t)3 * b + p) * kNH + 4 * jb) =
              make_float4(dv[0][s], dv[1][s], dv[2][s], dv[3][s]);
          *reinterpret_cast<float4*>(hout + ((int64_t)3 * b + p) * kNH + 4 * jb) = hh;
        }
      }
#pragma unroll
      for (int jj = 0; jj < 4; ++jj)
        *reinterpret_cast<float4*>(&sm.d[1][4 * jb + jj][4 * pb]) =
            make_float4(dv[jj][0], dv[jj][1], dv[jj][2], dv[jj][3]);
    }
    __syncthreads();
    f2 acc[4][2];
    // layers 3 -> 1: dh_{l-1} = W_l dz_l, dz_{l-1} = dh_{l-1} * silu'(z_{l-1})
#pragma unroll 1
    for (int l = 3; l >= 1; --l) {
      const int cur = l & 1, nxt = cur ^ 1;
      nrf_gemm_bwd(&sm.d[cur][0][0], sm.prm + oW1 + (l - 1) * kNH * kNH, kNH, pb, jb, acc);
      float dv[4][4];
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const int64_t p = p0 + 4 * pb + s;
        float4 zz = make_float4(0.f, 0.f, 0.f, 0.f);
        if (p < b) zz = *reinterpret_cast<const float4*>(z + ((int64_t)(l - 1) * b + p) * kNH + 4 * jb);
        float4 hh;
        dv[0][s] = acc_at(acc, 0, s) * nrf_dsilu_h(zz.x, hh.x);
        dv[1][s] = acc_at(acc, 1, s) * nrf_dsilu_h(zz.y, hh.y);
        dv[2][s] = acc_at(acc, 2, s) * nrf_dsilu_h(zz.z, hh.z);
        dv[3][s] = acc_at(acc, 3, s) * nrf_dsilu_h(zz.w, hh.w);
        if (p < b) {
          *reinterpret_cast<float4*>(dz + ((int64_t)(l - 1) * b + p) * kNH + 4 * jb) =
              make_float4(dv[0][s], dv[1][s], dv[2][s], dv[3][s]);
          *reinterpret_cast<float4*>(hout + ((int64_t)(l - 1) * b + p) * kNH + 4 * jb) = hh;
        }
      }
#pragma unroll
      for (int jj = 0; jj < 4; ++jj)
        *reinterpret_cast<float4*>(&sm.d[nxt][4 * jb + jj][4 * pb]) =
            make_float4(dv[jj][0], dv[jj][1], dv[jj][2], dv[jj][3]);
      __syncthreads();
    }
    // encoding deltas: denc = W0 dz0 (dz0 in d[0]); 10 row blocks of 4 (row 39 unused)
    if (jb < (kNE + 3) / 4) {
      nrf_gemm_bwd(&sm.d[0][0][0], sm.prm + oW0, kNE, pb, jb, acc);
#pragma unroll
      for (int ii = 0; ii < 4; ++ii)
        *reinterpret_cast<float4*>(&sm.denc[4 * jb + ii][4 * pb]) =
            make_float4(acc_at(acc, ii, 0), acc_at(acc, ii, 1), acc_at(acc, ii, 2), acc_at(acc, ii, 3));
    }
    __syncthreads();
    // d_points through the features: d/dx sin(f x) = f cos(f x), d/dx cos(f x) = -f sin(f x)
    if (tid < 3 * kNT) {
      const int p = tid & (kNT - 1), c = tid >> 6;
      if (p0 + p < b) {
        const float xc = sm.xs[p][c];
        float* er = encout + (p0 + p) * (kNE + 1);  // the encoding row, for the dW pass
        er[c] = xc;
        if (c == 0) er[kNE] = 0.f;
        float v = sm.denc[c][p];
        for (int band = 0; band < kNBands; ++band) {
          const float f = ldexpf(3.14159265358979323846f, band);
          const float s = xc * f;
          const float sn = sinf(s), cs = cosf(s);
          er[3 + 6 * band + c] = sn;
          er[3 + 6 * band + 3 + c] = cs;
          v += f * (cs * sm.denc[3 + 6 * band + c][p] - sn * sm.denc[3 + 6 * band + 3 + c][p]);
        }
        dp[(p0 + p) * 3 + c] = v;
      }
    }
  }
}

struct NrfDwSmem {
  float a[2][kNChunk][kNH];  // double-buffered point-major A rows (enc padded to 40, or SiLU(z_{l-1}))
  float d[2][kNChunk][kNH];  // double-buffered point-major delta rows
};

__device__ __forceinline__ void cp_async16_zfill(void* dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes)
               : "memory");
}

// One chunk of A and delta rows into buffer `buf` with 16-byte cp.async pieces;
// rows past n (and A columns past astride) are zero-filled.
__device__ __forceinline__ void nrf_dw_stage(NrfDwSmem& sm, int buf, const float* A, int astride, const float* D,
                                             int64_t q0, int n, int tid) {
  constexpr int kPieces = kNChunk * kNH / 4 / kNThr;
#pragma unroll
  for (int u = 0; u < kPieces; ++u) {
    const int e = tid + u * kNThr, p = e / (kNH / 4), i4 = e - p * (kNH / 4);
    const bool okA = p < n && 4 * i4 < astride, okD = p < n;
    cp_async16_zfill(&sm.a[buf][p][4 * i4], okA ? A + (q0 + p) * astride + 4 * i4 : A, okA ? 16 : 0);
    cp_async16_zfill(&sm.d[buf][p][4 * i4], okD ? D + (q0 + p) * kNH + 4 * i4 : D, okD ? 16 : 0);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// blockIdx.y = layer (0..3: 64-wide deltas; 4: output layer); each CTA sums
// chunks blockIdx.x, blockIdx.x + gridDim.x, ... into one partial:
// part[l] = [gridDim.x][kin * 64 + 64] (dW row-major, then db).  The layer
// inputs come from the backward pass (enc rows, h = SiLU(z) rows); chunk c+1
// is copied in by cp.async while chunk c is reduced.
__global__ void __launch_bounds__(kNThr) nrf_dw_kernel(int64_t b, const float* __restrict__ enc,
                                                       const float* __restrict__ h, const float* __restrict__ dz,
                                                       const float* __restrict__ d4g, float* __restrict__ part) {
  extern __shared__ __align__(16) unsigned char nrf_dyn[];
  NrfDwSmem& sm = *reinterpret_cast<NrfDwSmem*>(nrf_dyn);
  const int l = blockIdx.y, tid = threadIdx.x;
  const int64_t nchunks = (b + kNChunk - 1) / kNChunk;
  const int G = gridDim.x;
  const int64_t sz0 = kNE * kNH + kNH, sz = kNH * kNH + kNH;
  float* out = part + (l == 0 ? 0 : G * (sz0 + (int64_t)(l - 1) * sz)) +
               (int64_t)blockIdx.x * (l == 0 ? sz0 : (l < 4 ? sz : 65));
  const float* A = l == 0 ? enc : h + (int64_t)(l == 4 ? 3 : l - 1) * b * kNH;
  if (l == 4) {  // dW4[j] = sum_p h3[p][j] d4[p]; db4 = sum_p d4[p] (small: synchronous staging)
    float s4 = 0.f, sb4 = 0.f;
    for (int64_t c = blockIdx.x; c < nchunks; c += G) {
      const int64_t q0 = c * kNChunk;
      const int n = (int)min((int64_t)kNChunk, b - q0);
      __syncthreads();
      for (int e = tid; e < kNChunk * kNH / 4; e += kNThr) {
        const int p = e / (kNH / 4), i4 = e - p * (kNH / 4);
        *reinterpret_cast<float4*>(&sm.a[0][p][4 * i4]) =
            p < n ? *reinterpret_cast<const float4*>(A + (q0 + p) * kNH + 4 * i4) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if (tid < kNChunk) sm.d[0][tid][0] = tid < n ? d4g[q0 + tid] : 0.f;
      __syncthreads();
      if (tid < kNH) {
        for (int p = 0; p < n; ++p) s4 = fmaf(sm.a[0][p][tid], sm.d[0][p][0], s4);
      } else if (tid == kNH) {
        for (int p = 0; p < n; ++p) sb4 += sm.d[0][p][0];
      }
    }
    if (tid < kNH) out[tid] = s4;
    if (tid == kNH) out[kNH] = sb4;
    return;
  }
  const int kin = l == 0 ? kNE : kNH;
  const int astride = l == 0 ? kNE + 1 : kNH;  // floats per A row in global memory
  const float* D = dz + (int64_t)l * b * kNH;
  const int ib = tid >> 4, jb = tid & 15;
  f2 acc[4][2];
#pragma unroll
  for (int ii = 0; ii < 4; ++ii) acc[ii][0] = acc[ii][1] = bc2(0.f);
  f2 dba[2] = {bc2(0.f), bc2(0.f)};
  int buf = 0;
  int64_t c = blockIdx.x;
  if (c < nchunks) nrf_dw_stage(sm, 0, A, astride, D, c * kNChunk, (int)min((int64_t)kNChunk, b - c * kNChunk), tid);
  for (; c < nchunks; c += G) {
    const int64_t cn = c + G;
    if (cn < nchunks) {
      nrf_dw_stage(sm, buf ^ 1, A, astride, D, cn * kNChunk, (int)min((int64_t)kNChunk, b - cn * kNChunk), tid);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const int n = (int)min((int64_t)kNChunk, b - c * kNChunk);
    if (4 * ib < kin) {
      // rows past n are zero, so groups of 8 points may run past n
#pragma unroll 1
      for (int p0 = 0; p0 < n; p0 += 8) {
        float4 a[8];
        ulonglong2 dd[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          a[u] = *reinterpret_cast<const float4*>(&sm.a[buf][p0 + u][4 * ib]);
          dd[u] = *reinterpret_cast<const ulonglong2*>(&sm.d[buf][p0 + u][4 * jb]);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const f2 d0{dd[u].x}, d1{dd[u].y};
          acc[0][0] = fma2(bc2(a[u].x), d0, acc[0][0]);
          acc[0][1] = fma2(bc2(a[u].x), d1, acc[0][1]);
          acc[1][0] = fma2(bc2(a[u].y), d0, acc[1][0]);
          acc[1][1] = fma2(bc2(a[u].y), d1, acc[1][1]);
          acc[2][0] = fma2(bc2(a[u].z), d0, acc[2][0]);
          acc[2][1] = fma2(bc2(a[u].z), d1, acc[2][1]);
          acc[3][0] = fma2(bc2(a[u].w), d0, acc[3][0]);
          acc[3][1] = fma2(bc2(a[u].w), d1, acc[3][1]);
          if (ib == 0) {
            dba[0] = add2(dba[0], d0);
            dba[1] = add2(dba[1], d1);
          }
        }
      }
    }
    __syncthreads();  // the next iteration stages into this buffer
    buf ^= 1;
  }
#pragma unroll
  for (int ii = 0; ii < 4; ++ii) {
    const int i = 4 * ib + ii;
    if (i < kin) {
      *reinterpret_cast<float4*>(out + (int64_t)i * kNH + 4 * jb) =
          make_float4(lo(acc[ii][0]), hi(acc[ii][0]), lo(acc[ii][1]), hi(acc[ii][1]));
    }
  }
  if (ib == 0)
    *reinterpret_cast<float4*>(out + (int64_t)kin * kNH + 4 * jb) =
        make_float4(lo(dba[0]), hi(dba[0]), lo(dba[1]), hi(dba[1]));
}

// grads = fixed-order sum over the G partials of each layer.
__global__ void nrf_reduce_kernel(const float* __restrict__ part, int G, NrfGrads out) {
  const int64_t sz0 = kNE * kNH + kNH, sz = kNH * kNH + kNH;
  const int64_t total = sz0 + 3 * sz + 65;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    int l;
    int64_t e, base, size;
    if (o < sz0) {
      l = 0, e = o, base = 0, size = sz0;
    } else if (o < sz0 + 3 * sz) {
      l = 1 + (int)((o - sz0) / sz), e = (o - sz0) % sz, base = G * (sz0 + (int64_t)(l - 1) * sz), size = sz;
    } else {
      l = 4, e = o - sz0 - 3 * sz, base = G * (sz0 + 3 * sz), size = 65;
    }
    float s = 0.f;
    for (int c = 0; c < G; ++c) s += part[base + (int64_t)c * size + e];
    const int kin = l == 0 ? kNE : kNH, nout = l == 4 ? 1 : kNH;
    if (e < (int64_t)kin * nout)
      out.w[l][e] = s;
    else
      out.b[l][e - (int64_t)kin * nout] = s;
  }
}

#ifndef MG_NRF_DW_G
#define MG_NRF_DW_G 64
#endif
static int nrf_dw_grid(int64_t b) {
  const int64_t nchunks = (b + kNChunk - 1) / kNChunk;
  const int64_t g = MG_NRF_DW_G;
  return (int)(nchunks < g ? (nchunks < 1 ? 1 : nchunks) : g);
}

size_t nrf_backward_ws_bytes(int64_t b) {
  const int G = nrf_dw_grid(b);
  const size_t sz0 = kNE * kNH + kNH, sz = kNH * kNH + kNH;
  const size_t part = (size_t)G * (sz0 + 3 * sz + 65) * sizeof(float);
  const size_t dz = (size_t)4 * b * kNH * sizeof(float), d4 = (size_t)b * sizeof(float);
  const size_t enc = (size_t)b * (kNE + 1) * sizeof(float);
  auto al = [](size_t v) { return (v + 255) & ~(size_t)255; };
  return 2 * al(dz) + al(d4) + al(enc) + al(part);
}

static void nrf_attrs() {
  static bool done = false;
  if (done) return;
  cudaFuncSetAttribute(nrf_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(NrfFwdSmem));
  cudaFuncSetAttribute(nrf_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(NrfBwdSmem));
  cudaFuncSetAttribute(nrf_dw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(NrfDwSmem));
  done = true;
}

static unsigned nrf_tile_grid(const void* kern, size_t smem, int64_t b) {
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kNThr, smem);
  const int64_t tiles = (b + kNT - 1) / kNT;
  int64_t g = (int64_t)num_sms() * (per_sm > 0 ? per_sm : 1);
  return (unsigned)(tiles < g ? (tiles < 1 ? 1 : tiles) : g);
}

// MGAUSS_NRF_TC=0 selects the SIMT layer kernels (A/B); the tcgen05 layers are the default.
bool nrf_use_tc() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MGAUSS_NRF_TC");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

void launch_nrf_forward(const float* x, int64_t b, const float* const* w, const float* const* bias, float* pred_add,
                        float* r_out, float* t_out, float* z_out, cudaStream_t st) {
  if (b <= 0) return;
  if (nrf_use_tc()) {
    launch_nrf_forward_tc(x, b, w, bias, pred_add, r_out, t_out, z_out, st);
    return;
  }
  nrf_attrs();
  NrfParams P;
  for (int l = 0; l < 5; ++l) P.w[l] = w[l], P.b[l] = bias[l];
  const size_t smem = sizeof(NrfFwdSmem);
  MG_LAUNCH(nrf_fwd_kernel<<<nrf_tile_grid((const void*)nrf_fwd_kernel, smem, b), kNThr, smem, st>>>(
      x, b, P, pred_add, r_out, t_out, z_out));
}

void launch_nrf_backward(const float* x, int64_t b, const float* const* w, const float* const* bias, const float* up,
                         const float* t, const float* z, float* dp, float* const* dw, float* const* db, void* ws,
                         cudaStream_t st) {
  if (b <= 0) {  // no points: zero gradients
    for (int l = 0; l < 5; ++l) {
      const size_t kin = l == 0 ? kNE : kNH, nout = l == 4 ? 1 : kNH;
      cudaMemsetAsync(dw[l], 0, kin * nout * sizeof(float), st);
      cudaMemsetAsync(db[l], 0, nout * sizeof(float), st);
    }
    return;
  }
  nrf_attrs();
  NrfParams P;
  NrfGrads Gd;
  for (int l = 0; l < 5; ++l) P.w[l] = w[l], P.b[l] = bias[l], Gd.w[l] = dw[l], Gd.b[l] = db[l];
  auto al = [](size_t v) { return (v + 255) & ~(size_t)255; };
  char* p = (char*)ws;
  float* dz = (float*)p;
  p += al((size_t)4 * b * kNH * sizeof(float));
  float* d4 = (float*)p;
  p += al((size_t)b * sizeof(float));
  float* hb = (float*)p;
  p += al((size_t)4 * b * kNH * sizeof(float));
  float* enc = (float*)p;
  p += al((size_t)b * (kNE + 1) * sizeof(float));
  float* part = (float*)p;
  if (nrf_use_tc()) {
    launch_nrf_bwd_chain_tc(x, b, w, bias, up, t, z, dz, d4, dp, hb, enc, st);
  } else {
    const size_t smem = sizeof(NrfBwdSmem);
    MG_LAUNCH(nrf_bwd_kernel<<<nrf_tile_grid((const void*)nrf_bwd_kernel, smem, b), kNThr, smem, st>>>(
        x, b, P, up, t, z, dz, d4, dp, hb, enc));
  }
  const int G = nrf_dw_grid(b);
  MG_LAUNCH(nrf_dw_kernel<<<dim3(G, 5), kNThr, sizeof(NrfDwSmem), st>>>(b, enc, hb, dz, d4, part));
  const int64_t total = (kNE * kNH + kNH) + 3 * (kNH * kNH + kNH) + 65;
  MG_LAUNCH(nrf_reduce_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(part, G, Gd));
}

}  // namespace mg

namespace mg {

// Adam over the NRF parameter tensors (AdamState.step "nrf", train.py:251-271)
// in one single-CTA launch: the device step counter is read, used and
// incremented here so the update replays inside the step graph.
struct NrfAdamArgs {
  const float* g[10];
  float* p[10];
  float* m[10];
  float* v[10];
  int64_t n[10];
  int count;
};

__global__ void __launch_bounds__(1024) nrf_adam_kernel(NrfAdamArgs a, double* __restrict__ tstep, float lr,
                                                        double b1, double b2, float eps) {
  const double t = *tstep + 1.0;
  const float bc1 = (float)(1.0 - pow(b1, t)), bc2 = (float)(1.0 - pow(b2, t));
  const float fb1 = (float)b1, fb2 = (float)b2, a1 = (float)(1.0 - b1), a2 = (float)(1.0 - b2);
  for (int k = 0; k < a.count; ++k) {
    const float* __restrict__ g = a.g[k];
    float* __restrict__ p = a.p[k];
    float* __restrict__ m = a.m[k];
    float* __restrict__ v = a.v[k];
    for (int64_t i = threadIdx.x; i < a.n[k]; i += blockDim.x) {
      const float gi = g[i];
      const float mi = m[i] * fb1 + a1 * gi;
      const float vi = v[i] * fb2 + a2 * gi * gi;
      m[i] = mi;
      v[i] = vi;
      const float den = sqrtf(vi / bc2) + eps;
      p[i] -= lr * ((mi / bc1) / den);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) *tstep = t;
}

void launch_nrf_adam(const float* const* g, float* const* p, float* const* m, float* const* v, const int64_t* n,
                     int count, double* tstep, double lr, double b1, double b2, double eps, cudaStream_t st) {
  NrfAdamArgs a;
  a.count = count < 10 ? count : 10;
  for (int k = 0; k < a.count; ++k) a.g[k] = g[k], a.p[k] = p[k], a.m[k] = m[k], a.v[k] = v[k], a.n[k] = n[k];
  MG_LAUNCH(nrf_adam_kernel<<<1, 1024, 0, st>>>(a, tstep, (float)lr, b1, b2, (float)eps));
}

}  // namespace mg
