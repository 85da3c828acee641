// mg_nrf_tc.cu -- tensor-core (tcgen05, kind::tf32) building blocks of the
// residual-field MLP.  This file starts with a self-test GEMM that pins the
// descriptor / TMEM conventions of mg_tc.cuh on the device.
#include "mg_render.cuh"
#include "mg_tc.cuh"

namespace mg {

// D[128 x 64] = A[128 x 64] * B, B given transposed as Bt[64 (n)][64 (k)];
// split != 0: 3xTF32 (a_hi b_hi + a_hi b_lo + a_lo b_hi), else 1xTF32.
__global__ void __launch_bounds__(128) tc_selftest_kernel(const float* __restrict__ A, const float* __restrict__ Bt,
                                                          float* __restrict__ D, int split) {
  extern __shared__ __align__(1024) unsigned char dyn[];
  float* a_hi = reinterpret_cast<float*>(dyn);            // 32 KB
  float* a_lo = a_hi + 128 * 64;                          // 32 KB
  float* b_hi = a_lo + 128 * 64;                          // 16 KB
  float* b_lo = b_hi + 64 * 64;                           // 16 KB
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x, warp = t >> 5;
  char* ah = reinterpret_cast<char*>(a_hi);
  char* al = reinterpret_cast<char*>(a_lo);
  char* bh = reinterpret_cast<char*>(b_hi);
  char* bl = reinterpret_cast<char*>(b_lo);
  for (int k = 0; k < 64; ++k) {
    float h, l;
    tc::split_tf32(A[t * 64 + k], h, l);
    *reinterpret_cast<float*>(ah + tc::kmaj_off(t, k, 64)) = h;
    *reinterpret_cast<float*>(al + tc::kmaj_off(t, k, 64)) = l;
  }
  for (int e = t; e < 64 * 64; e += 128) {
    const int n = e >> 6, k = e & 63;
    float h, l;
    tc::split_tf32(Bt[e], h, l);
    *reinterpret_cast<float*>(bh + tc::kmaj_off(n, k, 64)) = h;
    *reinterpret_cast<float*>(bl + tc::kmaj_off(n, k, 64)) = l;
  }
  if (t == 0) {
    tc::mbar_init(&mbar, 1);
    tc::fence_init();
  }
  if (warp == 0) tc::tmem_alloc(&tslot, 64);
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  if (split == 2) {  // bf16x3: overwrite the tiles with three bf16 parts (2-byte K-major layout)
    unsigned short* a16 = reinterpret_cast<unsigned short*>(dyn);        // 3 x 16 KB
    unsigned short* b16 = a16 + 3 * 128 * 64;                            // 3 x 8 KB
    __syncthreads();
    for (int k = 0; k < 64; ++k) {
      unsigned short h[3];
      tc::split_bf16x3(A[t * 64 + k], h[0], h[1], h[2]);
      for (int q = 0; q < 3; ++q)
        *reinterpret_cast<unsigned short*>(reinterpret_cast<char*>(a16 + q * 128 * 64) + tc::kmaj_off2(t, k, 64)) = h[q];
    }
    for (int e = t; e < 64 * 64; e += 128) {
      const int n = e >> 6, k = e & 63;
      unsigned short h[3];
      tc::split_bf16x3(Bt[e], h[0], h[1], h[2]);
      for (int q = 0; q < 3; ++q)
        *reinterpret_cast<unsigned short*>(reinterpret_cast<char*>(b16 + q * 64 * 64) + tc::kmaj_off2(n, k, 64)) = h[q];
    }
    tc::fence_async_smem();
    __syncthreads();
    if (t == 0) {
      tc::fence_after();
      constexpr uint32_t idesc = tc::idesc_bf16(128, 64);
      const int ia[8] = {0, 0, 1, 0, 1, 2, 1, 2}, ib[8] = {0, 1, 0, 2, 1, 0, 2, 1};
      for (int s = 0; s < 4; ++s)
        for (int j = 0; j < 8; ++j)
          tc::mma_bf16(tmem, tc::kmaj_desc2(tc::smem_u32(a16 + ia[j] * 128 * 64) + 256 * s, 64),
                       tc::kmaj_desc2(tc::smem_u32(b16 + ib[j] * 64 * 64) + 256 * s, 64), idesc,
                       (s | j) ? 1u : 0u);
      tc::commit(&mbar);
    }
  } else if (t == 0) {
    constexpr uint32_t idesc = tc::idesc_tf32(128, 64);
    for (int s = 0; s < 8; ++s) {
      const uint64_t dah = tc::kmaj_desc(tc::smem_u32(ah) + 256 * s, 64);
      const uint64_t dal = tc::kmaj_desc(tc::smem_u32(al) + 256 * s, 64);
      const uint64_t dbh = tc::kmaj_desc(tc::smem_u32(bh) + 256 * s, 64);
      const uint64_t dbl = tc::kmaj_desc(tc::smem_u32(bl) + 256 * s, 64);
      tc::mma_tf32(tmem, dah, dbh, idesc, s > 0 ? 1u : 0u);
      if (split) {
        tc::mma_tf32(tmem, dah, dbl, idesc, 1u);
        tc::mma_tf32(tmem, dal, dbh, idesc, 1u);
      }
    }
    tc::commit(&mbar);
  }
  tc::mbar_wait(&mbar, 0);
  tc::fence_after();
  float v[32];
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  for (int half = 0; half < 2; ++half) {
    tc::tmem_ld32(tmem + lane_base + 32 * half, v);
#pragma unroll
    for (int i = 0; i < 32; ++i) D[t * 64 + 32 * half + i] = v[i];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free(tmem, 64);
}

void launch_tc_selftest(const float* A, const float* Bt, float* D, int split, cudaStream_t st) {
  const size_t smem = (128 * 64 * 2 + 64 * 64 * 2) * sizeof(float);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tc_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  MG_LAUNCH(tc_selftest_kernel<<<1, 128, smem, st>>>(A, Bt, D, split));
}

}  // namespace mg


namespace mg {

// ---------------------------------------------------------------------------
// Residual-field layers on the tensor cores (nrf.py:115-182), bf16x3.
//
// A CTA of 256 threads owns tiles of 128 points: warps w and w + 4 both serve
// the points of TMEM lane quarter w % 4 (one point per lane), warp w < 4 the
// hidden columns 0..31 and warp w >= 4 the columns 32..63.  Each 64-wide
// layer is one 128 x 64 x K GEMM on tcgen05 (kind::f16 with bf16 operands,
// float32 accumulator in TMEM) over a three-term bf16 split of both operands
// (x = x1 + x2 + x3, each the bf16 rounding of the remainder), issued by one
// thread as the 8 products a_i b_j with i + j <= 4: float32 precision (the
// 3xTF32 scheme measured ~7e-7 relative per product and missed the float64
// mirror on cancelling 20k-point bias sums).  The epilogue (bias, SiLU, the next
// layer's split operand as 8-byte stores into the K-major core-matrix tiles)
// runs per thread on its half row.  The weights
// of the four 64-wide layers stay in shared memory as K-major B operands: W^T
// (rows = outputs) for the forward, W (rows = inputs) for the backward chain.
// The Fourier features use sincospi(x) and angle doubling for the higher
// bands (2^b pi x, nrf.py:23-36).
// ---------------------------------------------------------------------------
namespace {
constexpr int kTM = 128;      // points per tile (MMA M)
constexpr int kTN = 64;       // hidden width (MMA N)
constexpr int kTE = 39;       // encoding width
constexpr int kTK0 = 48;      // padded layer-0 K (multiple of 16)
constexpr int kTBands = 6;
constexpr int kTThr = 256;
constexpr float kTOut = 0.099999994f;  // the largest float32 not above 0.1 (see mg_nrf.cu)

struct NrfTcSmem {
  unsigned short w[4][3][kTN * kTN];  // B operands (K-major core-matrix layout), three bf16 parts
  unsigned short a[3][kTM * kTN];     // A operand tile (K-major, K = 48 or 64), three bf16 parts
  float bias[4][kTN];
  float w4[kTN];
  float red[kTM];             // cross-half exchange (output-layer partial sums, encoding deltas)
  float red8x[kTM][12];
  float b4;
};

struct TcParams {
  const float* w[5];
  const float* b[5];
};

__device__ __forceinline__ float tc_sigmoid(float z) { return __frcp_rn(1.0f + __expf(-z)); }

// Four consecutive K values (k % 4 == 0) of one row, as three bf16 parts (8 bytes each).
__device__ __forceinline__ void put4(unsigned short* const (&part)[3], uint32_t off, float a, float b, float c,
                                     float d) {
  unsigned short h[4][3];
  tc::split_bf16x3(a, h[0][0], h[0][1], h[0][2]);
  tc::split_bf16x3(b, h[1][0], h[1][1], h[1][2]);
  tc::split_bf16x3(c, h[2][0], h[2][1], h[2][2]);
  tc::split_bf16x3(d, h[3][0], h[3][1], h[3][2]);
#pragma unroll
  for (int q = 0; q < 3; ++q)
    *reinterpret_cast<uint2*>(reinterpret_cast<char*>(part[q]) + off) =
        make_uint2((uint32_t)h[0][q] | ((uint32_t)h[1][q] << 16), (uint32_t)h[2][q] | ((uint32_t)h[3][q] << 16));
}

__device__ void tc_load_weights(NrfTcSmem& sm, const TcParams& P, bool transposed) {
  const int t = threadIdx.x, n = blockDim.x;
  for (int l = 0; l < 4; ++l) {
    const int kin = l == 0 ? kTE : kTN;
    unsigned short* const part[3] = {sm.w[l][0], sm.w[l][1], sm.w[l][2]};
    for (int e = t; e < kTN * kTN / 4; e += n) {
      const int r = e >> 4, c0 = (e & 15) * 4;  // B row r, K values c0..c0+3
      float v[4];
      if (transposed) {  // row r = output j, K = input i (< 48 for layer 0)
        if (l == 0 && c0 >= kTK0) continue;
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = c0 + q < kin ? P.w[l][(c0 + q) * kTN + r] : 0.f;
        put4(part, tc::kmaj_off2(r, c0, l == 0 ? kTK0 : kTN), v[0], v[1], v[2], v[3]);
      } else {  // row r = input i, K = output j
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = r < kin ? P.w[l][r * kTN + c0 + q] : 0.f;
        put4(part, tc::kmaj_off2(r, c0, kTN), v[0], v[1], v[2], v[3]);
      }
    }
  }
  for (int e = t; e < 4 * kTN; e += n) sm.bias[e >> 6][e & 63] = P.b[e >> 6][e & 63];
  for (int e = t; e < kTN; e += n) sm.w4[e] = P.w[4][e];
  if (t == 0) sm.b4 = P.b[4][0];
}

__device__ __forceinline__ void tc_issue(uint32_t tmem, const NrfTcSmem& sm, int l, int K, void* mbar) {
  constexpr uint32_t idesc = tc::idesc_bf16(kTM, kTN);
  constexpr int ia[8] = {0, 0, 1, 0, 1, 2, 1, 2}, ib[8] = {0, 1, 0, 2, 1, 0, 2, 1};  // i + j <= 3 (0-based)
  for (int s = 0; s < K / 16; ++s) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint64_t da = tc::kmaj_desc2(tc::smem_u32(sm.a[ia[j]]) + 256 * s, K);
      const uint64_t db = tc::kmaj_desc2(tc::smem_u32(sm.w[l][ib[j]]) + 256 * s, K);
      tc::mma_bf16(tmem, da, db, idesc, (s | j) ? 1u : 0u);
    }
  }
  tc::commit(mbar);
}

// A tile written by all threads -> visible to the tensor core -> one thread
// issues the layer -> everyone waits for the accumulator.
__device__ __forceinline__ void tc_run_layer(uint32_t tmem, NrfTcSmem& sm, int l, int K, uint64_t* mbar,
                                             uint32_t& phase) {
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    tc::fence_after();
    tc_issue(tmem, sm, l, K, mbar);
  }
  tc::mbar_wait(mbar, phase);
  phase ^= 1u;
  tc::fence_after();
}

// The Fourier features [20 H, 20 H + 20) of one point (nrf.py:23-36 column
// order: x, then per band sin(xyz), cos(xyz) at frequency 2^band pi; 39 + one
// zero pad) and their derivatives d feature / d x_c.  sin/cos(2^b pi x) come
// from sincospi(2^b0 x) (2^b0 x is exact) and angle doubling: <= 2e-6 from
// float64 at the top band -- closer to the reference's float64 than a float32
// sin of the rounded argument x * (2^b pi) (~1e-5 there).
template <int H>
__device__ __forceinline__ void tc_feats(const float (&xv)[3], float (&val)[20], float (&dval)[20]) {
#pragma unroll
  for (int i = 0; i < 20; ++i) val[i] = dval[i] = 0.f;
  if (H == 0) {
#pragma unroll
    for (int c = 0; c < 3; ++c) val[c] = xv[c], dval[c] = 1.f;
  }
  constexpr int b0 = H == 0 ? 0 : 2, b1 = H == 0 ? 2 : 5;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    float sn, cs;
    sincospif(xv[c] * (float)(1 << b0), &sn, &cs);
#pragma unroll
    for (int band = b0; band <= b1; ++band) {
      const float fr = 3.14159265358979323846f * (float)(1 << band);
      const int fs = 3 + 6 * band + c - 20 * H, fc = 6 + 6 * band + c - 20 * H;
      if (fs >= 0 && fs < 20) val[fs] = sn, dval[fs] = fr * cs;
      if (fc >= 0 && fc < 20) val[fc] = cs, dval[fc] = -fr * sn;
      const float s2 = 2.0f * sn * cs, c2 = fmaf(-2.0f * sn, sn, 1.0f);
      sn = s2, cs = c2;
    }
  }
}
// coordinate of feature f (f < 39)
__device__ __forceinline__ int tc_feat_coord(int f) { return f < 3 ? f : ((f - 3) % 6) % 3; }

__device__ __forceinline__ void ld_row32(const float* __restrict__ src, bool live, float (&v)[32]) {
  const float4* r = reinterpret_cast<const float4*>(src);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float4 q = live ? r[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    v[4 * i] = q.x, v[4 * i + 1] = q.y, v[4 * i + 2] = q.z, v[4 * i + 3] = q.w;
  }
}
__device__ __forceinline__ void st_row32(float* __restrict__ dst, const float (&v)[32]) {
  float4* r = reinterpret_cast<float4*>(dst);
#pragma unroll
  for (int i = 0; i < 8; ++i) r[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
}
}  // namespace

__global__ void __launch_bounds__(kTThr, 1) nrf_fwd_tc_kernel(const float* __restrict__ x, int64_t b, TcParams P,
                                                              float* __restrict__ pred_add,
                                                              float* __restrict__ r_out, float* __restrict__ t_out,
                                                              float* __restrict__ z_out) {
  extern __shared__ __align__(1024) unsigned char tc_dyn[];
  NrfTcSmem& sm = *reinterpret_cast<NrfTcSmem*>(tc_dyn);
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int row = 32 * (warp & 3) + lane, half = warp >> 2, c0 = 32 * half;
  tc_load_weights(sm, P, true);
  if (tid == 0) {
    tc::mbar_init(&mbar, 1);
    tc::fence_init();
  }
  if (warp == 0) tc::tmem_alloc(&tslot, kTN);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  const uint32_t taddr = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + c0;
  uint32_t phase = 0;
  unsigned short* const ap[3] = {sm.a[0], sm.a[1], sm.a[2]};
  const int64_t ntiles = (b + kTM - 1) / kTM;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t p = tile * kTM + row;
    const bool live = p < b;
    {
      float xv[3] = {0.f, 0.f, 0.f};
      if (live) xv[0] = x[3 * p], xv[1] = x[3 * p + 1], xv[2] = x[3 * p + 2];
      float e[20], de_unused[20];
      if (half)
        tc_feats<1>(xv, e, de_unused);
      else
        tc_feats<0>(xv, e, de_unused);
#pragma unroll
      for (int q = 0; q < 5; ++q)  // this half's 20 features, 4 per 8-byte store
        put4(ap, tc::kmaj_off2(row, 20 * half + 4 * q, kTK0), e[4 * q], e[4 * q + 1], e[4 * q + 2], e[4 * q + 3]);
      if (half) {  // K padding 40..47
        put4(ap, tc::kmaj_off2(row, 40, kTK0), 0.f, 0.f, 0.f, 0.f);
        put4(ap, tc::kmaj_off2(row, 44, kTK0), 0.f, 0.f, 0.f, 0.f);
      }
    }
    float z4 = 0.f;
#pragma unroll 1
    for (int l = 0; l < 4; ++l) {
      tc_run_layer(tmem, sm, l, l == 0 ? kTK0 : kTN, &mbar, phase);
      float v[32];
      tc::tmem_ld32(taddr, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] += sm.bias[l][c0 + i];
      if (z_out && live) st_row32(z_out + ((int64_t)l * b + p) * kTN + c0, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] *= tc_sigmoid(v[i]);
      if (l < 3) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          put4(ap, tc::kmaj_off2(row, c0 + 4 * q, kTN), v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) z4 = fmaf(sm.w4[c0 + i], v[i], z4);
      }
    }
    if (half) sm.red[row] = z4;
    __syncthreads();
    if (!half && live) {
      const float t = tanhf(sm.b4 + (z4 + sm.red[row]));
      const float r = kTOut * t;
      if (t_out) t_out[p] = t;
      if (r_out) r_out[p] = r;
      if (pred_add) pred_add[p] += r;
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free(tmem, kTN);
}

// Backward delta chain (nrf.py:147-182): d4 = u 0.1 (1 - t^2), dz3 = d4 w4
// silu'(z3), dz_{l-1} = (W_l dz_l) silu'(z_{l-1}) on the tensor cores,
// d_enc = W_0 dz_0, d_points through the sin/cos features.  Writes the same
// intermediates as nrf_bwd_kernel (dz, d4, SiLU(z) and the encoding rows)
// for the weight-gradient pass.
__global__ void __launch_bounds__(kTThr, 1) nrf_bwd_tc_kernel(const float* __restrict__ x, int64_t b, TcParams P,
                                                              const float* __restrict__ up,
                                                              const float* __restrict__ tin,
                                                              const float* __restrict__ z, float* __restrict__ dz,
                                                              float* __restrict__ d4g, float* __restrict__ dp,
                                                              float* __restrict__ hout,
                                                              float* __restrict__ encout) {
  extern __shared__ __align__(1024) unsigned char tc_dyn[];
  NrfTcSmem& sm = *reinterpret_cast<NrfTcSmem*>(tc_dyn);
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int row = 32 * (warp & 3) + lane, half = warp >> 2, c0 = 32 * half;
  tc_load_weights(sm, P, false);
  if (tid == 0) {
    tc::mbar_init(&mbar, 1);
    tc::fence_init();
  }
  if (warp == 0) tc::tmem_alloc(&tslot, kTN);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  const uint32_t taddr = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + c0;
  uint32_t phase = 0;
  unsigned short* const ap[3] = {sm.a[0], sm.a[1], sm.a[2]};
  const int64_t ntiles = (b + kTM - 1) / kTM;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t p = tile * kTM + row;
    const bool live = p < b;
    const int64_t pr = live ? p : 0;
    float d4 = 0.f;
    if (live) {
      const float t = tin[p];
      d4 = up[p] * kTOut * (1.0f - t * t);
      if (!half) d4g[p] = d4;
    }
    {  // layer 3 delta from the output layer (rank one)
      float zz[32], hv[32];
      ld_row32(z + ((int64_t)3 * b + pr) * kTN + c0, live, zz);
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float s = tc_sigmoid(zz[i]);
        hv[i] = zz[i] * s;
        zz[i] = d4 * sm.w4[c0 + i] * (s * (1.0f + zz[i] * (1.0f - s)));
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        put4(ap, tc::kmaj_off2(row, c0 + 4 * q, kTN), zz[4 * q], zz[4 * q + 1], zz[4 * q + 2], zz[4 * q + 3]);
      if (live) {
        st_row32(dz + ((int64_t)3 * b + p) * kTN + c0, zz);
        st_row32(hout + ((int64_t)3 * b + p) * kTN + c0, hv);
      }
    }
#pragma unroll 1
    for (int l = 3; l >= 1; --l) {  // dh_{l-1} = W_l dz_l, dz_{l-1} = dh_{l-1} silu'(z_{l-1})
      tc_run_layer(tmem, sm, l, kTN, &mbar, phase);
      float v[32], zz[32], hv[32];
      tc::tmem_ld32(taddr, v);
      ld_row32(z + ((int64_t)(l - 1) * b + pr) * kTN + c0, live, zz);
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float s = tc_sigmoid(zz[i]);
        hv[i] = zz[i] * s;
        v[i] *= s * (1.0f + zz[i] * (1.0f - s));
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        put4(ap, tc::kmaj_off2(row, c0 + 4 * q, kTN), v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      if (live) {
        st_row32(dz + ((int64_t)(l - 1) * b + p) * kTN + c0, v);
        st_row32(hout + ((int64_t)(l - 1) * b + p) * kTN + c0, hv);
      }
    }
    tc_run_layer(tmem, sm, 0, kTN, &mbar, phase);  // d_enc = W_0 dz_0 (B rows 39.. are zero)
    float de[32];
    tc::tmem_ld32(taddr, de);  // half 0: encoding deltas 0..31, half 1: 32..63 (39.. are 0)
    if (!half) {
#pragma unroll
      for (int i = 0; i < 12; ++i) sm.red8x[row][i] = de[20 + i];  // 20..31 belong to the upper half
    }
    __syncthreads();
    float dpart[3] = {0.f, 0.f, 0.f};
    if (live) {  // this half's features [20 half, 20 half + 20): encoding row + d_points share
      const float xv[3] = {x[3 * p], x[3 * p + 1], x[3 * p + 2]};
      float* er = encout + p * (kTE + 1) + 20 * half;
      float e[20], dv[20];
      if (half)
        tc_feats<1>(xv, e, dv);
      else
        tc_feats<0>(xv, e, dv);
#pragma unroll
      for (int k = 0; k < 20; ++k) {
        const int f = 20 * half + k;
        const float d = half ? (k < 12 ? sm.red8x[row][k] : de[k - 12]) : de[k];
        const float term = dv[k] * d;
        const int c = tc_feat_coord(f < kTE ? f : 0);
        dpart[0] += c == 0 ? term : 0.f;
        dpart[1] += c == 1 ? term : 0.f;
        dpart[2] += c == 2 ? term : 0.f;
      }
#pragma unroll
      for (int q = 0; q < 5; ++q)
        *reinterpret_cast<float4*>(er + 4 * q) = make_float4(e[4 * q], e[4 * q + 1], e[4 * q + 2], e[4 * q + 3]);
    }
    __syncthreads();  // the upper half's row copies are consumed
    if (half) {
      sm.red8x[row][0] = dpart[0];
      sm.red8x[row][1] = dpart[1];
      sm.red8x[row][2] = dpart[2];
    }
    __syncthreads();
    if (!half && live) {
#pragma unroll
      for (int c = 0; c < 3; ++c) dp[p * 3 + c] = dpart[c] + sm.red8x[row][c];
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_free(tmem, kTN);
}

static void tc_attrs() {
  static bool done = false;
  if (done) return;
  cudaFuncSetAttribute(nrf_fwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(NrfTcSmem));
  cudaFuncSetAttribute(nrf_bwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(NrfTcSmem));
  done = true;
}

static unsigned tc_grid(int64_t b) {
  const int64_t tiles = (b + kTM - 1) / kTM;
  const int64_t g = num_sms();
  return (unsigned)(tiles < g ? (tiles < 1 ? 1 : tiles) : g);
}

void launch_nrf_forward_tc(const float* x, int64_t b, const float* const* w, const float* const* bias,
                           float* pred_add, float* r_out, float* t_out, float* z_out, cudaStream_t st) {
  if (b <= 0) return;
  tc_attrs();
  TcParams P;
  for (int l = 0; l < 5; ++l) P.w[l] = w[l], P.b[l] = bias[l];
  MG_LAUNCH(nrf_fwd_tc_kernel<<<tc_grid(b), kTThr, sizeof(NrfTcSmem), st>>>(x, b, P, pred_add, r_out, t_out,
                                                                          z_out));
}

void launch_nrf_bwd_chain_tc(const float* x, int64_t b, const float* const* w, const float* const* bias,
                             const float* up, const float* t, const float* z, float* dz, float* d4, float* dp,
                             float* hout, float* enc, cudaStream_t st) {
  if (b <= 0) return;
  tc_attrs();
  TcParams P;
  for (int l = 0; l < 5; ++l) P.w[l] = w[l], P.b[l] = bias[l];
  MG_LAUNCH(nrf_bwd_tc_kernel<<<tc_grid(b), kTThr, sizeof(NrfTcSmem), st>>>(x, b, P, up, t, z, dz, d4, dp, hout,
                                                                          enc));
}

}  // namespace mg
