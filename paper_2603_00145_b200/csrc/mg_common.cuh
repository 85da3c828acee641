// mg_common.cuh -- shared device helpers for the B200 (sm_100a) Gaussian path.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define MG_WARP 32
#define MG_FULL 0xffffffffu

// Reference cutoff m <= 64 (_kernels.py:21).  Precisions are stored pre-scaled
// by kMScale = -0.5*log2(e), so m' = d^T P' d = -0.5*log2(e)*m and
// exp(-m/2) = 2^{m'}; the cutoff becomes m' >= kCutScaled.
#define MG_LOG2E 1.4426950408889634
static constexpr double kMScaleD = -0.5 * MG_LOG2E;
static constexpr float kMScale = (float)(-0.5 * MG_LOG2E);
static constexpr float kCutScaled = (float)(-32.0 * MG_LOG2E);  // = kMScale * 64

// ---------------------------------------------------------------------------
// Packed f32x2 arithmetic (sm_100a FFMA2/FMUL2/FADD2).  A scalar operand that
// is shared by both halves is passed as a float and ptxas encodes it as a
// broadcast (.F32) operand, so no duplicate register is needed.
// ---------------------------------------------------------------------------
// Packed pairs live in one 64-bit value so the register allocator keeps the
// halves in an aligned register pair (no re-pairing moves before FFMA2).
struct f2 {
  unsigned long long v;
};

__device__ __forceinline__ f2 mk2(float a, float b) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ f2 bc2(float a) { return mk2(a, a); }
__device__ __forceinline__ float lo(f2 a) {
  float x, y;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a.v));
  return x;
}
__device__ __forceinline__ float hi(f2 a) {
  float x, y;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a.v));
  return y;
}

__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  f2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d.v) : "l"(a.v), "l"(b.v), "l"(c.v));
  return d;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
  f2 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d.v) : "l"(a.v), "l"(b.v));
  return d;
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
  f2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d.v) : "l"(a.v), "l"(b.v));
  return d;
}
__device__ __forceinline__ f2 sub2(f2 a, f2 b) {
  f2 d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d.v) : "l"(a.v), "l"(b.v));
  return d;
}

// 2^x on the MUFU (SFU) pipe, flush-to-zero: one MUFU.EX2.
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Cutoff by flush-to-zero.  2^{m'} is scaled by kCutScale = 2^-79.83 with an
// FTZ multiply: the product is subnormal -- flushed to exactly 0 -- precisely
// when m' < -46.17, i.e. m > 64 (_kernels.py:21: the reference's skip), so the
// cutoff costs one packed FMUL2.FTZ per two pairs instead of a compare and a
// select per pair, and 2^{m'} itself keeps full precision (biasing the exponent
// argument instead lost ~3e-6 relative in the float32 add).  The weights that
// multiply the Gaussian factor carry the inverse scale kWeightScale ~ 1.08e24:
// the intensity alpha in the records (A.w) and the upstream in the point
// records (prec.w), so alpha' g' = alpha g and u' g' = u g.  Point upstreams
// must stay below ~3e14 in magnitude (the host layer checks).
static constexpr float kCutScale = 9.28205098304025e-25f;        // float(2^(-126 + 32 log2 e))
static constexpr double kWeightScaleD = 1.0773481010039219e24;  // 1 / kCutScale (float64)
static constexpr float kWeightScale = (float)kWeightScaleD;

__device__ __forceinline__ float mul_ftz(float a, float b) {
  float d;
  asm("mul.rn.ftz.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
  return d;
}
__device__ __forceinline__ f2 mul2_ftz(f2 a, f2 b) {
  f2 d;
  asm("mul.rn.ftz.f32x2 %0, %1, %2;" : "=l"(d.v) : "l"(a.v), "l"(b.v));
  return d;
}

// Cutoff-masked weight g' = 2^{m'} * kCutScale (0 when m > 64).
__device__ __forceinline__ float gauss_w(float ms) { return mul_ftz(ex2(ms), kCutScale); }
__device__ __forceinline__ f2 gauss_w2(f2 m) { return mul2_ftz(mk2(ex2(lo(m)), ex2(hi(m))), bc2(kCutScale)); }

// ---------------------------------------------------------------------------
// Warp reductions
// ---------------------------------------------------------------------------
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(MG_FULL, v, o);
  return v;
}

__device__ __forceinline__ int warp_excl_scan(int v, int lane, int* total) {
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(MG_FULL, x, o);
    if (lane >= o) x += y;
  }
  *total = __shfl_sync(MG_FULL, x, 31);
  return x - v;
}

// Transposed ("reduce-scatter") warp reduction of 32 per-lane values:
// afterwards lane l holds sum over lanes of v[l].  31 shuffles instead of 160.
__device__ __forceinline__ float warp_transpose_reduce32(float (&v)[32], int lane) {
#pragma unroll
  for (int half = 16; half >= 1; half >>= 1) {
    const bool upper = (lane & half) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      // keep the half of the values this lane is responsible for
      float send = upper ? v[i] : v[i + half];
      float keep = upper ? v[i + half] : v[i];
      float recv = __shfl_xor_sync(MG_FULL, send, half);
      v[i] = keep + recv;
    }
  }
  return v[0];
}

// ---------------------------------------------------------------------------
// Cell math, bit-exact with spatial.py:18-27 evaluated in float64.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int cell_of_d(double v, int g) {
  double half = (double)g / 2.0;
  double f = floor(__dmul_rn(__dadd_rn(v, 1.0), half));
  // clamp in floating point first so huge values do not overflow the int cast
  if (f < 0.0) f = 0.0;
  if (f > (double)(g - 1)) f = (double)(g - 1);
  return (int)f;
}

__device__ __forceinline__ int flat_cell(int ci, int cj, int ck, int g) { return (ci * g + cj) * g + ck; }

// Gaussian records, structure-of-arrays inside one float buffer of 12*N:
// A = float4[N] {mu.xyz, alpha} at 0, B = float4[N] {P'00,P'11,P'22,P'01} at
// 4N, C = float2[N] {P'02,P'12} at 8N, E = uint2[N] at 10N: the half-extents
// of the cutoff ellipsoid's axis box (three fp16, rounded up; +inf = no
// culling), read by the backward's candidate-window culling.  Warp-wide loads
// of consecutive records are fully coalesced (4 + 4 + 2 sectors per 32).
struct GaussSoA {
  const float4* A;
  const float4* B;
  const float2* C;
  const uint2* E;
};
struct GaussOut {
  float4* A;
  float4* B;
  float2* C;
  uint2* E;
};
inline GaussSoA gauss_soa(const float* base, int64_t n) {
  return GaussSoA{reinterpret_cast<const float4*>(base), reinterpret_cast<const float4*>(base + 4 * n),
                  reinterpret_cast<const float2*>(base + 8 * n), reinterpret_cast<const uint2*>(base + 10 * n)};
}
inline GaussOut gauss_out(float* base, int64_t n) {
  return GaussOut{reinterpret_cast<float4*>(base), reinterpret_cast<float4*>(base + 4 * n),
                  reinterpret_cast<float2*>(base + 8 * n), reinterpret_cast<uint2*>(base + 10 * n)};
}

// Host-side count of kernel launches issued by this library (all streams),
// read through mg_launch_count(); MG_LAUNCH bumps it at every launch site.
namespace mg {
long long& launch_counter();
}
#define MG_LAUNCH(...) (++::mg::launch_counter(), __VA_ARGS__)

// Device-side error codes (read by the host wrappers).
enum MgErr : int {
  MG_OK = 0,
  MG_ERR_DEGENERATE_QUAT = 1,
  MG_ERR_NONFINITE = 2,
};
