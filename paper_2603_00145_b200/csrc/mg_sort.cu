// mg_sort.cu -- device-wide exclusive scan, stable LSD radix sort of
// (uint32 key, int32 value) pairs, and CSR construction over G^3 cells.
//
// Replaces the stable argsort + bincount + cumsum of
// /root/reference/pkg/src/mgauss/spatial.py:46-66 (and the stable batch
// sort of train.py:390-397).  Stability (ties keep ascending input order)
// makes cell_indices bit-identical to numpy's argsort(kind="stable").
#include "mg_sort.cuh"
#include "mg_scan.cuh"

namespace mg {

// ---------------------------------------------------------------------------
// Exclusive scan (int32): the look-back scan of mg_scan.cuh over an array.
// ---------------------------------------------------------------------------
struct ArrayScanOp {
  const int* in;
  int* out;
  __device__ int count(int64_t e) const { return in[e]; }
  __device__ void emit(int64_t e, int off, int) const { out[e] = off; }
};

size_t scan_workspace_bytes(int64_t n) { return lookback_state_bytes(n); }

// out[i] = sum_{j<i} in[j]; out may alias in (each tile reads before it writes).
void excl_scan(const int* in, int* out, int64_t n, void* ws, cudaStream_t st) {
  lookback_scan(ArrayScanOp{in, out}, n, ws, st);
}

// ---------------------------------------------------------------------------
// Stable LSD radix sort, digits of <= 10 bits (2 passes up to 20-bit keys).
// ---------------------------------------------------------------------------
constexpr int kRsThreads = 256;
constexpr int kRsRounds = 8;
constexpr int kRsTile = kRsThreads * kRsRounds;  // 2048 elements per block
constexpr int kRsWarps = kRsThreads / 32;

template <int DB>
__global__ void __launch_bounds__(kRsThreads) rs_hist(const uint32_t* __restrict__ keys, int64_t n, int shift,
                                                      int* __restrict__ hist, int nblocks) {
  constexpr int NB = 1 << DB;
  __shared__ int cnt[NB];
  for (int d = threadIdx.x; d < NB; d += kRsThreads) cnt[d] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kRsTile;
#pragma unroll
  for (int r = 0; r < kRsRounds; ++r) {
    int64_t e = base + r * kRsThreads + threadIdx.x;
    if (e < n) atomicAdd(&cnt[(keys[e] >> shift) & (NB - 1)], 1);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < NB; d += kRsThreads) hist[d * nblocks + blockIdx.x] = cnt[d];
}

template <int DB>
__global__ void __launch_bounds__(kRsThreads) rs_scatter(const uint32_t* __restrict__ kin,
                                                         const int* __restrict__ vin, uint32_t* __restrict__ kout,
                                                         int* __restrict__ vout, int64_t n, int shift,
                                                         const int* __restrict__ offs, int nblocks) {
  constexpr int NB = 1 << DB;
  __shared__ int s_base[NB];
  __shared__ int s_wcnt[kRsWarps][NB];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int d = threadIdx.x; d < NB; d += kRsThreads) {
    s_base[d] = offs[d * nblocks + blockIdx.x];
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) s_wcnt[w][d] = 0;
  }
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kRsTile;
  const unsigned lt = (1u << lane) - 1u;
  for (int r = 0; r < kRsRounds; ++r) {
    int64_t e = base + r * kRsThreads + threadIdx.x;
    bool valid = e < n;
    uint32_t k = valid ? kin[e] : 0u;
    int v = valid ? vin[e] : 0;
    int d = valid ? (int)((k >> shift) & (NB - 1)) : NB;  // NB = sentinel digit
    unsigned peers = __match_any_sync(MG_FULL, d);
    int rank = __popc(peers & lt);
    if (valid && rank == 0) s_wcnt[warp][d] = __popc(peers);
    __syncthreads();
    for (int dgt = threadIdx.x; dgt < NB; dgt += kRsThreads) {
      // digit-major prefix across warps, in warp order (stable)
      int run = s_base[dgt];
#pragma unroll
      for (int w = 0; w < kRsWarps; ++w) {
        int c = s_wcnt[w][dgt];
        s_wcnt[w][dgt] = run;
        run += c;
      }
      s_base[dgt] = run;
    }
    __syncthreads();
    if (valid) {
      int pos = s_wcnt[warp][d] + rank;
      kout[pos] = k;
      vout[pos] = v;
    }
    __syncthreads();
    for (int dgt = threadIdx.x; dgt < NB; dgt += kRsThreads) {
#pragma unroll
      for (int w = 0; w < kRsWarps; ++w) s_wcnt[w][dgt] = 0;
    }
    __syncthreads();
  }
}

__global__ void iota_kernel(int* __restrict__ v, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (int)i;
}

static inline size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

size_t radix_workspace_bytes(int64_t n) {
  int64_t nb = (n + kRsTile - 1) / kRsTile;
  if (nb < 1) nb = 1;
  const size_t bins = (size_t)1 << 10;
  return 2 * align256((size_t)n * 4) + 2 * align256((size_t)n * 4) + 2 * align256(bins * nb * 4) +
         scan_workspace_bytes((int64_t)bins * nb);
}

template <int DB>
static void rs_pass(const uint32_t* kin, const int* vin, uint32_t* ko, int* vo, int64_t n, int shift, int* hist,
                    int* offs, int64_t nb, void* sws, cudaStream_t st) {
  MG_LAUNCH(rs_hist<DB><<<(unsigned)nb, kRsThreads, 0, st>>>(kin, n, shift, hist, (int)nb));
  excl_scan(hist, offs, ((int64_t)1 << DB) * nb, sws, st);
  MG_LAUNCH(rs_scatter<DB><<<(unsigned)nb, kRsThreads, 0, st>>>(kin, vin, ko, vo, n, shift, offs, (int)nb));
}

// Sorts (keys, values := 0..n-1) by the low `bits` bits of keys, stably.
// Results go to keys_out / vals_out.
void radix_sort_pairs(const uint32_t* keys_in, uint32_t* keys_out, int* vals_out, int64_t n, int bits, void* ws,
                      cudaStream_t st) {
  if (n <= 0) return;
  int64_t nb = (n + kRsTile - 1) / kRsTile;
  char* w = (char*)ws;
  uint32_t* kA = (uint32_t*)w;
  w += align256((size_t)n * 4);
  uint32_t* kB = (uint32_t*)w;
  w += align256((size_t)n * 4);
  int* vA = (int*)w;
  w += align256((size_t)n * 4);
  int* vB = (int*)w;
  w += align256((size_t)n * 4);
  int* hist = (int*)w;
  w += align256((size_t)1024 * nb * 4);
  int* offs = (int*)w;
  w += align256((size_t)1024 * nb * 4);
  void* sws = w;
  // fewest passes with digits of <= 8 bits (cheaper scatter prefix than 10-bit digits)
  int passes = (bits + 7) / 8;
  if (passes < 1) passes = 1;
  const int db = (bits + passes - 1) / passes;
  MG_LAUNCH(iota_kernel<<<(unsigned)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096), 256, 0, st>>>(vA, n));
  const uint32_t* kin = keys_in;
  const int* vin = vA;
  for (int p = 0; p < passes; ++p) {
    bool last = p == passes - 1;
    uint32_t* ko = last ? keys_out : ((p & 1) ? kA : kB);
    int* vo = last ? vals_out : ((p & 1) ? vA : vB);
    const int shift = db * p;
    switch (db) {
      case 1: case 2: case 3: case 4: case 5: case 6:
        rs_pass<6>(kin, vin, ko, vo, n, shift, hist, offs, nb, sws, st);
        break;
      case 7: case 8:
        rs_pass<8>(kin, vin, ko, vo, n, shift, hist, offs, nb, sws, st);
        break;
      default:
        rs_pass<10>(kin, vin, ko, vo, n, shift, hist, offs, nb, sws, st);
        break;
    }
    kin = ko;
    vin = vo;
  }
}

// ---------------------------------------------------------------------------
// CSR starts (ncell + 1) from sorted keys: starts[c] = #keys < c.
// ---------------------------------------------------------------------------
__global__ void csr_hist(const uint32_t* __restrict__ keys, int64_t n, int* __restrict__ cnt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[keys[i]], 1);
}

size_t csr_workspace_bytes(int64_t ncell) { return scan_workspace_bytes(ncell + 1); }

void csr_starts(const uint32_t* keys, int64_t n, int64_t ncell, int* starts, void* ws, cudaStream_t st) {
  cudaMemsetAsync(starts, 0, sizeof(int) * (size_t)(ncell + 1), st);
  if (n > 0) {
    int64_t blocks = (n + 255) / 256;
    if (blocks > 8192) blocks = 8192;
    MG_LAUNCH(csr_hist<<<(unsigned)blocks, 256, 0, st>>>(keys, n, starts));
  }
  excl_scan(starts, starts, ncell + 1, ws, st);
}

// ---------------------------------------------------------------------------
// Counting sort for dense cell keys in [0, ncell): the CSR is the exclusive
// scan of the per-cell counts, elements scatter to starts[key] + (atomic slot),
// and a rank pass restores stable order inside each cell (rank = # smaller
// original indices in the cell, O(cell size) per element).  Output identical
// to the stable LSD radix sort, in 4 kernels + 1 memset instead of 3 passes of
// hist/scan/scatter plus a separate CSR build.  Cost is sum(cell size^2): a
// pathological single huge cell is slow (still correct).
// ---------------------------------------------------------------------------
__global__ void cs_count(const uint32_t* __restrict__ keys, int64_t n, int* __restrict__ cnt,
                         int* __restrict__ slot) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    slot[i] = atomicAdd(&cnt[keys[i]], 1);
}

__global__ void cs_scatter(const uint32_t* __restrict__ keys, const int* __restrict__ slot, int64_t n,
                           const int* __restrict__ starts, uint32_t* __restrict__ keys_out, int* __restrict__ tmp) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = keys[i];
    const int p = starts[k] + slot[i];
    keys_out[p] = k;
    tmp[p] = (int)i;
  }
}

__global__ void cs_rank(const uint32_t* __restrict__ keys_out, const int* __restrict__ tmp, int64_t n,
                        const int* __restrict__ starts, int* __restrict__ vals_out) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = keys_out[p];
    const int s = starts[k], e = starts[k + 1];
    const int v = tmp[p];
    int r = 0;
    for (int q = s; q < e; ++q) r += tmp[q] < v;
    vals_out[s + r] = v;
  }
}

size_t counting_workspace_bytes(int64_t n, int64_t ncell) {
  const size_t a = (((size_t)(n > 0 ? n : 1) * 4) + 255) & ~(size_t)255;
  return 2 * a + scan_workspace_bytes(ncell + 1);
}

void counting_sort_pairs(const uint32_t* keys, uint32_t* keys_out, int* vals_out, int* starts, int64_t n,
                         int64_t ncell, void* ws, cudaStream_t st) {
  cudaMemsetAsync(starts, 0, sizeof(int) * (size_t)(ncell + 1), st);
  const size_t a = (((size_t)(n > 0 ? n : 1) * 4) + 255) & ~(size_t)255;
  int* slot = (int*)ws;
  int* tmp = (int*)((char*)ws + a);
  void* sws = (char*)ws + 2 * a;
  const unsigned blocks = (unsigned)((n + 255) / 256 < 8192 ? (n + 255) / 256 : 8192);
  if (n > 0) MG_LAUNCH(cs_count<<<blocks, 256, 0, st>>>(keys, n, starts, slot));
  excl_scan(starts, starts, ncell + 1, sws, st);
  if (n > 0) {
    MG_LAUNCH(cs_scatter<<<blocks, 256, 0, st>>>(keys, slot, n, starts, keys_out, tmp));
    MG_LAUNCH(cs_rank<<<blocks, 256, 0, st>>>(keys_out, tmp, n, starts, vals_out));
  }
}

int bits_for(int64_t maxval) {
  int b = 0;
  while (b < 32 && ((int64_t)1 << b) <= maxval) ++b;
  return b;
}

}  // namespace mg
