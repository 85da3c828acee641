// mg_sort.cu -- device-wide exclusive scan, stable LSD radix sort of
// (uint32 key, int32 value) pairs, and CSR construction over G^3 cells.
//
// Replaces the stable argsort + bincount + cumsum of
// /root/reference/pkg/src/mgauss/spatial.py:46-66 (and the stable batch
// sort of train.py:390-397).  Stability (ties keep ascending input order)
// makes cell_indices bit-identical to numpy's argsort(kind="stable").
#include "mg_sort.cuh"

namespace mg {

// ---------------------------------------------------------------------------
// Exclusive scan (int32), 3-phase, recursive over block sums.
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;  // 2048

__device__ __forceinline__ int block_excl_scan(int v, int* s_warp, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int wt;
  int x = warp_excl_scan(v, lane, &wt);
  if (lane == 0) s_warp[warp] = wt;
  __syncthreads();
  if (warp == 0) {
    int t = lane < (kScanThreads / 32) ? s_warp[lane] : 0;
    int tt;
    int e = warp_excl_scan(t, lane, &tt);
    if (lane < (kScanThreads / 32)) s_warp[lane] = e;
    if (lane == 0) s_warp[kScanThreads / 32] = tt;
  }
  __syncthreads();
  int r = x + s_warp[warp];
  *total = s_warp[kScanThreads / 32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kScanThreads) scan_tiles(const int* __restrict__ in, int* __restrict__ out,
                                                           int64_t n, int* __restrict__ tile_sums) {
  __shared__ int s_warp[kScanThreads / 32 + 1];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int v[kScanItems];
  int sum = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    int64_t e = base + i;
    v[i] = e < n ? in[e] : 0;
    sum += v[i];
  }
  int tot;
  int off = block_excl_scan(sum, s_warp, &tot);
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    int64_t e = base + i;
    if (e < n) out[e] = off;
    off += v[i];
  }
  if (threadIdx.x == 0 && tile_sums) tile_sums[blockIdx.x] = tot;
}

__global__ void scan_add(int* __restrict__ out, int64_t n, const int* __restrict__ tile_offs) {
  const int64_t e = (int64_t)blockIdx.x * kScanTile + threadIdx.x;
  const int add = tile_offs[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    int64_t k = e + (int64_t)i * kScanThreads;
    if (k < n) out[k] += add;
  }
}

size_t scan_workspace_bytes(int64_t n) {
  size_t b = 0;
  while (n > kScanTile) {
    int64_t tiles = (n + kScanTile - 1) / kScanTile;
    b += ((size_t)tiles * 2 * sizeof(int) + 255) & ~(size_t)255;
    n = tiles;
  }
  return b + 256;
}

// out[i] = sum_{j<i} in[j]; out may alias in.  Writes total to *total_dev if given.
void excl_scan(const int* in, int* out, int64_t n, void* ws, cudaStream_t st) {
  if (n <= 0) return;
  int64_t tiles = (n + kScanTile - 1) / kScanTile;
  if (tiles == 1) {
    MG_LAUNCH(scan_tiles<<<1, kScanThreads, 0, st>>>(in, out, n, nullptr));
    return;
  }
  int* sums = (int*)ws;
  int* offs = sums + tiles;
  size_t used = ((size_t)tiles * 2 * sizeof(int) + 255) & ~(size_t)255;
  MG_LAUNCH(scan_tiles<<<(unsigned)tiles, kScanThreads, 0, st>>>(in, out, n, sums));
  excl_scan(sums, offs, tiles, (char*)ws + used, st);
  MG_LAUNCH(scan_add<<<(unsigned)tiles, kScanThreads, 0, st>>>(out, n, offs));
}

// ---------------------------------------------------------------------------
// Stable LSD radix sort, 8-bit digits.
// ---------------------------------------------------------------------------
constexpr int kRsThreads = 256;
constexpr int kRsRounds = 8;
constexpr int kRsTile = kRsThreads * kRsRounds;  // 2048 elements per block
constexpr int kRsWarps = kRsThreads / 32;

__global__ void __launch_bounds__(kRsThreads) rs_hist(const uint32_t* __restrict__ keys, int64_t n, int shift,
                                                      int* __restrict__ hist, int nblocks) {
  __shared__ int cnt[256];
  cnt[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kRsTile;
#pragma unroll
  for (int r = 0; r < kRsRounds; ++r) {
    int64_t e = base + r * kRsThreads + threadIdx.x;
    if (e < n) atomicAdd(&cnt[(keys[e] >> shift) & 255u], 1);
  }
  __syncthreads();
  hist[threadIdx.x * nblocks + blockIdx.x] = cnt[threadIdx.x];
}

__global__ void __launch_bounds__(kRsThreads) rs_scatter(const uint32_t* __restrict__ kin,
                                                         const int* __restrict__ vin, uint32_t* __restrict__ kout,
                                                         int* __restrict__ vout, int64_t n, int shift,
                                                         const int* __restrict__ offs, int nblocks) {
  __shared__ int s_base[256];
  __shared__ int s_wcnt[kRsWarps][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  s_base[threadIdx.x] = offs[threadIdx.x * nblocks + blockIdx.x];
#pragma unroll
  for (int w = 0; w < kRsWarps; ++w) s_wcnt[w][threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kRsTile;
  const unsigned lt = (1u << lane) - 1u;
  for (int r = 0; r < kRsRounds; ++r) {
    int64_t e = base + r * kRsThreads + threadIdx.x;
    bool valid = e < n;
    uint32_t k = valid ? kin[e] : 0u;
    int v = valid ? vin[e] : 0;
    int d = valid ? (int)((k >> shift) & 255u) : 256;  // 256 = sentinel digit
    unsigned peers = __match_any_sync(MG_FULL, d);
    int rank = __popc(peers & lt);
    if (valid && rank == 0) s_wcnt[warp][d] = __popc(peers);
    __syncthreads();
    {
      // digit-major prefix across warps, in warp order (stable)
      int dgt = threadIdx.x;
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
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) s_wcnt[w][threadIdx.x] = 0;
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
  return 2 * align256((size_t)n * 4) + 2 * align256((size_t)n * 4) + 2 * align256((size_t)256 * nb * 4) +
         scan_workspace_bytes(256 * nb);
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
  w += align256((size_t)256 * nb * 4);
  int* offs = (int*)w;
  w += align256((size_t)256 * nb * 4);
  void* sws = w;
  int passes = (bits + 7) / 8;
  if (passes < 1) passes = 1;
  MG_LAUNCH(iota_kernel<<<(unsigned)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096), 256, 0, st>>>(vA, n));
  const uint32_t* kin = keys_in;
  const int* vin = vA;
  for (int p = 0; p < passes; ++p) {
    bool last = p == passes - 1;
    uint32_t* ko = last ? keys_out : ((p & 1) ? kA : kB);
    int* vo = last ? vals_out : ((p & 1) ? vA : vB);
    MG_LAUNCH(rs_hist<<<(unsigned)nb, kRsThreads, 0, st>>>(kin, n, 8 * p, hist, (int)nb));
    excl_scan(hist, offs, 256 * nb, sws, st);
    MG_LAUNCH(rs_scatter<<<(unsigned)nb, kRsThreads, 0, st>>>(kin, vin, ko, vo, n, 8 * p, offs, (int)nb));
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

int bits_for(int64_t maxval) {
  int b = 0;
  while (b < 32 && ((int64_t)1 << b) <= maxval) ++b;
  return b;
}

}  // namespace mg
