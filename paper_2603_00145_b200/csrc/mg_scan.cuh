// mg_scan.cuh -- single-pass device-wide exclusive scan (decoupled look-back)
// over a per-element functor, so a producer can scan counts and write its
// outputs at the scanned offsets in ONE kernel:
//   struct Op { __device__ int count(int64_t e) const;
//               __device__ void emit(int64_t e, int offset, int count) const; };
// Elements are visited in index order within a tile; every element gets
// emit(e, sum_{j<e} count(j), count(e)).
#pragma once
#include "mg_common.cuh"

namespace mg {

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

// Every tile publishes its aggregate (flag A) and then its inclusive prefix
// (flag P); a tile's exclusive prefix comes from a warp-parallel look-back
// over its predecessors.  Tile ids are handed out in launch order by an atomic
// ticket, so every predecessor is already running (forward progress).
constexpr unsigned long long kFlagA = 1ull << 32, kFlagP = 2ull << 32;

template <class Op>
__global__ void __launch_bounds__(kScanThreads) scan_lookback_op(const Op op, int64_t n,
                                                                 unsigned long long* __restrict__ state,
                                                                 int* __restrict__ ticket) {
  __shared__ int s_warp[kScanThreads / 32 + 1];
  __shared__ int s_tile, s_prefix;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1);
  __syncthreads();
  const int tile = s_tile;
  const int64_t base = (int64_t)tile * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int v[kScanItems];
  int sum = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    int64_t e = base + i;
    v[i] = e < n ? op.count(e) : 0;
    sum += v[i];
  }
  int tot;
  int off = block_excl_scan(sum, s_warp, &tot);
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {
    volatile unsigned long long* vs = state;
    if (tile == 0) {
      if (lane == 0) {
        vs[0] = kFlagP | (unsigned)tot;
        __threadfence();
        s_prefix = 0;
      }
    } else {
      if (lane == 0) {
        vs[tile] = kFlagA | (unsigned)tot;
        __threadfence();
      }
      int prefix = 0;
      int look = tile - 1;
      while (true) {
        const int t = look - lane;
        unsigned long long w = kFlagP;  // before tile 0: inclusive prefix 0
        if (t >= 0) {
          do {
            w = vs[t];
          } while ((w >> 32) == 0);
        }
        const unsigned pmask = __ballot_sync(MG_FULL, (w >> 32) == 2);
        const int first_p = pmask ? __ffs(pmask) - 1 : 32;  // lanes up to the first P contribute
        int val = (lane <= first_p) ? (int)(w & 0xffffffffu) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(MG_FULL, val, o);
        prefix += val;
        if (pmask) break;
        look -= 32;
      }
      if (lane == 0) {
        vs[tile] = kFlagP | (unsigned)(prefix + tot);
        __threadfence();
        s_prefix = prefix;
      }
    }
  }
  __syncthreads();
  off += s_prefix;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    int64_t e = base + i;
    if (e < n) op.emit(e, off, v[i]);
    off += v[i];
  }
}

inline size_t lookback_state_bytes(int64_t n) {
  int64_t tiles = (n + kScanTile - 1) / kScanTile;
  if (tiles < 1) tiles = 1;
  return (((size_t)tiles * 8 + 255) & ~(size_t)255) + 256;
}

// Enqueue the scan of n elements; ws >= lookback_state_bytes(n).
template <class Op>
void lookback_scan(const Op& op, int64_t n, void* ws, cudaStream_t st) {
  if (n <= 0) return;
  const int64_t tiles = (n + kScanTile - 1) / kScanTile;
  const size_t sb = ((size_t)tiles * 8 + 255) & ~(size_t)255;
  cudaMemsetAsync(ws, 0, sb + 4, st);
  MG_LAUNCH(scan_lookback_op<Op><<<(unsigned)tiles, kScanThreads, 0, st>>>(op, n, (unsigned long long*)ws,
                                                                          (int*)((char*)ws + sb)));
}

}  // namespace mg
