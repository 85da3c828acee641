// mg_volume.cu -- inference-time sampling of the Gaussian field on a dense,
// node-inclusive voxel grid (render.py:357-408: grid_coordinates +
// sample_volume, clip to [0, 1]).
//
// Voxel (i, j, k) sits at lo + i*spacing (float64, numpy order of
// operations).  Along each axis the voxels of one partition cell form a
// contiguous run, so a work item is a box of voxels that all share one
// cell -- and therefore one exact candidate set.  A warp owns an item:
// lanes hold voxels (V per lane, packed in f32x2), the candidate Gaussians
// stream through warp-uniform (broadcast) loads.  Slabs [i0, i1) of axis 0
// are independent, which is how inference shards across GPUs.
#include "mg_render.cuh"
#include "mg_sort.cuh"

namespace mg {

// Per-axis voxel coordinate (render.py:357-376).
__device__ __forceinline__ double axis_coord(int i, int n, double lo, double hi, double sp) {
  if (n == 1) return __dmul_rn(0.5, __dadd_rn(lo, hi));
  return __dadd_rn(lo, __dmul_rn((double)i, sp));
}

// axis a voxels [v0, v1): cell per voxel and "starts a run" flags.
__global__ void axis_cells_kernel(int n_all, int v0, int v1, double lo, double hi, double sp, int g,
                                  int* __restrict__ cells, int* __restrict__ flags) {
  int n = v1 - v0;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    int c = cell_of_d(axis_coord(v0 + t, n_all, lo, hi, sp), g);
    int cp = t > 0 ? cell_of_d(axis_coord(v0 + t - 1, n_all, lo, hi, sp), g) : -1;
    cells[t] = c;
    flags[t] = (c != cp) ? 1 : 0;
  }
}

__global__ void axis_runs_kernel(const int* __restrict__ cells, const int* __restrict__ flags,
                                 const int* __restrict__ scan, int n, int* __restrict__ run_start,
                                 int* __restrict__ run_cell, int* __restrict__ nruns) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    if (flags[t]) {
      run_start[scan[t]] = t;
      run_cell[scan[t]] = cells[t];
    }
    if (t == n - 1) {
      int nr = scan[t] + flags[t];
      *nruns = nr;
      run_start[nr] = n;  // sentinel
    }
  }
}

struct VolAxes {
  const int* rs[3];  // run starts (relative to axis origin), with sentinel
  const int* rc[3];  // run cells
  const int* nr;     // nruns[3]
  int v0[3];         // axis origins (slab offset on axis 0)
  int n[3];          // total voxels per axis
  double lo[3], hi[3], sp[3];
};

constexpr int kVolWarps = 4;

template <int V>
__device__ __forceinline__ void vol_chunk(const GaussSoA& grec, const int* __restrict__ gstart, int g,
                                          int r, const VolAxes& ax, int bx0, int by0, int bz0, int nbx, int nby,
                                          int nbz, int cell, int l0, int nvox, const float* __restrict__ residual,
                                          float* __restrict__ out, int64_t slab_i0, int lane) {
  constexpr int VP = V / 2;
  f2 px[VP], py[VP], pz[VP], acc[VP];
  float cx[V], cy[V], cz[V];
  int vid[V];
  const int nyz = nby * nbz;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    int l = l0 + lane + 32 * v;
    int lc = l < nvox ? l : 0;
    int bx = lc / nyz, rem = lc - bx * nyz, by = rem / nbz, bz = rem - by * nbz;
    int i = bx0 + bx, j = by0 + by, k = bz0 + bz;
    float x = (float)axis_coord(ax.v0[0] + i, ax.n[0], ax.lo[0], ax.hi[0], ax.sp[0]);
    float y = (float)axis_coord(j, ax.n[1], ax.lo[1], ax.hi[1], ax.sp[1]);
    float z = (float)axis_coord(k, ax.n[2], ax.lo[2], ax.hi[2], ax.sp[2]);
    vid[v] = l < nvox ? ((i * ax.n[1] + j) * ax.n[2] + k) : -1;
    cx[v] = x;
    cy[v] = y;
    cz[v] = z;
  }
#pragma unroll
  for (int q = 0; q < VP; ++q) {
    px[q] = mk2(cx[2 * q], cx[2 * q + 1]);
    py[q] = mk2(cy[2 * q], cy[2 * q + 1]);
    pz[q] = mk2(cz[2 * q], cz[2 * q + 1]);
  }
#pragma unroll
  for (int q = 0; q < VP; ++q) acc[q] = bc2(0.f);
  // candidate Gaussians: clipped (2r+1)^2 columns x k-window, warp-uniform walk
  int ck = cell % g, t = cell / g, cj = t % g, ci = t / g;
  int ilo = max(ci - r, 0), ihi = min(ci + r, g - 1), jlo = max(cj - r, 0), jhi = min(cj + r, g - 1);
  int klo = max(ck - r, 0), khi = min(ck + r, g - 1);
  for (int ii = ilo; ii <= ihi; ++ii) {
    for (int jj = jlo; jj <= jhi; ++jj) {
      int base = (ii * g + jj) * g;
      int a = __ldg(gstart + base + klo), b = __ldg(gstart + base + khi + 1);
      for (int gi = a; gi < b; ++gi) {
        const float4 A = __ldg(grec.A + gi), B = __ldg(grec.B + gi);
        const float2 C = __ldg(grec.C + gi);
        const float a01 = 2.f * B.w, a02 = 2.f * C.x, a12 = 2.f * C.y;
#pragma unroll
        for (int q = 0; q < VP; ++q) {
          f2 dx = sub2(px[q], bc2(A.x)), dy = sub2(py[q], bc2(A.y)), dz = sub2(pz[q], bc2(A.z));
          f2 t1 = fma2(bc2(a02), dz, fma2(bc2(a01), dy, mul2(bc2(B.x), dx)));
          f2 m = mul2(dx, t1);
          f2 t2 = fma2(bc2(a12), dz, mul2(bc2(B.y), dy));
          m = fma2(dy, t2, m);
          m = fma2(dz, mul2(bc2(B.z), dz), m);
          acc[q] = fma2(bc2(A.w), gauss_w2(m), acc[q]);
        }
      }
    }
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
    if (vid[v] >= 0) {
      float val = (v & 1) ? hi(acc[v / 2]) : lo(acc[v / 2]);
      int64_t o = (int64_t)vid[v];
      if (residual) val += residual[o];
      val = fminf(fmaxf(val, 0.f), 1.f);
      out[o] = val;
    }
  }
}

__global__ void __launch_bounds__(kVolWarps * 32) volume_kernel(const GaussSoA grec,
                                                                const int* __restrict__ gstart, int g, int r,
                                                                VolAxes ax, const float* __restrict__ residual,
                                                                float* __restrict__ out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nrx = ax.nr[0], nry = ax.nr[1], nrz = ax.nr[2];
  const int64_t nitems = (int64_t)nrx * nry * nrz;
  for (int64_t it = (int64_t)blockIdx.x * kVolWarps + warp; it < nitems; it += (int64_t)gridDim.x * kVolWarps) {
    int rz = (int)(it % nrz);
    int64_t t = it / nrz;
    int ry = (int)(t % nry);
    int rx = (int)(t / nry);
    int bx0 = ax.rs[0][rx], nbx = ax.rs[0][rx + 1] - bx0;
    int by0 = ax.rs[1][ry], nby = ax.rs[1][ry + 1] - by0;
    int bz0 = ax.rs[2][rz], nbz = ax.rs[2][rz + 1] - bz0;
    int cell = flat_cell(ax.rc[0][rx], ax.rc[1][ry], ax.rc[2][rz], g);
    int nvox = nbx * nby * nbz;
    if (nvox <= 64) {
      vol_chunk<2>(grec, gstart, g, r, ax, bx0, by0, bz0, nbx, nby, nbz, cell, 0, nvox, residual, out, 0, lane);
    } else {
      for (int l0 = 0; l0 < nvox; l0 += 128)
        vol_chunk<4>(grec, gstart, g, r, ax, bx0, by0, bz0, nbx, nby, nbz, cell, l0, nvox, residual, out, 0, lane);
    }
  }
}

// ---------------------------------------------------------------------------
// Tiled variant (dense inference): a block owns 2x2x2 voxel runs (8 cells,
// one warp each).  The union of their candidate windows -- at most
// (2 + 2r)^2 columns, each ONE contiguous CSR segment over the union
// k-range -- is staged in shared memory once per tile with cp.async, with a
// per-column table of cell starts; each warp then walks exactly its own
// cell's window from shared memory (broadcast LDS, no L2 round trips).  A
// tile whose union exceeds the staging capacity falls back to vol_chunk.
// ---------------------------------------------------------------------------
#ifndef MG_VOL_TILE
#define MG_VOL_TILE 1
#endif

#ifndef MG_VOL_TZ
#define MG_VOL_TZ 6  // runs per tile along k: 2 x 2 x 6 cells over 12 warps, 2 CTAs (2 x 104 KB) per SM
                     // (2 x 2 x 4 over 8 warps: 130 ms at C5; this shape: 116 ms)
#endif
#ifndef MG_VOL_FD
#define MG_VOL_FD 0  // forward-differencing cell pairs: 108 -> 115 ms at C5 (one pair per warp per tile: end-of-tile imbalance)
#endif
#ifndef MG_VOL_LPT
#define MG_VOL_LPT 1
#endif
#ifndef MG_VOL_WARPS
#define MG_VOL_WARPS 12  // warps per tile CTA; the tile's 2 x 2 x TZ cells are dealt round-robin
#endif
constexpr int kTileTZ = MG_VOL_TZ;
constexpr int kVolTileWarps = MG_VOL_WARPS;
// staged Gaussians per tile: the (2 + 2r)^2 x (TZ + 2r) union at one Gaussian per cell (r = 5), rounded up
constexpr int kTileCap = kTileTZ == 2 ? 1792 : (kTileTZ == 4 ? 2048 : ((144 * (kTileTZ + 10) + 63) / 64) * 64);
constexpr int kTileCols = 144;   // union columns ((2 + 2r)^2 at r = 5)
constexpr int kTileK = kTileTZ + 12 > 16 ? kTileTZ + 12 : 16;  // union k-cells + 1 (table width)

struct VolTileSmem {
  float4 A[kTileCap];
  float4 B[kTileCap];
  float2 C[kTileCap];
  int off[kTileCols][kTileK];  // absolute CSR index of union cell (column, KZ0 + k)
  int sb[kTileCols + 1];       // staged base of each column
  int geom[8];                 // UI0, UJ0, KZ0, ni, nj, nk, total, ok
  int order[4 * kTileTZ];      // the tile's cells, most voxel slots first (LPT hand-out)
  int next;                    // hand-out counter
};

template <int V>
__device__ __forceinline__ void vol_chunk_tile(const VolTileSmem& sm, int g, int r, const VolAxes& ax, int bx0,
                                               int by0, int bz0, int nbx, int nby, int nbz, int cell, int l0,
                                               int nvox, const float* __restrict__ residual,
                                               float* __restrict__ out, int lane) {
  constexpr int VP = V / 2;
  f2 px[VP], py[VP], pz[VP], acc[VP];
  float cx[V], cy[V], cz[V];
  int vid[V];
  const int nyz = nby * nbz;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    int l = l0 + lane + 32 * v;
    int lc = l < nvox ? l : 0;
    int bx = lc / nyz, rem = lc - bx * nyz, by = rem / nbz, bz = rem - by * nbz;
    int i = bx0 + bx, j = by0 + by, k = bz0 + bz;
    cx[v] = (float)axis_coord(ax.v0[0] + i, ax.n[0], ax.lo[0], ax.hi[0], ax.sp[0]);
    cy[v] = (float)axis_coord(j, ax.n[1], ax.lo[1], ax.hi[1], ax.sp[1]);
    cz[v] = (float)axis_coord(k, ax.n[2], ax.lo[2], ax.hi[2], ax.sp[2]);
    vid[v] = l < nvox ? ((i * ax.n[1] + j) * ax.n[2] + k) : -1;
  }
#pragma unroll
  for (int q = 0; q < VP; ++q) {
    px[q] = mk2(cx[2 * q], cx[2 * q + 1]);
    py[q] = mk2(cy[2 * q], cy[2 * q + 1]);
    pz[q] = mk2(cz[2 * q], cz[2 * q + 1]);
    acc[q] = bc2(0.f);
  }
  const int UI0 = sm.geom[0], UJ0 = sm.geom[1], KZ0 = sm.geom[2], nj = sm.geom[4];
  int ck = cell % g, t = cell / g, cj = t % g, ci = t / g;
  int ilo = max(ci - r, 0), ihi = min(ci + r, g - 1), jlo = max(cj - r, 0), jhi = min(cj + r, g - 1);
  const int klo = max(ck - r, 0) - KZ0, khi = min(ck + r, g - 1) - KZ0 + 1;
  for (int ii = ilo; ii <= ihi; ++ii) {
    for (int jj = jlo; jj <= jhi; ++jj) {
      const int c = (ii - UI0) * nj + (jj - UJ0);
      const int o0 = sm.off[c][0];
      const int a = sm.sb[c] + sm.off[c][klo] - o0, b = sm.sb[c] + sm.off[c][khi] - o0;
      for (int gi = a; gi < b; ++gi) {
        const float4 A = sm.A[gi], B = sm.B[gi];
        const float2 C = sm.C[gi];
        const float a01 = B.w, a02 = C.x, a12 = C.y;  // staged pre-doubled
#pragma unroll
        for (int q = 0; q < VP; ++q) {
          f2 dx = sub2(px[q], bc2(A.x)), dy = sub2(py[q], bc2(A.y)), dz = sub2(pz[q], bc2(A.z));
          f2 t1 = fma2(bc2(a02), dz, fma2(bc2(a01), dy, mul2(bc2(B.x), dx)));
          f2 m = mul2(dx, t1);
          f2 t2 = fma2(bc2(a12), dz, mul2(bc2(B.y), dy));
          m = fma2(dy, t2, m);
          m = fma2(dz, mul2(bc2(B.z), dz), m);
          acc[q] = fma2(bc2(A.w), gauss_w2(m), acc[q]);
        }
      }
    }
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
    if (vid[v] >= 0) {
      float val = (v & 1) ? hi(acc[v / 2]) : lo(acc[v / 2]);
      int64_t o = (int64_t)vid[v];
      if (residual) val += residual[o];
      out[o] = fminf(fmaxf(val, 0.f), 1.f);
    }
  }
}

// Forward-differencing pair walk (MG_VOL_FD): a warp takes two x-adjacent
// cells of the tile (same y and z runs); a lane owns one (x, y) column of
// voxels of one of them with all its z voxels (<= 6, packed in f32x2 pairs).
// Along a column dx, dy are shared, so per candidate the lane forms the
// (dx, dy) part of the quadratic form once,
//   m = [dx (P00 dx + 2 P01 dy) + P11 dy^2] + dz (2 P02 dx + 2 P12 dy + P22 dz),
// and each z voxel costs one packed subtract and two packed FMAs (~4.75 FP32-pipe
// instructions per pair instead of 6.5).  The walk covers the union of the two
// cells' windows (one extra i-column); a lane whose cell does not see a
// column weights it by 0.  Returns false (nothing written) when a run exceeds 6
// voxels along z -- the per-cell path handles those.
__device__ __forceinline__ bool vol_pair_fd(const VolTileSmem& sm, int g, int r, const VolAxes& ax, int rxA,
                                            int nrx, int ry, int rz, const float* __restrict__ residual,
                                            float* __restrict__ out, int lane) {
  const int by0 = ax.rs[1][ry], nby = ax.rs[1][ry + 1] - by0;
  const int bz0 = ax.rs[2][rz], nbz = ax.rs[2][rz + 1] - bz0;
  if (nbz > 6) return false;
  const bool hasB = rxA + 1 < nrx;
  const int bx0A = ax.rs[0][rxA], nbxA = ax.rs[0][rxA + 1] - bx0A;
  const int bx0B = hasB ? ax.rs[0][rxA + 1] : 0, nbxB = hasB ? ax.rs[0][rxA + 2] - bx0B : 0;
  const int ciA = ax.rc[0][rxA], ciB = hasB ? ax.rc[0][rxA + 1] : ciA;
  const int cj = ax.rc[1][ry], ck = ax.rc[2][rz];
  const int ncA = nbxA * nby, ntot = ncA + nbxB * nby;
  const int UI0 = sm.geom[0], UJ0 = sm.geom[1], KZ0 = sm.geom[2], nj = sm.geom[4];
  const int iu0 = max(min(ciA, ciB) - r, 0), iu1 = min(max(ciA, ciB) + r, g - 1);
  const int jlo = max(cj - r, 0), jhi = min(cj + r, g - 1);
  const int klo = max(ck - r, 0) - KZ0, khi = min(ck + r, g - 1) - KZ0 + 1;
  float zc[6];
#pragma unroll
  for (int t = 0; t < 6; ++t) zc[t] = (float)axis_coord(bz0 + min(t, nbz - 1), ax.n[2], ax.lo[2], ax.hi[2], ax.sp[2]);
  const f2 pz[3] = {mk2(zc[0], zc[1]), mk2(zc[2], zc[3]), mk2(zc[4], zc[5])};
  const int np = (nbz + 1) >> 1;  // packed z pairs in use (warp-uniform)
  for (int c0 = 0; c0 < ntot; c0 += 32) {
    const int c = c0 + lane;
    const bool active = c < ntot;
    const bool isB = c >= ncA;
    const int cc = active ? (isB ? c - ncA : c) : 0;
    const int bx = cc / nby, by = cc - bx * nby;
    const int i = (isB ? bx0B : bx0A) + bx, j = by0 + by;
    const float x = (float)axis_coord(ax.v0[0] + i, ax.n[0], ax.lo[0], ax.hi[0], ax.sp[0]);
    const float y = (float)axis_coord(j, ax.n[1], ax.lo[1], ax.hi[1], ax.sp[1]);
    const int ci = isB ? ciB : ciA;
    f2 acc[3] = {bc2(0.f), bc2(0.f), bc2(0.f)};
    for (int ii = iu0; ii <= iu1; ++ii) {
      const bool sees = active && ii >= ci - r && ii <= ci + r;
      for (int jj = jlo; jj <= jhi; ++jj) {
        const int col = (ii - UI0) * nj + (jj - UJ0);
        const int o0 = sm.off[col][0];
        const int a = sm.sb[col] + sm.off[col][klo] - o0, b = sm.sb[col] + sm.off[col][khi] - o0;
        for (int gi = a; gi < b; ++gi) {
          const float4 A = sm.A[gi], B = sm.B[gi];
          const float2 C = sm.C[gi];  // staged pre-doubled: B.w = 2P'01, C = (2P'02, 2P'12)
          const float al = sees ? A.w : 0.f;
          const float dx = x - A.x, dy = y - A.y;
          const float qa = fmaf(dy, B.y * dy, dx * fmaf(B.w, dy, B.x * dx));
          const float qb = fmaf(C.y, dy, C.x * dx);
          const f2 QA = bc2(qa), QB = bc2(qb);
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            if (q < np) {
              const f2 dz = sub2(pz[q], bc2(A.z));
              const f2 sz = fma2(dz, bc2(B.z), QB);
              const f2 m = fma2(dz, sz, QA);
              acc[q] = fma2(gauss_w2(m), bc2(al), acc[q]);
            }
          }
        }
      }
    }
    if (active) {
      const int64_t base = ((int64_t)i * ax.n[1] + j) * ax.n[2] + bz0;
#pragma unroll
      for (int t = 0; t < 6; ++t) {
        if (t < nbz) {
          float val = (t & 1) ? hi(acc[t >> 1]) : lo(acc[t >> 1]);
          if (residual) val += residual[base + t];
          out[base + t] = fminf(fmaxf(val, 0.f), 1.f);
        }
      }
    }
  }
  return true;
}

__device__ __forceinline__ void cpa16(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cpa8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

__global__ void __launch_bounds__(kVolTileWarps * 32) volume_tile_kernel(const GaussSoA grec, const int* __restrict__ gstart, int g,
                                                          int r, VolAxes ax, const float* __restrict__ residual,
                                                          float* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char vt_dyn[];
  VolTileSmem& sm = *reinterpret_cast<VolTileSmem*>(vt_dyn);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nrx = ax.nr[0], nry = ax.nr[1], nrz = ax.nr[2];
  const int tx = (nrx + 1) >> 1, ty = (nry + 1) >> 1, tz = (nrz + kTileTZ - 1) / kTileTZ;
  const int64_t ntiles = (int64_t)tx * ty * tz;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int iz = (int)(tile % tz);
    const int64_t tt = tile / tz;
    const int iy = (int)(tt % ty), ix = (int)(tt / ty);
    const int rx0 = 2 * ix, ry0 = 2 * iy, rz0 = kTileTZ * iz;  // < nrx, nry, nrz by the tile counts
    const int rx1 = min(rx0 + 1, nrx - 1), ry1 = min(ry0 + 1, nry - 1), rz1 = min(rz0 + kTileTZ - 1, nrz - 1);
    // union geometry (cells of a run pair are monotone along the axis)
    if (threadIdx.x == 0) {
      const int UI0 = max(ax.rc[0][rx0] - r, 0), UI1 = min(ax.rc[0][rx1] + r, g - 1);
      const int UJ0 = max(ax.rc[1][ry0] - r, 0), UJ1 = min(ax.rc[1][ry1] + r, g - 1);
      const int KZ0 = max(ax.rc[2][rz0] - r, 0), KZ1 = min(ax.rc[2][rz1] + r, g - 1);
      const int ni = UI1 - UI0 + 1, nj = UJ1 - UJ0 + 1, nk = KZ1 - KZ0 + 1;
      sm.geom[0] = UI0;
      sm.geom[1] = UJ0;
      sm.geom[2] = KZ0;
      sm.geom[3] = ni;
      sm.geom[4] = nj;
      sm.geom[5] = nk;
      sm.geom[7] = (ni * nj <= kTileCols && nk + 1 <= kTileK) ? 1 : 0;
    }
    __syncthreads();
    bool ok = sm.geom[7] != 0;
    if (ok) {
      const int UI0 = sm.geom[0], UJ0 = sm.geom[1], KZ0 = sm.geom[2], nj = sm.geom[4], nk = sm.geom[5];
      const int ncol = sm.geom[3] * nj;
      for (int e = threadIdx.x; e < ncol * (nk + 1); e += blockDim.x) {
        const int c = e / (nk + 1), k = e - c * (nk + 1);
        const int q = c / nj;
        const int64_t gi = ((int64_t)(UI0 + q) * g + UJ0 + (c - q * nj)) * g + KZ0 + k;
        sm.off[c][k] = __ldg(gstart + gi);
      }
      __syncthreads();
      if (warp == 0) {  // staged bases: exclusive scan of the column lengths
        int run = 0;
        for (int c0 = 0; c0 < ncol; c0 += 32) {
          const int c = c0 + lane;
          const int len = c < ncol ? sm.off[c][nk] - sm.off[c][0] : 0;
          int tot;
          const int ex = warp_excl_scan(len, lane, &tot);
          if (c < ncol) sm.sb[c] = run + ex;
          run += tot;
        }
        if (lane == 0) {
          sm.sb[ncol] = run;
          sm.geom[6] = run;
        }
      }
      __syncthreads();
      ok = sm.geom[6] <= kTileCap;
      if (ok) {
        for (int c = warp; c < ncol; c += blockDim.x >> 5) {
          const int e0 = sm.off[c][0], n = sm.off[c][nk] - e0, b0 = sm.sb[c];
          for (int t = lane; t < n; t += 32) {
            cpa16(&sm.A[b0 + t], grec.A + e0 + t);
            cpa16(&sm.B[b0 + t], grec.B + e0 + t);
            cpa8(&sm.C[b0 + t], grec.C + e0 + t);
          }
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
      }
      __syncthreads();
      if (ok) {  // off-diagonals doubled once here instead of per use (Horner form)
        for (int t = threadIdx.x; t < sm.geom[6]; t += blockDim.x) {
          sm.B[t].w *= 2.f;
          sm.C[t].x *= 2.f;
          sm.C[t].y *= 2.f;
        }
        __syncthreads();
      }
    }
#if MG_VOL_FD
    if (ok) {  // x-adjacent cell pairs, handed out from a shared counter
      if (threadIdx.x == 0) sm.next = 0;
      __syncthreads();
#pragma unroll 1
      for (;;) {
        int slot = 0;
        if (lane == 0) slot = atomicAdd(&sm.next, 1);
        slot = __shfl_sync(MG_FULL, slot, 0);
        if (slot >= 2 * kTileTZ) break;
        const int ry = ry0 + (slot & 1), rz = rz0 + (slot >> 1);
        if (ry < nry && rz < nrz && !vol_pair_fd(sm, g, r, ax, rx0, nrx, ry, rz, residual, out, lane)) {
          for (int rx = rx0; rx <= min(rx0 + 1, nrx - 1); ++rx) {  // long z runs: per-cell path
            const int bx0 = ax.rs[0][rx], nbx = ax.rs[0][rx + 1] - bx0;
            const int by0 = ax.rs[1][ry], nby = ax.rs[1][ry + 1] - by0;
            const int bz0 = ax.rs[2][rz], nbz = ax.rs[2][rz + 1] - bz0;
            const int cell = flat_cell(ax.rc[0][rx], ax.rc[1][ry], ax.rc[2][rz], g);
            const int nvox = nbx * nby * nbz;
            for (int l0 = 0; l0 < nvox; l0 += 128)
              vol_chunk_tile<4>(sm, g, r, ax, bx0, by0, bz0, nbx, nby, nbz, cell, l0, nvox, residual, out, lane);
          }
        }
      }
      __syncthreads();  // the staged tile is overwritten by the next one
      continue;
    }
#endif
#if MG_VOL_LPT
    // cells handed out dynamically, largest first (longest-processing-time):
    // 64-voxel cells take one 64-slot pass, larger ones 128-slot passes, so a
    // fixed round-robin deal left warps idle at the end-of-tile barrier
    if (threadIdx.x == 0) {
      int cost[4 * kTileTZ];
      for (int c = 0; c < 4 * kTileTZ; ++c) {
        const int rx = rx0 + ((c >> 2) & 1), ry = ry0 + ((c >> 1) & 1), rz = rz0 + (c & 1) + 2 * (c >> 3);
        int w = 0;
        if (rx < nrx && ry < nry && rz < nrz) {
          const int nv = (ax.rs[0][rx + 1] - ax.rs[0][rx]) * (ax.rs[1][ry + 1] - ax.rs[1][ry]) *
                         (ax.rs[2][rz + 1] - ax.rs[2][rz]);
          w = nv <= 64 ? 1 : 2 * ((nv + 127) / 128);
        }
        cost[c] = w;
        sm.order[c] = c;
      }
      for (int a = 1; a < 4 * kTileTZ; ++a) {  // insertion sort, descending cost
        const int v = sm.order[a];
        int b = a - 1;
        while (b >= 0 && cost[sm.order[b]] < cost[v]) {
          sm.order[b + 1] = sm.order[b];
          --b;
        }
        sm.order[b + 1] = v;
      }
      sm.next = 0;
    }
    __syncthreads();
#pragma unroll 1
    for (;;) {
    int slot = 0;
    if (lane == 0) slot = atomicAdd(&sm.next, 1);
    slot = __shfl_sync(MG_FULL, slot, 0);
    if (slot >= 4 * kTileTZ) break;
    const int c = sm.order[slot];
#else
    // this warp's runs (cells) of the tile's 2 x 2 x TZ, dealt round-robin
#pragma unroll 1
    for (int c = warp; c < 4 * kTileTZ; c += kVolTileWarps) {
#endif
    const int rx = rx0 + ((c >> 2) & 1), ry = ry0 + ((c >> 1) & 1), rz = rz0 + (c & 1) + 2 * (c >> 3);
    if (rx < nrx && ry < nry && rz < nrz) {
      const int bx0 = ax.rs[0][rx], nbx = ax.rs[0][rx + 1] - bx0;
      const int by0 = ax.rs[1][ry], nby = ax.rs[1][ry + 1] - by0;
      const int bz0 = ax.rs[2][rz], nbz = ax.rs[2][rz + 1] - bz0;
      const int cell = flat_cell(ax.rc[0][rx], ax.rc[1][ry], ax.rc[2][rz], g);
      const int nvox = nbx * nby * nbz;
      if (ok) {
        if (nvox <= 64)
          vol_chunk_tile<2>(sm, g, r, ax, bx0, by0, bz0, nbx, nby, nbz, cell, 0, nvox, residual, out, lane);
        else
          for (int l0 = 0; l0 < nvox; l0 += 128)
            vol_chunk_tile<4>(sm, g, r, ax, bx0, by0, bz0, nbx, nby, nbz, cell, l0, nvox, residual, out, lane);
      } else {
        if (nvox <= 64)
          vol_chunk<2>(grec, gstart, g, r, ax, bx0, by0, bz0, nbx, nby, nbz, cell, 0, nvox, residual, out, 0, lane);
        else
          for (int l0 = 0; l0 < nvox; l0 += 128)
            vol_chunk<4>(grec, gstart, g, r, ax, bx0, by0, bz0, nbx, nby, nbz, cell, l0, nvox, residual, out, 0,
                         lane);
      }
    }
    }
    __syncthreads();  // the staged tile is overwritten by the next one
  }
}

size_t volume_workspace_bytes(int nx, int ny, int nz) {
  int m = nx > ny ? nx : ny;
  m = m > nz ? m : nz;
  size_t per = (((size_t)(m + 1) * 4 + 255) & ~(size_t)255);
  return 3 * 5 * per + 256 + scan_workspace_bytes(m);
}

// Samples voxels [i0, i1) x [0, ny) x [0, nz); out is the slab (i1-i0, ny, nz),
// float32, clipped to [0, 1].  residual (optional) is added before the clip.
void launch_sample_volume(const float* grec_raw, int64_t n_gauss, const int* gstart, int g, int r, const int dims[3],
                          const double lo[3],
                          const double hi[3], int i0, int i1, const float* residual, float* out, void* ws,
                          cudaStream_t st) {
  int n[3] = {dims[0], dims[1], dims[2]};
  int m = n[0] > n[1] ? n[0] : n[1];
  m = m > n[2] ? m : n[2];
  size_t per = (((size_t)(m + 1) * 4 + 255) & ~(size_t)255);
  char* w = (char*)ws;
  int* nr = (int*)w;
  w += 256;
  VolAxes ax;
  ax.nr = nr;
  void* sws = w + 3 * 5 * per;
  for (int a = 0; a < 3; ++a) {
    int* cells = (int*)(w + (5 * a + 0) * per);
    int* flags = (int*)(w + (5 * a + 1) * per);
    int* scan = (int*)(w + (5 * a + 2) * per);
    int* rs = (int*)(w + (5 * a + 3) * per);
    int* rc = (int*)(w + (5 * a + 4) * per);
    int v0 = a == 0 ? i0 : 0, v1 = a == 0 ? i1 : n[a];
    ax.n[a] = n[a];
    ax.lo[a] = lo[a];
    ax.hi[a] = hi[a];
    ax.sp[a] = n[a] == 1 ? (hi[a] - lo[a]) : (hi[a] - lo[a]) / (double)(n[a] - 1);
    ax.v0[a] = 0;
    ax.rs[a] = rs;
    ax.rc[a] = rc;
    int cnt = v1 - v0;
    MG_LAUNCH(axis_cells_kernel<<<(cnt + 255) / 256, 256, 0, st>>>(n[a], v0, v1, lo[a], hi[a], ax.sp[a], g, cells, flags));
    excl_scan(flags, scan, cnt, sws, st);
    MG_LAUNCH(axis_runs_kernel<<<(cnt + 255) / 256, 256, 0, st>>>(cells, flags, scan, cnt, rs, rc, nr + a));
  }
  // axis-0 voxel indices inside the kernel are slab-relative; shift coordinates by i0
  ax.v0[0] = i0;
  int64_t maxitems = (int64_t)(i1 - i0) * n[1] * n[2];
  int64_t blocks = (maxitems + kVolWarps - 1) / kVolWarps;
  int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  // write offsets: kernel computes vid relative to the slab (i in [0, i1-i0))
  if (MG_VOL_TILE && 2 + 2 * r <= 12 && kTileTZ + 2 * r + 1 <= kTileK) {
    const size_t smem = sizeof(VolTileSmem);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(volume_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = true;
    }
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, volume_tile_kernel, kVolTileWarps * 32, smem);
    const int64_t tiles = (int64_t)((i1 - i0 + 1) / 2 + 1) * ((n[1] + 1) / 2 + 1) * (n[2] / kTileTZ + 1);
    int64_t tb = (int64_t)num_sms() * (per_sm > 0 ? per_sm : 1);
    if (tb > tiles) tb = tiles;
    MG_LAUNCH(volume_tile_kernel<<<(unsigned)tb, kVolTileWarps * 32, smem, st>>>(gauss_soa(grec_raw, n_gauss), gstart, g, r, ax,
                                                                   residual, out));
    return;
  }
  MG_LAUNCH(volume_kernel<<<(unsigned)blocks, kVolWarps * 32, 0, st>>>(gauss_soa(grec_raw, n_gauss), gstart, g, r, ax, residual,
                                                              out));
}

}  // namespace mg
