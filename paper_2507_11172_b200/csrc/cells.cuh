// cells.cuh -- device pieces of the row rebuild shared by the separate
// kernels (bin.cu, nlist.cu) and the fused gated rebuild (rebuild.cu).
#pragma once

#include "common.cuh"

namespace rb {

// Loads of data written earlier in the SAME kernel (the fused rebuild, whose
// phases are separated by grid barriers) must not take the read-only
// (non-coherent) path, which nvcc may pick for a plain load through a const
// __restrict__ pointer: kCoherent selects explicit weak loads cached in L1
// (ld.global.ca).  They see the other blocks' writes because every grid
// barrier ends with a __threadfence() (fence.sc: L1 invalidated) and a
// __syncthreads(), the cooperative-groups grid.sync() pattern; the rows and
// positions are re-read ~27x per phase, so L1 hits matter (RB_REBUILD_CG=1:
// the former L2-only loads, for A/B).
#ifndef RB_REBUILD_CG
#define RB_REBUILD_CG 0
#endif
template <bool kCoherent, typename T>
__device__ __forceinline__ T ldc(const T *p) {
    if constexpr (kCoherent) return RB_REBUILD_CG ? __ldcg(p) : __ldca(p);
    else return *p;
}

__device__ __forceinline__ int cell_index_1d(double x, double origin, double inv, int n) {
    // python int() truncates toward zero; numba's int() is the same fptosi
    double t = xmul(xsub(x, origin), inv);
    long long c = (long long)t;
    if (c < 0) c = 0;
    else if (c >= n) c = n - 1;
    return (int)c;
}

// cell of a coordinate in dimension d: the global index, mapped into the
// rank's window when the grid is a window of a decomposed periodic grid
__device__ __forceinline__ int cell_index(const rb_grid &g, int d, double x) {
    if (g.wrap[d] || !g.periodic) return cell_index_1d(x, g.origin[d], g.inv_cell[d], g.cells[d]);
    int c = cell_index_1d(x, g.origin[d], g.inv_cell[d], g.gcells[d]) - g.wlo[d];
    if (c < 0) c += g.gcells[d];
    if (c >= g.gcells[d]) c -= g.gcells[d];
    return c < g.cells[d] ? c : g.cells[d] - 1;  // outside the window: caller's error
}

// Rebuild gate: a binning launched inside a captured r-RESPA step runs only
// when the drift of that step flagged a rebuild (*flag == tag); flag == NULL
// means always (standalone passes).
__device__ __forceinline__ bool gate_closed(const int64_t *flag, const unsigned long long *status,
                                            int64_t tag) {
    if (!flag) return false;
    return *(volatile const int64_t *)flag != resolve_tag(tag, status);
}

constexpr int kScanThreads = 512;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int block_exclusive_scan(int v, int *warp_sums, int &total) {
    int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int nw = blockDim.x >> 5;
        int s = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, s, off);
            if (lane >= off) s += y;
        }
        if (lane < nw) warp_sums[lane] = s;
    }
    __syncthreads();
    int warp_off = warp ? warp_sums[warp - 1] : 0;
    total = warp_sums[(blockDim.x >> 5) - 1];
    __syncthreads();
    return warp_off + x - v;
}

// One warp per cell c: restore ascending particle order inside the cell (the
// atomic scatter is unordered), then gather the rank-ordered positions and
// the rank <-> particle maps.  Cells of up to 32 particles sort in registers
// (rank = number of smaller indices); larger cells fall back to a serial
// insertion sort by lane 0.
template <bool kCoherent = false>
__device__ __forceinline__ void cell_finish_one(int64_t c, int lane,
                                                const int32_t *__restrict__ start,
                                                int32_t *__restrict__ parts,
                                                int32_t *__restrict__ cell_of_rank,
                                                int32_t *__restrict__ rank_of,
                                                const double *__restrict__ pos,
                                                double *__restrict__ pr,
                                                double *__restrict__ x_ref) {
    const int b = ldc<kCoherent>(start + c), e = ldc<kCoherent>(start + c + 1), k = e - b;
    if (k <= 32) {
        const int v = lane < k ? ldc<kCoherent>(parts + b + lane) : 0x7fffffff;
        int rank = 0;
        for (int l = 0; l < k; l++) rank += __shfl_sync(0xffffffffu, v, l) < v ? 1 : 0;
        __syncwarp();
        if (lane < k) parts[b + rank] = v;
    } else if (lane == 0) {
        for (int a = b + 1; a < e; a++) {
            const int v = ldc<kCoherent>(parts + a);
            int q = a - 1;
            while (q >= b && parts[q] > v) {
                parts[q + 1] = parts[q];
                q--;
            }
            parts[q + 1] = v;
        }
    }
    __syncwarp();
    for (int r = b + lane; r < e; r += 32) {
        const int64_t p = parts[r];
        const double x = pos[3 * p], y = pos[3 * p + 1], z = pos[3 * p + 2];
        cell_of_rank[r] = (int32_t)c;
        pr[3 * (int64_t)r] = x;
        pr[3 * (int64_t)r + 1] = y;
        pr[3 * (int64_t)r + 2] = z;
        if (rank_of) rank_of[p] = r;
        if (x_ref) {
            x_ref[3 * p] = x;
            x_ref[3 * p + 1] = y;
            x_ref[3 * p + 2] = z;
        }
    }
}

template <bool kCoherent = false>
__device__ __forceinline__ void nlist_one(const rb_grid &g, int64_t r, int64_t n, const double *__restrict__ pr, const int32_t *__restrict__ cell_start,
            const int32_t *__restrict__ cell_of_rank, double rl2, int32_t capacity,
            int32_t *__restrict__ rows, int32_t *__restrict__ row_count,
            int32_t *__restrict__ max_count) {
    const int lane = threadIdx.x & 31;
    const Image im = make_image(g);
    const double xi = ldc<kCoherent>(pr + 3 * r), yi = ldc<kCoherent>(pr + 3 * r + 1),
                 zi = ldc<kCoherent>(pr + 3 * r + 2);
    const int cb = ldc<kCoherent>(cell_of_rank + r);
    const int cbz = cb % g.cells[2];
    const int cby = (cb / g.cells[2]) % g.cells[1];
    const int cbx = cb / (g.cells[2] * g.cells[1]);
    int32_t *row = rows + r * (int64_t)capacity;
    // 1. the (at most 27) valid neighbour cells, one per lane, sorted by flat
    //    id so that rows come out in ascending rank order
    int my_cell = 0x7fffffff;
    int nvalid = 0;
    for (int ob = 0; ob < g.n_offsets; ob += 32) {
        const int o = ob + lane;
        const int cc = o < g.n_offsets ? neighbor_cell(g, cbx, cby, cbz, o) : -1;
        const unsigned mv = __ballot_sync(0xffffffffu, cc >= 0);
        // lane nvalid + q receives the q-th valid cell of this chunk
        const int q = lane - nvalid;
        const unsigned src = (q >= 0 && q < __popc(mv)) ? __fns(mv, 0, q + 1) : 0u;
        const int v = __shfl_sync(0xffffffffu, cc, (int)(src & 31u));
        if (q >= 0 && q < __popc(mv)) my_cell = v;
        nvalid += __popc(mv);
    }
    // bitonic sort (ascending) of my_cell across the warp
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const int other = __shfl_xor_sync(0xffffffffu, my_cell, j);
            const bool take_min = ((lane & j) == 0) == ((lane & k) == 0);
            my_cell = take_min ? min(my_cell, other) : max(my_cell, other);
        }
    }
    int cstart = 0, ccount = 0;
    if (lane < nvalid) {
        cstart = ldc<kCoherent>(cell_start + my_cell);
        ccount = ldc<kCoherent>(cell_start + my_cell + 1) - cstart;
    }
    // 2. flattened candidate range over the sorted cells
    int incl = ccount;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    int count = 0;
    for (int base = 0; base < total; base += 32) {
        const int cand = base + lane;
        // owner lane of cand: first lane whose inclusive prefix exceeds cand
        int pos = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
            const int v = __shfl_sync(0xffffffffu, incl, pos + step - 1);
            if (v <= cand) pos += step;
        }
        const int owner_incl = __shfl_sync(0xffffffffu, incl, pos);
        const int owner_count = __shfl_sync(0xffffffffu, ccount, pos);
        const int owner_start = __shfl_sync(0xffffffffu, cstart, pos);
        bool keep = false;
        int j = 0;
        if (cand < total) {
            j = owner_start + (cand - (owner_incl - owner_count));
            if (j != r) {
                double dx, dy, dz;
                exact_disp(im, xi, yi, zi, ldc<kCoherent>(pr + 3 * j),
                           ldc<kCoherent>(pr + 3 * j + 1), ldc<kCoherent>(pr + 3 * j + 2), dx,
                           dy, dz);
                keep = exact_r2(dx, dy, dz) <= rl2;
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        const int slot = count + __popc(m & lanemask_lt());
        if (keep && slot < capacity) row[slot] = j;
        count += __popc(m);
    }
    if (lane == 0) {
        row_count[r] = count < capacity ? count : capacity;
        // longest row seen (also the overflow witness when > capacity); the
        // plain read first keeps the atomic off the common path
        if (count > *(volatile int32_t *)max_count) atomicMax(max_count, count);
    }
}


// mirror entries of row p (one warp): for each entry q > p a lane
// binary-searches p in the rank-sorted row q and writes BOTH mirror[p][k]
// and, by symmetry, mirror[q][that position] = k -- every pair once.
template <bool kCoherent = false>
__device__ __forceinline__ void mirror_one(int64_t p, int lane, const int32_t *__restrict__ rows,
                                           const int32_t *__restrict__ row_count,
                                           int32_t capacity, int32_t *__restrict__ mirror) {
        const int m = ldc<kCoherent>(row_count + p);
        const int32_t *rp = rows + p * (int64_t)capacity;
        for (int k = lane; k < m; k += 32) {
            const int q = kCoherent ? __ldcg(rp + k) : __ldg(rp + k);
            if (q <= p) continue;  // written by the warp of row q
            const int32_t *rq = rows + (int64_t)q * capacity;
            int lo = 0, hi = ldc<kCoherent>(row_count + q) - 1, pos = -1;
            while (lo <= hi) {
                const int mid = (lo + hi) >> 1;
                const int v = kCoherent ? __ldcg(rq + mid) : __ldg(rq + mid);
                if (v == (int)p) {
                    pos = mid;
                    break;
                }
                if (v < (int)p) lo = mid + 1;
                else hi = mid - 1;
            }
            mirror[p * (int64_t)capacity + k] = pos;
            if (pos >= 0) mirror[(int64_t)q * capacity + pos] = k;
        }
}

}  // namespace rb
