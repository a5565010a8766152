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
            int32_t *__restrict__ max_count, int cell = -1) {
    const int lane = threadIdx.x & 31;
    const Image im = make_image(g);
    const double xi = ldc<kCoherent>(pr + 3 * r), yi = ldc<kCoherent>(pr + 3 * r + 1),
                 zi = ldc<kCoherent>(pr + 3 * r + 2);
    const int cb = cell >= 0 ? cell : ldc<kCoherent>(cell_of_rank + r);
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

// ---------------------------------------------------------------------------
// Cell-staged rows: one CTA builds the rows of every particle of cell c.
// The (at most 27) neighbour cells, sorted by flat id as in nlist_one, are
// staged once into shared memory -- fp64 positions for the reference
// arithmetic, fp32 minimum-image coordinates relative to c's centre for a
// filter, ranks -- instead of every particle's warp gathering its ~27 x
// occupancy candidates from L2.  Per particle: pass 1 keeps the candidates
// whose fp32 distance is within r_list^2 (1 + 1e-3) (its error is ~1e-6 of
// that: a superset of the survivors), in candidate order; pass 2 decides
// them with the reference arithmetic (exact_disp, exact_r2, inclusive) and
// appends the survivors in order.  Rows are identical to nlist_one's:
// ascending rank, the same predicate.  A neighbourhood over nb_cap, or a
// particle with more than kRowsBuf filter survivors, falls back to
// nlist_one (the caller sees false / the particle is redone there).
// ---------------------------------------------------------------------------
constexpr int kRowsBuf = 256;  // filter survivors per particle (per warp)

// The fp32 filter compares minimum-image coordinates relative to the cell's
// centre; their difference is the pair's minimum image whenever the pair is
// within the cutoff only if every periodic dimension has >= 4 cells (a
// neighbour is at most 2 cells from the centre's image).  Smaller grids take
// nlist_one.
inline bool rows_staged_ok(const rb_grid &g) {
    if (!g.periodic) return true;
    for (int d = 0; d < 3; d++)
        if ((g.wrap[d] ? g.cells[d] : g.gcells[d]) < 4) return false;
    return true;
}

// staged particles per cell: 27 neighbour cells at twice the mean occupancy
// (and at least 24 per cell); a denser neighbourhood takes nlist_one
inline int rows_nb_cap(int64_t n, int64_t ncell) {
    const double mean = ncell > 0 ? (double)n / (double)ncell : 0.0;
    const double per = mean * 2.0 > 24.0 ? mean * 2.0 : 24.0;
    int cap = (int)(27.0 * per) + 64;
    cap = (cap + 31) / 32 * 32;
    return cap < 2048 ? cap : 2048;
}

struct RowsSmem {
    int32_t *cell, *start, *base;  // [28] sorted neighbour cells, first rank, staged prefix
    int32_t *misc;                 // total, self index, overflow
    double *x;                     // [nb_cap][3]
    float4 *f;                     // [nb_cap] fp32 relative coordinates
    int32_t *rank;                 // [nb_cap]
    int32_t *buf;                  // [warps][kRowsBuf]
};

__host__ __device__ inline size_t rows_smem_bytes(int nb_cap, int warps) {
    return 128 * sizeof(int32_t) + (size_t)nb_cap * (3 * sizeof(double) + sizeof(float4) +
                                                     sizeof(int32_t)) +
           (size_t)warps * kRowsBuf * sizeof(int32_t) + 64;
}

__device__ __forceinline__ RowsSmem rows_carve(char *base, int nb_cap) {
    RowsSmem s;
    s.cell = (int32_t *)base;
    s.start = s.cell + 28;
    s.base = s.start + 28;
    s.misc = s.base + 28;
    s.f = (float4 *)(base + 128 * sizeof(int32_t));
    s.x = (double *)(s.f + nb_cap);
    s.rank = (int32_t *)(s.x + 3 * (size_t)nb_cap);
    s.buf = s.rank + nb_cap;
    return s;
}

// false: the neighbourhood of c exceeds nb_cap (nothing written)
template <bool kCoherent>
__device__ bool nlist_cell(const rb_grid &g, int c, const double *__restrict__ pr,
                           const int32_t *__restrict__ cell_start, double rl2, float hi_f,
                           int32_t capacity, int32_t *__restrict__ rows,
                           int32_t *__restrict__ row_count, int32_t *__restrict__ max_count,
                           const RowsSmem &sm, int nb_cap) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int czz = c % g.cells[2], cyy = (c / g.cells[2]) % g.cells[1],
              cxx = c / (g.cells[2] * g.cells[1]);
    if (warp == 0) {  // the sorted neighbour cells, their ranks and staged offsets
        int my_cell = 0x7fffffff, nvalid = 0;
        for (int ob = 0; ob < g.n_offsets; ob += 32) {
            const int o = ob + lane;
            const int cc = o < g.n_offsets ? neighbor_cell(g, cxx, cyy, czz, o) : -1;
            const unsigned mv = __ballot_sync(0xffffffffu, cc >= 0);
            const int q = lane - nvalid;
            const unsigned src = (q >= 0 && q < __popc(mv)) ? __fns(mv, 0, q + 1) : 0u;
            const int v = __shfl_sync(0xffffffffu, cc, (int)(src & 31u));
            if (q >= 0 && q < __popc(mv)) my_cell = v;
            nvalid += __popc(mv);
        }
#pragma unroll
        for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
            for (int j = k >> 1; j > 0; j >>= 1) {
                const int other = __shfl_xor_sync(0xffffffffu, my_cell, j);
                const bool take_min = ((lane & j) == 0) == ((lane & k) == 0);
                my_cell = take_min ? min(my_cell, other) : max(my_cell, other);
            }
        }
        int cs = 0, cnt = 0;
        if (lane < nvalid) {
            cs = ldc<kCoherent>(cell_start + my_cell);
            cnt = ldc<kCoherent>(cell_start + my_cell + 1) - cs;
        }
        int incl = cnt;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += y;
        }
        if (lane < nvalid) {
            sm.cell[lane] = my_cell;
            sm.start[lane] = cs;
            sm.base[lane] = incl - cnt;
            if (my_cell == c) sm.misc[1] = lane;
        }
        if (lane == 31) {
            sm.base[nvalid] = incl;
            sm.misc[0] = incl;
            sm.misc[2] = nvalid;
        }
    }
    __syncthreads();
    const int total = sm.misc[0], self = sm.misc[1], ncells = sm.misc[2];
    if (total > nb_cap) {
        __syncthreads();  // every thread has read the header
        return false;
    }
    // stage: positions (exact), fp32 coordinates relative to c's centre
    // (minimum image), ranks
    double ctr[3];
    {
        const int cc[3] = {cxx, cyy, czz};
#pragma unroll
        for (int d = 0; d < 3; d++)
            ctr[d] = g.origin[d] + ((g.wrap[d] ? 0 : g.wlo[d]) + cc[d] + 0.5) / g.inv_cell[d];
    }
    for (int k = threadIdx.x; k < total; k += blockDim.x) {
        int j = 0;
        while (j + 1 < ncells && sm.base[j + 1] <= k) j++;
        const int q = sm.start[j] + (k - sm.base[j]);
        const double x = ldc<kCoherent>(pr + 3 * (int64_t)q),
                     y = ldc<kCoherent>(pr + 3 * (int64_t)q + 1),
                     z = ldc<kCoherent>(pr + 3 * (int64_t)q + 2);
        sm.x[3 * k] = x;
        sm.x[3 * k + 1] = y;
        sm.x[3 * k + 2] = z;
        double rel[3] = {x - ctr[0], y - ctr[1], z - ctr[2]};
        if (g.periodic) {
#pragma unroll
            for (int d = 0; d < 3; d++) rel[d] = fma(-g.box[d], rint(rel[d] / g.box[d]), rel[d]);
        }
        sm.f[k] = make_float4((float)rel[0], (float)rel[1], (float)rel[2], 0.0f);
        sm.rank[k] = q;
    }
    __syncthreads();
    const Image im = make_image(g);
    const int b0 = sm.base[self], b1 = sm.base[self + 1], r0 = sm.start[self];
    int32_t *buf = sm.buf + warp * kRowsBuf;
    for (int bi = b0 + warp; bi < b1; bi += nwarps) {
        const int64_t r = r0 + (bi - b0);
        const float4 fi = sm.f[bi];
        // pass 1: the fp32 filter, survivors in candidate order
        int nc = 0;
        for (int k0 = 0; k0 < total; k0 += 32) {
            const int k = k0 + lane;
            bool pass = false;
            if (k < total && k != bi) {
                const float4 o = sm.f[k];
                const float dx = fi.x - o.x, dy = fi.y - o.y, dz = fi.z - o.z;
                pass = fmaf(dz, dz, fmaf(dy, dy, dx * dx)) <= hi_f;
            }
            const unsigned mk = __ballot_sync(0xffffffffu, pass);
            const int at = nc + __popc(mk & lanemask_lt());
            if (pass && at < kRowsBuf) buf[at] = k;
            nc += __popc(mk);
        }
        __syncwarp();
        if (nc > kRowsBuf) {  // more filter survivors than the buffer: the L2 path
            nlist_one<kCoherent>(g, r, 0, pr, cell_start, nullptr, rl2, capacity, rows,
                                 row_count, max_count, c);
            __syncwarp();
            continue;
        }
        // pass 2: the reference arithmetic decides, survivors appended in order
        const double xi = sm.x[3 * bi], yi = sm.x[3 * bi + 1], zi = sm.x[3 * bi + 2];
        int32_t *row = rows + r * (int64_t)capacity;
        int count = 0;
        for (int c0 = 0; c0 < nc; c0 += 32) {
            const int ci = c0 + lane;
            bool keep = false;
            int k = 0;
            if (ci < nc) {
                k = buf[ci];
                double dx, dy, dz;
                exact_disp(im, xi, yi, zi, sm.x[3 * k], sm.x[3 * k + 1], sm.x[3 * k + 2], dx, dy,
                           dz);
                keep = exact_r2(dx, dy, dz) <= rl2;
            }
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            const int slot = count + __popc(m & lanemask_lt());
            if (keep && slot < capacity) row[slot] = sm.rank[k];
            count += __popc(m);
        }
        if (lane == 0) {
            row_count[r] = count < capacity ? count : capacity;
            if (count > *(volatile int32_t *)max_count) atomicMax(max_count, count);
        }
        __syncwarp();
    }
    __syncthreads();  // the staged neighbourhood is reused by the next cell
    return true;
}

}  // namespace rb
