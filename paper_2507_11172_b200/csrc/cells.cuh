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


// mirror entries of row p (one warp): for each entry q > p, the position of
// p in the rank-sorted row q.  Only these (upper) entries are written: the
// Newton-3 pass reads mirror[r][k] for rows[r][k] > r alone.  An 8-lane
// group serves one entry: it reads row q 32 entries at a time (one 128-byte
// line, four per lane) and counts the entries below p -- p < q sits in the
// lower half of row q, so one chunk, rarely two, instead of a ~7-load
// dependent binary search per lane; four entries per warp step.
template <bool kCoherent = false>
__device__ __forceinline__ void mirror_one(int64_t p, int lane, const int32_t *__restrict__ rows,
                                           const int32_t *__restrict__ row_count,
                                           int32_t capacity, int32_t *__restrict__ mirror) {
    const int m = ldc<kCoherent>(row_count + p);
    const int32_t *rp = rows + p * (int64_t)capacity;
    // first entry above p (rows ascend): the suffix this warp serves
    int first = m;
    for (int k0 = 0; k0 < m; k0 += 32) {
        const int k = k0 + lane;
        const unsigned b = __ballot_sync(0xffffffffu, k < m && ldc<kCoherent>(rp + k) > (int)p);
        if (b) {
            first = k0 + __ffs(b) - 1;
            break;
        }
    }
    const int grp = lane >> 3, sub = lane & 7;
    const unsigned gmask = 0xffu << (8 * grp);
    const bool vec = (capacity & 3) == 0;  // 16-byte aligned rows
    for (int k0 = first; k0 < m; k0 += 4) {
        const int k = k0 + grp;
        const bool valid = k < m;
        int q = 0, mq = 0;
        if (valid) {
            q = ldc<kCoherent>(rp + k);
            mq = ldc<kCoherent>(row_count + q);
        }
        const int32_t *rq = rows + (int64_t)q * capacity;
        int pos = -1;
        bool done = !valid;
        for (int base = 0; __any_sync(0xffffffffu, !done); base += 32) {
            int below = 0;
            bool hit = false, stop = false;
            if (!done) {
                const int at = base + 4 * sub;
                int v[4];
                if (vec && at + 4 <= capacity) {
                    const int4 w = ldc<kCoherent>(reinterpret_cast<const int4 *>(rq + at));
                    v[0] = w.x, v[1] = w.y, v[2] = w.z, v[3] = w.w;
                } else {
#pragma unroll
                    for (int t = 0; t < 4; t++) v[t] = at + t < capacity ? ldc<kCoherent>(rq + at + t) : 0;
                }
#pragma unroll
                for (int t = 0; t < 4; t++) {
                    const int x = at + t < mq ? v[t] : 0x7fffffff;  // past the row: above p
                    below += x < (int)p;
                    hit = hit || x == (int)p;
                    stop = stop || x >= (int)p;
                }
            }
            // group totals (xor tree inside the 8 lanes)
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) below += __shfl_xor_sync(0xffffffffu, below, o);
            const unsigned hb = __ballot_sync(0xffffffffu, hit) & gmask;
            const unsigned sb = __ballot_sync(0xffffffffu, stop) & gmask;
            if (!done && (sb || base + 32 >= mq)) {
                pos = hb ? base + below : -1;
                done = true;
            }
        }
        if (valid && sub == 0) mirror[p * (int64_t)capacity + k] = pos;
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
    if (g.n_offsets > 32) return false;  // one neighbour cell per lane
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
    int32_t *misc;                 // total, self index, cell count, mirror-search flag
    int32_t *slotc;                // [32] index of c among cell j's sorted neighbour cells
    int32_t *jc;                   // [3][32] coordinates of the sorted neighbour cells
    double *ctr;                   // [3] centre of c
    double *x;                     // [nb_cap][3]
    float4 *f;                     // [nb_cap] fp32 relative coordinates
    int32_t *rank;                 // [nb_cap]
    uint32_t *bits;                // [nb_cap] which of c's particles have k in their row
    int32_t *segn;                 // [warps][32] survivors per neighbour cell (directory)
    int32_t *buf;                  // [warps][kRowsBuf]
    uint8_t *cj;                   // [nb_cap] neighbour-cell index of staged particle k
};

// RB_ROWS_SMEM_X=0: the exact pass reads the candidates' fp64 positions from
// L1/L2 instead of staging them (24 bytes less shared memory per candidate)
#ifndef RB_ROWS_SMEM_X
#define RB_ROWS_SMEM_X 0
#endif
__host__ __device__ inline size_t rows_smem_bytes(int nb_cap, int warps) {
    return 288 * sizeof(int32_t) +
           (size_t)nb_cap * (RB_ROWS_SMEM_X * 3 * sizeof(double) + sizeof(float4) +
                             2 * sizeof(int32_t) + 1) +
           (size_t)warps * (kRowsBuf + 32) * sizeof(int32_t) + 64;
}

__device__ __forceinline__ RowsSmem rows_carve(char *base, int nb_cap) {
    RowsSmem s;
    s.cell = (int32_t *)base;
    s.start = s.cell + 28;
    s.base = s.start + 28;
    s.misc = s.base + 28;
    s.slotc = (int32_t *)base + 128;
    s.jc = (int32_t *)base + 160;
    s.ctr = (double *)((int32_t *)base + 256);
    s.f = (float4 *)(base + 288 * sizeof(int32_t));
    s.x = (double *)(s.f + nb_cap);
    s.rank = (int32_t *)(s.x + RB_ROWS_SMEM_X * 3 * (size_t)nb_cap);
    s.bits = (uint32_t *)(s.rank + nb_cap);
    s.segn = (int32_t *)(s.bits + nb_cap);
    s.buf = s.segn + (blockDim.x >> 5) * 32;
    s.cj = (uint8_t *)(s.buf + (blockDim.x >> 5) * kRowsBuf);
    return s;
}

// Mirror indices from the cell structure (the staged path's by-product; the
// fused rebuild and rb_nlist_rows_mirror).  A row lists its neighbour cells'
// members in flat-cell-id order, ascending rank inside each cell, so the
// position of p (in cell c) in the row of q (in cell c') is
//     dir[q][slot of c among c' 's sorted neighbour cells]   (survivors of
//         row q in the cells before c, written by c' 's CTA)
//   + #{x in c, x < p, q in row x}                            (c's CTA: a
//         bit per (staged q, particle of c), the predicate being symmetric)
// The CTA of c writes the second term and the slot into mirror[p][k] as
// `within | slot << 24` (kMirrorSearch where it cannot: a cell over 32
// particles or with a per-particle fallback); mirror_resolve adds the first.
// dir rows of particles whose rows were not built by the staged path are
// all kDirNone.
constexpr int32_t kMirrorSearch = -2;
constexpr int32_t kMirrorLower = -3;  // (rows phase) an entry of rank below the row's particle
constexpr uint16_t kDirNone = 0xffff;
constexpr int kDirStride = 32;  // uint16 per particle

// false: the neighbourhood of c exceeds nb_cap (nothing written).  mirror
// and dir non-null: the mirror partials and directory rows of c's particles
// are written too (see kMirrorSearch above).
template <bool kCoherent>
__device__ bool nlist_cell(const rb_grid &g, int c, const double *__restrict__ pr,
                           const int32_t *__restrict__ cell_start, double rl2, float hi_f,
                           int32_t capacity, int32_t *__restrict__ rows,
                           int32_t *__restrict__ row_count, int32_t *__restrict__ max_count,
                           const RowsSmem &sm, int nb_cap, int32_t *__restrict__ mirror = nullptr,
                           uint16_t *__restrict__ dir = nullptr) {
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
            sm.jc[lane] = my_cell / (g.cells[2] * g.cells[1]);
            sm.jc[32 + lane] = (my_cell / g.cells[2]) % g.cells[1];
            sm.jc[64 + lane] = my_cell % g.cells[2];
        }
        if (lane < 3) {
            const int cc = lane == 0 ? cxx : (lane == 1 ? cyy : czz);
            sm.ctr[lane] = g.origin[lane] +
                           ((g.wrap[lane] ? 0 : g.wlo[lane]) + cc + 0.5) / g.inv_cell[lane];
        }
        if (lane == 31) {
            sm.base[nvalid] = incl;
            sm.misc[0] = incl;
            sm.misc[2] = nvalid;
            sm.misc[3] = 0;
        }
    }
    __syncthreads();
    const int total = sm.misc[0], self = sm.misc[1], ncells = sm.misc[2];
    if (total > nb_cap) {
        __syncthreads();  // every thread has read the header
        return false;
    }
    const bool with_mirror = mirror != nullptr && dir != nullptr;
    if (with_mirror && threadIdx.x == 0 && sm.base[self + 1] - sm.base[self] > 32)
        sm.misc[3] = 1;  // more particles than bits: this cell's partials search
    // stage: positions (exact), fp32 coordinates relative to c's centre
    // (minimum image), ranks
    const double ctr[3] = {sm.ctr[0], sm.ctr[1], sm.ctr[2]};
    if (with_mirror) {
        // slotc[j]: the index of c among the sorted neighbour cells of cell j
        // (the neighbourhood relation is symmetric); a warp per cell j, a
        // lane per offset (rows grids have <= 32 offsets)
        const int o = lane < g.n_offsets ? lane : 0;
        const int ox = g.offsets[o][0], oy = g.offsets[o][1], oz = g.offsets[o][2];
        for (int j = warp; j < ncells; j += nwarps) {
            const int cc = lane < g.n_offsets
                               ? cell_at(g, sm.jc[j] + ox, sm.jc[32 + j] + oy, sm.jc[64 + j] + oz)
                               : -1;
            const int below = __popc(__ballot_sync(0xffffffffu, cc >= 0 && cc < c));
            if (lane == 0) sm.slotc[j] = below;
        }
    }
    for (int k = threadIdx.x; k < total; k += blockDim.x) {
        {
            // neighbour cell of staged index k: binary search of the prefix
            int j = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1)
                if (j + step < ncells && sm.base[j + step] <= k) j += step;
            const int q = sm.start[j] + (k - sm.base[j]);
            const double x = ldc<kCoherent>(pr + 3 * (int64_t)q),
                         y = ldc<kCoherent>(pr + 3 * (int64_t)q + 1),
                         z = ldc<kCoherent>(pr + 3 * (int64_t)q + 2);
            if (RB_ROWS_SMEM_X) {
                sm.x[3 * k] = x;
                sm.x[3 * k + 1] = y;
                sm.x[3 * k + 2] = z;
            }
            double rel[3] = {x - ctr[0], y - ctr[1], z - ctr[2]};
            if (g.periodic) {
#pragma unroll
                for (int d = 0; d < 3; d++)
                    rel[d] = fma(-g.box[d], rint(rel[d] * (1.0 / g.box[d])), rel[d]);
            }
            sm.f[k] = make_float4((float)rel[0], (float)rel[1], (float)rel[2], 0.0f);
            sm.rank[k] = q;
            sm.cj[k] = (uint8_t)j;
            sm.bits[k] = 0u;
        }
    }
    sm.segn[threadIdx.x] = 0;  // (blockDim.x == warps * 32)
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
            if (with_mirror) {  // no bits for this particle: the cell's partials search
                dir[r * kDirStride + lane] = kDirNone;
                if (lane == 0) sm.misc[3] = 1;
            }
            __syncwarp();
            continue;
        }
        // pass 2: the reference arithmetic decides, survivors appended in order
        const double xi = ldc<kCoherent>(pr + 3 * r), yi = ldc<kCoherent>(pr + 3 * r + 1),
                     zi = ldc<kCoherent>(pr + 3 * r + 2);
        int32_t *row = rows + r * (int64_t)capacity;
        int count = 0;
        for (int c0 = 0; c0 < nc; c0 += 32) {
            const int ci = c0 + lane;
            bool keep = false;
            int k = 0;
            if (ci < nc) {
                k = buf[ci];
                double dx, dy, dz;
                double px, py, pz;
                if (RB_ROWS_SMEM_X) {
                    px = sm.x[3 * k], py = sm.x[3 * k + 1], pz = sm.x[3 * k + 2];
                } else {
                    const int64_t q = sm.rank[k];
                    px = ldc<kCoherent>(pr + 3 * q), py = ldc<kCoherent>(pr + 3 * q + 1),
                    pz = ldc<kCoherent>(pr + 3 * q + 2);
                }
                exact_disp(im, xi, yi, zi, px, py, pz, dx, dy, dz);
                keep = exact_r2(dx, dy, dz) <= rl2;
            }
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            const int slot = count + __popc(m & lanemask_lt());
            if (keep && slot < capacity) row[slot] = sm.rank[k];
            if (with_mirror && keep) {
                if (bi - b0 < 32) atomicOr(&sm.bits[k], 1u << (bi - b0));
                atomicAdd(&sm.segn[warp * 32 + sm.cj[k]], 1);
                // (the staged index, for the partial below; lower entries
                // are marked, so the partial reads only this array)
                if (slot < capacity)
                    mirror[r * (int64_t)capacity + slot] = sm.rank[k] > (int)r ? k : kMirrorLower;
            }
            count += __popc(m);
        }
        if (lane == 0) {
            row_count[r] = count < capacity ? count : capacity;
            if (count > *(volatile int32_t *)max_count) atomicMax(max_count, count);
        }
        if (with_mirror) {  // directory row: survivors before each neighbour cell
            __syncwarp();
            const int v = sm.segn[warp * 32 + lane];
            int incl = v;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl += y;
            }
            dir[r * kDirStride + lane] = (uint16_t)(incl - v);
            sm.segn[warp * 32 + lane] = 0;
        }
        __syncwarp();
    }
    if (with_mirror) {
        __syncthreads();  // every particle's bits are in
        const bool search = sm.misc[3] != 0;
        for (int bi = b0 + warp; bi < b1; bi += nwarps) {
            const int64_t r = r0 + (bi - b0);
            if (dir[r * kDirStride] == kDirNone) continue;  // its rows came from nlist_one
            const int m = row_count[r];
            int32_t *mrow = mirror + r * (int64_t)capacity;
            const uint32_t below = (1u << (bi - b0 < 32 ? bi - b0 : 31)) - 1u;
            for (int k = lane; k < m; k += 32) {
                const int kk = mrow[k];
                if (kk == kMirrorLower) continue;  // only the upper entries are defined
                mrow[k] = search ? kMirrorSearch
                                 : (int32_t)(__popc(sm.bits[kk] & below) | (sm.slotc[sm.cj[kk]] << 24));
            }
        }
    }
    __syncthreads();  // the staged neighbourhood is reused by the next cell
    return true;
}

// Mirror entries of row p from the partials (one warp): pos = dir[q][slot] +
// within, -1 past the capacity (p fell off a truncated row q); the binary
// search where a partial or q's directory row is missing.
template <bool kCoherent = false>
__device__ __forceinline__ void mirror_resolve(int64_t p, int lane, const int32_t *__restrict__ rows,
                                               const int32_t *__restrict__ row_count,
                                               int32_t capacity, int32_t *__restrict__ mirror,
                                               const uint16_t *__restrict__ dir) {
    const int m = ldc<kCoherent>(row_count + p);
    const int32_t *rp = rows + p * (int64_t)capacity;
    int32_t *mp = mirror + p * (int64_t)capacity;
    const bool p_none = ldc<kCoherent>(dir + p * kDirStride) == kDirNone;
    // four entries per lane in flight (the phase is a chain of dependent
    // loads: row entry and partial, then q's directory word)
    constexpr int kU = 4;
    for (int k0 = lane; k0 < m; k0 += 32 * kU) {
        int q[kU];
        int32_t v[kU];
#pragma unroll
        for (int t = 0; t < kU; t++) {
            const int k = k0 + 32 * t;
            q[t] = k < m ? ldc<kCoherent>(rp + k) : -1;
            v[t] = k < m && !p_none ? ldc<kCoherent>(mp + k) : kMirrorSearch;
        }
        uint16_t d[kU];
#pragma unroll
        for (int t = 0; t < kU; t++) {
            const bool upper = q[t] > (int)p;
            d[t] = upper && v[t] != kMirrorSearch
                       ? ldc<kCoherent>(dir + (int64_t)q[t] * kDirStride + (v[t] >> 24))
                       : kDirNone;
        }
#pragma unroll
        for (int t = 0; t < kU; t++) {
            if (q[t] <= (int)p) continue;  // only the upper entries are defined
            int pos = -1;
            if (d[t] != kDirNone) {
                pos = (int)d[t] + (v[t] & 0xffffff);
                if (pos >= capacity) pos = -1;
            } else {  // binary search of p in the rank-sorted row q
                const int32_t *rq = rows + (int64_t)q[t] * capacity;
                int lo = 0, hi = ldc<kCoherent>(row_count + q[t]) - 1;
                while (lo <= hi) {
                    const int mid = (lo + hi) >> 1;
                    const int x = ldc<kCoherent>(rq + mid);
                    if (x == (int)p) {
                        pos = mid;
                        break;
                    }
                    if (x < (int)p) lo = mid + 1;
                    else hi = mid - 1;
                }
            }
            mp[k0 + 32 * t] = pos;
        }
    }
}

}  // namespace rb
