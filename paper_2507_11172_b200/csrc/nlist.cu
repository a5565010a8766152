// nlist.cu -- neighbour rows from the cell list.
//
// For each particle (rank order) one warp walks the canonical neighbour cells
// of its base cell (respamd/containers.py:319-333 / :403-423) as one
// flattened candidate range: lane l of a 32-wide chunk owns candidate l,
// located by a binary search over the warp-scanned cell counts.  The (at most
// 27) neighbour cells are sorted by flat id first, so every row lists its
// neighbours in ascending rank order -- the Newton-3 triplet pass relies on
// it (S+(i) is a row suffix; mirror indices come from a binary search).  The pair
// distance uses the reference arithmetic (a - b, single-shift minimum image,
// no FMA), and survivors (r^2 <= r_list^2, inclusive, self excluded) are
// appended with a ballot in candidate order, so rows are deterministic and
// equal to the reference's survivor lists (:437-474) when r_list == rc.
#include "common.cuh"

namespace rb {

constexpr int kNlistWarps = 8;

__device__ __forceinline__ void nlist_one(const rb_grid &g, int64_t r, int64_t n, const double *__restrict__ pr, const int32_t *__restrict__ cell_start,
            const int32_t *__restrict__ cell_of_rank, double rl2, int32_t capacity,
            int32_t *__restrict__ rows, int32_t *__restrict__ row_count,
            int32_t *__restrict__ max_count) {
    const int lane = threadIdx.x & 31;
    const Image im = make_image(g);
    const double xi = pr[3 * r], yi = pr[3 * r + 1], zi = pr[3 * r + 2];
    const int cb = cell_of_rank[r];
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
        cstart = cell_start[my_cell];
        ccount = cell_start[my_cell + 1] - cstart;
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
                exact_disp(im, xi, yi, zi, pr[3 * (j)], pr[3 * (j) + 1], pr[3 * (j) + 2], dx, dy, dz);
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

// grid-stride over particles (one warp each); a closed rebuild gate makes
// every block exit after one load, so the launch costs a few microseconds
__global__ void __launch_bounds__(kNlistWarps * 32)
    k_nlist(rb_grid g, int64_t n, const double *__restrict__ pr,
            const int32_t *__restrict__ cell_start, const int32_t *__restrict__ cell_of_rank,
            double rl2, int32_t capacity, int32_t *__restrict__ rows,
            int32_t *__restrict__ row_count, int32_t *__restrict__ max_count,
            const int64_t *flag, const unsigned long long *status, int64_t tag) {
    pdl_enter();
    if (flag && *(volatile const int64_t *)flag != resolve_tag(tag, status)) return;
    for (int64_t r = (int64_t)blockIdx.x * kNlistWarps + (threadIdx.x >> 5); r < n;
         r += (int64_t)gridDim.x * kNlistWarps)
        nlist_one(g, r, n, pr, cell_start, cell_of_rank, rl2, capacity, rows, row_count,
                  max_count);
}

// mirror[p][k] = position of p in the row of q = rows[p][k].  One warp per
// row p (grid-stride over rows); for each entry q > p a lane binary-searches
// p in the rank-sorted row q and writes BOTH mirror[p][k] and, by symmetry,
// mirror[q][that position] = k -- every pair is searched once.
constexpr int kMirrorWarps = 8;

__global__ void __launch_bounds__(kMirrorWarps * 32)
    k_mirror(int64_t n, const int32_t *__restrict__ rows, const int32_t *__restrict__ row_count,
             int32_t capacity, int32_t *__restrict__ mirror, const int64_t *flag,
             const unsigned long long *status, int64_t tag) {
    pdl_enter();
    if (flag && *(volatile const int64_t *)flag != resolve_tag(tag, status)) return;
    const int lane = threadIdx.x & 31;
    for (int64_t p = (int64_t)blockIdx.x * kMirrorWarps + (threadIdx.x >> 5); p < n;
         p += (int64_t)gridDim.x * kMirrorWarps) {
        const int m = row_count[p];
        const int32_t *rp = rows + p * (int64_t)capacity;
        for (int k = lane; k < m; k += 32) {
            const int q = __ldg(rp + k);
            if (q <= p) continue;  // written by the warp of row q
            const int32_t *rq = rows + (int64_t)q * capacity;
            int lo = 0, hi = row_count[q] - 1, pos = -1;
            while (lo <= hi) {
                const int mid = (lo + hi) >> 1;
                const int v = __ldg(rq + mid);
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
}

}  // namespace rb

using namespace rb;

extern "C" int rb_nlist(const rb_grid *g, int64_t n, const double *pos_r, const int32_t *cell_start, const int32_t *cell_of_rank,
                        double r_list, int32_t capacity, int32_t *rows, int32_t *row_count,
                        int32_t *max_count, const int64_t *rebuild_flag,
                        const unsigned long long *status, int64_t tag, void *stream) {
    if (!g || n < 0 || capacity <= 0 || !max_count) return RB_ERR_ARGUMENT;
    if (g->n_offsets <= 0 || g->n_offsets > RB_MAX_OFFSETS) return RB_ERR_GEOMETRY;
    if (n == 0) return RB_OK;
    const double rl2 = r_list * r_list;  // host-side rc*rc as containers.py:773
    int64_t blocks = (n + kNlistWarps - 1) / kNlistWarps;
    if (rebuild_flag && blocks > 148 * 8) blocks = 148 * 8;  // gated: grid-stride
    launch(k_nlist, dim3((unsigned)blocks), dim3(kNlistWarps * 32), 0, as_stream(stream), *g, n, pos_r, cell_start, cell_of_rank, rl2, capacity, rows, row_count, max_count,
        rebuild_flag, status, tag);
    note_launches(1);
    return launch_status();
}

extern "C" int rb_nlist_mirror(int64_t n, const int32_t *rows, const int32_t *row_count,
                               int32_t capacity, int32_t *mirror, const int64_t *rebuild_flag,
                               const unsigned long long *status, int64_t tag, void *stream) {
    if (n < 0 || capacity <= 0 || !rows || !row_count || !mirror) return RB_ERR_ARGUMENT;
    if (n == 0) return RB_OK;
    int64_t mblocks = (n + kMirrorWarps - 1) / kMirrorWarps;
    if (rebuild_flag && mblocks > 148 * 8) mblocks = 148 * 8;  // gated: grid-stride
    launch(k_mirror, dim3((unsigned)mblocks), dim3(kMirrorWarps * 32), 0, as_stream(stream), n,
           rows, row_count, capacity, mirror, rebuild_flag, status, tag);
    note_launches(1);
    return launch_status();
}
