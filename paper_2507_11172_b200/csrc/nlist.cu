// nlist.cu -- neighbour rows from the cell list.
//
// For each particle (rank order) one warp walks the canonical neighbour cells
// of its base cell (respamd/containers.py:319-333 / :403-423) as one
// flattened candidate range: lane l of a 32-wide chunk owns candidate l,
// located by a binary search over the warp-scanned cell counts.  The pair
// distance uses the reference arithmetic (a - b, single-shift minimum image,
// no FMA), and survivors (r^2 <= r_list^2, inclusive, self excluded) are
// appended with a ballot in candidate order, so rows are deterministic and
// equal to the reference's survivor lists (:437-474) when r_list == rc.
#include "common.cuh"

namespace rb {

constexpr int kNlistWarps = 8;

__global__ void __launch_bounds__(kNlistWarps * 32)
    k_nlist(rb_grid g, int64_t n, const double *__restrict__ xs, const double *__restrict__ ys,
            const double *__restrict__ zs, const int32_t *__restrict__ cell_start,
            const int32_t *__restrict__ cell_of_rank, double rl2, int32_t capacity,
            int32_t *__restrict__ rows, int32_t *__restrict__ row_count,
            int32_t *__restrict__ max_count) {
    const int lane = threadIdx.x & 31;
    const int64_t r = (int64_t)blockIdx.x * kNlistWarps + (threadIdx.x >> 5);
    if (r >= n) return;
    const Image im = make_image(g);
    const double xi = xs[r], yi = ys[r], zi = zs[r];
    const int cb = cell_of_rank[r];
    const int cbz = cb % g.cells[2];
    const int cby = (cb / g.cells[2]) % g.cells[1];
    const int cbx = cb / (g.cells[2] * g.cells[1]);
    int32_t *row = rows + r * (int64_t)capacity;
    int count = 0;
    for (int ob = 0; ob < g.n_offsets; ob += 32) {
        int o = ob + lane;
        int cstart = 0, ccount = 0;
        if (o < g.n_offsets) {
            int cc = neighbor_cell(g, cbx, cby, cbz, o);
            if (cc >= 0) {
                cstart = cell_start[cc];
                ccount = cell_start[cc + 1] - cstart;
            }
        }
        // inclusive scan of the chunk's cell counts
        int incl = ccount;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += y;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        for (int base = 0; base < total; base += 32) {
            const int cand = base + lane;
            // owner lane of cand: first lane whose inclusive prefix exceeds cand
            int pos = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                int v = __shfl_sync(0xffffffffu, incl, pos + step - 1);
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
                    exact_disp(im, xi, yi, zi, xs[j], ys[j], zs[j], dx, dy, dz);
                    keep = exact_r2(dx, dy, dz) <= rl2;
                }
            }
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            const int slot = count + __popc(m & lanemask_lt());
            if (keep && slot < capacity) row[slot] = j;
            count += __popc(m);
        }
    }
    if (lane == 0) {
        row_count[r] = count < capacity ? count : capacity;
        if (count > capacity) atomicMax(max_count, count);
    }
}

}  // namespace rb

using namespace rb;

extern "C" int rb_nlist(const rb_grid *g, int64_t n, const double *xs, const double *ys,
                        const double *zs, const int32_t *cell_start, const int32_t *cell_of_rank,
                        double r_list, int32_t capacity, int32_t *rows, int32_t *row_count,
                        int32_t *max_count, void *stream) {
    if (!g || n < 0 || capacity <= 0 || !max_count) return RB_ERR_ARGUMENT;
    if (g->n_offsets <= 0 || g->n_offsets > RB_MAX_OFFSETS) return RB_ERR_GEOMETRY;
    if (n == 0) return RB_OK;
    const double rl2 = r_list * r_list;  // host-side rc*rc as containers.py:773
    unsigned blocks = (unsigned)((n + kNlistWarps - 1) / kNlistWarps);
    k_nlist<<<blocks, kNlistWarps * 32, 0, as_stream(stream)>>>(
        *g, n, xs, ys, zs, cell_start, cell_of_rank, rl2, capacity, rows, row_count, max_count);
    note_launches(1);
    return launch_status();
}
