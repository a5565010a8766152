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
// By default the rows come from k_nlist_cells (cells.cuh nlist_cell: one CTA
// per cell, the neighbourhood staged in shared memory, identical rows);
// RB_ROWS_STAGED=0 keeps the warp-per-particle k_nlist.
#include <cstdlib>

#include "cells.cuh"

namespace rb {

constexpr int kNlistWarps = 8;

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

// Cell-staged rows (cells.cuh nlist_cell): one CTA per cell (grid-stride);
// a neighbourhood over nb_cap takes the per-particle path.
constexpr int kRowsWarps = 8;

__global__ void __launch_bounds__(kRowsWarps * 32)
    k_nlist_cells(rb_grid g, int32_t ncell, const double *__restrict__ pr,
                  const int32_t *__restrict__ cell_start, double rl2, float hi_f,
                  int32_t capacity, int32_t *__restrict__ rows, int32_t *__restrict__ row_count,
                  int32_t *__restrict__ max_count, int32_t nb_cap, int32_t *__restrict__ mirror,
                  uint16_t *__restrict__ dir, const int64_t *flag,
                  const unsigned long long *status, int64_t tag) {
    pdl_enter();
    if (flag && *(volatile const int64_t *)flag != resolve_tag(tag, status)) return;
    extern __shared__ __align__(16) char smem[];
    const RowsSmem sm = rows_carve(smem, nb_cap);
    const int warp = threadIdx.x >> 5;
    for (int c = blockIdx.x; c < ncell; c += gridDim.x) {
        if (!nlist_cell<false>(g, c, pr, cell_start, rl2, hi_f, capacity, rows, row_count,
                               max_count, sm, nb_cap, mirror, dir)) {
            const int b = cell_start[c], e = cell_start[c + 1];
            for (int r = b + warp; r < e; r += kRowsWarps) {
                nlist_one(g, r, 0, pr, cell_start, nullptr, rl2, capacity, rows, row_count,
                          max_count, c);
                if (dir) dir[(int64_t)r * kDirStride + (threadIdx.x & 31)] = kDirNone;
            }
            __syncthreads();
        }
    }
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
         p += (int64_t)gridDim.x * kMirrorWarps)
        mirror_one(p, lane, rows, row_count, capacity, mirror);
}

// mirror from the staged rows' partials and directory (cells.cuh)
__global__ void __launch_bounds__(kMirrorWarps * 32)
    k_mirror_resolve(int64_t n, const int32_t *__restrict__ rows,
                     const int32_t *__restrict__ row_count, int32_t capacity,
                     int32_t *__restrict__ mirror, const uint16_t *__restrict__ dir,
                     const int64_t *flag, const unsigned long long *status, int64_t tag) {
    pdl_enter();
    if (flag && *(volatile const int64_t *)flag != resolve_tag(tag, status)) return;
    const int lane = threadIdx.x & 31;
    for (int64_t p = (int64_t)blockIdx.x * kMirrorWarps + (threadIdx.x >> 5); p < n;
         p += (int64_t)gridDim.x * kMirrorWarps)
        mirror_resolve(p, lane, rows, row_count, capacity, mirror, dir);
}

}  // namespace rb

using namespace rb;

// rows (and, with mirror + dir, the staged path's mirror partials and
// directory); *staged_out: whether the staged path ran
static int nlist_launch(const rb_grid *g, int64_t n, const double *pos_r,
                        const int32_t *cell_start, const int32_t *cell_of_rank, double r_list,
                        int32_t capacity, int32_t *rows, int32_t *row_count, int32_t *max_count,
                        int32_t *mirror, uint16_t *dir, const int64_t *rebuild_flag,
                        const unsigned long long *status, int64_t tag, void *stream,
                        bool *staged_out) {
    *staged_out = false;
    if (!g || n < 0 || capacity <= 0 || !max_count) return RB_ERR_ARGUMENT;
    if (g->n_offsets <= 0 || g->n_offsets > RB_MAX_OFFSETS) return RB_ERR_GEOMETRY;
    if (n == 0) return RB_OK;
    const double rl2 = r_list * r_list;  // host-side rc*rc as containers.py:773
    static const bool staged = !(getenv("RB_ROWS_STAGED") && atoi(getenv("RB_ROWS_STAGED")) == 0);
    const int64_t ncell = (int64_t)g->cells[0] * g->cells[1] * g->cells[2];
    if (staged && rows_staged_ok(*g)) {
        const int nb_cap = rows_nb_cap(n, ncell);
        const size_t bytes = rows_smem_bytes(nb_cap, kRowsWarps);
        static size_t granted = 0;
        if (bytes > 48 * 1024 && bytes > granted) {
            cudaFuncSetAttribute(k_nlist_cells, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)bytes);
            granted = bytes;
        }
        int64_t blocks = ncell < 148 * 16 ? ncell : 148 * 16;
        launch(k_nlist_cells, dim3((unsigned)blocks), dim3(kRowsWarps * 32), bytes,
               as_stream(stream), *g, (int32_t)ncell, pos_r, cell_start, rl2,
               (float)(rl2 * (1.0 + 1e-3)), capacity, rows, row_count, max_count, nb_cap,
               mirror, dir, rebuild_flag, status, tag);
        note_launches(1);
        *staged_out = true;
        return launch_status();
    }
    int64_t blocks = (n + kNlistWarps - 1) / kNlistWarps;
    if (rebuild_flag && blocks > 148 * 8) blocks = 148 * 8;  // gated: grid-stride
    launch(k_nlist, dim3((unsigned)blocks), dim3(kNlistWarps * 32), 0, as_stream(stream), *g, n, pos_r, cell_start, cell_of_rank, rl2, capacity, rows, row_count, max_count,
        rebuild_flag, status, tag);
    note_launches(1);
    return launch_status();
}

extern "C" int rb_nlist(const rb_grid *g, int64_t n, const double *pos_r, const int32_t *cell_start, const int32_t *cell_of_rank,
                        double r_list, int32_t capacity, int32_t *rows, int32_t *row_count,
                        int32_t *max_count, const int64_t *rebuild_flag,
                        const unsigned long long *status, int64_t tag, void *stream) {
    NvtxRange nvtx_range("rows (rb_nlist)");
    bool staged = false;
    return nlist_launch(g, n, pos_r, cell_start, cell_of_rank, r_list, capacity, rows, row_count,
                        max_count, nullptr, nullptr, rebuild_flag, status, tag, stream, &staged);
}

extern "C" size_t rb_nlist_mirror_scratch_bytes(int64_t n) {
    return sizeof(uint16_t) * kDirStride * (size_t)(n > 0 ? n : 1);
}

extern "C" int rb_nlist_rows_mirror(const rb_grid *g, int64_t n, const double *pos_r,
                                    const int32_t *cell_start, const int32_t *cell_of_rank,
                                    double r_list, int32_t capacity, int32_t *rows,
                                    int32_t *row_count, int32_t *max_count, int32_t *mirror,
                                    void *scratch, size_t scratch_bytes,
                                    const int64_t *rebuild_flag,
                                    const unsigned long long *status, int64_t tag, void *stream) {
    NvtxRange nvtx_range("rows + mirror (rb_nlist_rows_mirror)");
    if (!mirror || !scratch || scratch_bytes < rb_nlist_mirror_scratch_bytes(n))
        return RB_ERR_ARGUMENT;
    uint16_t *dir = (uint16_t *)scratch;
    bool staged = false;
    int st = nlist_launch(g, n, pos_r, cell_start, cell_of_rank, r_list, capacity, rows,
                          row_count, max_count, mirror, dir, rebuild_flag, status, tag, stream,
                          &staged);
    if (st != RB_OK || n == 0) return st;
    if (!staged)
        return rb_nlist_mirror(n, rows, row_count, capacity, mirror, rebuild_flag, status, tag,
                               stream);
    int64_t mblocks = (n + kMirrorWarps - 1) / kMirrorWarps;
    if (rebuild_flag && mblocks > 148 * 8) mblocks = 148 * 8;  // gated: grid-stride
    launch(k_mirror_resolve, dim3((unsigned)mblocks), dim3(kMirrorWarps * 32), 0,
           as_stream(stream), n, rows, row_count, capacity, mirror, (const uint16_t *)dir,
           rebuild_flag, status, tag);
    note_launches(1);
    return launch_status();
}

extern "C" int rb_nlist_mirror(int64_t n, const int32_t *rows, const int32_t *row_count,
                               int32_t capacity, int32_t *mirror, const int64_t *rebuild_flag,
                               const unsigned long long *status, int64_t tag, void *stream) {
    NvtxRange nvtx_range("rows mirror (rb_nlist_mirror)");
    if (n < 0 || capacity <= 0 || !rows || !row_count || !mirror) return RB_ERR_ARGUMENT;
    if (n == 0) return RB_OK;
    int64_t mblocks = (n + kMirrorWarps - 1) / kMirrorWarps;
    if (rebuild_flag && mblocks > 148 * 8) mblocks = 148 * 8;  // gated: grid-stride
    launch(k_mirror, dim3((unsigned)mblocks), dim3(kMirrorWarps * 32), 0, as_stream(stream), n,
           rows, row_count, capacity, mirror, rebuild_flag, status, tag);
    note_launches(1);
    return launch_status();
}
