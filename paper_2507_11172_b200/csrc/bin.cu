// bin.cu -- linked-cell binning as a counting sort by cell index.
//
// Replaces respamd/containers.py:175-209 (_bin_particles).  The cell index is
// the reference's truncating int((x - origin) * inv_cell) clamped to
// [0, n-1] (:182-196), the flat id is (cx*ny + cy)*nz + cz (:197), and the
// order inside a cell is ascending particle index (the reference's serial
// stable scatter, :203-208).  Four HBM-bound passes:
//
//   k_bin_count    cell id per particle + histogram (integer atomics)
//   scan           exclusive scan of the histogram -> cell_start
//   k_bin_scatter  unordered scatter into the cell ranges
//   k_cell_finish  per-cell insertion sort by particle index (restores the
//                  reference's stable order) + gather of positions into rank
//                  order (SoA) and the rank -> cell map
#include <algorithm>

#include "cells.cuh"

namespace rb {

__global__ void k_bin_zero(int64_t ncell, int32_t *__restrict__ count, const int64_t *flag,
                           const unsigned long long *status, int64_t tag) {
    pdl_enter();
    if (gate_closed(flag, status, tag)) return;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < ncell;
         c += (int64_t)gridDim.x * blockDim.x)
        count[c] = 0;
}

__global__ void k_bin_count(rb_grid g, int64_t n, const double *__restrict__ pos,
                            int32_t *__restrict__ cell_of, int32_t *__restrict__ count,
                            const int64_t *flag, const unsigned long long *status, int64_t tag) {
    pdl_enter();
    if (gate_closed(flag, status, tag)) return;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double x = pos[3 * i], y = pos[3 * i + 1], z = pos[3 * i + 2];
        int cx = cell_index(g, 0, x);
        int cy = cell_index(g, 1, y);
        int cz = cell_index(g, 2, z);
        int c = (cx * g.cells[1] + cy) * g.cells[2] + cz;
        cell_of[i] = c;
        atomicAdd(&count[c], 1);
    }
}

__global__ void k_bin_scatter(int64_t n, const int32_t *__restrict__ cell_of,
                              int32_t *__restrict__ cursor, int32_t *__restrict__ parts,
                              const int64_t *flag, const unsigned long long *status, int64_t tag) {
    pdl_enter();
    if (gate_closed(flag, status, tag)) return;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int slot = atomicAdd(&cursor[cell_of[i]], 1);
        parts[slot] = (int32_t)i;
    }
}

constexpr int kFinishWarps = 8;

__global__ void __launch_bounds__(kFinishWarps * 32)
    k_cell_finish(int64_t ncell, const int32_t *__restrict__ start, int32_t *__restrict__ parts,
                  int32_t *__restrict__ cell_of_rank, int32_t *__restrict__ rank_of,
                  const double *__restrict__ pos, double *__restrict__ pr,
                  double *__restrict__ x_ref, const int64_t *flag,
                  const unsigned long long *status, int64_t tag) {
    pdl_enter();
    const int lane = threadIdx.x & 31;
    if (gate_closed(flag, status, tag)) return;
    for (int64_t c = (int64_t)blockIdx.x * kFinishWarps + (threadIdx.x >> 5); c < ncell;
         c += (int64_t)gridDim.x * kFinishWarps)
        cell_finish_one(c, lane, start, parts, cell_of_rank, rank_of, pos, pr, x_ref);
}

// ---------------------------------------------------------------------------
// exclusive scan of int32 counts into out[0..n] (out[n] = total)
// three phases: per-tile sums, scan of tile sums (one CTA), per-tile scan
// ---------------------------------------------------------------------------
__global__ void k_scan_tile_sums(int64_t n, const int32_t *__restrict__ in,
                                 int32_t *__restrict__ tile_sums, const int64_t *flag,
                                 const unsigned long long *status, int64_t tag) {
    pdl_enter();
    __shared__ int warp_sums[32];
    if (gate_closed(flag, status, tag)) return;
    int64_t base = (int64_t)blockIdx.x * kScanTile;
    int s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        int64_t i = base + (int64_t)threadIdx.x * kScanItems + k;
        if (i < n) s += in[i];
    }
    int total;
    block_exclusive_scan(s, warp_sums, total);
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

__global__ void k_scan_tile_offsets(int64_t ntiles, int32_t *__restrict__ tile_sums,
                                    const int64_t *flag, const unsigned long long *status,
                                    int64_t tag) {
    pdl_enter();
    __shared__ int warp_sums[32];
    if (gate_closed(flag, status, tag)) return;
    int carry = 0;
    for (int64_t base = 0; base < ntiles; base += blockDim.x) {
        int64_t i = base + threadIdx.x;
        int v = i < ntiles ? tile_sums[i] : 0;
        int total;
        int ex = block_exclusive_scan(v, warp_sums, total);
        if (i < ntiles) tile_sums[i] = carry + ex;
        carry += total;
    }
}

__global__ void k_scan_apply(int64_t n, const int32_t *__restrict__ in,
                             const int32_t *__restrict__ tile_off, int32_t *__restrict__ out,
                             int32_t *__restrict__ cursor, const int64_t *flag,
                             const unsigned long long *status, int64_t tag) {
    pdl_enter();
    __shared__ int warp_sums[32];
    if (gate_closed(flag, status, tag)) return;
    int64_t base = (int64_t)blockIdx.x * kScanTile;
    int vals[kScanItems];
    int s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        int64_t i = base + (int64_t)threadIdx.x * kScanItems + k;
        vals[k] = i < n ? in[i] : 0;
        s += vals[k];
    }
    int total;
    int ex = block_exclusive_scan(s, warp_sums, total) + tile_off[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        int64_t i = base + (int64_t)threadIdx.x * kScanItems + k;
        if (i < n) {
            out[i] = ex;
            cursor[i] = ex;
        }
        ex += vals[k];
        if (i == n - 1) out[n] = ex;
    }
}

static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// scratch layout: cell_of[n] | count[ncell] | cursor[ncell] | tiles[ntiles]
static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

}  // namespace rb

using namespace rb;

extern "C" size_t rb_bin_scratch_bytes(int64_t n, int64_t ncell) {
    int64_t ntiles = ceil_div(ncell > 0 ? ncell : 1, kScanTile);
    return align256(sizeof(int32_t) * (size_t)(n > 0 ? n : 1)) +
           2 * align256(sizeof(int32_t) * (size_t)ncell) +
           align256(sizeof(int32_t) * (size_t)ntiles);
}

extern "C" int rb_bin(const rb_grid *g, int64_t n, const double *pos, int32_t *cell_start,
                      int32_t *cell_particles, int32_t *cell_of_rank, double *pos_r,
                      int32_t *rank_of, double *x_ref, const int64_t *rebuild_flag,
                      const unsigned long long *status, int64_t tag, void *scratch,
                      size_t scratch_bytes, void *stream) {
    NvtxRange nvtx_range("bin (rb_bin)");
    if (!g || n < 0) return RB_ERR_ARGUMENT;
    int64_t ncell = (int64_t)g->cells[0] * g->cells[1] * g->cells[2];
    if (ncell <= 0) return RB_ERR_GEOMETRY;
    if (scratch_bytes < rb_bin_scratch_bytes(n, ncell)) return RB_ERR_ARGUMENT;
    cudaStream_t st = as_stream(stream);
    char *p = (char *)scratch;
    int32_t *cell_of = (int32_t *)p;
    p += align256(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    int32_t *count = (int32_t *)p;
    p += align256(sizeof(int32_t) * (size_t)ncell);
    int32_t *cursor = (int32_t *)p;
    p += align256(sizeof(int32_t) * (size_t)ncell);
    int32_t *tiles = (int32_t *)p;
    int64_t ntiles = ceil_div(ncell, kScanTile);
    const int64_t *fl = rebuild_flag;
    const int tb = 256;
    // gated launches use capped grid-stride grids so a closed gate is cheap
    auto cap = [&](int64_t b) { return (unsigned)(fl && b > 148 * 8 ? 148 * 8 : b); };
    launch(k_bin_zero, dim3((unsigned)std::min<int64_t>(ceil_div(ncell, tb), 148 * 8)), dim3(tb), 0, st, ncell, count, fl, status, tag);
    note_launches(1);
    if (n > 0) {
        launch(k_bin_count, dim3(cap(ceil_div(n, tb))), dim3(tb), 0, st, *g, n, pos, cell_of, count, fl,
                                                               status, tag);
        note_launches(1);
    }
    launch(k_scan_tile_sums, dim3((unsigned)ntiles), dim3(kScanThreads), 0, st, ncell, count, tiles, fl, status,
                                                                 tag);
    note_launches(1);
    launch(k_scan_tile_offsets, dim3(1), dim3(1024), 0, st, ntiles, tiles, fl, status, tag);
    note_launches(1);
    launch(k_scan_apply, dim3((unsigned)ntiles), dim3(kScanThreads), 0, st, ncell, count, tiles, cell_start,
                                                             cursor, fl, status, tag);
    note_launches(1);
    if (n > 0) {
        launch(k_bin_scatter, dim3(cap(ceil_div(n, tb))), dim3(tb), 0, st, n, cell_of, cursor,
                                                                 cell_particles, fl, status, tag);
        note_launches(1);
        launch(k_cell_finish, dim3(cap(ceil_div(ncell, kFinishWarps))), dim3(kFinishWarps * 32), 0, st, ncell, cell_start, cell_particles, cell_of_rank, rank_of, pos, pos_r, x_ref, fl,
            status, tag);
        note_launches(1);
    }
    return launch_status();
}
