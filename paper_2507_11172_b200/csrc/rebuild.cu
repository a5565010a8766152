#include <cstdlib>
// rebuild.cu -- the gated row rebuild of a captured r-RESPA step as ONE launch.
//
// Inside a captured step the rebuild (binning, rows, mirror: nine kernels)
// runs only when the step's drift flagged it.  Nine gated launches cost ~10 us
// of launch latency per step, a graph conditional node ~6 us; this kernel
// costs one PDL launch that exits at the gate.  When the gate is open it runs
// the same phases as rb_bin + rb_nlist + rb_nlist_mirror (identical results:
// the same device functions, cells.cuh), separated by grid-wide barriers:
//
//   zero counts | count | tile sums | tile offsets | scan apply | scatter |
//   cell finish (stable order, rank-ordered copy) | rows | mirror
//
// The grid is the co-resident capacity (occupancy x SMs of the current
// device) and the launch is cooperative (launch_coop): the driver makes
// every block resident before any runs, so the software barrier (count +
// generation words in the scratch) cannot wait on a block that is not
// scheduled -- not behind kernels of other streams, processes or MPS
// clients.  Data written by an earlier phase is read with L2-coherent loads
// (ldc<true>).
#include <algorithm>

#include "cells.cuh"

namespace rb {

constexpr int kRbThreads = 256;
constexpr int kRbItems = 4;
constexpr int kRbTile = kRbThreads * kRbItems;  // cells per scan tile
constexpr int kRbChunkMax = 8;  // ranks per counter grab (rows and mirror phases), at most

__device__ __forceinline__ void grid_barrier(unsigned *count, unsigned *gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g0 = *(volatile unsigned *)gen;
        __threadfence();
        if (atomicAdd(count, 1u) == gridDim.x - 1) {
            atomicExch(count, 0u);  // reusable: the next barrier counts from 0
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            while (*(volatile unsigned *)gen == g0) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

// phase profiling (RB_REBUILD_STOP=k: the kernel returns after phase k;
// timing experiments only, results are then incomplete)
__device__ int g_rebuild_stop = 99;

__global__ void __launch_bounds__(kRbThreads)
    k_rebuild(rb_grid g, int64_t n, const double *__restrict__ pos, int32_t *cell_start,
              int32_t *parts, int32_t *cell_of_rank, double *pr, int32_t *rank_of, double *x_ref,
              double rl2, int32_t capacity, int32_t *rows, int32_t *row_count,
              int32_t *max_count, int32_t *mirror, int32_t *cell_of, int32_t *count,
              int32_t *cursor, int32_t *tiles, unsigned *bar, uint16_t *dir, const int64_t *flag,
              const unsigned long long *status, int64_t tag, int32_t nb_cap, float hi_f) {
    pdl_enter();
    if (gate_closed(flag, status, tag)) return;  // the same answer in every block
    __shared__ int warp_sums[32];
    __shared__ int cell_grab;
    extern __shared__ __align__(16) char rows_smem[];
    const int64_t ncell = (int64_t)g.cells[0] * g.cells[1] * g.cells[2];
    const int64_t ntiles = (ncell + kRbTile - 1) / kRbTile;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    const int64_t warp = tid >> 5, nwarp = nth >> 5;
    unsigned *bcount = bar, *bgen = bar + 1;

    const int stop = g_rebuild_stop;
    unsigned long long *work = (unsigned long long *)(bar + 4);  // chunk counters (rows, mirror)
    if (tid == 0) work[0] = work[1] = 0;  // read only after later barriers
    // chunk: 1 rank per grab while there are few ranks per warp (the chunk is
    // the critical path), up to kRbChunkMax at 16+ ranks per warp
    const int64_t per_warp = n / (nwarp > 0 ? nwarp : 1);
    const int kRbChunk = per_warp >= 16 * kRbChunkMax ? kRbChunkMax
                         : (per_warp >= 32 ? (int)(per_warp / 16) : 1);
    for (int64_t c = tid; c < ncell; c += nth) count[c] = 0;
    if (stop <= 1) return;
    grid_barrier(bcount, bgen);
    // cell of every particle + histogram (bin.cu k_bin_count)
    for (int64_t i = tid; i < n; i += nth) {
        const int cx = cell_index(g, 0, pos[3 * i]);
        const int cy = cell_index(g, 1, pos[3 * i + 1]);
        const int cz = cell_index(g, 2, pos[3 * i + 2]);
        const int c = (cx * g.cells[1] + cy) * g.cells[2] + cz;
        cell_of[i] = c;
        atomicAdd(&count[c], 1);
    }
    if (stop <= 2) return;
    grid_barrier(bcount, bgen);
    // exclusive scan of the counts: tile sums, tile offsets, apply
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int s = 0;
#pragma unroll
        for (int k = 0; k < kRbItems; k++) {
            const int64_t i = t * kRbTile + (int64_t)threadIdx.x * kRbItems + k;
            if (i < ncell) s += ldc<true>(count + i);
        }
        int total;
        block_exclusive_scan(s, warp_sums, total);
        if (threadIdx.x == 0) tiles[t] = total;
    }
    if (stop <= 3) return;
    grid_barrier(bcount, bgen);
    if (blockIdx.x == 0) {
        int carry = 0;
        for (int64_t base = 0; base < ntiles; base += blockDim.x) {
            const int64_t i = base + threadIdx.x;
            const int v = i < ntiles ? ldc<true>(tiles + i) : 0;
            int total;
            const int ex = block_exclusive_scan(v, warp_sums, total);
            if (i < ntiles) tiles[i] = carry + ex;
            carry += total;
        }
    }
    if (stop <= 4) return;
    grid_barrier(bcount, bgen);
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int vals[kRbItems];
        int s = 0;
#pragma unroll
        for (int k = 0; k < kRbItems; k++) {
            const int64_t i = t * kRbTile + (int64_t)threadIdx.x * kRbItems + k;
            vals[k] = i < ncell ? ldc<true>(count + i) : 0;
            s += vals[k];
        }
        int total;
        int ex = block_exclusive_scan(s, warp_sums, total) + ldc<true>(tiles + t);
#pragma unroll
        for (int k = 0; k < kRbItems; k++) {
            const int64_t i = t * kRbTile + (int64_t)threadIdx.x * kRbItems + k;
            if (i < ncell) {
                cell_start[i] = ex;
                cursor[i] = ex;
            }
            ex += vals[k];
            if (i == ncell - 1) cell_start[ncell] = ex;
        }
    }
    if (stop <= 5) return;
    grid_barrier(bcount, bgen);
    // unordered scatter into the cell ranges (bin.cu k_bin_scatter)
    for (int64_t i = tid; i < n; i += nth) {
        const int slot = atomicAdd(&cursor[ldc<true>(cell_of + i)], 1);
        parts[slot] = (int32_t)i;
    }
    if (stop <= 6) return;
    grid_barrier(bcount, bgen);
    for (int64_t c = warp; c < ncell; c += nwarp)
        cell_finish_one<true>(c, lane, cell_start, parts, cell_of_rank, rank_of, pos, pr, x_ref);
    if (stop <= 7) return;
    grid_barrier(bcount, bgen);
    // rows: blocks take cells from a counter (cells.cuh nlist_cell: the cell's
    // neighbourhood staged in shared memory, one row per particle; the cells
    // in flight stay a compact window, so their neighbourhoods stay in L2);
    // nb_cap == 0 or a neighbourhood over it: warps per particle (nlist_one)
    if (nb_cap > 0) {
        const RowsSmem sm = rows_carve(rows_smem, nb_cap);
        const int wib = threadIdx.x >> 5, nwb = blockDim.x >> 5;
        for (;;) {
            if (threadIdx.x == 0) cell_grab = (int)atomicAdd(&work[0], 1ull);
            __syncthreads();
            const int c = cell_grab;
            __syncthreads();
            if (c >= ncell) break;
            if (!nlist_cell<true>(g, c, pr, cell_start, rl2, hi_f, capacity, rows, row_count,
                                  max_count, sm, nb_cap, mirror, dir)) {
                const int b = ldc<true>(cell_start + c), e = ldc<true>(cell_start + c + 1);
                for (int r = b + wib; r < e; r += nwb) {
                    nlist_one<true>(g, r, n, pr, cell_start, cell_of_rank, rl2, capacity, rows,
                                    row_count, max_count, c);
                    dir[(int64_t)r * kDirStride + lane] = kDirNone;  // mirror: searched
                }
                __syncthreads();
            }
        }
    } else {
        for (;;) {
            unsigned long long b0 = 0;
            if (lane == 0) b0 = atomicAdd(&work[0], (unsigned long long)kRbChunk);
            const int64_t b = (int64_t)__shfl_sync(0xffffffffu, b0, 0);
            if (b >= n) break;
            const int64_t e = b + kRbChunk < n ? b + kRbChunk : n;
            for (int64_t r = b; r < e; r++)
                nlist_one<true>(g, r, n, pr, cell_start, cell_of_rank, rl2, capacity, rows,
                                row_count, max_count);
        }
    }
    if (stop <= 8) return;
    grid_barrier(bcount, bgen);
    for (;;) {
        unsigned long long b0 = 0;
        if (lane == 0) b0 = atomicAdd(&work[1], (unsigned long long)kRbChunk);
        const int64_t b = (int64_t)__shfl_sync(0xffffffffu, b0, 0);
        if (b >= n) break;
        const int64_t e = b + kRbChunk < n ? b + kRbChunk : n;
        // staged rows: the partials + directory (cells.cuh mirror_resolve)
        if (nb_cap > 0)
            for (int64_t p = b; p < e; p++)
                mirror_resolve<true>(p, lane, rows, row_count, capacity, mirror, dir);
        else
            for (int64_t p = b; p < e; p++) mirror_one<true>(p, lane, rows, row_count, capacity, mirror);
    }
}

static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

// co-resident blocks of k_rebuild at `smem` dynamic bytes on the current
// device (the cooperative launch's grid)
static int rebuild_grid(size_t smem) {
    constexpr int kMaxDev = 64;
    static int blocks[kMaxDev] = {0};  // per device
    static size_t at[kMaxDev] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    const int d = dev < kMaxDev ? dev : kMaxDev - 1;
    if (!blocks[d] || at[d] != smem) {
        int sms = 0, per = 0;
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(k_rebuild, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_rebuild, kRbThreads, smem);
        blocks[d] = std::max(1, sms) * std::max(1, per);
        at[d] = smem;
    }
    return blocks[d];
}

}  // namespace rb

using namespace rb;

// scratch: barrier words (zero-filled once by the caller) | cell_of[n] |
// count[ncell] | cursor[ncell] | tile sums | mirror directory[n][32] (uint16)
extern "C" size_t rb_rebuild_scratch_bytes(int64_t n, int64_t ncell) {
    const int64_t ntiles = (std::max<int64_t>(ncell, 1) + kRbTile - 1) / kRbTile;
    return 256 + align256(sizeof(int32_t) * (size_t)std::max<int64_t>(n, 1)) +
           2 * align256(sizeof(int32_t) * (size_t)std::max<int64_t>(ncell, 1)) +
           align256(sizeof(int32_t) * (size_t)ntiles) +
           align256(sizeof(uint16_t) * kDirStride * (size_t)std::max<int64_t>(n, 1));
}

extern "C" int rb_rebuild(const rb_grid *g, int64_t n, const double *pos, int32_t *cell_start,
                          int32_t *cell_particles, int32_t *cell_of_rank, double *pos_r,
                          int32_t *rank_of, double *x_ref, double r_list, int32_t capacity,
                          int32_t *rows, int32_t *row_count, int32_t *max_count, int32_t *mirror,
                          const int64_t *rebuild_flag, const unsigned long long *status,
                          int64_t tag, void *scratch, size_t scratch_bytes, void *stream) {
    NvtxRange nvtx_range("rebuild (rb_rebuild)");
    if (!g || n < 0 || capacity <= 0 || !max_count || !rows || !row_count || !mirror || !scratch)
        return RB_ERR_ARGUMENT;
    if (g->n_offsets <= 0 || g->n_offsets > RB_MAX_OFFSETS) return RB_ERR_GEOMETRY;
    const int64_t ncell = (int64_t)g->cells[0] * g->cells[1] * g->cells[2];
    if (ncell <= 0) return RB_ERR_GEOMETRY;
    if (scratch_bytes < rb_rebuild_scratch_bytes(n, ncell)) return RB_ERR_ARGUMENT;
    if (n == 0) return RB_OK;
    char *p = (char *)scratch;
    unsigned *bar = (unsigned *)p;
    p += 256;
    int32_t *cell_of = (int32_t *)p;
    p += align256(sizeof(int32_t) * (size_t)n);
    int32_t *count = (int32_t *)p;
    p += align256(sizeof(int32_t) * (size_t)ncell);
    int32_t *cursor = (int32_t *)p;
    p += align256(sizeof(int32_t) * (size_t)ncell);
    int32_t *tiles = (int32_t *)p;
    p += align256(sizeof(int32_t) * (size_t)((ncell + kRbTile - 1) / kRbTile));
    uint16_t *dir = (uint16_t *)p;
    const double rl2 = r_list * r_list;  // host-side rc*rc as containers.py:773
    static const int stop = getenv("RB_REBUILD_STOP") ? atoi(getenv("RB_REBUILD_STOP")) : 0;
    if (stop > 0) cudaMemcpyToSymbol(g_rebuild_stop, &stop, sizeof(int));
    static const bool staged = !(getenv("RB_ROWS_STAGED") && atoi(getenv("RB_ROWS_STAGED")) == 0);
    const int nb_cap = staged && rows_staged_ok(*g) ? rows_nb_cap(n, ncell) : 0;
    const size_t smem = nb_cap > 0 ? rows_smem_bytes(nb_cap, kRbThreads / 32) : 0;
    const float hi_f = (float)(rl2 * (1.0 + 1e-3));
    launch_coop(k_rebuild, dim3((unsigned)rebuild_grid(smem)), dim3(kRbThreads), smem, as_stream(stream), *g,
           n, pos, cell_start, cell_particles, cell_of_rank, pos_r, rank_of, x_ref, rl2, capacity,
           rows, row_count, max_count, mirror, cell_of, count, cursor, tiles, bar, dir, rebuild_flag,
           status, tag, nb_cap, hi_f);
    note_launches(1);
    return launch_status();
}
