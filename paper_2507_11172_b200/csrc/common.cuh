// common.cuh -- shared device helpers for the sm_100a force-evaluation path.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include "../../include/respa_b200.h"

#define RB_MIN_DISTANCE_SQ (1e-10 * 1e-10)  // respamd/potentials.py:35-36

// Bounds checks of the checked build (-DRB_CHECKED, tools/checked_build.sh):
// every index-computed shared / global access of the hot kernels is
// checked and a violation printed (no trap: the run goes on and the test
// log is grepped for "RB_CHECK failed").  compute-sanitizer is closed on
// this pool; these checks plus the CPU-oracle comparisons stand in for it.
#ifdef RB_CHECKED
#include <cstdio>
#define RB_CHECK(c)                                                                          \
    do {                                                                                     \
        if (!(c)) printf("RB_CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c);             \
    } while (0)
#else
#define RB_CHECK(c) ((void)0)
#endif

namespace rb {

constexpr int kWarp = 32;

static inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// NVTX range around a C-ABI entry point (its launches): the phases of a
// step -- bin / rebuild, pair, triplet, kick / drift, halo -- show up by
// name under Nsight Systems (header-only NVTX3: no cost without a tool)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

// host-side count of kernel launches issued by this library (rb_launch_count)
void note_launches(int k);

// error of the last failed launch() on this host thread (consumed by launch_status)
extern thread_local cudaError_t g_launch_error;

static inline int launch_status() {
    cudaError_t e = cudaGetLastError();
    if (g_launch_error != cudaSuccess) {
        e = g_launch_error;
        g_launch_error = cudaSuccess;
    }
    return e == cudaSuccess ? RB_OK : RB_ERR_CUDA;
}

// ---------------------------------------------------------------------------
// Programmatic dependent launch.  Every kernel of the step path is launched
// with programmatic stream serialization and begins with pdl_enter(): it
// waits for the preceding kernel to complete (memory visible) before reading
// anything, then lets the following kernel launch, so consecutive kernels of
// a captured step overlap launch latency with execution instead of paying
// it as a gap.  A kernel must never return before pdl_enter() (completion
// of a kernel then implies completion of everything before it).
// RB_PDL=0 launches without the attribute (pdl_enter is then a no-op).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

bool pdl_on();

template <typename... KArgs, typename... Args>
static inline void launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                          cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_on() ? 1 : 0;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, ((KArgs)args)...);
    if (e != cudaSuccess) g_launch_error = e;
}

// A kernel whose blocks wait on one another (software grid barrier): a
// cooperative launch, so the driver guarantees that every block is resident
// (or fails the launch) -- never a hang behind kernels of other streams,
// processes or MPS clients.  Programmatic serialization as launch().
// Probed on B200 / driver 580 (tools/coop_pdl_probe.cu): the two attributes
// combine, eagerly and under stream capture.
template <typename... KArgs, typename... Args>
static inline void launch_coop(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                               cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_on() ? 2 : 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, ((KArgs)args)...);
    if (e != cudaSuccess) g_launch_error = e;
}

// ---------------------------------------------------------------------------
// Exact reference arithmetic.  nvcc contracts a*b+c into FMA by default; the
// reference (numba) rounds every mul and add separately, and the cutoff
// predicate must reproduce it bit for bit, so these use the _rn intrinsics
// that are never contracted.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }

// single-shift minimum image, respamd/containers.py:341-353 (d = a - b first),
// branch-free: d - s with s in {box, -box, +0} (d + box == d - (-box) and
// d - (+0) == d exactly in IEEE arithmetic, -0 included)
__device__ __forceinline__ double min_image(double d, double box, double half) {
    double s = d > half ? box : 0.0;
    s = d < -half ? -box : s;
    return xsub(d, s);
}

// r^2 = dx*dx + dy*dy + dz*dz rounded as numba evaluates it (left to right)
// 1/sqrt(x) for a normal double x: the hardware fp64 seed (MUFU.RSQ64H,
// ~2^-20 relative) and one third-order correction y (1 + r/2 + 3r^2/8),
// r = 1 - x y^2 (error ~ r^3, below double rounding).
__device__ __forceinline__ double rsqrt_nr(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double r = fma(-x * y, y, 1.0);
    return fma(y * r, fma(0.375, r, 0.5), y);
}

__device__ __forceinline__ double exact_r2(double dx, double dy, double dz) {
    return xadd(xadd(xmul(dx, dx), xmul(dy, dy)), xmul(dz, dz));
}

struct Image {
    double box[3];
    double half[3];
    int periodic;
};

__host__ __device__ inline Image make_image(const rb_grid &g) {
    Image im;
    for (int d = 0; d < 3; d++) {
        im.box[d] = g.box[d];
        im.half[d] = 0.5 * g.box[d];
    }
    im.periodic = g.periodic;
    return im;
}

// exact displacement a - b with the reference's minimum image
// (kImage = false: a particle for which image_free() holds -- no shift)
template <bool kImage = true>
__device__ __forceinline__ void exact_disp(const Image &im, double ax, double ay, double az,
                                           double bx, double by, double bz, double &dx,
                                           double &dy, double &dz) {
    dx = xsub(ax, bx);
    dy = xsub(ay, by);
    dz = xsub(az, bz);
    if (kImage && im.periodic) {
        dx = min_image(dx, im.box[0], im.half[0]);
        dy = min_image(dy, im.box[1], im.half[1]);
        dz = min_image(dz, im.box[2], im.half[2]);
    }
}

// True when the minimum image cannot change any outcome for partners of a
// particle at (x, y, z) (coordinates in [0, box), as the drift wraps them)
// under a cutoff `reach`: with x in [M, box - M], M > reach, a shifted
// difference d -/+ box has |.| > M for every partner in [0, box), so each
// partner inside the cutoff needs no shift (identical dx), and one outside
// stays outside unshifted (the shift only ever shortens |d|, exactly:
// Sterbenz).  M carries an absolute margin far above the rounding of d.
__device__ __forceinline__ bool image_free(const Image &im, double x, double y, double z,
                                           double reach) {
    if (!im.periodic) return true;
    const double m = reach + 1e-9 * (1.0 + im.box[0] + im.box[1] + im.box[2]);
    return x >= m && x <= im.box[0] - m && y >= m && y <= im.box[1] - m && z >= m &&
           z <= im.box[2] - m;
}

// ---------------------------------------------------------------------------
// status word: (tag << 8) | kind, reduced with atomicMin
// ---------------------------------------------------------------------------
__device__ __forceinline__ void record_status(unsigned long long *status, int64_t tag, int kind) {
    if (status) atomicMin(status, ((unsigned long long)tag << 8) | (unsigned long long)kind);
}

// Two adjacent status words in one volatile 16-byte load ({CLEAR, 0} for a
// null status); issued with a kernel's data loads it costs no extra round
// trip.  `p` is 16-byte aligned (status and status + 2).
__device__ __forceinline__ ulonglong2 ld_status2(const unsigned long long *p) {
    ulonglong2 r = make_ulonglong2(RB_STATUS_CLEAR, 0ull);
    if (p) asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];"
                        : "=l"(r.x), "=l"(r.y) : "l"(p));
    return r;
}

// Tag of the current kernel: the explicit value, or (tag < 0) the step
// counter kept in status[1] by rb_step_begin (lets a captured CUDA graph be
// replayed for many steps).
__device__ __forceinline__ int64_t resolve_tag(int64_t tag, const unsigned long long *status) {
    if (tag >= 0 || !status) return tag < 0 ? 0 : tag;
    return (int64_t)(*(volatile const unsigned long long *)(status + 1));
}

// True when a kernel of step `tag` whose own error kind is `kind` must not
// run: an earlier step failed, or an error of higher precedence (lower kind)
// was raised earlier in the same step.
__device__ __forceinline__ bool frozen_word(unsigned long long s, int64_t tag, int kind) {
    if (s == RB_STATUS_CLEAR) return false;
    long long t = (long long)(s >> 8);
    int k = (int)(s & 0xff);
    if (t < tag) return true;
    if (t == tag && k < kind && k != RB_KIND_NONFINITE && k != RB_KIND_CAPACITY) return true;
    return false;
}

__device__ __forceinline__ bool frozen(const unsigned long long *status, int64_t tag, int kind) {
    if (!status) return false;
    unsigned long long s = *(volatile const unsigned long long *)status;
    if (s == RB_STATUS_CLEAR) return false;
    long long t = (long long)(s >> 8);
    int k = (int)(s & 0xff);
    if (t < tag) return true;
    if (t == tag && k < kind && k != RB_KIND_NONFINITE && k != RB_KIND_CAPACITY) return true;
    return false;
}

// A rebuild vote froze the steps from its tag on (RB_KIND_REBUILD): the
// state-changing kernels of step `tag` or later (drift, kick, sample, halo
// pull) must not run either.
__device__ __forceinline__ bool rebuild_frozen(unsigned long long s, int64_t tag) {
    return s != RB_STATUS_CLEAR && (int)(s & 0xff) == RB_KIND_REBUILD &&
           (long long)(s >> 8) <= (long long)tag;
}

// warp-uniform variant: lane 0 reads, everyone agrees (needed before shuffles)
__device__ __forceinline__ bool warp_frozen(const unsigned long long *status, int64_t tag,
                                            int kind) {
    int f = 0;
    if ((threadIdx.x & 31) == 0) f = frozen(status, tag, kind) ? 1 : 0;
    return __shfl_sync(0xffffffffu, f, 0) != 0;
}

// ---------------------------------------------------------------------------
// warp helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <int kWidth>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
    for (int off = kWidth / 2; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off, kWidth);
    return v;
}

template <int kWidth>
__device__ __forceinline__ int group_sum_int(int v) {
#pragma unroll
    for (int off = kWidth / 2; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off, kWidth);
    return v;
}

// block-wide sum with a fixed tree (xor shuffles, then warp 0 over the
// per-warp partials); the result is valid in thread 0.  Every thread of the
// block must call it; `sh` holds >= 32 entries.
template <typename T>
__device__ __forceinline__ T block_tree_sum(T v, T *sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    T s = 0;
    if (warp == 0) {
        s = lane < (int)(blockDim.x >> 5) ? sh[lane] : (T)0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    }
    return s;
}

// neighbour cell of base cell (cx,cy,cz) at offset o; -1 when outside an
// open grid (respamd/containers.py:319-333)
// flat id of the cell at coordinates x (offset-shifted: in [0, 2 cells) on a
// wrapped dimension), -1 outside a non-wrapped one
__device__ __forceinline__ int cell_at(const rb_grid &g, int x, int y, int z) {
    int c[3] = {x, y, z};
#pragma unroll
    for (int d = 0; d < 3; d++) {
        if (g.wrap[d]) {
            if (c[d] >= g.cells[d]) c[d] -= g.cells[d];
        } else if (c[d] < 0 || c[d] >= g.cells[d]) {
            return -1;
        }
    }
    return (c[0] * g.cells[1] + c[1]) * g.cells[2] + c[2];
}

__device__ __forceinline__ int neighbor_cell(const rb_grid &g, int cx, int cy, int cz, int o) {
    int c[3];
#pragma unroll
    for (int d = 0; d < 3; d++) {
        int x = (d == 0 ? cx : (d == 1 ? cy : cz)) + g.offsets[o][d];
        if (g.wrap[d]) {
            // canonical offsets are already wrapped into [0, cells)
            if (x >= g.cells[d]) x -= g.cells[d];
        } else if (x < 0 || x >= g.cells[d]) {
            return -1;
        }
        c[d] = x;
    }
    return (c[0] * g.cells[1] + c[1]) * g.cells[2] + c[2];
}

}  // namespace rb
