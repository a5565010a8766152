// rdf.cu -- pair-distance histogram for the radial distribution function
// (respamd/observables.py:143-177).
//
// One thread per particle i counts every j != i (ordered pairs: the
// reference adds 2 per unordered pair, i.e. 1 per ordered pair), positions
// staged through shared-memory tiles.  The bin index repeats the
// reference's arithmetic bit for bit: d = x_i - x_j, single-shift minimum
// image, r^2 = (dx dx + dy dy) + dz dz without FMA, r^2 >= r_max^2 skipped,
// b = trunc(sqrt(r^2) * inv_width) clamped to bins - 1, with inv_width and
// r_max^2 computed by the host exactly as the reference does.  Counts go to
// a per-block shared histogram and then to the global int64 counts with
// integer atomics: the totals are exact and order independent.
#include "common.cuh"

namespace rb {

constexpr int kRdfThreads = 128;

__global__ void __launch_bounds__(kRdfThreads)
    k_rdf(int64_t n, const double *__restrict__ pos, double bx, double by, double bz,
          double r2_max, double inv_width, int bins, unsigned long long *__restrict__ counts) {
    pdl_enter();
    extern __shared__ __align__(16) unsigned char rdf_smem[];
    unsigned int *hist = reinterpret_cast<unsigned int *>(rdf_smem);
    double *tile = reinterpret_cast<double *>(rdf_smem + ((bins * 4 + 15) & ~15));
    for (int b = threadIdx.x; b < bins; b += kRdfThreads) hist[b] = 0u;
    const int64_t i = (int64_t)blockIdx.x * kRdfThreads + threadIdx.x;
    const bool active = i < n;
    double xi = 0.0, yi = 0.0, zi = 0.0;
    if (active) {
        xi = pos[3 * i];
        yi = pos[3 * i + 1];
        zi = pos[3 * i + 2];
    }
    const double hx = 0.5 * bx, hy = 0.5 * by, hz = 0.5 * bz;
    for (int64_t j0 = 0; j0 < n; j0 += kRdfThreads) {
        const int64_t jl = j0 + threadIdx.x;
        __syncthreads();
        for (int c = 0; c < 3; c++) tile[3 * threadIdx.x + c] = jl < n ? pos[3 * jl + c] : 0.0;
        __syncthreads();
        if (!active) continue;
        const int cnt = (int)(n - j0 < kRdfThreads ? n - j0 : kRdfThreads);
        for (int u = 0; u < cnt; u++) {
            if (j0 + u == i) continue;
            const double dx = min_image(xsub(xi, tile[3 * u]), bx, hx);
            const double dy = min_image(xsub(yi, tile[3 * u + 1]), by, hy);
            const double dz = min_image(xsub(zi, tile[3 * u + 2]), bz, hz);
            const double r2 = exact_r2(dx, dy, dz);
            if (r2 >= r2_max) continue;
            int b = (int)xmul(__dsqrt_rn(r2), inv_width);
            if (b >= bins) b = bins - 1;
            atomicAdd(hist + b, 1u);
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < bins; b += kRdfThreads)
        if (hist[b]) atomicAdd(counts + b, (unsigned long long)hist[b]);
}

}  // namespace rb

using namespace rb;

extern "C" int rb_distance_histogram(int64_t n, const double *pos, const double *box3_host,
                                     double r2_max, double inv_width, int32_t bins,
                                     int64_t *counts, void *stream) {
    if (n < 0 || bins < 1 || bins > 16384 || !box3_host || !counts || (n > 0 && !pos))
        return RB_ERR_ARGUMENT;
    if (n < 2) return RB_OK;
    const size_t smem = (size_t)((bins * 4 + 15) & ~15) + 3 * kRdfThreads * sizeof(double);
    static size_t granted = 0;
    if (smem > 48 * 1024 && smem > granted) {
        cudaFuncSetAttribute(k_rdf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        granted = smem;
    }
    launch(k_rdf, dim3((unsigned)((n + kRdfThreads - 1) / kRdfThreads)), dim3(kRdfThreads), smem,
           as_stream(stream), n, pos, box3_host[0], box3_host[1], box3_host[2], r2_max,
           inv_width, (int)bins, reinterpret_cast<unsigned long long *>(counts));
    note_launches(1);
    return launch_status();
}
