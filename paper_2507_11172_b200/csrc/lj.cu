// lj.cu -- Lennard-Jones pair pass over the neighbour rows.
//
// Replaces respamd/containers.py:282-370 (_c01_pair_kernel) with the same
// owner-computes discipline: each particle accumulates only its own force,
// every pair is visited from both sides and contributes phi/2 and
// scale*r^2/2 per visit (:364-365).  A group of kGroup lanes serves one
// particle: lanes stride over the row, then a fixed xor-shuffle tree sums the
// partials, so the result does not depend on scheduling.
//
// The cutoff predicate and the guard use the reference's exact pair-distance
// arithmetic; the LJ kernel itself (potentials.py:55-67) is restated with one
// reciprocal (hardware seed + a third-order correction) instead of two
// divides (agreement ~1e-16 relative).
#include <type_traits>

#include "common.cuh"

namespace rb {

#ifndef RB_LJ_GROUP
#define RB_LJ_GROUP 8
#endif
#ifndef RB_LJ_ROW_REGS
#define RB_LJ_ROW_REGS 10
#endif
constexpr int kLjGroup = RB_LJ_GROUP;   // lanes per particle
constexpr int kLjRowRegs = RB_LJ_ROW_REGS;  // row indices a lane holds at once
#ifndef RB_LJ_BATCH
#define RB_LJ_BATCH 2
#endif
constexpr int kLjBatch = RB_LJ_BATCH;  // neighbour positions in flight per lane
static_assert(kLjRowRegs % kLjBatch == 0, "row registers: whole batches");
constexpr int kLjThreads = 256;
// 1/x: the hardware fp64 seed (MUFU.RCP64H) and one third-order correction
// y (1 + e + e^2), e = 1 - x y (x is a squared distance, a normal double;
// relative error ~e^3, below double rounding)
__device__ __forceinline__ double lj_rcp(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-x, y, 1.0);
    return fma(y, fma(e, e, e), y);
}

#ifndef RB_LJ_MIN_BLOCKS
#define RB_LJ_MIN_BLOCKS 4  // 64 registers: 4 blocks of 256 per SM
#endif
// kScalars: accumulate the energy and virial (sample points); without it
// the pass writes forces only (energy_rank / virial_rank untouched)
template <bool kScalars>
__global__ void __launch_bounds__(kLjThreads, RB_LJ_MIN_BLOCKS)
    k_lj(rb_grid g, int64_t n, const double *__restrict__ pr, const int32_t *__restrict__ parts,
         const int32_t *__restrict__ rows, const int32_t *__restrict__ row_count,
         int32_t capacity, double rc, double rc2, double eps24, double eps4, double sigma2,
         double *__restrict__ forces, double *__restrict__ energy_rank,
         double *__restrict__ virial_rank, const uint8_t *__restrict__ owned,
         unsigned long long *status, int64_t tag) {
    pdl_enter();
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t r = gid / kLjGroup;
    const int sub = (int)(gid % kLjGroup);
    const bool active = r < n;
    // the pass is latency-bound: the first memory round trip carries the
    // status words, the row length, the own position and every row index of
    // this lane (up to kLjRowRegs; loaded up to the capacity and masked by
    // the length afterwards), the second the neighbour positions two entries
    // at a time; the accumulation order stays k = sub, sub + G, sub + 2G, ...
    int m = 0;
    double xi = 0.0, yi = 0.0, zi = 0.0;
    int jr[kLjRowRegs];
    const int32_t *row = rows + (active ? r : 0) * (int64_t)capacity;
    if (active) {
        m = row_count[r];
        xi = pr[3 * r];
        yi = pr[3 * r + 1];
        zi = pr[3 * r + 2];
    }
#pragma unroll
    for (int u = 0; u < kLjRowRegs; u++) {
        const int k = sub + u * kLjGroup;
        jr[u] = active && k < capacity ? __ldg(row + k) : -1;
    }
    const ulonglong2 s01 = ld_status2(status);
    const unsigned long long sw = __shfl_sync(0xffffffffu, s01.x, 0);  // one view per warp
    const int64_t cur = status ? (int64_t)__shfl_sync(0xffffffffu, s01.y, 0) : 0;
    const bool from_device = tag < 0;
    if (tag < 0) tag = cur;
    // the pair pass closes the device step (status[2]): the kick that ends it
    // may be folded into the next step's drift (rb_respa_kick_drift)
    if (from_device && status && gid == 0) status[2] = (unsigned long long)tag;
    if (status && frozen_word(sw, tag, RB_KIND_PAIR_MIN_SEPARATION)) return;
    const Image im = make_image(g);
    double fx = 0.0, fy = 0.0, fz = 0.0, e = 0.0, w = 0.0;
    bool bad = false;
    {  // (inactive lanes: empty rows; every lane takes part in the warp votes)
#pragma unroll
        for (int u = 0; u < kLjRowRegs; u++) {
            const int k = sub + u * kLjGroup;
            if (k >= m) jr[u] = -1;
        }
        const int self = active ? (int)r : 0;
        // branch-free visit: the kernel runs for every entry and the scale
        // is selected (zero beyond the cutoff, for an empty slot and for a
        // guarded pair, potentials.py:35-36), so the lanes never diverge
        auto visit = [&](auto image, bool valid, double px, double py, double pz) {
            double dx, dy, dz;
            exact_disp<decltype(image)::value>(im, xi, yi, zi, px, py, pz, dx, dy, dz);
            const double r2 = exact_r2(dx, dy, dz);
            const bool in = valid && r2 <= rc2;
            const bool guard = in && r2 < RB_MIN_DISTANCE_SQ;
            bad = bad || guard;
            const bool ok = in && !guard;
            const double inv_r2 = lj_rcp(r2);
            const double x = sigma2 * inv_r2;
            const double r6 = x * x * x;
            const double r12 = r6 * r6;
            // 2 r12 - r6 as one fma (2 r12 is exact: the same value)
            double scale = eps24 * fma(2.0, r12, -r6) * inv_r2;
            scale = ok ? scale : 0.0;
            fx = fma(scale, dx, fx);
            fy = fma(scale, dy, fy);
            fz = fma(scale, dz, fz);
            if (kScalars) {
                e += ok ? eps4 * (r12 - r6) : 0.0;
                w = fma(scale, r2, w);
            }
        };
        auto walk = [&](auto image) {
#pragma unroll
            for (int u = 0; u < kLjRowRegs; u += kLjBatch) {
                if (!__any_sync(0xffffffffu, jr[u] >= 0)) break;  // the warp's rows are done
                double px[kLjBatch], py[kLjBatch], pz[kLjBatch];
#pragma unroll
                for (int t = 0; t < kLjBatch; t++) {
                    const int q = jr[u + t] >= 0 ? jr[u + t] : self;
                    RB_CHECK(q >= 0 && q < n);
                    px[t] = pr[3 * q];
                    py[t] = pr[3 * q + 1];
                    pz[t] = pr[3 * q + 2];
                }
#pragma unroll
                for (int t = 0; t < kLjBatch; t++) visit(image, jr[u + t] >= 0, px[t], py[t], pz[t]);
            }
            for (int k = sub + kLjRowRegs * kLjGroup; k < m; k += kLjGroup) {  // long rows
                const int q = __ldg(row + k);
                visit(image, true, pr[3 * q], pr[3 * q + 1], pr[3 * q + 2]);
            }
        };
        // a warp whose particles all sit a cutoff away from the periodic
        // faces walks its rows without the minimum image (common.cuh
        // image_free: bit-identical outcomes; ~90% of warps at cfg4)
        if (__all_sync(0xffffffffu, !active || image_free(im, xi, yi, zi, rc)))
            walk(std::false_type{});
        else
            walk(std::true_type{});
    }
    fx = group_sum<kLjGroup>(fx);
    fy = group_sum<kLjGroup>(fy);
    fz = group_sum<kLjGroup>(fz);
    if (kScalars) {
        e = group_sum<kLjGroup>(e);
        w = group_sum<kLjGroup>(w);
    }
    if (active && bad) record_status(status, tag, RB_KIND_PAIR_MIN_SEPARATION);
    if (active && sub == 0) {
        const int64_t p = parts[r];
        forces[3 * p] = fx;
        forces[3 * p + 1] = fy;
        forces[3 * p + 2] = fz;
        if (kScalars) {
            // decomposed runs: only owned particles carry energy (phi/2 per visit)
            const double own = owned ? (double)owned[r] : 1.0;
            energy_rank[r] = own * (0.5 * e);
            virial_rank[r] = own * (0.5 * w);
        }
    }
}

}  // namespace rb

using namespace rb;

extern "C" int rb_lj_pass(const rb_grid *g, int64_t n, const double *pos_r, const int32_t *cell_particles, const int32_t *rows,
                          const int32_t *row_count, int32_t capacity, double rc, double epsilon,
                          double sigma, double *forces, double *energy_rank, double *virial_rank,
                          const uint8_t *owned, unsigned long long *status, int64_t tag,
                          void *stream) {
    NvtxRange nvtx_range("pair (rb_lj_pass)");
    if (!g || n < 0 || capacity <= 0) return RB_ERR_ARGUMENT;
    if (n == 0) return RB_OK;
    const int64_t threads = n * kLjGroup;
    unsigned blocks = (unsigned)((threads + kLjThreads - 1) / kLjThreads);
    // energy_rank == virial_rank == NULL: forces only (steps that are not
    // sample points, whose scalars nothing reads)
    auto kern = energy_rank && virial_rank ? k_lj<true> : k_lj<false>;
    launch(kern, dim3(blocks), dim3(kLjThreads), 0, as_stream(stream), *g, n, pos_r, cell_particles, rows, row_count, capacity, rc, rc * rc, 24.0 * epsilon,
        4.0 * epsilon, sigma * sigma, forces, energy_rank, virial_rank, owned, status, tag);
    note_launches(1);
    return launch_status();
}
