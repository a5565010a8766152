// atm.cu -- Axilrod-Teller-Muto triplet pass, C01 (owner-computes) form.
//
// The production pass is the Newton-3 kernel in atm3.cu; this C01 form is kept
// as an independent second enumeration (tests cross-check the two) and as the
// instrumentation of collect_triplet_visits.
//
// Replaces respamd/containers.py:373-535 (_c01_triplet_kernel).  One warp per
// base particle i (rank order), owner-computes like the reference: only the
// force on i is stored, every unique triplet is visited once from each of its
// three members (energy phi/3 per visit), so per-particle force sums need no
// atomics and are deterministic.
//
//   1. survivors: the row entries j with r_ij^2 <= rc^2 (reference pair
//      arithmetic), compacted into shared memory with their displacement
//      d_ij = x_i - x_j and a = r_ij^2 (containers.py:437-474);
//   2. candidates: every unordered survivor pair (j, k) -- the flat index
//      over the triangle is spread across the 32 lanes, so lanes stay busy
//      independent of the pattern structure.  r_jk^2 <= rc^2 is decided
//      bit-exactly (containers.py:497-515): a fused estimate from the
//      survivors' displacements settles every pair farther than 1e-10
//      (relative) from the cutoff, the rest are recomputed with the
//      reference's raw-position arithmetic.  When the box is smaller than
//      four cutoffs the estimate is not a valid minimum image and every
//      candidate takes the exact path.  (Enumerating all survivor pairs is
//      the reference's pattern loop :478-491: its patterns are exactly the
//      neighbour-cell pairs whose gap is within the cutoff, and pairs from
//      any other cell pair fail the r_jk test.)
//   3. accepted (j, k) go through a 64-entry warp queue in shared memory and
//      are evaluated 32 at a time with every lane busy; the ATM kernel
//      (potentials.py:82-114) is restated with one rsqrt.
//
// Per-visit virial: -(E_a a + E_b b); over the three visits of a triplet it
// sums to the reference's -2(E_a a + E_b b + E_c c) (:530).
#include "common.cuh"

namespace rb {

constexpr int kAtmWarps = 4;
constexpr int kAtmQueue = 64;
constexpr double kAtmMargin = 1e-10;

struct AtmWarpSmem {
    double *dx, *dy, *dz, *r2;
    int32_t *idx;
    uint32_t *qst;
    double *qc;
};

__host__ __device__ inline size_t atm_warp_bytes(int capacity) {
    size_t b = (size_t)capacity * (4 * sizeof(double) + sizeof(int32_t));
    b = (b + 15) & ~(size_t)15;
    b += (size_t)kAtmQueue * (sizeof(double) + sizeof(uint32_t));
    return (b + 15) & ~(size_t)15;
}

__device__ inline AtmWarpSmem atm_carve(char *base, int capacity) {
    AtmWarpSmem s;
    s.dx = (double *)base;
    s.dy = s.dx + capacity;
    s.dz = s.dy + capacity;
    s.r2 = s.dz + capacity;
    s.qc = s.r2 + capacity;
    s.idx = (int32_t *)(s.qc + kAtmQueue);
    s.qst = (uint32_t *)(s.idx + capacity);
    return s;
}

// (s, t), s < t, of the flat index c over the strict upper triangle of m x m
__device__ __forceinline__ void unflatten_pair(int c, int m, int &s, int &t) {
    const int b2 = 2 * m - 1;
    float disc = (float)b2 * (float)b2 - 8.0f * (float)c;
    int si = (int)(((float)b2 - sqrtf(fmaxf(disc, 0.0f))) * 0.5f);
    if (si < 0) si = 0;
    // off(s) = s*(2m-1-s)/2 = index of (s, s+1)
    while (si > 0 && si * (b2 - si) / 2 > c) si--;
    while ((si + 1) * (b2 - si - 1) / 2 <= c) si++;
    s = si;
    t = c - si * (b2 - si) / 2 + si + 1;
}

struct AtmAcc {
    double fx, fy, fz, e, w;
    int visits;
    bool bad;
};

// ATM energy and d/da, d/db without the factor nu (folded in once per
// particle); potentials.py:82-114 restated with rsqrt.
__device__ __forceinline__ void atm_visit(double a, double b, double c, double dijx, double dijy,
                                          double dijz, double dikx, double diky, double dikz,
                                          AtmAcc &acc) {
    if (a < RB_MIN_DISTANCE_SQ || b < RB_MIN_DISTANCE_SQ || c < RB_MIN_DISTANCE_SQ) {
        acc.bad = true;
        return;
    }
    const double u = a + b - c;
    const double v = a + c - b;
    const double w = b + c - a;
    const double p = u * v * w;
    const double s = a * b * c;
    const double rs = rsqrt(s);
    const double inv_s = rs * rs;
    const double s32 = inv_s * rs;
    const double s52 = s32 * inv_s;
    const double s72 = s52 * inv_s;
    const double uv = u * v, uw = u * w, vw = v * w;
    const double bc = b * c, ac = a * c;
    const double q = 0.9375 * p * s72;
    const double ea = (0.375 * (vw + uw - uv) - 1.5 * bc) * s52 - q * bc;
    const double eb = (0.375 * (vw - uw + uv) - 1.5 * ac) * s52 - q * ac;
    acc.fx += ea * dijx + eb * dikx;
    acc.fy += ea * dijy + eb * diky;
    acc.fz += ea * dijz + eb * dikz;
    acc.e += s32 + 0.375 * p * s52;
    acc.w += ea * a + eb * b;
    acc.visits += 1;
}

// kRows: instrumentation mode of _c01_triplet_visits_kernel (:538-660) --
// instead of evaluating, every accepted visit writes its sorted (i, j, k)
// particle indices at row_offset[r] + (visit ordinal), in enumeration order.
template <bool kExactImage, bool kRows>
__global__ void __launch_bounds__(kAtmWarps * 32)
    k_atm(rb_grid g, int64_t n, const double *__restrict__ pr, const int32_t *__restrict__ parts,
          const int32_t *__restrict__ rows, const int32_t *__restrict__ row_count,
          int32_t capacity, double rc2, double rc2_lo, double rc2_hi, double nu,
          double *__restrict__ forces, double *__restrict__ energy_rank,
          double *__restrict__ virial_rank, int32_t *__restrict__ visits_rank,
          unsigned long long *status, int64_t tag, const int64_t *__restrict__ row_offset,
          int32_t *__restrict__ visit_rows) {
    pdl_enter();
    extern __shared__ __align__(16) char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (r >= n) return;
    tag = resolve_tag(tag, status);
    if (!kRows && warp_frozen(status, tag, RB_KIND_TRIPLET_MIN_SEPARATION)) return;
    AtmWarpSmem sm = atm_carve(smem_raw + (size_t)warp * atm_warp_bytes(capacity), capacity);
    const Image im = make_image(g);
    const double xi = pr[3 * r], yi = pr[3 * r + 1], zi = pr[3 * r + 2];

    // 1. survivors
    const int m = row_count[r];
    const int32_t *row = rows + r * (int64_t)capacity;
    int cnt = 0;
    for (int base = 0; base < m; base += 32) {
        const int k = base + lane;
        bool keep = false;
        int j = 0;
        double dx = 0.0, dy = 0.0, dz = 0.0, r2 = 0.0;
        if (k < m) {
            j = row[k];
            exact_disp(im, xi, yi, zi, pr[3 * (j)], pr[3 * (j) + 1], pr[3 * (j) + 2], dx, dy, dz);
            r2 = exact_r2(dx, dy, dz);
            keep = r2 <= rc2;
        }
        const unsigned mk = __ballot_sync(0xffffffffu, keep);
        if (keep) {
            const int slot = cnt + __popc(mk & lanemask_lt());
            sm.dx[slot] = dx;
            sm.dy[slot] = dy;
            sm.dz[slot] = dz;
            sm.r2[slot] = r2;
            sm.idx[slot] = j;
        }
        cnt += __popc(mk);
    }
    __syncwarp();

    // 2 + 3. candidate pairs -> queue -> evaluation
    AtmAcc acc = {0.0, 0.0, 0.0, 0.0, 0.0, 0, false};
    const int total = cnt * (cnt - 1) / 2;
    int qn = 0;
    for (int base = 0; base < total; base += 32) {
        const int c = base + lane;
        bool accept = false;
        int s = 0, t = 0;
        double cval = 0.0;
        if (c < total) {
            unflatten_pair(c, cnt, s, t);
            bool exact = kExactImage;
            if (!kExactImage) {
                // x_j - x_k = d_ik - d_ij  (fused estimate)
                const double ex = sm.dx[t] - sm.dx[s];
                const double ey = sm.dy[t] - sm.dy[s];
                const double ez = sm.dz[t] - sm.dz[s];
                const double c2 = ex * ex + ey * ey + ez * ez;
                if (c2 <= rc2_lo) {
                    accept = true;
                    cval = c2;
                } else if (c2 <= rc2_hi) {
                    exact = true;
                }
            }
            if (exact) {
                const int j = sm.idx[s], k = sm.idx[t];
                double dx, dy, dz;
                exact_disp(im, pr[3 * (j)], pr[3 * (j) + 1], pr[3 * (j) + 2], pr[3 * (k)], pr[3 * (k) + 1], pr[3 * (k) + 2], dx, dy, dz);
                const double c2 = exact_r2(dx, dy, dz);
                accept = c2 <= rc2;
                cval = c2;
            }
        }
        const unsigned ma = __ballot_sync(0xffffffffu, accept);
        if (kRows) {
            if (accept) {
                const int64_t at = row_offset[r] + acc.visits + __popc(ma & lanemask_lt());
                int a0 = parts[r], a1 = parts[sm.idx[s]], a2 = parts[sm.idx[t]];
                int lo = min(a0, min(a1, a2)), hi = max(a0, max(a1, a2));
                visit_rows[3 * at] = lo;
                visit_rows[3 * at + 1] = a0 + a1 + a2 - lo - hi;
                visit_rows[3 * at + 2] = hi;
            }
            acc.visits += __popc(ma);
            continue;
        }
        if (accept) {
            const int slot = qn + __popc(ma & lanemask_lt());
            sm.qst[slot] = (uint32_t)s | ((uint32_t)t << 16);
            sm.qc[slot] = cval;
        }
        qn += __popc(ma);
        __syncwarp();
        if (qn >= 32) {
            const uint32_t st = sm.qst[lane];
            const int qs = st & 0xffff, qt = st >> 16;
            atm_visit(sm.r2[qs], sm.r2[qt], sm.qc[lane], sm.dx[qs], sm.dy[qs], sm.dz[qs], sm.dx[qt],
                      sm.dy[qt], sm.dz[qt], acc);
            __syncwarp();
            if (lane < qn - 32) {
                sm.qst[lane] = sm.qst[lane + 32];
                sm.qc[lane] = sm.qc[lane + 32];
            }
            __syncwarp();
            qn -= 32;
        }
    }
    if (kRows) return;
    if (lane < qn) {
        const uint32_t st = sm.qst[lane];
        const int qs = st & 0xffff, qt = st >> 16;
        atm_visit(sm.r2[qs], sm.r2[qt], sm.qc[lane], sm.dx[qs], sm.dy[qs], sm.dz[qs], sm.dx[qt],
                  sm.dy[qt], sm.dz[qt], acc);
    }

    // fixed-tree warp reduction
    const double fx = group_sum<32>(acc.fx);
    const double fy = group_sum<32>(acc.fy);
    const double fz = group_sum<32>(acc.fz);
    const double e = group_sum<32>(acc.e);
    const double w = group_sum<32>(acc.w);
    const int visits = group_sum_int<32>(acc.visits);
    const bool bad = __any_sync(0xffffffffu, acc.bad);
    if (lane == 0) {
        const int64_t p = parts[r];
        const double f2nu = -2.0 * nu;
        forces[3 * p] = f2nu * fx;
        forces[3 * p + 1] = f2nu * fy;
        forces[3 * p + 2] = f2nu * fz;
        energy_rank[r] = (nu / 3.0) * e;
        virial_rank[r] = -nu * w;
        visits_rank[r] = visits;
        if (bad) record_status(status, tag, RB_KIND_TRIPLET_MIN_SEPARATION);
    }
}

// cudaFuncSetAttribute is not stream-ordered: call it only when a launch
// needs more dynamic shared memory than already granted, so that replays and
// CUDA-graph captures after the first launch never touch it.
template <typename K>
static void grant_smem(K kernel, size_t bytes, size_t &granted) {
    if (bytes > 48 * 1024 && bytes > granted) {
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        granted = bytes;
    }
}

static size_t g_granted[3] = {0, 0, 0};

// warps per CTA: kAtmWarps unless the per-warp survivor buffers of a large
// row capacity do not fit 227 KB of shared memory; 0 if one warp does not fit
static size_t atm_launch_shape(int capacity, int &warps) {
    const size_t per = atm_warp_bytes(capacity);
    const size_t limit = 227 * 1024;
    warps = kAtmWarps;
    while (warps > 1 && (size_t)warps * per > limit) warps--;
    if ((size_t)warps * per > limit) return 0;
    return (size_t)warps * per;
}

}  // namespace rb

using namespace rb;

extern "C" int rb_atm_pass_c01(const rb_grid *g, int64_t n, const double *pos_r, const int32_t *cell_particles, const int32_t *rows,
                           const int32_t *row_count, int32_t capacity, double rc, double nu,
                           double *forces, double *energy_rank, double *virial_rank,
                           int32_t *visits_rank, unsigned long long *status, int64_t tag,
                           void *stream) {
    NvtxRange nvtx_range("triplet C01 (rb_atm_pass_c01)");
    if (!g || n < 0 || capacity <= 0 || capacity > 4096) return RB_ERR_ARGUMENT;
    if (n == 0) return RB_OK;
    const double rc2 = rc * rc;
    bool exact_image = false;
    if (g->periodic)
        for (int d = 0; d < 3; d++)
            if (!(g->box[d] > 4.0 * rc * (1.0 + 1e-12))) exact_image = true;
    int warps = 0;
    const size_t smem = atm_launch_shape(capacity, warps);
    if (!smem) return RB_ERR_ARGUMENT;
    const unsigned blocks = (unsigned)((n + warps - 1) / warps);
    cudaStream_t st = as_stream(stream);
    if (exact_image) {
        grant_smem(k_atm<true, false>, smem, g_granted[0]);
        launch(k_atm<true, false>, dim3(blocks), dim3(warps * 32), smem, st, *g, n, pos_r, cell_particles, rows, row_count, capacity, rc2, rc2, rc2, nu,
            forces, energy_rank, virial_rank, visits_rank, status, tag, nullptr, nullptr);
        note_launches(1);
    } else {
        grant_smem(k_atm<false, false>, smem, g_granted[1]);
        launch(k_atm<false, false>, dim3(blocks), dim3(warps * 32), smem, st, *g, n, pos_r, cell_particles, rows, row_count, capacity, rc2,
            rc2 * (1.0 - kAtmMargin), rc2 * (1.0 + kAtmMargin), nu, forces, energy_rank,
            virial_rank, visits_rank, status, tag, nullptr, nullptr);
        note_launches(1);
    }
    return launch_status();
}

// Instrumentation: sorted (i, j, k) rows of every accepted visit
// (collect_triplet_visits, containers.py:825-849).  row_offset[r] is the
// exclusive prefix of the visit counts rb_atm_pass reported per rank.
extern "C" int rb_atm_visit_rows(const rb_grid *g, int64_t n, const double *pos_r, const int32_t *cell_particles,
                                 const int32_t *rows, const int32_t *row_count, int32_t capacity,
                                 double rc, const int64_t *row_offset, int32_t *visit_rows,
                                 void *stream) {
    if (!g || n < 0 || capacity <= 0 || capacity > 4096 || !row_offset || !visit_rows)
        return RB_ERR_ARGUMENT;
    if (n == 0) return RB_OK;
    const double rc2 = rc * rc;
    int warps = 0;
    const size_t smem = atm_launch_shape(capacity, warps);
    if (!smem) return RB_ERR_ARGUMENT;
    const unsigned blocks = (unsigned)((n + warps - 1) / warps);
    // the instrumentation always takes the exact raw-position predicate
    grant_smem(k_atm<true, true>, smem, g_granted[2]);
    launch(k_atm<true, true>, dim3(blocks), dim3(warps * 32), smem, as_stream(stream), *g, n, pos_r, cell_particles, rows, row_count, capacity, rc2, rc2, rc2, 0.0, nullptr,
        nullptr, nullptr, nullptr, nullptr, 0, row_offset, visit_rows);
    note_launches(1);
    return launch_status();
}
