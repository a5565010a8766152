// direct.cu -- DirectSum on the device: every pair and every triplet of a
// non-periodic system, no cutoff (respamd/containers.py:663-739, 852-908).
//
// Pairs: one warp per particle i sums the LJ force of all j != i (lanes
// stride over j, fixed xor tree); each pair is visited from both sides,
// phi/2 and scale*r^2/2 per visit (owner-computes: no scatter,
// deterministic).
//
// Triplets: Newton-3, every unique i < j < k evaluated once.  The pairs
// (j, k) of base i are the pairs of its m = n-1-i followers, enumerated by
// rotation rounds as in atm3.cu (round d pairs follower s with (s+d) mod m)
// and taken T at a time (one per thread of the block, T = 256, or 1024 when
// only one block fits an SM): inside such a window all j are distinct and all
// k are distinct (m >= T: a window spans at most two rounds; m < T: a window
// is one round), so f_j and f_k go to
// the block's shared-memory force array in two conflict-free sub-steps.  The
// windows of all bases form one list; block b takes a contiguous slice of it
// (equal pair counts per block).  Each block leaves its force array in a
// per-block slab; a final kernel sums the slabs in block order.  No atomics:
// the result is bit-identical from run to run.
//
// Arithmetic: the reference's raw differences (d = x_a - x_b, no image),
// guard MIN_DISTANCE_SQ on every side (flag + skip), the ATM kernel in the
// form of atm3.cu (forces in units of 2 nu, E and the virial rescaled at the
// end).
#include "common.cuh"

namespace rb {

constexpr int kDpThreads = 128;  // pair pass: threads per block (4 particles)
constexpr int kDtMaxN = 8192;    // the per-block force array lives in shared memory

__global__ void __launch_bounds__(kDpThreads)
    k_direct_pairs(int64_t n, int64_t i_lo, int64_t i_hi, const double *__restrict__ pos,
                   double eps24, double eps4, double sigma2, double *__restrict__ forces,
                   double *__restrict__ energy, double *__restrict__ virial,
                   unsigned long long *status, int64_t tag) {
    pdl_enter();
    // one warp per particle i of [i_lo, i_hi); lanes stride over j, then a
    // fixed xor tree
    const int lane = threadIdx.x & 31;
    const int64_t i = i_lo + (((int64_t)blockIdx.x * kDpThreads + threadIdx.x) >> 5);
    const bool from_device = tag < 0;
    tag = resolve_tag(tag, status);
    // like the LJ pass: closes the device step (status[2], see lj.cu)
    if (from_device && status && blockIdx.x == 0 && threadIdx.x == 0) status[2] = (unsigned long long)tag;
    if (i >= i_hi) return;  // whole warps
    const double xi = pos[3 * i], yi = pos[3 * i + 1], zi = pos[3 * i + 2];
    double fx = 0.0, fy = 0.0, fz = 0.0, e = 0.0, w = 0.0;
    bool bad = false;
    for (int64_t j = lane; j < n; j += 32) {
        if (j == i) continue;
        const double dx = xsub(xi, pos[3 * j]);
        const double dy = xsub(yi, pos[3 * j + 1]);
        const double dz = xsub(zi, pos[3 * j + 2]);
        const double r2 = exact_r2(dx, dy, dz);
        if (r2 < RB_MIN_DISTANCE_SQ) {  // potentials.py:35-36
            bad = true;
            continue;
        }
        const double inv_r2 = 1.0 / r2;
        const double x = sigma2 * inv_r2;
        const double r6 = x * x * x;
        const double r12 = r6 * r6;
        const double scale = eps24 * (2.0 * r12 - r6) * inv_r2;
        fx += scale * dx;
        fy += scale * dy;
        fz += scale * dz;
        e += eps4 * (r12 - r6);
        w += scale * r2;
    }
    fx = group_sum<32>(fx);
    fy = group_sum<32>(fy);
    fz = group_sum<32>(fz);
    e = group_sum<32>(e);
    w = group_sum<32>(w);
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
        forces[3 * i] = fx;
        forces[3 * i + 1] = fy;
        forces[3 * i + 2] = fz;
        energy[i] = 0.5 * e;
        virial[i] = 0.5 * w;
        if (bad) record_status(status, tag, RB_KIND_PAIR_MIN_SEPARATION);
    }
}

// windows of base i (m = n-1-i followers) for T threads per block
__host__ __device__ inline int64_t dt_windows(int64_t m, int T) {
    if (m < 2) return 0;
    if (m >= T) return (m * (m - 1) / 2 + T - 1) / T;
    return m / 2;
}

// prefix[i] = windows of the bases < i, i = 0..n (one block)
__global__ void __launch_bounds__(1024) k_direct_prep(int64_t n, int T,
                                                      int64_t *__restrict__ prefix) {
    pdl_enter();
    __shared__ int64_t part[1024];
    const int64_t per = (n + 1023) / 1024;
    const int64_t b = threadIdx.x * per;
    int64_t sum = 0;
    for (int64_t i = b; i < b + per && i < n; i++) sum += dt_windows(n - 1 - i, T);
    part[threadIdx.x] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {  // serial scan of 1024 partials: negligible next to the pass
        int64_t run = 0;
        for (int t = 0; t < 1024; t++) {
            const int64_t v = part[t];
            part[t] = run;
            run += v;
        }
        prefix[n] = run;
    }
    __syncthreads();
    int64_t run = part[threadIdx.x];
    for (int64_t i = b; i < b + per && i < n; i++) {
        prefix[i] = run;
        run += dt_windows(n - 1 - i, T);
    }
}

template <int kT>
__global__ void __launch_bounds__(kT)
    k_direct_triplets(int64_t n, int64_t i_lo, int64_t i_hi, const double *__restrict__ pos,
                      const int64_t *__restrict__ prefix, double *__restrict__ slab,
                      double *__restrict__ part_ew, unsigned long long *status, int64_t tag) {
    pdl_enter();
    extern __shared__ __align__(16) double fsh[];  // [3][n]: x, y, z force components
    __shared__ double red[32];
    const int tid = threadIdx.x;
    tag = resolve_tag(tag, status);
    for (int64_t q = tid; q < 3 * n; q += kT) fsh[q] = 0.0;
    double *fxs = fsh, *fys = fsh + n, *fzs = fsh + 2 * n;
    // the windows of the bases [i_lo, i_hi), cut into equal block slices
    const int64_t first = prefix[i_lo], total = prefix[i_hi] - first;
    const int64_t lo = first + total * blockIdx.x / gridDim.x;
    const int64_t hi = first + total * (blockIdx.x + 1) / gridDim.x;
    // base of window `lo`: the last i with prefix[i] <= lo
    int64_t i = 0, top = n;
    while (top - i > 1) {
        const int64_t mid = (i + top) >> 1;
        if (prefix[mid] <= lo) i = mid; else top = mid;
    }
    double e_acc = 0.0, w_acc = 0.0;
    bool bad = false;
    __syncthreads();
    for (int64_t win = lo; win < hi; i++) {
        const int64_t m = n - 1 - i;
        const int64_t w_end = min(prefix[i + 1], hi);
        const double xi = pos[3 * i], yi = pos[3 * i + 1], zi = pos[3 * i + 2];
        double fix = 0.0, fiy = 0.0, fiz = 0.0;
        // this thread's pair in the first window of the slice: f = ww * T + tid
        // is (round d, follower s); later windows advance by T pairs
        const int mi = (int)m, pairs = mi * (mi - 1) / 2;
        int f = (int)(win - prefix[i]) * kT + tid;
        int d = f / (mi > 0 ? mi : 1) + 1, s0 = f - (d - 1) * mi;
        for (; win < w_end; win++) {
            int s;
            bool live;
            if (mi >= kT) {
                live = f < pairs;
                s = s0;
            } else {  // one round per window
                d = (int)(win - prefix[i]) + 1;
                live = tid < (2 * d == mi ? d : mi);
                s = tid;
            }
            int t = s + d;
            if (t >= mi) t -= mi;
            if (!live) s = t = 0;
            const int64_t j = i + 1 + s, k = i + 1 + t;
            double fj[3] = {0.0, 0.0, 0.0}, fk[3] = {0.0, 0.0, 0.0};
            bool in = live;
            if (live) {
                const double xj = pos[3 * j], yj = pos[3 * j + 1], zj = pos[3 * j + 2];
                const double xk = pos[3 * k], yk = pos[3 * k + 1], zk = pos[3 * k + 2];
                const double ijx = xsub(xi, xj), ijy = xsub(yi, yj), ijz = xsub(zi, zj);
                const double ikx = xsub(xi, xk), iky = xsub(yi, yk), ikz = xsub(zi, zk);
                const double jkx = xsub(xj, xk), jky = xsub(yj, yk), jkz = xsub(zj, zk);
                const double a = exact_r2(ijx, ijy, ijz);
                const double b = exact_r2(ikx, iky, ikz);
                const double c = exact_r2(jkx, jky, jkz);
                if (a < RB_MIN_DISTANCE_SQ || b < RB_MIN_DISTANCE_SQ || c < RB_MIN_DISTANCE_SQ) {
                    bad = true;  // containers.py:709-711: flag and skip
                    in = false;
                } else {
                    // potentials.py:82-114 with a = r_ij^2, b = r_ik^2, c = r_jk^2
                    const double tsum = a + b + c;
                    const double u = fma(-2.0, c, tsum);
                    const double v = fma(-2.0, b, tsum);
                    const double wv = fma(-2.0, a, tsum);
                    const double p = u * v * wv;
                    const double sp = a * b * c;
                    const double rs = rsqrt_nr(sp);  // seed + third-order step (atm3.cu)
                    const double inv_s = rs * rs;
                    const double s52 = rs * inv_s * inv_s;
                    const double s72 = s52 * inv_s;
                    const double uv = u * v, uw = u * wv, vw = v * wv;
                    const double S = uv + uw + vw;
                    const double A = 0.375 * s52;
                    const double K = fma(1.5, s52, 0.9375 * p * s72);
                    const double ea = fma(A, fma(-2.0, uv, S), -K * (b * c));
                    const double eb = fma(A, fma(-2.0, uw, S), -K * (a * c));
                    const double ec = fma(A, fma(-2.0, vw, S), -K * (a * b));
                    fix = fma(-ea, ijx, fma(-eb, ikx, fix));
                    fiy = fma(-ea, ijy, fma(-eb, iky, fiy));
                    fiz = fma(-ea, ijz, fma(-eb, ikz, fiz));
                    e_acc = fma(s52, fma(0.375, p, sp), e_acc);
                    w_acc = fma(ea, a, fma(eb, b, fma(ec, c, w_acc)));
                    fj[0] = fma(ea, ijx, -ec * jkx);
                    fj[1] = fma(ea, ijy, -ec * jky);
                    fj[2] = fma(ea, ijz, -ec * jkz);
                    fk[0] = fma(eb, ikx, ec * jkx);
                    fk[1] = fma(eb, iky, ec * jky);
                    fk[2] = fma(eb, ikz, ec * jkz);
                }
            }
            if (in) {
                fxs[j] += fj[0];
                fys[j] += fj[1];
                fzs[j] += fj[2];
            }
            __syncthreads();
            if (in) {
                fxs[k] += fk[0];
                fys[k] += fk[1];
                fzs[k] += fk[2];
            }
            __syncthreads();
            f += kT;
            s0 += kT;
            if (s0 >= mi) {  // T <= m: at most one wrap
                s0 -= mi;
                d += 1;
            }
        }
        // f_i of this base (fixed tree), added by thread 0
        const double sx = block_tree_sum<double>(fix, red);
        __syncthreads();
        const double sy = block_tree_sum<double>(fiy, red);
        __syncthreads();
        const double sz = block_tree_sum<double>(fiz, red);
        if (tid == 0) {
            fxs[i] += sx;
            fys[i] += sy;
            fzs[i] += sz;
        }
        __syncthreads();
    }
    double *mine = slab + (int64_t)blockIdx.x * 3 * n;
    for (int64_t q = tid; q < 3 * n; q += kT) mine[q] = fsh[q];
    const double es = block_tree_sum<double>(e_acc, red);
    __syncthreads();
    const double ws = block_tree_sum<double>(w_acc, red);
    const bool any_bad = __syncthreads_or(bad ? 1 : 0) != 0;
    if (tid == 0) {
        part_ew[2 * blockIdx.x] = es;
        part_ew[2 * blockIdx.x + 1] = ws;
        if (any_bad) record_status(status, tag, RB_KIND_TRIPLET_MIN_SEPARATION);
    }
}

// forces[i] = 2 nu sum_b slab[b][i] (block order); energy / virial sums
__global__ void k_direct_finish(int64_t n, int nb, const double *__restrict__ slab,
                                const double *__restrict__ part_ew, double two_nu, double nu,
                                double *__restrict__ forces, double *__restrict__ ew) {
    pdl_enter();
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // component c of i
    if (q < 3 * n) {
        const int64_t i = q / 3, c = q - 3 * i;
        double s = 0.0;
        for (int b = 0; b < nb; b++) s += slab[((int64_t)b * 3 + c) * n + i];
        forces[q] = two_nu * s;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        double e = 0.0, w = 0.0;
        for (int b = 0; b < nb; b++) {
            e += part_ew[2 * b];
            w += part_ew[2 * b + 1];
        }
        ew[0] = nu * e;
        ew[1] = -two_nu * w;
    }
}

// blocks per SM as shared memory allows (the force array is 24 n bytes),
static int dt_per_sm(int64_t n) {
    const size_t smem = (size_t)3 * (n > 0 ? n : 1) * sizeof(double) + 1024;
    int per_sm = (int)((227 * 1024) / (smem + 1024));
    if (per_sm > 8) per_sm = 8;
    if (per_sm < 1) per_sm = 1;
    return per_sm;
}

// 256-thread blocks (cheaper block barriers per window) unless the force
// array leaves room for one block per SM only (measured: 81-89 G triplets/s
// at n = 1024..4096 with 256, 58 vs 48 at n = 8192 with 1024)
static int dt_threads(int64_t n) { return dt_per_sm(n) == 1 ? 1024 : 256; }

static int dt_blocks(int64_t n) { return 148 * dt_per_sm(n); }

}  // namespace rb

using namespace rb;

extern "C" int rb_direct_pairs_range(int64_t n, const double *pos, int64_t i_lo, int64_t i_hi,
                                     double epsilon, double sigma, double *forces,
                                     double *energy_part, double *virial_part,
                                     unsigned long long *status, int64_t tag, void *stream) {
    if (n < 0 || i_lo < 0 || i_hi > n || i_lo > i_hi ||
        (n > 0 && (!pos || !forces || !energy_part || !virial_part)))
        return RB_ERR_ARGUMENT;
    if (i_hi == i_lo) return RB_OK;
    const int64_t threads = 32 * (i_hi - i_lo);
    launch(k_direct_pairs, dim3((unsigned)((threads + kDpThreads - 1) / kDpThreads)), dim3(kDpThreads),
           0, as_stream(stream), n, i_lo, i_hi, pos, 24.0 * epsilon, 4.0 * epsilon, sigma * sigma,
           forces, energy_part, virial_part, status, tag);
    note_launches(1);
    return launch_status();
}

extern "C" int rb_direct_pairs(int64_t n, const double *pos, double epsilon, double sigma,
                               double *forces, double *energy_part, double *virial_part,
                               unsigned long long *status, int64_t tag, void *stream) {
    return rb_direct_pairs_range(n, pos, 0, n, epsilon, sigma, forces, energy_part, virial_part,
                                 status, tag, stream);
}

extern "C" size_t rb_direct_scratch_bytes(int64_t n) {
    const int64_t nn = n > 0 ? n : 1;
    const int nb = dt_blocks(nn);
    return (size_t)(nn + 1) * sizeof(int64_t) + (size_t)nb * 3 * nn * sizeof(double) +
           (size_t)nb * 2 * sizeof(double) + 256;
}

extern "C" int rb_direct_triplets_range(int64_t n, const double *pos, int64_t i_lo,
                                        int64_t i_hi, double nu, double *forces,
                                        double *energy_virial, void *scratch,
                                        size_t scratch_bytes, unsigned long long *status,
                                        int64_t tag, void *stream) {
    if (n < 0 || i_lo < 0 || i_hi > n || i_lo > i_hi ||
        (n > 0 && (!pos || !forces || !energy_virial || !scratch)))
        return RB_ERR_ARGUMENT;
    if (n > kDtMaxN) return RB_ERR_CAPACITY;
    if (scratch_bytes < rb_direct_scratch_bytes(n)) return RB_ERR_ARGUMENT;
    if (n == 0) return RB_OK;
    cudaStream_t st = as_stream(stream);
    const int nb = dt_blocks(n);
    int64_t *prefix = (int64_t *)scratch;
    double *slab = (double *)(prefix + n + 1);
    double *part_ew = slab + (size_t)nb * 3 * n;
    const size_t smem = (size_t)3 * n * sizeof(double);
    const int T = dt_threads(n);
    launch(k_direct_prep, dim3(1), dim3(1024), 0, st, n, T, prefix);
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        launch(kern, dim3(nb), dim3(T), smem, st, n, i_lo, i_hi, pos, (const int64_t *)prefix,
               slab, part_ew, status, tag);
    };
    if (T == 1024)
        go(k_direct_triplets<1024>);
    else
        go(k_direct_triplets<256>);
    const int64_t q = 3 * n;
    launch(k_direct_finish, dim3((unsigned)((q + 255) / 256)), dim3(256), 0, st, n, nb,
           (const double *)slab, (const double *)part_ew, 2.0 * nu, nu, forces, energy_virial);
    note_launches(3);
    return launch_status();
}

extern "C" int rb_direct_triplets(int64_t n, const double *pos, double nu, double *forces,
                                  double *energy_virial, void *scratch, size_t scratch_bytes,
                                  unsigned long long *status, int64_t tag, void *stream) {
    return rb_direct_triplets_range(n, pos, 0, n, nu, forces, energy_virial, scratch,
                                    scratch_bytes, status, tag, stream);
}
