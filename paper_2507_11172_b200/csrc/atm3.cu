// atm3.cu -- Newton-3 Axilrod-Teller-Muto triplet pass: every unique triplet
// i < j < k (rank order) is evaluated exactly once, by the warp of its
// lowest-rank member i, and its three forces are delivered deterministically.
//
// Replaces respamd/containers.py:373-535 (_c01_triplet_kernel).  The C01
// reference evaluates each triplet three times (once per member, force on the
// base particle only); here the expensive kernel (potentials.py:82-114) runs
// once and the partial forces of j and k are accumulated without atomics:
//
//   phase 0  S+(i): the suffix of i's rank-sorted row with rank > i and
//            r_ij^2 <= rc^2 (reference arithmetic) -> per-warp slots in
//            shared memory (d_ij, r_ij^2, row index).
//   phase 1  candidate pairs of slots by ROUNDS: in round d slot s pairs
//            with slot (s + d) mod m, d = 1 .. m/2.  Every unordered slot
//            pair appears exactly once, and inside one round all first slots
//            are distinct and all second slots are distinct.  Per block of
//            rounds each lane tests its own slots' partners (r_jk^2 <= rc^2,
//            settled bit-exactly: fp32 estimate from d_ik - d_ij outside a
//            1e-5 band, fp64 estimate outside a 1e-10 band, else -- or when
//            the box is under four cutoffs -- the reference's raw-position
//            arithmetic) and keeps accept bits; one ballot per (round, slot
//            set) places every accepted pair in a round-major queue.
//   phase 2  the queue is evaluated 32 entries at a time (all lanes busy);
//            f_i stays in registers, f_j and f_k are added to the slot
//            accumulators in shared memory one round at a time, so no two
//            lanes of a sub-step touch the same slot and the order of the
//            additions is fixed by the enumeration.
//   phase 3  slot sums go to the TARGET's row, G[j][position of i in row j];
//            the gather kernel sums, for each particle p, its own part and
//            its row segment G[p][k] over the entries q < p -- in row order.
//
// Energies are phi per triplet (the reference's phi/3 per visit, summed), the
// virial -2(E_a a + E_b b + E_c c) per triplet (:530 summed over visits).
#include <cstdlib>

#include "common.cuh"

#include <type_traits>

namespace rb {

constexpr int kA3Warps = 4;
#ifndef RB_A3_MIN_BLOCKS
#define RB_A3_MIN_BLOCKS 8
#endif
constexpr int kA3MinBlocks = RB_A3_MIN_BLOCKS;  // register cap for occupancy
#ifndef RB_A3_PACKED
#define RB_A3_PACKED 1  // fp32x2 packed candidate filter
#endif
#ifndef RB_A3_QUEUE
#define RB_A3_QUEUE 512
#endif
constexpr int kA3Queue = RB_A3_QUEUE;  // entries: the carry of the last chunk + one round block
constexpr int kA3RoundBlock = 32;    // at most this many rounds per block (bits per word)
constexpr int kA3MaxSlots = 2047;    // queue entries pack s and t in 11 bits each
constexpr double kA3Margin = 1e-10;  // fp64 estimate vs the reference arithmetic
constexpr double kA3Band = 1e-5;     // fp32 filter vs the fp64 estimate

// per-warp shared memory, M slots (S+(i)) + a 64-entry queue
struct A3Smem {
    double2 *dxy;    // slots: (x, y) of d_ij = x_i - x_j
    double *dz, *r2; // slots: z of d_ij, r_ij^2
    double2 *axy;    // slot force accumulators (units of 2 nu), x and y
    double *az;      //   ... z
    float4 *f4;      // slots: d_ij in fp32 for the candidate filter
    int32_t *kidx;   // slot -> row index | owned << 30
    uint32_t *mask;  // slot -> accept bits of the current round block
    uint32_t *vote;  // per round of the block: the ballot of each slot set
    int32_t *vbase;  // per round of the block: queue offset of each slot set
    uint32_t *qe;    // queue: s | t << 11 | (round & 1023) << 22
};

#ifndef RB_A3_WINDOW
#define RB_A3_WINDOW 1  // phase 1 by 32-pair windows (no queue)
#endif

__host__ __device__ inline size_t a3_warp_bytes(int m) {
#if RB_A3_WINDOW
    // d_ij (x,y | z), r_ij^2, accumulators (x,y | z), row index
    size_t b = (size_t)m * (2 * sizeof(double2) + 3 * sizeof(double) + sizeof(int32_t)) + 16;
#else
    size_t b = (size_t)m * (2 * sizeof(double2) + 3 * sizeof(double) + sizeof(float4) +
                            2 * sizeof(int32_t));
    b += (size_t)kA3Queue * sizeof(uint32_t) + 16;  // + alignment pad of f4
    b += (size_t)2 * kA3RoundBlock * ((m + 31) / 32) * sizeof(uint32_t);
#endif
    return (b + 15) & ~(size_t)15;
}

// kM > 0: the slot count is a compile-time constant (every offset folds
// into the shared-memory addressing); kM == 0: runtime m
template <int kM>
__device__ __forceinline__ A3Smem a3_carve(char *base, int m_rt) {
    const int m = kM > 0 ? kM : m_rt;
    A3Smem s;
    s.dxy = (double2 *)base;
    s.axy = s.dxy + m;
    s.dz = (double *)(s.axy + m);
    s.r2 = s.dz + m;
    s.az = s.r2 + m;
#if RB_A3_WINDOW
    s.f4 = nullptr;
    s.kidx = (int32_t *)(s.az + m);
    s.mask = s.vote = s.qe = nullptr;
    s.vbase = nullptr;
    return s;
#endif
    s.f4 = (float4 *)(s.az + m + (m & 1));  // keep 16-byte alignment
    s.kidx = (int32_t *)(s.f4 + m);
    s.mask = (uint32_t *)(s.kidx + m);
    s.qe = s.mask + m;
    s.vote = s.qe + kA3Queue;
    s.vbase = (int32_t *)(s.vote + kA3RoundBlock * ((m + 31) / 32));
    return s;
}

struct A3Acc {
    double fx, fy, fz, e, w;
    int n;
    bool bad;
    int owned_i;     // decomposed runs: the base particle is owned by this rank
    bool slot_bad;   // some r_ij^2 of S+(i) is under the guard (checked per triplet then)
};

constexpr int kKidxMask = 0x3fffffff;

// share of a triplet's energy that belongs to this rank: (owned members)/3
// (the reference attributes phi/3 to each member, containers.py:524)
__device__ __forceinline__ double owned_share(int n_owned) {
    return n_owned == 3 ? 1.0 : (n_owned == 2 ? 2.0 / 3.0 : (n_owned == 1 ? 1.0 / 3.0 : 0.0));
}

// 1/sqrt(x) from an fp32 seed and two Newton steps (2^-23 -> 2^-46 ->
// rounding); CUDA's rsqrt for the rare arguments outside the fp32 range.
__device__ __forceinline__ double rsqrt_nr(double x) {
    if (x < 1e-30 || x > 1e30) return rsqrt(x);
    double y = (double)rsqrtf((float)x);
#pragma unroll
    for (int it = 0; it < 2; it++) {
        const double r = fma(-x * y, y, 1.0);  // 1 - x y^2
        y = fma(0.5 * y, r, y);
    }
    return y;
}

// Evaluate queue entry `q`: adds f_i, E, W to acc and returns f_j, f_k, all
// in units of 2 nu.  With a = r_ij^2, b = r_ik^2, c = r_jk^2, u = a+b-c,
// v = a+c-b, w = b+c-a, p = uvw, S = uv+uw+vw, s = abc (potentials.py:82-114):
//   E   = s^-5/2 (s + 3/8 p)
//   E_a = 3/8 s^-5/2 (S - 2uv) - bc (3/2 s^-5/2 + 15/16 p s^-7/2), b/c alike.
// The ATM kernel for slots (s, t) with a = r_ij^2, b = r_ik^2, c = r_jk^2
// and d_ij (ij, ijz), d_ik (ik, ikz), d_jk = x_j - x_k (jk*).
template <bool kOwned>
__device__ __forceinline__ bool a3_core(const A3Smem &sm, int s, int t, double a, double b,
                                        double c, double2 ij, double ijz, double2 ik, double ikz,
                                        double jkx, double jky, double jkz, A3Acc &acc,
                                        double fj[3], double fk[3]) {
    // guard (potentials.py:35-36): r_ij, r_ik under it were noted per slot
    if (c < RB_MIN_DISTANCE_SQ ||
        (acc.slot_bad && (a < RB_MIN_DISTANCE_SQ || b < RB_MIN_DISTANCE_SQ))) {
        acc.bad = true;
        fj[0] = fj[1] = fj[2] = fk[0] = fk[1] = fk[2] = 0.0;
        return false;
    }
    const double tsum = a + b + c;
    const double u = fma(-2.0, c, tsum);
    const double v = fma(-2.0, b, tsum);
    const double w = fma(-2.0, a, tsum);
    const double p = u * v * w;
    const double sp = a * b * c;
    const double rs = rsqrt_nr(sp);
    const double inv_s = rs * rs;
    const double s52 = rs * inv_s * inv_s;
    const double s72 = s52 * inv_s;
    const double uv = u * v, uw = u * w, vw = v * w;
    const double S = uv + uw + vw;
    const double A = 0.375 * s52;
    const double K = fma(1.5, s52, 0.9375 * p * s72);
    const double ea = fma(A, fma(-2.0, uv, S), -K * (b * c));
    const double eb = fma(A, fma(-2.0, uw, S), -K * (a * c));
    const double ec = fma(A, fma(-2.0, vw, S), -K * (a * b));
    acc.fx = fma(-ea, ij.x, fma(-eb, ik.x, acc.fx));
    acc.fy = fma(-ea, ij.y, fma(-eb, ik.y, acc.fy));
    acc.fz = fma(-ea, ijz, fma(-eb, ikz, acc.fz));
    if (kOwned) {
        const double share =
            owned_share(acc.owned_i + (sm.kidx[s] >> 30) + (sm.kidx[t] >> 30));
        acc.e = fma(share * s52, fma(0.375, p, sp), acc.e);
        acc.w = fma(share, fma(ea, a, fma(eb, b, ec * c)), acc.w);
    } else {
        acc.e = fma(s52, fma(0.375, p, sp), acc.e);
        acc.w = fma(ea, a, fma(eb, b, fma(ec, c, acc.w)));
    }
    acc.n += 1;
    fj[0] = fma(ea, ij.x, -ec * jkx);
    fj[1] = fma(ea, ij.y, -ec * jky);
    fj[2] = fma(ea, ijz, -ec * jkz);
    fk[0] = fma(eb, ik.x, ec * jkx);
    fk[1] = fma(eb, ik.y, ec * jky);
    fk[2] = fma(eb, ikz, ec * jkz);
    return true;
}


template <bool kExactImage, bool kOwned>
__device__ __forceinline__ bool a3_eval(const A3Smem &sm, int q, const Image &im,
                                        const int32_t *__restrict__ row,
                                        const double *__restrict__ pr, A3Acc &acc,
                                        double fj[3], double fk[3], int &s, int &t) {
    const uint32_t qe = sm.qe[q];
    s = (int)(qe & 0x7ffu);
    t = (int)((qe >> 11) & 0x7ffu);
    const double a = sm.r2[s], b = sm.r2[t];
    const double2 ij = sm.dxy[s], ik = sm.dxy[t];
    const double ijz = sm.dz[s], ikz = sm.dz[t];
    double jkx, jky, jkz;  // d_jk = x_j - x_k
    double c;
    if (kExactImage) {
        // the reference's raw-position minimum image (containers.py:497-513)
        const int j = row[sm.kidx[s] & kKidxMask], k = row[sm.kidx[t] & kKidxMask];
        exact_disp(im, pr[3 * j], pr[3 * j + 1], pr[3 * j + 2], pr[3 * k], pr[3 * k + 1],
                   pr[3 * k + 2], jkx, jky, jkz);
        c = exact_r2(jkx, jky, jkz);
    } else {
        jkx = ik.x - ij.x;
        jky = ik.y - ij.y;
        jkz = ikz - ijz;
        c = fma(jkz, jkz, fma(jky, jky, jkx * jkx));
    }
    return a3_core<kOwned>(sm, s, t, a, b, c, ij, ijz, ik, ikz, jkx, jky, jkz, acc, fj, fk);
}

__device__ __forceinline__ void a3_add(double2 *axy, double *az, int slot, const double f[3]) {
    double2 xy = axy[slot];
    xy.x += f[0];
    xy.y += f[1];
    axy[slot] = xy;
    az[slot] += f[2];
}

// evaluate the first `cnt` queue entries and fold f_j / f_k into the slot
// accumulators, one round-record at a time (records are contiguous runs; in
// one round all j slots are distinct and all k slots are distinct)
template <bool kExactImage, bool kOwned>
__device__ __forceinline__ void a3_chunk(const A3Smem &sm, int cnt, int lane, const Image &im,
                                         const int32_t *__restrict__ row,
                                         const double *__restrict__ pr, A3Acc &acc,
                                         int debug_mode, int offset) {
    double fj[3] = {0.0, 0.0, 0.0}, fk[3] = {0.0, 0.0, 0.0};
    int s = 0, t = 0, rec = -1;
    bool pending = false;
    if (lane < cnt) {
        pending = a3_eval<kExactImage, kOwned>(sm, offset + lane, im, row, pr, acc, fj, fk, s, t);
        rec = (int)(sm.qe[offset + lane] >> 22);
    }
    if (debug_mode == 4) {  // debug 4: no slot accumulation
        acc.fx += fj[0] + fk[0] + fj[1] + fk[1] + fj[2] + fk[2];
        return;
    }
    unsigned todo = __ballot_sync(0xffffffffu, pending);
    while (todo) {
        const int r0 = __shfl_sync(0xffffffffu, rec, __ffs(todo) - 1);
        const bool act = pending && rec == r0;
        if (act) a3_add(sm.axy, sm.az, s, fj);
        __syncwarp();
        if (act) a3_add(sm.axy, sm.az, t, fk);
        __syncwarp();
        if (act) pending = false;
        todo = __ballot_sync(0xffffffffu, pending);
    }
}

// r_jk^2 <= rc^2 for the slot pair (s, t), decided bit-exactly: fp32 estimate
// outside a 1e-5 band, fp64 estimate outside a 1e-10 band, else the
// reference's raw-position arithmetic.
template <bool kExactImage>
__device__ __forceinline__ bool a3_accept(const A3Smem &sm, const float4 &ps, int s, int t,
                                          const Image &im, const int32_t *__restrict__ row,
                                          const double *__restrict__ pr, double rc2,
                                          double rc2_lo, double rc2_hi, float rc2f_lo,
                                          float rc2f_hi) {
    if (kExactImage) {
        // box under four cutoffs: d_ik - d_ij need not be the minimum image
        const int jr = row[sm.kidx[s] & kKidxMask], kr = row[sm.kidx[t] & kKidxMask];
        double dx, dy, dz;
        exact_disp(im, pr[3 * jr], pr[3 * jr + 1], pr[3 * jr + 2], pr[3 * kr], pr[3 * kr + 1],
                   pr[3 * kr + 2], dx, dy, dz);
        return exact_r2(dx, dy, dz) <= rc2;
    }
    const float4 pt = sm.f4[t];
    const float ex = pt.x - ps.x, ey = pt.y - ps.y, ez = pt.z - ps.z;
    const float c2f = fmaf(ez, ez, fmaf(ey, ey, ex * ex));
    if (c2f <= rc2f_lo) return true;
    if (c2f > rc2f_hi) return false;
    const double2 js = sm.dxy[s], kt = sm.dxy[t];
    const double ex2 = kt.x - js.x, ey2 = kt.y - js.y, ez2 = sm.dz[t] - sm.dz[s];
    const double c2 = fma(ez2, ez2, fma(ey2, ey2, ex2 * ex2));
    if (c2 <= rc2_lo) return true;
    if (c2 > rc2_hi) return false;
    const int jr = row[sm.kidx[s] & kKidxMask], kr = row[sm.kidx[t] & kKidxMask];
    double dx, dy, dz;
    exact_disp(im, pr[3 * jr], pr[3 * jr + 1], pr[3 * jr + 2], pr[3 * kr], pr[3 * kr + 1],
               pr[3 * kr + 2], dx, dy, dz);
    return exact_r2(dx, dy, dz) <= rc2;
}

// Phase 1, window form.  The m(m-1)/2 slot pairs, enumerated round-major
// (round d = 1 .. m/2 pairs s with (s + d) mod m; for even m the last round
// only s < m/2), are taken 32 at a time: lane l of window w holds pair
// f = 32 w + l (m >= 32) or slot l of round w + 1 (m < 32).  Inside a window
// all first slots are distinct and all second slots are distinct (for
// m > 32 a window spans at most two rounds and s repeats only every m
// pairs), so the partial forces go to the shared-memory slot accumulators
// in two conflict-free sub-steps -- no queue, no serialisation, a fixed
// order.  Each lane decides r_jk^2 <= rc^2 bit-exactly (fp64 estimate from
// d_ik - d_ij outside a 1e-10 band, else the reference's raw-position
// arithmetic; always the latter when the box is under four cutoffs).
// One window step: the pair (s, t) of this lane (live) -- acceptance, the
// ATM kernel (a3_core) and the two conflict-free accumulator sub-steps.
template <bool kExactImage, bool kOwned>
__device__ __forceinline__ void a3_pair(const A3Smem &sm, bool live, int s, int t,
                                        const Image &im, const int32_t *__restrict__ row,
                                        const double *__restrict__ pr, double rc2, double rc2_lo,
                                        double rc2_hi, A3Acc &acc) {
    double fj[3], fk[3];
    bool hit = false;
    if (live) {
        const double2 ij = sm.dxy[s], ik = sm.dxy[t];
        const double ijz = sm.dz[s], ikz = sm.dz[t];
        double jkx, jky, jkz, c;
        bool in;
        if (kExactImage) {
            const int j = row[sm.kidx[s] & kKidxMask], k = row[sm.kidx[t] & kKidxMask];
            exact_disp(im, pr[3 * j], pr[3 * j + 1], pr[3 * j + 2], pr[3 * k], pr[3 * k + 1],
                       pr[3 * k + 2], jkx, jky, jkz);
            c = exact_r2(jkx, jky, jkz);
            in = c <= rc2;
        } else {
            jkx = ik.x - ij.x;
            jky = ik.y - ij.y;
            jkz = ikz - ijz;
            c = fma(jkz, jkz, fma(jky, jky, jkx * jkx));
            in = c <= rc2_lo;
            if (!in && c <= rc2_hi) {  // inside the band: the reference arithmetic decides
                const int j = row[sm.kidx[s] & kKidxMask], k = row[sm.kidx[t] & kKidxMask];
                double ex, ey, ez;
                exact_disp(im, pr[3 * j], pr[3 * j + 1], pr[3 * j + 2], pr[3 * k],
                           pr[3 * k + 1], pr[3 * k + 2], ex, ey, ez);
                in = exact_r2(ex, ey, ez) <= rc2;
            }
        }
        if (in)
            hit = a3_core<kOwned>(sm, s, t, sm.r2[s], sm.r2[t], c, ij, ijz, ik, ikz, jkx, jky,
                                  jkz, acc, fj, fk);
    }
    __syncwarp();
    if (hit) a3_add(sm.axy, sm.az, s, fj);
    __syncwarp();
    if (hit) a3_add(sm.axy, sm.az, t, fk);
}

template <bool kExactImage, bool kOwned>
__device__ __forceinline__ void a3_windows(const A3Smem &sm, int m, int lane, const Image &im,
                                           const int32_t *__restrict__ row,
                                           const double *__restrict__ pr, double rc2,
                                           double rc2_lo, double rc2_hi, A3Acc &acc) {
    if (m >= 32) {
        const int pairs = m * (m - 1) / 2;
        int s = lane, d = 1;  // pair f = f0 + lane is (round d, slot s)
        for (int f0 = 0; f0 < pairs; f0 += 32) {
            int t = s + d;
            if (t >= m) t -= m;
            a3_pair<kExactImage, kOwned>(sm, f0 + lane < pairs, s, t, im, row, pr, rc2, rc2_lo,
                                         rc2_hi, acc);
            s += 32;
            if (s >= m) {
                s -= m;
                d += 1;
            }
        }
    } else {
        for (int d = 1; 2 * d <= m; d++) {
            const int lim = 2 * d == m ? d : m;  // even m: the last round is half
            int t = lane + d;
            if (t >= m) t -= m;
            a3_pair<kExactImage, kOwned>(sm, lane < lim, lane, t, im, row, pr, rc2, rc2_lo,
                                         rc2_hi, acc);
        }
    }
    __syncwarp();
}

// One base particle r (rank order) per warp.  `ovf` (main pass with a
// reduced slot count): a base whose S+(r) does not fit is appended to the
// overflow list ovf[2..] (count ovf[0]) and left to k_atm3_overflow; the
// gather moves the count to ovf[1] and clears ovf[0].
template <bool kExactImage, bool kOwned, int kM>
__device__ __forceinline__ void a3_base(int64_t r, char *smem_raw, const rb_grid &g, int64_t n, const double *__restrict__ pr,
                                       const int32_t *__restrict__ rows,
                                       const int32_t *__restrict__ row_count,
                                       const int32_t *__restrict__ mirror, int32_t capacity,
                                       int32_t slots, double rc2, double rc2_lo, double rc2_hi,
                                       float rc2f_lo, float rc2f_hi, double *__restrict__ own,
                                       double *__restrict__ gbuf,
                                       double *__restrict__ energy_rank,
                                       double *__restrict__ virial_rank,
                                       int32_t *__restrict__ triplets_rank,
                                       const uint8_t *__restrict__ owned,
                                       unsigned long long *status, int64_t tag, int debug_mode,
                                       int32_t *ovf) {
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    tag = resolve_tag(tag, status);
    if (warp_frozen(status, tag, RB_KIND_TRIPLET_MIN_SEPARATION)) return;
    if (kM > 0) slots = kM;
    const A3Smem sm = a3_carve<kM>(smem_raw + (size_t)warp * a3_warp_bytes(slots), slots);
    const Image im = make_image(g);
    const double xi = pr[3 * r], yi = pr[3 * r + 1], zi = pr[3 * r + 2];
    const int rc_n = row_count[r];
    const int32_t *row = rows + r * (int64_t)capacity;
    const int32_t *mir = mirror + r * (int64_t)capacity;
    // partial forces go to the TARGET's row: G[q][position of i in row q], so
    // the gather of q reads its own row segment contiguously

    // ---- phase 0: S+(i), the row suffix with rank > i within rc
    int m = 0;
    bool slot_bad = false;
    for (int base = 0; base < rc_n; base += 32) {
        const int k = base + lane;
        bool keep = false;
        double dx = 0.0, dy = 0.0, dz = 0.0, r2 = 0.0;
        if (k < rc_n) {
            const int q = row[k];
            if (q > r) {
                exact_disp(im, xi, yi, zi, pr[3 * q], pr[3 * q + 1], pr[3 * q + 2], dx, dy, dz);
                r2 = exact_r2(dx, dy, dz);
                keep = r2 <= rc2;
                if (!keep) {  // beyond the three-body cutoff: contributes nothing
                    double *gq = gbuf + ((int64_t)q * capacity + mir[k]) * 3;
                    gq[0] = 0.0;
                    gq[1] = 0.0;
                    gq[2] = 0.0;
                }
            }
        }
        const unsigned mk = __ballot_sync(0xffffffffu, keep);
        if (m + __popc(mk) > slots) {  // S+(i) does not fit the shared-memory slots
            if (lane == 0) {
                if (ovf)
                    ovf[2 + atomicAdd(ovf, 1)] = (int32_t)r;
                else
                    record_status(status, tag, RB_KIND_CAPACITY);
            }
            return;
        }
        if (keep) {
            const int slot = m + __popc(mk & lanemask_lt());
            sm.dxy[slot] = make_double2(dx, dy);
            sm.dz[slot] = dz;
            sm.r2[slot] = r2;
            sm.kidx[slot] = k | ((kOwned ? (int)owned[row[k]] : 1) << 30);
#if !RB_A3_WINDOW
            sm.f4[slot] = make_float4((float)dx, (float)dy, (float)dz, 0.0f);
#endif
            sm.axy[slot] = make_double2(0.0, 0.0);
            sm.az[slot] = 0.0;
        }
        m += __popc(mk);
        slot_bad |= __any_sync(0xffffffffu, keep && r2 < RB_MIN_DISTANCE_SQ);
    }
    __syncwarp();

    // ---- phase 1: rounds.  Round d (1..m/2) pairs slot s with (s + d) mod m
    // (for even m the last round only s < m/2): every unordered pair once.
    // Per block of rounds: (A) each lane tests its own slots' partners and
    // keeps accept bits; (B) one ballot per (round, slot set) gives every
    // accepted pair its queue position in round-major order, each lane
    // writes its own pairs; (C) the queue is evaluated 32 entries at a time,
    // the incomplete tail carried to the next block.
    A3Acc acc = {0.0, 0.0, 0.0, 0.0, 0.0, 0, false, kOwned ? (int)owned[r] : 1, slot_bad};
#if RB_A3_WINDOW
    if (debug_mode != 1)  // debug 1: phases 0 and 3 only
        a3_windows<kExactImage, kOwned>(sm, m, lane, im, row, pr, rc2, rc2_lo, rc2_hi, acc);
#else
    const int rounds = debug_mode == 1 ? 0 : (m >> 1);  // debug 1: phases 0 and 3 only
    const int nsets = (m + 31) >> 5;
    const int block = max(1, min(kA3RoundBlock, (kA3Queue - 32) / max(m, 1)));
    int qn = 0;  // carried entries at the queue head
    for (int d0 = 1; d0 <= rounds; d0 += block) {
        const int dn = min(block, rounds - d0 + 1);
        // (A) accept bits
        for (int sg = 0; sg < nsets; sg++) {
            const int s = (sg << 5) + lane;
            uint32_t bits = 0u;
            if (s < m) {
                const float4 ps = sm.f4[s];
                const int elim = (2 * (d0 + dn - 1) == m && s >= d0 + dn - 1) ? dn - 1 : dn;
                int t = s + d0;
                if (t >= m) t -= m;
                int e = 0;
                if (!kExactImage && RB_A3_PACKED) {
                    // two partners per step with packed fp32x2 math; the rare
                    // pairs inside the band go through a3_accept
                    const float2 nx = make_float2(-ps.x, -ps.x), ny = make_float2(-ps.y, -ps.y),
                                 nz = make_float2(-ps.z, -ps.z);
                    for (; e + 1 < elim; e += 2) {
                        int t2 = t + 1;
                        if (t2 == m) t2 = 0;
                        const float4 p1 = sm.f4[t], p2 = sm.f4[t2];
                        const float2 ex = __fadd2_rn(make_float2(p1.x, p2.x), nx);
                        const float2 ey = __fadd2_rn(make_float2(p1.y, p2.y), ny);
                        const float2 ez = __fadd2_rn(make_float2(p1.z, p2.z), nz);
                        const float2 c2 = __ffma2_rn(ez, ez, __ffma2_rn(ey, ey, __fmul2_rn(ex, ex)));
                        if (c2.x <= rc2f_lo) bits |= 1u << e;
                        else if (c2.x <= rc2f_hi &&
                                 a3_accept<kExactImage>(sm, ps, s, t, im, row, pr, rc2, rc2_lo,
                                                        rc2_hi, rc2f_lo, rc2f_hi))
                            bits |= 1u << e;
                        if (c2.y <= rc2f_lo) bits |= 2u << e;
                        else if (c2.y <= rc2f_hi &&
                                 a3_accept<kExactImage>(sm, ps, s, t2, im, row, pr, rc2, rc2_lo,
                                                        rc2_hi, rc2f_lo, rc2f_hi))
                            bits |= 2u << e;
                        t = t2 + 1;
                        if (t == m) t = 0;
                    }
                }
                for (; e < elim; e++) {
                    if (a3_accept<kExactImage>(sm, ps, s, t, im, row, pr, rc2, rc2_lo, rc2_hi,
                                               rc2f_lo, rc2f_hi))
                        bits |= 1u << e;
                    if (++t == m) t = 0;
                }
            }
            if (s < m) sm.mask[s] = bits;
            if (debug_mode == 2) continue;
            // (B1) ballots per round of this set -> counts
            for (int e = 0; e < dn; e++) {
                const unsigned b = __ballot_sync(0xffffffffu, (bits >> e) & 1u);
                if (lane == 0) sm.vote[e * nsets + sg] = b;
            }
        }
        if (debug_mode == 2) continue;  // debug 2: accept bits only
        __syncwarp();
        // (B2) round-major offsets: vbase[e*nsets+sg] = exclusive prefix of the
        // vote counts (warp scan), then every lane places its own pairs
        const int nv = dn * nsets;
        int carry = qn;
        for (int v0 = 0; v0 < nv; v0 += 32) {
            const int c = v0 + lane < nv ? __popc(sm.vote[v0 + lane]) : 0;
            int incl = c;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl += y;
            }
            if (v0 + lane < nv) sm.vbase[v0 + lane] = carry + incl - c;
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        __syncwarp();
        for (int sg = 0; sg < nsets; sg++) {
            const int s = (sg << 5) + lane;
            uint32_t bits = s < m ? sm.mask[s] : 0u;
            while (bits) {
                const int e = __ffs(bits) - 1;
                bits &= bits - 1u;
                const int v = e * nsets + sg;
                const int pos = sm.vbase[v] + __popc(sm.vote[v] & lanemask_lt());
                int t = s + d0 + e;
                if (t >= m) t -= m;
                sm.qe[pos] = (uint32_t)s | ((uint32_t)t << 11) | ((uint32_t)((d0 + e) & 1023) << 22);
            }
        }
        qn = carry;
        __syncwarp();
        // (C) full chunks
        int done = 0;
        for (; done + 32 <= qn; done += 32) {
            if (debug_mode != 3)
                a3_chunk<kExactImage, kOwned>(sm, 32, lane, im, row, pr, acc, debug_mode, done);
        }
        __syncwarp();
        if (done > 0 && lane < qn - done) sm.qe[lane] = sm.qe[done + lane];
        qn -= done;
        __syncwarp();
    }
    if (qn > 0 && debug_mode != 3 && debug_mode != 2)
        a3_chunk<kExactImage, kOwned>(sm, qn, lane, im, row, pr, acc, debug_mode, 0);
    __syncwarp();
#endif

    // ---- phase 3: slot sums -> G[i][row index]; own part, scalars
    for (int sl = lane; sl < m; sl += 32) {
        const int k = sm.kidx[sl] & kKidxMask;
        const double2 xy = sm.axy[sl];
        double *gq = gbuf + ((int64_t)row[k] * capacity + mir[k]) * 3;
        gq[0] = xy.x;
        gq[1] = xy.y;
        gq[2] = sm.az[sl];
    }
    const double fx = group_sum<32>(acc.fx);
    const double fy = group_sum<32>(acc.fy);
    const double fz = group_sum<32>(acc.fz);
    const double e = group_sum<32>(acc.e);
    const double w = group_sum<32>(acc.w);
    const int nt = group_sum_int<32>(acc.n);
    const bool bad = __any_sync(0xffffffffu, acc.bad);
    if (lane == 0) {
        own[3 * r] = fx;
        own[3 * r + 1] = fy;
        own[3 * r + 2] = fz;
        energy_rank[r] = e;
        virial_rank[r] = w;
        triplets_rank[r] = nt;
        if (bad) record_status(status, tag, RB_KIND_TRIPLET_MIN_SEPARATION);
    }
}

template <bool kExactImage, bool kOwned, int kM>
__global__ void __launch_bounds__(kA3Warps * 32, kA3MinBlocks)
    k_atm3(rb_grid g, int64_t n, const double *__restrict__ pr, const int32_t *__restrict__ rows,
           const int32_t *__restrict__ row_count, const int32_t *__restrict__ mirror,
           int32_t capacity, int32_t slots, double rc2, double rc2_lo, double rc2_hi,
           float rc2f_lo, float rc2f_hi, double *__restrict__ own, double *__restrict__ gbuf,
           double *__restrict__ energy_rank, double *__restrict__ virial_rank,
           int32_t *__restrict__ triplets_rank, const uint8_t *__restrict__ owned,
           unsigned long long *status, int64_t tag, int debug_mode, int32_t *ovf) {
    pdl_enter();
    extern __shared__ __align__(16) char smem_raw[];
    const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (r >= n) return;
    a3_base<kExactImage, kOwned, kM>(r, smem_raw, g, n, pr, rows, row_count, mirror, capacity, slots, rc2, rc2_lo,
                            rc2_hi, rc2f_lo, rc2f_hi, own, gbuf, energy_rank, virial_rank,
                            triplets_rank, owned, status, tag, debug_mode, ovf);
}

// the bases listed by the main pass, with the full slot count
template <bool kExactImage, bool kOwned>
__global__ void __launch_bounds__(kA3Warps * 32)
    k_atm3_overflow(rb_grid g, int64_t n, const double *__restrict__ pr, const int32_t *__restrict__ rows,
           const int32_t *__restrict__ row_count, const int32_t *__restrict__ mirror,
           int32_t capacity, int32_t slots, double rc2, double rc2_lo, double rc2_hi,
           float rc2f_lo, float rc2f_hi, double *__restrict__ own, double *__restrict__ gbuf,
           double *__restrict__ energy_rank, double *__restrict__ virial_rank,
           int32_t *__restrict__ triplets_rank, const uint8_t *__restrict__ owned,
           unsigned long long *status, int64_t tag, int debug_mode, const int32_t *ovf) {
    pdl_enter();
    extern __shared__ __align__(16) char smem_raw[];
    const int wpb = blockDim.x >> 5;
    const int cnt = *(volatile const int32_t *)ovf;
    for (int64_t q = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); q < cnt;
         q += (int64_t)gridDim.x * wpb) {
        a3_base<kExactImage, kOwned, 0>(ovf[2 + q], smem_raw, g, n, pr, rows, row_count, mirror,
                                        capacity, slots, rc2, rc2_lo, rc2_hi, rc2f_lo, rc2f_hi,
                                        own, gbuf, energy_rank, virial_rank, triplets_rank,
                                        owned, status, tag, debug_mode, nullptr);
        __syncwarp();  // the warp's slots are reused by its next base
    }
}

// F(p) = 2 nu * (own(p) + sum over row entries k of p with q = row[k] < p of
// G[p][k]); the row prefix is walked in order by kG lanes, then a fixed xor
// tree.
constexpr int kGatherGroup = 8;

__global__ void k_atm3_gather(int64_t n, const int32_t *__restrict__ parts,
                              const int32_t *__restrict__ rows,
                              const int32_t *__restrict__ row_count,
                              const int32_t *__restrict__ mirror, int32_t capacity,
                              const double *__restrict__ own, const double *__restrict__ gbuf,
                              double two_nu, double nu, double *__restrict__ forces,
                              double *__restrict__ energy_rank, double *__restrict__ virial_rank,
                              const unsigned long long *status, int64_t tag, int32_t *ovf) {
    pdl_enter();
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // list empty for the next pass
        ovf[1] = ovf[0];                           // (count of this pass: diagnostic)
        ovf[0] = 0;
    }
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t p = gid / kGatherGroup;
    const int sub = (int)(gid % kGatherGroup);
    const bool active = p < n;
    tag = resolve_tag(tag, status);
    if (warp_frozen(status, tag, RB_KIND_TRIPLET_MIN_SEPARATION)) return;
    double fx = 0.0, fy = 0.0, fz = 0.0;
    if (active) {
        const int m = row_count[p];
        const int32_t *row = rows + p * (int64_t)capacity;
        const double *gp = gbuf + p * (int64_t)capacity * 3;
        for (int k = sub; k < m; k += kGatherGroup) {
            if (row[k] >= p) break;  // rows are rank-sorted: the prefix q < p
            fx += gp[3 * k];
            fy += gp[3 * k + 1];
            fz += gp[3 * k + 2];
        }
    }
    fx = group_sum<kGatherGroup>(fx);
    fy = group_sum<kGatherGroup>(fy);
    fz = group_sum<kGatherGroup>(fz);
    if (active && sub == 0) {
        const int64_t pp = parts ? parts[p] : p;
        forces[3 * pp] = two_nu * (own[3 * p] + fx);
        forces[3 * pp + 1] = two_nu * (own[3 * p + 1] + fy);
        forces[3 * pp + 2] = two_nu * (own[3 * p + 2] + fz);
        energy_rank[p] = nu * energy_rank[p];
        virial_rank[p] = -two_nu * virial_rank[p];
    }
}

template <typename K>
static void a3_grant(K kernel, size_t bytes, size_t &granted) {
    if (bytes > 48 * 1024 && bytes > granted) {
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        granted = bytes;
    }
}

}  // namespace rb

using namespace rb;

extern "C" size_t rb_atm_scratch_bytes(int64_t n, int32_t capacity) {
    // own (n x 3) + G (n x capacity x 3), doubles; overflow list (1 + n) int32
    const size_t nn = (size_t)(n > 0 ? n : 1);
    return nn * 3 * sizeof(double) * (size_t)(1 + capacity) + (nn + 2) * sizeof(int32_t);
}

namespace rb {
// Slots of the main launch.  S+(r) of most bases is about half a row; only
// bases whose neighbours mostly follow them in rank order (cells next to the
// periodic wrap of the cell order) approach a full row.  Sizing every warp's
// shared memory for the longest S+ costs occupancy, so the main launch takes
// about half the slots and lists the few longer bases for a second launch.
static int a3_fast_slots(int slot_capacity) {
    int f = ((slot_capacity * 11 / 20) + 31) / 32 * 32;  // ~0.55 of the full count
    f = f < 64 ? 64 : f;
    return f >= slot_capacity ? slot_capacity : f;
}

static int a3_warps_for(size_t per) {
    int warps = kA3Warps;
    while (warps > 1 && (size_t)warps * per > 227 * 1024) warps--;
    return (size_t)warps * per > 227 * 1024 ? 0 : warps;
}

template <bool kExactImage, bool kOwned, int kM>
static void a3_launch_main(cudaStream_t st, int64_t n, int warps, size_t per, const rb_grid &g,
                           const double *pos_r, const int32_t *rows, const int32_t *row_count,
                           const int32_t *mirror, int32_t capacity, int fast, double rc2,
                           double lo, double hi, float flo, float fhi, double *own, double *gbuf,
                           double *energy_rank, double *virial_rank, int32_t *triplets_rank,
                           const uint8_t *owned, unsigned long long *status, int64_t tag,
                           int debug_mode, int32_t *ovf) {
    static size_t granted = 0;
    a3_grant(k_atm3<kExactImage, kOwned, kM>, warps * per, granted);
    launch(k_atm3<kExactImage, kOwned, kM>, dim3((unsigned)((n + warps - 1) / warps)),
           dim3(warps * 32), warps * per, st, g, n, pos_r, rows, row_count, mirror, capacity,
           fast, rc2, lo, hi, flo, fhi, own, gbuf, energy_rank, virial_rank, triplets_rank, owned,
           status, tag, debug_mode, ovf);
    note_launches(1);
}

template <bool kExactImage, bool kOwned>
static void a3_launch(cudaStream_t st, const rb_grid &g, int64_t n, const double *pos_r,
                      const int32_t *rows, const int32_t *row_count, const int32_t *mirror,
                      int32_t capacity, int fast, int full, double rc2, double lo, double hi,
                      double *own, double *gbuf, double *energy_rank, double *virial_rank,
                      int32_t *triplets_rank, const uint8_t *owned, unsigned long long *status,
                      int64_t tag, int debug_mode, int32_t *ovf) {
    static size_t granted_ovf = 0;
    const float flo = (float)(rc2 * (1.0 - kA3Band)), fhi = (float)(rc2 * (1.0 + kA3Band));
    const size_t per = a3_warp_bytes(fast);
    const int warps = a3_warps_for(per);
    const bool split = fast < full;
    int32_t *list = split ? ovf : nullptr;
    // the common slot counts get compile-time layouts
    if (fast == 64)
        a3_launch_main<kExactImage, kOwned, 64>(st, n, warps, per, g, pos_r, rows, row_count,
                                                mirror, capacity, fast, rc2, lo, hi, flo, fhi, own,
                                                gbuf, energy_rank, virial_rank, triplets_rank,
                                                owned, status, tag, debug_mode, list);
    else if (fast == 96)
        a3_launch_main<kExactImage, kOwned, 96>(st, n, warps, per, g, pos_r, rows, row_count,
                                                mirror, capacity, fast, rc2, lo, hi, flo, fhi, own,
                                                gbuf, energy_rank, virial_rank, triplets_rank,
                                                owned, status, tag, debug_mode, list);
    else
        a3_launch_main<kExactImage, kOwned, 0>(st, n, warps, per, g, pos_r, rows, row_count,
                                               mirror, capacity, fast, rc2, lo, hi, flo, fhi, own,
                                               gbuf, energy_rank, virial_rank, triplets_rank,
                                               owned, status, tag, debug_mode, list);
    if (!split) return;
    const size_t per_full = a3_warp_bytes(full);
    const int wf = a3_warps_for(per_full);
    const int64_t need = (n + wf - 1) / wf;
    const unsigned blocks = (unsigned)(need < 148 * 4 ? need : 148 * 4);
    a3_grant(k_atm3_overflow<kExactImage, kOwned>, wf * per_full, granted_ovf);
    launch(k_atm3_overflow<kExactImage, kOwned>, dim3(blocks), dim3(wf * 32), wf * per_full, st,
           g, n, pos_r, rows, row_count, mirror, capacity, full, rc2, lo, hi, flo, fhi, own, gbuf,
           energy_rank, virial_rank, triplets_rank, owned, status, tag, debug_mode,
           (const int32_t *)ovf);
    note_launches(1);
}
}  // namespace rb

extern "C" int rb_atm_pass(const rb_grid *g, int64_t n, const double *pos_r, const int32_t *cell_particles, const int32_t *rows,
                           const int32_t *row_count, const int32_t *mirror, int32_t capacity,
                           int32_t slot_capacity, double rc, double nu, double *forces, double *energy_rank,
                           double *virial_rank, int32_t *triplets_rank, const uint8_t *owned,
                           void *scratch, size_t scratch_bytes, unsigned long long *status,
                           int64_t tag, void *stream) {
    if (!g || n < 0 || capacity <= 0 || capacity > 4096 || !mirror || !scratch) return RB_ERR_ARGUMENT;
    if (slot_capacity <= 0 || slot_capacity > capacity) slot_capacity = capacity;
    if (slot_capacity > kA3MaxSlots) return RB_ERR_CAPACITY;
    if (scratch_bytes < rb_atm_scratch_bytes(n, capacity)) return RB_ERR_ARGUMENT;
    if (n == 0) return RB_OK;
    const double rc2 = rc * rc;
    static const int debug_mode = getenv("RB_ATM_DEBUG") ? atoi(getenv("RB_ATM_DEBUG")) : 0;
    static const int no_split = getenv("RB_ATM_NO_SPLIT") ? atoi(getenv("RB_ATM_NO_SPLIT")) : 0;
    bool exact_image = false;
    if (g->periodic)
        for (int d = 0; d < 3; d++)
            if (!(g->box[d] > 4.0 * rc * (1.0 + 1e-12))) exact_image = true;
    if (!a3_warps_for(a3_warp_bytes(slot_capacity))) return RB_ERR_ARGUMENT;
    const int fast = no_split ? slot_capacity : a3_fast_slots(slot_capacity);
    cudaStream_t st = as_stream(stream);
    double *own = (double *)scratch;
    double *gbuf = own + 3 * n;
    int32_t *ovf = (int32_t *)(gbuf + (size_t)n * capacity * 3);
    const double lo = exact_image ? rc2 : rc2 * (1.0 - kA3Margin);
    const double hi = exact_image ? rc2 : rc2 * (1.0 + kA3Margin);
    auto go = [&](auto exact, auto with_owned) {
        a3_launch<decltype(exact)::value, decltype(with_owned)::value>(
            st, *g, n, pos_r, rows, row_count, mirror, capacity, fast, slot_capacity, rc2, lo, hi,
            own, gbuf, energy_rank, virial_rank, triplets_rank, owned, status, tag, debug_mode,
            ovf);
    };
    using T = std::true_type;
    using F = std::false_type;
    if (exact_image)
        owned ? go(T{}, T{}) : go(T{}, F{});
    else
        owned ? go(F{}, T{}) : go(F{}, F{});
    const int tb = 256;
    const int64_t threads = n * kGatherGroup;
    launch(k_atm3_gather, dim3((unsigned)((threads + tb - 1) / tb)), dim3(tb), 0, st, n, cell_particles, rows, row_count, mirror, capacity, own, gbuf, 2.0 * nu, nu, forces,
        energy_rank, virial_rank, status, tag, ovf);
    note_launches(1);
    return launch_status();
}
