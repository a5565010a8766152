// atm_core.cuh -- the Newton-3 ATM pair loop shared by the row-based
// (atm3.cu) and cell-based (atm_cells.cu) triplet passes: the per-warp slot
// layout of S+(i), the ATM kernel (potentials.py:82-114), the bit-exact
// r_jk acceptance and the conflict-free rotation-round enumeration of the
// slot pairs.
#pragma once

#include "common.cuh"

namespace rb {

#ifndef RB_A3_SHFL_IN
#define RB_A3_SHFL_IN 0
#endif
constexpr double kA3Margin = 1e-10;  // fp64 estimate vs the reference arithmetic

// per-warp shared memory: M slots of S+(i) plus one dummy slot (index M)
// that dead lanes of a window read and accumulate into, so the window loop
// has no branches around its shared-memory traffic.  16-byte rows (lanes
// reading consecutive slots are conflict-free): a slot's record is
// xy[s] = (x, y) and zr[s] = (z, r^2) of d_ij = x_i - x_j; its force sum
// (units of 2 nu) is axy[s], az[s].
struct A3Smem {
    double2 *xy, *zr;  // [M + 1]
    double2 *axy;      // [M + 1]
    double *az;        // [M + 1]
    double *ae;        // [M + 1] energy of the slot's triplets (owned shares, atm_rot.cuh)
    double *aw;        // [M + 1] scalar part of a slot's sum in the cross rounds (atm_rot.cuh)
    int32_t *kidx;     // row index | owned << 30
    int32_t *q;        // the slot's particle (rank) ...
    int32_t *mpos;     //   ... and the base's position in its row (G target)
};

__host__ __device__ inline size_t a3_warp_bytes(int m) {
    size_t b = (size_t)(m + 1) * (3 * sizeof(double2) + 3 * sizeof(double)) +
               (size_t)m * 3 * sizeof(int32_t);
    return (b + 15) & ~(size_t)15;
}

// kM > 0: the slot count is a compile-time constant (every offset folds
// into the shared-memory addressing); kM == 0: runtime m
template <int kM>
__device__ __forceinline__ A3Smem a3_carve(char *base, int m_rt) {
    const int m = kM > 0 ? kM : m_rt;
    A3Smem s;
    s.xy = (double2 *)base;
    s.zr = s.xy + (m + 1);
    s.axy = s.zr + (m + 1);
    s.az = (double *)(s.axy + (m + 1));
    s.ae = s.az + (m + 1);
    s.aw = s.ae + (m + 1);
    s.kidx = (int32_t *)(s.aw + (m + 1));
    s.q = s.kidx + m;
    s.mpos = s.q + m;
    return s;
}

__device__ __forceinline__ void ld_rec(const A3Smem &sm, int s, double &x, double &y, double &z,
                                       double &w) {
    RB_CHECK(s >= 0 && s <= 4096);
    const double2 a = sm.xy[s];
    const double2 b = sm.zr[s];
    x = a.x;
    y = a.y;
    z = b.x;
    w = b.y;
}

// slot s's force sum += f (x, y, z)
__device__ __forceinline__ void acc_add(const A3Smem &sm, int s, double fx, double fy, double fz) {
    RB_CHECK(s >= 0 && s <= 4096);
    double2 xy = sm.axy[s];
    double zz = sm.az[s];
    xy.x += fx;
    xy.y += fy;
    zz += fz;
    sm.axy[s] = xy;
    sm.az[s] = zz;
}

struct A3Acc {
    double e, w;     // per-triplet sums only where phase 3 cannot recover them
    int n;
    bool bad;
    int owned_i;     // decomposed runs: the base particle is owned by this rank
};

constexpr int kKidxMask = 0x3fffffff;

// share of a triplet's energy that belongs to this rank: (owned members)/3
// (the reference attributes phi/3 to each member, containers.py:524)
__device__ __forceinline__ double owned_share(int n_owned) {
    return n_owned == 3 ? 1.0 : (n_owned == 2 ? 2.0 / 3.0 : (n_owned == 1 ? 1.0 / 3.0 : 0.0));
}

// Acceptance thresholds on the high word of r_jk^2 (for positive doubles
// the order of the high words is the order of the values): below lo_hi the
// fp64 estimate is certainly under rc^2 (1 - 1e-10), above hi_hi certainly
// over rc^2 (1 + 1e-10); in between (values within ~2^-20 of rc^2), or under
// min_hi (the guard), the reference arithmetic decides.  Integer compares:
// no FP64 pipe work for the acceptance.
struct A3Cut {
    double rc2;
    int lo_hi, hi_hi, min_hi;
};

// The ATM kernel for one slot pair, all in units of nu (potentials.py:82-114).
// With a = r_ij^2, b = r_ik^2, c = r_jk^2, u = a+b-c, v = a+c-b, w = b+c-a,
// p = uvw, S = uv+uw+vw, s = abc:
//   E   = s^-5/2 (s + 3/8 p)
//   E_a = 3/8 s^-5/2 (S - 2uv) - bc (3/2 s^-5/2 + 15/16 p s^-7/2), b/c alike.
// Returns E_a, E_b, E_c; *e = E when kEnergy (decomposed runs and boxes
// under four cutoffs; elsewhere phase 3 recovers the energy from the virial:
// E is homogeneous of degree -9/2 in (a, b, c), so a E_a + b E_b + c E_c =
// -9/2 E per triplet).
template <bool kEnergy>
__device__ __forceinline__ void atm_scalars(double a, double b, double c, double &ea, double &eb,
                                            double &ec, double *e) {
    const double tsum = a + b + c;
    const double u = fma(-2.0, c, tsum);
    const double v = fma(-2.0, b, tsum);
    const double w = fma(-2.0, a, tsum);
    const double uv = u * v, uw = u * w, vw = v * w;
    const double p = uv * w;
    const double sp = a * b * c;
    const double rs = rsqrt_nr(sp);
    const double inv_s = rs * rs;
    const double s52 = rs * inv_s * inv_s;
    const double S = uv + uw + vw;
    const double A = 0.375 * s52;
    const double K = s52 * fma(0.9375 * p, inv_s, 1.5);
    ea = fma(A, fma(-2.0, uv, S), -K * (b * c));
    eb = fma(A, fma(-2.0, uw, S), -K * (a * c));
    ec = fma(A, fma(-2.0, vw, S), -K * (a * b));
    if (kEnergy) *e = s52 * fma(0.375, p, sp);
}

// One window step for one lane: slot pair (s, t) with d_ij = (ijx, ijy,
// ijz), a = r_ij^2 (from registers or the record of s).  Decides r_jk^2 <=
// rc^2 bit-exactly, evaluates the ATM kernel unconditionally and returns
// f_j, f_k (units of 2 nu) -- zero for a rejected pair (the scalars are
// selected, so the accumulation needs no predicate).
template <bool kExactImage, bool kOwned, bool kSlotBad>
__device__ __forceinline__ void a3_pair(const A3Smem &sm, bool live, int s, int t, double ijx,
                                        double ijy, double ijz, double a, double ikx, double iky,
                                        double ikz, double b, const rb_grid &g,
                                        const double *__restrict__ pr, const A3Cut &cut,
                                        A3Acc &acc, double fj[3], double fk[3]) {
    double jkx = ikx - ijx, jky = iky - ijy, jkz = ikz - ijz;
    double c = fma(jkz, jkz, fma(jky, jky, jkx * jkx));
    bool in;
    bool bad = false;
    if (kExactImage) {  // box under four cutoffs: d_ik - d_ij need not be a minimum image
        in = false;
        if (live) {
            const Image im = make_image(g);
            const int j = sm.q[s], k = sm.q[t];
            exact_disp(im, pr[3 * j], pr[3 * j + 1], pr[3 * j + 2], pr[3 * k], pr[3 * k + 1],
                       pr[3 * k + 2], jkx, jky, jkz);
            c = exact_r2(jkx, jky, jkz);
            in = c <= cut.rc2;
            bad = in && c < RB_MIN_DISTANCE_SQ;
        }
    } else {
        const int ch = __double2hiint(c);
        in = live && ch < cut.lo_hi && ch > cut.min_hi;
        const bool sus = live && !in && ch <= cut.hi_hi;
        if (__any_sync(0xffffffffu, sus)) {  // rare: the reference arithmetic decides
            if (sus) {
                const Image im = make_image(g);  // from the kernel parameters, on demand
                const int j = sm.q[s], k = sm.q[t];
                double ex, ey, ez;
                exact_disp(im, pr[3 * j], pr[3 * j + 1], pr[3 * j + 2], pr[3 * k],
                           pr[3 * k + 1], pr[3 * k + 2], ex, ey, ez);
                const double ce = exact_r2(ex, ey, ez);
                in = ce <= cut.rc2;
                bad = in && ce < RB_MIN_DISTANCE_SQ;
            }
        }
    }
    // guard (potentials.py:35-36) on r_ij / r_ik: only if phase 0 saw a slot
    // under it (uniform per base: the loop is instantiated for both)
    if (kSlotBad) bad = bad || (in && (a < RB_MIN_DISTANCE_SQ || b < RB_MIN_DISTANCE_SQ));
    acc.bad = acc.bad || bad;
    in = in && !bad;
    double ea, eb, ec, e;
    atm_scalars<kOwned || kExactImage>(a, b, c, ea, eb, ec, &e);
    if (kOwned) {
        const double share = owned_share(acc.owned_i + (sm.kidx[s] >> 30) + (sm.kidx[t] >> 30));
        if (in) {
            acc.e = fma(share, e, acc.e);
            acc.w = fma(share, fma(ea, a, fma(eb, b, ec * c)), acc.w);
        }
    } else if (kExactImage) {
        if (in) {
            acc.e += e;
            acc.w = fma(ea, a, fma(eb, b, fma(ec, c, acc.w)));
        }
    }
    acc.n += in ? 1 : 0;
    ea = in ? ea : 0.0;
    eb = in ? eb : 0.0;
    ec = in ? ec : 0.0;
    const double cx = ec * jkx, cy = ec * jky, cz = ec * jkz;
    fj[0] = fma(ea, ijx, -cx);
    fj[1] = fma(ea, ijy, -cy);
    fj[2] = fma(ea, ijz, -cz);
    fk[0] = fma(eb, ikx, cx);
    fk[1] = fma(eb, iky, cy);
    fk[2] = fma(eb, ikz, cz);
}

// Phase 1.  The m(m-1)/2 slot pairs by rotation rounds: round d = 1 .. m/2
// pairs slot s with (s + d) mod m (for even m the last round only s < m/2),
// so every unordered pair appears once.
//   m < 32: one round per step, lane = s: the partner's record is two
//     16-byte shared loads of slot t = (s + d) mod m (the loads of a round
//     are a rotation: conflict-free), f_j accumulates in the lane, f_k goes
//     by shuffle to the lane of t (in a round the targets are a permutation
//     of the lanes).  No accumulator read-modify-write in shared memory.
//     (RB_A3_SHFL_IN=1: the record by shuffle too -- fewer L1 wavefronts,
//     more instructions.)
//   m >= 32: the round-major pair order 32 at a time (lane l of step w holds
//     pair 32 w + l); inside a step all first slots are distinct and all
//     second slots are distinct, so f_j and f_k go to the shared
//     accumulators in two conflict-free sub-steps (dead lanes work on the
//     dummy slot M).
// No atomics; the order is fixed by the enumeration, so the sums are
// deterministic.  m < 32 leaves the slot sums in F (lane = slot), m >= 32
// in the shared accumulators.
template <bool kExactImage, bool kOwned, bool kSlotBad>
__device__ __forceinline__ void a3_windows(const A3Smem &sm, int m, int M, int lane,
                                           const rb_grid &g, const double *__restrict__ pr,
                                           const A3Cut &cut, A3Acc &acc, double F[3]) {
    double fj[3], fk[3];
    RB_CHECK(m >= 0 && m <= M);
    if (m >= 32) {
        const int pairs = m * (m - 1) / 2;
        int s = lane, d = 1;  // pair f0 + lane is (round d, slot s)
        for (int f0 = 0; f0 < pairs; f0 += 32) {
            const bool live = f0 + lane < pairs;
            int t = s + d;
            if (t >= m) t -= m;
            const int ss = live ? s : M, tt = live ? t : M;
            double ijx, ijy, ijz, a, ikx, iky, ikz, b;
            ld_rec(sm, ss, ijx, ijy, ijz, a);
            ld_rec(sm, tt, ikx, iky, ikz, b);
            a3_pair<kExactImage, kOwned, kSlotBad>(sm, live, ss, tt, ijx, ijy, ijz, a, ikx, iky,
                                                   ikz, b, g, pr, cut, acc, fj, fk);
            __syncwarp();
            acc_add(sm, ss, fj[0], fj[1], fj[2]);
            __syncwarp();
            acc_add(sm, tt, fk[0], fk[1], fk[2]);
            s += 32;
            if (s >= m) {
                s -= m;
                d += 1;
            }
        }
        __syncwarp();
        return;
    }
    constexpr unsigned kAll = 0xffffffffu;
    double ijx = 0.0, ijy = 0.0, ijz = 0.0, a = 0.0;
    if (lane < m) ld_rec(sm, lane, ijx, ijy, ijz, a);
    double aj0 = 0.0, aj1 = 0.0, aj2 = 0.0, ak0 = 0.0, ak1 = 0.0, ak2 = 0.0;
    const bool mine = lane < m;
    // partner t = (lane + d) mod m, sender of the k role src = (lane - d) mod m
    int t = lane + 1 >= m ? lane + 1 - m : lane + 1;
    int src = lane - 1 < 0 ? lane - 1 + m : lane - 1;
    if (!mine) t = src = lane;
    const int rounds = m >> 1;
    for (int d = 1; d <= rounds; d++) {
        const bool live = mine && (2 * d != m || lane < d);  // even m: the last round is half
#if RB_A3_SHFL_IN
        const double ikx = __shfl_sync(kAll, ijx, t), iky = __shfl_sync(kAll, ijy, t);
        const double ikz = __shfl_sync(kAll, ijz, t), b = __shfl_sync(kAll, a, t);
#else
        double ikx, iky, ikz, b;  // two 16-byte loads (conflict-free: t is a rotation)
        ld_rec(sm, t, ikx, iky, ikz, b);
#endif
        a3_pair<kExactImage, kOwned, kSlotBad>(sm, live, lane, t, ijx, ijy, ijz, a, ikx, iky, ikz,
                                               b, g, pr, cut, acc, fj, fk);
        aj0 += fj[0];
        aj1 += fj[1];
        aj2 += fj[2];
        ak0 += __shfl_sync(kAll, fk[0], src);  // zero from a rejected or dead pair
        ak1 += __shfl_sync(kAll, fk[1], src);
        ak2 += __shfl_sync(kAll, fk[2], src);
        if (mine) {
            t = t + 1 >= m ? t + 1 - m : t + 1;
            src = src - 1 < 0 ? src - 1 + m : src - 1;
        }
    }
    F[0] = aj0 + ak0;
    F[1] = aj1 + ak1;
    F[2] = aj2 + ak2;
}

}  // namespace rb
