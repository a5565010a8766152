// atm_rot.cuh -- register-resident slot-pair rounds of the Newton-3 ATM pass
// for S+(i) of up to 64 slots (boxes of at least four cutoffs: the hot
// 64-slot instance of k_atm3, undecomposed and -- with kE, the per-slot
// energy sums behind the owned shares -- decomposed runs).
//
// Every slot's force sum lives in registers of the lane that holds the slot
// (lane l holds slot l, and slot 32 + l when m > 32), so the pair loop moves
// no accumulator through shared memory.  The sum is kept as one scalar and one
// vector, F_y = D_y * sum(E_y + E_c) - sum(E_c * D_partner) (rot_eval /
// kRotSum below), which takes a pair from 58 to 43 FP64 instructions -- the
// loop is bound by the FP64 pipe.  The m(m-1)/2 slot pairs are taken in
// three kinds of rounds, each conflict-free and deterministic:
//
//   rotation rounds over a group of g <= 32 slots (lane = slot): round d
//     pairs slot s with (s + d) mod g, d = 1 .. g/2 (the last round of an
//     even g only s < g/2); the j role stays in the lane, the k role is pulled (as two
//     scalars) by the lane of its target (in a round the targets are a
//     permutation of the lanes).
//   cross rounds A x B (m > 32: A = slots 0..31 on all 32 lanes, B = slots
//     32..m-1, mB = m - 32 of them): round e pairs lane l's A slot with B slot
//     (l + e) mod mB, so all 32 lanes work in every round.  f_j stays in the
//     lane; f_k joins a systolic stream: the stream at lane l in round e is
//     the partial sum of B slot (l + e) mod mB, it moves one lane down per
//     round (lane 31 starts a new one) and lane 0 retires its stream (slot e)
//     into shared memory.  Streams still in flight after the last round are
//     summed per slot in lane order.
//
// The ATM kernel (potentials.py:82-114, atm_core.cuh atm_scalars) runs for
// every pair of a round and a rejected pair's scale is selected to zero (no
// divergence).  r_jk^2 <= rc^2 is decided on the fp64 estimate from
// D_k - D_j outside a 1e-10 band around rc^2; a pair inside the band (or
// under the guard distance) raises a per-lane flag and is found again and settled
// after the loop with the reference's raw-position arithmetic (the fix-up
// rounds, rarely entered), so the loop itself never branches.  A base with a
// slot under the guard distance is not taken here (k_atm3 lists it for the
// second launch, which runs the window loop of atm_core.cuh).
//
// The rounds of every group run through ONE inlined copy of the loop (and of
// each fix-up): the kernel's instruction footprint stays small (a warp in
// phase 0, one in the rotation loop and one in the cross loop share the SM's
// instruction cache).
//
// kE (decomposed runs): every pair also yields its energy E_t; a lane sums
// the energies of its slot's triplets (j role in the lane, k role by the same
// shuffle / stream as f_k) and of the pairs it evaluated (the base's sum), so
// k_atm3 weights them by owned shares, (o_i sum_t E_t + sum_s o_s E_s) / 3.
#pragma once

#include "atm_core.cuh"

namespace rb {

// 32-bit shared-memory address of a generic pointer into shared memory
__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void lds_rec(unsigned xy, unsigned zr, double &x, double &y,
                                        double &z, double &w) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(xy));
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(z), "=d"(w) : "r"(zr));
}

// Acceptance on the high word of c = r_jk^2 (A3Cut): in = min_hi < ch <
// lo_hi; undecided (band or guard) = !in && ch <= hi_hi.
struct RotCut {
    int base;       // min_hi + 1
    unsigned span;  // lo_hi - min_hi - 1
    int hi_hi;
};
__device__ __forceinline__ RotCut rot_cut(const A3Cut &cut) {
    RotCut r;
    r.base = cut.min_hi + 1;
    r.span = (unsigned)(cut.lo_hi - cut.min_hi - 1);
    r.hi_hi = cut.hi_hi;
    return r;
}

// The reference's acceptance and guard for slots s, t (raw positions)
__device__ __forceinline__ bool rot_exact_in(const A3Smem &sm, int s, int t, const rb_grid &g,
                                          const double *__restrict__ pr, const A3Cut &cut,
                                          bool &bad) {
    const Image im = make_image(g);
    const int j = sm.q[s], k = sm.q[t];
    double ex, ey, ez;
    exact_disp(im, pr[3 * j], pr[3 * j + 1], pr[3 * j + 2], pr[3 * k], pr[3 * k + 1],
               pr[3 * k + 2], ex, ey, ez);
    const double ce = exact_r2(ex, ey, ez);
    const bool in = ce <= cut.rc2;
    bad = in && ce < RB_MIN_DISTANCE_SQ;
    return in;
}

// FP64 constants of the pair loop that cannot ride as instruction immediates
// (a DFMA takes one): read from the constant bank as operands, so the loop
// does not rebuild them in registers every round.
static __constant__ double kRot38 = 0.375, kRot5 = 5.0;

// rsqrt_nr (common.cuh) with 3/8 from the constant bank
__device__ __forceinline__ double rot_rsqrt(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double r = fma(-x * y, y, 1.0);
    return fma(y * r, fma(kRot38, r, 0.5), y);
}

// The ATM scalars of one slot pair from the dot product g = D_j . D_k
// (D_j, D_k the slots' displacements from the base, a = r_ij^2, b = r_ik^2,
// c = r_jk^2 = a + b - 2 g).  In atm_scalars' notation u = 2 g, v = 2 (a - g),
// w = 2 (b - g), so with q = g (a - g)(b - g) = p / 8 and k = 1 + 5 q / s:
//   E_a = 3/2 s^-5/2 [a (b - g) - g (a - g) - k b c]
//   E_b = 3/2 s^-5/2 [b (a - g) - g (b - g) - k a c]
//   E_c = 3/2 s^-5/2 [c g - (a - g)(b - g) - k a b]
//   E   = s^-5/2 (s + 3 q)
// (the same polynomials, potentials.py:82-114, regrouped: 29 FP64
// instructions instead of 35 and no r_jk vector).  Returns the brackets
// e_a + e_c, e_b + e_c, e_c (units of 3/2 s^-5/2) and s52 = s^-5/2, zero
// unless `in`: the rounds below fold s52 into their accumulation.
template <bool kE>
__device__ __forceinline__ void rot_eval(bool in, double g, double a, double b, double c,
                                         double &eac, double &ebc, double &ec, double &s52,
                                         double &e) {
    // (two nearly coincident slots: the estimate c = a + b - 2 g can round to
    // zero or below and 0 * NaN reaches the sums -- of a pass that raises: the
    // pair is undecided, the reference arithmetic finds it under the guard,
    // and RB_KIND_TRIPLET_MIN_SEPARATION orders before RB_KIND_NONFINITE in
    // the status word.  A select on c here cost 1 % of the pass.
    // test_minimum_separation_between_slots_raises)
    const double ab = a * b;
    const double sp = ab * c;
    const double rs = rot_rsqrt(sp);
    const double inv_s = rs * rs;
    s52 = (rs * inv_s) * inv_s;
    s52 = in ? s52 : 0.0;
    const double va = a - g, wb = b - g;
    const double gva = g * va, gwb = g * wb, vawb = va * wb;
    const double q = gva * wb;
    const double k = fma(q * inv_s, kRot5, 1.0);
    const double ea = fma(-k, b * c, fma(a, wb, -gva));
    const double eb = fma(-k, a * c, fma(b, va, -gwb));
    ec = fma(-k, ab, fma(c, g, -vawb));
    eac = ea + ec;
    ebc = eb + ec;
    if (kE) e = s52 * fma(3.0, q, sp);  // the triplet's energy (units of nu), 0 if rejected
}

// A slot's force sum in the rounds (units of 3 nu): with f_j = E_a D_j -
// E_c (D_k - D_j) = (E_a + E_c) D_j - E_c D_k and f_k = (E_b + E_c) D_k -
// E_c D_j, slot y's sum is D_y * S[0] - (S[1], S[2], S[3]): S[0] the sum of
// (E_y + E_c) over the slot's pairs, S[1..3] the sum of E_c * (the partner's
// D).  A pair costs the j role 1 + 3 and the k role 1 + 3 FP64 instructions
// (instead of 3 + 3 + 3 for the two force vectors and 3 + 3 to add them), and
// the k role travels as two scalars.  S[4]: the slot's energy sum (kE).
constexpr int kRotSum = 5;

// One pair of the fast loop: `live` lanes accept on the fp64 estimate of
// c = a + b - 2 g (a few ulp of a + b from the raw-position value: far inside
// the 1e-10 band); undecided pairs contribute nothing here and set `und`
// (whether or not the lane is live: the fix-ups test rot_undecided again).
template <bool kE>
__device__ __forceinline__ void rot_fast(bool live, double sx, double sy, double sz, double a,
                                         double tx, double ty, double tz, double b,
                                         const RotCut &rc, A3Acc &acc, bool &und, double &eac,
                                         double &ebc, double &ec, double &s52, double &e) {
    const double g = fma(sz, tz, fma(sy, ty, sx * tx));
    const double c = fma(-2.0, g, a + b);
    const int ch = __double2hiint(c);
    const bool inr = (unsigned)(ch - rc.base) < rc.span;
    und = !inr && ch <= rc.hi_hi;
    const bool in = live && inr;
    acc.n += in ? 1 : 0;
    rot_eval<kE>(in, g, a, b, c, eac, ebc, ec, s52, e);
}

// rot_fast's verdict on a pair again (the same arithmetic, for the fix-ups)
__device__ __forceinline__ bool rot_undecided(double sx, double sy, double sz, double a, double tx,
                                              double ty, double tz, double b, const RotCut &rc) {
    const double g = fma(sz, tz, fma(sy, ty, sx * tx));
    const double c = fma(-2.0, g, a + b);
    const int ch = __double2hiint(c);
    return !((unsigned)(ch - rc.base) < rc.span) && ch <= rc.hi_hi;
}

// The fix-up pair: `live` lanes decide with the reference arithmetic.
template <bool kE>
__device__ __forceinline__ void rot_slow(const A3Smem &sm, bool live, int s, int t, double sx,
                                         double sy, double sz, double a, double tx, double ty,
                                         double tz, double b, const rb_grid &g,
                                         const double *__restrict__ pr, const A3Cut &cut,
                                         A3Acc &acc, double &eac, double &ebc, double &ec,
                                         double &s52, double &e) {
    const double dot = fma(sz, tz, fma(sy, ty, sx * tx));
    const double c = fma(-2.0, dot, a + b);
    bool bad = false;
    bool in = live && rot_exact_in(sm, s, t, g, pr, cut, bad);
    acc.bad = acc.bad || bad;
    in = in && !bad;
    acc.n += in ? 1 : 0;
    rot_eval<kE>(in, dot, a, b, c, eac, ebc, ec, s52, e);
}

// position of a slot record (the z half of the second 16-byte row)
__device__ __forceinline__ void lds_pos(unsigned xy, unsigned zr, double &x, double &y,
                                        double &z) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(xy));
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(z) : "r"(zr));
}

// Rotation rounds over slots [off, off + gm) on lanes 0 .. gm-1 (2 <= gm <=
// 32); lanes >= gm mirror lane (lane mod gm) and contribute nothing.  Adds
// each slot's sums to S of its lane (kRotSum above).  The k role of round d
// comes from the lane of slot (s - d) mod gm as two scalars; that slot's
// displacement is a second conflict-free shared load.
template <bool kE>
__device__ __forceinline__ void rot_rounds(const A3Smem &sm, int off, int gm, int lane,
                                           const rb_grid &g, const double *__restrict__ pr,
                                           const A3Cut &cut, A3Acc &acc, double S[kRotSum]) {
    constexpr unsigned kAll = 0xffffffffu;
    const bool mine = lane < gm;
    const int s = mine ? lane : lane % gm;
    const unsigned xy0 = smem_u32(sm.xy + off), zr0 = smem_u32(sm.zr + off);
    double sx, sy, sz, a;
    lds_rec(xy0 + 16 * s, zr0 + 16 * s, sx, sy, sz, a);
    const RotCut rc = rot_cut(cut);
    const unsigned zro = zr0 - xy0;  // (a constant of the instance)
    const unsigned end = xy0 + 16u * (unsigned)gm;
    // partner t = (s + d) mod gm and sender of the k role src = (s - d) mod
    // gm, as shared-memory addresses of their records
    unsigned tp = xy0 + 16u * (unsigned)(s + 1 >= gm ? s + 1 - gm : s + 1);
    int src = s - 1 < 0 ? s - 1 + gm : s - 1;
    unsigned up = xy0 + 16u * (unsigned)src;
    const int rounds = gm >> 1;
    // the lane's last live round: gm/2 (even gm: only s < gm/2 start a pair
    // in the last round), none for a mirror lane
    const int lim = !mine ? 0 : ((gm & 1) || lane < rounds ? rounds : rounds - 1);
    bool und = false;  // some round of this lane is undecided
#pragma unroll 1
    for (int d = 1; d <= rounds; d++) {
        RB_CHECK(tp >= xy0 && tp < end && up == xy0 + 16u * (unsigned)src && src >= 0 &&
                 src < gm && off + gm <= 64);
        double tx, ty, tz, b, ux, uy, uz;
        lds_rec(tp, tp + zro, tx, ty, tz, b);  // conflict-free: a rotation
        lds_pos(up, up + zro, ux, uy, uz);
        bool u;
        double eac, ebc, ec, s52, e = 0.0;
        rot_fast<kE>(d <= lim, sx, sy, sz, a, tx, ty, tz, b, rc, acc, u, eac, ebc, ec, s52, e);
        und = und || u;
        const double ecs = s52 * ec, ebs = s52 * ebc;  // zero from a rejected pair
        S[0] = fma(s52, eac, S[0]);
        S[1] = fma(ecs, tx, S[1]);
        S[2] = fma(ecs, ty, S[2]);
        S[3] = fma(ecs, tz, S[3]);
        const double rb = __shfl_sync(kAll, ebs, src), rc_ = __shfl_sync(kAll, ecs, src);
        S[0] += rb;
        S[1] = fma(rc_, ux, S[1]);
        S[2] = fma(rc_, uy, S[2]);
        S[3] = fma(rc_, uz, S[3]);
        if (kE) {  // the slot energy sums of both members, the base's sum
            acc.e += e;
            S[4] += e;
            S[4] += __shfl_sync(kAll, e, src);
        }
        tp += 16u;
        tp = tp == end ? xy0 : tp;
        up = up == xy0 ? end : up;
        up -= 16u;
        src = (int)((up - xy0) >> 4);
    }
    if (__any_sync(kAll, und)) {  // fix-up rounds (rare)
#pragma unroll 1
        for (int d = 1; d <= rounds; d++) {
            const int t = (s + d) % gm;
            const int sr = (s - d + gm) % gm;
            double tx, ty, tz, b, ux, uy, uz;
            lds_rec(xy0 + 16 * t, zr0 + 16 * t, tx, ty, tz, b);
            const bool mysus = d <= lim && rot_undecided(sx, sy, sz, a, tx, ty, tz, b, rc);
            if (!__any_sync(kAll, mysus)) continue;
            lds_pos(xy0 + 16 * sr, zr0 + 16 * sr, ux, uy, uz);
            double eac, ebc, ec, s52, e = 0.0;
            rot_slow<kE>(sm, mysus, off + s, off + t, sx, sy, sz, a, tx, ty, tz, b, g, pr, cut,
                         acc, eac, ebc, ec, s52, e);
            const double ecs = s52 * ec, ebs = s52 * ebc;
            S[0] = fma(s52, eac, S[0]);
            S[1] = fma(ecs, tx, S[1]);
            S[2] = fma(ecs, ty, S[2]);
            S[3] = fma(ecs, tz, S[3]);
            const double rb = __shfl_sync(kAll, ebs, sr), rc_ = __shfl_sync(kAll, ecs, sr);
            S[0] += rb;
            S[1] = fma(rc_, ux, S[1]);
            S[2] = fma(rc_, uy, S[2]);
            S[3] = fma(rc_, uz, S[3]);
            if (kE) {
                acc.e += e;
                S[4] += e;
                S[4] += __shfl_sync(kAll, e, sr);
            }
        }
    }
}

// Cross rounds A x B (m > 32): adds the A sums to S (lane = A slot) and
// leaves the B sums (lane = B slot, lanes < mb) in G.  A stream carries a B
// slot's five sums (the lane's own D_j is the partner of its k role).
template <bool kE>
__device__ __forceinline__ void rot_cross(const A3Smem &sm, int m, int lane, const rb_grid &g,
                                          const double *__restrict__ pr, const A3Cut &cut,
                                          A3Acc &acc, double S[kRotSum], double G[kRotSum]) {
    constexpr unsigned kAll = 0xffffffffu;
    const int mb = m - 32;
    const unsigned xy0 = smem_u32(sm.xy), zr0 = smem_u32(sm.zr);
    double sx, sy, sz, a;
    lds_rec(xy0 + 16 * lane, zr0 + 16 * lane, sx, sy, sz, a);
    const RotCut rc = rot_cut(cut);
    double R[kRotSum] = {0.0, 0.0, 0.0, 0.0, 0.0};
    const unsigned bbeg = 16u * 32u, bend = 16u * (unsigned)m;
    unsigned boff = bbeg + 16u * (unsigned)(lane % mb);  // B slot (lane + e) mod mb
    bool und = false;
    const unsigned ret0 = smem_u32(sm.axy + 32), retz0 = smem_u32(sm.az + 32),
                   retw0 = smem_u32(sm.aw + 32);
#pragma unroll 1
    for (int e = 0; e < mb; e++) {
        RB_CHECK(boff >= bbeg && boff < bend && mb <= 32 && m <= 64);
        double tx, ty, tz, b;
        lds_rec(xy0 + boff, zr0 + boff, tx, ty, tz, b);
        bool u;
        double eac, ebc, ec, s52, en = 0.0;
        rot_fast<kE>(true, sx, sy, sz, a, tx, ty, tz, b, rc, acc, u, eac, ebc, ec, s52, en);
        und = und || u;
        const double ecs = s52 * ec;
        S[0] = fma(s52, eac, S[0]);
        S[1] = fma(ecs, tx, S[1]);
        S[2] = fma(ecs, ty, S[2]);
        S[3] = fma(ecs, tz, S[3]);
        R[0] = fma(s52, ebc, R[0]);
        R[1] = fma(ecs, sx, R[1]);
        R[2] = fma(ecs, sy, R[2]);
        R[3] = fma(ecs, sz, R[3]);
        if (kE) {
            acc.e += en;
            S[4] += en;
            R[4] += en;
        }
        if (lane == 0) {  // the stream of B slot e leaves the warp
            asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(ret0 + 16u * e), "d"(R[1]),
                         "d"(R[2]));
            asm volatile("st.shared.f64 [%0], %1;" ::"r"(retz0 + 8u * e), "d"(R[3]));
            asm volatile("st.shared.f64 [%0], %1;" ::"r"(retw0 + 8u * e), "d"(R[0]));
            if (kE) sm.ae[32 + e] = R[4];
        }
        // every stream moves one lane down; lane 31 starts the next one
        R[0] = __shfl_down_sync(kAll, R[0], 1);
        R[1] = __shfl_down_sync(kAll, R[1], 1);
        R[2] = __shfl_down_sync(kAll, R[2], 1);
        R[3] = __shfl_down_sync(kAll, R[3], 1);
        if (kE) R[4] = __shfl_down_sync(kAll, R[4], 1);
        if (lane == 31) R[0] = R[1] = R[2] = R[3] = R[4] = 0.0;
        boff += 16u;
        boff = boff == bend ? bbeg : boff;
    }
    __syncwarp();
    // streams still in flight: lane l (0..30) holds B slot (l + mb) mod mb
    // = l mod mb (after the last shift)
    sm.axy[lane] = make_double2(R[1], R[2]);
    sm.az[lane] = R[3];
    sm.aw[lane] = R[0];
    if (kE) sm.ae[lane] = R[4];
    if (__any_sync(kAll, und)) {  // fix-up (rare): lane by lane, in order
#pragma unroll 1
        for (int e = 0; e < mb; e++) {
            bool mine_und;
            {
                const int bslot = 32 + (lane + e) % mb;
                double tx, ty, tz, b;
                lds_rec(xy0 + 16 * bslot, zr0 + 16 * bslot, tx, ty, tz, b);
                mine_und = rot_undecided(sx, sy, sz, a, tx, ty, tz, b, rc);
            }
            unsigned who = __ballot_sync(kAll, mine_und);
            while (who) {
                const int L = __ffs(who) - 1;
                who &= who - 1;
                if (lane == L) {
                    const int bslot = 32 + (lane + e) % mb;
                    double tx, ty, tz, b;
                    lds_rec(xy0 + 16 * bslot, zr0 + 16 * bslot, tx, ty, tz, b);
                    double eac, ebc, ec, s52, en = 0.0;
                    rot_slow<kE>(sm, true, lane, bslot, sx, sy, sz, a, tx, ty, tz, b, g, pr, cut,
                                 acc, eac, ebc, ec, s52, en);
                    const double ecs = s52 * ec;
                    S[0] = fma(s52, eac, S[0]);
                    S[1] = fma(ecs, tx, S[1]);
                    S[2] = fma(ecs, ty, S[2]);
                    S[3] = fma(ecs, tz, S[3]);
                    acc_add(sm, bslot, ecs * sx, ecs * sy, ecs * sz);
                    sm.aw[bslot] += s52 * ebc;
                    if (kE) {
                        acc.e += en;
                        S[4] += en;
                        sm.ae[bslot] += en;
                    }
                }
                __syncwarp();
            }
        }
    }
    __syncwarp();
    G[0] = G[1] = G[2] = G[3] = G[4] = 0.0;
    if (lane < mb) {
        const double2 r = sm.axy[32 + lane];
        G[0] = sm.aw[32 + lane];
        G[1] = r.x;
        G[2] = r.y;
        G[3] = sm.az[32 + lane];
        if (kE) G[4] = sm.ae[32 + lane];
        for (int l = lane; l < 31; l += mb) {  // in lane order
            const double2 q = sm.axy[l];
            G[0] += sm.aw[l];
            G[1] += q.x;
            G[2] += q.y;
            G[3] += sm.az[l];
            if (kE) G[4] += sm.ae[l];
        }
    }
    __syncwarp();
}

// slot `sl`'s force sum (units of 2 nu) from its round sums: 3/2 (D S[0] -
// (S[1], S[2], S[3])), into the shared accumulators phase 3 reads
template <bool kE>
__device__ __forceinline__ void rot_store(const A3Smem &sm, int sl, const double S[kRotSum]) {
    double dx, dy, dz, r2;
    ld_rec(sm, sl, dx, dy, dz, r2);
    sm.axy[sl] = make_double2(1.5 * fma(dx, S[0], -S[1]), 1.5 * fma(dy, S[0], -S[2]));
    sm.az[sl] = 1.5 * fma(dz, S[0], -S[3]);
    if (kE) sm.ae[sl] = S[4];
}

// Phase 1 for m <= 64 slots: the slot sums (units of 2 nu) end in the shared
// accumulators sm.axy / sm.az (phase 3 reads them).
template <bool kE>
__device__ __forceinline__ void a3_rot(const A3Smem &sm, int m, int lane, const rb_grid &g,
                                       const double *__restrict__ pr, const A3Cut &cut,
                                       A3Acc &acc) {
    double S[kRotSum] = {0.0, 0.0, 0.0, 0.0, 0.0};
    int off = 0, gm = m < 32 ? m : 32;
    // group A (or all of a short S+), then the cross rounds, then group B
    // through the same loop
#pragma unroll 1
    for (int grp = 0;; grp++) {
        if (gm >= 2) rot_rounds<kE>(sm, off, gm, lane, g, pr, cut, acc, S);
        if (grp == 1 || m <= 32) break;
        double G[kRotSum];
        rot_cross<kE>(sm, m, lane, g, pr, cut, acc, S, G);
        rot_store<kE>(sm, lane, S);  // the A sums are complete
#pragma unroll
        for (int c = 0; c < kRotSum; c++) S[c] = G[c];
        off = 32;
        gm = m - 32;
    }
    if (lane < gm) rot_store<kE>(sm, off + lane, S);  // (a group may have fewer than 32 slots)
    __syncwarp();
}

}  // namespace rb
