// atm_rot.cuh -- register-resident slot-pair rounds of the Newton-3 ATM pass
// for S+(i) of up to 64 slots (boxes of at least four cutoffs: the hot
// 64-slot instance of k_atm3, undecomposed and -- with kE, the per-slot
// energy sums behind the owned shares -- decomposed runs).
//
// Every slot's force sum lives in a register of the lane that holds the slot
// (lane l holds slot l, and slot 32 + l when m > 32), so the pair loop moves
// no accumulator through shared memory.  The m(m-1)/2 slot pairs are taken in
// three kinds of rounds, each conflict-free and deterministic:
//
//   rotation rounds over a group of g <= 32 slots (lane = slot): round d
//     pairs slot s with (s + d) mod g, d = 1 .. g/2 (the last round of an
//     even g only s < g/2); f_j stays in the lane, f_k is pulled by the lane
//     of its target (in a round the targets are a permutation of the lanes).
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
// under the guard distance) is recorded in a per-lane bit mask and settled
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

// f_j, f_k (units of 2 nu) of the pair with D_j = (sx, sy, sz), a = r_ij^2,
// D_k = (tx, ty, tz), b = r_ik^2, scaled to zero unless `in`.
template <bool kE>
__device__ __forceinline__ void rot_eval(bool in, double sx, double sy, double sz, double a,
                                         double tx, double ty, double tz, double b, double jkx,
                                         double jky, double jkz, double c, double fj[3],
                                         double fk[3], double &e) {
    // atm_scalars with the common factor s^-5/2 selected (every E_x is a
    // multiple of it)
    const double tsum = a + b + c;
    const double u = fma(-2.0, c, tsum);
    const double v = fma(-2.0, b, tsum);
    const double w = fma(-2.0, a, tsum);
    const double uv = u * v, uw = u * w, vw = v * w;
    const double p = uv * w;
    const double sp = a * b * c;
    const double rs = rsqrt_nr(sp);
    const double inv_s = rs * rs;
    double s52 = rs * inv_s * inv_s;
    s52 = in ? s52 : 0.0;
    const double S = uv + uw + vw;
    const double A = 0.375 * s52;
    const double K = s52 * fma(0.9375 * p, inv_s, 1.5);
    const double ea = fma(A, fma(-2.0, uv, S), -K * (b * c));
    const double eb = fma(A, fma(-2.0, uw, S), -K * (a * c));
    const double ec = fma(A, fma(-2.0, vw, S), -K * (a * b));
    const double cx = ec * jkx, cy = ec * jky, cz = ec * jkz;
    fj[0] = fma(ea, sx, -cx);
    fj[1] = fma(ea, sy, -cy);
    fj[2] = fma(ea, sz, -cz);
    fk[0] = fma(eb, tx, cx);
    fk[1] = fma(eb, ty, cy);
    fk[2] = fma(eb, tz, cz);
    if (kE) e = s52 * fma(0.375, p, sp);  // the triplet's energy (units of nu), 0 if rejected
}

// One pair of the fast loop: `live` lanes accept on the fp64 estimate;
// undecided pairs contribute nothing here and set `und`.
template <bool kE>
__device__ __forceinline__ void rot_fast(bool live, double sx, double sy, double sz, double a,
                                         double tx, double ty, double tz, double b,
                                         const RotCut &rc, A3Acc &acc, bool &und, double fj[3],
                                         double fk[3], double &e) {
    const double jkx = tx - sx, jky = ty - sy, jkz = tz - sz;
    const double c = fma(jkz, jkz, fma(jky, jky, jkx * jkx));
    const int ch = __double2hiint(c);
    const bool inr = (unsigned)(ch - rc.base) < rc.span;
    und = live && !inr && ch <= rc.hi_hi;
    const bool in = live && inr;
    acc.n += in ? 1 : 0;
    rot_eval<kE>(in, sx, sy, sz, a, tx, ty, tz, b, jkx, jky, jkz, c, fj, fk, e);
}

// The fix-up pair: `live` lanes decide with the reference arithmetic.
template <bool kE>
__device__ __forceinline__ void rot_slow(const A3Smem &sm, bool live, int s, int t, double sx,
                                         double sy, double sz, double a, double tx, double ty,
                                         double tz, double b, const rb_grid &g,
                                         const double *__restrict__ pr, const A3Cut &cut,
                                         A3Acc &acc, double fj[3], double fk[3], double &e) {
    const double jkx = tx - sx, jky = ty - sy, jkz = tz - sz;
    const double c = fma(jkz, jkz, fma(jky, jky, jkx * jkx));
    bool bad = false;
    bool in = live && rot_exact_in(sm, s, t, g, pr, cut, bad);
    acc.bad = acc.bad || bad;
    in = in && !bad;
    acc.n += in ? 1 : 0;
    rot_eval<kE>(in, sx, sy, sz, a, tx, ty, tz, b, jkx, jky, jkz, c, fj, fk, e);
}

// Rotation rounds over slots [off, off + gm) on lanes 0 .. gm-1 (2 <= gm <=
// 32); lanes >= gm mirror lane (lane mod gm) and contribute nothing.  Adds
// each slot's sum to F of its lane.
template <bool kE>
__device__ __forceinline__ void rot_rounds(const A3Smem &sm, int off, int gm, int lane,
                                           const rb_grid &g, const double *__restrict__ pr,
                                           const A3Cut &cut, A3Acc &acc, double F[4]) {
    constexpr unsigned kAll = 0xffffffffu;
    const bool mine = lane < gm;
    const int s = mine ? lane : lane % gm;
    const unsigned xy0 = smem_u32(sm.xy + off), zr0 = smem_u32(sm.zr + off);
    double sx, sy, sz, a;
    lds_rec(xy0 + 16 * s, zr0 + 16 * s, sx, sy, sz, a);
    const RotCut rc = rot_cut(cut);
    const unsigned end = 16u * (unsigned)gm;
    // partner t = (s + d) mod gm as a byte offset, sender of the k role
    // src = (s - d) mod gm
    unsigned toff = 16u * (unsigned)(s + 1 >= gm ? s + 1 - gm : s + 1);
    int src = s - 1 < 0 ? s - 1 + gm : s - 1;
    const int rounds = gm >> 1;
    // the lane's last live round: gm/2 (even gm: only s < gm/2 start a pair
    // in the last round), none for a mirror lane
    const int lim = !mine ? 0 : ((gm & 1) || lane < rounds ? rounds : rounds - 1);
    unsigned und = 0;  // bit d: round d is undecided on this lane
    double fj[3], fk[3];
#pragma unroll 1
    for (int d = 1; d <= rounds; d++) {
        RB_CHECK(toff < end && src >= 0 && src < gm && off + gm <= 64);
        double tx, ty, tz, b;
        lds_rec(xy0 + toff, zr0 + toff, tx, ty, tz, b);  // conflict-free: a rotation
        bool u;
        double e = 0.0;
        rot_fast<kE>(d <= lim, sx, sy, sz, a, tx, ty, tz, b, rc, acc, u, fj, fk, e);
        und |= u ? 1u << d : 0u;
        F[0] += fj[0];
        F[1] += fj[1];
        F[2] += fj[2];
        F[0] += __shfl_sync(kAll, fk[0], src);  // zero from a rejected pair
        F[1] += __shfl_sync(kAll, fk[1], src);
        F[2] += __shfl_sync(kAll, fk[2], src);
        if (kE) {  // the slot energy sums of both members, the base's sum
            acc.e += e;
            F[3] += e;
            F[3] += __shfl_sync(kAll, e, src);
        }
        toff += 16u;
        toff = toff == end ? 0u : toff;
        src = src == 0 ? gm - 1 : src - 1;
    }
    if (__any_sync(kAll, und != 0)) {  // fix-up rounds (rare)
#pragma unroll 1
        for (int d = 1; d <= rounds; d++) {
            const bool mysus = (und >> d) & 1u;
            if (!__any_sync(kAll, mysus)) continue;
            const int t = (s + d) % gm;
            const int sr = (s - d + gm) % gm;
            double tx, ty, tz, b;
            lds_rec(xy0 + 16 * t, zr0 + 16 * t, tx, ty, tz, b);
            double e = 0.0;
            rot_slow<kE>(sm, mysus, off + s, off + t, sx, sy, sz, a, tx, ty, tz, b, g, pr, cut,
                         acc, fj, fk, e);
            F[0] += fj[0];
            F[1] += fj[1];
            F[2] += fj[2];
            F[0] += __shfl_sync(kAll, fk[0], sr);
            F[1] += __shfl_sync(kAll, fk[1], sr);
            F[2] += __shfl_sync(kAll, fk[2], sr);
            if (kE) {
                acc.e += e;
                F[3] += e;
                F[3] += __shfl_sync(kAll, e, sr);
            }
        }
    }
}

// Cross rounds A x B (m > 32): adds the A sums to F (lane = A slot) and
// leaves the B sums (lane = B slot, lanes < mb) in G.
template <bool kE>
__device__ __forceinline__ void rot_cross(const A3Smem &sm, int m, int lane, const rb_grid &g,
                                          const double *__restrict__ pr, const A3Cut &cut,
                                          A3Acc &acc, double F[4], double G[4]) {
    constexpr unsigned kAll = 0xffffffffu;
    const int mb = m - 32;
    const unsigned xy0 = smem_u32(sm.xy), zr0 = smem_u32(sm.zr);
    double sx, sy, sz, a;
    lds_rec(xy0 + 16 * lane, zr0 + 16 * lane, sx, sy, sz, a);
    const RotCut rc = rot_cut(cut);
    double R[4] = {0.0, 0.0, 0.0, 0.0};
    double fj[3], fk[3];
    const unsigned bbeg = 16u * 32u, bend = 16u * (unsigned)m;
    unsigned boff = bbeg + 16u * (unsigned)(lane % mb);  // B slot (lane + e) mod mb
    unsigned und = 0;
    const unsigned ret0 = smem_u32(sm.axy + 32), retz0 = smem_u32(sm.az + 32);
#pragma unroll 1
    for (int e = 0; e < mb; e++) {
        RB_CHECK(boff >= bbeg && boff < bend && mb <= 32 && m <= 64);
        double tx, ty, tz, b;
        lds_rec(xy0 + boff, zr0 + boff, tx, ty, tz, b);
        bool u;
        double en = 0.0;
        rot_fast<kE>(true, sx, sy, sz, a, tx, ty, tz, b, rc, acc, u, fj, fk, en);
        und |= u ? 1u << e : 0u;
        F[0] += fj[0];
        F[1] += fj[1];
        F[2] += fj[2];
        R[0] += fk[0];
        R[1] += fk[1];
        R[2] += fk[2];
        if (kE) {
            acc.e += en;
            F[3] += en;
            R[3] += en;
        }
        if (lane == 0) {  // the stream of B slot e leaves the warp
            asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(ret0 + 16u * e), "d"(R[0]),
                         "d"(R[1]));
            asm volatile("st.shared.f64 [%0], %1;" ::"r"(retz0 + 8u * e), "d"(R[2]));
            if (kE) sm.ae[32 + e] = R[3];
        }
        // every stream moves one lane down; lane 31 starts the next one
        R[0] = __shfl_down_sync(kAll, R[0], 1);
        R[1] = __shfl_down_sync(kAll, R[1], 1);
        R[2] = __shfl_down_sync(kAll, R[2], 1);
        if (kE) R[3] = __shfl_down_sync(kAll, R[3], 1);
        if (lane == 31) R[0] = R[1] = R[2] = R[3] = 0.0;
        boff += 16u;
        boff = boff == bend ? bbeg : boff;
    }
    __syncwarp();
    // streams still in flight: lane l (0..30) holds B slot (l + mb) mod mb
    // = l mod mb (after the last shift)
    sm.axy[lane] = make_double2(R[0], R[1]);
    sm.az[lane] = R[2];
    if (kE) sm.ae[lane] = R[3];
    if (__any_sync(kAll, und != 0)) {  // fix-up (rare): lane by lane, in order
#pragma unroll 1
        for (int e = 0; e < mb; e++) {
            unsigned who = __ballot_sync(kAll, (und >> e) & 1u);
            while (who) {
                const int L = __ffs(who) - 1;
                who &= who - 1;
                if (lane == L) {
                    const int bslot = 32 + (lane + e) % mb;
                    double tx, ty, tz, b;
                    lds_rec(xy0 + 16 * bslot, zr0 + 16 * bslot, tx, ty, tz, b);
                    double en = 0.0;
                    rot_slow<kE>(sm, true, lane, bslot, sx, sy, sz, a, tx, ty, tz, b, g, pr, cut,
                                 acc, fj, fk, en);
                    F[0] += fj[0];
                    F[1] += fj[1];
                    F[2] += fj[2];
                    acc_add(sm, bslot, fk[0], fk[1], fk[2]);
                    if (kE) {
                        acc.e += en;
                        F[3] += en;
                        sm.ae[bslot] += en;
                    }
                }
                __syncwarp();
            }
        }
    }
    __syncwarp();
    G[0] = G[1] = G[2] = G[3] = 0.0;
    if (lane < mb) {
        const double2 r = sm.axy[32 + lane];
        G[0] = r.x;
        G[1] = r.y;
        G[2] = sm.az[32 + lane];
        if (kE) G[3] = sm.ae[32 + lane];
        for (int l = lane; l < 31; l += mb) {  // in lane order
            const double2 q = sm.axy[l];
            G[0] += q.x;
            G[1] += q.y;
            G[2] += sm.az[l];
            if (kE) G[3] += sm.ae[l];
        }
    }
    __syncwarp();
}

// Phase 1 for m <= 64 slots: the slot sums (units of 2 nu) end in the shared
// accumulators sm.axy / sm.az (phase 3 reads them).
template <bool kE>
__device__ __forceinline__ void a3_rot(const A3Smem &sm, int m, int lane, const rb_grid &g,
                                       const double *__restrict__ pr, const A3Cut &cut,
                                       A3Acc &acc) {
    double F[4] = {0.0, 0.0, 0.0, 0.0};
    int off = 0, gm = m < 32 ? m : 32;
    // group A (or all of a short S+), then the cross rounds, then group B
    // through the same loop
#pragma unroll 1
    for (int grp = 0;; grp++) {
        if (gm >= 2) rot_rounds<kE>(sm, off, gm, lane, g, pr, cut, acc, F);
        if (grp == 1 || m <= 32) break;
        double G[4];
        rot_cross<kE>(sm, m, lane, g, pr, cut, acc, F, G);
        sm.axy[lane] = make_double2(F[0], F[1]);  // the A sums are complete
        sm.az[lane] = F[2];
        if (kE) sm.ae[lane] = F[3];
        F[0] = G[0];
        F[1] = G[1];
        F[2] = G[2];
        F[3] = G[3];
        off = 32;
        gm = m - 32;
    }
    if (lane < gm) {  // (a group may have fewer than 32 slots)
        sm.axy[off + lane] = make_double2(F[0], F[1]);
        sm.az[off + lane] = F[2];
        if (kE) sm.ae[off + lane] = F[3];
    }
    __syncwarp();
}

}  // namespace rb
