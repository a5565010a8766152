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
//   phase 1  the slot pairs by ROUNDS: in round d slot s pairs with slot
//            (s + d) mod m, d = 1 .. m/2, so every unordered pair appears
//            exactly once.  The pairs are taken round-major, 32 per window
//            (one lane each): inside a window all first slots are distinct
//            and all second slots are distinct.  Each lane settles
//            r_jk^2 <= rc^2 bit-exactly (fp64 estimate from d_ik - d_ij
//            outside a 1e-10 band, else -- or when the box is under four
//            cutoffs -- the reference's raw-position arithmetic), evaluates
//            the ATM kernel, keeps f_i in registers and adds f_j, f_k to the
//            slot accumulators in shared memory in two conflict-free
//            sub-steps (no atomics; the order is fixed by the enumeration).
//   phase 3  slot sums go to the TARGET's row, G[j][position of i in row j];
//            the gather kernel sums, for each particle p, its own part and
//            its row segment G[p][k] over the entries q < p -- in row order.
//
// Energies are phi per triplet (the reference's phi/3 per visit, summed), the
// virial -2(E_a a + E_b b + E_c c) per triplet (:530 summed over visits).
#include <cstdlib>
#include <cstring>

#include <algorithm>

#include "atm_core.cuh"
#include "atm_rot.cuh"

#include <type_traits>

namespace rb {

#ifndef RB_A3_WARPS
#define RB_A3_WARPS 4
#endif
constexpr int kA3Warps = RB_A3_WARPS;
// (6 blocks of 4 warps, 80 registers: with the 43-instruction rounds the pass
// is throughput-bound on pipes its warps share, and fewer warps without
// spills win -- 5 / 6 / 7 / 8 blocks per SM: cfg4 5.76 / 5.61 / 5.64 / 5.72 ms,
// cfg2 0.116 / 0.116 / 0.120 / 0.124 ms, cfg3@2.5 0.752 / 0.734 / 0.744 ms / -)
#ifndef RB_A3_MIN_BLOCKS
#define RB_A3_MIN_BLOCKS 6
#endif
constexpr int kA3MinBlocks = RB_A3_MIN_BLOCKS;  // register cap for occupancy
constexpr int kA3MaxSlots = 4096;
// G entries are padded to 4 doubles (32 bytes, sector-aligned): every partial
// force write covers a whole DRAM sector, so the scattered writes need no
// read-modify-write fill (24-byte entries straddle sectors written at
// different times by different bases)
constexpr int kGStride = 4;    // longest S+(i) a warp takes (rows are <= 4096)

// Phase 0: S+(r), the suffix of r's rank-sorted row with rank > r and
// r_ir^2 <= rc^2 (reference arithmetic), into the warp's slots.  Returns m,
// or -1 when S+(r) does not fit `slots` (the base is then listed in `ovf`
// for the full-slot launch, or a capacity error is recorded).  Row entries
// beyond the three-body cutoff get a zero G partial (the gather reads every
// entry of the row prefix).
template <bool kOwned>
__device__ __forceinline__ int a3_slots(int64_t r, const A3Smem &sm, const Image &im,
                                        double xi, double yi, double zi, int rc_n,
                                        int chunk_first, const double *__restrict__ pr,
                                        const int32_t *__restrict__ row,
                                        const int32_t *__restrict__ mir, int32_t capacity,
                                        int32_t slots, double rc2, double *__restrict__ gbuf,
                                        const uint8_t *__restrict__ owned,
                                        unsigned long long *status, int64_t tag, int32_t *ovf,
                                        bool &slot_bad, int32_t *split_out) {
    const int lane = threadIdx.x & 31;
    int m = 0;
    int below = 0;  // row entries of rank < r from `first` on (the prefix ends inside them)
    slot_bad = false;
    // (warp-uniform: a base a cutoff away from the periodic faces needs no
    // minimum image, common.cuh image_free)
    const bool image = !image_free(im, xi, yi, zi, sqrt(rc2));
    int first = 0;
    {
        const int nchunks = (rc_n + 31) >> 5;
        const unsigned b = __ballot_sync(0xffffffffu, lane < nchunks && chunk_first < r);
        first = b ? 32 * (__popc(b) - 1) : 0;
        if (nchunks > 32) first = 0;  // longer rows than one ballot covers: scan all
    }
    // two chunks per iteration: both rows' (and mirror) loads, then both
    // positions' loads are in flight together
    for (int base = first; base < rc_n; base += 64) {
        int q2[2], mk2[2];
        double px[2], py[2], pz[2];
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int k = base + 32 * h + lane;
            q2[h] = k < rc_n ? row[k] : -1;
            mk2[h] = k < rc_n ? mir[k] : 0;
        }
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int q = q2[h] > r ? q2[h] : (int)r;  // (own position: a harmless load)
            px[h] = pr[3 * q];
            py[h] = pr[3 * q + 1];
            pz[h] = pr[3 * q + 2];
        }
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int k = base + 32 * h + lane;
            const int q = q2[h];
            bool keep = false;
            double dx = 0.0, dy = 0.0, dz = 0.0, r2 = 0.0;
            if (q > r) {
                exact_disp<false>(im, xi, yi, zi, px[h], py[h], pz[h], dx, dy, dz);
                if (image) {
                    dx = min_image(dx, im.box[0], im.half[0]);
                    dy = min_image(dy, im.box[1], im.half[1]);
                    dz = min_image(dz, im.box[2], im.half[2]);
                }
                r2 = exact_r2(dx, dy, dz);
                keep = r2 <= rc2;
                // beyond the three-body cutoff: contributes nothing.  (A row
                // truncated at its capacity has no mirror entry, -1: that pass
                // is reported as a capacity error and repeated; nothing is
                // written for it.)
                if (!keep && mk2[h] >= 0) {
                    RB_CHECK(mk2[h] < capacity);
                    double2 *gq = (double2 *)(gbuf + ((int64_t)q * capacity + mk2[h]) * kGStride);
                    gq[0] = make_double2(0.0, 0.0);
                    gq[1] = make_double2(0.0, 0.0);
                }
            }
            below += __popc(__ballot_sync(0xffffffffu, k < rc_n && q >= 0 && q < r));
            const unsigned mk = __ballot_sync(0xffffffffu, keep);
            if (m + __popc(mk) > slots) {  // S+(i) does not fit the shared-memory slots
                if (lane == 0) {
                    if (ovf)
                        ovf[2 + atomicAdd(ovf, 1)] = (int32_t)r;
                    else
                        record_status(status, tag, RB_KIND_CAPACITY);
                }
                return -1;
            }
            if (keep) {
                const int slot = m + __popc(mk & lanemask_lt());
                RB_CHECK(slot < slots && k < capacity && mk2[h] < capacity);
                sm.xy[slot] = make_double2(dx, dy);
                sm.zr[slot] = make_double2(dz, r2);
                sm.axy[slot] = make_double2(0.0, 0.0);
                sm.az[slot] = 0.0;
                sm.kidx[slot] = k | ((kOwned ? (int)owned[q] : 1) << 30);
                sm.q[slot] = q;
                sm.mpos[slot] = mk2[h];
            }
            m += __popc(mk);
            slot_bad |= __any_sync(0xffffffffu, keep && r2 < RB_MIN_DISTANCE_SQ);
        }
    }
    // the row prefix of ranks below r: the entries whose bases may write
    // G[r][k] (the gather reads exactly these)
    if (lane == 0 && split_out) *split_out = first + below;
    __syncwarp();
    return m;
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
                                       int32_t slots, const A3Cut &cut,
                                       double *__restrict__ own,
                                       double *__restrict__ gbuf,
                                       double *__restrict__ energy_rank,
                                       double *__restrict__ virial_rank,
                                       int32_t *__restrict__ triplets_rank,
                                       const uint8_t *__restrict__ owned,
                                       unsigned long long *status, int64_t tag, int debug_mode,
                                       int32_t *ovf, int32_t *__restrict__ splits) {
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int32_t *row = rows + r * (int64_t)capacity;
    const int32_t *mir = mirror + r * (int64_t)capacity;
    // phase 0 is latency-bound: the first memory round trip carries the
    // status words, the base's position and row length, and the first entry
    // of every 32-entry chunk of its row (rows are rank-sorted: S+(i) starts
    // in the last chunk whose first entry precedes i)
    const ulonglong2 s01 = ld_status2(status);
    const double xi = pr[3 * r], yi = pr[3 * r + 1], zi = pr[3 * r + 2];
    const int rc_n = row_count[r];
    const int chunk_first = 32 * lane < capacity ? row[32 * lane] : 0x7fffffff;
    const unsigned long long swd = __shfl_sync(0xffffffffu, s01.x, 0);  // one view per warp
    if (tag < 0) tag = status ? (int64_t)__shfl_sync(0xffffffffu, s01.y, 0) : 0;
    if (status && frozen_word(swd, tag, RB_KIND_TRIPLET_MIN_SEPARATION)) return;
    if (kM > 0) slots = kM;
    const A3Smem sm = a3_carve<kM>(smem_raw + (size_t)warp * a3_warp_bytes(slots), slots);
    const Image im = make_image(g);
    // partial forces go to the TARGET's row: G[q][position of i in row q], so
    // the gather of q reads its own row segment contiguously

    // ---- phase 0: S+(i), the row suffix with rank > i within rc
    bool slot_bad = false;
    const int m = a3_slots<kOwned>(r, sm, im, xi, yi, zi, rc_n, chunk_first, pr,
                                   row, mir, capacity, slots, cut.rc2, gbuf, owned, status, tag,
                                   ovf, slot_bad, splits + r);
    if (m < 0) return;
    // the fast instance (standard case, 64 slots) takes only bases without a
    // slot under the guard distance: the others go to the second launch
    constexpr bool kFast = !kExactImage && kM == 64;
    if (kFast && slot_bad) {
        if (lane == 0) ovf[2 + atomicAdd(ovf, 1)] = (int32_t)r;
        return;
    }

    // ---- phase 1: the slot pairs, 32 per window (a3_windows)
    A3Acc acc = {0.0, 0.0, 0, false, kOwned ? (int)owned[r] : 1};
    double F[3] = {0.0, 0.0, 0.0};
    // debug 1: phases 0 and 3 only; 2 / 3: phase 1 of the bases with m < 32 /
    // m >= 32 only (timing split, tuning only)
    const int dm = debug_mode & 15;
    if (dm != 1 && !(dm == 2 && m >= 32) && !(dm == 3 && m < 32)) {
        if constexpr (kFast) {
            // register-resident rounds (atm_rot.cuh); decomposed runs also sum
            // each slot's triplet energies for the owned shares
            a3_rot<kOwned>(sm, m, lane, g, pr, cut, acc);
        } else if (slot_bad) {
            a3_windows<kExactImage, kOwned, true>(sm, m, slots, lane, g, pr, cut, acc, F);
        } else {
            a3_windows<kExactImage, kOwned, false>(sm, m, slots, lane, g, pr, cut, acc, F);
        }
    }

    // ---- phase 3: slot sums -> G[i][row index]; own part, scalars.  Per
    // triplet f_i + f_j + f_k = 0, so the base's own force is minus the sum
    // of everything its triplets gave the slots (fixed lane order and tree)
    // Likewise the virial: per triplet x_i.f_i + x_j.f_j + x_k.f_k =
    // -(d_ij.f_j + d_ik.f_k) = -2(E_a a + E_b b + E_c c), so the base's sum is
    // sum_s d_is . (slot sum s) in the units of acc.w, and the energy is
    // -1/4.5 of it (atm_scalars).  Decomposed runs weight each triplet by its
    // owned share, and under four cutoffs d_jk is its own image: both keep
    // the per-triplet sums.
    double sx = 0.0, sy = 0.0, sz = 0.0, sw = 0.0, so = 0.0;
    for (int sl = lane; sl < m; sl += 32) {
        double ax = F[0], ay = F[1], az = F[2];  // m < 32: the lane's register sums
        if (kFast || m >= 32) {
            const double2 axy = sm.axy[sl];
            ax = axy.x;
            ay = axy.y;
            az = sm.az[sl];
        }
        RB_CHECK(sm.q[sl] >= 0 && sm.q[sl] < n && sm.mpos[sl] < capacity);
        if (sm.mpos[sl] >= 0) {  // (-1: a truncated row, see a3_slots)
            double2 *gq = (double2 *)(gbuf + ((int64_t)sm.q[sl] * capacity + sm.mpos[sl]) * kGStride);
            gq[0] = make_double2(ax, ay);  // one whole 32-byte sector
            gq[1] = make_double2(az, 0.0);
        }
        sx += ax;
        sy += ay;
        sz += az;
        if (!kOwned && !kExactImage) {
            double dx, dy, dz, r2;
            ld_rec(sm, sl, dx, dy, dz, r2);
            sw = fma(dx, ax, fma(dy, ay, fma(dz, az, sw)));
        }
        // owned members' shares of the slot's triplet energies
        if (kFast && kOwned && (sm.kidx[sl] >> 30)) so += sm.ae[sl];
    }
    const double fx = -group_sum<32>(sx);
    const double fy = -group_sum<32>(sy);
    const double fz = -group_sum<32>(sz);
    double w, e;
    if (kFast && kOwned) {
        // share (o_i + o_j + o_k)/3 per triplet: (o_i/3) sum_t E_t + (1/3) sum_s
        // o_s E_s, E_s the energy of slot s's triplets; the virial per
        // triplet is -9/2 E (Euler: E is homogeneous of degree -9/2)
        e = (acc.owned_i * group_sum<32>(acc.e) + group_sum<32>(so)) * (1.0 / 3.0);
        w = -4.5 * e;
    } else {
        w = group_sum<32>(kOwned || kExactImage ? acc.w : sw);
        e = kOwned || kExactImage ? group_sum<32>(acc.e) : w * (-1.0 / 4.5);
    }
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
           int32_t capacity, int32_t slots, A3Cut cut,
           double *__restrict__ own, double *__restrict__ gbuf,
           double *__restrict__ energy_rank, double *__restrict__ virial_rank,
           int32_t *__restrict__ triplets_rank, const uint8_t *__restrict__ owned,
           unsigned long long *status, int64_t tag, int debug_mode, int32_t *ovf,
           int32_t *work, int32_t *splits) {
    pdl_enter();
    extern __shared__ __align__(16) char smem_raw[];
    if (!work) {  // one base per warp
        const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
        if (r >= n) return;
        a3_base<kExactImage, kOwned, kM>(r, smem_raw, g, n, pr, rows, row_count, mirror,
                                         capacity, slots, cut, own, gbuf,
                                         energy_rank, virial_rank, triplets_rank, owned, status,
                                         tag, debug_mode, ovf, splits);
        return;
    }
    // persistent warps: the next base comes from a global counter (reset by
    // the gather), fetched one base ahead, so no warp idles behind the
    // slowest base of its block; every base writes only its own outputs
    const int lane = threadIdx.x & 31;
    int r = 0;
    if (lane == 0) r = atomicAdd(work, 1);
    r = __shfl_sync(0xffffffffu, r, 0);
    while (r < n) {
        int nxt = 0;
        if (lane == 0) nxt = atomicAdd(work, 1);
        a3_base<kExactImage, kOwned, kM>(r, smem_raw, g, n, pr, rows, row_count, mirror, capacity,
                                         slots, cut, own, gbuf, energy_rank,
                                         virial_rank, triplets_rank, owned, status, tag,
                                         debug_mode, ovf, splits);
        __syncwarp();  // the warp's slots are reused by its next base
        r = __shfl_sync(0xffffffffu, nxt, 0);
    }
}

// the bases listed by the main pass, with the full slot count
template <bool kExactImage, bool kOwned>
__global__ void __launch_bounds__(kA3Warps * 32)
    k_atm3_overflow(rb_grid g, int64_t n, const double *__restrict__ pr, const int32_t *__restrict__ rows,
           const int32_t *__restrict__ row_count, const int32_t *__restrict__ mirror,
           int32_t capacity, int32_t slots, A3Cut cut,
           double *__restrict__ own, double *__restrict__ gbuf,
           double *__restrict__ energy_rank, double *__restrict__ virial_rank,
           int32_t *__restrict__ triplets_rank, const uint8_t *__restrict__ owned,
           unsigned long long *status, int64_t tag, int debug_mode, const int32_t *ovf,
           int32_t *splits) {
    pdl_enter();
    extern __shared__ __align__(16) char smem_raw[];
    const int wpb = blockDim.x >> 5;
    const int cnt = *(volatile const int32_t *)ovf;
    for (int64_t q = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); q < cnt;
         q += (int64_t)gridDim.x * wpb) {
        a3_base<kExactImage, kOwned, 0>(ovf[2 + q], smem_raw, g, n, pr, rows, row_count, mirror,
                                        capacity, slots, cut,
                                        own, gbuf, energy_rank, virial_rank, triplets_rank,
                                        owned, status, tag, debug_mode, nullptr, splits);
        __syncwarp();  // the warp's slots are reused by its next base
    }
}

// F(p) = 2 nu * (own(p) + sum over row entries k of p with q = row[k] < p of
// G[p][k]); the row prefix is walked in order by kG lanes, then a fixed xor
// tree.
constexpr int kGatherGroup = 8;

__global__ void k_atm3_gather(int64_t n, const int32_t *__restrict__ parts,
                              const int32_t *__restrict__ splits, int32_t capacity,
                              const double *__restrict__ own, const double *__restrict__ gbuf,
                              const double *__restrict__ e_s, const double *__restrict__ w_s,
                              const int32_t *__restrict__ n_s, double two_nu, double nu,
                              double *__restrict__ forces, double *__restrict__ energy_rank,
                              double *__restrict__ virial_rank,
                              int32_t *__restrict__ triplets_rank,
                              const unsigned long long *status, int64_t tag, int32_t *ovf) {
    pdl_enter();
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // list empty for the next pass
        ovf[1] = ovf[0];                           // (count of this pass: diagnostic)
        ovf[0] = 0;
        ovf[-1] = 0;                               // base counter of the persistent pass
    }
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t p = gid / kGatherGroup;
    const int sub = (int)(gid % kGatherGroup);
    const bool active = p < n;
    tag = resolve_tag(tag, status);
    if (warp_frozen(status, tag, RB_KIND_TRIPLET_MIN_SEPARATION)) return;
    double fx = 0.0, fy = 0.0, fz = 0.0;
    if (active) {
        // the row prefix of ranks below p (its base recorded the length,
        // a3_slots): exactly the entries G[p][k] its bases wrote, summed in
        // row order by kGatherGroup lanes; no row indices are read
        const int sp = splits[p];
        RB_CHECK(sp >= 0 && sp <= capacity);
        const double2 *gp = (const double2 *)(gbuf + p * (int64_t)capacity * kGStride);
        for (int k = sub; k < sp; k += kGatherGroup) {
            const double2 xy = gp[2 * k];
            fx += xy.x;
            fy += xy.y;
            fz += gp[2 * k + 1].x;
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
        energy_rank[p] = nu * e_s[p];
        virial_rank[p] = -two_nu * w_s[p];
        triplets_rank[p] = n_s[p];
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

static size_t a3_header_bytes(size_t n) { return ((n + 3) * sizeof(int32_t) + 255) & ~(size_t)255; }

extern "C" size_t rb_atm_scratch_bytes(int64_t n, int32_t capacity) {
    // header at a fixed offset (independent of n, which a decomposed run
    // changes between passes): the persistent pass's base counter, the
    // overflow count, a diagnostic copy of it, then the overflow list (n);
    // after it (256-byte aligned) own (n x 3), the per-base energy and
    // virial sums (n each) and triplet counts (n int32, 8-byte padded) --
    // every output the caller sees is written by the gather, so the triplet
    // kernels may run concurrently with the pair pass -- then G
    // (n x capacity x 4: 32-byte entries, aligned) doubles
    const size_t nn = (size_t)(n > 0 ? n : 1);
    return a3_header_bytes(nn) + nn * 5 * sizeof(double) +
           2 * ((nn * sizeof(int32_t) + 7) & ~(size_t)7) + 32 +
           nn * kGStride * sizeof(double) * (size_t)capacity;
}

namespace rb {
// Slots of the main launch.  A slot costs 60 bytes of shared memory: up to
// 96 slots a warp holds the longest S+(i) outright and one launch does all
// (64 and 96 have compile-time layouts).  Larger counts take about half the
// slots in the main launch and
// list the few longer bases for a second, full-slot launch: S+(i) of most
// bases is about half a row, only bases whose neighbours mostly follow them
// in rank order (cells next to the periodic wrap of the cell order) approach
// a full row.
static int a3_fast_slots(int slot_capacity) {
    if (slot_capacity <= 96) return slot_capacity;  // measured: one launch is faster here
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
                           const int32_t *mirror, int32_t capacity, int fast, const A3Cut &cut, double *own, double *gbuf,
                           double *energy_rank, double *virial_rank, int32_t *triplets_rank,
                           const uint8_t *owned, unsigned long long *status, int64_t tag,
                           int debug_mode, int32_t *ovf, int32_t *work, int32_t *splits) {
    static size_t granted = 0;
    static int resident = 0;  // co-resident blocks per SM at this shared-memory size
    static const int64_t persist_min =
        getenv("RB_ATM_PERSIST_MIN") ? atoll(getenv("RB_ATM_PERSIST_MIN")) : 1;
    static size_t resident_for = 0;
    auto kern = k_atm3<kExactImage, kOwned, kM>;
    a3_grant(kern, warps * per, granted);
    int64_t blocks = (n + warps - 1) / warps;
    if (work) {
        if (resident_for != warps * per) {
            int per_sm = 0, dev = 0, sms = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, warps * 32, warps * per);
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            resident = std::max(1, per_sm) * std::max(1, sms);
            resident_for = warps * per;
        }
        // measured (B200, skin rows, kernel_bench): persistent warps win at
        // every size once the core runs unconditionally (cfg2 -3 %,
        // cfg3@2.5 -12 %, cfg4 0 %); RB_ATM_PERSIST_MIN = minimum bases
        // per resident warp (tuning only)
        if (n > persist_min * (int64_t)resident * warps) blocks = std::min<int64_t>(blocks, resident);
        else work = nullptr;
    }
    launch(kern, dim3((unsigned)blocks), dim3(warps * 32),
           warps * per, st, g, n, pos_r, rows, row_count, mirror, capacity, fast, cut,
           own, gbuf, energy_rank, virial_rank, triplets_rank, owned, status, tag, debug_mode,
           ovf, work, splits);
    note_launches(1);
}

template <bool kExactImage, bool kOwned>
static void a3_launch(cudaStream_t st, const rb_grid &g, int64_t n, const double *pos_r,
                      const int32_t *rows, const int32_t *row_count, const int32_t *mirror,
                      int32_t capacity, int fast, int full, const A3Cut &cut,
                      double *own, double *gbuf, double *energy_rank, double *virial_rank,
                      int32_t *triplets_rank, const uint8_t *owned, unsigned long long *status,
                      int64_t tag, int debug_mode, int32_t *ovf, int32_t *work, int32_t *splits) {
    static size_t granted_ovf = 0;
    // the standard case runs the fast instance (64 slots, register-resident
    // rounds) and always lists bases beyond it -- S+ over 64 slots, or a slot
    // under the guard distance -- for the second launch
    constexpr bool kStd = !kExactImage;
    if (kStd) fast = std::min(64, full);
    const size_t per = a3_warp_bytes(kStd ? 64 : fast);
    const int warps = a3_warps_for(per);
    const bool split = kStd || fast < full;
    int32_t *list = split ? ovf : nullptr;
    // the common slot counts get compile-time layouts
    if (kStd)
        a3_launch_main<kExactImage, kOwned, 64>(st, n, warps, per, g, pos_r, rows, row_count,
                                                mirror, capacity, 64, cut, own,
                                                gbuf, energy_rank, virial_rank, triplets_rank,
                                                owned, status, tag, debug_mode, list, work,
                                                splits);
    else if (fast == 64)
        a3_launch_main<kExactImage, kOwned, 64>(st, n, warps, per, g, pos_r, rows, row_count,
                                                mirror, capacity, fast, cut, own,
                                                gbuf, energy_rank, virial_rank, triplets_rank,
                                                owned, status, tag, debug_mode, list, work,
                                                splits);
    else if (fast == 96)
        a3_launch_main<kExactImage, kOwned, 96>(st, n, warps, per, g, pos_r, rows, row_count,
                                                mirror, capacity, fast, cut, own,
                                                gbuf, energy_rank, virial_rank, triplets_rank,
                                                owned, status, tag, debug_mode, list, work,
                                                splits);
    else
        a3_launch_main<kExactImage, kOwned, 0>(st, n, warps, per, g, pos_r, rows, row_count,
                                               mirror, capacity, fast, cut, own,
                                               gbuf, energy_rank, virial_rank, triplets_rank,
                                               owned, status, tag, debug_mode, list, work,
                                               splits);
    if (!split) return;
    const size_t per_full = a3_warp_bytes(full);
    const int wf = a3_warps_for(per_full);
    const int64_t need = (n + wf - 1) / wf;
    const unsigned blocks = (unsigned)(need < 148 * 4 ? need : 148 * 4);
    a3_grant(k_atm3_overflow<kExactImage, kOwned>, wf * per_full, granted_ovf);
    launch(k_atm3_overflow<kExactImage, kOwned>, dim3(blocks), dim3(wf * 32), wf * per_full, st,
           g, n, pos_r, rows, row_count, mirror, capacity, full, cut, own, gbuf,
           energy_rank, virial_rank, triplets_rank, owned, status, tag, debug_mode,
           (const int32_t *)ovf, splits);
    note_launches(1);
}
}  // namespace rb

extern "C" int rb_atm_pass_part(const rb_grid *g, int64_t n, const double *pos_r,
                                const int32_t *cell_particles, const int32_t *rows,
                                const int32_t *row_count, const int32_t *mirror, int32_t capacity,
                                int32_t slot_capacity, double rc, double nu, double *forces,
                                double *energy_rank, double *virial_rank, int32_t *triplets_rank,
                                const uint8_t *owned, void *scratch, size_t scratch_bytes,
                                unsigned long long *status, int64_t tag, int32_t part,
                                void *stream) {
    NvtxRange nvtx_range("triplet (rb_atm_pass_part)");
    if (part < 0 || part > 2) return RB_ERR_ARGUMENT;
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
    int32_t *work_word = (int32_t *)scratch;
    int32_t *ovf = work_word + 1;
    double *own = (double *)((char *)scratch + a3_header_bytes((size_t)n));
    double *e_s = own + 3 * n, *w_s = e_s + n;
    int32_t *n_s = (int32_t *)(w_s + n);
    // the row prefix length of every base (a3_slots), read by the gather
    int32_t *splits = (int32_t *)((char *)n_s + (((size_t)n * sizeof(int32_t) + 7) & ~(size_t)7));
    double *gbuf = (double *)((char *)splits + (((size_t)n * sizeof(int32_t) + 7) & ~(size_t)7));
    gbuf = (double *)(((uintptr_t)gbuf + 31) & ~(uintptr_t)31);  // whole 32-byte sectors
    auto hiword = [](double x) {
        int64_t b;
        memcpy(&b, &x, sizeof b);
        return (int)(b >> 32);
    };
    A3Cut cut;
    cut.rc2 = rc2;
    cut.lo_hi = hiword(rc2 * (1.0 - kA3Margin));
    cut.hi_hi = hiword(rc2 * (1.0 + kA3Margin));
    cut.min_hi = hiword(RB_MIN_DISTANCE_SQ);
    static const bool persist = !(getenv("RB_ATM_PERSIST") && atoi(getenv("RB_ATM_PERSIST")) == 0);
    int32_t *work = persist ? work_word : nullptr;
    auto go = [&](auto exact, auto with_owned) {
        a3_launch<decltype(exact)::value, decltype(with_owned)::value>(
            st, *g, n, pos_r, rows, row_count, mirror, capacity, fast, slot_capacity, cut,
            own, gbuf, e_s, w_s, n_s, owned, status, tag, debug_mode, ovf, work, splits);
    };
    using T = std::true_type;
    using F = std::false_type;
    if (part != 2) {
        if (exact_image)
            owned ? go(T{}, T{}) : go(T{}, F{});
        else
            owned ? go(F{}, T{}) : go(F{}, F{});
    }
    if (part == 1) return launch_status();
    const int tb = 256;
    const int64_t threads = n * kGatherGroup;
    launch(k_atm3_gather, dim3((unsigned)((threads + tb - 1) / tb)), dim3(tb), 0, st, n, cell_particles, splits, capacity, own, gbuf, e_s, w_s, n_s, 2.0 * nu, nu, forces,
        energy_rank, virial_rank, triplets_rank, status, tag, ovf);
    note_launches(1);
    return launch_status();
}

extern "C" int rb_atm_pass(const rb_grid *g, int64_t n, const double *pos_r, const int32_t *cell_particles, const int32_t *rows,
                           const int32_t *row_count, const int32_t *mirror, int32_t capacity,
                           int32_t slot_capacity, double rc, double nu, double *forces, double *energy_rank,
                           double *virial_rank, int32_t *triplets_rank, const uint8_t *owned,
                           void *scratch, size_t scratch_bytes, unsigned long long *status,
                           int64_t tag, void *stream) {
    return rb_atm_pass_part(g, n, pos_r, cell_particles, rows, row_count, mirror, capacity,
                            slot_capacity, rc, nu, forces, energy_rank, virial_rank, triplets_rank,
                            owned, scratch, scratch_bytes, status, tag, 0, stream);
}
