// atm_cells.cu -- cell-based Newton-3 ATM triplet pass.
//
// Replaces respamd/containers.py:373-535 (_c01_triplet_kernel) with the same
// results as the row-based pass (atm3.cu) -- every unique triplet i < j < k
// (rank order) evaluated once by the warp of its lowest-rank member, forces
// delivered deterministically -- but organised around linked cells
// (containers.py:50-72) instead of Verlet rows:
//
//   * the base of a triplet is its member whose cell comes first in the
//     lexicographic order of the signed stencil offsets between the members'
//     cells (same cell: the lowest rank).  With at least four cells per
//     periodic dimension the offsets of three mutually neighbouring cells
//     add up exactly, so this is a total order on every triplet -- each is
//     evaluated once -- and, unlike rank order (which wraps at the box
//     faces), every cell's forward neighbourhood is the same 13 cells.
//   * one CTA per base cell (persistent CTAs on a cell counter).  It stages
//     the cell and its 13 forward stencil neighbours, in offset order, into
//     shared memory: fp64 positions, fp32 copies, ranks.
//   * S+(i) from shared memory: an fp32 distance filter (band 1e-3 relative
//     around rc^2; the staged fp32 copies are minimum-image coordinates
//     relative to the base cell's centre) compacts the candidates, the
//     reference arithmetic (exact_disp / exact_r2, bit-exact predicate)
//     decides them; the slots and the pair loop are atm_core.cuh's.
//   * partial forces of the slots go to a per-warp target accumulator in
//     shared memory (bases are assigned to warps statically, so the
//     grouping of the sums is fixed); after the cell, the warps' sums are
//     added in warp order and written once per (target, source cell) into
//     G2[p][o] (32-byte entries, o = the stencil offset from the source
//     cell to p's cell).
//   * k_atm_cells_gather: F(p) = 2 nu (own(p) + sum over the forward stencil
//     offsets o of G2[p][o]), in offset order.
//
// Memory traffic per pass is the staged positions (L2-resident), one G2
// write and read per (particle, source cell) and the per-base outputs --
// no neighbour rows, no scattered 24-byte partial-force writes.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "atm_core.cuh"

namespace rb {

#ifndef RB_AC_WARPS
#define RB_AC_WARPS 4
#endif
#ifndef RB_AC_MIN_BLOCKS
#define RB_AC_MIN_BLOCKS 3
#endif
constexpr int kACWarps = RB_AC_WARPS;
constexpr int kACMaxOffsets = 27;   // reach-1 stencils (cell size >= the cutoff)
constexpr float kACBand = 1e-3f;    // fp32 filter band around rc^2 (relative)

struct ACLayout {
    int nb_cap, slots;
    size_t nbx, nbf, nbr, ta_xy, ta_z, warp, hdr, total;
};

__host__ __device__ inline size_t ac_align(size_t x) { return (x + 15) & ~(size_t)15; }

// dynamic shared memory of one CTA: header (staged cells), the staged
// neighbourhood, kACWarps target accumulators, kACWarps slot sets
__host__ __device__ inline ACLayout ac_layout(int nb_cap, int slots) {
    ACLayout l;
    l.nb_cap = nb_cap;
    l.slots = slots;
    size_t o = 0;
    l.hdr = o;
    o += ac_align(4 * (kACMaxOffsets + 1) * sizeof(int32_t) + 16 * sizeof(int32_t));
    l.nbx = o;
    o += ac_align((size_t)nb_cap * 3 * sizeof(double));
    l.nbf = o;
    o += ac_align((size_t)nb_cap * sizeof(float4));
    l.nbr = o;
    o += ac_align((size_t)nb_cap * sizeof(int32_t));
    l.ta_xy = o;
    o += ac_align((size_t)kACWarps * nb_cap * sizeof(double2));
    l.ta_z = o;
    o += ac_align((size_t)kACWarps * nb_cap * sizeof(double));
    l.warp = o;
    o += (size_t)kACWarps * ac_align(a3_warp_bytes(slots));
    l.total = o;
    return l;
}

// the stencil neighbour of cell (cx, cy, cz) at offset o and its inverse
__device__ __forceinline__ int ac_source_cell(const rb_grid &g, int t, int o) {
    int c[3];
    int tz = t % g.cells[2];
    int ty = (t / g.cells[2]) % g.cells[1];
    int tx = t / (g.cells[2] * g.cells[1]);
    const int tc[3] = {tx, ty, tz};
#pragma unroll
    for (int d = 0; d < 3; d++) {
        int x = tc[d] - g.offsets[o][d];
        if (g.wrap[d]) {
            if (x < 0) x += g.cells[d];
        } else if (x < 0 || x >= g.cells[d]) {
            return -1;
        }
        c[d] = x;
    }
    return (c[0] * g.cells[1] + c[1]) * g.cells[2] + c[2];
}

// signed stencil offset (canonical offsets are stored mod n in wrapped
// dimensions) and the forward half: lexicographically >= (0, 0, 0)
__device__ __forceinline__ int ac_signed(const rb_grid &g, int o, int d) {
    const int v = g.offsets[o][d];
    return g.wrap[d] && v > g.cells[d] / 2 ? v - g.cells[d] : v;
}
__device__ __forceinline__ bool ac_forward(const rb_grid &g, int o) {
    const int x = ac_signed(g, o, 0), y = ac_signed(g, o, 1), z = ac_signed(g, o, 2);
    return x > 0 || (x == 0 && (y > 0 || (y == 0 && z >= 0)));
}

template <bool kOwned>
__global__ void __launch_bounds__(kACWarps * 32, RB_AC_MIN_BLOCKS)
    k_atm_cells(rb_grid g, int32_t ncell, const double *__restrict__ pr,
                const int32_t *__restrict__ cell_start, const uint8_t *__restrict__ owned,
                A3Cut cut, float hi_f, int32_t nb_cap, int32_t slots,
                double *__restrict__ own, double *__restrict__ e_s, double *__restrict__ w_s,
                int32_t *__restrict__ n_s, double4 *__restrict__ g2,
                unsigned long long *status, int64_t tag, int32_t *work) {
    pdl_enter();
    extern __shared__ __align__(16) char smem[];
    const ACLayout L = ac_layout(nb_cap, slots);
    int32_t *h_cell = (int32_t *)(smem + L.hdr);           // [kACMaxOffsets] staged cell ids
    int32_t *h_start = h_cell + (kACMaxOffsets + 1);       // [..] their first rank
    int32_t *h_base = h_start + (kACMaxOffsets + 1);       // [..+1] staged index prefix
    int32_t *h_off = h_base + (kACMaxOffsets + 1);         // [..] their offset index
    int32_t *h_misc = h_off + (kACMaxOffsets + 1);         // cell, ncells staged, total, self
    double *nbx = (double *)(smem + L.nbx);
    float4 *nbf = (float4 *)(smem + L.nbf);
    int32_t *nbr = (int32_t *)(smem + L.nbr);
    double2 *ta_xy = (double2 *)(smem + L.ta_xy);
    double *ta_z = (double *)(smem + L.ta_z);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const A3Smem sm = a3_carve<0>(smem + L.warp + (size_t)warp * ac_align(a3_warp_bytes(slots)),
                                  slots);
    double2 *my_ta_xy = ta_xy + (size_t)warp * nb_cap;
    double *my_ta_z = ta_z + (size_t)warp * nb_cap;
    tag = resolve_tag(tag, status);
    const Image im = make_image(g);
    const double ibox[3] = {1.0 / g.box[0], 1.0 / g.box[1], 1.0 / g.box[2]};
    const int cells_yz = g.cells[1] * g.cells[2];
    for (;;) {
        if (tid == 0) {
            h_misc[0] = atomicAdd(work, 1);
            h_misc[4] = status && frozen(status, tag, RB_KIND_TRIPLET_MIN_SEPARATION);
        }
        __syncthreads();
        const int c = h_misc[0];
        if (c >= ncell) break;
        if (h_misc[4]) {  // an earlier error of the step: the pass's outputs are not used
            __syncthreads();
            continue;
        }
        // ---- the staged cells: c and its forward stencil neighbours, offset order
        if (warp == 0) {
            const int cx = c / cells_yz, cy = (c / g.cells[2]) % g.cells[1], cz = c % g.cells[2];
            int nc = -1, cnt = 0;
            if (lane < g.n_offsets && ac_forward(g, lane)) {
                nc = neighbor_cell(g, cx, cy, cz, lane);
                if (nc >= 0) cnt = cell_start[nc + 1] - cell_start[nc];
            }
            const unsigned keep = __ballot_sync(0xffffffffu, nc >= 0);
            const int j = __popc(keep & lanemask_lt());
            int x = cnt;  // inclusive scan of the staged counts (offset order)
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, off);
                if (lane >= off) x += y;
            }
            if (nc >= 0) {
                h_cell[j] = nc;
                h_start[j] = cell_start[nc];
                h_base[j] = x - cnt;
                h_off[j] = lane;
                if (nc == c) h_misc[3] = j;
            }
            if (lane == 31) {
                h_misc[1] = __popc(keep);
                h_misc[2] = x;
                h_base[__popc(keep)] = x;
            }
        }
        __syncthreads();
        const int total = h_misc[2], self = h_misc[3];
        double ctr[3];  // centre of cell c (global frame; windows offset by wlo)
        {
            const int cc[3] = {c / cells_yz, (c / g.cells[2]) % g.cells[1], c % g.cells[2]};
#pragma unroll
            for (int d = 0; d < 3; d++)
                ctr[d] = g.origin[d] + ((g.wrap[d] ? 0 : g.wlo[d]) + cc[d] + 0.5) / g.inv_cell[d];
        }
        if (total > nb_cap) {  // the neighbourhood does not fit: capacity error, retried larger
            if (tid == 0) record_status(status, tag, RB_KIND_CAPACITY);
            __syncthreads();
            continue;
        }
        // ---- stage positions (fp64 and fp32) and ranks; clear the accumulators
        for (int k = tid; k < total; k += blockDim.x) {
            int j = 0;
            while (h_base[j + 1] <= k) j++;
            const int r = h_start[j] + (k - h_base[j]);
            const double x = pr[3 * r], y = pr[3 * r + 1], z = pr[3 * r + 2];
            nbx[3 * k] = x;
            nbx[3 * k + 1] = y;
            nbx[3 * k + 2] = z;
            // fp32 copy relative to the base cell's centre, minimum image
            // (whatever cell the particle drifted into since the binning)
            double rel[3] = {x - ctr[0], y - ctr[1], z - ctr[2]};
            if (g.periodic) {
#pragma unroll
                for (int d = 0; d < 3; d++) rel[d] = fma(-g.box[d], rint(rel[d] * ibox[d]), rel[d]);
            }
            nbf[k] = make_float4((float)rel[0], (float)rel[1], (float)rel[2], 0.0f);
            nbr[k] = r;
        }
        for (int k = tid; k < kACWarps * total; k += blockDim.x) {
            const int w = k / total, kk = k - w * total;
            ta_xy[(size_t)w * nb_cap + kk] = make_double2(0.0, 0.0);
            ta_z[(size_t)w * nb_cap + kk] = 0.0;
        }
        __syncthreads();
        // ---- the bases of cell c, statically over the warps in snake order
        // (0 1 2 3 3 2 1 0 0 1 ...: S+ shrinks along the cell's rank order)
        const int bb0 = h_base[self], bb1 = h_base[self + 1];
        for (int q = 0;; q++) {
            const int round = q, lanew = (round & 1) ? kACWarps - 1 - warp : warp;
            const int bi = bb0 + round * kACWarps + lanew;
            if (bi >= bb1) break;
            const int r = nbr[bi];
            const double xi = nbx[3 * bi], yi = nbx[3 * bi + 1], zi = nbx[3 * bi + 2];
            const float4 fi = nbf[bi];
            // phase 0a: fp32 filter over the staged neighbourhood -> candidates
            // (in the slot accumulator area, as ints, until phase 1)
            int32_t *cand = reinterpret_cast<int32_t *>(sm.axy);
            const int cand_cap = (slots + 1) * 4;  // axy + az hold (slots + 1) * 24 bytes
            int nc = 0;
            bool over = false;
            for (int k0 = 0; k0 < total; k0 += 32) {
                const int k = k0 + lane;
                bool pass = false;
                if (k < total && (k > bi || k < bb0)) {  // forward cells, or later in c
                    const float4 o = nbf[k];  // relative to c's centre: no minimum image
                    const float dx = fi.x - o.x, dy = fi.y - o.y, dz = fi.z - o.z;
                    pass = fmaf(dz, dz, fmaf(dy, dy, dx * dx)) <= hi_f;
                }
                const unsigned mk = __ballot_sync(0xffffffffu, pass);
                if (nc + __popc(mk) > cand_cap) {
                    over = true;
                    break;
                }
                if (pass) {
                    RB_CHECK(nc + __popc(mk & lanemask_lt()) < cand_cap);
                    cand[nc + __popc(mk & lanemask_lt())] = k;
                }
                nc += __popc(mk);
            }
            __syncwarp();
            // phase 0b: the reference arithmetic on the candidates -> slots
            int m = 0;
            bool slot_bad = false;
            for (int c0 = 0; c0 < nc && !over; c0 += 32) {
                const int ci = c0 + lane;
                bool keep = false;
                int k = 0;
                double dx = 0.0, dy = 0.0, dz = 0.0, r2 = 0.0;
                if (ci < nc) {
                    k = cand[ci];
                    RB_CHECK(k >= 0 && k < total);
                    exact_disp(im, xi, yi, zi, nbx[3 * k], nbx[3 * k + 1], nbx[3 * k + 2], dx, dy,
                               dz);
                    r2 = exact_r2(dx, dy, dz);
                    keep = r2 <= cut.rc2;
                }
                const unsigned mk = __ballot_sync(0xffffffffu, keep);
                if (m + __popc(mk) > slots) {
                    over = true;
                    break;
                }
                __syncwarp();  // the candidates of this window are read before slots overwrite
                if (keep) {
                    const int s = m + __popc(mk & lanemask_lt());
                    sm.xy[s] = make_double2(dx, dy);
                    sm.zr[s] = make_double2(dz, r2);
                    sm.kidx[s] = k | ((kOwned ? (int)owned[nbr[k]] : 1) << 30);
                    sm.q[s] = nbr[k];
                }
                m += __popc(mk);
                slot_bad |= __any_sync(0xffffffffu, keep && r2 < RB_MIN_DISTANCE_SQ);
            }
            if (over) {  // S+(i) does not fit the slots: capacity error, retried larger
                if (lane == 0) record_status(status, tag, RB_KIND_CAPACITY);
                __syncwarp();
                continue;
            }
            __syncwarp();
            for (int s = lane; s < m; s += 32) {
                sm.axy[s] = make_double2(0.0, 0.0);
                sm.az[s] = 0.0;
            }
            __syncwarp();
            // phase 1: the slot pairs (atm_core.cuh)
            A3Acc acc = {0.0, 0.0, 0, false, kOwned ? (int)owned[r] : 1};
            double F[3] = {0.0, 0.0, 0.0};
            if (slot_bad)
                a3_windows<false, kOwned, true>(sm, m, slots, lane, g, pr, cut, acc, F);
            else
                a3_windows<false, kOwned, false>(sm, m, slots, lane, g, pr, cut, acc, F);
            // phase 3: slot sums -> the warp's target accumulator (targets of
            // one base are distinct); f_i = -sum, the virial from the slot sums
            double sx = 0.0, sy = 0.0, sz = 0.0, sw = 0.0;
            for (int s = lane; s < m; s += 32) {
                double ax = F[0], ay = F[1], az = F[2];
                if (m >= 32) {
                    const double2 a = sm.axy[s];
                    ax = a.x;
                    ay = a.y;
                    az = sm.az[s];
                }
                const int k = sm.kidx[s] & kKidxMask;
                RB_CHECK(k < total && total <= nb_cap);
                double2 t = my_ta_xy[k];
                t.x += ax;
                t.y += ay;
                my_ta_xy[k] = t;
                my_ta_z[k] += az;
                sx += ax;
                sy += ay;
                sz += az;
                if (!kOwned) {
                    double dx, dy, dz, r2;
                    ld_rec(sm, s, dx, dy, dz, r2);
                    sw = fma(dx, ax, fma(dy, ay, fma(dz, az, sw)));
                }
            }
            const double fx = -group_sum<32>(sx);
            const double fy = -group_sum<32>(sy);
            const double fz = -group_sum<32>(sz);
            const double w = group_sum<32>(kOwned ? acc.w : sw);
            const double e = kOwned ? group_sum<32>(acc.e) : w * (-1.0 / 4.5);
            const int nt = group_sum_int<32>(acc.n);
            const bool bad = __any_sync(0xffffffffu, acc.bad);
            if (lane == 0) {
                own[3 * r] = fx;
                own[3 * r + 1] = fy;
                own[3 * r + 2] = fz;
                e_s[r] = e;
                w_s[r] = w;
                n_s[r] = nt;
                if (bad) record_status(status, tag, RB_KIND_TRIPLET_MIN_SEPARATION);
            }
            __syncwarp();
        }
        __syncthreads();
        // ---- flush: G2[p][o] = sum over the warps (in warp order) for every
        // staged particle p (zero where no base of c reached it)
        for (int k = tid; k < total; k += blockDim.x) {
            int j = 0;
            while (h_base[j + 1] <= k) j++;
            double x = 0.0, y = 0.0, z = 0.0;
#pragma unroll
            for (int w = 0; w < kACWarps; w++) {
                const double2 t = ta_xy[(size_t)w * nb_cap + k];
                x += t.x;
                y += t.y;
                z += ta_z[(size_t)w * nb_cap + k];
            }
            RB_CHECK(j < kACMaxOffsets && h_off[j] < g.n_offsets);
            g2[(size_t)nbr[k] * kACMaxOffsets + h_off[j]] = make_double4(x, y, z, 0.0);
        }
        __syncthreads();
    }
}

// F(p) = 2 nu (own(p) + sum over the forward offsets o, in order, of
// G2[p][o]); kG lanes per particle, fixed xor tree
constexpr int kACGather = 4;

__global__ void k_atm_cells_gather(rb_grid g, int64_t n, const int32_t *__restrict__ parts,
                                   const int32_t *__restrict__ cell_of_rank,
                                   const double *__restrict__ own,
                                   const double4 *__restrict__ g2, const double *__restrict__ e_s,
                                   const double *__restrict__ w_s, const int32_t *__restrict__ n_s,
                                   double two_nu, double nu, double *__restrict__ forces,
                                   double *__restrict__ energy_rank,
                                   double *__restrict__ virial_rank,
                                   int32_t *__restrict__ triplets_rank,
                                   const unsigned long long *status, int64_t tag, int32_t *work) {
    pdl_enter();
    if (blockIdx.x == 0 && threadIdx.x == 0) *work = 0;  // the cell counter of the next pass
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t p = gid / kACGather;
    const int sub = (int)(gid % kACGather);
    const bool active = p < n;
    tag = resolve_tag(tag, status);
    if (warp_frozen(status, tag, RB_KIND_TRIPLET_MIN_SEPARATION)) return;
    double fx = 0.0, fy = 0.0, fz = 0.0;
    if (active) {
        const int t = cell_of_rank[p];
        for (int o = sub; o < g.n_offsets; o += kACGather) {
            if (ac_forward(g, o) && ac_source_cell(g, t, o) >= 0) {
                const double4 v = g2[(size_t)p * kACMaxOffsets + o];
                fx += v.x;
                fy += v.y;
                fz += v.z;
            }
        }
    }
    fx = group_sum<kACGather>(fx);
    fy = group_sum<kACGather>(fy);
    fz = group_sum<kACGather>(fz);
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

// the largest staged neighbourhood of any cell (sizes nb_cap)
__global__ void k_atm_cells_nbmax(rb_grid g, int32_t ncell, const int32_t *__restrict__ cell_start,
                                  int32_t *out) {
    const int cells_yz = g.cells[1] * g.cells[2];
    int best = 0;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncell; c += gridDim.x * blockDim.x) {
        const int cx = c / cells_yz, cy = (c / g.cells[2]) % g.cells[1], cz = c % g.cells[2];
        int tot = 0;
        for (int o = 0; o < g.n_offsets; o++) {
            const int nc = ac_forward(g, o) ? neighbor_cell(g, cx, cy, cz, o) : -1;
            if (nc >= 0) tot += cell_start[nc + 1] - cell_start[nc];
        }
        best = max(best, tot);
    }
    for (int off = 16; off > 0; off >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, off));
    if ((threadIdx.x & 31) == 0) atomicMax(out, best);
}

}  // namespace rb

using namespace rb;

// scratch: header (cell counter), own (n x 3), e_s, w_s (n), n_s (n int32),
// G2 (n x 27 x 4 doubles)
static size_t ac_header_bytes() { return 256; }

extern "C" size_t rb_atm_cells_scratch_bytes(int64_t n) {
    const size_t nn = (size_t)(n > 0 ? n : 1);
    return ac_header_bytes() + nn * 5 * sizeof(double) + ac_align(nn * sizeof(int32_t)) + 32 +
           nn * kACMaxOffsets * sizeof(double4);
}

extern "C" size_t rb_atm_cells_smem_bytes(int32_t nb_cap, int32_t slot_capacity) {
    return ac_layout(nb_cap, slot_capacity).total;
}

extern "C" int rb_atm_cells_supported(const rb_grid *g, double rc) {
    if (!g || g->n_offsets <= 0 || g->n_offsets > kACMaxOffsets) return 0;
    for (int d = 0; d < 3; d++) {
        if (g->cells[d] <= 0) return 0;
        // the forward order needs additive offsets: >= 4 cells per wrapped dimension
        if (g->wrap[d] && g->cells[d] < 4) return 0;
        // every pair within rc lies in the reach-1 stencil: cell size >= rc
        // (containers.py:262: reach 1 iff rc / size <= 1 + 1e-12)
        if (!(rc * g->inv_cell[d] <= 1.0 + 1e-9)) return 0;
        // the pair loop's d_ik - d_ij is a minimum image only in boxes of at
        // least four cutoffs (atm3.cu keeps the exact-image path)
        if (g->periodic && !(g->box[d] > 4.0 * rc * (1.0 + 1e-12))) return 0;
        // the fp32 filter's error (~1e-7 of the box per coordinate) stays
        // far inside its 1e-3 band
        if (!(g->box[d] <= 400.0 * rc)) return 0;
    }
    return 1;
}

extern "C" int rb_atm_pass_cells(const rb_grid *g, int64_t n, const double *pos_r,
                                 const int32_t *cell_particles, const int32_t *cell_start,
                                 const int32_t *cell_of_rank, int32_t nb_cap,
                                 int32_t slot_capacity, double rc, double nu, double *forces,
                                 double *energy_rank, double *virial_rank,
                                 int32_t *triplets_rank, const uint8_t *owned, void *scratch,
                                 size_t scratch_bytes, unsigned long long *status, int64_t tag,
                                 int32_t part, void *stream) {
    NvtxRange nvtx_range("triplet (rb_atm_pass_cells)");
    if (part < 0 || part > 2) return RB_ERR_ARGUMENT;
    if (!g || n < 0 || !scratch || !cell_start || !cell_of_rank) return RB_ERR_ARGUMENT;
    if (!rb_atm_cells_supported(g, rc)) return RB_ERR_ARGUMENT;
    if (nb_cap < 32 || slot_capacity < 32 || slot_capacity > 256) return RB_ERR_ARGUMENT;
    if (scratch_bytes < rb_atm_cells_scratch_bytes(n)) return RB_ERR_ARGUMENT;
    if (n == 0) return RB_OK;
    const ACLayout L = ac_layout(nb_cap, slot_capacity);
    if (L.total > 227 * 1024) return RB_ERR_CAPACITY;
    cudaStream_t st = as_stream(stream);
    int32_t *work = (int32_t *)scratch;
    double *own = (double *)((char *)scratch + ac_header_bytes());
    double *e_s = own + 3 * n, *w_s = e_s + n;
    int32_t *n_s = (int32_t *)(w_s + n);
    // G2 entries are 32-byte aligned (one sector each) whatever n is
    const uintptr_t g2a = ((uintptr_t)((char *)n_s + (size_t)n * sizeof(int32_t)) + 31) & ~(uintptr_t)31;
    double4 *g2 = (double4 *)g2a;
    const int32_t ncell = g->cells[0] * g->cells[1] * g->cells[2];
    const double rc2 = rc * rc;
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
    const float hi_f = (float)(rc2 * (1.0 + kACBand));
    if (part != 2) {
        static int resident = 0, resident_dev = -1;
        static size_t resident_bytes = 0, granted = 0, granted_o = 0;
        int dev = 0;
        cudaGetDevice(&dev);
        auto go = [&](auto kern, size_t &gr) {
            if (L.total > gr) {
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)L.total);
                gr = L.total;
            }
            if (resident_dev != dev || resident_bytes != L.total) {
                int per_sm = 0, sms = 0;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kACWarps * 32,
                                                              L.total);
                cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
                resident = std::max(1, per_sm) * std::max(1, sms);
                resident_dev = dev;
                resident_bytes = L.total;
            }
            const int blocks = std::max(1, std::min(resident, ncell));
            launch(kern, dim3((unsigned)blocks), dim3(kACWarps * 32), L.total, st, *g, ncell,
                   pos_r, cell_start, owned, cut, hi_f, nb_cap, slot_capacity, own, e_s, w_s,
                   n_s, g2, status, tag, work);
            note_launches(1);
        };
        if (owned)
            go(k_atm_cells<true>, granted_o);
        else
            go(k_atm_cells<false>, granted);
    }
    if (part == 1) return launch_status();
    const int tb = 256;
    const int64_t threads = n * kACGather;
    launch(k_atm_cells_gather, dim3((unsigned)((threads + tb - 1) / tb)), dim3(tb), 0, st, *g, n,
           cell_particles, cell_of_rank, own, (const double4 *)g2, e_s, w_s, n_s, 2.0 * nu, nu,
           forces, energy_rank, virial_rank, triplets_rank, status, tag, work);
    note_launches(1);
    return launch_status();
}

extern "C" int rb_atm_cells_nb_max(const rb_grid *g, const int32_t *cell_start, int32_t *out,
                                   void *stream) {
    if (!g || !cell_start || !out) return RB_ERR_ARGUMENT;
    const int32_t ncell = g->cells[0] * g->cells[1] * g->cells[2];
    cudaStream_t st = as_stream(stream);
    if (cudaMemsetAsync(out, 0, sizeof(int32_t), st) != cudaSuccess) return RB_ERR_CUDA;
    const int blocks = std::max(1, std::min(148 * 4, (ncell + 255) / 256));
    k_atm_cells_nbmax<<<blocks, 256, 0, st>>>(*g, ncell, cell_start, out);
    note_launches(1);
    return launch_status();
}
