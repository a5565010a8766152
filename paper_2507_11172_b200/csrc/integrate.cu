// integrate.cu -- fused r-RESPA kick/drift, deterministic reductions and the
// measurement helpers bench.py uses.
//
// The updates restate the numpy statements of respamd/integrators.py:148-170
// with numpy's rounding order (every product and sum rounded separately, so
// the _rn intrinsics keep nvcc from contracting them into FMAs):
//
//   drift (tag = i+1):  if i % s == 0:  v = v + half_respa*f3          (:149-150)
//                       x = x + (dt*v + half_drift*f2_old)              (:151)
//                       wrap into [0, box)                              (:152-153)
//   kick  (tag = i+1):  v = v + half_dt*(f2_old + f2_new)              (:158)
//                       if (i+1) % s == 0:  v = v + half_respa*f3       (:165)
//
// Arrays are the reference's (n,3) AoS, handled as flat 3n streams.
#include "common.cuh"

#include <atomic>
#include <cstdlib>

namespace rb {

static std::atomic<long long> g_launches{0};
void note_launches(int k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
thread_local cudaError_t g_launch_error = cudaSuccess;
bool pdl_on() {
    static const bool on = !(getenv("RB_PDL") && atoi(getenv("RB_PDL")) == 0);
    return on;
}

// numpy float remainder (npy_divmod) followed by the edge fix of
// respamd/model.py:279-280
__device__ __forceinline__ double wrap_coord(double x, double box) {
    // one box away at most after a step: fmod's value without its loop
    // (x - box is exact for box <= x < 2 box, Sterbenz)
    double r;
    if (x >= 0.0 && x < box) r = x;
    else if (x >= box && x < 2.0 * box) r = x - box;
    else if (x < 0.0 && x > -box) r = x;
    else r = fmod(x, box);
    if (r != 0.0) {
        if (r < 0.0) r = xadd(r, box);
    } else {
        r = 0.0;  // copysign(0, box) with box > 0
    }
    if (r >= box) r = 0.0;
    return r;
}

// Four lanes per particle, lane c < 3 on component c of the AoS arrays
// (coalesced: a warp covers 8 particles = 24 contiguous doubles per array;
// lane 3 idles).  A thread serves kU particles a grid stride apart and issues
// every load of all of them -- and both status words -- before the first
// use: the pass is one memory round trip per thread, so the bytes in flight
// per SM (not the instruction count) set its speed (ncu, cfg4: one particle
// per thread left DRAM at 29 % with 60 % of the stalls on the status round
// trip).  Besides the drift it (a) scatters the new position into the
// rank-ordered copy the force kernels read, and (b) compares against the
// positions of the last neighbour-row build: a particle that moved more than
// skin/2 flags a rebuild of the rows in this very step (*rebuild_flag = tag),
// so every pair within rc is always inside the rows built at rc + skin.  The
// displacement norm is gathered by shuffles into lane 0 of the group.
#ifndef RB_DRIFT_U
#define RB_DRIFT_U 4
#endif
template <int kU>
__global__ void k_drift(int64_t n, double *__restrict__ pos, double *__restrict__ vel,
                        double *__restrict__ f2_old, const double *__restrict__ f3,
                        double bx, double by, double bz, int periodic, double dt,
                        double half_drift, double half_respa, int kick3,
                        const int32_t *__restrict__ rank_of, double *__restrict__ pr,
                        const double *__restrict__ x_ref, double skin_half2,
                        int64_t *rebuild_flag, unsigned long long *status, int64_t tag,
                        int advance, cudaGraphConditionalHandle cond,
                        const double *__restrict__ f2_new, double half_dt, int kick_prev,
                        int kick3_prev, double *__restrict__ publish, int64_t pub_stride) {
    pdl_enter();
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;  // a multiple of 4
    const int c = (int)(gt & 3);
    // every load of the step first (one memory round trip; the status words
    // ride along), the decisions after
    double v[kU], fo[kU], fnew[kU], f3v[kU], px[kU], xr[kU];
    int32_t ro[kU];
    bool act[kU];
    int64_t ix[kU];
#pragma unroll
    for (int u = 0; u < kU; u++) {
        const int64_t p = (gt + u * stride) >> 2;
        act[u] = p < n && c < 3;
        ix[u] = 3 * p + c;
        v[u] = fo[u] = fnew[u] = f3v[u] = px[u] = xr[u] = 0.0;
        ro[u] = 0;
        if (act[u]) {
            const int64_t i = ix[u];
            v[u] = vel[i];
            fo[u] = f2_old[i];
            px[u] = pos[i];
            if (kick_prev) fnew[u] = f2_new[i];
            if (kick3 || (kick_prev && kick3_prev)) f3v[u] = f3[i];
            if (x_ref) xr[u] = x_ref[i];
            if (pr && rank_of) ro[u] = rank_of[p];
        }
    }
    const ulonglong2 s01 = ld_status2(status);
    // status[2] (the last CLOSED step) is written by the previous step's
    // pair pass / kick only: loaded with the rest
    const ulonglong2 s23 = advance ? ld_status2(status + 2) : make_ulonglong2(0ull, 0ull);
    // a step-opening drift numbers its step from the last CLOSED step
    // (status[2], written by the step's pair pass and kick) and publishes it
    // in status[1]: no kernel reads the word another block of it writes.
    const unsigned long long sw = s01.x;  // the error word as this step found it
    if (advance) {
        tag = (int64_t)s23.x + 1;
        if (rebuild_frozen(sw, tag)) return;  // a speculative window stopped here
        if (gt == 0) status[1] = (unsigned long long)tag;
    } else if (tag < 0) {
        tag = status ? (int64_t)s01.y : 0;
    }
    if (rebuild_frozen(sw, tag)) return;
    if (kick_prev) {
        // the kick that closes the previous step (tag - 1), folded in: the
        // same updates and error rules as k_kick (integrators.py:158-165)
        const int64_t tp = tag - 1;
        bool go = true, do3 = kick3_prev != 0;
        if (sw != RB_STATUS_CLEAR) {
            const long long t = (long long)(sw >> 8);
            const int k = (int)(sw & 0xff);
            if (t < tp || (t == tp && k == RB_KIND_PAIR_MIN_SEPARATION)) go = false;
            if (t == tp && k == RB_KIND_TRIPLET_MIN_SEPARATION) do3 = false;
        }
#pragma unroll
        for (int u = 0; u < kU; u++) {
            if (go && act[u]) {
                double w = xadd(v[u], xmul(half_dt, xadd(fo[u], fnew[u])));
                if (do3) w = xadd(w, xmul(half_respa, f3v[u]));
                v[u] = w;
                vel[ix[u]] = w;
                f2_old[ix[u]] = fnew[u];
                fo[u] = fnew[u];
                if (!isfinite(w)) record_status(status, tp, RB_KIND_NONFINITE);
            }
        }
    }
    // an earlier step failed: freeze (errors of this step do not stop it)
    const bool run = sw == RB_STATUS_CLEAR || (long long)(sw >> 8) >= tag;
    const double box = c == 0 ? bx : (c == 1 ? by : bz);
#pragma unroll
    for (int u = 0; u < kU; u++) {
        const int64_t i = ix[u];
        double d = 0.0;
        if (run && act[u]) {
            double w = v[u];
            if (kick3) {
                w = xadd(w, xmul(half_respa, f3v[u]));
                vel[i] = w;
            }
            double xc = xadd(px[u], xadd(xmul(dt, w), xmul(half_drift, fo[u])));
            if (periodic) xc = wrap_coord(xc, box);
            pos[i] = xc;
            if (!isfinite(xc)) record_status(status, tag, RB_KIND_NONFINITE);
            if (pr && rank_of) pr[3 * (int64_t)ro[u] + c] = xc;
            if (publish) {  // the copy peers pull their ghosts from (rb_halo_pull),
                            // the half of this step's parity
                publish[(tag & 1) * 3 * pub_stride + i] = xc;
                __threadfence_system();
            }
            if (x_ref) {
                d = xc - xr[u];
                if (periodic) d = min_image(d, box, 0.5 * box);
            }
        }
        if (x_ref && rebuild_flag) {  // uniform: every lane takes the shuffles
            const double dy = __shfl_down_sync(0xffffffffu, d, 1);
            const double dz = __shfl_down_sync(0xffffffffu, d, 2);
            if (run && act[u] && c == 0) {
                const double d2 = d * d + dy * dy + dz * dz;
                if (!(d2 <= skin_half2)) {  // also catches NaN
                    // the first thread to flag this step counts a rebuild step
                    const unsigned long long was =
                        atomicExch(reinterpret_cast<unsigned long long *>(rebuild_flag),
                                   (unsigned long long)tag);
                    if ((int64_t)was != tag && status) atomicAdd(status + 3, 1ull);
                    if (cond) cudaGraphSetConditional(cond, 1u);
                }
            }
        }
    }
}

// kU entries a grid stride apart per thread, all loads first (k_drift)
template <int kU>
__global__ void k_kick(int64_t n3, double *__restrict__ vel, double *__restrict__ f2_old,
                       const double *__restrict__ f2_new, const double *__restrict__ f3,
                       double half_dt, double half_respa, int kick3, unsigned long long *status,
                       int64_t tag) {
    pdl_enter();
    const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    // loads first, the status words with them (one round trip)
    double v[kU], fo[kU], fnew[kU], f3v[kU];
#pragma unroll
    for (int u = 0; u < kU; u++) {
        const int64_t i = i0 + u * stride;
        v[u] = fo[u] = fnew[u] = f3v[u] = 0.0;
        if (i < n3) {
            v[u] = vel[i];
            fo[u] = f2_old[i];
            fnew[u] = f2_new[i];
            if (kick3) f3v[u] = f3[i];
        }
    }
    const ulonglong2 s01 = ld_status2(status);
    const bool from_device = tag < 0;
    if (tag < 0) tag = status ? (int64_t)s01.y : 0;
    if (status && rebuild_frozen(s01.x, tag)) return;  // (the step stays open)
    if (from_device && status && i0 == 0) status[2] = (unsigned long long)tag;  // closes the step
    bool do_kick2 = true, do_kick3 = kick3 != 0;
    const unsigned long long s = s01.x;
    if (s != RB_STATUS_CLEAR) {
        const long long t = (long long)(s >> 8);
        const int k = (int)(s & 0xff);
        if (t < tag) return;
        if (t == tag && k == RB_KIND_PAIR_MIN_SEPARATION) return;  // raised before :158
        if (t == tag && k == RB_KIND_TRIPLET_MIN_SEPARATION) do_kick3 = false;  // before :165
    }
#pragma unroll
    for (int u = 0; u < kU; u++) {
        const int64_t i = i0 + u * stride;
        if (i >= n3) continue;
        double w = v[u];
        if (do_kick2) w = xadd(w, xmul(half_dt, xadd(fo[u], fnew[u])));
        if (do_kick3) w = xadd(w, xmul(half_respa, f3v[u]));
        vel[i] = w;
        f2_old[i] = fnew[u];  // np.copyto(f2_old, forces_2b), integrators.py:159
        if (!isfinite(w)) record_status(status, tag, RB_KIND_NONFINITE);
    }
}

// ---------------------------------------------------------------------------
// deterministic sums: the partition depends only on n, each CTA sums its
// contiguous slice with a fixed per-thread stride and a fixed tree, then one
// CTA sums the partials in index order.
// ---------------------------------------------------------------------------
constexpr int kRedThreads = 256;
constexpr int kRedMaxBlocks = 592;  // 4 x 148 SMs

__host__ __device__ inline int red_blocks(int64_t n) {
    int64_t b = (n + 1023) / 1024;  // ~4 entries per thread: latency, not bandwidth
    if (b < 1) b = 1;
    if (b > kRedMaxBlocks) b = kRedMaxBlocks;
    return (int)b;
}


template <typename Tin, typename Tacc, bool kSquare>
__global__ void k_partial_sum(int64_t n, const Tin *__restrict__ in, Tacc *__restrict__ partial) {
    pdl_enter();
    __shared__ Tacc sh[32];
    const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
    const int64_t b = (int64_t)blockIdx.x * chunk;
    const int64_t e = b + chunk < n ? b + chunk : n;
    Tacc acc = 0;
    for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x) {
        Tacc v = (Tacc)in[i];
        acc += kSquare ? v * v : v;
    }
    Tacc s = block_tree_sum<Tacc>(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

template <typename Tacc>
__global__ void k_final_sum(int nb, const Tacc *__restrict__ partial, Tacc *__restrict__ out) {
    pdl_enter();
    __shared__ Tacc sh[32];
    Tacc acc = 0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) acc += partial[i];
    Tacc s = block_tree_sum<Tacc>(acc, sh);
    if (threadIdx.x == 0) out[0] = s;
}

// Sample point of the device loop in one launch: the five sums of a trace
// row (sum v^2 over 3n, E2, W2, E3, W3 over the n rank entries), each with
// the partition and trees of k_partial_sum/k_final_sum (bit-identical to the
// separate reductions); the block that finishes last (ticket) folds the
// partials in index order and writes the trace row.
constexpr int kSampleQ = 5;

// block_tree_sum of five values at once: the same shuffle tree and the same
// warp-0 fold per value (bit-identical), one __syncthreads for all five
__device__ __forceinline__ void block_tree_sum5(double v[kSampleQ], double (*sh)[32]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < kSampleQ; q++) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], off);
        if (lane == 0) sh[q][warp] = v[q];
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int q = 0; q < kSampleQ; q++) {
            double t = lane < (int)(blockDim.x >> 5) ? sh[q][lane] : 0.0;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
            v[q] = t;
        }
    }
}

__global__ void __launch_bounds__(kRedThreads)
    k_sample(int64_t n, const double *__restrict__ vel, const double *__restrict__ e2,
             const double *__restrict__ w2, const double *__restrict__ e3,
             const double *__restrict__ w3, double *__restrict__ sums,
             const unsigned long long *status, int64_t interval, double *trace,
             double *__restrict__ partial, unsigned int *ticket) {
    pdl_enter();
    __shared__ double sh[kSampleQ][32];
    __shared__ bool last;
    // the partitions of k_partial_sum: 3n components for sum v^2, n rank
    // entries for E2, W2, E3, W3; every thread accumulates its stride in
    // index order.  The first four elements of both partitions are loaded
    // together (one memory round trip for the usual sizes).
    const int64_t len = 3 * n;
    const int nbA = red_blocks(len), nbB = red_blocks(n);
    const int bid = (int)blockIdx.x;
    int64_t ia = 0, ea = 0, ib = 0, eb = 0;
    if (bid < nbA) {
        const int64_t chunk = (len + nbA - 1) / nbA;
        ia = (int64_t)bid * chunk + threadIdx.x;
        ea = (int64_t)bid * chunk + chunk < len ? (int64_t)bid * chunk + chunk : len;
    }
    if (bid < nbB) {
        const int64_t chunk = (n + nbB - 1) / nbB;
        ib = (int64_t)bid * chunk + threadIdx.x;
        eb = (int64_t)bid * chunk + chunk < n ? (int64_t)bid * chunk + chunk : n;
    }
    constexpr int kPre = 4;
    double va[kPre], vb[kPre][4];
#pragma unroll
    for (int u = 0; u < kPre; u++) {
        const int64_t i = ia + (int64_t)u * blockDim.x, j = ib + (int64_t)u * blockDim.x;
        va[u] = i < ea ? vel[i] : 0.0;
        vb[u][0] = j < eb ? e2[j] : 0.0;
        vb[u][1] = j < eb ? w2[j] : 0.0;
        vb[u][2] = j < eb ? e3[j] : 0.0;
        vb[u][3] = j < eb ? w3[j] : 0.0;
    }
    double acc[kSampleQ] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int u = 0; u < kPre; u++) {
        if (ia + (int64_t)u * blockDim.x < ea) acc[0] += va[u] * va[u];
        if (ib + (int64_t)u * blockDim.x < eb) {
#pragma unroll
            for (int q = 0; q < 4; q++) acc[1 + q] += vb[u][q];
        }
    }
    for (int64_t i = ia + (int64_t)kPre * blockDim.x; i < ea; i += blockDim.x)
        acc[0] += vel[i] * vel[i];
    for (int64_t j = ib + (int64_t)kPre * blockDim.x; j < eb; j += blockDim.x) {
        acc[1] += e2[j];
        acc[2] += w2[j];
        acc[3] += e3[j];
        acc[4] += w3[j];
    }
    block_tree_sum5(acc, sh);
    if (threadIdx.x == 0) {
        if (bid < nbA) partial[bid] = acc[0];
        if (bid < nbB)
            for (int q = 1; q < kSampleQ; q++) partial[q * kRedMaxBlocks + bid] = acc[q];
        __threadfence();
        last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double out[kSampleQ];
#pragma unroll
    for (int q = 0; q < kSampleQ; q++) {
        const int nb = q == 0 ? nbA : nbB;
        out[q] = 0.0;
        for (int i = threadIdx.x; i < nb; i += blockDim.x)
            out[q] += *(volatile const double *)(partial + q * kRedMaxBlocks + i);
    }
    block_tree_sum5(out, sh);
    // a step a speculative window froze records nothing (it is run again)
    const bool fz = status && rebuild_frozen(status[0], (int64_t)status[1]);
    if (threadIdx.x == 0 && fz) *ticket = 0u;
    if (threadIdx.x == 0 && !fz) {
        for (int q = 0; q < kSampleQ; q++) sums[q] = out[q];
        if (trace) {
            const int64_t tag = (int64_t)status[1];
            double *row = trace + 8 * (tag / interval);
            row[0] = (double)tag;
            for (int q = 0; q < kSampleQ; q++) row[1 + q] = out[q];
            row[6] = 0.0;
            row[7] = 0.0;
        }
        *ticket = 0u;  // ready for the next launch
    }
}

template <typename Tin, typename Tacc, bool kSquare>
static int reduce_launch(int64_t n, const Tin *in, Tacc *out, void *scratch, void *stream) {
    cudaStream_t st = as_stream(stream);
    const int nb = red_blocks(n);
    Tacc *partial = (Tacc *)scratch;
    launch(k_partial_sum<Tin, Tacc, kSquare>, dim3(nb), dim3(kRedThreads), 0, st, n, in, partial);
    note_launches(1);
    launch(k_final_sum<Tacc>, dim3(1), dim3(kRedThreads), 0, st, nb, partial, out);
    note_launches(1);
    return launch_status();
}

// ---------------------------------------------------------------------------
// measurement helpers
// ---------------------------------------------------------------------------
constexpr int kPeakChains = 8;

__global__ void k_fp64_fma(int iters, double seed, double *sink) {
    double a[kPeakChains];
#pragma unroll
    for (int c = 0; c < kPeakChains; c++) a[c] = seed + c * 1e-3 + threadIdx.x * 1e-9;
    const double m = 0.999999999, k = 1e-9;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int u = 0; u < 16; u++) {
#pragma unroll
            for (int c = 0; c < kPeakChains; c++) a[c] = fma(a[c], m, k);
        }
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < kPeakChains; c++) s += a[c];
    if (s == 12345.678) sink[0] = s;  // keep the chains alive
}

__global__ void k_step_begin(unsigned long long *status) {
    pdl_enter();
    status[2] = status[1];
    status[1] += 1ull;
}

// trace row (tag / interval): [tag, sum v^2, E2, W2, E3, W3, 0, 0]
__global__ void k_trace_record(const unsigned long long *status, int64_t interval, double *trace,
                               const double *sumsq, const double *e2, const double *w2,
                               const double *e3, const double *w3) {
    pdl_enter();
    const int64_t tag = (int64_t)status[1];
    double *row = trace + 8 * (tag / interval);
    row[0] = (double)tag;
    row[1] = *sumsq;
    row[2] = *e2;
    row[3] = *w2;
    row[4] = *e3;
    row[5] = *w3;
    row[6] = 0.0;
    row[7] = 0.0;
}

// the rebuild vote of the current step (rb_vote_flag / rb_vote_freeze)
__global__ void k_vote_flag(const int64_t *rebuild_flag, const unsigned long long *status,
                            int64_t *flag) {
    pdl_enter();
    *flag = rebuild_flag[0] == (int64_t)status[1] ? 1 : 0;
}
__global__ void k_vote_freeze(const int64_t *flag, unsigned long long *status) {
    pdl_enter();
    if (*flag > 0 && status[0] == RB_STATUS_CLEAR)
        status[0] = (status[1] << 8) | (unsigned long long)RB_KIND_REBUILD;
}

__global__ void k_flush(int4 *buf, int64_t n16, int v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16;
         i += (int64_t)gridDim.x * blockDim.x)
        buf[i] = make_int4(v, v, v, v);
}

}  // namespace rb

using namespace rb;

static int drift_launch(int64_t n, double *pos, double *vel, double *f2_old, const double *f2_new,
                        const double *f3, const double *box3_host, int32_t periodic, double dt,
                        double half_dt, double half_drift, double half_respa, int32_t kick3,
                        int32_t kick_prev, int32_t kick3_prev, const int32_t *rank_of,
                        double *pos_r, const double *x_ref, double skin, int64_t *rebuild_flag,
                        unsigned long long *status, int64_t tag, int32_t advance_step,
                        uint64_t rebuild_cond, void *stream, double *publish = nullptr,
                        int64_t pub_stride = 0) {
    if (n < 0 || !box3_host) return RB_ERR_ARGUMENT;
    if (advance_step && (!status || tag >= 0)) return RB_ERR_ARGUMENT;
    if (n == 0) return advance_step ? rb_step_begin(status, stream) : RB_OK;
    const int tb = 256;
    const double half = 0.5 * skin;
    constexpr int kU = RB_DRIFT_U;
    launch(k_drift<kU>, dim3((unsigned)((4 * n + (int64_t)tb * kU - 1) / ((int64_t)tb * kU))),
           dim3(tb), 0, as_stream(stream), n, pos,
           vel, f2_old, f3, box3_host[0], box3_host[1], box3_host[2], periodic, dt, half_drift,
           half_respa, kick3, rank_of, pos_r, x_ref, half * half * (1.0 - 1e-9), rebuild_flag,
           status, tag, advance_step ? 1 : 0, (cudaGraphConditionalHandle)rebuild_cond, f2_new,
           half_dt, kick_prev ? 1 : 0, kick3_prev ? 1 : 0, publish, pub_stride);
    note_launches(1);
    return launch_status();
}

extern "C" int rb_respa_drift(int64_t n, double *pos, double *vel, const double *f2_old,
                              const double *f3, const double *box3_host, int32_t periodic,
                              double dt, double half_drift, double half_respa, int32_t kick3,
                              const int32_t *rank_of, double *pos_r, const double *x_ref,
                              double skin, int64_t *rebuild_flag, unsigned long long *status,
                              int64_t tag, int32_t advance_step, uint64_t rebuild_cond,
                              void *stream) {
    NvtxRange nvtx_range("drift (rb_respa_drift)");
    return drift_launch(n, pos, vel, const_cast<double *>(f2_old), nullptr, f3, box3_host,
                        periodic, dt, 0.0, half_drift, half_respa, kick3, 0, 0, rank_of, pos_r,
                        x_ref, skin, rebuild_flag, status, tag, advance_step, rebuild_cond,
                        stream);
}

extern "C" int rb_respa_drift_publish(int64_t n, double *pos, double *vel, const double *f2_old,
                                      const double *f3, const double *box3_host, int32_t periodic,
                                      double dt, double half_drift, double half_respa,
                                      int32_t kick3, const int32_t *rank_of, double *pos_r,
                                      const double *x_ref, double skin, int64_t *rebuild_flag,
                                      unsigned long long *status, int64_t tag,
                                      int32_t advance_step, double *publish, int64_t stride,
                                      void *stream) {
    NvtxRange nvtx_range("drift+publish (rb_respa_drift_publish)");
    if (!publish || stride < n || !advance_step) return RB_ERR_ARGUMENT;
    return drift_launch(n, pos, vel, const_cast<double *>(f2_old), nullptr, f3, box3_host,
                        periodic, dt, 0.0, half_drift, half_respa, kick3, 0, 0, rank_of, pos_r,
                        x_ref, skin, rebuild_flag, status, tag, advance_step, 0, stream, publish,
                        stride);
}

extern "C" int rb_respa_kick_drift(int64_t n, double *pos, double *vel, double *f2_old,
                                   const double *f2_new, const double *f3,
                                   const double *box3_host, int32_t periodic, double dt,
                                   double half_dt, double half_drift, double half_respa,
                                   int32_t kick3_prev, int32_t kick3, const int32_t *rank_of,
                                   double *pos_r, const double *x_ref, double skin,
                                   int64_t *rebuild_flag, unsigned long long *status,
                                   uint64_t rebuild_cond, void *stream) {
    NvtxRange nvtx_range("kick+drift (rb_respa_kick_drift)");
    if (!status || !f2_new) return RB_ERR_ARGUMENT;
    return drift_launch(n, pos, vel, f2_old, f2_new, f3, box3_host, periodic, dt, half_dt,
                        half_drift, half_respa, kick3, 1, kick3_prev, rank_of, pos_r, x_ref, skin,
                        rebuild_flag, status, -1, 1, rebuild_cond, stream);
}

extern "C" int rb_respa_kick(int64_t n, double *vel, double *f2_old, const double *f2_new,
                             const double *f3, double half_dt, double half_respa, int32_t kick3,
                             unsigned long long *status, int64_t tag, void *stream) {
    NvtxRange nvtx_range("kick (rb_respa_kick)");
    if (n < 0) return RB_ERR_ARGUMENT;
    const int64_t n3 = 3 * n;
    if (n == 0 && (tag >= 0 || !status)) return RB_OK;  // (tag < 0: still closes the step)
    const int tb = 256;
    constexpr int kU = RB_DRIFT_U;
    const int64_t per = (int64_t)tb * kU;
    launch(k_kick<kU>, dim3(n3 > 0 ? (unsigned)((n3 + per - 1) / per) : 1u), dim3(tb), 0,
           as_stream(stream), n3, vel, f2_old, f2_new, f3, half_dt, half_respa, kick3, status,
           tag);
    note_launches(1);
    return launch_status();
}

extern "C" size_t rb_reduce_scratch_bytes(int64_t n) {
    return (size_t)kRedMaxBlocks * sizeof(double);
}

extern "C" size_t rb_sample_scratch_bytes(int64_t n) {
    return (size_t)kSampleQ * kRedMaxBlocks * sizeof(double) + 256;
}

extern "C" int rb_sample(int64_t n, const double *vel, const double *e2_rank,
                         const double *w2_rank, const double *e3_rank, const double *w3_rank,
                         double *sums, const unsigned long long *status, int64_t sample_interval,
                         double *trace, void *scratch, size_t scratch_bytes, void *stream) {
    NvtxRange nvtx_range("sample (rb_sample)");
    if (n < 0 || !vel || !e2_rank || !w2_rank || !e3_rank || !w3_rank || !sums || !scratch)
        return RB_ERR_ARGUMENT;
    if (scratch_bytes < rb_sample_scratch_bytes(n)) return RB_ERR_ARGUMENT;
    if (trace && (!status || sample_interval <= 0)) return RB_ERR_ARGUMENT;
    // every sum keeps its own partition (the v^2 sum spans 3n entries)
    const int nb = red_blocks(3 * n);
    double *partial = (double *)scratch;
    unsigned int *ticket = (unsigned int *)(partial + kSampleQ * kRedMaxBlocks);
    launch(k_sample, dim3(nb), dim3(kRedThreads), 0, as_stream(stream), n, vel, e2_rank, w2_rank, e3_rank,
                                                       w3_rank, sums, status, sample_interval,
                                                       trace, partial, ticket);
    note_launches(1);
    return launch_status();
}

extern "C" int rb_reduce_sum_f64(int64_t n, const double *in, double *out, void *scratch,
                                 void *stream) {
    if (n < 0 || !out || !scratch) return RB_ERR_ARGUMENT;
    return reduce_launch<double, double, false>(n, in, out, scratch, stream);
}

extern "C" int rb_reduce_sumsq_f64(int64_t n, const double *in, double *out, void *scratch,
                                   void *stream) {
    if (n < 0 || !out || !scratch) return RB_ERR_ARGUMENT;
    return reduce_launch<double, double, true>(n, in, out, scratch, stream);
}

extern "C" int rb_reduce_sum_i32(int64_t n, const int32_t *in, int64_t *out, void *scratch,
                                 void *stream) {
    if (n < 0 || !out || !scratch) return RB_ERR_ARGUMENT;
    return reduce_launch<int32_t, long long, false>(n, in, (long long *)out, scratch, stream);
}

extern "C" int rb_fp64_peak(int32_t iters, double *tflops, void *stream) {
    if (iters <= 0 || !tflops) return RB_ERR_ARGUMENT;
    cudaStream_t st = as_stream(stream);
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double *sink = nullptr;
    if (cudaMalloc(&sink, sizeof(double)) != cudaSuccess) return RB_ERR_CUDA;
    const int threads = 512, blocks = sms * 4;
    k_fp64_fma<<<blocks, threads, 0, st>>>(iters / 4 + 1, 1.0, sink);
    note_launches(1);  // warm-up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    k_fp64_fma<<<blocks, threads, 0, st>>>(iters, 1.0, sink);
    note_launches(1);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    const double flops = 2.0 * (double)blocks * threads * (double)iters * 16.0 * kPeakChains;
    *tflops = flops / ((double)ms * 1e-3) / 1e12;
    return launch_status();
}

extern "C" int rb_step_begin(unsigned long long *status, void *stream) {
    if (!status) return RB_ERR_ARGUMENT;
    launch(k_step_begin, dim3(1), dim3(1), 0, as_stream(stream), status);
    note_launches(1);
    return launch_status();
}

extern "C" int rb_trace_record(const unsigned long long *status, int64_t sample_interval,
                               double *trace, const double *sumsq, const double *e2,
                               const double *w2, const double *e3, const double *w3,
                               void *stream) {
    if (!status || !trace || sample_interval <= 0) return RB_ERR_ARGUMENT;
    launch(k_trace_record, dim3(1), dim3(1), 0, as_stream(stream), status, sample_interval, trace, sumsq, e2, w2,
                                                   e3, w3);
    note_launches(1);
    return launch_status();
}

extern "C" int rb_l2_flush(void *buf, size_t bytes, void *stream) {
    if (!buf) return RB_ERR_ARGUMENT;
    static int v = 0;
    v++;
    k_flush<<<148 * 8, 256, 0, as_stream(stream)>>>((int4 *)buf, (int64_t)(bytes / 16), v);
    note_launches(1);
    return launch_status();
}

extern "C" int rb_abi_version(void) { return RB_ABI_VERSION; }

extern "C" long long rb_launch_count(void) { return g_launches.load(); }

extern "C" size_t rb_grid_bytes(void) { return sizeof(rb_grid); }

extern "C" const char *rb_status_string(int status) {
    switch (status) {
        case RB_OK: return "ok";
        case RB_ERR_MIN_SEPARATION: return "minimum separation violated";
        case RB_ERR_GEOMETRY: return "invalid cell-grid geometry";
        case RB_ERR_CUDA: return "CUDA launch error";
        case RB_ERR_CAPACITY: return "neighbour-row capacity exceeded";
        case RB_ERR_ARGUMENT: return "invalid argument";
        case RB_NOT_CAPTURING: return "stream is not capturing";
        default: return "unknown status";
    }
}

extern "C" int rb_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

extern "C" int rb_event_create(void **event) {
    if (!event) return RB_ERR_ARGUMENT;
    cudaEvent_t e;
    if (cudaEventCreateWithFlags(&e, cudaEventDefault) != cudaSuccess) return RB_ERR_CUDA;
    *event = (void *)e;
    return RB_OK;
}

extern "C" int rb_event_destroy(void *event) {
    return cudaEventDestroy((cudaEvent_t)event) == cudaSuccess ? RB_OK : RB_ERR_CUDA;
}

extern "C" int rb_event_record(void *event, void *stream) {
    // external: inside a stream capture this becomes an event-record node
    return cudaEventRecordWithFlags((cudaEvent_t)event, as_stream(stream),
                                    cudaEventRecordExternal) == cudaSuccess
               ? RB_OK
               : RB_ERR_CUDA;
}

extern "C" int rb_event_elapsed(void *start, void *end, float *ms) {
    if (!ms) return RB_ERR_ARGUMENT;
    if (cudaEventSynchronize((cudaEvent_t)end) != cudaSuccess) return RB_ERR_CUDA;
    return cudaEventElapsedTime(ms, (cudaEvent_t)start, (cudaEvent_t)end) == cudaSuccess
               ? RB_OK
               : RB_ERR_CUDA;
}

extern "C" int rb_vote_flag(const int64_t *rebuild_flag, const unsigned long long *status,
                            int64_t *flag, void *stream) {
    if (!rebuild_flag || !status || !flag) return RB_ERR_ARGUMENT;
    launch(k_vote_flag, dim3(1), dim3(1), 0, as_stream(stream), rebuild_flag, status, flag);
    note_launches(1);
    return launch_status();
}

extern "C" int rb_vote_freeze(const int64_t *flag, unsigned long long *status, void *stream) {
    if (!flag || !status) return RB_ERR_ARGUMENT;
    launch(k_vote_freeze, dim3(1), dim3(1), 0, as_stream(stream), flag, status);
    note_launches(1);
    return launch_status();
}
