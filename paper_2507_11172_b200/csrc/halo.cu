// halo.cu -- ghost-position pack / unpack for the domain-decomposed loop
// (SURVEY §8b "halo pack/unpack for multi-GPU").
//
// Between row rebuilds every step sends the owners' new positions along the
// staged (x -> y -> z) send lists kept at the last rebuild: pack gathers the
// listed local rows into a contiguous message, unpack writes a received
// message into the ghost rows and their rank-ordered copy the force kernels
// read.  Plain 24-byte records, one thread per record.  rb_halo_pull is the
// peer-memory form of the same refresh (no messages).
#include <cstring>

#include "common.cuh"

namespace rb {

__global__ void k_halo_pack(int64_t n, const int32_t *__restrict__ idx,
                            const double *__restrict__ pos, double *__restrict__ buf) {
    pdl_enter();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t p = idx[i];
    buf[3 * i] = pos[3 * p];
    buf[3 * i + 1] = pos[3 * p + 1];
    buf[3 * i + 2] = pos[3 * p + 2];
}

__global__ void k_halo_unpack(int64_t n, const double *__restrict__ buf, int64_t first,
                              double *__restrict__ pos, const int32_t *__restrict__ rank_of,
                              double *__restrict__ pos_r) {
    pdl_enter();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t p = first + i;
    const double x = buf[3 * i], y = buf[3 * i + 1], z = buf[3 * i + 2];
    pos[3 * p] = x;
    pos[3 * p + 1] = y;
    pos[3 * p + 2] = z;
    if (pos_r) {
        const int64_t r = rank_of[p];
        pos_r[3 * r] = x;
        pos_r[3 * r + 1] = y;
        pos_r[3 * r + 2] = z;
    }
}

// Peer-memory ghost refresh: every ghost row reads its owner's position
// straight from the owner's published copy (peer memory mapped over
// NVLink / NVSwitch with CUDA IPC), one thread per ghost row.  The
// publishing drift of every rank completed before the step's rebuild vote,
// which every rank passes before launching this kernel; the copy is double
// buffered by the parity of the device step counter (status[1]) so an
// owner's next drift cannot overwrite what a slower peer still reads, and a
// captured step replays at either parity.
__global__ void k_halo_pull(int64_t n, const int32_t *__restrict__ src_rank,
                            const int32_t *__restrict__ src_index,
                            const unsigned long long *__restrict__ peers, int64_t stride,
                            const unsigned long long *__restrict__ status, int64_t first,
                            double *__restrict__ pos, const int32_t *__restrict__ rank_of,
                            double *__restrict__ pos_r) {
    pdl_enter();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (rebuild_frozen(status[0], (int64_t)status[1])) return;  // (a frozen window step)
    // the half the owners' drifts of this step (status[1]) published into
    const int64_t half = (int64_t)(status[1] & 1ull) * 3 * stride;
    const double *src = reinterpret_cast<const double *>(peers[src_rank[i]]) + half +
                        3 * (int64_t)src_index[i];
    const double x = __ldcv(src), y = __ldcv(src + 1), z = __ldcv(src + 2);
    const int64_t p = first + i;
    pos[3 * p] = x;
    pos[3 * p + 1] = y;
    pos[3 * p + 2] = z;
    if (pos_r) {
        const int64_t r = rank_of[p];
        pos_r[3 * r] = x;
        pos_r[3 * r + 1] = y;
        pos_r[3 * r + 2] = z;
    }
}

}  // namespace rb

using namespace rb;

extern "C" int rb_halo_pull(int64_t n, const int32_t *src_rank, const int32_t *src_index,
                            const uint64_t *peers, int64_t stride,
                            const unsigned long long *status, int64_t first, double *pos,
                            const int32_t *rank_of, double *pos_r, void *stream) {
    NvtxRange nvtx_range("halo (rb_halo_pull)");
    if (n < 0 || first < 0 || stride < 0 ||
        (n > 0 && (!src_rank || !src_index || !peers || !status || !pos || (pos_r && !rank_of))))
        return RB_ERR_ARGUMENT;
    if (n == 0) return RB_OK;
    launch(k_halo_pull, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, as_stream(stream), n,
           src_rank, src_index, reinterpret_cast<const unsigned long long *>(peers), stride,
           status, first, pos, rank_of, pos_r);
    note_launches(1);
    return launch_status();
}

// ---- CUDA IPC for the published copies (one allocation per rank) --------
extern "C" int rb_ipc_alloc(int64_t bytes, void **ptr) {
    if (bytes <= 0 || !ptr) return RB_ERR_ARGUMENT;
    *ptr = nullptr;
    if (cudaMalloc(ptr, (size_t)bytes) != cudaSuccess) return RB_ERR_CUDA;
    return cudaMemset(*ptr, 0, (size_t)bytes) == cudaSuccess ? RB_OK : RB_ERR_CUDA;
}

extern "C" int rb_ipc_free(void *ptr) {
    if (!ptr) return RB_OK;
    return cudaFree(ptr) == cudaSuccess ? RB_OK : RB_ERR_CUDA;
}

extern "C" int rb_ipc_handle(void *ptr, uint8_t *handle64) {
    if (!ptr || !handle64) return RB_ERR_ARGUMENT;
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, ptr) != cudaSuccess) return RB_ERR_CUDA;
    memcpy(handle64, &h, 64);
    return RB_OK;
}

extern "C" int rb_ipc_open(const uint8_t *handle64, void **ptr) {
    if (!handle64 || !ptr) return RB_ERR_ARGUMENT;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, 64);
    *ptr = nullptr;
    return cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess
               ? RB_OK : RB_ERR_CUDA;
}

extern "C" int rb_ipc_close(void *ptr) {
    if (!ptr) return RB_OK;
    return cudaIpcCloseMemHandle(ptr) == cudaSuccess ? RB_OK : RB_ERR_CUDA;
}

extern "C" int rb_halo_pack(int64_t n, const int32_t *idx, const double *pos, double *buf,
                            void *stream) {
    NvtxRange nvtx_range("halo (rb_halo_pack)");
    if (n < 0 || (n > 0 && (!idx || !pos || !buf))) return RB_ERR_ARGUMENT;
    if (n == 0) return RB_OK;
    launch(k_halo_pack, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, as_stream(stream), n,
           idx, pos, buf);
    note_launches(1);
    return launch_status();
}

extern "C" int rb_halo_unpack(int64_t n, const double *buf, int64_t first, double *pos,
                              const int32_t *rank_of, double *pos_r, void *stream) {
    NvtxRange nvtx_range("halo (rb_halo_unpack)");
    if (n < 0 || first < 0 || (n > 0 && (!buf || !pos || (pos_r && !rank_of))))
        return RB_ERR_ARGUMENT;
    if (n == 0) return RB_OK;
    launch(k_halo_unpack, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, as_stream(stream), n,
           buf, first, pos, rank_of, pos_r);
    note_launches(1);
    return launch_status();
}
