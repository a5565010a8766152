// halo.cu -- ghost-position pack / unpack for the domain-decomposed loop
// (SURVEY §8b "halo pack/unpack for multi-GPU").
//
// Between row rebuilds every step sends the owners' new positions along the
// staged (x -> y -> z) send lists kept at the last rebuild: pack gathers the
// listed local rows into a contiguous message, unpack writes a received
// message into the ghost rows and their rank-ordered copy the force kernels
// read.  Plain 24-byte records, one thread per record.
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

}  // namespace rb

using namespace rb;

extern "C" int rb_halo_pack(int64_t n, const int32_t *idx, const double *pos, double *buf,
                            void *stream) {
    if (n < 0 || (n > 0 && (!idx || !pos || !buf))) return RB_ERR_ARGUMENT;
    if (n == 0) return RB_OK;
    launch(k_halo_pack, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, as_stream(stream), n,
           idx, pos, buf);
    note_launches(1);
    return launch_status();
}

extern "C" int rb_halo_unpack(int64_t n, const double *buf, int64_t first, double *pos,
                              const int32_t *rank_of, double *pos_r, void *stream) {
    if (n < 0 || first < 0 || (n > 0 && (!buf || !pos || (pos_r && !rank_of))))
        return RB_ERR_ARGUMENT;
    if (n == 0) return RB_OK;
    launch(k_halo_unpack, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, as_stream(stream), n,
           buf, first, pos, rank_of, pos_r);
    note_launches(1);
    return launch_status();
}
