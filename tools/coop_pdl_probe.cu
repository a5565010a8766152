// coop_pdl_probe.cu -- does a cooperative launch accept the programmatic
// stream serialization attribute too, eagerly and under stream capture?
// (decides how rb_rebuild launches its grid-barrier kernel)
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>

__global__ void k_prev(int *x) { if (threadIdx.x == 0) atomicAdd(x, 1); }
__global__ void k_coop(int *x) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    cooperative_groups::this_grid().sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(x, 100);
}

static cudaError_t go(cudaStream_t st, int *x, int blocks, bool pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute a[2];
    a[0].id = cudaLaunchAttributeCooperative;
    a[0].val.cooperative = 1;
    a[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = a;
    cfg.numAttrs = pdl ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, k_coop, x);
}

int main() {
    int *x;
    cudaMalloc(&x, 4);
    cudaMemset(x, 0, 4);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    int per = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_coop, 256, 0);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = per * sms;
    k_prev<<<1, 32, 0, st>>>(x);
    cudaError_t e1 = go(st, x, blocks, true);
    cudaError_t s1 = cudaStreamSynchronize(st);
    printf("eager coop+pdl: launch %s sync %s\n", cudaGetErrorString(e1), cudaGetErrorString(s1));
    cudaGetLastError();
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    k_prev<<<1, 32, 0, st>>>(x);
    cudaError_t e2 = go(st, x, blocks, true);
    cudaError_t c2 = cudaStreamEndCapture(st, &g);
    printf("captured coop+pdl: launch %s end %s\n", cudaGetErrorString(e2), cudaGetErrorString(c2));
    if (c2 == cudaSuccess) {
        cudaError_t i2 = cudaGraphInstantiate(&ge, g, 0);
        cudaError_t l2 = i2 == cudaSuccess ? cudaGraphLaunch(ge, st) : i2;
        cudaError_t s2 = cudaStreamSynchronize(st);
        printf("  instantiate %s launch %s sync %s\n", cudaGetErrorString(i2), cudaGetErrorString(l2),
               cudaGetErrorString(s2));
    }
    cudaGetLastError();
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    k_prev<<<1, 32, 0, st>>>(x);
    cudaError_t e3 = go(st, x, blocks, false);
    cudaError_t c3 = cudaStreamEndCapture(st, &g);
    printf("captured coop only: launch %s end %s\n", cudaGetErrorString(e3), cudaGetErrorString(c3));
    if (c3 == cudaSuccess) {
        cudaError_t i3 = cudaGraphInstantiate(&ge, g, 0);
        cudaError_t l3 = i3 == cudaSuccess ? cudaGraphLaunch(ge, st) : i3;
        cudaError_t s3 = cudaStreamSynchronize(st);
        printf("  instantiate %s launch %s sync %s\n", cudaGetErrorString(i3), cudaGetErrorString(l3),
               cudaGetErrorString(s3));
    }
    int h = 0;
    cudaMemcpy(&h, x, 4, cudaMemcpyDeviceToHost);
    printf("counter %d\n", h);
    return 0;
}
