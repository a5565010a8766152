// graph.cu -- conditional rebuild node for captured r-RESPA steps.
//
// The device loop (integrators.DeviceRespa) replays one CUDA graph per step;
// the row rebuild (binning + rows + mirror, nine kernels) is needed only on
// the steps whose drift flagged it (Verlet skin, integrators.py docstring).
// Instead of nine gated launches that exit at once, the drift sets a graph
// conditional together with the rebuild flag, and an IF node holds the
// rebuild.  The body kernels keep their own gate check, so a body that runs
// is exactly the gated launch sequence.
#include <mutex>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace rb {

namespace {
struct OpenCond {
    cudaStream_t parent = nullptr;
    cudaStream_t body = nullptr;
    cudaGraphNode_t node = nullptr;
    bool open = false;
};
thread_local OpenCond g_open;
thread_local cudaStream_t g_body_stream = nullptr;
}  // namespace

}  // namespace rb

using namespace rb;

extern "C" int rb_rebuild_cond_create(void *stream, uint64_t *handle) {
    if (!handle) return RB_ERR_ARGUMENT;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaGraph_t graph = nullptr;
    if (cudaStreamGetCaptureInfo(as_stream(stream), &cs, nullptr, &graph) != cudaSuccess)
        return RB_ERR_CUDA;
    if (cs != cudaStreamCaptureStatusActive) return RB_NOT_CAPTURING;
    cudaGraphConditionalHandle h;
    if (cudaGraphConditionalHandleCreate(&h, graph, 0, cudaGraphCondAssignDefault) != cudaSuccess)
        return RB_ERR_CUDA;
    *handle = (uint64_t)h;
    return RB_OK;
}

extern "C" int rb_rebuild_cond_begin(uint64_t handle, void *stream, void **body_stream) {
    if (!handle || !body_stream || g_open.open) return RB_ERR_ARGUMENT;
    cudaStream_t s = as_stream(stream);
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaGraph_t graph = nullptr;
    const cudaGraphNode_t *deps = nullptr;
    size_t nd = 0;
    if (cudaStreamGetCaptureInfo(s, &cs, nullptr, &graph, &deps, &nd) != cudaSuccess)
        return RB_ERR_CUDA;
    if (cs != cudaStreamCaptureStatusActive) return RB_NOT_CAPTURING;
    if (!g_body_stream && cudaStreamCreateWithFlags(&g_body_stream, cudaStreamNonBlocking) !=
                              cudaSuccess)
        return RB_ERR_CUDA;
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = (cudaGraphConditionalHandle)handle;
    p.conditional.type = cudaGraphCondTypeIf;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    if (cudaGraphAddNode(&node, graph, deps, nd, &p) != cudaSuccess) return RB_ERR_CUDA;
    if (cudaStreamBeginCaptureToGraph(g_body_stream, p.conditional.phGraph_out[0], nullptr,
                                      nullptr, 0, cudaStreamCaptureModeRelaxed) != cudaSuccess)
        return RB_ERR_CUDA;
    g_open.parent = s;
    g_open.body = g_body_stream;
    g_open.node = node;
    g_open.open = true;
    *body_stream = (void *)g_body_stream;
    return RB_OK;
}

extern "C" int rb_rebuild_cond_end(void *stream) {
    if (!g_open.open || g_open.parent != as_stream(stream)) return RB_ERR_ARGUMENT;
    g_open.open = false;
    cudaGraph_t body = nullptr;
    if (cudaStreamEndCapture(g_open.body, &body) != cudaSuccess) return RB_ERR_CUDA;
    if (cudaStreamUpdateCaptureDependencies(g_open.parent, &g_open.node, 1,
                                            cudaStreamSetCaptureDependencies) != cudaSuccess)
        return RB_ERR_CUDA;
    return RB_OK;
}

// ---- reusable step graphs (domain loop) ---------------------
// A decomposed run captures one graph per step kind for every row epoch
// (counts and lists change at each rebuild, the kernel sequence does not):
// rb_graph_end instantiates the first capture and afterwards updates the
// existing executable in place (cudaGraphExecUpdate, falling back to a new
// instantiation if the topology changed), which costs a fraction of an
// instantiation.  Thread-local capture mode: other host threads (e.g. a
// communication library's watchdog) do not invalidate it.
// kernels per executable, so graph launches count in rb_launch_count
static std::mutex g_graph_mu;
static std::unordered_map<uint64_t, int> g_graph_kernels;

static int count_kernel_nodes(cudaGraph_t g) {
    size_t n = 0;
    if (cudaGraphGetNodes(g, nullptr, &n) != cudaSuccess || n == 0) return 0;
    std::vector<cudaGraphNode_t> nodes(n);
    if (cudaGraphGetNodes(g, nodes.data(), &n) != cudaSuccess) return 0;
    int k = 0;
    for (size_t i = 0; i < n; i++) {
        cudaGraphNodeType t;
        if (cudaGraphNodeGetType(nodes[i], &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) k++;
    }
    return k;
}

extern "C" long long rb_launch_count(void);
static thread_local long long g_capture_mark = 0;

extern "C" int rb_graph_begin(void *stream) {
    if (!stream) return RB_ERR_ARGUMENT;  // the legacy default stream cannot capture
    g_capture_mark = rb_launch_count();
    return cudaStreamBeginCapture(as_stream(stream), cudaStreamCaptureModeThreadLocal) ==
                   cudaSuccess
               ? RB_OK : RB_ERR_CUDA;
}

extern "C" int rb_graph_end(void *stream, uint64_t *exec) {
    if (!stream || !exec) return RB_ERR_ARGUMENT;
    cudaGraph_t g = nullptr;
    // captured launches did not run: they count when the graph is launched
    note_launches((int)(g_capture_mark - rb_launch_count()));
    if (cudaStreamEndCapture(as_stream(stream), &g) != cudaSuccess || !g) return RB_ERR_CUDA;
    cudaGraphExec_t ex = reinterpret_cast<cudaGraphExec_t>(*exec);
    bool ok = false;
    if (ex) {
        cudaGraphExecUpdateResultInfo info;
        ok = cudaGraphExecUpdate(ex, g, &info) == cudaSuccess;
        if (!ok) {
            (void)cudaGetLastError();
            cudaGraphExecDestroy(ex);
            ex = nullptr;
        }
    }
    if (!ok) ok = cudaGraphInstantiate(&ex, g, 0) == cudaSuccess;
    const int kernels = count_kernel_nodes(g);
    cudaGraphDestroy(g);
    if (!ok) {
        *exec = 0;
        return RB_ERR_CUDA;
    }
    *exec = reinterpret_cast<uint64_t>(ex);
    std::lock_guard<std::mutex> lock(g_graph_mu);
    g_graph_kernels[*exec] = kernels;
    return RB_OK;
}

extern "C" int rb_graph_launch(uint64_t exec, void *stream) {
    if (!exec) return RB_ERR_ARGUMENT;
    if (cudaGraphLaunch(reinterpret_cast<cudaGraphExec_t>(exec), as_stream(stream)) != cudaSuccess)
        return RB_ERR_CUDA;
    std::lock_guard<std::mutex> lock(g_graph_mu);
    const auto it = g_graph_kernels.find(exec);
    if (it != g_graph_kernels.end()) note_launches(it->second);
    return RB_OK;
}

extern "C" int rb_graph_destroy(uint64_t exec) {
    if (!exec) return RB_OK;
    {
        std::lock_guard<std::mutex> lock(g_graph_mu);
        g_graph_kernels.erase(exec);
    }
    return cudaGraphExecDestroy(reinterpret_cast<cudaGraphExec_t>(exec)) == cudaSuccess
               ? RB_OK : RB_ERR_CUDA;
}
