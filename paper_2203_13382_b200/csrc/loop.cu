// loop.cu — device-resident MGRIT convergence loop (mgrit.py:355-373).
//
// The reference's solve() checks ||r_k|| against the stop rule on the host
// after every V-cycle.  Here the V-cycle is captured ONCE into the body of a
// CUDA-graph WHILE node, followed by a one-thread check kernel that appends
// r_k to a device history, applies the same stop rule (same fp64 operations
// and comparisons as the Python loop) and clears the node's condition when
// the solve stops.  A whole solve is then one graph launch and one host
// synchronisation at the end instead of a host round trip per iteration.
#include <cmath>
#include <cstdio>

#include "internal.cuh"

namespace mgrit {
namespace {

// ctrl (device int32[4]): [0] completed iterations, [1] state, [2] max_iters
// par  (device double[2]): rtol, divergence_factor
// hist (device double[max_iters + 1]): hist[0] = r0, hist[k] = r_k
__global__ void loop_init_kernel(const double *r0_sumsq, double *hist, int32_t *ctrl, double *par,
                                 double rtol, double divergence_factor, int32_t max_iters) {
    if (threadIdx.x != 0) return;
    hist[0] = sqrt(r0_sumsq[0]);
    ctrl[0] = 0;
    ctrl[1] = MGRIT_LOOP_RUNNING;
    ctrl[2] = max_iters;
    par[0] = rtol;
    par[1] = divergence_factor;
}

__global__ void loop_check_kernel(cudaGraphConditionalHandle h, const double *sumsq, const int32_t *status,
                                  double *hist, int32_t *ctrl, const double *par) {
    if (threadIdx.x != 0) return;
    const int it = ctrl[0] + 1;
    ctrl[0] = it;
    const double r0 = hist[0];
    int state = MGRIT_LOOP_RUNNING;
    if (status[0] != 0) {
        // non-finite GMRES input: the reference raises -> "diverged" (mgrit.py:363-366)
        hist[it] = __longlong_as_double(0x7ff8000000000000LL);
        state = MGRIT_LOOP_DIVERGED;
    } else {
        const double r = sqrt(sumsq[0]);
        hist[it] = r;
        if (!isfinite(r) || r >= __dmul_rn(par[1], r0)) state = MGRIT_LOOP_DIVERGED;
        else if (r <= __dmul_rn(par[0], r0)) state = MGRIT_LOOP_CONVERGED;
        else if (it >= ctrl[2]) state = MGRIT_LOOP_MAX_ITERS;
    }
    ctrl[1] = state;
    cudaGraphSetConditional(h, state == MGRIT_LOOP_RUNNING ? 1u : 0u);
}

struct Loop {
    cudaGraph_t graph = nullptr;
    cudaGraph_t body = nullptr;        // owned by the conditional node
    cudaGraphExec_t exec = nullptr;
    cudaGraphConditionalHandle handle = 0;
    cudaStream_t capture = nullptr;    // stream the body is being captured on
};

int fail(const char *what, cudaError_t e) {
    set_error(what, e);
    return MGRIT_ECUDA;
}

}  // namespace
}  // namespace mgrit

using namespace mgrit;

extern "C" int mgrit_loop_begin(void *stream, void **loop_out) {
    if (!stream || !loop_out) return MGRIT_EINVAL;  // the legacy stream cannot be captured
    *loop_out = nullptr;
    Loop *lp = new Loop();
    cudaError_t e = cudaGraphCreate(&lp->graph, 0);
    if (e == cudaSuccess)
        e = cudaGraphConditionalHandleCreate(&lp->handle, lp->graph, 1u, cudaGraphCondAssignDefault);
    cudaGraphNode_t node;
    cudaGraphNodeParams p = {};
    if (e == cudaSuccess) {
        p.type = cudaGraphNodeTypeConditional;
        p.conditional.handle = lp->handle;
        p.conditional.type = cudaGraphCondTypeWhile;
        p.conditional.size = 1;
        e = cudaGraphAddNode(&node, lp->graph, nullptr, 0, &p);
    }
    if (e == cudaSuccess) {
        lp->body = p.conditional.phGraph_out[0];
        lp->capture = (cudaStream_t)stream;
        // relaxed: API calls the host code makes meanwhile (attribute and
        // occupancy queries, frees) cannot invalidate the capture
        e = cudaStreamBeginCaptureToGraph(lp->capture, lp->body, nullptr, nullptr, 0,
                                          cudaStreamCaptureModeRelaxed);
    }
    if (e != cudaSuccess) {
        if (lp->graph) cudaGraphDestroy(lp->graph);
        delete lp;
        return fail("loop_begin", e);
    }
    *loop_out = lp;
    return MGRIT_OK;
}

extern "C" int mgrit_loop_check(void *loop, const double *sumsq, const int32_t *status, double *hist,
                                int32_t *ctrl, const double *par, void *stream) {
    Loop *lp = (Loop *)loop;
    if (!lp || !sumsq || !status || !hist || !ctrl || !par || (cudaStream_t)stream != lp->capture)
        return MGRIT_EINVAL;
    loop_check_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(lp->handle, sumsq, status, hist, ctrl, par);
    return check_launch("loop_check");
}

extern "C" int mgrit_loop_end(void *loop, void *stream) {
    Loop *lp = (Loop *)loop;
    if (!lp || (cudaStream_t)stream != lp->capture) return MGRIT_EINVAL;
    cudaGraph_t captured = nullptr;
    cudaError_t e = cudaStreamEndCapture(lp->capture, &captured);
    lp->capture = nullptr;
    if (e != cudaSuccess) return fail("loop_end (capture)", e);
    e = cudaGraphInstantiate(&lp->exec, lp->graph, 0);
    if (e != cudaSuccess) return fail("loop_end (instantiate)", e);
    return MGRIT_OK;
}

extern "C" int mgrit_loop_init(const double *r0_sumsq, double *hist, int32_t *ctrl, double *par, double rtol,
                               double divergence_factor, int32_t max_iters, void *stream) {
    if (!r0_sumsq || !hist || !ctrl || !par || max_iters < 1) return MGRIT_EINVAL;
    loop_init_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(r0_sumsq, hist, ctrl, par, rtol, divergence_factor,
                                                         max_iters);
    return check_launch("loop_init");
}

extern "C" int mgrit_loop_launch(void *loop, void *stream) {
    Loop *lp = (Loop *)loop;
    if (!lp || !lp->exec) return MGRIT_EINVAL;
    cudaError_t e = cudaGraphLaunch(lp->exec, (cudaStream_t)stream);
    return e == cudaSuccess ? MGRIT_OK : fail("loop_launch", e);
}

extern "C" void mgrit_loop_destroy(void *loop) {
    Loop *lp = (Loop *)loop;
    if (!lp) return;
    if (lp->capture) {
        // abandon an unfinished capture; the half-built graph is leaked on
        // purpose (destroying a graph whose conditional body capture was
        // invalidated is not safe on every driver)
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(lp->capture, &g);
        cudaGetLastError();
        delete lp;
        return;
    }
    if (lp->exec) cudaGraphExecDestroy(lp->exec);
    if (lp->graph) cudaGraphDestroy(lp->graph);
    delete lp;
}

// Kernel nodes in the captured loop body (one V-cycle + the stop test): the
// kernels one iteration of the device-resident solve launches.  Memset /
// memcpy nodes (2D row copies) are not kernels and are not counted.
extern "C" int64_t mgrit_loop_body_kernels(void *loop) {
    Loop *lp = (Loop *)loop;
    if (!lp || !lp->body || lp->capture) return -1;
    size_t count = 0;
    if (cudaGraphGetNodes(lp->body, nullptr, &count) != cudaSuccess) return -1;
    if (count == 0) return 0;
    cudaGraphNode_t *nodes = new cudaGraphNode_t[count];
    int64_t kernels = 0;
    if (cudaGraphGetNodes(lp->body, nodes, &count) == cudaSuccess) {
        for (size_t i = 0; i < count; ++i) {
            cudaGraphNodeType t;
            if (cudaGraphNodeGetType(nodes[i], &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++kernels;
        }
    } else {
        kernels = -1;
    }
    delete[] nodes;
    return kernels;
}
