// host_common.cuh -- host-side plumbing of the C-ABI: error capture (guard,
// CK, fail -> w1mg_last_error) and the context (stream, workspace buffers,
// cached CUDA graphs, events).  Included once, by capi.cu.
#pragma once

namespace {

thread_local std::string g_err;

struct Fail {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw Fail{code, msg}; }

#define CK(expr)                                                                        \
    do {                                                                                \
        cudaError_t e_ = (expr);                                                        \
        if (e_ != cudaSuccess)                                                          \
            fail(e_ == cudaErrorMemoryAllocation ? W1MG_ENOMEM : W1MG_ECUDA,            \
                 std::string(#expr) + ": " + cudaGetErrorString(e_));                  \
    } while (0)

template <class F>
int guard(F&& f) {
    try {
        f();
        return W1MG_OK;
    } catch (const Fail& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return W1MG_ENOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return W1MG_ECUDA;
    }
}

void check_pnorm(int p) {
    if (p < 0 || p > 2) fail(W1MG_ELOGIC, "bad PNorm");
}
void check_n(int n) {
    if (n < 1) fail(W1MG_EINVAL, "GridSpec: cells_per_side must be positive");
}

}  // namespace

// ---------------------------------------------------------------- context
struct w1mg_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    struct Buf {
        void* p = nullptr;
        size_t bytes = 0;
    };
    std::map<std::string, Buf> bufs;
    std::map<std::string, cudaGraphExec_t> graphs;
    int* pinned = nullptr;  // 2 ints for the done-count pipeline
    cudaEvent_t ev[2] = {nullptr, nullptr};
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    std::vector<cudaEvent_t> lev_ev;  // start/end per level of the last cascade
    int lev_count = 0;
    long launches = 0;
    int num_sms = 148;
    std::map<int, w1mg_dev::DctPlan> dct;  // Poisson DCT plans per m (dct_kernels.cuh)

    void* buf(const std::string& name, size_t bytes) {
        Buf& b = bufs[name];
        if (b.bytes < bytes) {
            if (b.p) {
                CK(cudaFree(b.p));
                // any cached graph may hold the old pointer
                for (auto& g : graphs) cudaGraphExecDestroy(g.second);
                graphs.clear();
            }
            b.p = nullptr;
            b.bytes = 0;
            CK(cudaMalloc(&b.p, bytes));
            b.bytes = bytes;
        }
        return b.p;
    }
    template <class T>
    T* get(const std::string& name, size_t count) {
        return static_cast<T*>(buf(name, count * sizeof(T)));
    }
};
