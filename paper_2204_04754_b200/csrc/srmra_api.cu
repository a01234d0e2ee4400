// srmra_api.cu — the C ABI of libsrmra.so (declared and documented in include/srmra.h).
// Host-side: argument validation, device buffers, path choice, the per-iteration launch
// sequence (prep -> E/M path kernel -> pack -> [NCCL all-reduce] -> finalize/projection) and
// the NCCL communicator (libnccl.so.2 is dlopen'ed on first use, so single-GPU use has no NCCL
// dependency and, inside a PyTorch process, the already-loaded NCCL is reused).
#include <algorithm>
#include <chrono>
#include <dlfcn.h>
#include <unistd.h>
#include <math.h>
#include <nccl.h>
#include <stdio.h>
#include <string.h>

#include <string>
#include <vector>

#include "srmra_internal.cuh"

using namespace srmra;

static thread_local std::string g_init_err;

cudaEvent_t srmra_ctx::prof_event() {
    if (ev_used == ev_pool.size()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        ev_pool.push_back(e);
    }
    return ev_pool[ev_used++];
}

// ---------------------------------------------------------------- NCCL (dlopen)
namespace {
struct NcclApi {
    bool loaded = false;
    std::string err;
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclAllReduce) AllReduce = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
    decltype(&ncclCommGetAsyncError) CommGetAsyncError = nullptr;
    decltype(&ncclCommAbort) CommAbort = nullptr;
};
NcclApi& nccl() {
    static NcclApi api;
    if (!api.loaded && api.err.empty()) {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.err = std::string("cannot dlopen libnccl.so.2: ") + dlerror();
            return api;
        }
        api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
        api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
        api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
        api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
        api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
        api.CommGetAsyncError = (decltype(api.CommGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
        api.CommAbort = (decltype(api.CommAbort))dlsym(h, "ncclCommAbort");
        if (!api.GetUniqueId || !api.CommInitRank || !api.AllReduce || !api.CommDestroy || !api.GetErrorString ||
            !api.CommGetAsyncError || !api.CommAbort)
            api.err = "libnccl.so.2 lacks a required symbol";
        else
            api.loaded = true;
    }
    return api;
}

int fail(srmra_ctx* c, int code, const std::string& msg) {
    if (c) {
        c->err = msg;
        if (code == SRMRA_ERR_CUDA || code == SRMRA_ERR_NCCL) c->failed = true;
    } else {
        g_init_err = msg;
    }
    return code;
}

int cuda_fail(srmra_ctx* c, cudaError_t e, const char* where) {
    std::string m = std::string(where) + ": " + cudaGetErrorString(e);
    if (e == cudaErrorMemoryAllocation) return fail(c, SRMRA_ERR_OOM, m);
    return fail(c, SRMRA_ERR_CUDA, m);
}

#define CK(call)                                                   \
    do {                                                           \
        cudaError_t e_ = (call);                                   \
        if (e_ != cudaSuccess) return cuda_fail(c, e_, #call);     \
    } while (0)

// Wait for the context stream.  With an NCCL communicator the wait polls ncclCommGetAsyncError (SURVEY §5:
// a dead peer must not hang the caller): an asynchronous NCCL error, or opt.nccl_timeout_ms without
// completion, aborts the communicator and fails the context.
int stream_wait(srmra_ctx* c) {
    if (!c->nccl_comm) {
        const cudaError_t e = cudaStreamSynchronize(c->stream);
        return e == cudaSuccess ? SRMRA_OK : cuda_fail(c, e, "cudaStreamSynchronize");
    }
    NcclApi& api = nccl();
    const auto t0 = std::chrono::steady_clock::now();
    for (int spin = 0;; ++spin) {
        const cudaError_t e = cudaStreamQuery(c->stream);
        if (e == cudaSuccess) return SRMRA_OK;
        if (e != cudaErrorNotReady) return cuda_fail(c, e, "cudaStreamQuery");
        ncclResult_t ae = ncclSuccess;
        const ncclResult_t r = api.CommGetAsyncError((ncclComm_t)c->nccl_comm, &ae);
        std::string why;
        if (r != ncclSuccess) why = std::string("ncclCommGetAsyncError: ") + api.GetErrorString(r);
        else if (ae != ncclSuccess && ae != ncclInProgress) why = std::string("NCCL asynchronous error: ") + api.GetErrorString(ae);
        else if (c->opt.nccl_timeout_ms > 0 &&
                 std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count() >
                     c->opt.nccl_timeout_ms)
            why = "stream did not complete within nccl_timeout_ms (peer lost?)";
        if (!why.empty()) {
            api.CommAbort((ncclComm_t)c->nccl_comm);
            c->nccl_comm = nullptr;
            return fail(c, SRMRA_ERR_NCCL, why);
        }
        if (spin > 64) usleep(20);
    }
}

#define SYNC()                                   \
    do {                                         \
        const int rc_ = stream_wait(c);          \
        if (rc_ != SRMRA_OK) return rc_;         \
    } while (0)

template <typename T>
cudaError_t dalloc(T** p, size_t count) {
    if (count == 0) count = 1;
    return cudaMalloc((void**)p, sizeof(T) * count);
}

bool all_finite_f(const float* a, size_t n) {
    for (size_t k = 0; k < n; ++k)
        if (!isfinite(a[k])) return false;
    return true;
}

int check_rho(const double* r, int L, std::vector<double>& out) {
    double s = 0;
    for (int k = 0; k < L; ++k) {
        if (!isfinite(r[k]) || r[k] < 0) return -1;
        s += r[k];
    }
    if (fabs(s - 1.0) > 1e-6) return -1;
    out.resize(L);
    for (int k = 0; k < L; ++k) out[k] = r[k] / s;
    return 0;
}

int choose_path(int requested, int L, int Ll, int K) {
    if (requested == SRMRA_PATH_DIRECT) return direct_supported(L, Ll, K) ? SRMRA_PATH_DIRECT : -1;
    if (requested == SRMRA_PATH_FFT) return fft_supported(L, Ll, K) ? SRMRA_PATH_FFT : -1;
    if (requested == SRMRA_PATH_GEMM) return gemm_supported(L, Ll, K) ? SRMRA_PATH_GEMM : -1;
    // AUTO: measured choice ("Path choice"): FFT < direct < GEMM in time wherever compiled
    if (fft_supported(L, Ll, K)) return SRMRA_PATH_FFT;
    if (direct_supported(L, Ll, K)) return SRMRA_PATH_DIRECT;
    if (gemm_supported(L, Ll, K)) return SRMRA_PATH_GEMM;
    return -1;
}

// The captured FFT iteration bakes in the E/M kernel instantiation: drop it when that changes.
void drop_graphs(srmra_ctx* c) {
    if (c->graph) cudaGraphExecDestroy(c->graph);
    if (c->graph_prof) cudaGraphExecDestroy(c->graph_prof);
    if (c->graph_prof_src) cudaGraphDestroy(c->graph_prof_src);
    c->graph = nullptr;
    c->graph_prof = nullptr;
    c->graph_prof_src = nullptr;
    for (int k = 0; k < 4; ++k) c->prof_nodes[k] = nullptr;
    c->graph_failed = false;
}

// FFT path: switch the E/M kernel between the separable and the joint-prior variant (NEXT-3)
int fft_joint_mode(srmra_ctx* c, bool on) {
    if (c->path != SRMRA_PATH_FFT || c->fft_joint == on) return SRMRA_OK;
    SYNC();
    drop_graphs(c);
    const cudaError_t e = fft_plan_joint(c, on);
    if (e != cudaSuccess) return fail(c, SRMRA_ERR_UNSUPPORTED, std::string("FFT joint-prior plan: ") + cudaGetErrorString(e));
    return SRMRA_OK;
}

// Upload y and theta_0 (host) and run the per-observation init kernels.  ysrc: Y_HOST = host y,
// Y_DEVICE = y already in d_y (srmra_generate), Y_NONE = no observations yet (srmra_init with y NULL:
// d_y zeroed, the context needs srmra_load / srmra_generate before iterating).
enum { Y_HOST = 0, Y_DEVICE = 1, Y_NONE = 2 };
int upload(srmra_ctx* c, const float* y, const float* x0, const std::vector<double>& r1,
           const std::vector<double>& r2, int ysrc = Y_HOST) {
    const size_t ny = (size_t)c->n_local * c->Ll2;
    // pinned caller buffers give an asynchronous DMA; pageable ones are staged by the driver.  FFT path:
    // y goes over in ~4 MB chunks on the copy stream and each chunk's init kernels (||y_i||^2, Yhat_i)
    // run on the context stream as soon as it has landed, overlapping the transfer
    CK(cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));  // before k_ynorm may set bit 1
    const bool chunked = ysrc == Y_HOST && c->path == SRMRA_PATH_FFT && c->copy_stream && ny;
    if (chunked) {
        static const int64_t chunk_bytes = [] {  // ~4 MB per chunk (SRMRA_H2D_CHUNK_MB overrides)
            const char* e = getenv("SRMRA_H2D_CHUNK_MB");
            const int64_t mb = e ? atoll(e) : 4;
            return (mb > 0 ? mb : 4) << 20;
        }();
        const int64_t per = std::max<int64_t>(1, chunk_bytes / (int64_t)(sizeof(float) * c->Ll2));
        for (int64_t o = 0; o < c->n_local; o += per) {
            const int64_t m = std::min<int64_t>(per, c->n_local - o);
            CK(cudaMemcpyAsync(c->d_y + o * c->Ll2, y + o * c->Ll2, sizeof(float) * m * c->Ll2,
                               cudaMemcpyHostToDevice, c->copy_stream));
            CK(cudaEventRecord(c->copy_event, c->copy_stream));
            CK(cudaStreamWaitEvent(c->stream, c->copy_event, 0));  // binds to this record
            CK(launch_init_obs(c, o, m));
            CK(launch_fft_init(c, o, m));
        }
    } else if (ny && ysrc == Y_HOST) {
        CK(cudaMemcpyAsync(c->d_y, y, sizeof(float) * ny, cudaMemcpyHostToDevice, c->stream));
    } else if (ny && ysrc == Y_NONE) {
        CK(cudaMemsetAsync(c->d_y, 0, sizeof(float) * ny, c->stream));
    }
    std::vector<double> x64(c->L2), rho(2 * c->L);
    for (int k = 0; k < c->L2; ++k) x64[k] = (double)x0[k];
    for (int k = 0; k < c->L; ++k) { rho[k] = r1[k]; rho[c->L + k] = r2[k]; }
    CK(cudaMemcpyAsync(c->d_x64, x64.data(), sizeof(double) * c->L2, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_x32, x0, sizeof(float) * c->L2, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_rho, rho.data(), sizeof(double) * 2 * c->L, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemsetAsync(c->d_iter, 0, sizeof(int), c->stream));
    c->joint = false;  // (rho1, rho2): a separable prior again
    {
        const int rcj = fft_joint_mode(c, false);
        if (rcj != SRMRA_OK) return rcj;
    }
    CK(cudaMemsetAsync(c->d_run, 0, 2 * sizeof(int), c->stream));
    CK(cudaMemsetAsync(c->d_rtol, 0, sizeof(double), c->stream));
    c->n_proj = 0;
    if (!chunked) CK(launch_init_obs(c, 0, c->n_local));
    if (c->path == SRMRA_PATH_GEMM) CK(launch_gemm_init(c));
    if (c->path == SRMRA_PATH_FFT) {
        if (!chunked) CK(launch_fft_init(c, 0, c->n_local));
        CK(launch_fft_tail(c, TAIL_PREP));  // Xhat and logit bias of theta_0
    }
    int flag = 0;
    CK(cudaMemcpyAsync(&flag, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    SYNC();  // host vectors above go out of scope
    c->iters_done = 0;
    if (flag & 2) {  // k_ynorm found a non-finite observation value
        c->needs_load = true;
        CK(cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
        return fail(c, SRMRA_ERR_INVALID_ARG, "y not finite");
    }
    c->needs_load = ysrc == Y_NONE && c->n_local > 0;
    return SRMRA_OK;
}

// srmra_load_iterate on the FFT path (one rank, built-in projection): upload y and theta_0 and run the first EM iteration
// with its E/M step split over `stream_chunks` observation ranges — range j's E/M kernel starts as soon as its chunked
// host->device copies and init kernels are done, while range j+1 is still in flight on the copy stream.  Each range
// writes its own per-CTA partial slots; the tail then reduces all of them in its fixed order (the same float64 sums,
// grouped by range).  Same result as upload + one iteration up to the float32 rounding of the per-CTA partials.
int upload_streamed(srmra_ctx* c, const float* y, const float* x0, const std::vector<double>& r1,
                    const std::vector<double>& r2) {
    const int S = c->stream_chunks > 0 ? c->stream_chunks : 8;
    const int PB = fft_partial_bins(c->KK, c->Ll);
    const size_t slots = (size_t)S * c->fft_grid;
    if (!c->d_part_s || c->stream_chunks != S) {
        if (c->d_part_s) cudaFree(c->d_part_s);
        if (c->d_llpart_s) cudaFree(c->d_llpart_s);
        c->d_part_s = nullptr;
        c->d_llpart_s = nullptr;
        if (dalloc(&c->d_part_s, slots * PB) != cudaSuccess || dalloc(&c->d_llpart_s, slots) != cudaSuccess) {
            cudaGetLastError();
            return fail(c, SRMRA_ERR_OOM, "srmra_load_iterate: partial slots");
        }
        c->stream_chunks = S;
    }
    CK(cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
    std::vector<double> x64(c->L2), rho(2 * c->L);
    for (int k = 0; k < c->L2; ++k) x64[k] = (double)x0[k];
    for (int k = 0; k < c->L; ++k) { rho[k] = r1[k]; rho[c->L + k] = r2[k]; }
    CK(cudaMemcpyAsync(c->d_x64, x64.data(), sizeof(double) * c->L2, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_x32, x0, sizeof(float) * c->L2, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_rho, rho.data(), sizeof(double) * 2 * c->L, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemsetAsync(c->d_iter, 0, sizeof(int), c->stream));
    c->joint = false;
    {
        const int rcj = fft_joint_mode(c, false);
        if (rcj != SRMRA_OK) return rcj;
    }
    CK(cudaMemsetAsync(c->d_run, 0, 2 * sizeof(int), c->stream));
    CK(cudaMemsetAsync(c->d_rtol, 0, sizeof(double), c->stream));
    c->n_proj = 0;
    CK(launch_fft_tail(c, TAIL_PREP));  // Xhat and logit bias of theta_0, before the first range's E/M kernel
    static const int64_t chunk_bytes = [] {
        const char* e = getenv("SRMRA_H2D_CHUNK_MB");
        const int64_t mb = e ? atoll(e) : 4;
        return (mb > 0 ? mb : 4) << 20;
    }();
    const int64_t per = std::max<int64_t>(1, chunk_bytes / (int64_t)(sizeof(float) * c->Ll2));
    const int64_t range = (c->n_local + S - 1) / S;
    for (int j = 0; j < S; ++j) {
        const int64_t r0 = j * range, r1e = std::min<int64_t>(c->n_local, r0 + range);
        float2* part = c->d_part_s + (size_t)j * c->fft_grid * PB;
        double* llp = c->d_llpart_s + (size_t)j * c->fft_grid;
        for (int64_t o = r0; o < r1e; o += per) {
            const int64_t m = std::min<int64_t>(per, r1e - o);
            CK(cudaMemcpyAsync(c->d_y + o * c->Ll2, y + o * c->Ll2, sizeof(float) * m * c->Ll2, cudaMemcpyHostToDevice,
                               c->copy_stream));
            CK(cudaEventRecord(c->copy_event, c->copy_stream));
            CK(cudaStreamWaitEvent(c->stream, c->copy_event, 0));
            CK(launch_init_obs(c, o, m));
            CK(launch_fft_init(c, o, m));
        }
        c->em_off = r0;
        c->em_n = std::max<int64_t>(0, r1e - r0);
        c->em_part = part;
        c->em_llpart = llp;
        const cudaError_t e = c->em_n > 0 ? launch_fft_em(c) : cudaSuccess;
        c->em_n = -1;
        if (e != cudaSuccess) return cuda_fail(c, e, "launch_fft_em (range)");
        if (r1e <= r0) {  // an empty range still owns slots the tail reads
            CK(cudaMemsetAsync(part, 0, sizeof(float2) * (size_t)c->fft_grid * PB, c->stream));
            CK(cudaMemsetAsync(llp, 0, sizeof(double) * c->fft_grid, c->stream));
        }
    }
    c->tail_part = c->d_part_s;
    c->tail_llpart = c->d_llpart_s;
    c->tail_nparts = (int)slots;
    const cudaError_t et = launch_fft_tail(c, TAIL_REDUCE | TAIL_FOLD | TAIL_FINALIZE | TAIL_PREP);
    c->tail_nparts = 0;
    if (et != cudaSuccess) return cuda_fail(c, et, "launch_fft_tail (streamed)");
    int flag = 0;
    CK(cudaMemcpyAsync(&flag, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    SYNC();
    c->iters_done = 1;
    if (flag & 2) {
        c->needs_load = true;
        CK(cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
        return fail(c, SRMRA_ERR_INVALID_ARG, "y not finite");
    }
    c->needs_load = false;
    return SRMRA_OK;
}

// Sum a device float64 buffer over all ranks on the context stream: the options' exchange provider if
// one is set, else ncclAllReduce (no-op for world 1).
int exchange(srmra_ctx* c, double* buf, size_t n) {
    if (c->opt.world <= 1 || n == 0) return SRMRA_OK;
    if (c->opt.allreduce) {
        if (c->opt.allreduce(buf, (uint64_t)n, (void*)c->stream, c->opt.allreduce_user) != 0)
            return fail(c, SRMRA_ERR_NCCL, "exchange provider (srmra_options.allreduce) failed");
        return SRMRA_OK;
    }
    NcclApi& api = nccl();
    ncclResult_t r = api.AllReduce(buf, buf, n, ncclFloat64, ncclSum, (ncclComm_t)c->nccl_comm, c->stream);
    if (r != ncclSuccess) return fail(c, SRMRA_ERR_NCCL, std::string("ncclAllReduce: ") + api.GetErrorString(r));
    return SRMRA_OK;
}

// The one data-path collective: sum this rank's sufficient statistics over all ranks.
// FFT path: the compact float64 accumulators (U, V, row sums, pair line, LL) — the fold after it is
// linear, so fold(sum) = sum(fold) — plus, with a joint prior, the per-shift posterior mass;
// GEMM / direct paths: the packed b | class mass | marginals | LL, and with a joint prior the per-shift
// posterior mass colsum that finalize divides by the global total (d_colsum sits right after the pack,
// so it is the same single collective).
int allreduce_stats(srmra_ctx* c) {
    if (c->opt.world <= 1) return SRMRA_OK;
    if (c->path != SRMRA_PATH_FFT)
        return exchange(c, c->d_pack, (size_t)c->pk.total + (c->joint ? (size_t)c->L2 : 0));
    int rc = exchange(c, c->d_bhat, fft_bhat_doubles(c->KK, c->Ll));
    if (rc == SRMRA_OK && c->fft_joint) rc = exchange(c, c->d_jacc, fft_joint_bins(c->KK, c->Ll));
    return rc;
}


// A converged srmra_run leaves the device stop flag set, which makes the E/M and tail kernels return at
// once (so that the remaining enqueued replays are no-ops).  Every launch outside iterate() clears it first.
int clear_stop(srmra_ctx* c) {
    CK(cudaMemsetAsync(c->d_run, 0, sizeof(int), c->stream));
    return SRMRA_OK;
}

int record(srmra_ctx* c) {
    if (!c->prof || c->path == SRMRA_PATH_FFT) return SRMRA_OK;  // FFT: the E/M kernel stamps itself
    cudaEvent_t e = c->prof_event();
    if (!e) return fail(c, SRMRA_ERR_CUDA, "cudaEventCreate failed");
    CK(cudaEventRecord(e, c->stream));
    return SRMRA_OK;
}

// E + M over the local shard at the current theta, up to the (local) sufficient statistics:
// FFT path: the E/M kernel only (the previous tail, or the load-time tail, already prepared Xhat and
// the logit bias; the reduce is the first phase of the tail); direct: prep, E/M, pack.
// With profiling on, events bracket the dominant E/M kernel (records 2 and 3 of the quadruple).
int local_estep_mstep(srmra_ctx* c) {
    int rc;
    if (c->path == SRMRA_PATH_FFT) {
        if ((rc = record(c))) return rc;
        CK(launch_fft_em(c));
        if ((rc = record(c))) return rc;
    } else if (c->path == SRMRA_PATH_GEMM) {
        CK(launch_prep(c));
        if ((rc = record(c))) return rc;
        CK(launch_gemm_em(c, nullptr, nullptr));  // x copies, GEMM1, softmax, GEMM2, fold
        if ((rc = record(c))) return rc;
        CK(launch_pack(c));
    } else if (c->path == SRMRA_PATH_DIRECT) {
        CK(launch_prep(c));
        if ((rc = record(c))) return rc;
        CK(launch_direct_em(c));
        if ((rc = record(c))) return rc;
        CK(launch_pack(c));
    } else {
        return fail(c, SRMRA_ERR_UNSUPPORTED, "path not available");
    }
    return SRMRA_OK;
}


// Run control of the FFT graph path: stop flag, first iteration of the run, tolerance (0 = none).
int set_run_control(srmra_ctx* c, double rel_tol) {
    c->h_run[0] = 0;
    c->h_run[1] = c->iters_done;
    c->h_rtol = rel_tol > 0 ? rel_tol : 0.0;
    // pageable sources: the copies are staged before the calls return
    CK(cudaMemcpyAsync(c->d_run, c->h_run, 2 * sizeof(int), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_rtol, &c->h_rtol, sizeof(double), cudaMemcpyHostToDevice, c->stream));
    return SRMRA_OK;
}

// After a denoiser hook replaced x64: the float32 copy and (FFT path) the next iteration's spectra
int refresh_after_denoise(srmra_ctx* c) {
    if (c->path == SRMRA_PATH_FFT) CK(launch_fft_tail(c, TAIL_PREP));  // also writes x32
    else CK(launch_x32_from_x64(c));
    return SRMRA_OK;
}

// n_iters EM iterations of Algorithm 2 (srmra_em_iter: rel_tol = 0; srmra_run: the stopping rule)
int iterate(srmra_ctx* c, int32_t n_iters, double rel_tol) {
    // one rank, or NCCL ranks (every rank records the same all-reduced LL_t, so the device stopping rule
    // takes the same decision everywhere); a host exchange provider or a denoiser hook needs the host loop
    const bool device_loop = c->path == SRMRA_PATH_FFT && !c->denoiser && (c->opt.world == 1 || !c->opt.allreduce);
    int rc;
    if ((rc = set_run_control(c, device_loop ? rel_tol : 0.0)) != SRMRA_OK) return rc;
    // FFT path: replay a captured CUDA graph of one iteration (E/M kernel + cooperative tail; world > 1:
    // E/M kernel, reduce-only tail, ncclAllReduce, fold / finalize / prep tail); the tail takes t and the
    // projection flag from the device counter.  With profiling on, the
    // graph variant carries 4 event-record nodes that are re-pointed to fresh pool events per replay.
    if (device_loop && !c->graph_failed && n_iters > 0) {
        cudaGraphExec_t* exec = &c->graph;  // profiling needs no event nodes: the E/M kernel stamps itself
        if (!*exec) {
            cudaGraph_t g = nullptr;
            cudaEvent_t ph[4] = {nullptr, nullptr, nullptr, nullptr};
            bool ok = true;
            const bool prof_nodes = false;
            if (prof_nodes)
                for (int k = 0; k < 4 && ok; ++k) ok = cudaEventCreate(&ph[k]) == cudaSuccess;
            ok = ok && cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
            if (ok) {
                bool l = true;
                if (prof_nodes) l = l && cudaEventRecordWithFlags(ph[0], c->stream, cudaEventRecordExternal) == cudaSuccess;
                if (prof_nodes) l = l && cudaEventRecordWithFlags(ph[1], c->stream, cudaEventRecordExternal) == cudaSuccess;
                l = l && launch_fft_em(c) == cudaSuccess;
                if (prof_nodes) l = l && cudaEventRecordWithFlags(ph[2], c->stream, cudaEventRecordExternal) == cudaSuccess;
                if (c->opt.world > 1) {
                    l = l && launch_fft_tail(c, TAIL_REDUCE) == cudaSuccess;
                    l = l && allreduce_stats(c) == SRMRA_OK;
                    l = l && launch_fft_tail(c, TAIL_FOLD | TAIL_FINALIZE | TAIL_PREP) == cudaSuccess;
                } else {
                    l = l && launch_fft_tail(c, TAIL_REDUCE | TAIL_FOLD | TAIL_FINALIZE | TAIL_PREP) == cudaSuccess;
                }
                if (prof_nodes) l = l && cudaEventRecordWithFlags(ph[3], c->stream, cudaEventRecordExternal) == cudaSuccess;
                ok = cudaStreamEndCapture(c->stream, &g) == cudaSuccess && l;
            }
            if (ok && prof_nodes) {  // find the event-record nodes by their placeholder events
                size_t nn = 0;
                ok = cudaGraphGetNodes(g, nullptr, &nn) == cudaSuccess;
                std::vector<cudaGraphNode_t> nodes(nn);
                ok = ok && cudaGraphGetNodes(g, nodes.data(), &nn) == cudaSuccess;
                for (size_t k = 0; ok && k < nn; ++k) {
                    cudaGraphNodeType ty;
                    if (cudaGraphNodeGetType(nodes[k], &ty) != cudaSuccess || ty != cudaGraphNodeTypeEventRecord) continue;
                    cudaEvent_t ev;
                    if (cudaGraphEventRecordNodeGetEvent(nodes[k], &ev) != cudaSuccess) continue;
                    for (int j = 0; j < 4; ++j)
                        if (ev == ph[j]) c->prof_nodes[j] = nodes[k];
                }
                for (int j = 0; j < 4; ++j) ok = ok && c->prof_nodes[j] != nullptr;
            }
            if (ok) ok = cudaGraphInstantiate(exec, g, 0) == cudaSuccess;
            // the profiling variant keeps its graph: exec-node updates refer to the graph's node handles
            if (g && ok && prof_nodes) c->graph_prof_src = g;
            else if (g) cudaGraphDestroy(g);
            if (!ok) {
                cudaGetLastError();  // clear the capture error; stream launches are used instead
                *exec = nullptr;
                c->graph_failed = true;
                c->failed = false;   // an NCCL call refused under capture is not a context failure
                c->err.clear();
            }
            // placeholders must outlive the exec (destroying them invalidates its event-record nodes)
            for (int k = 0; k < 4; ++k) {
                if (ok && prof_nodes) c->prof_ph[k] = ph[k];
                else if (ph[k]) cudaEventDestroy(ph[k]);
            }
        }
        if (*exec) {
            if (rel_tol > 0) c->iters_stale = true;  // the device may stop before n_iters
            for (int it = 0; it < n_iters; ++it) {
                CK(cudaGraphLaunch(*exec, c->stream));
                c->iters_done++;
            }
            return SRMRA_OK;
        }
    }
    const int t0 = c->iters_done;
    for (int it = 0; it < n_iters; ++it) {
        const int t = c->iters_done;
        if ((rc = record(c)) != SRMRA_OK) return rc;
        if ((rc = local_estep_mstep(c)) != SRMRA_OK) return rc;
        const int F = c->opt.proj_every;
        const bool proj_step = F > 0 && ((t + 1) % F == 0);
        const int project = proj_step && !c->denoiser;  // the built-in stand-in projection
        if (c->path == SRMRA_PATH_FFT) {
            // reduce -> [all-reduce] -> fold / update -> projection / next prep: one cooperative kernel
            // (two when the NCCL all-reduce has to sit between the reduce and the fold)
            const int rest = TAIL_FOLD | TAIL_FINALIZE | TAIL_PREP;
            if (c->opt.world > 1) {
                CK(launch_fft_tail(c, TAIL_REDUCE));
                if ((rc = allreduce_stats(c)) != SRMRA_OK) return rc;
                CK(launch_fft_tail(c, rest));
            } else {
                CK(launch_fft_tail(c, TAIL_REDUCE | rest));
            }
        } else {
            if ((rc = allreduce_stats(c)) != SRMRA_OK) return rc;
            CK(launch_finalize(c, t, project));
        }
        if ((rc = record(c)) != SRMRA_OK) return rc;
        c->iters_done++;
        if (proj_step && c->denoiser) {  // Algorithm 2: x <- D(x, sigma_j), sigma_j = 2^(-(j-1)/10)
            const double sig = pow(2.0, -(double)(c->n_proj++) / 10.0);
            if (c->denoiser(c->d_x64, c->L, sig, (void*)c->stream, c->denoiser_user) != 0)
                return fail(c, SRMRA_ERR_NUMERIC, "denoiser hook failed");
            if ((rc = refresh_after_denoise(c)) != SRMRA_OK) return rc;
        }
        if (rel_tol > 0 && t - t0 >= 1 && t < c->opt.trace_cap) {  // host-side stopping rule
            double ll[2];
            CK(cudaMemcpyAsync(ll, c->d_trace + (t - 1), 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
            SYNC();
            if (fabs(ll[1] - ll[0]) <= rel_tol * fabs(ll[1])) break;
        }
    }
    return SRMRA_OK;
}

// Iterations actually run: the FFT tail's device counter is authoritative (a converged srmra_run
// turns the remaining enqueued iterations into no-ops); other paths count on the host.
int sync_iters(srmra_ctx* c) {
    if (c->path == SRMRA_PATH_FFT) {
        int t = 0;
        CK(cudaMemcpyAsync(&t, c->d_iter, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        SYNC();
        c->iters_done = t;
    }
    c->iters_stale = false;
    return SRMRA_OK;
}

}  // namespace

// ==================================================================== ABI
namespace srmra {
// NCCL sum of a device float64 buffer over all ranks, on the context stream (no-op for world 1);
// the moments call (k_moments.cu) uses it for its raw sums.
int allreduce_doubles(srmra_ctx* c, double* buf, size_t n) { return exchange(c, buf, n); }
}  // namespace srmra

namespace {
// Every call on a context runs on the context's device and restores the caller's current device
// (a process may hold contexts on several GPUs).
struct DevGuard {
    int prev = -1;
    explicit DevGuard(const srmra_ctx* c) {
        int cur = -1;
        if (c && cudaGetDevice(&cur) == cudaSuccess && cur != c->device && cudaSetDevice(c->device) == cudaSuccess)
            prev = cur;
    }
    ~DevGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};
}  // namespace

extern "C" {

void srmra_default_options(srmra_options* o) {
    if (!o) return;
    memset(o, 0, sizeof(*o));
    o->path = SRMRA_PATH_AUTO;
    o->proj_every = 1;
    o->floor_tau = -1.0;
    o->device = -1;
    o->rank = 0;
    o->world = 1;
    o->nccl_id = nullptr;
    o->stream = nullptr;
    o->trace_cap = 4096;
    o->allreduce = nullptr;
    o->allreduce_user = nullptr;
    o->grid_cap = 0;
    o->nccl_timeout_ms = 0;
}

const char* srmra_last_error(const srmra_ctx* ctx) { return ctx ? ctx->err.c_str() : g_init_err.c_str(); }

int srmra_nccl_unique_id(void* out128) {
    if (!out128) return fail(nullptr, SRMRA_ERR_INVALID_ARG, "out128 is NULL");
    NcclApi& api = nccl();
    if (!api.loaded) return fail(nullptr, SRMRA_ERR_NCCL, api.err);
    ncclUniqueId id;
    ncclResult_t r = api.GetUniqueId(&id);
    if (r != ncclSuccess) return fail(nullptr, SRMRA_ERR_NCCL, api.GetErrorString(r));
    memcpy(out128, &id, sizeof(id));
    return SRMRA_OK;
}

int srmra_init(srmra_ctx** out, const float* y, int32_t n_local, int32_t L_high, int32_t L_low, int32_t K,
               double sigma, const float* x0, const double* rho1_0, const double* rho2_0,
               const srmra_options* opt_in) {
    srmra_ctx* c = nullptr;  // errors before the context exists go to g_init_err
    if (!out) return fail(c, SRMRA_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    srmra_options opt;
    srmra_default_options(&opt);
    if (opt_in) opt = *opt_in;
    if (L_high <= 0 || L_low <= 0 || K <= 0 || n_local < 0)
        return fail(c, SRMRA_ERR_INVALID_ARG, "sizes must be positive (n_local >= 0)");
    if ((int64_t)K * L_low != L_high) return fail(c, SRMRA_ERR_INVALID_ARG, "K * L_low != L_high");
    if (!(sigma > 0) || !isfinite(sigma)) return fail(c, SRMRA_ERR_INVALID_ARG, "sigma must be finite and > 0");
    if (!x0 || !rho1_0 || !rho2_0) return fail(c, SRMRA_ERR_INVALID_ARG, "NULL input");
    if (opt.world < 1 || opt.rank < 0 || opt.rank >= opt.world) return fail(c, SRMRA_ERR_INVALID_ARG, "bad rank/world");
    if (opt.world > 1 && !opt.nccl_id && !opt.allreduce)
        return fail(c, SRMRA_ERR_INVALID_ARG, "world > 1 needs nccl_id or an exchange provider (allreduce)");
    if (opt.proj_every < 0) return fail(c, SRMRA_ERR_INVALID_ARG, "proj_every < 0");
    if (opt.trace_cap < 1) opt.trace_cap = 4096;
    if (!all_finite_f(x0, (size_t)L_high * L_high)) return fail(c, SRMRA_ERR_INVALID_ARG, "x0 not finite");
    std::vector<double> r1, r2;
    if (check_rho(rho1_0, L_high, r1) || check_rho(rho2_0, L_high, r2))
        return fail(c, SRMRA_ERR_INVALID_ARG, "rho must be >= 0, finite and sum to 1 (within 1e-6)");
    if (K * K > 256 || L_high > 4096) return fail(c, SRMRA_ERR_UNSUPPORTED, "K^2 > 256 or L_high > 4096");
    const int path = choose_path(opt.path, L_high, L_low, K);
    if (path < 0) return fail(c, SRMRA_ERR_UNSUPPORTED, "no compiled path supports this shape / path request");

    int dev = opt.device;
    cudaError_t ce;
    if (dev < 0) {
        if ((ce = cudaGetDevice(&dev)) != cudaSuccess) return cuda_fail(c, ce, "cudaGetDevice");
    }
    cudaDeviceProp prop;
    if ((ce = cudaGetDeviceProperties(&prop, dev)) != cudaSuccess) return cuda_fail(c, ce, "cudaGetDeviceProperties");
    if (prop.major != 10 || prop.minor != 0)
        return fail(c, SRMRA_ERR_UNSUPPORTED, "libsrmra is built for sm_100a (B200); device is sm_" +
                                                  std::to_string(prop.major) + std::to_string(prop.minor));
    if ((ce = cudaSetDevice(dev)) != cudaSuccess) return cuda_fail(c, ce, "cudaSetDevice");

    c = new srmra_ctx();
    c->opt = opt;
    c->device = dev;
    c->num_sms = prop.multiProcessorCount;
    {  // stream-ordered temporaries (moments, evaluation) are reused across calls instead of returned to the OS
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
    c->L = L_high; c->Ll = L_low; c->K = K; c->KK = K * K;
    c->L2 = L_high * L_high; c->Ll2 = L_low * L_low; c->Lh = L_low / 2 + 1;
    c->n_local = n_local;
    c->sigma = sigma;
    c->inv_s2 = 1.0 / (sigma * sigma);
    c->inv_2s2 = 0.5 / (sigma * sigma);
    c->path = path;
    c->pk.b = 0;
    c->pk.cmass = c->L2;
    c->pk.m1 = c->pk.cmass + c->KK;
    c->pk.m2 = c->pk.m1 + c->L;
    c->pk.ll = c->pk.m2 + c->L;
    c->pk.total = c->pk.ll + 1;

    auto bail = [&](int code) { g_init_err = c->err; srmra_free(c); return code; };
    int rc;
#define CKI(call)                                                                   \
    do {                                                                            \
        cudaError_t e_ = (call);                                                    \
        if (e_ != cudaSuccess) return bail(cuda_fail(c, e_, #call));               \
    } while (0)

    if (opt.stream) {
        c->stream = (cudaStream_t)opt.stream;
    } else {
        CKI(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
    }
    if (path == SRMRA_PATH_FFT) {
        CKI(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        CKI(cudaEventCreateWithFlags(&c->copy_event, cudaEventDisableTiming));
    }
    const size_t ny = (size_t)n_local * c->Ll2;
    CKI(dalloc(&c->d_y, ny));
    CKI(dalloc(&c->d_ynorm, n_local));
    CKI(dalloc(&c->d_llobs, n_local));
    CKI(dalloc(&c->d_x64, c->L2));
    CKI(dalloc(&c->d_x32, c->L2));
    CKI(dalloc(&c->d_xtmp, c->L2));
    CKI(dalloc(&c->d_rho, 2 * c->L));
    CKI(dalloc(&c->par.f32, 2 * c->L + c->KK));
    CKI(dalloc(&c->par.f64, 2 * c->KK + 2));
    CKI(cudaMemset(c->par.f64, 0, sizeof(double) * (2 * c->KK + 2)));
    // pack | colsum in one buffer: with a joint prior both are all-reduced by one collective
    CKI(dalloc(&c->d_pack, c->pk.total + c->L2));
    c->d_colsum = c->d_pack + c->pk.total;
    CKI(dalloc(&c->d_trace, opt.trace_cap));
    CKI(dalloc(&c->d_flag, 1));
    CKI(dalloc(&c->d_counter, 1));
    CKI(cudaMemset(c->d_counter, 0, sizeof(unsigned)));
    CKI(dalloc(&c->d_iter, 1));
    CKI(dalloc(&c->d_emt, 2 * (size_t)opt.trace_cap));
    CKI(cudaMemset(c->d_emt, 0, sizeof(unsigned long long) * 2 * (size_t)opt.trace_cap));
    CKI(dalloc(&c->d_run, 2));
    CKI(cudaMemset(c->d_run, 0, 2 * sizeof(int)));
    CKI(dalloc(&c->d_rtol, 1));
    CKI(cudaMemset(c->d_rtol, 0, sizeof(double)));
    if (getenv("SRMRA_TAIL_STAMPS")) {
        CKI(dalloc(&c->d_stamps, 16));
        CKI(cudaMemset(c->d_stamps, 0, 16 * sizeof(unsigned long long)));
    }
    if (path == SRMRA_PATH_FFT) {
        CKI(dalloc(&c->d_yhat, (size_t)n_local * fft_yhat_stride(c->Ll)));
        CKI(dalloc(&c->d_ysum, n_local));
        CKI(dalloc(&c->d_xhat, fft_xhat_float2(c->KK, c->Ll)));
        CKI(cudaMemset(c->d_xhat, 0, sizeof(float2) * fft_xhat_float2(c->KK, c->Ll)));
        CKI(dalloc(&c->d_bhat, fft_bhat_doubles(c->KK, c->Ll)));
        if (c->Ll == 128) CKI(dalloc(&c->d_xcoef, fft128_coef_float4(c->KK)));
        CKI(fft_plan(c));
        std::vector<double> tw(2 * (size_t)c->Ll);  // cos / sin (2 pi j / L_low), float64
        for (int j = 0; j < c->Ll; ++j) {
            tw[j] = cos(2.0 * M_PI * j / c->Ll);
            tw[c->Ll + j] = sin(2.0 * M_PI * j / c->Ll);
        }
        CKI(dalloc(&c->d_tw, tw.size()));
        CKI(cudaMemcpy(c->d_tw, tw.data(), sizeof(double) * tw.size(), cudaMemcpyHostToDevice));
        CKI(dalloc(&c->d_part, fft_part_float2(c)));
        CKI(dalloc(&c->d_llpart, c->fft_grid));
    }
    if (path == SRMRA_PATH_GEMM) {
        size_t fr = 0, tot = 0;
        CKI(cudaMemGetInfo(&fr, &tot));
        if (gemm_bytes(c) + (size_t)(1u << 30) > fr)
            return bail(fail(c, SRMRA_ERR_OOM, "gemm path: scores / posterior buffers exceed free device memory"));
        CKI(gemm_alloc(c));
    }
    CKI(cudaMemsetAsync(c->d_llobs, 0, sizeof(double) * (n_local ? n_local : 1), c->stream));

    // global N and the NCCL communicator
    c->n_global = n_local;
    if (opt.world > 1) {
        if (!opt.allreduce) {
            NcclApi& api = nccl();
            if (!api.loaded) return bail(fail(c, SRMRA_ERR_NCCL, api.err));
            ncclUniqueId id;
            memcpy(&id, opt.nccl_id, sizeof(id));
            ncclComm_t comm;
            ncclResult_t r = api.CommInitRank(&comm, opt.world, id, opt.rank);
            if (r != ncclSuccess) return bail(fail(c, SRMRA_ERR_NCCL, std::string("ncclCommInitRank: ") + api.GetErrorString(r)));
            c->nccl_comm = comm;
        }
        double* d_n = c->d_pack;  // scratch for the one-off N all-reduce
        double hn = (double)n_local;
        CKI(cudaMemcpyAsync(d_n, &hn, sizeof(double), cudaMemcpyHostToDevice, c->stream));
        if ((rc = exchange(c, d_n, 1)) != SRMRA_OK) return bail(rc);
        CKI(cudaMemcpyAsync(&hn, d_n, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        if ((rc = stream_wait(c)) != SRMRA_OK) return bail(rc);
        c->n_global = (int64_t)llround(hn);
    }
    c->tau = opt.floor_tau >= 0 ? opt.floor_tau : 1e-12 * (double)c->n_global;

    if ((rc = upload(c, y, x0, r1, r2, y ? Y_HOST : Y_NONE)) != SRMRA_OK) return bail(rc);
    *out = c;
    return SRMRA_OK;
}

int srmra_load(srmra_ctx* c, const float* y, const float* x0, const double* rho1_0, const double* rho2_0) {
    DevGuard dg_(c);
    if (!c) return fail(nullptr, SRMRA_ERR_INVALID_ARG, "ctx is NULL");
    if (c->failed) return SRMRA_ERR_STATE;
    if (!x0 || !rho1_0 || !rho2_0 || (c->n_local > 0 && !y)) return fail(c, SRMRA_ERR_INVALID_ARG, "NULL input");
    if (!all_finite_f(x0, (size_t)c->L2)) return fail(c, SRMRA_ERR_INVALID_ARG, "x0 not finite");
    std::vector<double> r1, r2;
    if (check_rho(rho1_0, c->L, r1) || check_rho(rho2_0, c->L, r2))
        return fail(c, SRMRA_ERR_INVALID_ARG, "rho must be >= 0, finite and sum to 1 (within 1e-6)");
    return upload(c, y, x0, r1, r2);
}

int srmra_load_iterate(srmra_ctx* c, const float* y, const float* x0, const double* rho1_0, const double* rho2_0,
                       int32_t n_iters) {
    DevGuard dg_(c);
    if (!c) return fail(nullptr, SRMRA_ERR_INVALID_ARG, "ctx is NULL");
    if (c->failed) return SRMRA_ERR_STATE;
    if (n_iters < 0) return fail(c, SRMRA_ERR_INVALID_ARG, "n_iters < 0");
    if (!x0 || !rho1_0 || !rho2_0 || (c->n_local > 0 && !y)) return fail(c, SRMRA_ERR_INVALID_ARG, "NULL input");
    if (!all_finite_f(x0, (size_t)c->L2)) return fail(c, SRMRA_ERR_INVALID_ARG, "x0 not finite");
    std::vector<double> r1, r2;
    if (check_rho(rho1_0, c->L, r1) || check_rho(rho2_0, c->L, r2))
        return fail(c, SRMRA_ERR_INVALID_ARG, "rho must be >= 0, finite and sum to 1 (within 1e-6)");
    // the streamed first iteration: FFT path, one rank, the built-in projection (a denoiser hook or a host exchange
    // needs the host loop around every iteration)
    const bool streamed = n_iters > 0 && c->path == SRMRA_PATH_FFT && c->copy_stream && c->n_local > 0 &&
                          c->opt.world == 1 && !c->denoiser;
    int rc;
    if (!streamed) {
        if ((rc = upload(c, y, x0, r1, r2)) != SRMRA_OK) return rc;
        return n_iters > 0 ? iterate(c, n_iters, 0.0) : SRMRA_OK;
    }
    if ((rc = upload_streamed(c, y, x0, r1, r2)) != SRMRA_OK) return rc;
    return n_iters > 1 ? iterate(c, n_iters - 1, 0.0) : SRMRA_OK;
}

int srmra_generate(srmra_ctx* c, const float* x_true, const double* rho1_true, const double* rho2_true, uint64_t seed,
                   int64_t first_index, const float* x0, const double* rho1_0, const double* rho2_0,
                   int32_t* shifts_out) {
    DevGuard dg_(c);
    if (!c) return fail(nullptr, SRMRA_ERR_INVALID_ARG, "ctx is NULL");
    if (c->failed) return SRMRA_ERR_STATE;
    if (!x_true || !rho1_true || !rho2_true || !x0 || !rho1_0 || !rho2_0)
        return fail(c, SRMRA_ERR_INVALID_ARG, "NULL input");
    if (first_index < 0) return fail(c, SRMRA_ERR_INVALID_ARG, "first_index < 0");
    if (!all_finite_f(x_true, (size_t)c->L2) || !all_finite_f(x0, (size_t)c->L2))
        return fail(c, SRMRA_ERR_INVALID_ARG, "x_true / x0 not finite");
    std::vector<double> t1, t2, r1, r2;
    if (check_rho(rho1_true, c->L, t1) || check_rho(rho2_true, c->L, t2) || check_rho(rho1_0, c->L, r1) ||
        check_rho(rho2_0, c->L, r2))
        return fail(c, SRMRA_ERR_INVALID_ARG, "rho must be >= 0, finite and sum to 1 (within 1e-6)");
    // inverse-CDF tables: sequential float64 partial sums of the caller's pmfs (as given, not renormalised)
    std::vector<double> cdf(2 * c->L);
    int last[2] = {0, 0};
    for (int a = 0; a < 2; ++a) {
        const double* r = a ? rho2_true : rho1_true;
        double s = 0.0;
        for (int k = 0; k < c->L; ++k) {
            s += r[k];
            cdf[a * c->L + k] = s;
            if (r[k] > 0) last[a] = k;
        }
    }
    const size_t bytes = sizeof(float) * c->L2 + sizeof(double) * 2 * c->L + sizeof(int) * 2 * (size_t)c->n_local;
    unsigned char* tmp = nullptr;
    CK(cudaMallocAsync(&tmp, bytes, c->stream));
    double* d_cdf = reinterpret_cast<double*>(tmp);
    float* d_x = reinterpret_cast<float*>(tmp + sizeof(double) * 2 * c->L);
    int* d_sh = reinterpret_cast<int*>(tmp + sizeof(double) * 2 * c->L + sizeof(float) * c->L2);
    cudaError_t e = cudaMemcpyAsync(d_cdf, cdf.data(), sizeof(double) * 2 * c->L, cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_x, x_true, sizeof(float) * c->L2, cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess) e = launch_generate(c, d_x, d_cdf, last[0], last[1], seed, first_index, shifts_out ? d_sh : nullptr);
    if (e == cudaSuccess && shifts_out && c->n_local > 0)
        e = cudaMemcpyAsync(shifts_out, d_sh, sizeof(int) * 2 * (size_t)c->n_local, cudaMemcpyDeviceToHost, c->stream);
    cudaFreeAsync(tmp, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);  // host tables go out of scope
    if (e != cudaSuccess) return cuda_fail(c, e, "srmra_generate");
    return upload(c, nullptr, x0, r1, r2, Y_DEVICE);
}

int srmra_get_observations(srmra_ctx* c, int64_t first, int64_t count, float* y_out) {
    DevGuard dg_(c);
    if (!c) return fail(nullptr, SRMRA_ERR_INVALID_ARG, "ctx is NULL");
    if (c->failed) return SRMRA_ERR_STATE;
    if (first < 0 || count < 0 || first + count > c->n_local || (count > 0 && !y_out))
        return fail(c, SRMRA_ERR_INVALID_ARG, "range outside [0, n_local) or NULL output");
    if (count == 0) return SRMRA_OK;
    CK(cudaMemcpyAsync(y_out, c->d_y + first * c->Ll2, sizeof(float) * count * c->Ll2, cudaMemcpyDeviceToHost, c->stream));
    SYNC();
    return SRMRA_OK;
}

int srmra_em_iter(srmra_ctx* c, int32_t n_iters) {
    DevGuard dg_(c);
    if (!c) return fail(nullptr, SRMRA_ERR_INVALID_ARG, "ctx is NULL");
    if (c->failed) return SRMRA_ERR_STATE;
    if (n_iters < 0) return fail(c, SRMRA_ERR_INVALID_ARG, "n_iters < 0");
    if (c->needs_load) return fail(c, SRMRA_ERR_STATE, "no valid observations (srmra_init with y NULL, or a rejected srmra_load): srmra_load / srmra_generate first");
    int rc;
    // after a device-loop srmra_run with a tolerance the host count may exceed the iterations run
    if (c->iters_stale && (rc = sync_iters(c)) != SRMRA_OK) return rc;
    return iterate(c, n_iters, 0.0);
}

int srmra_run(srmra_ctx* c, int32_t max_iters, double rel_tol) {
    DevGuard dg_(c);
    if (!c) return fail(nullptr, SRMRA_ERR_INVALID_ARG, "ctx is NULL");
    if (c->failed) return SRMRA_ERR_STATE;
    if (max_iters < 0 || !(rel_tol == rel_tol)) return fail(c, SRMRA_ERR_INVALID_ARG, "max_iters < 0 or rel_tol NaN");
    if (c->needs_load) return fail(c, SRMRA_ERR_STATE, "no valid observations (srmra_init with y NULL, or a rejected srmra_load): srmra_load / srmra_generate first");
    int rc;
    if ((rc = sync_iters(c)) != SRMRA_OK) return rc;  // the run's first iteration index
    c->n_proj = 0;
    return iterate(c, max_iters, rel_tol);
}

int srmra_relative_error(srmra_ctx* c, const float* x_true, double* err_out, int32_t* s1_out, int32_t* s2_out) {
    DevGuard dg_(c);
    if (!c || !x_true) return fail(c, SRMRA_ERR_INVALID_ARG, "NULL argument");
    if (c->failed) return SRMRA_ERR_STATE;
    std::vector<double> xr(c->L2), corr(c->L2), xh(c->L2);
    double nr = 0.0;
    for (int p = 0; p < c->L2; ++p) {
        xr[p] = (double)x_true[p];
        nr += xr[p] * xr[p];
    }
    if (!(nr > 0.0) || !isfinite(nr)) return fail(c, SRMRA_ERR_INVALID_ARG, "x_true must be finite and non-zero");
    double* d = nullptr;
    CK(cudaMallocAsync(&d, sizeof(double) * 2 * c->L2, c->stream));
    cudaError_t e = cudaMemcpyAsync(d, xr.data(), sizeof(double) * c->L2, cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess) e = launch_shift_corr(c, d, d + c->L2);
    if (e == cudaSuccess) e = cudaMemcpyAsync(corr.data(), d + c->L2, sizeof(double) * c->L2, cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(xh.data(), c->d_x64, sizeof(double) * c->L2, cudaMemcpyDeviceToHost, c->stream);
    cudaFreeAsync(d, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "srmra_relative_error");
    int best = 0;  // the minimiser maximises the correlation; ties: the smallest flattened shift
    for (int s = 1; s < c->L2; ++s)
        if (corr[s] > corr[best]) best = s;
    // the distance at the minimiser directly (||x_hat||^2 + ||x||^2 - 2 corr cancels for small errors)
    const int L = c->L, b1 = best / L, b2 = best % L;
    double d2 = 0.0;
    for (int p1 = 0; p1 < L; ++p1)
        for (int p2 = 0; p2 < L; ++p2) {
            const double d = xh[(size_t)((p1 - b1 + L) % L) * L + (p2 - b2 + L) % L] - xr[(size_t)p1 * L + p2];
            d2 += d * d;
        }
    if (err_out) *err_out = sqrt(d2) / sqrt(nr);
    if (s1_out) *s1_out = best / c->L;
    if (s2_out) *s2_out = best % c->L;
    return SRMRA_OK;
}

int srmra_set_joint_rho(srmra_ctx* c, const double* rho) {
    DevGuard dg_(c);
    if (!c || !rho) return fail(c, SRMRA_ERR_INVALID_ARG, "NULL argument");
    if (c->failed) return SRMRA_ERR_STATE;
    if (c->path == SRMRA_PATH_FFT && c->Ll > 64)
        return fail(c, SRMRA_ERR_UNSUPPORTED, "joint shift prior on the FFT path: L_low <= 64 (init with path = gemm | direct)");
    std::vector<double> r(rho, rho + c->L2);
    double s = 0.0;
    for (double v : r) {
        if (!isfinite(v) || v < 0) return fail(c, SRMRA_ERR_INVALID_ARG, "joint rho must be finite and >= 0");
        s += v;
    }
    if (fabs(s - 1.0) > 1e-6) return fail(c, SRMRA_ERR_INVALID_ARG, "joint rho must sum to 1 (within 1e-6)");
    std::vector<double> marg(2 * (size_t)c->L, 0.0);
    for (int s1 = 0; s1 < c->L; ++s1)
        for (int s2 = 0; s2 < c->L; ++s2) {
            const double v = r[(size_t)s1 * c->L + s2] / s;
            r[(size_t)s1 * c->L + s2] = v;
            marg[s1] += v;
            marg[c->L + s2] += v;
        }
    if (!c->d_rhoj) {
        CK(cudaMalloc(&c->d_rhoj, sizeof(double) * c->L2));
        CK(cudaMalloc(&c->d_lrj, sizeof(float) * c->L2));
    }
    if (c->path == SRMRA_PATH_FFT && !c->d_ljp) {
        CK(cudaMalloc(&c->d_ljp, sizeof(float2) * ((c->KK + 1) / 2) * (size_t)c->Ll * c->Ll));
        CK(cudaMalloc(&c->d_jpart, sizeof(float) * (size_t)std::max(1, c->fft_part_cap) * fft_joint_bins(c->KK, c->Ll)));
        CK(cudaMalloc(&c->d_jacc, sizeof(double) * fft_joint_bins(c->KK, c->Ll)));
    }
    CK(cudaMemcpyAsync(c->d_rhoj, r.data(), sizeof(double) * c->L2, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_rho, marg.data(), sizeof(double) * 2 * c->L, cudaMemcpyHostToDevice, c->stream));
    SYNC();
    if (c->path == SRMRA_PATH_FFT) {
        int rc;
        if ((rc = sync_iters(c)) != SRMRA_OK) return rc;
        if ((rc = fft_joint_mode(c, true)) != SRMRA_OK) return rc;
        c->joint = true;
        if ((rc = clear_stop(c)) != SRMRA_OK) return rc;
        CK(launch_fft_tail(c, TAIL_PREP));  // the per-shift log2 prior table of the E/M kernel
        SYNC();
        return SRMRA_OK;
    }
    c->joint = true;
    return SRMRA_OK;
}

int srmra_get_joint_rho(srmra_ctx* c, double* out) {
    DevGuard dg_(c);
    if (!c || !out) return fail(c, SRMRA_ERR_INVALID_ARG, "NULL argument");
    if (c->failed) return SRMRA_ERR_STATE;
    if (!c->joint) return fail(c, SRMRA_ERR_STATE, "no joint shift prior set (srmra_set_joint_rho)");
    CK(cudaMemcpyAsync(out, c->d_rhoj, sizeof(double) * c->L2, cudaMemcpyDeviceToHost, c->stream));
    SYNC();
    return SRMRA_OK;
}

int srmra_moments(srmra_ctx* c, double* m1, double* m2) {
    DevGuard dg_(c);
    if (!c) return fail(nullptr, SRMRA_ERR_INVALID_ARG, "ctx is NULL");
    if (c->failed) return SRMRA_ERR_STATE;
    if (c->needs_load) return fail(c, SRMRA_ERR_STATE, "no valid observations (srmra_init with y NULL, or a rejected srmra_load)");
    if (!m1 && !m2) return fail(c, SRMRA_ERR_INVALID_ARG, "both outputs NULL");
    std::string err;
    const int rc = moments(c, m1, m2, err);
    if (rc == SRMRA_ERR_CUDA) return fail(c, rc, err);
    return rc;
}

static int mom_fail(srmra_ctx* c, int rc, const std::string& err) {
    if (rc == SRMRA_OK || rc == SRMRA_ERR_NCCL) return rc;  // NCCL failures were recorded by allreduce_doubles
    return fail(c, rc, err);
}

int srmra_mom_set_moments(srmra_ctx* c, const double* m1, const double* m2) {
    DevGuard dg_(c);
    if (!c) return fail(nullptr, SRMRA_ERR_INVALID_ARG, "ctx is NULL");
    if (c->failed) return SRMRA_ERR_STATE;
    if ((m1 == nullptr) != (m2 == nullptr)) return fail(c, SRMRA_ERR_INVALID_ARG, "m1 and m2: both or neither");
    if (!m1 && c->needs_load) return fail(c, SRMRA_ERR_STATE, "no valid observations (srmra_init with y NULL, or a rejected srmra_load)");
    if (!mom_supported(c)) return fail(c, SRMRA_ERR_UNSUPPORTED, "moment objective compiled for L_low <= 64");
    if (m1) {
        for (int a = 0; a < c->Ll2; ++a)
            if (!isfinite(m1[a])) return fail(c, SRMRA_ERR_INVALID_ARG, "m1 not finite");
        for (size_t a = 0; a < (size_t)c->Ll2 * c->Ll2; ++a)
            if (!isfinite(m2[a])) return fail(c, SRMRA_ERR_INVALID_ARG, "m2 not finite");
    }
    std::string err;
    return mom_fail(c, mom_set(c, m1, m2, err), err);
}

int srmra_mom_objective(srmra_ctx* c, const double* x, const double* rho1, const double* rho2, double* f,
                        double* grad_x, double* grad_rho1, double* grad_rho2) {
    DevGuard dg_(c);
    if (!c) return fail(nullptr, SRMRA_ERR_INVALID_ARG, "ctx is NULL");
    if (c->failed) return SRMRA_ERR_STATE;
    if (!x || !rho1 || !rho2) return fail(c, SRMRA_ERR_INVALID_ARG, "NULL theta");
    if (!mom_ready(c)) return fail(c, SRMRA_ERR_STATE, "no moments set (srmra_mom_set_moments)");
    std::string err;
    return mom_fail(c, mom_objective(c, x, rho1, rho2, f, grad_x, grad_rho1, grad_rho2, err), err);
}

int srmra_mom_run(srmra_ctx* c, int32_t max_steps, int32_t F, double gtol, double* f_out, int32_t* steps_out) {
    DevGuard dg_(c);
    if (!c) return fail(nullptr, SRMRA_ERR_INVALID_ARG, "ctx is NULL");
    if (c->failed) return SRMRA_ERR_STATE;
    if (max_steps < 0 || F < 0 || !(gtol >= 0.0)) return fail(c, SRMRA_ERR_INVALID_ARG, "max_steps < 0, F < 0 or gtol < 0");
    if (!mom_ready(c)) return fail(c, SRMRA_ERR_STATE, "no moments set (srmra_mom_set_moments)");
    int rc;
    if ((rc = sync_iters(c)) != SRMRA_OK) return rc;
    std::string err;
    int steps = 0;
    rc = mom_run(c, max_steps, F, gtol, f_out, &steps, err);
    if (steps_out) *steps_out = steps;
    if (rc != SRMRA_OK) return mom_fail(c, rc, err);
    c->joint = false;  // the estimate is (x, rho1, rho2) again
    if ((rc = fft_joint_mode(c, false)) != SRMRA_OK) return rc;
    if ((rc = clear_stop(c)) != SRMRA_OK) return rc;
    if ((rc = refresh_after_denoise(c)) != SRMRA_OK) return rc;  // EM can continue from the MoM estimate
    SYNC();
    return SRMRA_OK;
}

int srmra_set_denoiser(srmra_ctx* c, srmra_denoiser_fn fn, void* user) {
    if (!c) return fail(nullptr, SRMRA_ERR_INVALID_ARG, "ctx is NULL");
    if (c->failed) return SRMRA_ERR_STATE;
    c->denoiser = fn;
    c->denoiser_user = user;
    return SRMRA_OK;
}

int srmra_profile(srmra_ctx* c, int32_t enable) {
    DevGuard dg_(c);
    if (!c) return fail(nullptr, SRMRA_ERR_INVALID_ARG, "ctx is NULL");
    if (c->failed) return SRMRA_ERR_STATE;
    SYNC();
    c->prof = enable != 0;
    c->ev_used = 0;
    if (c->path == SRMRA_PATH_FFT && c->prof) {  // arm the E/M launch stamps of the window
        int rc;
        if ((rc = sync_iters(c)) != SRMRA_OK) return rc;
        c->prof_t0 = c->iters_done;
        std::vector<unsigned long long> arm(2 * (size_t)c->opt.trace_cap);
        for (size_t k = 0; k < arm.size(); k += 2) {
            arm[k] = ~0ull;
            arm[k + 1] = 0ull;
        }
        CK(cudaMemcpy(c->d_emt, arm.data(), sizeof(unsigned long long) * arm.size(), cudaMemcpyHostToDevice));
    }
    return SRMRA_OK;
}

int srmra_profile_read(srmra_ctx* c, double* em_ms, double* iter_ms, int32_t* n_iters) {
    DevGuard dg_(c);
    if (!c) return fail(nullptr, SRMRA_ERR_INVALID_ARG, "ctx is NULL");
    if (c->failed) return SRMRA_ERR_STATE;
    SYNC();
    double em = 0, tot = 0;
    int n = 0;
    if (c->path == SRMRA_PATH_FFT) {
        // E/M launch duration = last-CTA end - first-CTA start (globaltimer ns); iteration = the time
        // between consecutive E/M starts (the window's last iteration contributes its E/M time only)
        int rc;
        if ((rc = sync_iters(c)) != SRMRA_OK) return rc;
        const int t1 = std::min(c->iters_done, c->opt.trace_cap);
        const int m = t1 - c->prof_t0;
        if (m > 0) {
            std::vector<unsigned long long> st(2 * (size_t)m);
            CK(cudaMemcpy(st.data(), c->d_emt + 2 * (size_t)c->prof_t0, sizeof(unsigned long long) * st.size(),
                          cudaMemcpyDeviceToHost));
            for (int k = 0; k < m; ++k, ++n) {
                em += (double)(st[2 * k + 1] - st[2 * k]) * 1e-6;
                if (k + 1 < m) tot += (double)(st[2 * k + 2] - st[2 * k]) * 1e-6;
            }
            if (m > 1) tot *= (double)m / (m - 1);  // per-iteration mean over the m - 1 full intervals
        }
        c->prof_t0 = c->iters_done;
        if (em_ms) *em_ms = em;
        if (iter_ms) *iter_ms = tot;
        if (n_iters) *n_iters = n;
        return SRMRA_OK;
    }
    for (size_t k = 0; k + 4 <= c->ev_used; k += 4, ++n) {
        float a = 0, b = 0;
        CK(cudaEventElapsedTime(&a, c->ev_pool[k + 1], c->ev_pool[k + 2]));
        CK(cudaEventElapsedTime(&b, c->ev_pool[k], c->ev_pool[k + 3]));
        em += a;
        tot += b;
    }
    c->ev_used = 0;
    if (em_ms) *em_ms = em;
    if (iter_ms) *iter_ms = tot;
    if (n_iters) *n_iters = n;
    return SRMRA_OK;
}

int srmra_get_estimate(srmra_ctx* c, float* x_out, double* rho1_out, double* rho2_out, double* loglik_out,
                       int32_t* iters_done) {
    DevGuard dg_(c);
    if (!c) return fail(nullptr, SRMRA_ERR_INVALID_ARG, "ctx is NULL");
    if (c->failed) return SRMRA_ERR_STATE;
    if (x_out) CK(cudaMemcpyAsync(x_out, c->d_x32, sizeof(float) * c->L2, cudaMemcpyDeviceToHost, c->stream));
    if (rho1_out) CK(cudaMemcpyAsync(rho1_out, c->d_rho, sizeof(double) * c->L, cudaMemcpyDeviceToHost, c->stream));
    if (rho2_out) CK(cudaMemcpyAsync(rho2_out, c->d_rho + c->L, sizeof(double) * c->L, cudaMemcpyDeviceToHost, c->stream));
    double ll = NAN;
    int flag = 0;
    int rc;
    if ((rc = sync_iters(c)) != SRMRA_OK) return rc;
    const int t = c->iters_done;
    if (t > 0 && t <= c->opt.trace_cap)
        CK(cudaMemcpyAsync(&ll, c->d_trace + (t - 1), sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(&flag, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    SYNC();
    if (loglik_out) *loglik_out = ll;
    if (iters_done) *iters_done = t;
    if (flag) return fail(c, SRMRA_ERR_NUMERIC, "non-finite log-likelihood or estimate");
    return SRMRA_OK;
}

int srmra_get_loglik_trace(srmra_ctx* c, double* out, int32_t cap, int32_t* n) {
    DevGuard dg_(c);
    if (!c) return fail(nullptr, SRMRA_ERR_INVALID_ARG, "ctx is NULL");
    if (c->failed) return SRMRA_ERR_STATE;
    int rc;
    if ((rc = sync_iters(c)) != SRMRA_OK) return rc;
    int m = c->iters_done < c->opt.trace_cap ? c->iters_done : c->opt.trace_cap;
    if (m > cap) m = cap;
    if (m > 0 && out) CK(cudaMemcpyAsync(out, c->d_trace, sizeof(double) * m, cudaMemcpyDeviceToHost, c->stream));
    SYNC();
    if (n) *n = c->iters_done;
    return SRMRA_OK;
}

int srmra_get_stats(srmra_ctx* c, double* b, double* cmass, double* m1, double* m2) {
    DevGuard dg_(c);
    if (!c) return fail(nullptr, SRMRA_ERR_INVALID_ARG, "ctx is NULL");
    if (c->failed) return SRMRA_ERR_STATE;
    if (b) CK(cudaMemcpyAsync(b, c->d_pack + c->pk.b, sizeof(double) * c->L2, cudaMemcpyDeviceToHost, c->stream));
    if (cmass) CK(cudaMemcpyAsync(cmass, c->d_pack + c->pk.cmass, sizeof(double) * c->KK, cudaMemcpyDeviceToHost, c->stream));
    if (m1) CK(cudaMemcpyAsync(m1, c->d_pack + c->pk.m1, sizeof(double) * c->L, cudaMemcpyDeviceToHost, c->stream));
    if (m2) CK(cudaMemcpyAsync(m2, c->d_pack + c->pk.m2, sizeof(double) * c->L, cudaMemcpyDeviceToHost, c->stream));
    SYNC();
    return SRMRA_OK;
}

int srmra_get_obs_loglik(srmra_ctx* c, double* out) {
    DevGuard dg_(c);
    if (!c || !out) return fail(c, SRMRA_ERR_INVALID_ARG, "NULL argument");
    if (c->failed) return SRMRA_ERR_STATE;
    if (c->n_local) CK(cudaMemcpyAsync(out, c->d_llobs, sizeof(double) * c->n_local, cudaMemcpyDeviceToHost, c->stream));
    SYNC();
    return SRMRA_OK;
}

int srmra_local_stats(srmra_ctx* c, double* out) {
    DevGuard dg_(c);
    if (!c || !out) return fail(c, SRMRA_ERR_INVALID_ARG, "NULL argument");
    if (c->failed) return SRMRA_ERR_STATE;
    int rc;
    if ((rc = sync_iters(c)) != SRMRA_OK || (rc = clear_stop(c)) != SRMRA_OK) return rc;
    const bool prof = c->prof;
    c->prof = false;  // keep the profiling records aligned to whole iterations
    rc = local_estep_mstep(c);
    c->prof = prof;
    if (rc != SRMRA_OK) return rc;
    if (c->path == SRMRA_PATH_FFT) CK(launch_fft_tail(c, TAIL_REDUCE | TAIL_FOLD));  // local, no update
    CK(cudaMemcpyAsync(out, c->d_pack, sizeof(double) * c->pk.total, cudaMemcpyDeviceToHost, c->stream));
    SYNC();
    return SRMRA_OK;
}

int srmra_get_path(const srmra_ctx* c) { return c ? c->path : SRMRA_ERR_INVALID_ARG; }

int srmra_debug_timestamps(srmra_ctx* c, uint64_t* out8) {
    DevGuard dg_(c);
    if (!c || !out8) return fail(c, SRMRA_ERR_INVALID_ARG, "NULL argument");
    if (!c->d_stamps) return fail(c, SRMRA_ERR_STATE, "set SRMRA_TAIL_STAMPS before srmra_init");
    CK(cudaMemcpyAsync(out8, c->d_stamps, 8 * sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream));
    SYNC();
    // re-arm the cross-block extremes: [6] earliest tail-block start (min), [7] latest tail-block end (max)
    const uint64_t arm[2] = {~0ull, 0ull};
    CK(cudaMemcpy(c->d_stamps + 6, arm, sizeof(arm), cudaMemcpyHostToDevice));
    CK(cudaMemset(c->d_stamps + 2, 0, 2 * sizeof(uint64_t)));  // [2] / [3]: slowest block's fold / prep item loop
    return SRMRA_OK;
}

int srmra_launches_per_iter(const srmra_ctx* c) {
    if (!c) return SRMRA_ERR_INVALID_ARG;
    if (c->path == SRMRA_PATH_DIRECT) return 3 + (c->n_local > 0 ? 1 : 0);  // prep, pack, finalize [, em]
    // prep, x copies, pack, finalize [, GEMM1, softmax, GEMM2, fold]
    if (c->path == SRMRA_PATH_GEMM) return 4 + (c->n_local > 0 ? 4 : 0);
    return fft_launches_per_iter(c);  // [em,] tail [, reduce-only tail when world > 1]
}

void srmra_free(srmra_ctx* c) {
    DevGuard dg_(c);
    if (!c) return;
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->nccl_comm) {
        NcclApi& api = nccl();
        if (api.loaded) api.CommDestroy((ncclComm_t)c->nccl_comm);
    }
    void* bufs[] = {c->d_y, c->d_yhat, c->d_ysum, c->d_ynorm, c->d_llobs, c->d_x64, c->d_x32, c->d_xtmp, c->d_rho,
                    c->par.f32, c->par.f64, c->d_xhat, c->d_xcoef, c->d_bhat, c->d_pack, c->d_trace, c->d_flag,
                    c->d_part, c->d_llpart, c->d_tw, c->d_counter, c->d_stamps, c->d_part_s, c->d_llpart_s};
    for (void* p : bufs)
        if (p) cudaFree(p);
    gemm_free(c);
    if (c->graph) cudaGraphExecDestroy(c->graph);
    if (c->graph_prof) cudaGraphExecDestroy(c->graph_prof);
    if (c->graph_prof_src) cudaGraphDestroy(c->graph_prof_src);
    for (int k = 0; k < 4; ++k)
        if (c->prof_ph[k]) cudaEventDestroy(c->prof_ph[k]);
    if (c->d_iter) cudaFree(c->d_iter);
    if (c->d_run) cudaFree(c->d_run);
    if (c->d_emt) cudaFree(c->d_emt);
    if (c->d_rhoj) cudaFree(c->d_rhoj);
    if (c->d_ljp) cudaFree(c->d_ljp);
    if (c->d_jpart) cudaFree(c->d_jpart);
    if (c->d_jacc) cudaFree(c->d_jacc);
    mom_free(c);
    if (c->d_lrj) cudaFree(c->d_lrj);
    if (c->d_rtol) cudaFree(c->d_rtol);
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    if (c->copy_event) cudaEventDestroy(c->copy_event);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

}  // extern "C"
