// capi.cu -- extern "C" boundary (include/vxq.h).  Every entry point catches, maps the
// failure to a VXQ_ERR_* code and leaves a thread-local message for vxq_last_error().
#include <cmath>
#include <cstring>
#include <string>

#include "vxq_internal.h"

namespace {
thread_local std::string g_last_error;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        g_last_error.clear();
        return VXQ_OK;
    } catch (const vxq::Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return VXQ_ERR_OOM;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return VXQ_ERR_CUDA;
    }
}

void check_outputs(const vxq_outputs* out) {
    VXQ_REQUIRE(out != nullptr, "outputs must not be null");
    VXQ_REQUIRE(out->states && out->energies, "outputs.states and outputs.energies are required");
}

struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        VXQ_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() { cudaSetDevice(prev); }
};
}  // namespace

struct vxq_problem {
    vxq::Problem* p;
};

namespace {
struct SessionBox {
    vxq::Session* S;
    int device;
    vxq_run_opts opts;
};
void retain_mempool_public() { vxq::retain_mempool(); }
}  // namespace

extern "C" {

int vxq_abi_version(void) { return VXQ_ABI_VERSION; }

const char* vxq_last_error(void) { return g_last_error.c_str(); }

int vxq_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int vxq_pa_schedule(double lambda0, int64_t T, double* out) {
    return guarded([&] {
        VXQ_REQUIRE(T >= 0 && (T == 0 || out), "invalid schedule arguments");
        vxq::pa_schedule(lambda0, T, out);
    });
}

int vxq_sbm_schedule(double a0, int64_t T, double* out) {
    return guarded([&] {
        VXQ_REQUIRE(T >= 0 && (T == 0 || out), "invalid schedule arguments");
        vxq::sbm_schedule(a0, T, out);
    });
}

int vxq_sa_schedule(double T_init, double T_final, int64_t sweeps, double* out) {
    return guarded([&] {
        VXQ_REQUIRE(sweeps >= 0 && (sweeps == 0 || out), "invalid schedule arguments");
        vxq::sa_schedule(T_init, T_final, sweeps, out);
    });
}

int vxq_problem_create(int64_t n, int64_t num_couplings, const int64_t* rows,
                       const int64_t* cols, const double* values, const double* h,
                       double offset, int device, vxq_problem** out) {
    return guarded([&] {
        VXQ_REQUIRE(out != nullptr, "out must not be null");
        *out = nullptr;
        DeviceGuard dg(device);
        vxq::Problem* p =
            vxq::problem_create(n, num_couplings, rows, cols, values, h, offset, device);
        *out = new vxq_problem{p};
    });
}

int vxq_problem_generate(int32_t family, int64_t n, uint64_t seed, int device,
                         vxq_problem** out) {
    return guarded([&] {
        VXQ_REQUIRE(out != nullptr, "out must not be null");
        *out = nullptr;
        int ndev = 0;
        VXQ_CUDA(cudaGetDeviceCount(&ndev));
        VXQ_REQUIRE(device >= 0 && device < ndev, "invalid CUDA device ordinal");
        DeviceGuard dg(device);
        *out = new vxq_problem{vxq::problem_generate(family, n, seed, device)};
    });
}

int vxq_problem_export(const vxq_problem* p, int64_t* rows, int64_t* cols, double* values,
                       double* h, double* offset) {
    return guarded([&] {
        VXQ_REQUIRE(p, "null problem");
        DeviceGuard dg(p->p->device);
        vxq::problem_export(p->p, rows, cols, values, h, offset);
    });
}

int vxq_problem_destroy(vxq_problem* p) {
    return guarded([&] {
        if (!p) return;
        delete p->p;
        delete p;
    });
}

int vxq_problem_info(const vxq_problem* p, int64_t* info5) {
    return guarded([&] {
        VXQ_REQUIRE(p && info5, "null argument");
        info5[0] = p->p->n;
        info5[1] = p->p->m;
        info5[2] = p->p->nnz;
        info5[3] = p->p->max_row_nnz;
        info5[4] = p->p->uniform_magnitude ? 1 : 0;
    });
}

int vxq_problem_lambda0(vxq_problem* p, double* out) {
    return guarded([&] {
        VXQ_REQUIRE(p && out, "null argument");
        DeviceGuard dg(p->p->device);
        vxq::StreamScope ss(nullptr);
        *out = vxq::problem_lambda0(p->p, ss.s);
    });
}

int vxq_problem_c0(vxq_problem* p, double* out) {
    return guarded([&] {
        VXQ_REQUIRE(p && out, "null argument");
        DeviceGuard dg(p->p->device);
        vxq::StreamScope ss(nullptr);
        *out = vxq::problem_c0(p->p, ss.s);
    });
}

int vxq_problem_eig_info(vxq_problem* p, double* info6) {
    return guarded([&] {
        VXQ_REQUIRE(p && info6, "null argument");
        DeviceGuard dg(p->p->device);
        vxq::StreamScope ss(nullptr);
        const double c0 = vxq::problem_c0(p->p, ss.s);
        const vxq::EigInfo& e = p->p->eig;
        info6[0] = e.value;
        info6[1] = e.theta;
        info6[2] = e.residual;
        info6[3] = (double)e.iterations;
        info6[4] = (double)e.method;
        info6[5] = c0;
    });
}

int vxq_dense_eligible(const vxq_problem* p, int32_t solver, int64_t replicas, double q_cap,
                       double init_noise, int32_t* out) {
    return guarded([&] {
        VXQ_REQUIRE(p && out, "null argument");
        VXQ_REQUIRE(solver == 0 || solver == 1, "solver must be 0 (PA) or 1 (SBM)");
        VXQ_REQUIRE(replicas > 0, "replicas must be positive");
        const vxq::Problem* P = p->p;
        bool e;
        if (P->uniform_magnitude) e = vxq::dense_eligible(P, replicas);
        else e = vxq::dense_general_eligible(P, replicas) &&
                 (solver == 0 || vxq::dense_sbm_fp16_ok(q_cap, init_noise));
        *out = e ? 1 : 0;
    });
}

int vxq_pa_solve(vxq_problem* p, const vxq_pa_params* prm, const vxq_run_opts* opts,
                 vxq_outputs* out) {
    return guarded([&] {
        VXQ_REQUIRE(p && prm, "null argument");
        check_outputs(out);
        // PaParams.validate (common.py:109-116)
        VXQ_REQUIRE(prm->steps > 0, "steps must be positive");
        VXQ_REQUIRE(prm->learning_rate > 0, "learning_rate must be positive");
        VXQ_REQUIRE(prm->momentum >= 0 && prm->momentum < 1, "momentum must lie in [0, 1)");
        VXQ_REQUIRE(std::isnan(prm->lambda0) || prm->lambda0 > 0, "lambda0 must be positive");
        VXQ_REQUIRE(prm->replicas > 0, "replicas must be positive");
        DeviceGuard dg(p->p->device);
        vxq::StreamScope ss(opts ? opts->stream : nullptr);
        vxq::pa_solve(p->p, prm, opts, out, ss.s);
    });
}

int vxq_sa_solve(vxq_problem* p, const vxq_sa_params* prm, const vxq_run_opts* opts,
                 vxq_outputs* out) {
    return guarded([&] {
        VXQ_REQUIRE(p && prm, "null argument");
        check_outputs(out);
        // SaParams.validate (common.py:84-91)
        VXQ_REQUIRE(prm->sweeps > 0, "sweeps must be positive");
        VXQ_REQUIRE(prm->replicas > 0, "replicas must be positive");
        if (!std::isnan(prm->T_init) && !std::isnan(prm->T_final))
            VXQ_REQUIRE(prm->T_init >= prm->T_final && prm->T_final > 0,
                        "need T_init >= T_final > 0");
        DeviceGuard dg(p->p->device);
        vxq::StreamScope ss(opts ? opts->stream : nullptr);
        vxq::sa_solve(p->p, prm, opts, out, ss.s);
    });
}

int vxq_sbm_solve(vxq_problem* p, const vxq_sbm_params* prm, const vxq_run_opts* opts,
                  vxq_outputs* out) {
    return guarded([&] {
        VXQ_REQUIRE(p && prm, "null argument");
        check_outputs(out);
        // SbmParams.validate (common.py:136-144)
        VXQ_REQUIRE(prm->steps > 0, "steps must be positive");
        VXQ_REQUIRE(prm->dt > 0, "dt must be positive");
        VXQ_REQUIRE(prm->a0 > 0, "a0 must be positive");
        VXQ_REQUIRE(std::isnan(prm->c0) || prm->c0 > 0, "c0 must be positive");
        VXQ_REQUIRE(prm->q_cap > 0, "q_cap must be positive");
        VXQ_REQUIRE(prm->init_noise > 0, "init_noise must be positive");
        VXQ_REQUIRE(prm->replicas > 0, "replicas must be positive");
        DeviceGuard dg(p->p->device);
        vxq::StreamScope ss(opts ? opts->stream : nullptr);
        vxq::sbm_solve(p->p, prm, opts, out, ss.s);
    });
}

int vxq_sbm_integrate(int64_t n, const int64_t* bt_indptr, const int32_t* bt_indices,
                      const double* bt_data, const double* g, int64_t R, double* Q,
                      double* P, const double* a_sched, int64_t T, double dt, double a0,
                      double c0, double q_cap, const vxq_run_opts* opts) {
    return guarded([&] {
        VXQ_REQUIRE(n >= 1 && R >= 1 && T >= 0, "invalid sizes");
        VXQ_REQUIRE(bt_indptr && g && Q && P && (T == 0 || a_sched), "null argument");
        int dev = 0;
        VXQ_CUDA(cudaGetDevice(&dev));
        vxq::StreamScope ss(opts ? opts->stream : nullptr);
        vxq::sbm_integrate(n, bt_indptr, bt_indices, bt_data, g, R, Q, P, a_sched, T, dt, a0,
                           c0, q_cap, opts, ss.s);
    });
}

int vxq_energies(vxq_problem* p, const int8_t* states, int64_t R, double* energies,
                 const vxq_run_opts* opts) {
    return guarded([&] {
        VXQ_REQUIRE(p && states && energies && R >= 0, "null argument");
        if (R == 0) return;
        DeviceGuard dg(p->p->device);
        vxq::StreamScope ss(opts ? opts->stream : nullptr);
        cudaStream_t s = ss.s;
        const int64_t n = p->p->n;
        const int64_t W = vxq::ceil_div(R, 32);
        const bool on_dev = opts && opts->outputs_on_device;
        vxq::DevBuf<int8_t> st;
        const int8_t* sd = states;
        if (!on_dev) {
            st = vxq::DevBuf<int8_t>(n * R, s);
            VXQ_CUDA(cudaMemcpyAsync(st.get(), states, n * R, cudaMemcpyHostToDevice, s));
            sd = st.get();
        }
        vxq::DevBuf<uint32_t> sb(n * W, s);
        vxq::pack_states_to_bits(sd, n, R, W, sb.get(), s);
        vxq::DevBuf<double> e;
        double* ed = energies;
        if (!on_dev) {
            e = vxq::DevBuf<double>(R, s);
            ed = e.get();
        }
        vxq::energies_from_bits(p->p, sb.get(), W, R, ed, s);
        if (!on_dev)
            VXQ_CUDA(cudaMemcpyAsync(energies, ed, R * sizeof(double), cudaMemcpyDeviceToHost, s));
        VXQ_CUDA(cudaStreamSynchronize(s));
    });
}

int vxq_exchange_row_bytes(int32_t solver, int64_t replicas, int32_t precision, int64_t* out) {
    return guarded([&] {
        VXQ_REQUIRE(out && replicas > 0 && (solver == 0 || solver == 1), "invalid arguments");
        *out = vxq::exchange_row_bytes(solver, replicas, precision);
    });
}

int vxq_session_create(vxq_problem* p, int32_t solver, const vxq_pa_params* pa,
                       const vxq_sbm_params* sbm, int64_t row_begin, int64_t row_end,
                       int64_t rows_alloc, void* xbuf0, void* xbuf1, const vxq_run_opts* opts,
                       vxq_session** out) {
    return guarded([&] {
        VXQ_REQUIRE(p && out && (solver == 0 ? pa != nullptr : sbm != nullptr), "null argument");
        *out = nullptr;
        VXQ_CUDA(cudaSetDevice(p->p->device));
        retain_mempool_public();
        cudaStream_t st = opts && opts->stream ? (cudaStream_t)opts->stream : nullptr;
        bool own = false;
        if (!st) {
            VXQ_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            own = true;
        }
        vxq::Session* S = vxq::session_create(p->p, solver, pa, sbm, row_begin, row_end,
                                              rows_alloc, xbuf0, xbuf1, opts, st);
        vxq::session_set_own_stream(S, own);
        *out = reinterpret_cast<vxq_session*>(new SessionBox{S, p->p->device,
                                                             opts ? *opts : vxq_run_opts{}});
    });
}

int vxq_session_step(vxq_session* s, int64_t t) {
    return guarded([&] {
        VXQ_REQUIRE(s, "null session");
        SessionBox* b = reinterpret_cast<SessionBox*>(s);
        VXQ_CUDA(cudaSetDevice(b->device));
        vxq::session_step(b->S, t);
    });
}

int vxq_session_finish(vxq_session* s, vxq_outputs* out) {
    return guarded([&] {
        VXQ_REQUIRE(s, "null session");
        check_outputs(out);
        SessionBox* b = reinterpret_cast<SessionBox*>(s);
        VXQ_CUDA(cudaSetDevice(b->device));
        vxq::session_finish(b->S, out, &b->opts);
    });
}

int vxq_session_set_peers(vxq_session* s, int32_t world, int32_t rank, uint32_t epoch,
                          void* const* xbuf0, void* const* xbuf1, uint64_t* const* flags) {
    return guarded([&] {
        VXQ_REQUIRE(s, "null session");
        SessionBox* b = reinterpret_cast<SessionBox*>(s);
        VXQ_CUDA(cudaSetDevice(b->device));
        vxq::session_set_peers(b->S, world, rank, epoch, xbuf0, xbuf1, flags);
    });
}

int vxq_exchange_alloc(int device, int64_t bytes, void** out) {
    return guarded([&] {
        VXQ_REQUIRE(out && bytes > 0, "invalid exchange allocation");
        *out = nullptr;
        DeviceGuard dg(device);
        void* p = nullptr;
        VXQ_CUDA(cudaMalloc(&p, (size_t)bytes));  // plain cudaMalloc: IPC-shareable
        // zeroing must be complete before the IPC handle reaches another process (peers
        // write into this memory with no ordering against our stream)
        cudaError_t e = cudaMemset(p, 0, (size_t)bytes);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            cudaFree(p);
            VXQ_CUDA(e);
        }
        *out = p;
    });
}

int vxq_exchange_free(void* ptr) {
    return guarded([&] {
        if (ptr) VXQ_CUDA(cudaFree(ptr));
    });
}

int vxq_ipc_handle(const void* dev_ptr, void* handle_out) {
    return guarded([&] {
        VXQ_REQUIRE(dev_ptr && handle_out, "null argument");
        static_assert(sizeof(cudaIpcMemHandle_t) == VXQ_IPC_HANDLE_BYTES, "IPC handle size");
        cudaIpcMemHandle_t h;
        VXQ_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)));
        memcpy(handle_out, &h, sizeof(h));
    });
}

int vxq_ipc_open(const void* handle, int device, void** dev_ptr) {
    return guarded([&] {
        VXQ_REQUIRE(handle && dev_ptr, "null argument");
        *dev_ptr = nullptr;
        DeviceGuard dg(device);
        cudaIpcMemHandle_t h;
        memcpy(&h, handle, sizeof(h));
        VXQ_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    });
}

int vxq_ipc_close(void* dev_ptr) {
    return guarded([&] {
        if (dev_ptr) VXQ_CUDA(cudaIpcCloseMemHandle(dev_ptr));
    });
}

int vxq_session_destroy(vxq_session* s) {
    return guarded([&] {
        if (!s) return;
        SessionBox* b = reinterpret_cast<SessionBox*>(s);
        cudaSetDevice(b->device);
        vxq::session_destroy(b->S);
        delete b;
    });
}

}  // extern "C"
