// vxq_internal.h -- internal types shared by the vxq translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <mutex>
#include <vector>

#include "vxq_common.cuh"

namespace vxq {

// Maximum 32-bit limbs of the exact fixed-point energy accumulator.
constexpr int kMaxLimbs = 8;

struct DenseOperand;  // dense tcgen05 path (dense_tc.cu)
struct NbrBlocks;     // row-block neighbour lists of the blocked sparse SBM step (dynamics.cu)

// lambda_max of the SBM coupling matrix (eigen.cu, eig_extreme "max")
constexpr int kEigDense = 0;       // n <= 512: full-dimension Lanczos, full reorthogonalisation
constexpr int kEigLanczos = 1;     // Lanczos to ARPACK's tol, theta + explicit residual
constexpr int kEigGershgorin = 2;  // no convergence: Gershgorin bound
struct EigInfo {
    double value = NAN;     // what eig_extreme returns
    double theta = NAN;     // largest Ritz value
    double residual = NAN;  // ||B y - theta y|| / ||y|| (Lanczos)
    int64_t iterations = 0;
    int method = -1;
};

// A device-resident Ising problem (the reference's IsingModel, model.py:113-200).
struct Problem {
    int device = 0;
    int64_t n = 0, m = 0, nnz = 0;
    double offset = 0.0;

    // symmetric coupling CSR, ascending columns per row (both triangles, zero diagonal)
    int64_t* indptr = nullptr;     // [n+1]
    int32_t* indices = nullptr;    // [nnz]
    double* data64 = nullptr;      // [nnz]
    float* data32 = nullptr;       // [nnz]
    int32_t* lower_count = nullptr;  // [n] entries with j < i in row i
    double* h64 = nullptr;         // [n]
    float* h32 = nullptr;          // [n]
    double* g64 = nullptr;         // [n]  -h  (SBM drive, bifurcation.py:57)
    float* g32 = nullptr;          // [n]
    int32_t* coo_i = nullptr;      // [m] couplings i<j (energy evaluation)
    int32_t* coo_j = nullptr;      // [m]
    double* coo_v = nullptr;       // [m] coupling values (COO order)

    // exact energy: every coefficient as an L-limb two's-complement integer * 2^e_low
    int limbs = 0;
    int e_low = 0;
    uint32_t* coef_fx = nullptr;   // [m][limbs]
    uint32_t* h_fx = nullptr;      // [n][limbs]
    uint32_t offset_fx[kMaxLimbs] = {0};
    uint32_t mag_fx[kMaxLimbs] = {0};  // +|J_ij| when uniform_magnitude
    bool energy_ok = true;         // false if the dynamic range exceeds kMaxLimbs*32 bits

    int64_t max_row_nnz = 0;
    bool uniform_magnitude = false;  // all |J_ij| equal (e.g. SK +-1/sqrt(N))
    double magnitude = 0.0;

    std::mutex mu;  // guards the lazy caches below
    double lambda0 = NAN;
    double c0 = NAN;
    EigInfo eig;      // how c0 was obtained (vxq_problem_eig_info)
    int h_zero = -1;  // cached problem_h_zero (-1 = unknown)
    DenseOperand* dense = nullptr;
    NbrBlocks* nbr_blocks = nullptr;  // built on the first blocked-SBM eligibility check
    int nbr_blocks_state = 0;         // 0 unknown, 1 built (eligible), -1 not eligible

    ~Problem();
};

// Keep the device's stream-ordered pool from trimming at every synchronize, so repeated
// solves reuse workspace instead of going back to the driver (once per device).
inline void retain_mempool() {
    static std::mutex mu;
    static bool done[64] = {false};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
    std::lock_guard<std::mutex> g(mu);
    if (done[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done[dev] = true;
}

// run-scoped stream holder
struct StreamScope {
    cudaStream_t s = nullptr;
    bool owned = false;
    explicit StreamScope(void* user) {
        retain_mempool();
        if (user) {
            s = (cudaStream_t)user;
        } else {
            VXQ_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
            owned = true;
        }
    }
    ~StreamScope() {
        if (owned && s) cudaStreamDestroy(s);
    }
};

// stream-ordered device buffer
template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t count = 0;
    cudaStream_t s = nullptr;
    DevBuf() = default;
    DevBuf(size_t n, cudaStream_t st) : count(n), s(st) {
        if (n) VXQ_CUDA(cudaMallocAsync((void**)&p, n * sizeof(T), st));
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), count(o.count), s(o.s) { o.p = nullptr; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        release();
        p = o.p; count = o.count; s = o.s; o.p = nullptr;
        return *this;
    }
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
    }
    T* get() const { return p; }
};

// ---- problem.cu
Problem* problem_create(int64_t n, int64_t m, const int64_t* rows, const int64_t* cols,
                        const double* values, const double* h, double offset, int device);
double problem_lambda0(Problem* p, cudaStream_t s);
void encode_energy(Problem* P, cudaStream_t s);
// replace h / offset (host or device pointer) and re-derive everything that depends on them
void problem_set_fields(Problem* P, const double* h, double offset, cudaStream_t s);
// generate.cu: device-side instance families (0 = qubo_deg6, BASELINE config 5)
Problem* problem_generate(int family, int64_t n, uint64_t seed, int device);
void problem_export(Problem* P, int64_t* rows, int64_t* cols, double* values, double* h,
                    double* offset);
double problem_c0(Problem* p, cudaStream_t s);

// ---- eigen.cu: lambda_max of the operator w_ij = sign * data[k] (eig_extreme "max")
EigInfo eig_max(const Problem* p, double sign, cudaStream_t s);

// ---- energy.cu
// energies of bit-packed spins sb[n][W] (bit (r%32) of word r/32) for replicas r < R
// q2 (optional, uniform-magnitude problems): per replica 2*sum_{i<j} K_ij s_i s_j with
// J = c K, already computed (dense tensor-core energy step); only h/offset are summed here.
void energies_from_bits(Problem* p, const uint32_t* sb, int64_t W, int64_t R,
                        double* energies_dev, cudaStream_t s, const long long* q2 = nullptr);
void pack_states_to_bits(const int8_t* states_dev, int64_t n, int64_t R, int64_t W,
                         uint32_t* sb, cudaStream_t s);
void bits_to_states(const uint32_t* sb, int64_t n, int64_t R, int64_t W, int8_t* states_dev,
                    cudaStream_t s);
void stable_order(const double* energies_dev, int64_t R, int64_t* order_dev, cudaStream_t s);

// CUDA-event timer on one stream (the library's loop_ms)
struct EventTimer {
    cudaEvent_t a = nullptr, b = nullptr;
    cudaStream_t s;
    explicit EventTimer(cudaStream_t st) : s(st) {
        VXQ_CUDA(cudaEventCreate(&a));
        VXQ_CUDA(cudaEventCreate(&b));
    }
    void start() { VXQ_CUDA(cudaEventRecord(a, s)); }
    void stop() { VXQ_CUDA(cudaEventRecord(b, s)); }
    double ms() {
        float v = 0;
        VXQ_CUDA(cudaEventSynchronize(b));
        VXQ_CUDA(cudaEventElapsedTime(&v, a, b));
        return v;
    }
    ~EventTimer() {
        if (a) cudaEventDestroy(a);
        if (b) cudaEventDestroy(b);
    }
};

// ---- dynamics.cu
// exact energies, +-1 states and best-first order from bit-packed spins sb[n][W]
// (x/m outputs must be NULL); the common tail of every solver
void finish_from_bits(Problem* p, int64_t R, int64_t W, const uint32_t* sb,
                      const vxq_run_opts* opts, vxq_outputs* out, cudaStream_t s);
void pa_solve(Problem* p, const vxq_pa_params* prm, const vxq_run_opts* opts, vxq_outputs* out,
              cudaStream_t s);
void sbm_solve(Problem* p, const vxq_sbm_params* prm, const vxq_run_opts* opts,
               vxq_outputs* out, cudaStream_t s);
void sbm_integrate(int64_t n, const int64_t* bt_indptr, const int32_t* bt_indices,
                   const double* bt_data, const double* g, int64_t R, double* Q, double* P,
                   const double* a_sched, int64_t T_, double dt, double a0, double c0,
                   double q_cap, const vxq_run_opts* opts, cudaStream_t s);

// row-partitioned sessions (dynamics.cu)
struct Session;
int64_t exchange_row_bytes(int solver, int64_t R, int prec);
Session* session_create(Problem* p, int solver, const vxq_pa_params* pa,
                        const vxq_sbm_params* sbm, int64_t row_begin, int64_t row_end,
                        int64_t rows_alloc, void* xbuf0, void* xbuf1, const vxq_run_opts* opts,
                        cudaStream_t s);
void session_step(Session* S, int64_t t);
void session_finish(Session* S, vxq_outputs* out, const vxq_run_opts* opts);
void session_set_peers(Session* S, int world, int rank, uint32_t epoch, void* const* xbuf0,
                       void* const* xbuf1, uint64_t* const* flags);
void session_destroy(Session* S);
void session_set_own_stream(Session* S, bool own);

// ---- dense_tc.cu (tcgen05 path)
bool dense_eligible(const Problem* p, int64_t R);
bool dense_general_eligible(const Problem* p, int64_t R);
bool dense_sbm_fp16_ok(double q_cap, double amp);  // |q| stays in the fp16 q-plane range
int sbm_fixed_point_shift(double q_cap, double amp);  // exact SBM path: 2^S scaling of q
int dense_last_kind();  // VXQ_DENSE_KIND_* of the calling thread's last dense loop
void dense_pa_general_loop(Problem* p, int64_t R, int64_t R_pad, int V, int64_t W,
                           const std::vector<double>& sched, float eta, float alpha,
                           uint64_t seed, int64_t rbegin, float* x_il, float* m_il, uint32_t* sb,
                           cudaStream_t s, double* loop_ms, int64_t* launches);
void dense_pa_loop(Problem* p, int64_t R, int64_t R_pad, int V, int64_t W,
                   const std::vector<double>& sched, float eta, float alpha, uint64_t seed,
                   int64_t rbegin, float* x_il, float* m_il, uint32_t* sb, long long* q2,
                   cudaStream_t s, double* loop_ms, int64_t* launches,
                   double* trace_out = nullptr, bool trace_on_dev = false,
                   uint32_t* sb_best = nullptr);
// h == 0 everywhere (cached per problem): the dense path's in-kernel energies are exact
bool problem_h_zero(Problem* p, cudaStream_t s);

void dense_sbm_loop(Problem* p, int64_t R, int64_t R_pad, int V, int64_t W,
                    const std::vector<double>& a_sched, double dt, double a0, double c0,
                    double q_cap, double amp, uint64_t seed, int64_t rbegin, float* q_il,
                    float* p_il, uint32_t* sb, long long* q2, cudaStream_t s, double* loop_ms,
                    int64_t* launches, double* trace_out = nullptr, bool trace_on_dev = false);

// ---- host schedules (bit-exact with the reference's Python expressions)
void pa_schedule(double lam0, int64_t T, double* out);   // lam0 * (1.0 - t / T)
void sbm_schedule(double a0, int64_t T, double* out);    // np.linspace(0.0, a0, T)

// ---- anneal.cu (simulated annealing, annealing.py:24-74)
void sa_solve(Problem* p, const vxq_sa_params* prm, const vxq_run_opts* opts, vxq_outputs* out,
              cudaStream_t s);
void sa_schedule(double T_init, double T_final, int64_t sweeps, double* out);

}  // namespace vxq
