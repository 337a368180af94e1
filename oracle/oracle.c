/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  CPU restatement of the reference's
 * batched multi-replica dynamics loop (qubokit PA / SBM), used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg as the CHECKER.
 * Nothing in the product package may link or call this file.
 *
 * Reference algorithm (read-only, /root/reference/pkg/src/qubokit):
 *   - replica streams      generators.py:35-40, solvers/common.py:64-65
 *                          (numpy Philox4x64-10, key=(seed,0), jumped(r) => ctr word 2 = r)
 *   - PA loop              solvers/parallel_annealing.py:41-45
 *   - SBM integrate        solvers/bifurcation.py:37-47
 *   - sign_pm              model.py:36-38   (sign(0) = +1)
 *   - field_scale (lambda0) model.py:194-200, parallel_annealing.py:23-25
 *
 * Arithmetic order follows numpy's evaluation of the reference lines exactly
 * (each binary op rounds once; compile with -ffp-contract=off so no FMA is
 * formed).  The coupling field is summed per output row over the symmetric
 * CSR in ascending column order, starting from 0.0 -- this is bit-for-bit the
 * order scipy's csc_matvecs uses for `X @ A_csr` (the reference's operator for
 * n > 2048, model.py:185-187), checked in tests/test_oracle.py.
 *
 * Layout: states are replica-major (R, n) row-major, as in the reference.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

/* ---------------- Philox4x64-10 (numpy bit generator) ---------------- */
#define PH_M0 0xD2E7470EE14C6C93ULL
#define PH_M1 0xCA5A826395121157ULL
#define PH_W0 0x9E3779B97F4A7C15ULL
#define PH_W1 0xBB67AE8584CAA73BULL

static void philox4x64_10(const uint64_t ctr_in[4], uint64_t key0, uint64_t key1,
                          uint64_t out[4]) {
    uint64_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint64_t k0 = key0, k1 = key1;
    for (int r = 0; r < 10; ++r) {
        unsigned __int128 p0 = (unsigned __int128)PH_M0 * c0;
        unsigned __int128 p1 = (unsigned __int128)PH_M1 * c2;
        uint64_t n0 = (uint64_t)(p1 >> 64) ^ c1 ^ k0;
        uint64_t n1 = (uint64_t)p1;
        uint64_t n2 = (uint64_t)(p0 >> 64) ^ c3 ^ k1;
        uint64_t n3 = (uint64_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += PH_W0; k1 += PH_W1;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* raw 64-bit draw k of stream rng_stream(seed, replica) */
uint64_t orc_philox_raw(uint64_t seed, uint64_t replica, uint64_t k) {
    uint64_t ctr[4] = {k / 4 + 1, 0, replica, 0}, out[4];
    philox4x64_10(ctr, seed, 0, out);
    return out[k % 4];
}

/* numpy Generator.uniform(lo, hi): lo + (hi - lo) * ((raw >> 11) * 2^-53) */
void orc_uniform(uint64_t seed, uint64_t replica, uint64_t first, int64_t count,
                 double lo, double hi, double* out) {
    double range = hi - lo;
    for (int64_t k = 0; k < count; ++k) {
        uint64_t raw = orc_philox_raw(seed, replica, first + (uint64_t)k);
        double u = (double)(raw >> 11) * (1.0 / 9007199254740992.0);
        out[k] = lo + range * u;
    }
}

/* ---------------- field scale (lambda0 source), model.py:194-200 ----------------
 * row_i = |h_i| + sum over np.add.at(rows) then np.add.at(cols), i.e. the j>i
 * couplings ascending, then the j<i couplings ascending.  COO input i<j sorted. */
double orc_field_scale(int64_t n, int64_t m, const int64_t* rows, const int64_t* cols,
                       const double* values, const double* h, double* row_out) {
    for (int64_t i = 0; i < n; ++i) row_out[i] = fabs(h[i]);
    for (int64_t k = 0; k < m; ++k) row_out[rows[k]] += fabs(values[k]);
    for (int64_t k = 0; k < m; ++k) row_out[cols[k]] += fabs(values[k]);
    double mx = row_out[0];
    for (int64_t i = 1; i < n; ++i) if (row_out[i] > mx) mx = row_out[i];
    return mx;
}

/* ---------------- PA loop, parallel_annealing.py:41-45 ---------------- */
#define PA_BODY(T)                                                                  \
    for (int64_t t = 0; t < steps; ++t) {                                           \
        T lam = lam_sched[t];                                                       \
        for (int64_t r = 0; r < R; ++r) {                                           \
            T* x = X + r * n; T* mm = M + r * n;                                    \
            for (int64_t i = 0; i < n; ++i) sgn[i] = (x[i] >= (T)0) ? (T)1 : (T)-1; \
            for (int64_t i = 0; i < n; ++i) {                                       \
                T f = (T)0;                                                         \
                for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k)                 \
                    f = f + data[k] * sgn[indices[k]];                              \
                T grad = (lam * x[i] + f) + hv[i];                                  \
                T mn = alpha * mm[i] - eta * grad;                                  \
                T xn = x[i] + mn;                                                   \
                xn = xn < (T)-1 ? (T)-1 : (xn > (T)1 ? (T)1 : xn);                  \
                mm[i] = mn; xnew[i] = xn;                                           \
            }                                                                       \
            memcpy(x, xnew, sizeof(T) * n);                                         \
        }                                                                           \
    }

void orc_pa_run_f64(int64_t n, int64_t R, const int64_t* indptr, const int32_t* indices,
                    const double* data, const double* hv, const double* lam_sched,
                    int64_t steps, double eta, double alpha, double* X, double* M,
                    double* sgn, double* xnew) {
    PA_BODY(double)
}

void orc_pa_run_f32(int64_t n, int64_t R, const int64_t* indptr, const int32_t* indices,
                    const float* data, const float* hv, const float* lam_sched,
                    int64_t steps, float eta, float alpha, float* X, float* M,
                    float* sgn, float* xnew) {
    PA_BODY(float)
}

/* ---------------- SBM integrate, bifurcation.py:37-47 ----------------
 * B given as CSR of B^T rows (field_i = sum_j B[j,i] q_j, ascending j), g.
 * P += dt * (-(Q*Q + a0 - a_t) * Q + c0 * (Q @ B + g))
 * Q += (dt * a0) * P;  over = |Q| > q_cap -> clip Q, P = 0                  */
#define SBM_BODY(T)                                                                 \
    for (int64_t t = 0; t < steps; ++t) {                                           \
        T a_t = a_sched[t];                                                         \
        for (int64_t r = 0; r < R; ++r) {                                           \
            T* q = Q + r * n; T* p = P + r * n;                                     \
            for (int64_t i = 0; i < n; ++i) {                                       \
                T f = (T)0;                                                         \
                for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k)                 \
                    f = f + data[k] * q[indices[k]];                                \
                T qi = q[i];                                                        \
                T inner = -((qi * qi + a0) - a_t);                                  \
                T force = inner * qi + c0 * (f + g[i]);                             \
                pnew[i] = p[i] + dt * force;                                        \
            }                                                                       \
            for (int64_t i = 0; i < n; ++i) {                                       \
                T qn = q[i] + dta0 * pnew[i];                                       \
                T pn = pnew[i];                                                     \
                if (fabs((double)qn) > (double)q_cap) {                             \
                    qn = qn < -q_cap ? -q_cap : q_cap;                              \
                    pn = (T)0;                                                      \
                }                                                                   \
                q[i] = qn; p[i] = pn;                                               \
            }                                                                       \
        }                                                                           \
    }

void orc_sbm_run_f64(int64_t n, int64_t R, const int64_t* indptr, const int32_t* indices,
                     const double* data, const double* g, const double* a_sched,
                     int64_t steps, double dt, double a0, double c0, double q_cap,
                     double dta0, double* Q, double* P, double* pnew) {
    SBM_BODY(double)
}

void orc_sbm_run_f32(int64_t n, int64_t R, const int64_t* indptr, const int32_t* indices,
                     const float* data, const float* g, const float* a_sched,
                     int64_t steps, float dt, float a0, float c0, float q_cap,
                     float dta0, float* Q, float* P, float* pnew) {
    SBM_BODY(float)
}

/* ---------------- SA, solvers/annealing.py:24-74 ----------------
 * Replica r = stream rng_stream(seed, rbegin + r):
 *   S = 2 * integers(0, 2, n) - 1   (32-bit half i of the raw draws, low half first; the
 *                                    Lemire step for range 2 is the top bit, no rejection)
 *   U[s, i] = random() from raw draw ceil(n/2) + s*n + i    (chunking keeps stream order)
 *   F = S @ A + h  (CSR ascending column from 0.0, then + h; annealing.py:42-43)
 *   E = energies(S) - offset  (passed in as E0: correctly rounded exact, see energy_exact)
 * sweep s, spin i (annealing.py:56-70):
 *   dE = -2.0 * S_i * F_i;  accept = U < exp(minimum(-dE / T_s, 0.0))
 *   accept: S_i = -S_i; E += dE; F_j += 2.0 * S_i * A_ij  (j in row i)
 *   after each sweep: E < best_E -> best = (E, S)                                      */
void orc_sa_init_spins(int64_t n, uint64_t seed, uint64_t replica, int8_t* S) {
    uint64_t blk[4], q_cached = ~0ULL;
    for (int64_t i = 0; i < n; ++i) {
        uint64_t q = (uint64_t)i >> 1;
        if ((q >> 2) != q_cached) {
            uint64_t ctr[4] = {(q >> 2) + 1, 0, replica, 0};
            philox4x64_10(ctr, seed, 0, blk);
            q_cached = q >> 2;
        }
        uint64_t raw = blk[q & 3];
        uint64_t bit = (i & 1) ? (raw >> 63) : ((raw >> 31) & 1ULL);
        S[i] = bit ? 1 : -1;
    }
}

#define SA_BODY(T)                                                                       \
    for (int64_t r = 0; r < R; ++r) {                                                    \
        const uint64_t rg = (uint64_t)(rbegin + r);                                      \
        int8_t* S = S_work;                                                              \
        orc_sa_init_spins(n, seed, rg, S);                                               \
        for (int64_t i = 0; i < n; ++i) {                                                \
            T f = (T)0;                                                                  \
            for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k)                          \
                f = f + (S[indices[k]] > 0 ? data[k] : -data[k]);                        \
            F[i] = f + hv[i];                                                            \
        }                                                                                \
        double E = E0[r], bestE = E;                                                     \
        memcpy(best + r * n, S, (size_t)n);                                              \
        uint64_t kdraw = (uint64_t)(n + 1) / 2, blk[4], qc = ~0ULL;                      \
        for (int64_t s = 0; s < sweeps; ++s) {                                           \
            const double Tt = temps[s];                                                  \
            for (int64_t i = 0; i < n; ++i) {                                            \
                const uint64_t q = kdraw >> 2;                                           \
                if (q != qc) {                                                           \
                    uint64_t ctr[4] = {q + 1, 0, rg, 0};                                 \
                    philox4x64_10(ctr, seed, 0, blk);                                    \
                    qc = q;                                                              \
                }                                                                        \
                const uint64_t raw = blk[kdraw & 3];                                     \
                ++kdraw;                                                                 \
                const double u = (double)(raw >> 11) * (1.0 / 9007199254740992.0);      \
                const double dE = (-2.0 * (double)S[i]) * (double)F[i];                  \
                double x = -dE / Tt;                                                     \
                if (!isnan(x) && !(x < 0.0)) x = 0.0;                                    \
                if (u < exp(x)) {                                                        \
                    S[i] = (int8_t)-S[i];                                                \
                    E = E + dE;                                                          \
                    const T d2 = (T)(2 * S[i]);                                          \
                    for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k)                   \
                        F[indices[k]] = F[indices[k]] + d2 * data[k];                    \
                }                                                                        \
            }                                                                            \
            if (E < bestE) {                                                             \
                bestE = E;                                                               \
                memcpy(best + r * n, S, (size_t)n);                                      \
            }                                                                            \
        }                                                                                \
        bestE_out[r] = bestE;                                                            \
    }

void orc_sa_run_f64(int64_t n, int64_t R, const int64_t* indptr, const int32_t* indices,
                    const double* data, const double* hv, const double* temps, int64_t sweeps,
                    uint64_t seed, int64_t rbegin, const double* E0, int8_t* best,
                    double* bestE_out, double* F, int8_t* S_work) {
    SA_BODY(double)
}

void orc_sa_run_f32(int64_t n, int64_t R, const int64_t* indptr, const int32_t* indices,
                    const float* data, const float* hv, const double* temps, int64_t sweeps,
                    uint64_t seed, int64_t rbegin, const double* E0, int8_t* best,
                    double* bestE_out, float* F, int8_t* S_work) {
    SA_BODY(float)
}
