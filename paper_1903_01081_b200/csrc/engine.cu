// B200 EMT step-loop engine: persistent sm_100a kernel + C ABI (include/emt_b200.h).
//
// Design: one warp owns one scenario lane for the whole run.
// The lane's arena (the reference's slot layout, proj/docs/schedule_format.md)
// and its constant-table column live in shared memory; the warp walks the
// schedule's layers in order (proj/src/exec.cpp:364-374), its 32 threads
// taking the layer's processes in parallel (write sets are disjoint per layer,
// proj/src/schedule.cpp:229-254), with __syncwarp between layers. The
// factorize / solve singletons run warp-cooperatively: sparse LU rows in the
// reference's up-looking order and level-scheduled triangular sweeps that keep
// every row's subtraction sequence, so results are bit-identical to the
// reference's lu_factor / lu_solve (proj/src/sparse.cpp:79-172). Compiled with
// -fmad=false: no FMA contraction, like the reference's -ffp-contract=off.
// Scenario lanes are independent, so there is no grid-wide synchronisation:
// a launch advances every lane by N passes and streams waveform rows to HBM.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <future>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "../../include/emt_b200.h"
#include "codegen.hpp"
#include "host_schedule.hpp"
#include "jit.hpp"

namespace emtb200 {

// Engine-side developer switches (kernel forcing, profiling counters, line-coupling
// mode): read only in a developer build (build.py --dev), like the generator knobs.
inline const char* dev_env(const char* name) {
#ifdef EMTB200_DEV_KNOBS
    return std::getenv(name);
#else
    (void)name;
    return nullptr;
#endif
}

constexpr unsigned kFull = 0xffffffffu;
constexpr double kDefaultDivergence = 1e12;  // kDivergenceLimit, kernels.hpp:24

// Per-lane error record in global memory: code (1+ErrorCode), step, index.
struct LaneError {
    int code, step, index, layer;
};

// Argument block of the generated kernel (layout mirrored in codegen.cpp).
struct CgArgs {
    double* arena;
    const double* ctab;
    double* waves;
    unsigned char* refac;
    int* lane_err;
    int* events;
    int* n_events;
    int max_events;
    int step0, nsteps, row0;
    double div_limit;
    double* ring;  // line-end history mirror, lane-major [batch lane][ring slot - ring_lo]
    long long ring_lo, ring_cols;
    unsigned int* progress;  // persistent line-coupled run: passes completed per CTA (else null)
    int min_k, nblocks;
    long long* prof;         // phase profiler accumulators (EMTB200_CG_PROF=1), else null
    const double* srctab;    // this launch's AC source values [pass][source] (emt_src_kernel)
    int prog_off;            // this engine's first CTA in the (possibly shared) progress array
    int sys_scope;           // 1: peers on other GPUs (system-scope acquire/release, uncached ring reads)
    int* pick;               // full-chip launch: lane-group claim counter (else null, see launch_ctas)
};

struct DevPlan {
    int W;          // lanes owned by this engine
    int lane_begin; // first owned lane of the batch (line-end peers are batch lane indices)
    double* ring;   // line-end history mirror [batch lane][ring_cols], see emt_engine_ring
    int ring_lo, ring_cols;
    int lpb;        // lanes (warps) per block
    int use_smem;   // arena + consts in shared memory (else lane-major global scratch)
    int lane_stride;  // doubles per lane in the working area
    int ext_pad;      // consts start inside the lane's area
    int extent, consts, nch, nlatch, layers, nodes, comps, dim, nnz, nwatch;
    int v_base, mat, l, u, scratch, fcount;
    int n_fwd, n_bwd;
    double dt, div_limit;

    const int* layer_begin;  // layers+1, into the regular process list
    const int* layer_flags;  // bit0 factorize, bit1 solve
    const int4* procA;       // code, out, out2, state
    const int4* procB;       // par, par_len, in_base, in_count
    const int* proc_id;
    const int* port_slot;
    const double* port_sign;
    const int* ch_slot;
    const int* latch_live;
    const int* latch_shadow;
    const int* row_ptr;
    const int* col_idx;
    const int* ment_ptr;
    const int* ment_slot;
    const double* ment_sign;
    const int* gat_ptr;
    const int* gat_slot;
    const int* fin;  // 5 per component
    const int* watch;
    const int* l_row_ptr;
    const int* l_col;
    const int* u_row_ptr;
    const int* u_col;
    const int* fwd_ptr;
    const int* fwd_rows;
    const int* bwd_ptr;
    const int* bwd_rows;

    double* arena;         // extent x W (slot-major, lanes innermost): resident state between launches
    const double* ctab;    // consts x W
    double* work;          // lane-major scratch when !use_smem: W x lane_stride
    double* waves;         // rows x nch x W
    unsigned char* refactored;  // per recorded row: some lane refactorized
    LaneError* lane_err;        // per lane
    int* events;                // triples step, lane, process
    int* n_events;
    int max_events;
};

__device__ __forceinline__ double rd(const double* A, int slot) { return slot < 0 ? 0.0 : A[slot]; }

// glibc's cos, operation for operation (libmcos.cuh): the reference's std::cos bits
__device__ __forceinline__ int emt_lo32(double d) { return __double2loint(d); }
#define EMT_LIBMCOS_TEXT(...) __VA_ARGS__
#define EMT_HD __device__ __forceinline__
#define EMT_TABLE __device__ const
#include "libmcos.cuh"
#undef EMT_LIBMCOS_TEXT
#undef EMT_HD
#undef EMT_TABLE

__global__ void emt_cos_kernel(const double* __restrict__ x, double* __restrict__ y, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        y[i] = emt_libm_cos(x[i]);
}

// kern::source_value (proj/include/emtgrid/kernels.hpp:68-70)
__device__ __forceinline__ double source_value(double mag, double omega, double phase, double t) {
    return omega == 0.0 ? mag : mag * emt_libm_cos(omega * t + phase);
}

// One non-singleton process for this lane: Engine::run_proc, proj/src/exec.cpp:77-311.
__device__ __forceinline__ void run_regular(const DevPlan& P, double* __restrict__ A, const double* __restrict__ C,
                                            int k, double t, int step, int lane) {
    const int4 a = __ldg(&P.procA[k]);  // code, out, out2, state
    const int4 b = __ldg(&P.procB[k]);  // par, par_len, in_base, in_count
    const int* in = P.port_slot + b.z;
    const double* sg = P.port_sign + b.z;
    const double* par = C + b.x;
    double* st = A + a.w;
    switch (a.x) {
        case kNortonResistor:
            A[a.y] = par[0];
            A[a.z] = 0.0;
            break;
        case kNortonInductor: {  // h = i_prev + g*v_prev (kernels.hpp:71-73)
            const double vs = rd(A, __ldg(in + 1)) - rd(A, __ldg(in + 0));
            const double g = par[0];
            A[a.y] = g;
            A[a.z] = rd(A, __ldg(in + 2)) + g * vs;
            break;
        }
        case kNortonCapacitor: {  // h = -i_prev - g*v_prev (kernels.hpp:74-76)
            const double vs = rd(A, __ldg(in + 1)) - rd(A, __ldg(in + 0));
            const double g = par[0];
            A[a.y] = g;
            A[a.z] = -rd(A, __ldg(in + 2)) - g * vs;
            break;
        }
        case kNortonSeriesRL: {  // h = decay*i_prev + g*v_prev (kernels.hpp:77-79)
            const double vs = rd(A, __ldg(in + 1)) - rd(A, __ldg(in + 0));
            const double g = par[0];
            A[a.y] = g;
            A[a.z] = par[1] * rd(A, __ldg(in + 2)) + g * vs;
            break;
        }
        case kNortonVoltageSource: {
            const double g = par[0];
            A[a.y] = g;
            A[a.z] = g * source_value(par[1], par[2], par[3], t);
            break;
        }
        case kNortonCurrentSource:
            A[a.y] = 0.0;
            A[a.z] = source_value(par[0], par[1], par[2], t);
            break;
        case kNortonControlledSource:
            A[a.y] = 0.0;
            A[a.z] = par[0] * (b.w > 3 ? rd(A, __ldg(in + 3)) : 0.0);
            break;
        case kNortonSwitch: {  // proj/src/exec.cpp:151-165; state = [now, changed]
            int now = par[2] != 0.0 ? 1 : 0;
            for (int j = 3; j < b.y; ++j)
                if (t >= par[j]) now ^= 1;
            const double changed = static_cast<double>(now) != st[0] ? 1.0 : 0.0;
            st[1] = changed;
            st[0] = static_cast<double>(now);
            A[a.y] = now != 0 ? par[0] : par[1];
            A[a.z] = 0.0;
            if (changed != 0.0 && P.events != nullptr) {
                const int slot = atomicAdd(P.n_events, 1);
                if (slot < P.max_events) {
                    P.events[3 * slot + 0] = step;
                    P.events[3 * slot + 1] = lane;
                    P.events[3 * slot + 2] = __ldg(&P.proc_id[k]);
                }
            }
            break;
        }
        case kNortonBergeron: {  // line end (extension): oracle/emt_oracle.c case K_BERG
            const double vs = rd(A, __ldg(in + 1)) - rd(A, __ldg(in + 0));
            const double beta = par[0] * vs + A[a.z];
            const int L = static_cast<int>(par[6]);
            const int w = step % L;
            st[w] = beta;  // the lane's arena copy (written back at launch end)
            const size_t cols = static_cast<size_t>(P.ring_cols);
            P.ring[static_cast<size_t>(P.lane_begin + lane) * cols + static_cast<size_t>(a.w - P.ring_lo + w)] = beta;
            const int K = static_cast<int>(par[3]);
            const size_t pl = static_cast<size_t>(par[4]);
            const size_t pr = static_cast<size_t>(par[5]) - static_cast<size_t>(P.ring_lo);
            int q1 = (step + 1 - K) % L;
            if (q1 < 0) q1 += L;
            const int q0 = q1 == 0 ? L - 1 : q1 - 1;
            // entries of earlier launches (a launch spans < K passes): read through L2
            const double b1 = __ldcg(P.ring + pl * cols + pr + static_cast<size_t>(q1));
            const double b0 = __ldcg(P.ring + pl * cols + pr + static_cast<size_t>(q0));
            A[a.y] = 0.0;
            A[a.z] = -(par[1] * b1 + par[2] * b0);
            break;
        }
        case kInjectionPair: {
            const double h = rd(A, __ldg(in + 0));
            A[a.y] = h;
            A[a.y + 1] = -h;
            break;
        }
        case kCtlGain:
            A[a.y] = par[0] * (__ldg(sg + 0) * rd(A, __ldg(in + 0)));
            break;
        case kCtlSum: {  // signs applied before sequential accumulation (exec.cpp:245-253)
            double acc = 0.0;
            for (int j = 0; j < b.w; ++j) acc += __ldg(sg + j) * rd(A, __ldg(in + j));
            A[a.y] = acc;
            break;
        }
        case kCtlIntegrator: {  // y = y_prev + dt/2 (u + u_prev) (kernels.hpp:80-82)
            const double u = __ldg(sg + 0) * rd(A, __ldg(in + 0));
            const double y = st[0] + par[0] * (u + st[1]);
            st[0] = y;
            st[1] = u;
            A[a.y] = y;
            break;
        }
        case kCtlFirstOrderLag: {  // kernels.hpp:83-85
            const double u = __ldg(sg + 0) * rd(A, __ldg(in + 0));
            const double y = par[0] * st[0] + par[1] * (u + st[1]);
            st[0] = y;
            st[1] = u;
            A[a.y] = y;
            break;
        }
        case kCtlLimiter: {  // kernels.hpp:86-88
            const double u = __ldg(sg + 0) * rd(A, __ldg(in + 0));
            const double lo = par[0], hi = par[1];
            A[a.y] = u < lo ? lo : (u > hi ? hi : u);
            break;
        }
        case kCtlPiController: {  // exec.cpp:283-292
            const double u = __ldg(sg + 0) * rd(A, __ldg(in + 0));
            st[0] = st[0] + par[1] * (u + st[1]);
            st[1] = u;
            A[a.y] = par[0] * u + st[0];
            break;
        }
        case kCtlComparator:
            A[a.y] = __ldg(sg + 0) * rd(A, __ldg(in + 0)) >= __ldg(sg + 1) * rd(A, __ldg(in + 1)) ? 1.0 : 0.0;
            break;
        case kCtlConstant:
            A[a.y] = par[0];
            break;
        case kCtlDelay:
            A[a.y] = __ldg(sg + 0) * rd(A, __ldg(in + 0));
            break;
        default:
            break;
    }
}

__device__ __forceinline__ void lane_fail(const DevPlan& P, int lane, int code, int step, int index, int layer,
                                          int tl) {
    if (tl == 0) {
        LaneError e{code, step, index, layer};
        P.lane_err[lane] = e;
    }
}

// FactorizeSystem for one lane (exec.cpp:175-204 + lu_factor, sparse.cpp:79-145).
// Refactorizing only lanes whose watch slots are set gives the same factors
// the reference computes for every lane (unchanged lanes re-derive identical
// values); the per-row `refactored` flag reproduces its global factor_count.
__device__ int warp_factorize(const DevPlan& P, double* __restrict__ A, int tl, int lane, int step, int row,
                              int layer) {
    bool set = false;
    for (int q = tl; q < P.nwatch; q += 32) set |= (A[__ldg(&P.watch[q])] != 0.0);
    if (!__any_sync(kFull, set)) return 0;

    double* G = A + P.mat;
    for (int k = tl; k < P.nnz; k += 32) {
        double d = 0.0;
        for (int q = __ldg(&P.ment_ptr[k]); q < __ldg(&P.ment_ptr[k + 1]); ++q)
            d += __ldg(&P.ment_sign[q]) * A[__ldg(&P.ment_slot[q])];
        G[k] = d;
    }
    __syncwarp();
    double m = 0.0;  // max |A| of the lane, sparse.cpp:84-90
    for (int k = tl; k < P.nnz; k += 32) {
        const double x = fabs(G[k]);
        m = m < x ? x : m;
    }
    for (int off = 16; off > 0; off >>= 1) {
        const double o = __shfl_xor_sync(kFull, m, off);
        m = m < o ? o : m;
    }
    double* S = A + P.scratch;
    double* Lv = A + P.l;
    double* Uv = A + P.u;
    for (int i = 0; i < P.dim; ++i) {
        const int lb = __ldg(&P.l_row_ptr[i]), le = __ldg(&P.l_row_ptr[i + 1]);
        const int ub = __ldg(&P.u_row_ptr[i]), ue = __ldg(&P.u_row_ptr[i + 1]);
        for (int k = lb + tl; k < le; k += 32) S[__ldg(&P.l_col[k])] = 0.0;
        for (int k = ub + tl; k < ue; k += 32) S[__ldg(&P.u_col[k])] = 0.0;
        __syncwarp();
        for (int k = __ldg(&P.row_ptr[i]) + tl; k < __ldg(&P.row_ptr[i + 1]); k += 32)
            S[__ldg(&P.col_idx[k])] = G[k];
        __syncwarp();
        for (int k = lb; k < le; ++k) {
            const int col = __ldg(&P.l_col[k]);
            const int cb = __ldg(&P.u_row_ptr[col]), ce = __ldg(&P.u_row_ptr[col + 1]);
            const double lik = S[col] / Uv[cb];
            if (tl == 0) Lv[k] = lik;
            for (int j = cb + 1 + tl; j < ce; j += 32) S[__ldg(&P.u_col[j])] -= lik * Uv[j];
            __syncwarp();
        }
        for (int k = ub + tl; k < ue; k += 32) Uv[k] = S[__ldg(&P.u_col[k])];
        __syncwarp();
        if (!(fabs(Uv[ub]) > 1e-12 * m)) {
            lane_fail(P, lane, 8 /*SingularMatrix*/, step, i, layer, tl);
            return 1;
        }
    }
    for (int q = tl; q < P.nwatch; q += 32) A[__ldg(&P.watch[q])] = 0.0;
    if (tl == 0) {
        A[P.fcount] += 1.0;
        P.refactored[row] = 1;
    }
    __syncwarp();
    return 0;
}

// SolveSystem for one lane (exec.cpp:205-239 + lu_solve, sparse.cpp:147-172).
__device__ int warp_solve(const DevPlan& P, double* __restrict__ A, int tl, int lane, int step, int layer) {
    double* v = A + P.v_base;
    for (int node = tl; node < P.nodes; node += 32) {  // canonical gather order, exec.cpp:207-214
        double acc = 0.0;
        for (int q = __ldg(&P.gat_ptr[node]); q < __ldg(&P.gat_ptr[node + 1]); ++q) acc += A[__ldg(&P.gat_slot[q])];
        v[node] = acc;
    }
    __syncwarp();
    if (P.nodes > 0) {
        const double* Lv = A + P.l;
        const double* Uv = A + P.u;
        for (int lv = 0; lv < P.n_fwd; ++lv) {
            for (int r = __ldg(&P.fwd_ptr[lv]) + tl; r < __ldg(&P.fwd_ptr[lv + 1]); r += 32) {
                const int i = __ldg(&P.fwd_rows[r]);
                double x = v[i];
                for (int k = __ldg(&P.l_row_ptr[i]); k < __ldg(&P.l_row_ptr[i + 1]); ++k)
                    x -= Lv[k] * v[__ldg(&P.l_col[k])];
                v[i] = x;
            }
            __syncwarp();
        }
        for (int lv = 0; lv < P.n_bwd; ++lv) {
            for (int r = __ldg(&P.bwd_ptr[lv]) + tl; r < __ldg(&P.bwd_ptr[lv + 1]); r += 32) {
                const int i = __ldg(&P.bwd_rows[r]);
                const int ub = __ldg(&P.u_row_ptr[i]);
                double x = v[i];
                for (int k = ub + 1; k < __ldg(&P.u_row_ptr[i + 1]); ++k) x -= Uv[k] * v[__ldg(&P.u_col[k])];
                x /= Uv[ub];
                v[i] = x;
            }
            __syncwarp();
        }
    }
    for (int c = tl; c < P.comps; c += 32) {  // i = g (v_b - v_a) + h, exec.cpp:220-228
        const int* f = P.fin + 5 * c;
        const double vs = rd(A, __ldg(f + 4)) - rd(A, __ldg(f + 3));
        A[__ldg(f + 0)] = A[__ldg(f + 1)] * vs + A[__ldg(f + 2)];
    }
    int bad = INT_MAX;  // first diverged node index, exec.cpp:229-237
    for (int node = tl; node < P.nodes; node += 32)
        if (!(fabs(v[node]) <= P.div_limit)) bad = min(bad, node);
    for (int off = 16; off > 0; off >>= 1) bad = min(bad, __shfl_xor_sync(kFull, bad, off));
    __syncwarp();
    if (bad != INT_MAX) {
        lane_fail(P, lane, 7 /*NonFiniteState*/, step, bad, layer, tl);
        return 1;
    }
    return 0;
}

__global__ void __launch_bounds__(1024, 1)
emt_step_kernel(const DevPlan P, const int step0, const int nsteps, const int row0) {
    extern __shared__ double smem[];
    const int wid = threadIdx.x >> 5;
    const int tl = threadIdx.x & 31;
    const int lane = blockIdx.x * P.lpb + wid;
    if (lane >= P.W) return;
    if (P.lane_err[lane].code != 0) return;  // lane already failed: frozen

    double* A = P.use_smem ? smem + static_cast<size_t>(wid) * P.lane_stride
                           : P.work + static_cast<size_t>(lane) * P.lane_stride;
    double* C = A + P.ext_pad;
    for (int s = tl; s < P.extent; s += 32) A[s] = P.arena[static_cast<size_t>(s) * P.W + lane];
    for (int s = tl; s < P.consts; s += 32) C[s] = P.ctab[static_cast<size_t>(s) * P.W + lane];
    __syncwarp();

    int err = 0;
    int it = 0;
    for (; it < nsteps; ++it) {
        const int step = step0 + it;
        const int row = row0 + it;
        const double t = static_cast<double>(step + 1) * P.dt;  // exec.cpp:366
        for (int layer = 0; layer < P.layers; ++layer) {
            const int e = __ldg(&P.layer_begin[layer + 1]);
            for (int k = __ldg(&P.layer_begin[layer]) + tl; k < e; k += 32) run_regular(P, A, C, k, t, step, lane);
            const int fl = __ldg(&P.layer_flags[layer]);
            if (fl != 0) {
                __syncwarp();
                if (fl & 1) err = warp_factorize(P, A, tl, lane, step, row, layer);
                if (!err && (fl & 2)) err = warp_solve(P, A, tl, lane, step, layer);
                if (err) break;
            }
            __syncwarp();
        }
        if (err) break;
        // record (exec.cpp:313-321) then latch (exec.cpp:323-329)
        double* wrow = P.waves + static_cast<size_t>(row) * P.nch * P.W;
        for (int ch = tl; ch < P.nch; ch += 32) wrow[static_cast<size_t>(ch) * P.W + lane] = rd(A, __ldg(&P.ch_slot[ch]));
        for (int q = tl; q < P.nlatch; q += 32) A[__ldg(&P.latch_shadow[q])] = A[__ldg(&P.latch_live[q])];
        __syncwarp();
    }
    for (int s = tl; s < P.extent; s += 32) P.arena[static_cast<size_t>(s) * P.W + lane] = A[s];
}

#include "system_kernel.cuh"

// ----------------------------------------------------------------- host side

thread_local std::string g_last_error;

emt_status set_error(int code, const std::string& msg) {
    g_last_error = msg;
    return static_cast<emt_status>(code);
}

#define CUDA_TRY(expr)                                                                              \
    do {                                                                                            \
        cudaError_t _e = (expr);                                                                    \
        if (_e != cudaSuccess)                                                                      \
            return set_error(EMT_CUDA_ERROR, std::string(#expr) + ": " + cudaGetErrorString(_e));  \
    } while (0)

}  // namespace emtb200

using namespace emtb200;

// A specialised kernel being generated and compiled on a host thread while the
// engine already runs the (bit-identical) generic kernel (EMT_FLAG_ASYNC_JIT).
struct PendingJit {
    std::future<void> done;
    GeneratedKernel gen;
    JitModule jit;
    Failure fail;
    std::string log;
    double gen_s = 0.0;
    bool ok = false;
};

struct emt_engine {
    Schedule sched;
    int device = 0;
    int lane_begin = 0;
    int W = 1;  // lanes owned
    int width = 1;  // lanes of the whole batch (the caller's arena / const-table width)
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;  // D2H of finished waveform chunks (emt_engine_run)
    cudaStream_t h2d_stream = nullptr;   // staged batch uploads (emt_engine_stage)
    cudaEvent_t stage_done = nullptr, commit_done = nullptr;
    double* d_stage_arena = nullptr;     // next batch, lane slice (extent x W)
    double* d_stage_ctab = nullptr;      // next batch constants (consts x W)
    double* d_stage_ring = nullptr;      // next batch ring mirror (width x cols)
    std::vector<double> stage_ring_host;
    bool staged = false, staged_ctab = false;
    std::vector<double> staged_fcount;
    int staged_base_fc = 0;
    std::vector<int> inv_slots;          // constant slots compiled in as immediates ...
    std::vector<double> inv_vals;        // ... and their values (emt_engine_load checks them)
    std::vector<cudaEvent_t> chunk_done;
    DevPlan plan{};
    std::vector<void*> allocations;
    size_t smem_bytes = 0;
    int grid = 1;
    int block = 32;
    int step = 0;       // absolute next pass index
    int rows = 0;       // recorded rows
    int capacity = 0;   // rows the waveform store can hold
    double* d_waves = nullptr;
    unsigned char* d_refactored = nullptr;
    int launches = 0;
    int max_chunk = INT_MAX;  // passes per launch; < K when line ends couple lanes across CTAs
    double* d_ring = nullptr;   // line-end history mirror (owned unless attached)
    bool ring_owned = true;
    bool ring_shared = false;  // mirror shared with other engines (attach_lines): write own rows only
    unsigned int* d_progress = nullptr;  // persistent line-coupled mode: per-CTA pass counters
    bool progress_owned = true;
    int prog_off = 0, prog_total = 0;    // shared progress array (emt_engine_attach_lines)
    int sys_scope = 0;
    long long* d_prof = nullptr;         // 32 warps x 64 markers of cycle sums (profiling builds)
    double* d_srctab = nullptr;          // per-launch AC source table (gen.nsrc columns)
    size_t srctab_cap = 0;               // doubles
    bool persistent_lines = false;
    int min_k = 0;
    int failed = 0;
    int max_events = 1 << 16;
    double divergence_limit = kDefaultDivergence;
    std::vector<double> host_ctab;       // consts x W (this engine's lanes)
    int kernel_mode = EMT_KERNEL_GENERIC;
    SysPlan sys{};               // EMT_KERNEL_SYSTEM tables (system_kernel.cuh)
    size_t sys_smem = 0;
    GeneratedKernel gen;
    JitModule jit;
    std::string summary;
    std::vector<double> initial_fcount;  // per owned lane, from the initial arena
    int base_factor_count = 0;           // global lane 0's initial fcount (ExecStats, exec.cpp:376)

    std::unique_ptr<PendingJit> pending;  // async JIT in flight (EMT_FLAG_ASYNC_JIT)
    int claim_grid = 0;                   // full-chip launch of the specialised kernel: CTAs (= SMs), else 0
    size_t claim_smem = 0;                // its dynamic shared memory (forces one CTA per SM)
    int* d_pick = nullptr;                // [0] CTAs started, [1 + g] lane group g taken (codegen.cpp bid_code)
    int switched_at = -1;                 // pass at which the engine moved to the specialised kernel

    ~emt_engine() {
        if (pending && pending->done.valid()) pending->done.wait();  // the thread reads sched
        if (device >= 0) cudaSetDevice(device);
        if (pending && pending->ok && pending->jit.module && driver()) driver()->ModuleUnload(pending->jit.module);
        if (jit.module && driver()) driver()->ModuleUnload(jit.module);
        for (void* p : allocations) cudaFree(p);
        if (d_ring && ring_owned) cudaFree(d_ring);
        if (d_progress && progress_owned) cudaFree(d_progress);
        if (d_prof) cudaFree(d_prof);
        if (d_srctab) cudaFree(d_srctab);
        if (d_waves) cudaFree(d_waves);
        if (d_pick) cudaFree(d_pick);
        if (d_refactored) cudaFree(d_refactored);
        for (cudaEvent_t ev : chunk_done) cudaEventDestroy(ev);
        if (copy_stream) cudaStreamDestroy(copy_stream);
        if (h2d_stream) cudaStreamDestroy(h2d_stream);
        if (stage_done) cudaEventDestroy(stage_done);
        if (commit_done) cudaEventDestroy(commit_done);
        if (d_stage_arena) cudaFree(d_stage_arena);
        if (d_stage_ctab) cudaFree(d_stage_ctab);
        if (d_stage_ring) cudaFree(d_stage_ring);
        if (stream) cudaStreamDestroy(stream);
    }

    template <typename T>
    emt_status upload(const std::vector<T>& host, const T*& dev) {
        T* p = nullptr;
        const size_t bytes = std::max<size_t>(sizeof(T), host.size() * sizeof(T));
        CUDA_TRY(cudaMalloc(&p, bytes));
        allocations.push_back(p);
        if (!host.empty()) CUDA_TRY(cudaMemcpy(p, host.data(), host.size() * sizeof(T), cudaMemcpyHostToDevice));
        dev = p;
        return EMT_OK;
    }
};

namespace {

/// CTAs of the specialised kernel: gen.lpc scenario lanes each (32, or 16 / 8)
int cta_count(const emt_engine* e) {
    const int lpc = e->gen.lpc > 0 ? e->gen.lpc : 32;
    return (e->W + lpc - 1) / lpc;
}

#define EMT_TRY(expr)                          \
    do {                                       \
        emt_status _s = (expr);                \
        if (_s != EMT_OK) return _s;           \
    } while (0)

/// Checks done by interpret before stepping (exec.cpp:340-357).
emt_status validate(const Schedule& s, int64_t initial_len, int width) {
    if (initial_len != static_cast<int64_t>(s.extent) * width)
        return set_error(EMT_DIMENSION_MISMATCH, "initial state size " + std::to_string(initial_len) +
                                                     " does not match extent " + std::to_string(s.extent) +
                                                     " x width " + std::to_string(width));
    for (const Proc& p : s.procs) {
        if (p.code < 0 || p.code >= kKernelCount)
            return set_error(EMT_UNKNOWN_KIND, "process " + std::to_string(p.id) + ": kernel code " +
                                                   std::to_string(p.code) + " is not registered");
    }
    if (static_cast<int>(s.l_col.size()) != s.l_nnz || static_cast<int>(s.u_col.size()) != s.u_nnz)
        return set_error(EMT_MALFORMED_DOCUMENT, "schedule LU fill sizes are inconsistent");
    return EMT_OK;
}

emt_status build_plan(emt_engine* e, const double* const_table, int width, const double* initial) {
    Schedule& s = e->sched;
    DevPlan& P = e->plan;
    const int W = e->W;
    P.W = W;
    P.lane_begin = e->lane_begin;
    P.extent = s.extent;
    P.consts = s.consts;
    P.nch = static_cast<int>(s.channel_slot.size());
    P.nlatch = static_cast<int>(s.latch_live.size());
    P.layers = s.layers;
    P.nodes = s.nodes;
    P.comps = s.comps;
    P.dim = s.dim;
    P.nnz = static_cast<int>(s.col_idx.size());
    P.nwatch = static_cast<int>(s.watch.size());
    P.v_base = s.v_base;
    P.mat = s.matrix;
    P.l = s.l;
    P.u = s.u;
    P.scratch = s.scratch;
    P.fcount = s.fcount;
    P.dt = s.dt;
    P.div_limit = e->divergence_limit;

    // regular processes per layer + singleton flags
    std::vector<int4> pa, pb;
    std::vector<int> pid, layer_begin{0}, layer_flags;
    for (int L = 0; L < s.layers; ++L) {
        int flags = 0;
        for (int k = s.layer_begin[static_cast<size_t>(L)]; k < s.layer_begin[static_cast<size_t>(L) + 1]; ++k) {
            const Proc& p = s.procs[static_cast<size_t>(k)];
            if (p.code == kFactorizeSystem) { flags |= 1; continue; }
            if (p.code == kSolveSystem) { flags |= 2; continue; }
            pa.push_back(make_int4(p.code, p.out, p.out2, p.state));
            pb.push_back(make_int4(p.par, p.par_len, p.in_base, p.in_count));
            pid.push_back(p.id);
        }
        layer_begin.push_back(static_cast<int>(pa.size()));
        layer_flags.push_back(flags);
    }
    std::vector<int> fwd_ptr, fwd_rows, bwd_ptr, bwd_rows;
    triangular_levels(s, fwd_ptr, fwd_rows, bwd_ptr, bwd_rows);
    P.n_fwd = static_cast<int>(fwd_ptr.size()) - 1;
    P.n_bwd = static_cast<int>(bwd_ptr.size()) - 1;
    std::vector<int> fin = s.finalize;

    EMT_TRY(e->upload(layer_begin, P.layer_begin));
    EMT_TRY(e->upload(layer_flags, P.layer_flags));
    EMT_TRY(e->upload(pa, P.procA));
    EMT_TRY(e->upload(pb, P.procB));
    EMT_TRY(e->upload(pid, P.proc_id));
    EMT_TRY(e->upload(s.port_slot, P.port_slot));
    EMT_TRY(e->upload(s.port_sign, P.port_sign));
    EMT_TRY(e->upload(s.channel_slot, P.ch_slot));
    EMT_TRY(e->upload(s.latch_live, P.latch_live));
    EMT_TRY(e->upload(s.latch_shadow, P.latch_shadow));
    EMT_TRY(e->upload(s.row_ptr, P.row_ptr));
    EMT_TRY(e->upload(s.col_idx, P.col_idx));
    EMT_TRY(e->upload(s.mentry_ptr, P.ment_ptr));
    EMT_TRY(e->upload(s.mentry_slot, P.ment_slot));
    EMT_TRY(e->upload(s.mentry_sign, P.ment_sign));
    EMT_TRY(e->upload(s.gather_ptr, P.gat_ptr));
    EMT_TRY(e->upload(s.gather_slot, P.gat_slot));
    EMT_TRY(e->upload(fin, P.fin));
    EMT_TRY(e->upload(s.watch, P.watch));
    EMT_TRY(e->upload(s.l_row_ptr, P.l_row_ptr));
    EMT_TRY(e->upload(s.l_col, P.l_col));
    EMT_TRY(e->upload(s.u_row_ptr, P.u_row_ptr));
    EMT_TRY(e->upload(s.u_col, P.u_col));
    EMT_TRY(e->upload(fwd_ptr, P.fwd_ptr));
    EMT_TRY(e->upload(fwd_rows, P.fwd_rows));
    EMT_TRY(e->upload(bwd_ptr, P.bwd_ptr));
    EMT_TRY(e->upload(bwd_rows, P.bwd_rows));

    // lane slice of the const table and the initial arena (slot-major, lanes innermost)
    std::vector<double> ctab(static_cast<size_t>(s.consts) * W), arena(static_cast<size_t>(s.extent) * W);
    const double* src_c = const_table != nullptr ? const_table : s.const_table.data();
    for (int k = 0; k < s.consts; ++k)
        for (int l = 0; l < W; ++l)
            ctab[static_cast<size_t>(k) * W + l] =
                src_c[static_cast<size_t>(k) * width + static_cast<size_t>(e->lane_begin + l)];
    for (int k = 0; k < s.extent; ++k)
        for (int l = 0; l < W; ++l)
            arena[static_cast<size_t>(k) * W + l] =
                initial[static_cast<size_t>(k) * width + static_cast<size_t>(e->lane_begin + l)];
    e->host_ctab = ctab;
    for (int k = 0; k < s.consts; ++k) {
        const double* row = ctab.data() + static_cast<size_t>(k) * W;
        bool inv = true;
        for (int l = 1; l < W && inv; ++l) inv = std::memcmp(&row[l], &row[0], sizeof(double)) == 0;
        if (inv) {
            e->inv_slots.push_back(k);
            e->inv_vals.push_back(row[0]);
        }
    }
    // Bergeron line ends read peer rings written >= K-1 passes earlier: a launch
    // may span at most K-1 passes so that every entry it reads was written by an
    // earlier launch (the kernel boundary orders the cross-CTA stores; across
    // GPUs the ring exchange between launches does), and the ring must hold the
    // 2K-1 entries live across one launch. Peers may be any lane of the batch:
    // their rings are read from the mirror, which emt_engine_ring exposes.
    int ring_lo = INT_MAX, ring_hi = -1;
    for (const Proc& p : s.procs) {
        if (p.code != kNortonBergeron) continue;
        if (p.par_len < 7 || p.state < 0 || p.state_len < 1)
            return set_error(EMT_MALFORMED_DOCUMENT, "line end " + std::to_string(p.id) + ": bad record");
        ring_lo = std::min(ring_lo, p.state);
        ring_hi = std::max(ring_hi, p.state + p.state_len);
        for (int l = 0; l < W; ++l) {
            auto c = [&](int j) { return ctab[static_cast<size_t>(p.par + j) * W + l]; };
            const int K = static_cast<int>(c(3)), L = static_cast<int>(c(6));
            const long long pl = static_cast<long long>(c(4));
            if (K < 2 || L != p.state_len || L < 2 * K - 1 || pl < 0 || pl >= width)
                return set_error(EMT_MALFORMED_DOCUMENT, "line end " + std::to_string(p.id) + " lane " +
                                                             std::to_string(e->lane_begin + l) +
                                                             ": needs K >= 2, ring L >= 2K-1 and a peer lane in the batch");
            e->max_chunk = std::min(e->max_chunk, K - 1);
        }
    }
    P.ring = nullptr;
    P.ring_lo = 0;
    P.ring_cols = 0;
    if (ring_hi > ring_lo) {
        for (const Proc& p : s.procs) {  // peer ring slots must lie in the mirrored range
            if (p.code != kNortonBergeron) continue;
            for (int l = 0; l < W; ++l) {
                const int pr = static_cast<int>(ctab[static_cast<size_t>(p.par + 5) * W + l]);
                if (pr < ring_lo || pr + p.state_len > ring_hi)
                    return set_error(EMT_MALFORMED_DOCUMENT, "line end " + std::to_string(p.id) + ": peer ring slot");
            }
        }
        P.ring_lo = ring_lo;
        P.ring_cols = ring_hi - ring_lo;
        std::vector<double> mirror(static_cast<size_t>(width) * P.ring_cols);
        for (int l = 0; l < width; ++l)
            for (int c = 0; c < P.ring_cols; ++c)
                mirror[static_cast<size_t>(l) * P.ring_cols + c] =
                    initial[static_cast<size_t>(ring_lo + c) * width + static_cast<size_t>(l)];
        CUDA_TRY(cudaMalloc(&e->d_ring, mirror.size() * sizeof(double)));
        CUDA_TRY(cudaMemcpy(e->d_ring, mirror.data(), mirror.size() * sizeof(double), cudaMemcpyHostToDevice));
        P.ring = e->d_ring;
    }
    e->initial_fcount.resize(static_cast<size_t>(W));
    for (int l = 0; l < W; ++l) e->initial_fcount[static_cast<size_t>(l)] = arena[static_cast<size_t>(s.fcount) * W + l];
    e->base_factor_count = static_cast<int>(initial[static_cast<size_t>(s.fcount) * width]);
    const double* dc = nullptr;
    const double* da = nullptr;
    EMT_TRY(e->upload(ctab, dc));
    EMT_TRY(e->upload(arena, da));
    P.ctab = dc;
    P.arena = const_cast<double*>(da);

    std::vector<LaneError> errs(static_cast<size_t>(W), LaneError{0, 0, 0, 0});
    const LaneError* de = nullptr;
    EMT_TRY(e->upload(errs, de));
    P.lane_err = const_cast<LaneError*>(de);
    std::vector<int> ev(static_cast<size_t>(3 * e->max_events + 3), 0), nev(1, 0);
    const int* dev_ev = nullptr;
    const int* dev_nev = nullptr;
    EMT_TRY(e->upload(ev, dev_ev));
    EMT_TRY(e->upload(nev, dev_nev));
    P.events = const_cast<int*>(dev_ev);
    P.n_events = const_cast<int*>(dev_nev);
    P.max_events = e->max_events;

    // work-area geometry: arena then constants per lane
    P.ext_pad = (s.extent + 1) & ~1;
    P.lane_stride = P.ext_pad + ((s.consts + 1) & ~1);
    const size_t lane_bytes = static_cast<size_t>(P.lane_stride) * sizeof(double);
    int dev_smem = 0, sms = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, e->device));
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, e->device));
    const int max_lpb_smem = static_cast<int>(static_cast<size_t>(dev_smem) / lane_bytes);
    P.use_smem = max_lpb_smem >= 1 ? 1 : 0;
    int lpb = (W + sms - 1) / sms;  // one CTA per SM when the batch is large enough
    lpb = std::max(1, std::min(lpb, 32));
    if (P.use_smem) lpb = std::min(lpb, max_lpb_smem);
    P.lpb = lpb;
    P.work = nullptr;
    if (!P.use_smem) {
        double* w = nullptr;
        CUDA_TRY(cudaMalloc(&w, lane_bytes * static_cast<size_t>(W)));
        e->allocations.push_back(w);
        P.work = w;
    }
    e->block = 32 * lpb;
    e->grid = (W + lpb - 1) / lpb;
    e->smem_bytes = P.use_smem ? lane_bytes * static_cast<size_t>(lpb) : 0;
    CUDA_TRY(cudaFuncSetAttribute(emt_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(std::max<size_t>(e->smem_bytes, 0))));
    return EMT_OK;
}

/// Tables of the one-CTA-per-lane system kernel (system_kernel.cuh): forward column
/// blocks of 32 with their tiles and trailing segments, and the backward stream
/// (rows descending: the row's U entries past the diagonal, the diagonal, its reciprocal).
emt_status build_system_plan(emt_engine* e) {
    const Schedule& s = e->sched;
    const DevPlan& P = e->plan;
    SysPlan& S = e->sys;
    if (s.nodes > 0 && s.dim != s.nodes)
        return set_error(EMT_MALFORMED_DOCUMENT, "system kernel: matrix dimension differs from the node count");
    const int dim = s.dim;
    S.nblk = (dim + 31) / 32;
    std::vector<int> kin(static_cast<size_t>(dim));
    std::vector<unsigned> mask(static_cast<size_t>(dim), 0u), blk(static_cast<size_t>(std::max(1, S.nblk)), 0u);
    std::vector<std::vector<int4>> segs(static_cast<size_t>(std::max(1, S.nblk)));
    for (int r = 0; r < dim; ++r) {
        const int b = r / 32, kb = s.l_row_ptr[static_cast<size_t>(r)], ke = s.l_row_ptr[static_cast<size_t>(r) + 1];
        int k = kb;
        while (k < ke) {  // runs of entries per column block, ascending
            const int cb = s.l_col[static_cast<size_t>(k)] / 32;
            int k1 = k;
            while (k1 < ke && s.l_col[static_cast<size_t>(k1)] / 32 == cb) ++k1;
            if (cb < b) {
                segs[static_cast<size_t>(cb)].push_back(make_int4(r, k, k1, 0));
            } else {  // cb == b: the row's own tile (strictly lower: columns < r)
                kin[static_cast<size_t>(r)] = k;
                for (int q = k; q < k1; ++q) mask[static_cast<size_t>(r)] |= 1u << (s.l_col[static_cast<size_t>(q)] - 32 * b);
            }
            k = k1;
        }
        if (mask[static_cast<size_t>(r)] == 0u) kin[static_cast<size_t>(r)] = ke;
        blk[static_cast<size_t>(b)] |= mask[static_cast<size_t>(r)];
    }
    // shared memory left for a forward round's products once everything else is laid
    // out (below): bigger rounds mean fewer round barriers per forward block
    int dev_smem_q = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&dev_smem_q, cudaDevAttrMaxSharedMemoryPerBlockOptin, e->device));
    int max_u_off = 1;
    for (int r = 0; r < dim; ++r)
        max_u_off = std::max(max_u_off, s.u_row_ptr[static_cast<size_t>(r) + 1] - s.u_row_ptr[static_cast<size_t>(r)] - 1);
    const long long fixed = static_cast<long long>(kSysRing) * kSysChunk * 12 + 8 * kSysRing + 16 + 2 * 4 * 8 +
                            2LL * (max_u_off + 8) * 8 + 32 * 33 * 8 + 8LL * std::max(1, dim) + 1024;
    const int fcap = static_cast<int>(std::max(1024LL, std::min(16384LL, (dev_smem_q - fixed) / 8 / 1024 * 1024)));
    S.fcap = fcap;
    // forward rounds: each block's trailing segments (one row's terms in the block's
    // columns, <= 32) packed into rounds whose products fit the shared buffer in a
    // transposed layout: term j of the round's piece p sits at j * P' + p (P' = pieces
    // rounded up to odd), so a warp reading term j of 32 pieces is bank-conflict free
    std::vector<int> rnd_ptr{0}, fsrc, fcol, fdst;
    std::vector<int4> rnd, piece;
    for (int b = 0; b < std::max(1, S.nblk); ++b) {
        const auto& sv = segs[static_cast<size_t>(b)];
        size_t i0 = 0;
        do {  // one round: pieces [i0, i1)
            size_t i1 = i0;
            int maxlen = 0;
            while (i1 < sv.size()) {
                const int len = sv[i1].z - sv[i1].y;
                const int np = (static_cast<int>(i1 - i0) + 1) | 1;
                if (i1 > i0 && np * std::max(maxlen, len) > fcap) break;
                maxlen = std::max(maxlen, len);
                ++i1;
            }
            const int pp = static_cast<int>(i1 - i0) | 1;
            const int e0 = static_cast<int>(fsrc.size()), p0 = static_cast<int>(piece.size());
            for (size_t i = i0; i < i1; ++i) {
                const int4& sg = sv[i];
                const int pi = static_cast<int>(i - i0);
                piece.push_back(make_int4(sg.x, pi, sg.z - sg.y, pp));
                for (int q = sg.y; q < sg.z; ++q) {
                    fsrc.push_back(q);
                    fcol.push_back(s.l_col[static_cast<size_t>(q)]);
                    fdst.push_back((q - sg.y) * pp + pi);
                }
            }
            rnd.push_back(make_int4(e0, static_cast<int>(fsrc.size()), p0, static_cast<int>(piece.size())));
            i0 = i1;
        } while (i0 < sv.size());  // every block has >= 1 (possibly empty) round: it stages the next tile
        rnd_ptr.push_back(static_cast<int>(rnd.size()));
    }
    if (fsrc.empty()) {  // one placeholder entry (never read as an L value)
        fsrc.push_back(-1);
        fcol.push_back(0);
        fdst.push_back(0);
    }
    std::vector<int> tsrc(static_cast<size_t>(std::max(1, S.nblk)) * 1024, -1);
    for (int r = 0; r < dim; ++r) {
        const int b = r / 32, j = r % 32;
        for (int q = kin[static_cast<size_t>(r)]; q < s.l_row_ptr[static_cast<size_t>(r) + 1]; ++q)
            tsrc[static_cast<size_t>(b) * 1024 + j * 32 + (s.l_col[static_cast<size_t>(q)] - 32 * b)] = q;
    }
    if (s.l_col.empty()) std::fill(tsrc.begin(), tsrc.end(), -1);
    S.fstream_len = static_cast<long long>(fsrc.size());
    int max_urow = 1;
    for (int r = 0; r < dim; ++r) max_urow = std::max(max_urow, s.u_row_ptr[static_cast<size_t>(r) + 1] - s.u_row_ptr[static_cast<size_t>(r)] - 1);
    S.fact_threads = std::min(kSysThreads, 32 * ((max_urow + 31) / 32));
    std::vector<int4> lent(std::max<size_t>(1, s.l_col.size()), make_int4(0, 0, 0, 0));
    for (size_t k = 0; k < s.l_col.size(); ++k) {
        const int c = s.l_col[k];
        lent[k] = make_int4(c, s.u_row_ptr[static_cast<size_t>(c)], s.u_row_ptr[static_cast<size_t>(c) + 1], 0);
    }
    std::vector<int> bcol, bsrc, brow_len;
    S.pmax = 1;
    for (int i = dim - 1; i >= 0; --i) {
        const int ub = s.u_row_ptr[static_cast<size_t>(i)], ue = s.u_row_ptr[static_cast<size_t>(i) + 1];
        brow_len.push_back(2 * (ue - ub - 1) + (ue - ub > 1 && s.u_col[static_cast<size_t>(ub) + 1] == i + 1 ? 1 : 0));
        S.pmax = std::max(S.pmax, ue - ub - 1);
        for (int k = ub + 1; k < ue; ++k) {
            bcol.push_back(s.u_col[static_cast<size_t>(k)]);
            bsrc.push_back(k);
        }
        bcol.push_back(0);  // diagonal
        bsrc.push_back(ub);
        bcol.push_back(0);  // its reciprocal
        bsrc.push_back(-1 - ub);
    }
    const size_t padded = std::max<size_t>(kSysChunk, (bcol.size() + kSysChunk - 1) / kSysChunk * kSysChunk);
    bcol.resize(padded, 0);
    bsrc.resize(padded, INT_MIN);
    S.stream_len = static_cast<long long>(padded);
    S.stream_chunks = static_cast<int>(padded / kSysChunk);
    const int* d = nullptr;
    EMT_TRY(e->upload(kin, S.fwd_kin));
    EMT_TRY(e->upload(mask, S.fwd_mask));
    EMT_TRY(e->upload(blk, S.blk_cols));
    EMT_TRY(e->upload(rnd_ptr, S.rnd_ptr));
    EMT_TRY(e->upload(rnd, S.rnd));
    EMT_TRY(e->upload(piece, S.piece));
    EMT_TRY(e->upload(fsrc, S.fsrc));
    EMT_TRY(e->upload(fcol, S.fcol));
    EMT_TRY(e->upload(fdst, S.fdst));
    EMT_TRY(e->upload(tsrc, S.tsrc));
    EMT_TRY(e->upload(lent, S.lent));
    EMT_TRY(e->upload(bcol, S.bcol));
    EMT_TRY(e->upload(bsrc, S.bsrc));
    EMT_TRY(e->upload(brow_len, d));
    S.brow = d;
    CUDA_TRY(cudaMalloc(&S.bval, padded * sizeof(double) * static_cast<size_t>(e->W)));
    e->allocations.push_back(S.bval);
    CUDA_TRY(cudaMalloc(&S.fval, static_cast<size_t>(S.fstream_len) * sizeof(double) * static_cast<size_t>(e->W)));
    e->allocations.push_back(S.fval);
    CUDA_TRY(cudaMalloc(&S.tval, tsrc.size() * sizeof(double) * static_cast<size_t>(e->W)));
    e->allocations.push_back(S.tval);
    CUDA_TRY(cudaMalloc(&S.frcp, static_cast<size_t>(std::max(1, dim)) * sizeof(double) * static_cast<size_t>(e->W)));
    e->allocations.push_back(S.frcp);
    S.work = nullptr;
    if (e->W > 1) {
        CUDA_TRY(cudaMalloc(&S.work, static_cast<size_t>(P.lane_stride) * sizeof(double) * static_cast<size_t>(e->W)));
        e->allocations.push_back(S.work);
    }
    // dynamic shared memory: TMA ring (values, columns), mbarriers, the forward tile, v
    size_t off = 0;
    S.smem_ring_v = static_cast<int>(off);
    off += static_cast<size_t>(kSysRing) * kSysChunk * sizeof(double);
    S.smem_ring_c = static_cast<int>(off);
    off += static_cast<size_t>(kSysRing) * kSysChunk * sizeof(int);
    S.smem_mbar = static_cast<int>(off);
    off += static_cast<size_t>(kSysRing) * 8;
    S.smem_flags = static_cast<int>(off);
    off += 16;
    S.smem_desc = static_cast<int>(off);
    off += 2 * 4 * sizeof(double);
    S.smem_pbuf = static_cast<int>(off);
    S.pmax += 8;  // room for the zero padding to a multiple of eight terms
    off += 2 * static_cast<size_t>(S.pmax) * sizeof(double);
    S.smem_fp = static_cast<int>(off);
    off += static_cast<size_t>(S.fcap) * sizeof(double);
    S.smem_tile = static_cast<int>(off);
    off += 32 * 33 * sizeof(double);
    S.smem_xs = static_cast<int>(off);
    off += static_cast<size_t>(std::max(1, dim)) * sizeof(double);
    if (S.pmax + 2 > (kSysRing - 1) * kSysChunk)  // a row's stream entries must fit in the ring at once
        return set_error(EMT_CAPACITY_EXCEEDED, "system kernel: a U row of " + std::to_string(S.pmax) + " entries");
    int dev_smem = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, e->device));
    if (off + 1024 > static_cast<size_t>(dev_smem))  // static shared: s_flag, s_bad
        return set_error(EMT_CAPACITY_EXCEEDED, "system kernel: " + std::to_string(dim) +
                                                    " nodes exceed the shared-memory copy of v");
    e->sys_smem = off;
    S.prof = nullptr;
    const char* pf = dev_env("EMTB200_CG_PROF");
    if (pf && std::strcmp(pf, "0") != 0) {
        CUDA_TRY(cudaMalloc(&e->d_prof, 32 * 64 * sizeof(long long)));
        CUDA_TRY(cudaMemset(e->d_prof, 0, 32 * 64 * sizeof(long long)));
        S.prof = e->d_prof;
    }
    CUDA_TRY(cudaFuncSetAttribute(emt_system_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(off)));
    return EMT_OK;
}

/// Full-chip launch of the specialised kernel (generated prologue: `bid_code`,
/// codegen.cpp): one CTA per SM, the CTAs on SMs 0..groups-1 claim the lane groups.
/// A launch of fewer CTAs than SMs runs up to 13% slower on some B200s, the same
/// groups spread over more TPCs slower still (profiles/ab/placement_r2.log). Needs one
/// CTA per SM (the dynamic shared memory is raised above half an SM's when smaller)
/// and at most one lane group per SM; otherwise, and for engines whose progress words
/// are shared with peer engines (emt_engine_attach_lines), the launch stays one CTA
/// per group.
void setup_claim(emt_engine* e) {
    e->claim_grid = 0;
    if (e->kernel_mode != EMT_KERNEL_SPECIALISED || dev_env("EMTB200_NOCLAIM")) return;
    int sms = 0, per_sm = 0, optin = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, e->device) != cudaSuccess ||
        cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, e->device) != cudaSuccess ||
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, e->device) != cudaSuccess)
        return;
    if (cta_count(e) > sms) return;
    const size_t need = std::max<size_t>(e->gen.smem_bytes, static_cast<size_t>(per_sm) / 2 + 1024);
    if (need > static_cast<size_t>(optin)) return;
    if (driver()->FuncSetAttribute(e->jit.function, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
                                   static_cast<int>(need)) != CUDA_SUCCESS)
        return;
    if (e->d_pick == nullptr && cudaMalloc(&e->d_pick, sizeof(int) * (1 + static_cast<size_t>(sms))) != cudaSuccess) return;
    e->claim_grid = sms;
    e->claim_smem = need;
}

/// Adopts the asynchronously compiled specialised kernel once it is ready (or, with
/// `block`, waits for it). Launches stay stream-ordered, so switching between two
/// launches needs no synchronisation; both kernels produce the same bits.
void adopt_pending(emt_engine* e, bool block) {
    if (!e->pending) return;
    PendingJit& p = *e->pending;
    if (!block && p.done.wait_for(std::chrono::seconds(0)) != std::future_status::ready) return;
    p.done.get();
    if (p.ok) {
        e->gen = std::move(p.gen);
        e->jit = p.jit;
        p.jit = JitModule{};
        p.ok = false;
        e->kernel_mode = EMT_KERNEL_SPECIALISED;
        e->switched_at = e->step;
        char b[200];
        std::snprintf(b, sizeof b, " codegen=%.3fs jit=%.3fs%s (async JIT: generic kernel for passes 0..%d)", p.gen_s,
                      e->jit.compile_seconds, e->jit.cached ? " (cached)" : "", e->step - 1);
        e->summary = "specialised kernel: " + e->gen.summary + b;
        setup_claim(e);
        if (e->claim_grid > 0) e->summary += " launch=full-chip(" + std::to_string(e->claim_grid) + ")";
    } else {
        e->summary += " (specialised kernel unavailable: " + (p.fail.message.empty() ? p.log.substr(0, 300) : p.fail.message) + ")";
    }
    e->pending.reset();
}

emt_status check_lane_errors(emt_engine* e) {
    std::vector<LaneError> errs(static_cast<size_t>(e->W));
    CUDA_TRY(cudaMemcpy(errs.data(), e->plan.lane_err, errs.size() * sizeof(LaneError), cudaMemcpyDeviceToHost));
    // The reference throws at the first failing (step, layer); within it, the
    // lowest row/node index, then the lowest lane (sparse.cpp:135-143, exec.cpp:229-237).
    const LaneError* best = nullptr;
    int best_lane = -1;
    // a failing CTA releases its line-coupled peers, which then record code 64: the
    // cause is the other error, so 64 is reported only when it is the only one
    bool cause = false;
    for (const LaneError& x : errs) cause = cause || (x.code != 0 && x.code != 64);
    for (int l = 0; l < e->W; ++l) {
        const LaneError& x = errs[static_cast<size_t>(l)];
        if (x.code == 0 || (cause && x.code == 64)) continue;
        if (best == nullptr || x.step < best->step || (x.step == best->step && x.layer < best->layer) ||
            (x.step == best->step && x.layer == best->layer && x.index < best->index)) {
            best = &x;
            best_lane = l;
        }
    }
    if (best == nullptr) return EMT_OK;
    e->failed = 1;
    const int glane = e->lane_begin + best_lane;
    if (best->code == EMT_INEXACT_DIVISION)
        return set_error(EMT_INEXACT_DIVISION, "backward-substitution quotient below 2^-900 (step " +
                                                   std::to_string(best->step) + ", lane " + std::to_string(glane) +
                                                   "); rerun with EMT_FLAG_EXACT_DIVISION");
    if (best->code == 64 && best->index == -2)  // system kernel (system_kernel.cuh)
        return set_error(EMT_CUDA_ERROR, "system kernel: backward-sweep handoff wait timed out (step " +
                                             std::to_string(best->step) + ", lane " + std::to_string(glane) + ")");
    if (best->code == 64)  // written by the line-coupled persistent kernel (codegen.cpp)
        return set_error(EMT_CUDA_ERROR, "line-coupling progress wait timed out or a peer CTA / rank failed (step " +
                                             std::to_string(best->step) + ", lane " + std::to_string(glane) + ")");
    if (best->code == EMT_SINGULAR_MATRIX)
        return set_error(best->code, "row " + std::to_string(best->index) + ": zero pivot below tolerance" +
                                         (e->sched.width > 1 ? " in lane " + std::to_string(glane) : std::string()) +
                                         " (step " + std::to_string(best->step) + ")");
    return set_error(best->code, "node index " + std::to_string(best->index) + ": node voltage diverged (step " +
                                     std::to_string(best->step) + ", lane " + std::to_string(glane) + ")");
}


/// Grows the waveform store to `capacity_steps` rows, keeping recorded rows.
emt_status emt_engine_reserve_keep(emt_engine* e, int capacity_steps) {
    CUDA_TRY(cudaSetDevice(e->device));
    CUDA_TRY(cudaStreamSynchronize(e->stream));
    if (e->copy_stream) CUDA_TRY(cudaStreamSynchronize(e->copy_stream));
    if (capacity_steps <= e->capacity) return EMT_OK;
    const size_t row = static_cast<size_t>(e->plan.nch) * e->W;
    double* w = nullptr;
    unsigned char* f = nullptr;
    CUDA_TRY(cudaMalloc(&w, std::max<size_t>(8, row * capacity_steps * sizeof(double))));
    CUDA_TRY(cudaMalloc(&f, static_cast<size_t>(capacity_steps)));
    CUDA_TRY(cudaMemset(f, 0, static_cast<size_t>(capacity_steps)));
    if (e->rows > 0) {
        CUDA_TRY(cudaMemcpy(w, e->d_waves, row * e->rows * sizeof(double), cudaMemcpyDeviceToDevice));
        CUDA_TRY(cudaMemcpy(f, e->d_refactored, static_cast<size_t>(e->rows), cudaMemcpyDeviceToDevice));
    }
    if (e->d_waves) cudaFree(e->d_waves);
    if (e->d_refactored) cudaFree(e->d_refactored);
    e->d_waves = w;
    e->d_refactored = f;
    e->capacity = capacity_steps;
    return EMT_OK;
}

}  // namespace

extern "C" {

const char* emt_last_error(void) { return g_last_error.c_str(); }

const char* emt_version(void) {
#ifdef EMTB200_DEV_KNOBS
    return "emtb200 persistent-warp engine; sm_100a; -fmad=false; DEVELOPER BUILD (EMTB200_* environment knobs live)";
#else
    return "emtb200 persistent-warp engine; sm_100a; -fmad=false";
#endif
}

static emt_status engine_create(const char* schedule_text, const double* const_table, int32_t width,
                                const double* initial, int64_t initial_len, const emt_config* cfg, emt_engine** out);

// C ABI entry points doing host-side work (parsing, planning, code generation) turn any
// C++ exception (e.g. std::bad_alloc) into a status instead of unwinding into C callers.
emt_status emt_engine_create(const char* schedule_text, const double* const_table, int32_t width,
                             const double* initial, int64_t initial_len, const emt_config* cfg,
                             emt_engine** out) {
    try {
        return engine_create(schedule_text, const_table, width, initial, initial_len, cfg, out);
    } catch (const std::exception& ex) {
        return set_error(EMT_CUDA_ERROR, std::string("internal error: ") + ex.what());
    } catch (...) {
        return set_error(EMT_CUDA_ERROR, "internal error");
    }
}

static emt_status engine_create(const char* schedule_text, const double* const_table, int32_t width,
                                const double* initial, int64_t initial_len, const emt_config* cfg,
                                emt_engine** out) {
    if (out == nullptr || schedule_text == nullptr) return set_error(EMT_INVALID_HANDLE, "null argument");
    *out = nullptr;
    auto e = std::make_unique<emt_engine>();
    Failure f;
    if (!parse_schedule(schedule_text, e->sched, f))
        return set_error(f.code, (f.where.empty() ? "" : f.where + ": ") + f.message);
    if (width <= 0) width = e->sched.width;
    if (const_table == nullptr && width != e->sched.width)
        return set_error(EMT_DIMENSION_MISMATCH, "width differs from the schedule and no const table was given");
    lu_symbolic(e->sched);
    EMT_TRY(validate(e->sched, initial_len, width));
    emt_config c{};
    if (cfg != nullptr) c = *cfg;
    e->device = c.device;
    e->lane_begin = c.lane_begin;
    e->width = width;
    e->W = c.lane_count > 0 ? c.lane_count : width - c.lane_begin;
    if (e->lane_begin < 0 || e->W < 1 || e->lane_begin + e->W > width)
        return set_error(EMT_NON_POSITIVE_INPUT, "lane range outside the batch");
    CUDA_TRY(cudaSetDevice(e->device));
    CUDA_TRY(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
    EMT_TRY(build_plan(e.get(), const_table, width, initial));
    if (c.lanes_per_block > 0) {
        e->plan.lpb = std::min(c.lanes_per_block, 32);
        const size_t lane_bytes = static_cast<size_t>(e->plan.lane_stride) * sizeof(double);
        e->block = 32 * e->plan.lpb;
        e->grid = (e->W + e->plan.lpb - 1) / e->plan.lpb;
        e->smem_bytes = e->plan.use_smem ? lane_bytes * static_cast<size_t>(e->plan.lpb) : 0;
        CUDA_TRY(cudaFuncSetAttribute(emt_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(e->smem_bytes)));
    }
    e->kernel_mode = EMT_KERNEL_GENERIC;
    e->summary = "generic table-driven kernel, grid=" + std::to_string(e->grid) + " block=" + std::to_string(e->block);
    if (c.kernel == EMT_KERNEL_SYSTEM) {
        EMT_TRY(build_system_plan(e.get()));
        e->kernel_mode = EMT_KERNEL_SYSTEM;
        e->summary = "system kernel: one " + std::to_string(kSysThreads) + "-thread CTA per lane, grid=" +
                     std::to_string(e->W) + " fwd_blocks=" + std::to_string(e->sys.nblk) +
                     " stream_chunks=" + std::to_string(e->sys.stream_chunks) + " fcap=" + std::to_string(e->sys.fcap) + " smem=" + std::to_string(e->sys_smem);
        *out = e.release();
        return EMT_OK;
    }
    const char* kenv = dev_env("EMTB200_KERNEL");
    if (c.kernel == EMT_KERNEL_AUTO && kenv && std::strcmp(kenv, "tsimt") == 0) c.kernel = EMT_KERNEL_TSIMT;
    if (c.kernel == EMT_KERNEL_TSIMT) {
        CodegenOptions opt;
        opt.warps = c.warps_per_group > 0 ? c.warps_per_group : 4;
        opt.lane_begin = e->lane_begin;
        Failure gf;
        std::string log;
        const auto t0 = std::chrono::steady_clock::now();
        bool ok = generate_tsimt(e->sched, e->host_ctab, e->W, opt, e->gen, gf);
        const double gen_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (ok) ok = jit_load(e->gen.source, e->gen.name, e->device, e->jit, log);
        if (ok && driver()->FuncSetAttribute(e->jit.function, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
                                             static_cast<int>(e->gen.smem_bytes)) != CUDA_SUCCESS) {
            ok = false;
            log = "cuFuncSetAttribute(max dynamic smem) failed";
        }
        if (ok) {  // record tables are read through L1: leave it most of the SRAM
            const int carve = dev_env("EMTB200_TS_CARVEOUT") ? std::atoi(dev_env("EMTB200_TS_CARVEOUT")) : 25;
            driver()->FuncSetAttribute(e->jit.function, CU_FUNC_ATTRIBUTE_PREFERRED_SHARED_MEMORY_CARVEOUT, carve);
        }
        if (!ok)
            return set_error(gf.code ? gf.code : EMT_CUDA_ERROR,
                             "task-SIMT kernel unavailable: " + (gf.message.empty() ? log.substr(0, 2000) : gf.message));
        e->kernel_mode = EMT_KERNEL_TSIMT;
        char b[160];
        std::snprintf(b, sizeof b, " codegen=%.3fs jit=%.3fs%s", gen_s, e->jit.compile_seconds, e->jit.cached ? " (cached)" : "");
        e->summary = "task-SIMT kernel: " + e->gen.summary + b;
        *out = e.release();
        return EMT_OK;
    }
    if (c.kernel == EMT_KERNEL_AUTO && (c.flags & EMT_FLAG_ASYNC_JIT) && e->plan.use_smem && e->plan.ring == nullptr &&
        !(c.flags & EMT_FLAG_TENSOR_SOLVE)) {
        // run the generic kernel now; generate + NVRTC-compile the specialised one on a
        // host thread and switch to it at the first launch after it is ready
        CodegenOptions opt;
        opt.warps = c.warps_per_group > 0 ? c.warps_per_group : 8;
        opt.auto_warps = c.warps_per_group <= 0;
        opt.exact_division = (c.flags & EMT_FLAG_EXACT_DIVISION) != 0;
        int dev_smem = 0;
        CUDA_TRY(cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, e->device));
        opt.smem_budget = static_cast<size_t>(dev_smem);
        opt.lane_begin = e->lane_begin;
        e->pending = std::make_unique<PendingJit>();
        PendingJit* p = e->pending.get();
        const Schedule* sc = &e->sched;
        const std::vector<double>* ct = &e->host_ctab;
        const int W = e->W, dev = e->device;
        p->done = std::async(std::launch::async, [p, sc, ct, W, dev, opt]() {
            try {  // nothing may escape the thread: get() would rethrow it across the C ABI
                cudaSetDevice(dev);
                const auto t0 = std::chrono::steady_clock::now();
                p->ok = generate_kernel(*sc, *ct, W, opt, p->gen, p->fail);
                p->gen_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                if (p->ok) p->ok = jit_load(p->gen.source, p->gen.name, dev, p->jit, p->log);
                if (p->ok && driver()->FuncSetAttribute(p->jit.function, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
                                                        static_cast<int>(p->gen.smem_bytes)) != CUDA_SUCCESS) {
                    p->ok = false;
                    p->log = "cuFuncSetAttribute(max dynamic smem) failed";
                }
            } catch (const std::exception& ex) {
                p->ok = false;
                p->log = std::string("async JIT failed: ") + ex.what();
            } catch (...) {
                p->ok = false;
                p->log = "async JIT failed";
            }
        });
        e->summary += " (async JIT of the specialised kernel in flight)";
        *out = e.release();
        return EMT_OK;
    }
    if (c.kernel != EMT_KERNEL_GENERIC) {
        CodegenOptions opt;
        opt.warps = c.warps_per_group > 0 ? c.warps_per_group : 8;
        opt.auto_warps = c.warps_per_group <= 0;
        opt.tensor_solve = (c.flags & EMT_FLAG_TENSOR_SOLVE) != 0;
        opt.exact_division = (c.flags & EMT_FLAG_EXACT_DIVISION) != 0;
        int dev_smem = 0;
        CUDA_TRY(cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, e->device));
        opt.smem_budget = static_cast<size_t>(dev_smem);
        Failure gf;
        std::string log;
        const auto t0 = std::chrono::steady_clock::now();
        opt.lane_begin = e->lane_begin;
        bool ok = generate_kernel(e->sched, e->host_ctab, e->W, opt, e->gen, gf);
        const double gen_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (ok) ok = jit_load(e->gen.source, e->gen.name, e->device, e->jit, log);
        if (ok) {
            if (driver()->FuncSetAttribute(e->jit.function, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
                                           static_cast<int>(e->gen.smem_bytes)) != CUDA_SUCCESS) {
                ok = false;
                log = "cuFuncSetAttribute(max dynamic smem) failed";
            }
        }
        if (ok) {
            e->kernel_mode = EMT_KERNEL_SPECIALISED;
            const char* pf = dev_env("EMTB200_CG_PROF");
            if (pf && std::strcmp(pf, "0") != 0) {
                CUDA_TRY(cudaMalloc(&e->d_prof, 32 * 64 * sizeof(long long)));
                CUDA_TRY(cudaMemset(e->d_prof, 0, 32 * 64 * sizeof(long long)));
            }
            // Line-coupled lanes in one engine: one persistent launch with per-CTA
            // progress words instead of relaunching every K-1 passes (all CTAs must
            // be co-resident: one 32-lane CTA per SM at most).
            int sms = 0;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, e->device);
            const char* pe = dev_env("EMTB200_LINE_PERSISTENT");
            if (e->plan.ring != nullptr && e->max_chunk != INT_MAX && cta_count(e.get()) <= sms &&
                !(pe && std::strcmp(pe, "0") == 0)) {
                CUDA_TRY(cudaMalloc(&e->d_progress, sizeof(unsigned int) * static_cast<size_t>(cta_count(e.get()))));
                CUDA_TRY(cudaMemset(e->d_progress, 0, sizeof(unsigned int) * static_cast<size_t>(cta_count(e.get()))));
                e->min_k = e->max_chunk + 1;
                e->max_chunk = INT_MAX;
                e->persistent_lines = true;
            }
            char b[160];
            std::snprintf(b, sizeof b, " codegen=%.3fs jit=%.3fs%s", gen_s, e->jit.compile_seconds,
                          e->jit.cached ? " (cached)" : "");
            e->summary = "specialised kernel: " + e->gen.summary + b;
            setup_claim(e.get());
            if (e->claim_grid > 0) e->summary += " launch=full-chip(" + std::to_string(e->claim_grid) + ")";
        } else if (c.kernel == EMT_KERNEL_SPECIALISED) {
            return set_error(gf.code ? gf.code : EMT_CUDA_ERROR,
                             "specialised kernel unavailable: " + (gf.message.empty() ? log : gf.message));
        } else if (!e->plan.use_smem && build_system_plan(e.get()) == EMT_OK) {
            // the lane does not fit in shared memory: a whole CTA per lane instead of one warp
            e->kernel_mode = EMT_KERNEL_SYSTEM;
            e->summary = "system kernel: one " + std::to_string(kSysThreads) + "-thread CTA per lane, grid=" +
                         std::to_string(e->W) + " fwd_blocks=" + std::to_string(e->sys.nblk) +
                         " stream_chunks=" + std::to_string(e->sys.stream_chunks) + " fcap=" + std::to_string(e->sys.fcap) + " smem=" + std::to_string(e->sys_smem) +
                         " (specialised kernel unavailable: " + (gf.message.empty() ? log.substr(0, 300) : gf.message) + ")";
        } else {
            e->summary += " (specialised kernel unavailable: " + (gf.message.empty() ? log.substr(0, 300) : gf.message) + ")";
        }
    }
    *out = e.release();
    return EMT_OK;
}

void emt_engine_destroy(emt_engine* engine) { delete engine; }

emt_status emt_engine_shape(const emt_engine* e, int32_t* lanes, int32_t* channels, int32_t* extent,
                            int32_t* consts, int32_t* steps, int32_t* nodes, int32_t* l_nnz, int32_t* u_nnz,
                            int32_t* layers) {
    if (e == nullptr) return set_error(EMT_INVALID_HANDLE, "null engine");
    if (lanes) *lanes = e->W;
    if (channels) *channels = static_cast<int32_t>(e->sched.channel_slot.size());
    if (extent) *extent = e->sched.extent;
    if (consts) *consts = e->sched.consts;
    if (steps) *steps = e->sched.steps;
    if (nodes) *nodes = e->sched.nodes;
    if (l_nnz) *l_nnz = static_cast<int32_t>(e->sched.l_col.size());
    if (u_nnz) *u_nnz = static_cast<int32_t>(e->sched.u_col.size());
    if (layers) *layers = e->sched.layers;
    return EMT_OK;
}

emt_status emt_engine_reserve(emt_engine* e, int32_t capacity_steps) {
    if (e == nullptr) return set_error(EMT_INVALID_HANDLE, "null engine");
    if (capacity_steps < 0) return set_error(EMT_NON_POSITIVE_INPUT, "negative capacity");
    CUDA_TRY(cudaSetDevice(e->device));
    CUDA_TRY(cudaStreamSynchronize(e->stream));
    if (e->rows > 0 && e->d_refactored) {
        // the recording window restarts: carry its refactorisations into the base
        // counts, so factor_count and the fcount slot keep counting from pass 0
        std::vector<unsigned char> flags(static_cast<size_t>(e->rows));
        CUDA_TRY(cudaMemcpy(flags.data(), e->d_refactored, flags.size(), cudaMemcpyDeviceToHost));
        int fc = 0;
        for (unsigned char f : flags) fc += f ? 1 : 0;
        e->base_factor_count += fc;
        for (double& x : e->initial_fcount) x += fc;
    }
    if (capacity_steps > e->capacity) {
        if (e->d_waves) cudaFree(e->d_waves);
        if (e->d_refactored) cudaFree(e->d_refactored);
        e->d_waves = nullptr;
        e->d_refactored = nullptr;
        const size_t row = static_cast<size_t>(e->plan.nch) * e->W;
        CUDA_TRY(cudaMalloc(&e->d_waves, std::max<size_t>(8, row * capacity_steps * sizeof(double))));
        CUDA_TRY(cudaMalloc(&e->d_refactored, std::max<size_t>(1, static_cast<size_t>(capacity_steps))));
        e->capacity = capacity_steps;
    }
    if (e->d_refactored) CUDA_TRY(cudaMemset(e->d_refactored, 0, static_cast<size_t>(std::max(1, e->capacity))));
    e->rows = 0;
    return EMT_OK;
}

emt_status emt_engine_advance(emt_engine* e, int32_t steps, int32_t sync) {
    if (e == nullptr) return set_error(EMT_INVALID_HANDLE, "null engine");
    if (steps < 0) return set_error(EMT_NON_POSITIVE_INPUT, "negative step count");
    if (e->failed) return set_error(EMT_INVALID_HANDLE, "engine stopped after an error: " + g_last_error);
    if (steps == 0) return EMT_OK;
    if (e->rows + steps > e->capacity)
        return set_error(EMT_CAPACITY_EXCEEDED, "waveform store holds " + std::to_string(e->capacity) + " rows");
    CUDA_TRY(cudaSetDevice(e->device));
    adopt_pending(e, false);
    if (steps > e->max_chunk) {
        for (int done = 0; done < steps;) {
            const int n = std::min(e->max_chunk, steps - done);
            EMT_TRY(emt_engine_advance(e, n, 0));
            done += n;
        }
        if (sync) return emt_engine_sync(e);
        return EMT_OK;
    }
    if (e->kernel_mode == EMT_KERNEL_SPECIALISED || e->kernel_mode == EMT_KERNEL_TSIMT) {
        CgArgs a{e->plan.arena, e->plan.ctab, e->d_waves, e->d_refactored, reinterpret_cast<int*>(e->plan.lane_err),
                 e->plan.events, e->plan.n_events, e->plan.max_events, e->step, steps, e->rows, e->plan.div_limit,
                 e->plan.ring, e->plan.ring_lo, e->plan.ring_cols,
                 e->persistent_lines ? e->d_progress : nullptr, e->min_k,
                 e->prog_total > 0 ? e->prog_total : static_cast<int>(cta_count(e)), e->d_prof, e->d_srctab,
                 e->prog_off, e->sys_scope, nullptr};
        if (e->gen.nsrc > 0 && e->jit.function2 != nullptr) {  // the launch's source value table first
            const size_t need = static_cast<size_t>(steps) * e->gen.nsrc;
            if (need > e->srctab_cap) {
                if (e->d_srctab) cudaFree(e->d_srctab);
                e->d_srctab = nullptr;
                CUDA_TRY(cudaMalloc(&e->d_srctab, need * sizeof(double)));
                e->srctab_cap = need;
            }
            a.srctab = e->d_srctab;
            double* tab = e->d_srctab;
            int s0 = e->step, ns = steps;
            const double* ct = e->plan.ctab;
            void* tp[] = {&tab, &s0, &ns, &ct};
            const CUresult r2 = driver()->LaunchKernel(e->jit.function2, static_cast<unsigned>((need + 255) / 256), 1, 1, 256, 1, 1, 0,
                                                       reinterpret_cast<CUstream>(e->stream), tp, nullptr);
            if (r2 != CUDA_SUCCESS) return set_error(EMT_CUDA_ERROR, "cuLaunchKernel(emt_src_kernel) failed");
            e->launches += 1;  // kernel_launches counts every kernel of ours
        }
        void* params[] = {&a};
        const bool ts = e->kernel_mode == EMT_KERNEL_TSIMT;
        unsigned grid = static_cast<unsigned>(ts ? e->W : cta_count(e));
        unsigned smem = static_cast<unsigned>(e->gen.smem_bytes);
        if (!ts && e->claim_grid > 0 && e->progress_owned) {  // full-chip launch: CTAs on SMs 0..groups-1 claim the lane groups
            CUDA_TRY(cudaMemsetAsync(e->d_pick, 0, sizeof(int) * (1 + static_cast<size_t>(cta_count(e))), e->stream));
            a.pick = e->d_pick;
            grid = static_cast<unsigned>(e->claim_grid);
            smem = static_cast<unsigned>(e->claim_smem);
        }
        const CUresult r = driver()->LaunchKernel(e->jit.function, grid, 1, 1, static_cast<unsigned>(32 * e->gen.warps), 1, 1,
                                          smem, reinterpret_cast<CUstream>(e->stream), params, nullptr);
        if (r != CUDA_SUCCESS) {
            const char* msg = nullptr;
            driver()->GetErrorString(r, &msg);
            return set_error(EMT_CUDA_ERROR, std::string("cuLaunchKernel: ") + (msg ? msg : "?"));
        }
    } else if (e->kernel_mode == EMT_KERNEL_SYSTEM) {
        DevPlan P = e->plan;
        P.waves = e->d_waves;
        P.refactored = e->d_refactored;
        emt_system_kernel<<<e->W, kSysThreads, e->sys_smem, e->stream>>>(P, e->sys, e->step, steps, e->rows);
        CUDA_TRY(cudaGetLastError());
    } else {
        DevPlan P = e->plan;
        P.waves = e->d_waves;
        P.refactored = e->d_refactored;
        emt_step_kernel<<<e->grid, e->block, e->smem_bytes, e->stream>>>(P, e->step, steps, e->rows);
        CUDA_TRY(cudaGetLastError());
    }
    e->launches += 1;
    e->step += steps;
    e->rows += steps;
    if (sync) return emt_engine_sync(e);
    return EMT_OK;
}

emt_status emt_engine_sync(emt_engine* e) {
    if (e == nullptr) return set_error(EMT_INVALID_HANDLE, "null engine");
    CUDA_TRY(cudaSetDevice(e->device));
    CUDA_TRY(cudaStreamSynchronize(e->stream));
    return check_lane_errors(e);
}

emt_status emt_engine_read_waves(emt_engine* e, int32_t row0, int32_t rows, double* waves, double* time) {
    if (e == nullptr) return set_error(EMT_INVALID_HANDLE, "null engine");
    if (row0 < 0 || rows < 0 || row0 + rows > e->rows) return set_error(EMT_NON_POSITIVE_INPUT, "row range");
    EMT_TRY(emt_engine_sync(e));
    const size_t row = static_cast<size_t>(e->plan.nch) * e->W;
    if (waves != nullptr && rows > 0)
        CUDA_TRY(cudaMemcpy(waves, e->d_waves + row * row0, row * rows * sizeof(double), cudaMemcpyDeviceToHost));
    if (time != nullptr) {
        const int first_step = e->step - e->rows;
        for (int r = 0; r < rows; ++r) time[r] = static_cast<double>(first_step + row0 + r + 1) * e->sched.dt;
    }
    return EMT_OK;
}

emt_status emt_engine_read_state(emt_engine* e, double* arena) {
    if (e == nullptr) return set_error(EMT_INVALID_HANDLE, "null engine");
    CUDA_TRY(cudaSetDevice(e->device));
    CUDA_TRY(cudaStreamSynchronize(e->stream));
    CUDA_TRY(cudaMemcpy(arena, e->plan.arena, static_cast<size_t>(e->sched.extent) * e->W * sizeof(double),
                        cudaMemcpyDeviceToHost));
    // The reference bumps every lane's fcount on each batch refactorization
    // (exec.cpp:201-202); lanes refactorize individually here, so rebuild it.
    emt_exec_stats st{};
    EMT_TRY(emt_engine_stats(e, &st));
    const int passes = st.factor_count - e->base_factor_count;
    for (int l = 0; l < e->W; ++l)
        arena[static_cast<size_t>(e->sched.fcount) * e->W + l] = e->initial_fcount[static_cast<size_t>(l)] + passes;
    return EMT_OK;
}

emt_status emt_engine_read_events(emt_engine* e, emt_switch_event* events, int32_t max, int32_t* count) {
    if (e == nullptr) return set_error(EMT_INVALID_HANDLE, "null engine");
    CUDA_TRY(cudaSetDevice(e->device));
    CUDA_TRY(cudaStreamSynchronize(e->stream));
    int n = 0;
    CUDA_TRY(cudaMemcpy(&n, e->plan.n_events, sizeof(int), cudaMemcpyDeviceToHost));
    if (count) *count = n;
    const int take = std::min(std::min(n, e->max_events), std::max(0, max));
    if (events != nullptr && take > 0) {
        std::vector<int> raw(static_cast<size_t>(3 * take));
        CUDA_TRY(cudaMemcpy(raw.data(), e->plan.events, raw.size() * sizeof(int), cudaMemcpyDeviceToHost));
        std::vector<emt_switch_event> ev(static_cast<size_t>(take));
        for (int k = 0; k < take; ++k)
            ev[static_cast<size_t>(k)] = {raw[3 * k], raw[3 * k + 1] + e->lane_begin, raw[3 * k + 2]};
        std::sort(ev.begin(), ev.end(), [](const emt_switch_event& a, const emt_switch_event& b) {
            if (a.step != b.step) return a.step < b.step;
            if (a.lane != b.lane) return a.lane < b.lane;
            return a.process < b.process;
        });
        std::memcpy(events, ev.data(), ev.size() * sizeof(emt_switch_event));
    }
    return EMT_OK;
}

emt_status emt_engine_stats(emt_engine* e, emt_exec_stats* stats) {
    if (e == nullptr || stats == nullptr) return set_error(EMT_INVALID_HANDLE, "null argument");
    CUDA_TRY(cudaSetDevice(e->device));
    CUDA_TRY(cudaStreamSynchronize(e->stream));
    std::vector<unsigned char> flags(static_cast<size_t>(std::max(1, e->rows)));
    if (e->rows > 0)
        CUDA_TRY(cudaMemcpy(flags.data(), e->d_refactored, static_cast<size_t>(e->rows), cudaMemcpyDeviceToHost));
    int fc = 0;
    for (int r = 0; r < e->rows; ++r) fc += flags[static_cast<size_t>(r)] ? 1 : 0;
    // fcount slot of the arena carries refactorizations before this recording window
    stats->factor_count = fc + e->base_factor_count;
    int n = 0;
    CUDA_TRY(cudaMemcpy(&n, e->plan.n_events, sizeof(int), cudaMemcpyDeviceToHost));
    stats->switch_events = n;
    stats->kernel_launches = e->launches;
    return EMT_OK;
}

emt_status emt_engine_stage(emt_engine* e, const double* initial, int64_t initial_len, const double* const_table) {
    if (e == nullptr || initial == nullptr) return set_error(EMT_INVALID_HANDLE, "null argument");
    const Schedule& s = e->sched;
    if (initial_len != static_cast<int64_t>(s.extent) * e->width)
        return set_error(EMT_DIMENSION_MISMATCH, "initial state size " + std::to_string(initial_len) +
                                                     " does not match extent " + std::to_string(s.extent) +
                                                     " x width " + std::to_string(e->width));
    if (e->staged) return set_error(EMT_NON_POSITIVE_INPUT, "a staged batch is waiting for emt_engine_commit");
    const size_t W = static_cast<size_t>(e->W), width = static_cast<size_t>(e->width), lb = static_cast<size_t>(e->lane_begin);
    // (also while an async JIT is in flight: its kernel compiles the same constants in)
    if (const_table != nullptr &&
        (e->kernel_mode == EMT_KERNEL_SPECIALISED || e->kernel_mode == EMT_KERNEL_TSIMT || e->pending != nullptr)) {
        // constants compiled in as immediates must keep their values (an isomorphic batch)
        for (size_t q = 0; q < e->inv_slots.size(); ++q) {
            const double* row = const_table + static_cast<size_t>(e->inv_slots[q]) * width + lb;
            for (size_t l = 0; l < W; ++l)
                if (std::memcmp(&row[l], &e->inv_vals[q], sizeof(double)) != 0)
                    return set_error(EMT_TOPOLOGY_MISMATCH, "constant slot " + std::to_string(e->inv_slots[q]) +
                                                                " is compiled into the specialised kernel; "
                                                                "create a new engine for this batch");
        }
    }
    if (const_table != nullptr && e->plan.ring != nullptr) {  // line ends: same ring geometry and K bounds
        for (const Proc& p : s.procs) {
            if (p.code != kNortonBergeron) continue;
            for (size_t l = 0; l < W; ++l) {
                auto c = [&](int j) { return const_table[static_cast<size_t>(p.par + j) * width + lb + l]; };
                const int K = static_cast<int>(c(3)), pr = static_cast<int>(c(5));
                const long long pl = static_cast<long long>(c(4));
                if (K < 2 || static_cast<int>(c(6)) != p.state_len || K - 1 < (e->persistent_lines ? e->min_k : e->max_chunk + 1) - 1 ||
                    pl < 0 || pl >= e->width || pr < e->plan.ring_lo || pr + p.state_len > e->plan.ring_lo + e->plan.ring_cols)
                    return set_error(EMT_TOPOLOGY_MISMATCH, "line end " + std::to_string(p.id) + ": the new batch changes the line geometry");
            }
        }
    }
    CUDA_TRY(cudaSetDevice(e->device));
    if (e->h2d_stream == nullptr) {
        CUDA_TRY(cudaStreamCreateWithFlags(&e->h2d_stream, cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreateWithFlags(&e->stage_done, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&e->commit_done, cudaEventDisableTiming));
        CUDA_TRY(cudaEventRecord(e->commit_done, e->stream));
        CUDA_TRY(cudaMalloc(&e->d_stage_arena, static_cast<size_t>(s.extent) * W * sizeof(double)));
        CUDA_TRY(cudaMalloc(&e->d_stage_ctab, std::max<size_t>(1, static_cast<size_t>(s.consts)) * W * sizeof(double)));
        if (e->plan.ring != nullptr)
            CUDA_TRY(cudaMalloc(&e->d_stage_ring, width * static_cast<size_t>(e->plan.ring_cols) * sizeof(double)));
    }
    // staging buffers are free once the previous commit's device copies ran
    CUDA_TRY(cudaStreamWaitEvent(e->h2d_stream, e->commit_done, 0));
    if (const_table != nullptr)
        CUDA_TRY(cudaMemcpy2DAsync(e->d_stage_ctab, W * sizeof(double), const_table + lb, width * sizeof(double),
                                   W * sizeof(double), static_cast<size_t>(s.consts), cudaMemcpyHostToDevice, e->h2d_stream));
    // arena lane slice: one strided (2D) copy, contiguous when the engine owns every lane
    CUDA_TRY(cudaMemcpy2DAsync(e->d_stage_arena, W * sizeof(double), initial + lb, width * sizeof(double), W * sizeof(double),
                               static_cast<size_t>(s.extent), cudaMemcpyHostToDevice, e->h2d_stream));
    if (e->plan.ring != nullptr) {  // mirror = the new batch's ring slots, every lane, lane-major
        CUDA_TRY(cudaStreamSynchronize(e->h2d_stream));  // the host staging vector is reused
        e->stage_ring_host.assign(width * static_cast<size_t>(e->plan.ring_cols), 0.0);
        for (size_t l = 0; l < width; ++l)
            for (int c = 0; c < e->plan.ring_cols; ++c)
                e->stage_ring_host[l * e->plan.ring_cols + c] = initial[static_cast<size_t>(e->plan.ring_lo + c) * width + l];
        CUDA_TRY(cudaMemcpyAsync(e->d_stage_ring, e->stage_ring_host.data(), e->stage_ring_host.size() * sizeof(double),
                                 cudaMemcpyHostToDevice, e->h2d_stream));
    }
    CUDA_TRY(cudaEventRecord(e->stage_done, e->h2d_stream));
    e->staged_fcount.resize(W);
    for (size_t l = 0; l < W; ++l) e->staged_fcount[l] = initial[static_cast<size_t>(s.fcount) * width + lb + l];
    e->staged_base_fc = static_cast<int>(initial[static_cast<size_t>(s.fcount) * width]);
    e->staged_ctab = const_table != nullptr;
    e->staged = true;
    return EMT_OK;
}

emt_status emt_engine_commit(emt_engine* e) {
    if (e == nullptr) return set_error(EMT_INVALID_HANDLE, "null engine");
    if (!e->staged) return set_error(EMT_NON_POSITIVE_INPUT, "no staged batch");
    const Schedule& s = e->sched;
    const size_t W = static_cast<size_t>(e->W);
    CUDA_TRY(cudaSetDevice(e->device));
    CUDA_TRY(cudaStreamWaitEvent(e->stream, e->stage_done, 0));
    // the staged buffers become the live ones (no device copy): launches enqueued from
    // here on read them, and the next stage writes the old ones only after commit_done,
    // i.e. after every launch that used them
    auto swap_owned = [e](double*& live, double*& staged) {
        for (void*& a : e->allocations)
            if (a == live) a = staged;
        std::swap(live, staged);
    };
    swap_owned(e->plan.arena, e->d_stage_arena);
    if (e->staged_ctab) {
        double* ct = const_cast<double*>(e->plan.ctab);
        swap_owned(ct, e->d_stage_ctab);
        e->plan.ctab = ct;
    }
    (void)s;
    if (e->plan.ring != nullptr) {
        // an attached (shared) mirror holds other engines' rows too: write only this engine's lanes
        const size_t cols = static_cast<size_t>(e->plan.ring_cols);
        const size_t r0 = e->ring_shared ? static_cast<size_t>(e->lane_begin) : 0;
        const size_t nr = e->ring_shared ? W : static_cast<size_t>(e->width);
        CUDA_TRY(cudaMemcpyAsync(e->plan.ring + r0 * cols, e->d_stage_ring + r0 * cols, nr * cols * sizeof(double),
                                 cudaMemcpyDefault, e->stream));
    }
    CUDA_TRY(cudaEventRecord(e->commit_done, e->stream));
    e->initial_fcount = e->staged_fcount;
    e->base_factor_count = e->staged_base_fc;
    CUDA_TRY(cudaMemsetAsync(e->plan.lane_err, 0, W * sizeof(LaneError), e->stream));
    CUDA_TRY(cudaMemsetAsync(e->plan.n_events, 0, sizeof(int), e->stream));
    if (e->d_progress)
        CUDA_TRY(cudaMemsetAsync(e->d_progress + e->prog_off, 0, sizeof(unsigned int) * static_cast<size_t>(cta_count(e)), e->stream));
    if (e->d_refactored) CUDA_TRY(cudaMemsetAsync(e->d_refactored, 0, static_cast<size_t>(std::max(1, e->capacity)), e->stream));
    e->step = 0;
    e->rows = 0;
    e->failed = 0;
    e->staged = false;
    return EMT_OK;
}

emt_status emt_engine_load(emt_engine* e, const double* initial, int64_t initial_len, const double* const_table) {
    if (e == nullptr) return set_error(EMT_INVALID_HANDLE, "null engine");
    CUDA_TRY(cudaSetDevice(e->device));
    CUDA_TRY(cudaStreamSynchronize(e->stream));
    if (e->copy_stream) CUDA_TRY(cudaStreamSynchronize(e->copy_stream));
    EMT_TRY(emt_engine_stage(e, initial, initial_len, const_table));
    EMT_TRY(emt_engine_commit(e));
    // commit's history copy into a shared line mirror and the progress-word reset are
    // queued on the engine stream; other ranks read both as soon as the host returns
    if (e->ring_shared || e->d_progress) CUDA_TRY(cudaStreamSynchronize(e->stream));
    return EMT_OK;
}

emt_status emt_engine_profile(emt_engine* e, int64_t* cycles, int32_t n) {
    if (e == nullptr || cycles == nullptr) return set_error(EMT_INVALID_HANDLE, "null argument");
    if (e->d_prof == nullptr) return set_error(EMT_NON_POSITIVE_INPUT, "engine built without EMTB200_CG_PROF=1");
    CUDA_TRY(cudaSetDevice(e->device));
    CUDA_TRY(cudaStreamSynchronize(e->stream));
    CUDA_TRY(cudaMemcpy(cycles, e->d_prof, sizeof(long long) * static_cast<size_t>(std::min(n, 32 * 64)), cudaMemcpyDeviceToHost));
    return EMT_OK;
}

emt_status emt_engine_ring(emt_engine* e, void** device_ptr, int32_t* lanes, int32_t* cols, int32_t* max_chunk) {
    if (e == nullptr) return set_error(EMT_INVALID_HANDLE, "null engine");
    if (device_ptr) *device_ptr = e->plan.ring;
    if (lanes) *lanes = e->plan.ring ? e->width : 0;
    if (cols) *cols = e->plan.ring_cols;
    if (max_chunk) *max_chunk = e->persistent_lines ? e->min_k - 1 : (e->max_chunk == INT_MAX ? 0 : e->max_chunk);
    return EMT_OK;
}

emt_status emt_engine_attach_lines(emt_engine* e, void* mirror, void* progress, int32_t cta_offset, int32_t total_ctas,
                                   int32_t system_scope) {
    if (e == nullptr || mirror == nullptr || progress == nullptr) return set_error(EMT_INVALID_HANDLE, "null argument");
    if (e->plan.ring == nullptr) return set_error(EMT_NON_POSITIVE_INPUT, "schedule has no line ends");
    if (e->kernel_mode != EMT_KERNEL_SPECIALISED)
        return set_error(EMT_NON_POSITIVE_INPUT, "device-side line exchange needs the specialised kernel");
    const int nctas = cta_count(e);
    if (cta_offset < 0 || total_ctas < cta_offset + nctas) return set_error(EMT_NON_POSITIVE_INPUT, "progress range");
    CUDA_TRY(cudaSetDevice(e->device));
    CUDA_TRY(cudaStreamSynchronize(e->stream));
    // this engine's rows of the current mirror (the initial histories) into the shared one
    const size_t cols = static_cast<size_t>(e->plan.ring_cols);
    CUDA_TRY(cudaMemcpy(static_cast<double*>(mirror) + static_cast<size_t>(e->lane_begin) * cols,
                        e->plan.ring + static_cast<size_t>(e->lane_begin) * cols, static_cast<size_t>(e->W) * cols * sizeof(double),
                        cudaMemcpyDefault));
    CUDA_TRY(cudaMemset(static_cast<unsigned int*>(progress) + cta_offset, 0, sizeof(unsigned int) * static_cast<size_t>(nctas)));
    if (e->ring_owned && e->d_ring) cudaFree(e->d_ring);
    e->d_ring = static_cast<double*>(mirror);
    e->ring_owned = false;
    e->ring_shared = true;
    e->plan.ring = e->d_ring;
    if (e->d_progress && e->progress_owned) cudaFree(e->d_progress);
    e->d_progress = static_cast<unsigned int*>(progress);
    e->progress_owned = false;
    if (!e->persistent_lines) {
        e->min_k = e->max_chunk + 1;
        e->max_chunk = INT_MAX;
        e->persistent_lines = true;
    }
    e->prog_off = cta_offset;
    e->prog_total = total_ctas;
    e->sys_scope = system_scope ? 1 : 0;
    // the D2D history copy and the memset may still be in flight on the legacy stream
    CUDA_TRY(cudaDeviceSynchronize());
    return EMT_OK;
}

emt_status emt_engine_ctas(const emt_engine* e, int32_t* ctas, int32_t* lanes_per_cta) {
    if (e == nullptr) return set_error(EMT_INVALID_HANDLE, "null engine");
    if (ctas) *ctas = cta_count(e);
    if (lanes_per_cta) *lanes_per_cta = e->kernel_mode == EMT_KERNEL_SPECIALISED ? e->gen.lpc : 0;
    return EMT_OK;
}

emt_status emt_ipc_alloc(int32_t device, int64_t bytes, void** ptr, void* handle) {
    if (ptr == nullptr || handle == nullptr || bytes <= 0) return set_error(EMT_INVALID_HANDLE, "null argument");
    CUDA_TRY(cudaSetDevice(device));
    CUDA_TRY(cudaMalloc(ptr, static_cast<size_t>(bytes)));
    CUDA_TRY(cudaMemset(*ptr, 0, static_cast<size_t>(bytes)));
    cudaIpcMemHandle_t h;
    CUDA_TRY(cudaIpcGetMemHandle(&h, *ptr));
    std::memcpy(handle, &h, sizeof h);
    return EMT_OK;
}

emt_status emt_ipc_open(int32_t device, const void* handle, void** ptr) {
    if (ptr == nullptr || handle == nullptr) return set_error(EMT_INVALID_HANDLE, "null argument");
    CUDA_TRY(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    CUDA_TRY(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return EMT_OK;
}

emt_status emt_ipc_close(void* ptr) {
    CUDA_TRY(cudaIpcCloseMemHandle(ptr));
    return EMT_OK;
}

emt_status emt_source_cos(int32_t device, const double* x, double* y, int64_t n) {
    if (n < 0 || (n > 0 && (x == nullptr || y == nullptr))) return set_error(EMT_NON_POSITIVE_INPUT, "bad arguments");
    if (n == 0) return EMT_OK;
    CUDA_TRY(cudaSetDevice(device));
    double* d = nullptr;
    CUDA_TRY(cudaMalloc(&d, 2 * static_cast<size_t>(n) * sizeof(double)));
    cudaError_t rc = cudaMemcpy(d, x, static_cast<size_t>(n) * sizeof(double), cudaMemcpyHostToDevice);
    if (rc == cudaSuccess) {
        const long long blocks = std::min<long long>((n + 255) / 256, 148LL * 8);
        emt_cos_kernel<<<static_cast<unsigned>(blocks), 256>>>(d, d + n, n);
        rc = cudaGetLastError();
    }
    if (rc == cudaSuccess) rc = cudaMemcpy(y, d + n, static_cast<size_t>(n) * sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (rc != cudaSuccess) return set_error(EMT_CUDA_ERROR, std::string("emt_source_cos: ") + cudaGetErrorString(rc));
    return EMT_OK;
}

emt_status emt_ipc_free(void* ptr) {
    CUDA_TRY(cudaFree(ptr));
    return EMT_OK;
}

emt_status emt_engine_attach_ring(emt_engine* e, void* device_ptr) {
    if (e == nullptr || device_ptr == nullptr) return set_error(EMT_INVALID_HANDLE, "null argument");
    if (e->plan.ring == nullptr) return set_error(EMT_NON_POSITIVE_INPUT, "schedule has no line ends");
    CUDA_TRY(cudaSetDevice(e->device));
    CUDA_TRY(cudaStreamSynchronize(e->stream));
    const size_t bytes = static_cast<size_t>(e->width) * e->plan.ring_cols * sizeof(double);
    CUDA_TRY(cudaMemcpy(device_ptr, e->plan.ring, bytes, cudaMemcpyDeviceToDevice));
    if (e->ring_owned && e->d_ring) cudaFree(e->d_ring);
    e->d_ring = static_cast<double*>(device_ptr);
    e->ring_owned = false;
    if (e->persistent_lines) {  // peers on other GPUs: back to launches of K-1 passes + host exchange
        e->persistent_lines = false;
        e->max_chunk = e->min_k - 1;
    }
    e->plan.ring = e->d_ring;
    return EMT_OK;
}

emt_status emt_engine_run_async(emt_engine* e, int32_t steps, int32_t chunk, double* waves) {
    if (e == nullptr) return set_error(EMT_INVALID_HANDLE, "null engine");
    if (steps < 0) return set_error(EMT_NON_POSITIVE_INPUT, "negative step count");
    if (e->rows + steps > e->capacity) EMT_TRY(emt_engine_reserve_keep(e, e->rows + steps));
    if (chunk <= 0) chunk = std::max(1, std::min<int>(steps, 256));
    CUDA_TRY(cudaSetDevice(e->device));
    if (waves != nullptr && e->copy_stream == nullptr)
        CUDA_TRY(cudaStreamCreateWithFlags(&e->copy_stream, cudaStreamNonBlocking));
    const int nchunks = (steps + chunk - 1) / chunk;
    while (waves != nullptr && static_cast<int>(e->chunk_done.size()) < std::min(nchunks, 64)) {
        cudaEvent_t ev;
        CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        e->chunk_done.push_back(ev);
    }
    const size_t row = static_cast<size_t>(e->plan.nch) * e->W;
    for (int c = 0; c < nchunks; ++c) {
        const int n = std::min(chunk, steps - c * chunk);
        const int r0 = e->rows;
        EMT_TRY(emt_engine_advance(e, n, 0));
        if (waves == nullptr) continue;
        // chunk c's rows go to the host while chunk c+1 computes
        cudaEvent_t ev = e->chunk_done[static_cast<size_t>(c) % e->chunk_done.size()];
        CUDA_TRY(cudaEventRecord(ev, e->stream));
        CUDA_TRY(cudaStreamWaitEvent(e->copy_stream, ev, 0));
        CUDA_TRY(cudaMemcpyAsync(waves + row * static_cast<size_t>(c) * chunk, e->d_waves + row * r0,
                                 row * n * sizeof(double), cudaMemcpyDeviceToHost, e->copy_stream));
    }
    return EMT_OK;
}

emt_status emt_engine_wait(emt_engine* e) {
    if (e == nullptr) return set_error(EMT_INVALID_HANDLE, "null engine");
    CUDA_TRY(cudaSetDevice(e->device));
    if (e->copy_stream) CUDA_TRY(cudaStreamSynchronize(e->copy_stream));
    return emt_engine_sync(e);
}

emt_status emt_engine_run(emt_engine* e, int32_t steps, int32_t chunk, double* waves) {
    EMT_TRY(emt_engine_run_async(e, steps, chunk, waves));
    return emt_engine_wait(e);
}

emt_status emt_emit_program(const char* schedule_text, char** source) {
    if (schedule_text == nullptr || source == nullptr) return set_error(EMT_INVALID_HANDLE, "null argument");
    Schedule s;
    Failure f;
    if (!parse_schedule(schedule_text, s, f)) return set_error(f.code ? f.code : EMT_MALFORMED_DOCUMENT, f.where + ": " + f.message);
    lu_symbolic(s);
    std::string out;
    if (!emit_program(s, s.const_table, s.width, out, f)) return set_error(f.code ? f.code : EMT_CAPACITY_EXCEEDED, f.where + ": " + f.message);
    *source = static_cast<char*>(std::malloc(out.size() + 1));
    if (*source == nullptr) return set_error(EMT_CUDA_ERROR, "out of host memory");
    std::memcpy(*source, out.c_str(), out.size() + 1);
    return EMT_OK;
}

emt_status emt_codegen(const char* schedule_text, const double* const_table, int32_t width, int32_t warps,
                       int32_t compile, const char* arch, const char** source, const char** summary) {
    thread_local std::string src_out, sum_out;
    Schedule s;
    Failure f;
    if (schedule_text == nullptr || !parse_schedule(schedule_text, s, f))
        return set_error(f.code ? f.code : EMT_INVALID_HANDLE, f.where + ": " + f.message);
    lu_symbolic(s);
    if (width <= 0) width = s.width;
    if (const_table == nullptr && width != s.width) return set_error(EMT_DIMENSION_MISMATCH, "width without const table");
    std::vector<double> ct(const_table ? const_table : s.const_table.data(),
                           (const_table ? const_table : s.const_table.data()) + static_cast<size_t>(s.consts) * width);
    CodegenOptions opt;
    opt.warps = warps > 0 ? warps : 4;
    GeneratedKernel g;
    const bool ts = warps < 0 && warps > -100;  // negative warp count selects the task-SIMT generator
    if (ts) opt.warps = -warps;
    if (warps <= -100) {  // -100 - w: lane-SIMT kernel with the shared-G tensor-core solve
        opt.warps = -100 - warps > 0 ? -100 - warps : 8;
        opt.tensor_solve = true;
    }
    if (!(ts ? generate_tsimt(s, ct, width, opt, g, f) : generate_kernel(s, ct, width, opt, g, f)))
        return set_error(f.code, f.message);
    src_out = g.source;
    sum_out = g.summary;
    if (compile) {
        std::vector<char> cubin;
        std::string log;
        const auto t0 = std::chrono::steady_clock::now();
        if (!jit_compile(g.source, arch ? arch : "sm_100a", cubin, log))
            return set_error(EMT_CUDA_ERROR, "NVRTC: " + log.substr(0, 4000));
        char b[96];
        std::snprintf(b, sizeof b, " nvrtc=%.3fs cubin=%zuB", std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(),
                      cubin.size());
        sum_out += b;
    }
    if (source) *source = src_out.c_str();
    if (summary) *summary = sum_out.c_str();
    return EMT_OK;
}

emt_status emt_engine_read_refactor_steps(emt_engine* e, int32_t* steps, int32_t max, int32_t* count) {
    if (e == nullptr) return set_error(EMT_INVALID_HANDLE, "null engine");
    CUDA_TRY(cudaSetDevice(e->device));
    CUDA_TRY(cudaStreamSynchronize(e->stream));
    std::vector<unsigned char> flags(static_cast<size_t>(std::max(1, e->rows)));
    if (e->rows > 0)
        CUDA_TRY(cudaMemcpy(flags.data(), e->d_refactored, static_cast<size_t>(e->rows), cudaMemcpyDeviceToHost));
    const int first_step = e->step - e->rows;
    int n = 0;
    for (int r = 0; r < e->rows; ++r) {
        if (!flags[static_cast<size_t>(r)]) continue;
        if (steps != nullptr && n < max) steps[n] = first_step + r;
        ++n;
    }
    if (count) *count = n;
    return EMT_OK;
}

// ---- multi-device engine: the executor call of SURVEY §8(b) (emt_create / emt_run)
// over one lane-shard engine per listed device, run concurrently from one host thread.
struct emt_multi {
    std::vector<emt_engine*> shards;
    std::vector<int> lo, hi;  // lane range of each shard
    int width = 1, channels = 0;
    std::string detail;
    ~emt_multi() {
        for (emt_engine* e : shards) emt_engine_destroy(e);
    }
};

emt_status emt_create(const char* cgmsched_text, const double* initial, int64_t extent, int32_t width,
                      const int32_t* devices, int32_t ndev, emt_multi** out) {
    if (out == nullptr || cgmsched_text == nullptr || initial == nullptr)
        return set_error(EMT_INVALID_HANDLE, "null argument");
    *out = nullptr;
    if (width < 1 || extent < 0) return set_error(EMT_NON_POSITIVE_INPUT, "width must be >= 1");
    const int n = std::max(1, std::min<int>(ndev > 0 ? ndev : 1, width));
    auto m = std::make_unique<emt_multi>();
    m->width = width;
    for (int d = 0; d < n; ++d) {  // contiguous lane shards (sharding.shard_bounds)
        const int lo = static_cast<int>(static_cast<long long>(width) * d / n);
        const int hi = static_cast<int>(static_cast<long long>(width) * (d + 1) / n);
        emt_config c{};
        c.device = devices != nullptr && ndev > 0 ? devices[d] : 0;
        c.lane_begin = lo;
        c.lane_count = hi - lo;
        emt_engine* e = nullptr;
        EMT_TRY(emt_engine_create(cgmsched_text, nullptr, width, initial, extent * width, &c, &e));
        m->shards.push_back(e);
        m->lo.push_back(lo);
        m->hi.push_back(hi);
    }
    m->channels = static_cast<int>(m->shards[0]->sched.channel_slot.size());
    *out = m.release();
    return EMT_OK;
}

emt_status emt_run(emt_multi* m, int32_t steps, int32_t warmup, double* waves, emt_exec_stats* stats) {
    if (m == nullptr) return set_error(EMT_INVALID_HANDLE, "null engine");
    if (steps < 0) return set_error(EMT_NON_POSITIVE_INPUT, "negative step count");
    const int warm = std::max(0, std::min(warmup, steps));
    struct Ev {
        cudaEvent_t a = nullptr, b = nullptr;
        int dev = 0;
        ~Ev() {
            cudaSetDevice(dev);
            if (a) cudaEventDestroy(a);
            if (b) cudaEventDestroy(b);
        }
    };
    std::vector<Ev> ev(m->shards.size());
    auto fail = [m](emt_status st) {
        m->detail = g_last_error;
        return st;
    };
    for (size_t k = 0; k < m->shards.size(); ++k) {  // enqueue every shard, then wait
        emt_engine* e = m->shards[k];
        ev[k].dev = e->device;
        if (emt_status st = emt_engine_reserve(e, steps)) return fail(st);
        CUDA_TRY(cudaSetDevice(e->device));
        CUDA_TRY(cudaEventCreate(&ev[k].a));
        CUDA_TRY(cudaEventCreate(&ev[k].b));
        if (emt_status st = emt_engine_advance(e, warm, 0)) return fail(st);
        CUDA_TRY(cudaEventRecord(ev[k].a, e->stream));
        if (emt_status st = emt_engine_advance(e, steps - warm, 0)) return fail(st);
        CUDA_TRY(cudaEventRecord(ev[k].b, e->stream));
    }
    // the first shard (lowest lanes) that failed reports, as the reference reports its lowest lane
    for (emt_engine* e : m->shards)
        if (emt_status st = emt_engine_sync(e)) return fail(st);
    float worst = 0.f;
    std::set<int> refac;
    emt_exec_stats sum{};
    std::vector<double> rows;
    for (size_t k = 0; k < m->shards.size(); ++k) {
        emt_engine* e = m->shards[k];
        float ms = 0.f;
        CUDA_TRY(cudaSetDevice(e->device));
        cudaEventElapsedTime(&ms, ev[k].a, ev[k].b);
        worst = std::max(worst, ms);
        if (waves != nullptr && steps > 0) {  // shard rows (rows x channels x W) into the batch layout
            const int W = m->hi[k] - m->lo[k];
            rows.resize(static_cast<size_t>(steps) * m->channels * W);
            if (emt_status st = emt_engine_read_waves(e, 0, steps, rows.data(), nullptr)) return fail(st);
            for (int r = 0; r < steps; ++r)
                for (int c = 0; c < m->channels; ++c)
                    std::memcpy(waves + (static_cast<size_t>(r) * m->channels + c) * m->width + m->lo[k],
                                rows.data() + (static_cast<size_t>(r) * m->channels + c) * W, sizeof(double) * W);
        }
        std::vector<int32_t> rs(static_cast<size_t>(std::max(1, steps)));
        int32_t cnt = 0;
        if (emt_status st = emt_engine_read_refactor_steps(e, rs.data(), static_cast<int32_t>(rs.size()), &cnt)) return fail(st);
        for (int q = 0; q < std::min<int>(cnt, static_cast<int>(rs.size())); ++q) refac.insert(rs[static_cast<size_t>(q)]);
        emt_exec_stats st{};
        if (emt_status s2 = emt_engine_stats(e, &st)) return fail(s2);
        sum.kernel_launches += st.kernel_launches;
        sum.switch_events += st.switch_events;
        if (k == 0) sum.factor_count = st.factor_count - static_cast<int>(refac.size());  // the base count
    }
    if (stats) {
        // a refactorisation pass of ANY lane counts once (exec.cpp:200-201): the union over shards
        stats->factor_count = sum.factor_count + static_cast<int>(refac.size());
        stats->measured_steps = steps - warm;
        stats->measured_seconds = static_cast<double>(worst) * 1e-3;  // slowest device
        stats->kernel_launches = sum.kernel_launches;
        stats->switch_events = sum.switch_events;
    }
    return EMT_OK;
}

const char* emt_error_detail(const emt_multi* m) { return m ? m->detail.c_str() : ""; }

void emt_destroy(emt_multi* m) { delete m; }

int32_t emt_engine_kernel(const emt_engine* e) { return e ? e->kernel_mode : 0; }

emt_status emt_engine_wait_jit(emt_engine* e) {
    if (e == nullptr) return set_error(EMT_INVALID_HANDLE, "null engine");
    CUDA_TRY(cudaSetDevice(e->device));
    adopt_pending(e, true);
    return EMT_OK;
}
const char* emt_engine_source(const emt_engine* e) { return e ? e->gen.source.c_str() : ""; }
const char* emt_engine_summary(const emt_engine* e) { return e ? e->summary.c_str() : ""; }

void* emt_engine_device_waves(emt_engine* e) { return e ? e->d_waves : nullptr; }
void* emt_engine_stream(emt_engine* e) { return e ? e->stream : nullptr; }

static emt_status interpret_once(const char* schedule_text, const double* initial, int64_t initial_len, int32_t steps,
                                 const emt_exec_options* options, emt_config c, double* waves, double* time,
                                 emt_exec_stats* stats);

static emt_status interpret_retry(const char* schedule_text, const double* initial, int64_t initial_len,
                                  int32_t steps, const emt_exec_options* options, const emt_config* cfg,
                                  double* waves, double* time, emt_exec_stats* stats);

emt_status emt_interpret(const char* schedule_text, const double* initial, int64_t initial_len, int32_t steps,
                         const emt_exec_options* options, const emt_config* cfg, double* waves, double* time,
                         emt_exec_stats* stats) {
    try {
        return interpret_retry(schedule_text, initial, initial_len, steps, options, cfg, waves, time, stats);
    } catch (const std::exception& ex) {
        return set_error(EMT_CUDA_ERROR, std::string("internal error: ") + ex.what());
    } catch (...) {
        return set_error(EMT_CUDA_ERROR, "internal error");
    }
}

emt_status emt_execute_parallel(const char* schedule_text, const double* initial, int64_t initial_len,
                                int32_t workers, int32_t steps, const emt_exec_options* options,
                                const emt_config* cfg, double* waves, double* time, emt_exec_stats* stats) {
    // execute_parallel (proj/src/exec.cpp:385-389): same contract and results as
    // interpret; the worker count is validated as there, the device does the work
    if (workers < 1) return set_error(EMT_NON_POSITIVE_INPUT, "worker count must be at least 1");
    return emt_interpret(schedule_text, initial, initial_len, steps, options, cfg, waves, time, stats);
}

static emt_status interpret_retry(const char* schedule_text, const double* initial, int64_t initial_len,
                                  int32_t steps, const emt_exec_options* options, const emt_config* cfg,
                                  double* waves, double* time, emt_exec_stats* stats) {
    if (steps < 0) return set_error(EMT_NON_POSITIVE_INPUT, "negative step count");
    emt_config c{};
    if (cfg) c = *cfg;
    c.lane_begin = 0;
    c.lane_count = 0;
    const emt_status st = interpret_once(schedule_text, initial, initial_len, steps, options, c, waves, time, stats);
    if (st != EMT_INEXACT_DIVISION || (c.flags & EMT_FLAG_EXACT_DIVISION)) return st;
    // a quotient left the fast division's exact range: the same run with the IEEE
    // fallback compiled into every backward row (bit-identical to the reference)
    c.flags |= EMT_FLAG_EXACT_DIVISION;
    return interpret_once(schedule_text, initial, initial_len, steps, options, c, waves, time, stats);
}

static emt_status interpret_once(const char* schedule_text, const double* initial, int64_t initial_len, int32_t steps,
                                 const emt_exec_options* options, emt_config c, double* waves, double* time,
                                 emt_exec_stats* stats) {
    emt_engine* raw = nullptr;
    EMT_TRY(emt_engine_create(schedule_text, nullptr, 0, initial, initial_len, &c, &raw));
    std::unique_ptr<emt_engine> e(raw);
    if (options && options->divergence_limit > 0) e->plan.div_limit = options->divergence_limit;
    const int warm = options ? std::max(0, std::min<int>(options->warmup_steps, steps)) : 0;
    EMT_TRY(emt_engine_reserve(e.get(), steps));
    struct Events {  // released on every return path
        cudaEvent_t t0 = nullptr, t1 = nullptr;
        ~Events() {
            if (t0) cudaEventDestroy(t0);
            if (t1) cudaEventDestroy(t1);
        }
    } ev;
    CUDA_TRY(cudaEventCreate(&ev.t0));
    CUDA_TRY(cudaEventCreate(&ev.t1));
    EMT_TRY(emt_engine_advance(e.get(), warm, 0));
    CUDA_TRY(cudaEventRecord(ev.t0, e->stream));
    EMT_TRY(emt_engine_advance(e.get(), steps - warm, 0));
    CUDA_TRY(cudaEventRecord(ev.t1, e->stream));
    emt_status st = emt_engine_sync(e.get());
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev.t0, ev.t1);
    if (st != EMT_OK) return st;
    EMT_TRY(emt_engine_read_waves(e.get(), 0, steps, waves, time));
    if (stats) {
        EMT_TRY(emt_engine_stats(e.get(), stats));
        stats->measured_steps = steps - warm;
        stats->measured_seconds = static_cast<double>(ms) * 1e-3;
    }
    return EMT_OK;
}

}  // extern "C"
