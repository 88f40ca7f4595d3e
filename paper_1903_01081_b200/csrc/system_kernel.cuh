// Large single-system step loop (EMT_KERNEL_SYSTEM): one 1024-thread CTA per lane.
//
// For systems whose arena does not fit in shared memory (gen_scale_case, the
// paper's large-scale case: proj/src/bench.cpp:54-117), one
// warp per lane (the generic kernel) leaves the GPU idle. Here a whole CTA owns
// the lane, the arena stays in HBM/L2, and every phase of a pass is spread over
// the block while every floating-point operation keeps the reference's order:
//
//  * layers (exec.cpp:364-374): the layer's processes in parallel over 1024
//    threads (write sets are disjoint per layer), __syncthreads between layers;
//  * FactorizeSystem (exec.cpp:175-204): the reference's up-looking rows, each
//    elimination's scratch-row update spread over the block (sys_factorize), then
//    the block rebuilds the factor streams below;
//  * SolveSystem (exec.cpp:205-239): the gather in parallel per node into a
//    shared-memory copy of v; the forward sweep in column blocks of 32 — warp 0
//    resolves the block's own lower-triangular tile with register shuffles, then
//    the whole block applies the block's columns to every later row ("trailing
//    segments"); each row still subtracts its terms in ascending column order,
//    exactly as lu_solve does (sparse.cpp:152-160), only the rows progress in
//    parallel; the backward sweep by warp 0 streaming U (rows descending) from
//    HBM through a TMA bulk-copy ring (cp.async.bulk + mbarrier) — each row's
//    products in parallel over the lanes and its subtraction chain in ascending
//    column order (sparse.cpp:161-170); finalize and the divergence check in
//    parallel (lowest failing node wins, exec.cpp:229-237).
//
// What bounds it: the backward sweep. In the reference's order row i subtracts
// its smallest column first, which is the row finished last, so no term of row i
// can start before row i+1 is done: with the fill of a shared root node the
// whole sweep is ONE dependency chain of u_nnz dependent subtractions, and the
// pass costs at least u_nnz x the FP64 add latency.
#pragma once
// (included by engine.cu inside namespace emtb200: uses DevPlan, run_regular, warp_factorize)

constexpr int kSysThreads = 1024;
constexpr int kSysChunkLog = 10;
constexpr int kSysChunk = 1 << kSysChunkLog;  // backward-stream entries per TMA bulk copy
constexpr int kSysRing = 4;      // chunks in flight

struct SysPlan {
    int nblk;                // forward column blocks of 32
    const int* fwd_kin;      // dim: first L index of row r whose column lies in r's own block
    const unsigned* fwd_mask;  // dim: bit c = row r has an L entry in column 32*(r/32)+c
    const unsigned* blk_cols;  // nblk: OR of the block's row masks
    const int* rnd_ptr;      // nblk+1: rounds of each block's trailing update
    const int4* rnd;         // (entry begin, entry end, piece begin, piece end): <= fcap entries per round
    const int4* piece;       // (row, p, count, P'): a row's terms of one round, ascending column, at fp[j * P' + p]
    const int* fsrc;         // forward stream: L index of each entry (block, then row, then column order)
    const int* fcol;         //                 its column
    const int* fdst;         //                 its slot in the round's product buffer
    double* fval;            // W x fstream_len: the lane's L values in stream order (rebuilt with the factors)
    long long fstream_len;
    const int* tsrc;         // nblk x 1024: L index at tile (row j, column c) of block b, or -1
    double* tval;            // W x nblk x 1024: the lane's dense diagonal tiles (0 where absent)
    long long stream_len;    // backward stream entries, padded to kSysChunk
    int stream_chunks;
    const int* bcol;         // stream_len: column of each entry (0 for the diagonal / reciprocal / padding)
    const int* bsrc;         // stream_len: U index of the entry, -1-k for 1/U[k], INT_MIN padding
    const int* brow;         // dim, rows descending: 2 * off-diagonal entries + (first column == row + 1)
    double* bval;            // W x stream_len: the lane's stream values (rebuilt at launch start and after each factorisation)
    double* work;            // lane-major working arena when W > 1 (W == 1 runs on the arena itself)
    double* frcp;            // W x dim: pivot reciprocals 1/U(c,c) of the lane's current factors
    const int4* lent;        // l_nnz: (column c, U row begin, U row end, -) of every L entry (factorisation)
    int fact_threads;        // threads taking part in an elimination step: 32 x ceil(longest U row / 32)
    int smem_xs;             // byte offsets in dynamic shared memory
    int smem_tile;
    int smem_ring_v;
    int smem_ring_c;
    int smem_mbar;
    int smem_flags;          // frontier + two row-ready words (backward producer / consumer)
    int smem_desc;           // [2][4] u_{r,r+1}, diagonal, reciprocal
    int smem_pbuf;           // [2][pmax] products of the rows in flight
    int smem_fp;             // [fcap] products of a forward round
    int fcap;                // forward-round capacity (the shared memory left, 1024..16384 entries)
    int pmax;                // longest U row past the diagonal
    long long* prof;         // developer phase profile (EMTB200_CG_PROF=1): cycles per phase, else null
};

// phase profile: thread 0 adds the cycles since `t` to prof[k] (developer builds only)
__device__ __forceinline__ void sys_mark(const SysPlan& S, long long& t, int k) {
    if (S.prof != nullptr && threadIdx.x == 0) {
        const long long now = clock64();
        S.prof[k] += now - t;
        t = now;
    }
    __syncwarp();
}

// Spin bound of the backward producer / consumer handoff (~1 s): a wait that never
// ends stops the lane with code 64 instead of hanging the GPU.
constexpr unsigned kSysSpinLimit = 1u << 26;


__device__ __forceinline__ unsigned sys_smem_addr(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// One TMA bulk copy of stream chunk `c` (values and columns) into the ring slot of
// its sequence number `q` (slot q % kSysRing; the slot's mbarrier completes one phase per chunk).
__device__ __forceinline__ void sys_issue_chunk(const SysPlan& S, const double* src_v, unsigned char* sm, long long c,
                                                long long q) {
    const int slot = static_cast<int>(q % kSysRing);
    double* dv = reinterpret_cast<double*>(sm + S.smem_ring_v) + static_cast<size_t>(slot) * kSysChunk;
    int* dc = reinterpret_cast<int*>(sm + S.smem_ring_c) + static_cast<size_t>(slot) * kSysChunk;
    unsigned long long* mb = reinterpret_cast<unsigned long long*>(sm + S.smem_mbar) + slot;
    const unsigned bytes_v = kSysChunk * sizeof(double), bytes_c = kSysChunk * sizeof(int);
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sys_smem_addr(mb)), "r"(bytes_v + bytes_c)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(sys_smem_addr(dv)),
        "l"(src_v + static_cast<size_t>(c) * kSysChunk), "r"(bytes_v), "r"(sys_smem_addr(mb))
        : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(sys_smem_addr(dc)),
        "l"(S.bcol + static_cast<size_t>(c) * kSysChunk), "r"(bytes_c), "r"(sys_smem_addr(mb))
        : "memory");
}

__device__ __forceinline__ void sys_wait_chunk(const SysPlan& S, unsigned char* sm, long long seq) {
    unsigned long long* mb = reinterpret_cast<unsigned long long*>(sm + S.smem_mbar) + static_cast<int>(seq % kSysRing);
    const unsigned parity = static_cast<unsigned>((seq / kSysRing) & 1);
    unsigned done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(sys_smem_addr(mb)), "r"(parity)
            : "memory");
    }
}

// IEEE division out of line: an inline `x / d` in one arm of the guarded-Markstein
// selection is if-converted by the compiler, i.e. evaluated (slow path included) for
// every quotient, also when the fast arm is taken
__device__ __noinline__ double sys_div_ieee(double x, double d) { return x / d; }

// Pivot reciprocal with the Markstein range of codegen.cpp (EMT_RCP): NaN outside [2^-60, 2^960].
__device__ __forceinline__ double sys_rcp(double u) {
    return (fabs(u) >= 0x1p-60 && fabs(u) <= 0x1p960) ? 1.0 / u : __longlong_as_double(0x7ff8000000000000LL);
}

// The lane's factor streams from its current factors: the backward stream (U entries,
// diagonal, reciprocal), the forward stream (L values in round order) and the dense
// diagonal tiles. Run at launch start and after every factorisation.
__device__ __forceinline__ void sys_build_stream(const DevPlan& P, const SysPlan& S, const double* __restrict__ A,
                                                 double* __restrict__ bv, double* __restrict__ fv,
                                                 double* __restrict__ tv) {
    const double* Uv = A + P.u;
    const double* Lv = A + P.l;
    for (long long e = threadIdx.x; e < S.stream_len; e += kSysThreads) {
        const int s = __ldg(&S.bsrc[e]);
        bv[e] = s >= 0 ? Uv[s] : (s == INT_MIN ? 0.0 : sys_rcp(Uv[-1 - s]));
    }
    for (long long e = threadIdx.x; e < S.fstream_len; e += kSysThreads) {
        const int k = __ldg(&S.fsrc[e]);
        fv[e] = k >= 0 ? Lv[k] : 0.0;  // -1: the placeholder entry of an empty stream
    }
    for (long long q = threadIdx.x; q < static_cast<long long>(S.nblk) * 1024; q += kSysThreads) {
        const int s = __ldg(&S.tsrc[q]);
        tv[q] = s >= 0 ? Lv[s] : 0.0;
    }
}

__device__ __forceinline__ void sys_cp_async(void* dst, const void* src, int bytes) {
    if (bytes == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sys_smem_addr(dst)), "l"(src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sys_smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void sys_cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void sys_cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

constexpr int kSysFD = 4;  // factorisation: elimination steps whose operands are in flight (cp.async)
static_assert(kSysFD * kSysThreads <= kSysRing * kSysChunk, "factorisation pipeline must fit the TMA ring");

// FactorizeSystem for one lane on the whole block (exec.cpp:175-204 + lu_factor,
// sparse.cpp:79-145): the reference's up-looking rows, one row at a time; within a
// row the eliminations run in ascending column order, each one's update of the
// scratch row spread over the block (the scratch row lives in shared memory). The
// quotient S[c] / U(c,c) is the guarded Markstein division (the IEEE quotient bit
// for bit) with the reciprocal kept per row. Returns the block-uniform error flag.
__device__ int sys_factorize(const DevPlan& P, const SysPlan& S, double* __restrict__ A, unsigned char* sm, int lane,
                             int step, int row, int layer) {
    const int tid = threadIdx.x, tl = tid & 31, wid = tid >> 5;
    double* Sx = reinterpret_cast<double*>(sm + S.smem_xs);
    __shared__ double s_max[32];
    double* G = A + P.mat;
    double m = 0.0;  // max |A| of the lane, sparse.cpp:84-90 (std::max keeps m on NaN)
    for (int k = tid; k < P.nnz; k += kSysThreads) {
        double d = 0.0;
        for (int q = __ldg(&P.ment_ptr[k]); q < __ldg(&P.ment_ptr[k + 1]); ++q)
            d += __ldg(&P.ment_sign[q]) * A[__ldg(&P.ment_slot[q])];
        G[k] = d;
        const double x = fabs(d);
        m = m < x ? x : m;
    }
    for (int off = 16; off > 0; off >>= 1) {
        const double o = __shfl_xor_sync(kFull, m, off);
        m = m < o ? o : m;
    }
    if (tl == 0) s_max[wid] = m;
    __syncthreads();
    m = 0.0;
    for (int w = 0; w < kSysThreads / 32; ++w) m = m < s_max[w] ? s_max[w] : m;
    double* Lv = A + P.l;
    double* Uv = A + P.u;
    double* R = S.frcp + static_cast<size_t>(lane) * static_cast<size_t>(P.dim > 0 ? P.dim : 1);
    double* fuv = reinterpret_cast<double*>(sm + S.smem_ring_v);  // [kSysFD][1024] (the TMA ring is idle here)
    int* fuc = reinterpret_cast<int*>(sm + S.smem_ring_c);
    double* fdr = reinterpret_cast<double*>(sm + S.smem_desc);    // [kSysFD][2]
    int4* fde = reinterpret_cast<int4*>(sm + S.smem_pbuf);        // [kSysFD] lent entries (pbuf idle here)
    long long tf = clock64();
    for (int i = 0; i < P.dim; ++i) {
        const int lb = __ldg(&P.l_row_ptr[i]), le = __ldg(&P.l_row_ptr[i + 1]);
        const int ub = __ldg(&P.u_row_ptr[i]), ue = __ldg(&P.u_row_ptr[i + 1]);
        // operands of the row's first eliminations in flight (cp.async into the idle TMA
        // ring): each thread's U entry and column, thread 0 the pivot and its reciprocal
        const int n = le - lb;
        // e4 = lent[k] (c, U row [cb, ce)), loaded one elimination before its issue so
        // that no step waits on it; thread 0 keeps it in shared memory for the step
        auto issue = [&](const int4 e4, int slot) {
            const int j = e4.y + 1 + tid;
            if (j < e4.z) {
                sys_cp_async(fuv + slot * kSysThreads + tid, Uv + j, 8);
                sys_cp_async(fuc + slot * kSysThreads + tid, P.u_col + j, 4);
            }
            if (tid == 0) {
                sys_cp_async(fdr + 2 * slot, Uv + e4.y, 8);
                sys_cp_async(fdr + 2 * slot + 1, R + e4.x, 8);
                fde[slot] = e4;
            }
        };
        const int nft = S.fact_threads;  // the other warps skip the eliminations (nothing to update)
        int4 e_nx = make_int4(0, 0, 0, 0);
        if (tid < nft) {
            for (int q = 0; q < kSysFD - 1; ++q) {
                if (q < n) issue(__ldg(&S.lent[lb + q]), q);
                sys_cp_commit();
            }
            if (kSysFD - 1 < n) e_nx = __ldg(&S.lent[lb + kSysFD - 1]);
        }
        // scatter row i of A over the union pattern, fill positions zero (sparse.cpp:94-110)
        for (int q = lb + tid; q < le; q += kSysThreads) Sx[__ldg(&P.l_col[q])] = 0.0;
        for (int q = ub + tid; q < ue; q += kSysThreads) Sx[__ldg(&P.u_col[q])] = 0.0;
        __syncthreads();
        for (int q = __ldg(&P.row_ptr[i]) + tid; q < __ldg(&P.row_ptr[i + 1]); q += kSysThreads)
            Sx[__ldg(&P.col_idx[q])] = G[q];
        sys_cp_wait<kSysFD - 2>();
        __syncthreads();
        sys_mark(S, tf, 12);  // factorisation: row set-up
        // eliminate with the settled rows, ascending columns (sparse.cpp:112-124); the
        // participating warps synchronise on named barrier 1 only
        if (tid < nft)
        for (int sidx = 0; sidx < n; ++sidx) {
            const int k = lb + sidx, slot = sidx % kSysFD;
            if (sidx + kSysFD - 1 < n) issue(e_nx, (sidx + kSysFD - 1) % kSysFD);
            sys_cp_commit();
            if (sidx + kSysFD < n) e_nx = __ldg(&S.lent[k + kSysFD]);
            const int4 e4 = fde[slot];
            const double x = Sx[e4.x], d = fdr[2 * slot], r = fdr[2 * slot + 1];
            // x / d: Markstein while |x r| is in range; a zero x (three in four L entries of the
            // gen_scale_case factors are exact zeros) gives x r = the signed zero x / d whenever
            // 1/d is in range (not NaN); anything else takes the IEEE division
            const double q0 = x * r;
            const double lik = (fabs(q0) >= 0x1p-900 && fabs(q0) <= 0x1p900) ? __fma_rn(__fma_rn(-d, q0, x), r, q0)
                               : (x == 0.0 && r == r)                          ? q0
                                                                               : sys_div_ieee(x, d);
            if (tid == 0) Lv[k] = lik;
            const int j = e4.y + 1 + tid;
            if (j < e4.z) {
                const int cj = fuc[slot * kSysThreads + tid];
                Sx[cj] = Sx[cj] - lik * fuv[slot * kSysThreads + tid];
            }
            for (int jj = j + kSysThreads; jj < e4.z; jj += kSysThreads) {  // U rows longer than the block
                const int cj = __ldg(&P.u_col[jj]);
                Sx[cj] = Sx[cj] - lik * Uv[jj];
            }
            sys_cp_wait<kSysFD - 2>();
            asm volatile("bar.sync 1, %0;\n" ::"r"(nft) : "memory");
        }
        __syncthreads();
        sys_mark(S, tf, 13);  // factorisation: eliminations
        if (S.prof != nullptr && tid == 0) S.prof[15] += n;
        for (int q = ub + tid; q < ue; q += kSysThreads) Uv[q] = Sx[__ldg(&P.u_col[q])];
        const double piv = Sx[i];  // U(i, i), first in its row (sparse.cpp:126-131)
        if (tid == 0) R[i] = sys_rcp(piv);
        if (!(fabs(piv) > 1e-12 * m)) {  // sparse.cpp:133-143
            if (tid == 0) lane_fail(P, lane, 8 /*SingularMatrix*/, step, i, layer, 0);
            return 1;
        }
        __syncthreads();
        sys_mark(S, tf, 14);  // factorisation: U row, pivot
    }
    // the scratch row's final contents (every column is some row's diagonal, so all are written)
    double* scr = A + P.scratch;
    for (int c = tid; c < P.dim; c += kSysThreads) scr[c] = Sx[c];
    for (int q = tid; q < P.nwatch; q += kSysThreads) A[__ldg(&P.watch[q])] = 0.0;
    if (tid == 0) {
        A[P.fcount] += 1.0;
        P.refactored[row] = 1;
    }
    return 0;
}

// SolveSystem for one lane on the whole block (exec.cpp:205-239 + lu_solve, sparse.cpp:147-172).
// Returns the block-uniform error flag. `seq` is warp 0's running count of stream chunks.
__device__ int sys_solve(const DevPlan& P, const SysPlan& S, double* __restrict__ A, const double* __restrict__ bv,
                         const double* __restrict__ fv, const double* __restrict__ tv, unsigned char* sm, long long& seq, int lane, int step, int layer, long long& tp) {
    const int tid = threadIdx.x, wid = tid >> 5, tl = tid & 31;
    double* xs = reinterpret_cast<double*>(sm + S.smem_xs);
    double* tile = reinterpret_cast<double*>(sm + S.smem_tile);  // [32][33]
    __shared__ int s_bad, s_stall;
    if (tid == 0) {
        s_bad = INT_MAX;
        s_stall = 0;
        volatile int* fl = reinterpret_cast<volatile int*>(sm + S.smem_flags);
        fl[0] = P.dim;  // frontier: rows >= frontier are final
        fl[1] = -1;
        fl[2] = -1;
    }
    if (P.dim > 0) {
    // stream chunks of this pass: in flight during the gather and the forward sweep
    if (tid == 32) {  // warp 1 owns the ring
        for (int c = 0; c < kSysRing && c < S.stream_chunks; ++c) sys_issue_chunk(S, bv, sm, c, seq + c);
    }
    // gather in the canonical order (exec.cpp:207-214)
    for (int node = tid; node < P.nodes; node += kSysThreads) {
        double acc = 0.0;
        for (int q = __ldg(&P.gat_ptr[node]); q < __ldg(&P.gat_ptr[node + 1]); ++q) acc += A[__ldg(&P.gat_slot[q])];
        xs[node] = acc;
    }
    __syncthreads();
    sys_mark(S, tp, 11);  // gather
    double* fp = reinterpret_cast<double*>(sm + S.smem_fp);
    auto stage_tile = [&](int b) {  // block b's dense lower-triangular tile, one coalesced load per thread
        tile[(tid >> 5) * 33 + tl] = tv[static_cast<size_t>(b) * 1024 + tid];
    };
    stage_tile(0);
    __syncthreads();
    unsigned cols_next = __ldg(&S.blk_cols[0]);
    unsigned m_next = tl < P.dim ? __ldg(&S.fwd_mask[tl]) : 0u;
    for (int b = 0; b < S.nblk; ++b) {
        const unsigned cols = cols_next, m = m_next;  // loaded one block ahead
        if (b + 1 < S.nblk) {
            cols_next = __ldg(&S.blk_cols[b + 1]);
            m_next = 32 * (b + 1) + tl < P.dim ? __ldg(&S.fwd_mask[32 * (b + 1) + tl]) : 0u;
        }
        if (wid == 0 && cols != 0u) {  // rows 32b.. resolve their in-block terms, ascending column
            const int r = 32 * b + tl;
            const bool ok = r < P.dim;
            double x = ok ? xs[r] : 0.0;
            unsigned cm = cols;
            while (cm) {
                const int c = __ffs(cm) - 1;
                cm &= cm - 1;
                const double vc = __shfl_sync(kFull, x, c);
                if ((m >> c) & 1u) x = x - tile[tl * 33 + c] * vc;
            }
            if (ok) xs[r] = x;
        }
        __syncthreads();
        sys_mark(S, tp, 8);  // forward tile chains
        // every later row applies this block's columns, a round at a time: the round's
        // products in parallel (coalesced stream loads), then each row subtracts its
        // products in ascending column order (sparse.cpp:152-160)
        for (int q = __ldg(&S.rnd_ptr[b]); q < __ldg(&S.rnd_ptr[b + 1]); ++q) {
            const int4 rd4 = __ldg(&S.rnd[q]);
            for (int e0 = rd4.x + tid; e0 < rd4.y; e0 += 4 * kSysThreads) {  // four loads in flight per thread
                double v[4];
                int c[4], d[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int e = e0 + u * kSysThreads;
                    v[u] = e < rd4.y ? fv[e] : 0.0;
                    c[u] = e < rd4.y ? __ldg(&S.fcol[e]) : 0;
                    d[u] = e < rd4.y ? __ldg(&S.fdst[e]) : 0;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int e = e0 + u * kSysThreads;
                    if (e < rd4.y) fp[d[u]] = v[u] * xs[c[u]];
                }
            }
            if (q == __ldg(&S.rnd_ptr[b]) && b + 1 < S.nblk) stage_tile(b + 1);
            __syncthreads();
            sys_mark(S, tp, 9);  // forward round products
            for (int pc = rd4.z + tid; pc < rd4.w; pc += kSysThreads) {
                const int4 pi = __ldg(&S.piece[pc]);
                const double* f = fp + pi.y;
                double x = xs[pi.x];
#pragma unroll 4
                for (int j = 0; j < pi.z; ++j) x = x - f[j * pi.w];
                xs[pi.x] = x;
            }
            __syncthreads();
            sys_mark(S, tp, 10);  // forward round chains
        }
    }
    sys_mark(S, tp, 2);  // gather + forward
    // backward sweep, rows descending. Warp 1 (producer) streams U through the TMA ring
    // and writes row r's products u_rj * v_j for every column j >= r+2 into a
    // double-buffered row slot as soon as rows >= r+2 are final, i.e. while warp 0
    // (consumer) still runs row r+1's chain. Warp 0 forms the product with v_{r+1}
    // (which it just computed, the row's first term when present), subtracts the row's
    // products in ascending column order (sparse.cpp:164-168) eight at a time with the
    // next eight loads in flight, and divides (sparse.cpp:169-170). Products are
    // zero-padded to a multiple of eight: x - (+0) == x bit for bit (also for x = -0).
    // The consumer's chain is the pass's critical path.
    volatile int* flags = reinterpret_cast<volatile int*>(sm + S.smem_flags);  // [0] frontier, [1..2] row ready
    double* pbuf = reinterpret_cast<double*>(sm + S.smem_pbuf);                // [2][pmax]
    double* desc = reinterpret_cast<double*>(sm + S.smem_desc);                // [2][4]: u_{r,r+1}, diag, rcp
    if (wid == 1) {
        const double* rv = reinterpret_cast<const double*>(sm + S.smem_ring_v);
        const int* rc = reinterpret_cast<const int*>(sm + S.smem_ring_c);
        const long long seq0 = seq;  // this pass's chunk c has sequence number seq0 + c
        long long waited = 0, recycled = 0;
        long long pos = 0;
        auto ready = [&](long long idx) {  // chunks up to idx landed
            const long long need = idx >> kSysChunkLog;
            while (waited <= need) {
                sys_wait_chunk(S, sm, seq0 + waited);
                ++waited;
            }
        };
        auto recycle = [&](long long below) {  // chunks wholly below `below` are consumed: refill their slots
            const long long upto = below >> kSysChunkLog;
            if (recycled < upto) {
                __syncwarp();
                while (recycled < upto) {
                    if (tl == 0 && recycled + kSysRing < S.stream_chunks)
                        sys_issue_chunk(S, bv, sm, recycled + kSysRing, seq0 + recycled + kSysRing);
                    ++recycled;
                }
            }
        };
        auto slot = [&](long long e) {
            return static_cast<int>((seq0 + (e >> kSysChunkLog)) & (kSysRing - 1)) * kSysChunk + static_cast<int>(e & (kSysChunk - 1));
        };
        long long t_pwait = 0;  // developer profile (S.prof)
        int inf_next = __ldg(&S.brow[0]);
        for (int r = P.dim - 1; r >= 0; --r) {
            const int inf = inf_next;
            if (r > 0) inf_next = __ldg(&S.brow[P.dim - r]);
            const int len = inf >> 1;
            const bool adj = (inf & 1) != 0;
            const int buf = r & 1;
            ready(pos + len + 1);
            // row data not depending on fresh rows, loaded before the wait
            const double u0 = adj ? rv[slot(pos)] : 0.0, d = rv[slot(pos + len)], rcp = rv[slot(pos + len + 1)];
            // rows >= r+2 final (this also frees the buffer row r+2 used)
            const long long c0 = S.prof ? clock64() : 0;
            __syncwarp();
            unsigned spins = 0;
            while (flags[0] > r + 2 && ++spins < kSysSpinLimit) {
            }
            if (spins >= kSysSpinLimit) {
                if (tl == 0) s_stall = 1;
                break;
            }
            __threadfence_block();
            if (S.prof) t_pwait += clock64() - c0;
            double* pb = pbuf + buf * S.pmax;
            const int t0 = adj ? 1 : 0, tend = t0 + ((len - t0 + 7) & ~7);
            for (int t = tl + t0; t < tend; t += 32) {
                const long long e = pos + t;
                pb[t] = t < len ? rv[slot(e)] * xs[rc[slot(e)]] : 0.0;
            }
            if (tl == 0) {
                desc[buf * 4 + 0] = u0;
                desc[buf * 4 + 1] = d;
                desc[buf * 4 + 2] = rcp;
            }
            __syncwarp();
            __threadfence_block();
            if (tl == 0) flags[1 + buf] = r;
            pos += len + 2;
            recycle(pos);
        }
        recycle(S.stream_len);
        seq = seq0 + S.stream_chunks;
        if (S.prof && tl == 0) S.prof[7] += t_pwait;
        __syncwarp();
    } else if (wid == 0) {
        double last = 0.0;  // v_{i+1}, just computed
        long long t_wait = 0, t_chain = 0;  // developer profile (S.prof)
        int inf_next = __ldg(&S.brow[0]);
        for (int i = P.dim - 1; i >= 0; --i) {
            const int inf = inf_next;
            if (i > 0) inf_next = __ldg(&S.brow[P.dim - i]);
            const int len = inf >> 1;
            const bool adj = (inf & 1) != 0;
            const int buf = i & 1;
            double x = xs[i];
            const long long c0 = S.prof ? clock64() : 0;
            __syncwarp();
            unsigned spins = 0;
            while (flags[1 + buf] != i && ++spins < kSysSpinLimit) {
            }
            if (spins >= kSysSpinLimit) {
                if (tl == 0) s_stall = 1;
                break;
            }
            // one fence: acquires row i's products and releases v_{i+1} (stored at the end
            // of the previous row) before the frontier moves to i+1
            __threadfence_block();
            if (tl == 0) flags[0] = i + 1;
            const long long c1 = S.prof ? clock64() : 0;
            const double* pb = pbuf + buf * S.pmax;
            const double u1 = desc[buf * 4 + 0], d = desc[buf * 4 + 1], rcp = desc[buf * 4 + 2];
            int t = 0;
            if (adj) {
                x = x - u1 * last;
                t = 1;
            }
            if (len > t) {  // groups of eight (zero-padded), the next group's loads in flight
                double q0 = pb[t], q1 = pb[t + 1], q2 = pb[t + 2], q3 = pb[t + 3];
                double q4 = pb[t + 4], q5 = pb[t + 5], q6 = pb[t + 6], q7 = pb[t + 7];
#pragma unroll 2
                for (t += 8; t < len; t += 8) {
                    const double n0 = pb[t], n1 = pb[t + 1], n2 = pb[t + 2], n3 = pb[t + 3];
                    const double n4 = pb[t + 4], n5 = pb[t + 5], n6 = pb[t + 6], n7 = pb[t + 7];
                    x = x - q0; x = x - q1; x = x - q2; x = x - q3;
                    x = x - q4; x = x - q5; x = x - q6; x = x - q7;
                    q0 = n0; q1 = n1; q2 = n2; q3 = n3; q4 = n4; q5 = n5; q6 = n6; q7 = n7;
                }
                x = x - q0; x = x - q1; x = x - q2; x = x - q3;
                x = x - q4; x = x - q5; x = x - q6; x = x - q7;
            }
            // x / d: Markstein's correction of x * (1/d) is the IEEE quotient while
            // 1/d is in range (else NaN) and |q0| stays in [2^-900, 2^900]
            const double q0 = x * rcp;
            const double mk = __fma_rn(__fma_rn(-d, q0, x), rcp, q0);
            if (__builtin_expect(fabs(q0) >= 0x1p-900 && fabs(q0) <= 0x1p900, 1))
                x = mk;
            else if (x == 0.0 && rcp == rcp)  // signed zero quotient (1/d in range)
                x = q0;
            else
                x = sys_div_ieee(x, d);
            last = x;
            if (tl == 0) xs[i] = x;
            if (S.prof) {
                const long long c2 = clock64();
                t_wait += c1 - c0;
                t_chain += c2 - c1;
            }
            __syncwarp();
        }
        if (S.prof && tl == 0) {
            S.prof[5] += t_wait;
            S.prof[6] += t_chain;
        }
        __syncwarp();
    }
    }  // P.dim > 0
    __syncthreads();
    sys_mark(S, tp, 3);  // backward
    double* v = A + P.v_base;
    for (int node = tid; node < P.nodes; node += kSysThreads) {
        const double x = xs[node];
        v[node] = x;
        if (!(fabs(x) <= P.div_limit)) atomicMin(&s_bad, node);  // first diverged node, exec.cpp:229-237
    }
    __syncthreads();
    for (int c = tid; c < P.comps; c += kSysThreads) {  // i = g (v_b - v_a) + h, exec.cpp:220-228
        const int* f = P.fin + 5 * c;
        const double vs = rd(A, __ldg(f + 4)) - rd(A, __ldg(f + 3));
        A[__ldg(f + 0)] = A[__ldg(f + 1)] * vs + A[__ldg(f + 2)];
    }
    sys_mark(S, tp, 4);  // write-back, divergence, finalize
    if (s_stall) {  // a backward handoff wait timed out (never expected): report, do not hang
        if (tid == 0) lane_fail(P, lane, 64, step, -2, layer, 0);
        return 1;
    }
    const int bad = s_bad;
    if (bad != INT_MAX) {
        if (tid == 0) lane_fail(P, lane, 7 /*NonFiniteState*/, step, bad, layer, 0);
        return 1;
    }
    return 0;
}

__global__ void __launch_bounds__(kSysThreads, 1)
emt_system_kernel(const DevPlan P, const SysPlan S, const int step0, const int nsteps, const int row0) {
    extern __shared__ __align__(128) unsigned char sys_smem[];
    const int tid = threadIdx.x;
    const int lane = blockIdx.x;
    if (P.lane_err[lane].code != 0) return;  // lane already failed: frozen
    double* A;
    const double* C;
    if (P.W == 1) {  // the arena and constant table are the lane's own (slot-major with one lane)
        A = P.arena;
        C = P.ctab;
    } else {
        A = S.work + static_cast<size_t>(lane) * P.lane_stride;
        double* Cw = A + P.ext_pad;
        for (int s = tid; s < P.extent; s += kSysThreads) A[s] = P.arena[static_cast<size_t>(s) * P.W + lane];
        for (int s = tid; s < P.consts; s += kSysThreads) Cw[s] = P.ctab[static_cast<size_t>(s) * P.W + lane];
        C = Cw;
    }
    if (tid < kSysRing) {
        unsigned long long* mb = reinterpret_cast<unsigned long long*>(sys_smem + S.smem_mbar) + tid;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sys_smem_addr(mb)) : "memory");
    }
    double* tile = reinterpret_cast<double*>(sys_smem + S.smem_tile);
    for (int q = tid; q < 32 * 33; q += kSysThreads) tile[q] = 0.0;
    __syncthreads();
    double* bv = S.bval + static_cast<size_t>(lane) * S.stream_len;
    double* fv = S.fval + static_cast<size_t>(lane) * S.fstream_len;
    double* tv = S.tval + static_cast<size_t>(lane) * S.nblk * 1024;
    sys_build_stream(P, S, A, bv, fv, tv);
    asm volatile("fence.proxy.async.global;\n" ::: "memory");  // generic stores -> TMA reads
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncthreads();

    long long seq = 0;  // warp 1: stream chunks issued so far (ring slot / mbarrier phase)
    long long tp = clock64();
    int err = 0;
    for (int it = 0; it < nsteps; ++it) {
        const int step = step0 + it;
        const int row = row0 + it;
        const double t = static_cast<double>(step + 1) * P.dt;  // exec.cpp:366
        for (int layer = 0; layer < P.layers; ++layer) {
            const int e = __ldg(&P.layer_begin[layer + 1]);
            for (int k = __ldg(&P.layer_begin[layer]) + tid; k < e; k += kSysThreads) run_regular(P, A, C, k, t, step, lane);
            const int fl = __ldg(&P.layer_flags[layer]);
            if (fl != 0) {
                __syncthreads();
                sys_mark(S, tp, 0);  // layers
                if (fl & 1) {
                    bool set = false;
                    for (int q = tid; q < P.nwatch; q += kSysThreads) set |= (A[__ldg(&P.watch[q])] != 0.0);
                    if (__syncthreads_or(set)) {
                        err = sys_factorize(P, S, A, sys_smem, lane, step, row, layer);
                        __syncthreads();
                        sys_mark(S, tp, 1);  // factorisation
                        if (!err) {
                            sys_build_stream(P, S, A, bv, fv, tv);
                            asm volatile("fence.proxy.async.global;\n" ::: "memory");
                        }
                        __syncthreads();
                    }
                }
                if (!err && (fl & 2)) err = sys_solve(P, S, A, bv, fv, tv, sys_smem, seq, lane, step, layer, tp);
                if (err) break;
            }
            __syncthreads();
        }
        if (err) break;
        // record (exec.cpp:313-321) then latch (exec.cpp:323-329)
        double* wrow = P.waves + static_cast<size_t>(row) * P.nch * P.W;
        for (int ch = tid; ch < P.nch; ch += kSysThreads)
            wrow[static_cast<size_t>(ch) * P.W + lane] = rd(A, __ldg(&P.ch_slot[ch]));
        __syncthreads();
        for (int q = tid; q < P.nlatch; q += kSysThreads) A[__ldg(&P.latch_shadow[q])] = A[__ldg(&P.latch_live[q])];
        __syncthreads();
        sys_mark(S, tp, 0);  // layers, record, latch
    }
    if (P.W != 1) {
        __syncthreads();
        for (int s = tid; s < P.extent; s += kSysThreads) P.arena[static_cast<size_t>(s) * P.W + lane] = A[s];
    }
}

