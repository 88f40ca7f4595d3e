// Schedule -> specialised sm_100a kernel source. See codegen.hpp and DESIGN.md §4.
//
// Semantics are those of the reference's per-process kernels
// (Engine::run_proc, /root/reference/proj/src/exec.cpp:77-311, and the
// code-database templates proj/data/codedb/cpp/*.tpl). The generator
//  1. turns the schedule's sequential process order into a dependency DAG of
//     fine-grained tasks (one per Norton update, gather node, triangular-solve
//     row, finalize component, control block, channel record, latch);
//  2. list-schedules the DAG onto the CTA's warps in barrier-separated phases;
//  3. emits, per component / block type, one compact loop over a constant-
//     memory task table (warp-uniform records, one scenario lane per thread),
//     and a per-warp phase program of (type, table range) segments.
// Compact loops keep the whole step in the instruction cache (a fully
// unrolled straight-line variant measured instruction-fetch bound, see
// profiles/ncu_r1b_cg8.json). Within a task every floating-point operation
// keeps the reference's order; NVRTC compiles with --fmad=false.
#include "codegen.hpp"

#include <algorithm>
#include <climits>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <set>
#include <sstream>

namespace emtb200 {

namespace {

// glibc's cos, operation for operation (libmcos.cuh), pasted into every generated source
#define EMT_LIBMCOS_TEXT(...) const char* const kLibmCosSrc = #__VA_ARGS__;
#include "libmcos.cuh"
#undef EMT_LIBMCOS_TEXT

std::string libm_cos_prelude() {
    return std::string("__device__ __forceinline__ int emt_lo32(double d) { return __double2loint(d); }\n"
                       // pivot reciprocal for the guarded Markstein division: NaN outside [2^-60, 2^960]
                       "#define EMT_RCP(u) ((fabs(u) >= 0x1p-60 && fabs(u) <= 0x1p960) ? 1.0 / (u) : "
                       "__longlong_as_double(0x7ff8000000000000LL))\n"
                       "__device__ __noinline__ double emt_div_ieee(double x, double d) { return x / d; }\n"
                       "#define EMT_HD __device__ __forceinline__\n#define EMT_TABLE __device__ const\n") +
           kLibmCosSrc + "\n";
}

// Generator tuning knobs. The product library ignores the environment: knob()
// returns the measured-best default. A developer build (build.py --dev, which
// defines EMTB200_DEV_KNOBS) reads EMTB200_CG_* overrides for A/B experiments,
// and the engine summary then lists every override in effect.
#ifdef EMTB200_DEV_KNOBS
std::string g_knobs_used;
int knob(const char* name, int dflt) {
    const char* v = std::getenv(name);
    if (!(v && *v)) return dflt;
    const int x = std::atoi(v);
    if (x != dflt && g_knobs_used.find(name) == std::string::npos)
        g_knobs_used += std::string(g_knobs_used.empty() ? "" : ",") + name + "=" + v;
    return x;
}
#else
int knob(const char*, int dflt) { return dflt; }
#endif

/// Per-warp bodies of a warp-major region ("    switch (warp) {" + one
/// "    case w: {" ... "    } break;" per warp + "    }"), false if the text differs.
bool split_warp_cases(const std::string& code, int G, std::vector<std::string>& bodies) {
    const std::string head = "    switch (warp) {\n", brk = "    } break;\n";
    if (code.compare(0, head.size(), head) != 0) return false;
    bodies.assign(static_cast<size_t>(G), std::string());
    size_t pos = head.size();
    for (int w = 0; w < G; ++w) {
        const std::string ch = "    case " + std::to_string(w) + ": {\n";
        if (code.compare(pos, ch.size(), ch) != 0) return false;
        pos += ch.size();
        const std::string nxt = brk + (w + 1 < G ? "    case " + std::to_string(w + 1) + ": {\n" : std::string("    }\n"));
        const size_t e = code.find(nxt, pos);
        if (e == std::string::npos) return false;
        bodies[static_cast<size_t>(w)] = code.substr(pos, e - pos);
        pos = e + brk.size();
    }
    return code.compare(pos, std::string::npos, "    }\n") == 0;
}

std::string dev_knob_note() {
#ifdef EMTB200_DEV_KNOBS
    return " devbuild" + (g_knobs_used.empty() ? std::string() : " knobs=" + g_knobs_used);
#else
    return std::string();
#endif
}

std::string lit(double v) {
    if (std::isnan(v) || std::isinf(v)) {
        long long bits;
        std::memcpy(&bits, &v, sizeof bits);
        char b[64];
        std::snprintf(b, sizeof b, "__longlong_as_double(0x%llxLL)", static_cast<unsigned long long>(bits));
        return b;
    }
    char b[64];
    std::snprintf(b, sizeof b, "(%a)", v);
    return b;
}

// Task kinds of the compact kernel; record strides in ints.
enum Kind {
    K_IND, K_CAP, K_SRL, K_VSRC, K_ISRC, K_CSRC, K_SW, K_GATHER, K_FWD, K_BWD, K_FINC, K_FINS,
    K_GAIN, K_SUM, K_INTEG, K_LAG, K_PI, K_LIM, K_CMP, K_CONST, K_DELAY, K_REC, K_LATCH, K_BERG,
    K_VSRCP, K_ISRCP, K_SRCPRE, K_VSRCT, K_ISRCT, K_NKINDS
};
const char* const kKindName[K_NKINDS] = {"IND", "CAP", "SRL", "VSRC", "ISRC", "CSRC", "SW", "GATHER",
                                         "FWD", "BWD", "FINC", "FINS", "GAIN", "SUM", "INTEG", "LAG",
                                         "PI", "LIM", "CMP", "CONST", "DELAY", "REC", "LATCH", "BERG",
                                         "VSRCP", "ISRCP", "SRCPRE", "VSRCT", "ISRCT"};
// kinds whose tasks never depend on another task of the same kind: eligible
// for the unrolled (loads-first) loop when a segment has no internal edges
bool unrollable(int k) { return k != K_SW; }

struct Task {
    int kind = 0;
    std::vector<int> f;                      // integer record fields (shared-memory offsets, flags)
    std::vector<int> ck;                     // constant-table slots of the constant fields
    std::vector<std::pair<int, int>> terms;  // variable-length operand list
    std::vector<int> reads, writes;          // arena slots, for dependencies
    int cost = 1;
    int region = 0;  // 0: before FactorizeSystem, 1: after
    bool fused = false;  // Norton task that also recomputes its own i_prev (finalize fused away)
    bool out_alias = false;  // integrator / lag whose output slot aliases its state slot (out == y == state0)
};

enum Cls { kNone = 0, kHot, kDerived, kContrib, kSolver, kChg, kAlias };

struct Gen {
    const Schedule& s;
    const std::vector<double>& ct;
    int W;
    CodegenOptions opt;

    std::vector<int> cls;            // per arena slot
    std::vector<int> derived_const;  // derived slot: const slot (or -1: literal 0.0)
    std::vector<int> contrib_h, contrib_sign;
    std::vector<int> hot_index;      // shared-memory slot (index 0 is the constant-0.0 slot)
    std::vector<int> hot_slots;      // arena slot per shared slot (-1 for the zero slot)
    int l_base_smem = -1, u_base_smem = -1;
    std::vector<int> vc_index;       // per const slot: shared slot caching a lane-varying constant, or -1
    std::vector<int> vc_slots;       // const slot per cached shared slot (in order)
    int vc_base = 0;                 // first shared slot of the constant cache
    bool chg_flag = false;           // switch "changed" slots replaced by one per-lane flag
    std::vector<int> chg_slots;
    std::vector<Task> tasks;
    int fact_layer = 0, solve_layer = 0;
    std::set<int> iread;        // arena slots some process / channel / latch reads
    std::vector<int> lazy_fin;  // components whose current no task reads: finalized once per launch

    bool lazy_i = true;
    bool dmma = false;  // shared-G tensor-core solve: the triangular sweeps become V = G^-1 I (DMMA)
    // AC sources (lane-invariant omega != 0): m cos(w t + p) for pass n+1 is computed
    // during pass n's solve, off the Norton phase's critical path; virtual slots
    // extent + j hold the values (shared memory only, never in the arena)
    bool presrc = false;
    std::map<int, int> pre_of;   // source process id -> j
    std::vector<std::array<int, 3>> pre_ck;  // j -> const slots (m, w, p)
    int pre_base = 0;
    // pivot reciprocals 1/u_ii in shared memory (rcp_base + row): the backward sweep's
    // division becomes q0 = x*r, x/u = fma(fma(-u, q0, x), r, q0) (Markstein; correctly
    // rounded for normal-range operands, tools/micro/divcheck.c). Range guard: the
    // reciprocal is NaN when |u| leaves [2^-60, 2^960] (EMT_RCP); with |q0| >= 2^-900
    // that keeps r and q0 normal and |x| >= 2^-960, so the remainder fma is exact and
    // the result is x / u bit for bit. Rows only AND |q0| >= 2^-900 into the divergence
    // predicate; the cold path tells a zero quotient (exact: x is never -0) from a
    // nonzero one below the bound, which stops the launch (EMT_INEXACT_DIVISION, and
    // emt_interpret reruns with the IEEE branch per row, EMT_FLAG_EXACT_DIVISION;
    // tests/golden/subnormal_decay). Huge q0 needs no test: |x| > 1e12 already fails
    // the divergence check, which reports the same node as IEEE division would.
    bool rcp = false;
    int rcp_base = -1;
    // shared factors: when G is the same constant matrix in every lane and nothing
    // changes it (no switches), every lane's refactorisation produces the same L, U
    // and pivot reciprocals; one copy per CTA (SH, broadcast reads) replaces the
    // per-lane [slot][lane] copies, which frees room for the reciprocals
    bool lu_shared = false;
    long long sh_base = -1;  // double offset of SH from the dynamic shared-memory base
    // finalize fusion: an L / C / RL component whose current only its own next-pass
    // Norton update reads gets i_prev = g (vb - va) + h recomputed there (the same
    // operands and order as the finalize), and its finalize runs once per launch
    bool fusefin = false;
    std::set<int> fused;  // component (= Norton process) ids
    // control outputs that always equal the block's first state slot (integrator and
    // first-order lag store y to both): readers use the state slot, the output slot is
    // written back once per launch (shared memory and one store per pass saved)
    std::map<int, int> alias_of;  // output slot -> state slot
    // lane-invariant AC sources tabulated per launch (emt_src_kernel): process id -> table column
    bool srctab = false;
    std::map<int, int> tab_of;
    std::vector<std::array<int, 3>> tab_ck;  // source -> const slots (m, w, p)
    std::vector<int> tab_var;                // source -> 1 when its value differs per lane
    int tab_shared() const { int n = 0; for (int v : tab_var) n += v == 0; return n; }
    /// table column of source j for this thread's lane (row = one pass)
    std::string tab_col(int j) const {
        const int ns = tab_shared();
        if (tab_var[static_cast<size_t>(j)] == 0) return std::to_string(j);
        return "(" + std::to_string(ns) + " + " + std::to_string(j - ns) + " * W_ + gl)";
    }
    int ls = 32;     // doubles between consecutive slots of one lane in S[] (32 lanes per CTA; 1 in task-SIMT)
    int unit = 256;  // record offset units per slot (bytes of a 32-lane row; 1 = slot index in task-SIMT)
    Gen(const Schedule& sc, const std::vector<double>& c, int w, const CodegenOptions& o) : s(sc), ct(c), W(w), opt(o) {
        lazy_i = knob("EMTB200_CG_LAZYI", 1) != 0;
    }

    /// Shared-G check for the tensor-core solve: no switches, the dirty flag is
    /// the only watch slot, and every conductance term of G is a lane-invariant
    /// constant — then G (and G^-1) is the same for every lane and every pass.
    bool shared_g() const {
        if (s.nodes <= 0 || s.dim != s.nodes || s.nodes > 64) return false;
        for (const Proc& p : s.procs)
            if (p.code == kNortonSwitch) return false;
        for (int x : s.watch)
            if (x != s.dirty) return false;
        for (int x : s.mentry_slot) {
            if (x < 0 || cls[static_cast<size_t>(x)] != kDerived) return false;
            const int k = derived_const[static_cast<size_t>(x)];
            if (k >= 0 && !invariant(k)) return false;
        }
        return true;
    }

    /// G^-1 (row-major, dim x dim): G assembled as FactorizeSystem does
    /// (exec.cpp:185-192), inverted by Gauss-Jordan with partial pivoting in
    /// long double and rounded once to double.
    bool g_inverse(std::vector<double>& inv) const {
        const int n = s.dim;
        std::vector<long double> a(static_cast<size_t>(n) * 2 * n, 0.0L);
        for (int i = 0; i < n; ++i) {
            for (int k = s.row_ptr[static_cast<size_t>(i)]; k < s.row_ptr[static_cast<size_t>(i) + 1]; ++k) {
                double gk = 0.0;
                for (int q = s.mentry_ptr[static_cast<size_t>(k)]; q < s.mentry_ptr[static_cast<size_t>(k) + 1]; ++q) {
                    const int x = s.mentry_slot[static_cast<size_t>(q)];
                    const int c = derived_const[static_cast<size_t>(x)];
                    gk = gk + s.mentry_sign[static_cast<size_t>(q)] * (c < 0 ? 0.0 : c0(c));
                }
                a[static_cast<size_t>(i) * 2 * n + static_cast<size_t>(s.col_idx[static_cast<size_t>(k)])] = gk;
            }
            a[static_cast<size_t>(i) * 2 * n + static_cast<size_t>(n + i)] = 1.0L;
        }
        for (int c = 0; c < n; ++c) {
            int piv = c;
            for (int r = c + 1; r < n; ++r)
                if (fabsl(a[static_cast<size_t>(r) * 2 * n + c]) > fabsl(a[static_cast<size_t>(piv) * 2 * n + c])) piv = r;
            if (a[static_cast<size_t>(piv) * 2 * n + c] == 0.0L) return false;
            if (piv != c)
                for (int j = 0; j < 2 * n; ++j) std::swap(a[static_cast<size_t>(c) * 2 * n + j], a[static_cast<size_t>(piv) * 2 * n + j]);
            const long double d = a[static_cast<size_t>(c) * 2 * n + c];
            for (int j = 0; j < 2 * n; ++j) a[static_cast<size_t>(c) * 2 * n + j] /= d;
            for (int r = 0; r < n; ++r) {
                if (r == c) continue;
                const long double f = a[static_cast<size_t>(r) * 2 * n + c];
                if (f == 0.0L) continue;
                for (int j = 0; j < 2 * n; ++j) a[static_cast<size_t>(r) * 2 * n + j] -= f * a[static_cast<size_t>(c) * 2 * n + j];
            }
        }
        inv.assign(static_cast<size_t>(n) * n, 0.0);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                inv[static_cast<size_t>(i) * n + j] = static_cast<double>(a[static_cast<size_t>(i) * 2 * n + n + j]);
        return true;
    }

    /// Deferred finalize (exec.cpp:220-228) of the currents no task reads, and the
    /// aliased control outputs (= their state slot).
    std::string emit_lazy_finalize() const {
        std::ostringstream o;
        for (const auto& kv : alias_of)
            o << "      A[(size_t)" << kv.first << " * W_] = " << R(kv.second) << ";\n";
        for (int c : lazy_fin) {
            const int* f = s.finalize.data() + 5 * c;
            std::string gx;
            if (f[1] < 0) gx = "(0.0)";
            else if (cls[static_cast<size_t>(f[1])] == kDerived) gx = R(f[1]);
            else gx = "S[" + std::to_string(hot_index[static_cast<size_t>(f[1])] * ls) + "]";
            o << "      { const double vs = " << R(f[4]) << " - " << R(f[3]) << "; A[(size_t)" << f[0]
              << " * W_] = " << gx << " * vs + " << R(f[2]) << "; }\n";
        }
        return o.str();
    }

    bool invariant(int k) const {
        const double* row = ct.data() + static_cast<size_t>(k) * W;
        for (int l = 1; l < W; ++l)
            if (std::memcmp(&row[l], &row[0], sizeof(double)) != 0) return false;
        return true;
    }
    double c0(int k) const { return ct[static_cast<size_t>(k) * W]; }
    /// shared-memory byte offset of an arena slot relative to the lane base
    int off(int slot) const {
        if (slot < 0) return 0;  // ground sentinel reads the zero slot
        if (slot >= s.extent) return (pre_base + slot - s.extent) * unit;  // precomputed source value
        if (cls[static_cast<size_t>(slot)] == kAlias) return off(alias_of.at(slot));
        if (cls[static_cast<size_t>(slot)] == kDerived && derived_const[static_cast<size_t>(slot)] < 0) return 0;
        if (hot_index[static_cast<size_t>(slot)] < 0) return 0;  // pass 1 (offsets not assigned yet)
        return hot_index[static_cast<size_t>(slot)] * unit;
    }
    int dep_slot(int slot) const {
        if (slot >= 0 && slot < s.extent && cls[static_cast<size_t>(slot)] == kContrib) return contrib_h[static_cast<size_t>(slot)];
        if (slot >= 0 && slot < s.extent && cls[static_cast<size_t>(slot)] == kAlias) return alias_of.at(slot);
        return slot;
    }
    // L/U operand codes: >= 0 a shared-memory byte offset (or arena slot); < 0 the
    // shared-factor entry SH[-(code + 1)]
    int lu_l(int k) const {
        if (lu_shared) return -(1 + k);
        return l_base_smem >= 0 ? (l_base_smem + k) * unit : s.l + k;
    }
    int lu_u(int k) const {
        if (lu_shared) return -(1 + static_cast<int>(s.l_col.size()) + k);
        return u_base_smem >= 0 ? (u_base_smem + k) * unit : s.u + k;
    }
    int sh_rcp(int i) const { return static_cast<int>(s.l_col.size() + s.u_col.size()) + i; }
    /// G is a lane-invariant constant and nothing refactorises it differently per lane
    bool factor_shared() const {
        if (s.nodes <= 0 || s.dim <= 0) return false;
        for (const Proc& p : s.procs)
            if (p.code == kNortonSwitch) return false;
        for (int x : s.watch)
            if (x != s.dirty) return false;
        for (int x : s.mentry_slot) {
            if (x < 0 || cls[static_cast<size_t>(x)] != kDerived) return false;
            const int k = derived_const[static_cast<size_t>(x)];
            if (k >= 0 && !invariant(k)) return false;
        }
        return true;
    }

    // ---- expressions for the straight-line refactorization
    std::string C(int k) const {
        if (invariant(k)) return lit(c0(k));
        return "__ldg(C + " + std::to_string(static_cast<long long>(k) * W) + ")";
    }
    std::string R(int slot) const {
        if (slot < 0) return "(0.0)";
        if (cls[static_cast<size_t>(slot)] == kAlias) return R(alias_of.at(slot));
        if (cls[static_cast<size_t>(slot)] == kDerived) {
            const int k = derived_const[static_cast<size_t>(slot)];
            return k < 0 ? std::string("(0.0)") : C(k);
        }
        return "S[" + std::to_string(hot_index[static_cast<size_t>(slot)] * ls) + "]";
    }
    std::string Wr(int slot) const { return "S[" + std::to_string(hot_index[static_cast<size_t>(slot)] * ls) + "]"; }
    std::string Lw(int k, const std::string& v) const {
        if (lu_shared) return "SH[" + std::to_string(k) + "] = " + v + ";";
        if (l_base_smem >= 0) return "S[" + std::to_string((l_base_smem + k) * ls) + "] = " + v + ";";
        return "if (live) A[" + std::to_string(static_cast<long long>(s.l + k) * W) + "] = " + v + ";";
    }
    std::string Uw(int k, const std::string& v) const {
        if (lu_shared) return "SH[" + std::to_string(s.l_col.size() + static_cast<size_t>(k)) + "] = " + v + ";";
        if (u_base_smem >= 0) return "S[" + std::to_string((u_base_smem + k) * ls) + "] = " + v + ";";
        return "if (live) A[" + std::to_string(static_cast<long long>(s.u + k) * W) + "] = " + v + ";";
    }

    void classify() {
        const size_t n = static_cast<size_t>(s.extent);
        pre_of.clear();
        pre_ck.clear();
        tab_of.clear();
        tab_ck.clear();
        tab_var.clear();
        if (srctab)
            for (int pass = 0; pass < 2; ++pass)  // shared columns first, then per-lane ones
                for (const Proc& p : s.procs) {
                    const int wk = p.code == kNortonVoltageSource ? p.par + 2 : p.code == kNortonCurrentSource ? p.par + 1 : -1;
                    if (wk < 0 || (invariant(wk) && c0(wk) == 0.0)) continue;  // DC (or omega varying incl. 0: below)
                    bool ok = true;  // omega must be nonzero in every lane
                    for (int l = 0; l < W && ok; ++l) ok = ct[static_cast<size_t>(wk) * W + l] != 0.0;
                    if (!ok) continue;
                    const bool shared = invariant(wk) && invariant(wk - 1) && invariant(wk + 1);
                    if (shared != (pass == 0)) continue;
                    tab_of[p.id] = static_cast<int>(tab_ck.size());
                    tab_ck.push_back({wk - 1, wk, wk + 1});
                    tab_var.push_back(shared ? 0 : 1);
                }
        if (presrc)
            for (const Proc& p : s.procs) {
                const int wk = p.code == kNortonVoltageSource ? p.par + 2 : p.code == kNortonCurrentSource ? p.par + 1 : -1;
                if (wk < 0 || !invariant(wk) || c0(wk) == 0.0) continue;
                const int mk = wk - 1;
                pre_of[p.id] = static_cast<int>(pre_ck.size());
                pre_ck.push_back({mk, wk, wk + 1});
            }
        iread.clear();
        for (const Proc& p : s.procs) {
            // ports a kernel actually reads (exec.cpp:85-309): Norton records carry
            // [v_a, v_b, i_prev(, actuator)] whatever the kind uses
            int lo = 0, hi = p.in_count;
            if (p.code == kNortonResistor || p.code == kNortonVoltageSource || p.code == kNortonCurrentSource ||
                p.code == kNortonSwitch)
                hi = 0;
            else if (p.code == kNortonControlledSource)
                lo = 3;
            else if (p.code == kNortonBergeron)
                hi = std::min(hi, 2);
            for (int j = lo; j < hi; ++j) iread.insert(s.port_slot[static_cast<size_t>(p.in_base + j)]);
        }
        for (int x : s.channel_slot) iread.insert(x);
        for (int x : s.latch_live) iread.insert(x);
        fused.clear();
        if (fusefin) {
            std::map<int, int> readers;  // slot -> number of reading ports / channels / latches
            for (const Proc& p : s.procs) {
                int lo = 0, hi = p.in_count;
                if (p.code == kNortonResistor || p.code == kNortonVoltageSource || p.code == kNortonCurrentSource ||
                    p.code == kNortonSwitch)
                    hi = 0;
                else if (p.code == kNortonControlledSource)
                    lo = 3;
                else if (p.code == kNortonBergeron)
                    hi = std::min(hi, 2);
                for (int j = lo; j < hi; ++j) readers[s.port_slot[static_cast<size_t>(p.in_base + j)]] += 1;
            }
            for (int x : s.channel_slot) readers[x] += 1;
            for (int x : s.latch_live) readers[x] += 1;
            for (const Proc& p : s.procs) {
                if (p.code != kNortonInductor && p.code != kNortonCapacitor && p.code != kNortonSeriesRL) continue;
                if (p.id < 0 || p.id >= s.comps || p.in_count < 3) continue;
                const int* f = s.finalize.data() + 5 * p.id;
                const int* in = s.port_slot.data() + p.in_base;
                if (f[0] < 0 || f[0] != in[2] || f[2] != p.out2 || f[3] != in[0] || f[4] != in[1] || f[1] != p.out) continue;
                if (readers[f[0]] != 1) continue;
                fused.insert(p.id);
            }
        }
        cls.assign(n, kNone);
        derived_const.assign(n, -2);
        contrib_h.assign(n, -1);
        contrib_sign.assign(n, 0);
        hot_index.assign(n, -1);
        auto mark_range = [&](int base, int len) {
            for (int k = 0; k < len; ++k)
                if (base + k >= 0 && base + k < s.extent) cls[static_cast<size_t>(base + k)] = kSolver;
        };
        mark_range(s.matrix, static_cast<int>(s.col_idx.size()));
        mark_range(s.l, static_cast<int>(s.l_col.size()));
        mark_range(s.u, static_cast<int>(s.u_col.size()));
        mark_range(s.scratch, s.dim);
        if (s.fcount >= 0) cls[static_cast<size_t>(s.fcount)] = kSolver;
        for (const auto& kv : alias_of) {
            cls[static_cast<size_t>(kv.first)] = kAlias;
        }
        for (const Proc& p : s.procs) {
            // Norton outputs that are constants every pass (exec.cpp:85-150)
            if (p.code < kNortonSwitch && p.out >= 0) {
                cls[static_cast<size_t>(p.out)] = kDerived;
                derived_const[static_cast<size_t>(p.out)] =
                    (p.code == kNortonCurrentSource || p.code == kNortonControlledSource) ? -1 : p.par;
            }
            if (p.code == kNortonBergeron && p.out >= 0) {  // g = 0 (the 1/Zc resistor is stamped separately)
                cls[static_cast<size_t>(p.out)] = kDerived;
                derived_const[static_cast<size_t>(p.out)] = -1;
            }
            if ((p.code == kNortonResistor || p.code == kNortonSwitch) && p.out2 >= 0) {
                cls[static_cast<size_t>(p.out2)] = kDerived;
                derived_const[static_cast<size_t>(p.out2)] = -1;
            }
            if (p.code == kInjectionPair && p.out >= 0 && p.in_count >= 1) {  // contrib = +-h (exact)
                const int h = s.port_slot[static_cast<size_t>(p.in_base)];
                for (int d = 0; d < 2; ++d) {
                    cls[static_cast<size_t>(p.out + d)] = kContrib;
                    contrib_h[static_cast<size_t>(p.out + d)] = h;
                    contrib_sign[static_cast<size_t>(p.out + d)] = d == 0 ? 1 : -1;
                }
            }
        }
    }

    void add(Task&& t, int region) {
        t.region = region;
        tasks.push_back(std::move(t));
    }

    void reads(Task& t, std::initializer_list<int> sl) const {
        for (int x : sl)
            if (x >= 0) t.reads.push_back(dep_slot(x));
    }

    // One non-singleton process (exec.cpp:85-309) -> task record.
    void emit_proc(const Proc& p, int region) {
        const int* in = s.port_slot.data() + p.in_base;
        const double* sg = s.port_sign.data() + p.in_base;
        auto IN = [&](int j) { return j < p.in_count ? in[j] : -1; };
        auto NEG = [&](int j) { return sg[j] < 0 ? 1 : 0; };
        Task t;
        switch (p.code) {
            case kNortonResistor:
            case kInjectionPair:
                return;  // constants / exact aliases of h
            case kNortonInductor:
            case kNortonCapacitor:
            case kNortonSeriesRL:
                t.kind = p.code == kNortonInductor ? K_IND : p.code == kNortonCapacitor ? K_CAP : K_SRL;
                reads(t, {IN(0), IN(1), IN(2)});
                if (fused.count(p.id)) {
                    t.fused = true;
                    t.reads.push_back(p.out2);
                }
                t.writes = {p.out2};
                t.f = {off(IN(0)), off(IN(1)), off(IN(2)), off(p.out2)};
                t.ck = {p.par};
                if (p.code == kNortonSeriesRL) t.ck.push_back(p.par + 1);
                t.cost = 10;
                break;
            case kNortonVoltageSource:
                if (tab_of.count(p.id)) {
                    t.kind = K_VSRCT;
                    t.writes = {p.out2};
                    t.f = {off(p.out2), tab_of.at(p.id)};
                    t.ck = {p.par};
                    t.cost = 30;
                    break;
                }
                if (pre_of.count(p.id)) {
                    const int vs = s.extent + pre_of.at(p.id);
                    t.kind = K_VSRCP;
                    t.reads = {vs};
                    t.writes = {p.out2};
                    t.f = {off(p.out2), off(vs)};
                    t.ck = {p.par};
                    t.cost = 8;
                    break;
                }
                t.kind = K_VSRC;
                t.writes = {p.out2};
                t.f = {off(p.out2)};
                t.ck = {p.par, p.par + 1, p.par + 2, p.par + 3};
                t.cost = invariant(p.par + 2) && c0(p.par + 2) == 0.0 ? 6 : 90;
                break;
            case kNortonCurrentSource:
                if (tab_of.count(p.id)) {
                    t.kind = K_ISRCT;
                    t.writes = {p.out2};
                    t.f = {off(p.out2), tab_of.at(p.id)};
                    t.cost = 30;
                    break;
                }
                if (pre_of.count(p.id)) {
                    const int vs = s.extent + pre_of.at(p.id);
                    t.kind = K_ISRCP;
                    t.reads = {vs};
                    t.writes = {p.out2};
                    t.f = {off(p.out2), off(vs)};
                    t.cost = 6;
                    break;
                }
                t.kind = K_ISRC;
                t.writes = {p.out2};
                t.f = {off(p.out2)};
                t.ck = {p.par, p.par + 1, p.par + 2};
                t.cost = invariant(p.par + 1) && c0(p.par + 1) == 0.0 ? 5 : 90;
                break;
            case kNortonControlledSource:
                t.kind = K_CSRC;
                if (p.in_count > 3) reads(t, {IN(3)});
                t.writes = {p.out2};
                t.f = {off(p.out2), p.in_count > 3 ? off(IN(3)) : 0};
                t.ck = {p.par};
                t.cost = 6;
                break;
            case kNortonBergeron:  // line end (extension): oracle/emt_oracle.c case K_BERG
                t.kind = K_BERG;
                reads(t, {IN(0), IN(1), p.out2});
                t.writes = {p.out2};  // + its ring in HBM (not a shared-memory slot: peers read it)
                t.f = {off(IN(0)), off(IN(1)), off(p.out2), p.state, p.state_len};
                for (int j = 0; j < 6; ++j) t.ck.push_back(p.par + j);
                t.cost = 40;
                break;
            case kNortonSwitch:  // exec.cpp:151-165
                t.kind = K_SW;
                t.reads = {p.state};
                t.writes = {p.state, p.state + 1, p.out};
                t.f = {off(p.state), off(p.state + 1), off(p.out), p.id};
                for (int j = 0; j < p.par_len; ++j) t.ck.push_back(p.par + j);
                t.cost = 14 + 3 * (p.par_len - 3);
                break;
            case kCtlGain:
                t.kind = K_GAIN;
                reads(t, {IN(0)});
                t.writes = {p.out};
                t.f = {off(p.out), off(IN(0)), NEG(0)};
                t.ck = {p.par};
                t.cost = 6;
                break;
            case kCtlSum:
                t.kind = K_SUM;
                for (int j = 0; j < p.in_count; ++j) {
                    reads(t, {IN(j)});
                    t.terms.push_back({off(IN(j)), NEG(j)});
                }
                t.writes = {p.out};
                t.f = {off(p.out)};
                t.cost = 6 + 4 * p.in_count;
                break;
            case kCtlIntegrator:
            case kCtlFirstOrderLag:
            case kCtlPiController:
                t.kind = p.code == kCtlIntegrator ? K_INTEG : p.code == kCtlFirstOrderLag ? K_LAG : K_PI;
                reads(t, {IN(0), p.state, p.state + 1});
                t.writes = {p.state, p.state + 1, p.out};
                if (p.out >= 0 && alias_of.count(p.out)) {
                    t.writes = {p.state, p.state + 1};
                    t.out_alias = true;
                }
                t.f = {off(p.out), off(IN(0)), off(p.state), off(p.state + 1), NEG(0)};
                t.ck = {p.par};
                if (p.code != kCtlIntegrator) t.ck.push_back(p.par + 1);
                t.cost = 10;
                break;
            case kCtlLimiter:
                t.kind = K_LIM;
                reads(t, {IN(0)});
                t.writes = {p.out};
                t.f = {off(p.out), off(IN(0)), NEG(0)};
                t.ck = {p.par, p.par + 1};
                t.cost = 7;
                break;
            case kCtlComparator:
                t.kind = K_CMP;
                reads(t, {IN(0), IN(1)});
                t.writes = {p.out};
                t.f = {off(p.out), off(IN(0)), off(IN(1)), NEG(0), NEG(1)};
                t.cost = 7;
                break;
            case kCtlConstant:
                t.kind = K_CONST;
                t.writes = {p.out};
                t.f = {off(p.out)};
                t.ck = {p.par};
                t.cost = 3;
                break;
            case kCtlDelay:
                t.kind = K_DELAY;
                reads(t, {IN(0)});
                t.writes = {p.out};
                t.f = {off(p.out), off(IN(0)), NEG(0)};
                t.cost = 4;
                break;
            default:
                return;
        }
        add(std::move(t), region);
    }

    // SolveSystem (exec.cpp:205-239): gather, lu_solve rows, finalize.
    void emit_solve(int region) {
        const int v = s.v_base;
        for (int node = 0; node < s.nodes; ++node) {
            Task t;
            t.kind = K_GATHER;
            for (int q = s.gather_ptr[static_cast<size_t>(node)]; q < s.gather_ptr[static_cast<size_t>(node) + 1]; ++q) {
                const int slot = s.gather_slot[static_cast<size_t>(q)];
                t.reads.push_back(dep_slot(slot));
                if (slot >= 0 && cls[static_cast<size_t>(slot)] == kContrib)
                    t.terms.push_back({off(contrib_h[static_cast<size_t>(slot)]),
                                       contrib_sign[static_cast<size_t>(slot)] < 0 ? 1 : 0});
                else
                    t.terms.push_back({off(slot), 0});
            }
            t.writes = {v + node};
            t.f = {off(v + node)};
            t.cost = 8 + 4 * static_cast<int>(t.terms.size());
            add(std::move(t), region);
        }
        if (dmma) region = 2;  // finalize and everything after reads V from the DMMA block
        if (s.nodes > 0 && !dmma) {
            for (int i = 0; i < s.dim; ++i) {  // forward, unit L (sparse.cpp:152-160)
                const int lb = s.l_row_ptr[static_cast<size_t>(i)], le = s.l_row_ptr[static_cast<size_t>(i) + 1];
                if (lb == le) continue;
                Task t;
                t.kind = K_FWD;
                t.reads.push_back(v + i);
                for (int k = lb; k < le; ++k) {
                    const int c = s.l_col[static_cast<size_t>(k)];
                    t.reads.push_back(v + c);
                    t.terms.push_back({lu_l(k), off(v + c)});
                }
                t.writes = {v + i};
                t.f = {off(v + i)};
                t.cost = 8 + 5 * (le - lb);
                add(std::move(t), region);
            }
            for (int i = s.dim - 1; i >= 0; --i) {  // backward (sparse.cpp:161-171) + divergence check
                const int ub = s.u_row_ptr[static_cast<size_t>(i)], ue = s.u_row_ptr[static_cast<size_t>(i) + 1];
                Task t;
                t.kind = K_BWD;
                t.reads.push_back(v + i);
                for (int k = ub + 1; k < ue; ++k) {
                    const int c = s.u_col[static_cast<size_t>(k)];
                    t.reads.push_back(v + c);
                    t.terms.push_back({lu_u(k), off(v + c)});
                }
                t.writes = {v + i};
                t.f = {off(v + i), lu_u(ub), i, lu_shared ? -(2 + i) : rcp_base >= 0 ? (rcp_base + i) * unit : -1};
                t.cost = 40 + 5 * (ue - ub - 1);
                add(std::move(t), region);
            }
        }
        for (int c = 0; c < s.comps; ++c) {  // i = g (v_b - v_a) + h
            const int* f = s.finalize.data() + 5 * c;
            if (fused.count(c)) {  // recomputed by its next-pass Norton update; arena copy once per launch
                lazy_fin.push_back(c);
                continue;
            }
            if (lazy_i && f[0] >= 0 && !iread.count(f[0])) {
                // nothing reads this current inside a pass: computing it from the
                // launch's final v, g, h gives the bits the last pass would have
                lazy_fin.push_back(c);
                continue;
            }
            Task t;
            t.reads = {dep_slot(f[1]), dep_slot(f[2])};
            if (f[3] >= 0) t.reads.push_back(f[3]);
            if (f[4] >= 0) t.reads.push_back(f[4]);
            t.writes = {f[0]};
            const bool gconst = f[1] >= 0 && cls[static_cast<size_t>(f[1])] == kDerived && derived_const[static_cast<size_t>(f[1])] >= 0;
            t.kind = gconst ? K_FINC : K_FINS;
            t.f = {off(f[0]), off(f[2]), off(f[3]), off(f[4])};
            if (gconst) t.ck = {derived_const[static_cast<size_t>(f[1])]};
            else t.f.push_back(off(f[1]));
            t.cost = 9;
            add(std::move(t), region);
        }
    }

    void emit_all(int& fact_count) {
        tasks.clear();
        lazy_fin.clear();
        int region = 0;
        fact_count = 0;
        for (int L = 0; L < s.layers; ++L) {
            for (int k = s.layer_begin[static_cast<size_t>(L)]; k < s.layer_begin[static_cast<size_t>(L) + 1]; ++k) {
                const Proc& p = s.procs[static_cast<size_t>(k)];
                if (p.code == kFactorizeSystem) {
                    ++fact_count;
                    region = 1;
                    fact_layer = L;
                    continue;
                }
                if (p.code == kSolveSystem) {
                    solve_layer = L;
                    emit_solve(region);
                    if (dmma) region = 2;
                    continue;
                }
                emit_proc(p, region);
            }
        }
        for (size_t j = 0; j < pre_ck.size(); ++j) {  // next pass's source values
            Task t;
            t.kind = K_SRCPRE;
            const int vs = s.extent + static_cast<int>(j);
            t.writes = {vs};
            t.f = {off(vs)};
            t.ck = {pre_ck[j][0], pre_ck[j][1], pre_ck[j][2]};
            t.cost = 90;
            add(std::move(t), dmma ? 2 : 1);
        }
        for (size_t ch = 0; ch < s.channel_slot.size(); ++ch) {  // record (exec.cpp:313-321)
            Task t;
            t.kind = K_REC;
            const int slot = s.channel_slot[ch];
            if (slot >= 0) t.reads.push_back(dep_slot(slot));
            t.f = {static_cast<int>(ch), off(slot)};
            t.cost = 4;
            add(std::move(t), dmma ? 2 : 1);
        }
        for (size_t q = 0; q < s.latch_live.size(); ++q) {  // latch (exec.cpp:323-329)
            Task t;
            t.kind = K_LATCH;
            t.reads = {s.latch_live[q]};
            t.writes = {s.latch_shadow[q]};
            t.f = {off(s.latch_live[q]), off(s.latch_shadow[q])};
            t.cost = 3;
            add(std::move(t), dmma ? 2 : 1);
        }
    }

    // Shared-memory layout per 32-lane group ([slot][lane] doubles): slot 0 holds
    // 0.0 (ground / derived zeros); then every arena slot the step loop reads or
    // writes, the watch slots and the switch conductances the refactorization
    // reads; then lane-varying constants the step reads (cached once per
    // launch); then L and U when they fit. Switch "changed" slots are always 0
    // at the end of a pass (FactorizeSystem clears them), so when every switch
    // updates before the factorization point they collapse into one per-lane
    // refactor flag instead of a slot each.
    bool assign_hot(bool& lu_smem, size_t& smem_bytes) {
        chg_flag = true;
        chg_slots.clear();
        for (const Proc& p : s.procs)
            if (p.code == kNortonSwitch) chg_slots.push_back(p.state + 1);
        for (const Task& t : tasks)
            if (t.kind == K_SW && t.region != 0) chg_flag = false;
        if (chg_flag)
            for (int x : chg_slots) cls[static_cast<size_t>(x)] = kChg;
        std::set<int> need;
        for (const Task& t : tasks) {
            for (int x : t.reads)
                if (x >= 0 && x < s.extent && cls[static_cast<size_t>(x)] == kNone) need.insert(x);
            for (int x : t.writes)
                if (x >= 0 && x < s.extent && cls[static_cast<size_t>(x)] == kNone) need.insert(x);
        }
        for (int x : s.watch)
            if (x >= 0 && cls[static_cast<size_t>(x)] == kNone) need.insert(x);
        for (int x : s.mentry_slot)
            if (x >= 0 && cls[static_cast<size_t>(x)] == kNone) need.insert(x);
        hot_slots.assign(1, -1);
        for (int x : need) {
            cls[static_cast<size_t>(x)] = kHot;
            hot_index[static_cast<size_t>(x)] = static_cast<int>(hot_slots.size());
            hot_slots.push_back(x);
        }
        const size_t per_slot = static_cast<size_t>(ls) * sizeof(double);
        const size_t fixed = 2 * static_cast<size_t>(ls) * sizeof(int) +  // serr + refactor flags
                             (lu_shared ? (s.l_col.size() + s.u_col.size() + static_cast<size_t>(s.dim)) * sizeof(double) : 0);
        pre_base = static_cast<int>(hot_slots.size());
        size_t used = (hot_slots.size() + pre_ck.size()) * per_slot + fixed;
        if (used > opt.smem_budget) return false;
        std::set<int> vc;
        for (const Task& t : tasks)
            for (int k : t.ck)
                if (!invariant(k)) vc.insert(k);
        vc_index.assign(static_cast<size_t>(s.consts), -1);
        vc_slots.clear();
        vc_base = static_cast<int>(hot_slots.size() + pre_ck.size());
        if (used + vc.size() * per_slot <= opt.smem_budget) {
            for (int k : vc) {
                vc_index[static_cast<size_t>(k)] = vc_base + static_cast<int>(vc_slots.size());
                vc_slots.push_back(k);
            }
            used += vc.size() * per_slot;
        }
        const int next = vc_base + static_cast<int>(vc_slots.size());
        const size_t lu = (s.l_col.size() + s.u_col.size()) * per_slot;
        lu_smem = !lu_shared && opt.lu_in_smem && used + lu <= opt.smem_budget;
        if (lu_smem) {
            l_base_smem = next;
            u_base_smem = l_base_smem + static_cast<int>(s.l_col.size());
            used += lu;
        }
        rcp_base = -1;
        const size_t rb = static_cast<size_t>(s.dim) * per_slot;
        if (rcp && lu_smem && s.dim > 0) {
            if (used + rb > opt.smem_budget && !vc_slots.empty()) {
                // make room: lane-varying constants are then read from the const table (L1)
                used -= vc_slots.size() * per_slot;
                std::fill(vc_index.begin(), vc_index.end(), -1);
                vc_slots.clear();
                l_base_smem = vc_base;
                u_base_smem = l_base_smem + static_cast<int>(s.l_col.size());
            }
            if (used + rb <= opt.smem_budget) {
                rcp_base = u_base_smem + static_cast<int>(s.u_col.size());
                used += rb;
            }
        }
        smem_bytes = used;
        return true;
    }

    int smem_slots() const {
        return vc_base + static_cast<int>(vc_slots.size()) +
               (l_base_smem >= 0 ? static_cast<int>(s.l_col.size() + s.u_col.size()) : 0) + (rcp_base >= 0 ? s.dim : 0);
    }

    // Refactorization (FactorizeSystem, exec.cpp:175-204; lu_factor, sparse.cpp:79-145)
    // as straight-line code for one lane per thread; lanes whose watch slots
    // are clear skip it (their factors would be recomputed bit-identically).
    std::string emit_refactor() const {
        std::ostringstream o;
        o << "      bool need = false;\n";
        for (int x : s.watch)
            if (x >= 0 && cls[static_cast<size_t>(x)] != kChg) o << "      need = need || (" << R(x) << " != 0.0);\n";
        if (chg_flag) o << "      need = need || (needS[lane] != 0);\n";
        o << "      if (need) {\n";
        const int nnz = static_cast<int>(s.col_idx.size());
        for (int k = 0; k < nnz; ++k) {
            o << "        double G" << k << " = 0.0;";
            for (int q = s.mentry_ptr[static_cast<size_t>(k)]; q < s.mentry_ptr[static_cast<size_t>(k) + 1]; ++q)
                o << " G" << k << " = G" << k << " + " << lit(s.mentry_sign[static_cast<size_t>(q)]) << " * "
                  << R(s.mentry_slot[static_cast<size_t>(q)]) << ";";
            o << " if (live) A[" << static_cast<long long>(s.matrix + k) * W << "] = G" << k << ";\n";
        }
        o << "        double mx = 0.0;\n";
        for (int k = 0; k < nnz; ++k) o << "        { const double x = fabs(G" << k << "); mx = mx < x ? x : mx; }\n";
        // last row touching each scratch column: final scratch contents (sparse.cpp:92-131)
        std::vector<int> last_row(static_cast<size_t>(s.dim), -1);
        for (int i = 0; i < s.dim; ++i) {
            for (int k = s.l_row_ptr[static_cast<size_t>(i)]; k < s.l_row_ptr[static_cast<size_t>(i) + 1]; ++k)
                last_row[static_cast<size_t>(s.l_col[static_cast<size_t>(k)])] = i;
            for (int k = s.u_row_ptr[static_cast<size_t>(i)]; k < s.u_row_ptr[static_cast<size_t>(i) + 1]; ++k)
                last_row[static_cast<size_t>(s.u_col[static_cast<size_t>(k)])] = i;
        }
        for (size_t k = 0; k < s.u_col.size(); ++k) o << "        double u" << k << ";\n";
        for (int i = 0; i < s.dim; ++i) {
            const int lb = s.l_row_ptr[static_cast<size_t>(i)], le = s.l_row_ptr[static_cast<size_t>(i) + 1];
            const int ub = s.u_row_ptr[static_cast<size_t>(i)], ue = s.u_row_ptr[static_cast<size_t>(i) + 1];
            o << "        {\n";
            std::set<int> cols;
            for (int k = lb; k < le; ++k) cols.insert(s.l_col[static_cast<size_t>(k)]);
            for (int k = ub; k < ue; ++k) cols.insert(s.u_col[static_cast<size_t>(k)]);
            for (int c : cols) o << "          double w" << c << " = 0.0;\n";
            for (int k = s.row_ptr[static_cast<size_t>(i)]; k < s.row_ptr[static_cast<size_t>(i) + 1]; ++k)
                o << "          w" << s.col_idx[static_cast<size_t>(k)] << " = G" << k << ";\n";
            for (int k = lb; k < le; ++k) {
                const int col = s.l_col[static_cast<size_t>(k)];
                const int cb = s.u_row_ptr[static_cast<size_t>(col)], ce = s.u_row_ptr[static_cast<size_t>(col) + 1];
                o << "          { const double lik = w" << col << " / u" << cb << "; " << Lw(k, "lik");
                for (int j = cb + 1; j < ce; ++j) {
                    const int c = s.u_col[static_cast<size_t>(j)];
                    o << " w" << c << " = w" << c << " - lik * u" << j << ";";
                }
                o << " }\n";
            }
            for (int k = ub; k < ue; ++k) {
                const int c = s.u_col[static_cast<size_t>(k)];
                o << "          u" << k << " = w" << c << "; " << Uw(k, "u" + std::to_string(k));
                if (k == ub && rcp_base >= 0) o << " S[" << (rcp_base + i) * ls << "] = EMT_RCP(u" << k << ");";
                if (k == ub && lu_shared) o << " SH[" << sh_rcp(i) << "] = EMT_RCP(u" << k << ");";
                o << "\n";
            }
            for (int c : cols)
                if (last_row[static_cast<size_t>(c)] == i)
                    o << "          if (live) A[" << static_cast<long long>(s.scratch + c) * W << "] = w" << c << ";\n";
            o << "          if (!(fabs(u" << ub << ") > " << lit(1e-12) << " * mx)) { srow = " << i << "; goto fact_done; }\n";
            o << "        }\n";
        }
        for (int x : s.watch)
            if (x >= 0 && cls[static_cast<size_t>(x)] != kChg) o << "        " << Wr(x) << " = 0.0;\n";
        if (chg_flag) o << "        needS[lane] = 0;\n";
        o << "      fact_done:;\n";
        o << "      }\n";
        return o.str();
    }
};

struct Sched {
    std::vector<std::vector<std::vector<int>>> phases;  // [phase][warp] -> task ids
};

// List scheduling of one region's DAG onto `G` warps with global barriers,
// simulated in estimated cycles. A task is visible to a warp when all its
// predecessors ran on that warp or finished before the latest barrier; warps
// take the visible ready task with the longest remaining path (critical path
// first). A barrier is inserted when no warp has visible work, or when the
// earliest-idle warp starves while enough work waits behind the barrier.
Sched schedule_region(const std::vector<Task>& tasks, const std::vector<int>& ids,
                      const std::vector<std::vector<int>>& deps, int G, double* makespan, long barrier_cost = 100) {
    const long kBarrier = knob("EMTB200_CG_BARRIER", knob("EMTB200_CG_COSTV2", 1) ? barrier_cost : 200);
    Sched out;
    const size_t n = ids.size();
    if (n == 0) {
        if (makespan) *makespan = 0;
        return out;
    }
    std::map<int, int> local;
    for (size_t i = 0; i < n; ++i) local[ids[i]] = static_cast<int>(i);
    std::vector<std::vector<int>> pred(n), succ(n);
    for (size_t i = 0; i < n; ++i)
        for (int d : deps[static_cast<size_t>(ids[i])]) {
            auto it = local.find(d);
            if (it == local.end()) continue;  // other region: ordered by the region barrier
            pred[i].push_back(it->second);
            succ[static_cast<size_t>(it->second)].push_back(static_cast<int>(i));
        }
    std::vector<long> cost(n), bottom(n, 0);
    for (size_t i = 0; i < n; ++i) cost[i] = std::max(1, tasks[static_cast<size_t>(ids[i])].cost);
    for (size_t k = n; k-- > 0;) {
        long b = 0;
        for (int sx : succ[k]) b = std::max(b, bottom[static_cast<size_t>(sx)]);
        bottom[k] = cost[k] + b;
    }
    std::vector<int> missing(n), warp_of(n, -1), epoch(n, -1);
    for (size_t i = 0; i < n; ++i) missing[i] = static_cast<int>(pred[i].size());
    std::set<std::pair<long, int>> ready;  // (-bottom, i)
    for (size_t i = 0; i < n; ++i)
        if (missing[i] == 0) ready.insert({-bottom[i], static_cast<int>(i)});
    std::vector<long> T(static_cast<size_t>(G), 0);
    std::vector<std::vector<std::pair<int, int>>> plan(static_cast<size_t>(G));
    int nb = 0;
    size_t done = 0;
    auto visible = [&](int i, int w) {
        for (int d : pred[static_cast<size_t>(i)])
            if (warp_of[static_cast<size_t>(d)] != w && epoch[static_cast<size_t>(d)] >= nb) return false;
        return true;
    };
    auto barrier = [&]() {
        const long b = *std::max_element(T.begin(), T.end()) + kBarrier;
        std::fill(T.begin(), T.end(), b);
        ++nb;
    };
    while (done < n) {
        std::vector<int> order(static_cast<size_t>(G));
        for (int w = 0; w < G; ++w) order[static_cast<size_t>(w)] = w;
        std::sort(order.begin(), order.end(), [&](int a, int b) { return T[static_cast<size_t>(a)] < T[static_cast<size_t>(b)]; });
        int pick_w = -1, pick_i = -1;
        bool first_starves = false;
        for (size_t oi = 0; oi < order.size() && pick_w < 0; ++oi) {
            const int w = order[oi];
            for (const auto& r : ready) {
                if (visible(r.second, w)) {
                    pick_w = w;
                    pick_i = r.second;
                    break;
                }
            }
            if (oi == 0 && pick_w < 0) first_starves = true;
        }
        if (pick_w < 0) {
            barrier();
            continue;
        }
        if (first_starves) {
            long waiting = 0;
            for (const auto& r : ready)
                if (!visible(r.second, order[0])) waiting += cost[static_cast<size_t>(r.second)];
            const long spread = T[static_cast<size_t>(order.back())] - T[static_cast<size_t>(order[0])];
            if (waiting >= kBarrier && spread >= kBarrier / 2) {
                barrier();
                continue;
            }
        }
        const size_t i = static_cast<size_t>(pick_i);
        ready.erase({-bottom[i], pick_i});
        T[static_cast<size_t>(pick_w)] += cost[i];
        warp_of[i] = pick_w;
        epoch[i] = nb;
        plan[static_cast<size_t>(pick_w)].push_back({ids[i], nb});
        ++done;
        for (int sx : succ[i])
            if (--missing[static_cast<size_t>(sx)] == 0) ready.insert({-bottom[static_cast<size_t>(sx)], sx});
    }
    out.phases.assign(static_cast<size_t>(nb) + 1, std::vector<std::vector<int>>(static_cast<size_t>(G)));
    for (int w = 0; w < G; ++w)
        for (const auto& pr : plan[static_cast<size_t>(w)])
            out.phases[static_cast<size_t>(pr.second)][static_cast<size_t>(w)].push_back(pr.first);
    while (out.phases.size() > 1) {
        bool empty = true;
        for (const auto& v : out.phases.back()) empty = empty && v.empty();
        if (!empty) break;
        out.phases.pop_back();
    }
    if (makespan) *makespan = static_cast<double>(*std::max_element(T.begin(), T.end()));
    return out;
}

// Kind-major topological re-order of one (phase, warp) list, then split into
// same-kind segments; a segment is "independent" when none of its tasks
// depends on another task of the segment.
struct Segment {
    int kind, first, count, indep;
};

std::vector<Segment> segments_of(const std::vector<int>& list, const std::vector<std::vector<int>>& deps,
                                 std::vector<Task>& tasks, std::vector<int>& ordered) {
    std::set<int> in(list.begin(), list.end());
    std::map<int, int> missing;
    std::map<int, std::vector<int>> succ;
    for (int id : list) {
        int m = 0;
        for (int d : deps[static_cast<size_t>(id)])
            if (in.count(d)) {
                ++m;
                succ[d].push_back(id);
            }
        missing[id] = m;
    }
    std::map<int, int> pos;
    for (size_t i = 0; i < list.size(); ++i) pos[list[i]] = static_cast<int>(i);
    auto key = [&](int id) {
        const Task& t = tasks[static_cast<size_t>(id)];
        return t.kind * 1000000 + static_cast<int>(t.terms.size()) * 1000 + static_cast<int>(t.ck.size());
    };
    std::set<std::pair<std::pair<int, int>, int>> ready;  // ((segment key, pos), id)
    for (int id : list)
        if (missing[id] == 0) ready.insert({{key(id), pos[id]}, id});
    ordered.clear();
    int cur_kind = -1;
    while (!ready.empty()) {
        auto it = ready.begin();
        for (auto jt = ready.begin(); jt != ready.end(); ++jt)
            if (jt->first.first == cur_kind) {  // keep same-kind runs together
                it = jt;
                break;
            }
        const int id = it->second;
        cur_kind = it->first.first;
        ready.erase(it);
        ordered.push_back(id);
        for (int sx : succ[id])
            if (--missing[sx] == 0) ready.insert({{key(sx), pos[sx]}, sx});
    }
    std::vector<Segment> segs;
    for (size_t i = 0; i < ordered.size();) {
        size_t j = i;
        const int kind = tasks[static_cast<size_t>(ordered[i])].kind;
        std::set<int> members;
        bool indep = unrollable(kind);
        const size_t nterm = tasks[static_cast<size_t>(ordered[i])].terms.size();
        const size_t ncst = tasks[static_cast<size_t>(ordered[i])].ck.size();
        while (j < ordered.size() && tasks[static_cast<size_t>(ordered[j])].kind == kind &&
               tasks[static_cast<size_t>(ordered[j])].terms.size() == nterm &&
               tasks[static_cast<size_t>(ordered[j])].ck.size() == ncst) {
            for (int d : deps[static_cast<size_t>(ordered[j])])
                if (members.count(d)) indep = false;
            members.insert(ordered[j]);
            ++j;
        }
        segs.push_back({kind, static_cast<int>(i), static_cast<int>(j - i), indep ? 1 : 0});
        i = j;
    }
    return segs;
}

// ---- device-side code templates --------------------------------------------
// Per kind: operand loads / compute / store, with {I<n>} = integer record field
// n and {C<n>} = constant field n of the task at unroll index @. A segment's
// loop bounds and table bases are compile-time constants inside a warp-uniform
// branch, so records come through the uniform datapath (LDCU) and shared-memory
// accesses become LDS [lane_base + uniform offset].
struct KindCode {
    const char* loads;
    const char* compute;
    const char* store;
};

const KindCode kCode[K_NKINDS] = {
    /*IND*/ {"const double vs@ = LD({I1}) - LD({I0}); const double ip@ = LD({I2}); const double g@ = {C0};",
             "const double h@ = ip@ + g@ * vs@;", "ST({I3}, h@);"},
    /*CAP*/ {"const double vs@ = LD({I1}) - LD({I0}); const double ip@ = LD({I2}); const double g@ = {C0};",
             "const double h@ = -ip@ - g@ * vs@;", "ST({I3}, h@);"},
    /*SRL*/ {"const double vs@ = LD({I1}) - LD({I0}); const double ip@ = LD({I2}); const double g@ = {C0}; const double d@ = {C1};",
             "const double h@ = d@ * ip@ + g@ * vs@;", "ST({I3}, h@);"},
    /*VSRC*/ {"const double g@ = {C0}; const double m@ = {C1}; const double w@ = {C2}; const double p@ = {C3};",
              "const double h@ = g@ * (w@ == 0.0 ? m@ : m@ * emt_libm_cos(w@ * t + p@));", "ST({I0}, h@);"},
    /*ISRC*/ {"const double m@ = {C0}; const double w@ = {C1}; const double p@ = {C2};",
              "const double h@ = w@ == 0.0 ? m@ : m@ * emt_libm_cos(w@ * t + p@);", "ST({I0}, h@);"},
    /*CSRC*/ {"const double k@ = {C0}; const double x@ = LD({I1});", "const double h@ = k@ * x@;", "ST({I0}, h@);"},
    /*SW*/ {nullptr, nullptr, nullptr},
    /*GATHER*/ {nullptr, nullptr, nullptr},
    /*FWD*/ {nullptr, nullptr, nullptr},
    /*BWD*/ {nullptr, nullptr, nullptr},
    /*FINC*/ {"const double vs@ = LD({I3}) - LD({I2}); const double h@ = LD({I1}); const double g@ = {C0};",
              "const double i@ = g@ * vs@ + h@;", "ST({I0}, i@);"},
    /*FINS*/ {"const double vs@ = LD({I3}) - LD({I2}); const double h@ = LD({I1}); const double g@ = LD({I4});",
              "const double i@ = g@ * vs@ + h@;", "ST({I0}, i@);"},
    /*GAIN*/ {"const double x@ = SGN(LD({I1}), {I2}); const double k@ = {C0};", "const double y@ = k@ * x@;",
              "ST({I0}, y@);"},
    /*SUM*/ {nullptr, nullptr, nullptr},
    /*INTEG*/ {"const double u@ = SGN(LD({I1}), {I4}); const double s0@ = LD({I2}); const double s1@ = LD({I3}); const double c0@ = {C0};",
               "const double y@ = s0@ + c0@ * (u@ + s1@);", "ST({I2}, y@); ST({I3}, u@); ST({I0}, y@);"},
    /*LAG*/ {"const double u@ = SGN(LD({I1}), {I4}); const double s0@ = LD({I2}); const double s1@ = LD({I3}); const double c0@ = {C0}; const double c1@ = {C1};",
             "const double y@ = c0@ * s0@ + c1@ * (u@ + s1@);", "ST({I2}, y@); ST({I3}, u@); ST({I0}, y@);"},
    /*PI*/ {"const double u@ = SGN(LD({I1}), {I4}); const double s0@ = LD({I2}); const double s1@ = LD({I3}); const double kp@ = {C0}; const double ki@ = {C1};",
            "const double y@ = s0@ + ki@ * (u@ + s1@); const double o@ = kp@ * u@ + y@;",
            "ST({I2}, y@); ST({I3}, u@); ST({I0}, o@);"},
    /*LIM*/ {"const double u@ = SGN(LD({I1}), {I2}); const double lo@ = {C0}; const double hi@ = {C1};",
             "const double y@ = u@ < lo@ ? lo@ : (u@ > hi@ ? hi@ : u@);", "ST({I0}, y@);"},
    /*CMP*/ {"const double a@ = SGN(LD({I1}), {I3}); const double b@ = SGN(LD({I2}), {I4});",
             "const double y@ = a@ >= b@ ? 1.0 : 0.0;", "ST({I0}, y@);"},
    /*CONST*/ {"const double y@ = {C0};", "", "ST({I0}, y@);"},
    /*DELAY*/ {"const double y@ = SGN(LD({I1}), {I2});", "", "ST({I0}, y@);"},
    /*REC*/ {"const double y@ = LD({I1});", "",
             "if (live) a.waves[((size_t)(a.row0 + it) * NCH + {I0}) * W_ + gl] = y@;"},
    /*LATCH*/ {"const double y@ = LD({I0});", "", "ST({I1}, y@);"},
    /*BERG*/ {"const double vs@ = LD({I1}) - LD({I0}); const double hp@ = LD({I2}); const double y2@ = {C0}; "
             "const double c1@ = {C1}; const double c0@ = {C2}; const int K@ = (int)({C3}); "
             "const long long pl@ = (long long)({C4}); const long long pr@ = (long long)({C5}) - a.ring_lo;",
             "const double be@ = y2@ * vs@ + hp@; int q1@ = (step + 1 - K@) % {I4}; if (q1@ < 0) q1@ += {I4}; "
             "const int q0@ = q1@ == 0 ? {I4} - 1 : q1@ - 1; "
             "const double b1@ = a.sys_scope ? __ldcv(a.ring + pl@ * a.ring_cols + pr@ + q1@) : __ldcg(a.ring + pl@ * a.ring_cols + pr@ + q1@); "
             "const double b0@ = a.sys_scope ? __ldcv(a.ring + pl@ * a.ring_cols + pr@ + q0@) : __ldcg(a.ring + pl@ * a.ring_cols + pr@ + q0@); "
             "const double h@ = -(c1@ * b1@ + c0@ * b0@);",
             "ST({I2}, h@); if (live) { const int w@ = step % {I4}; A[(size_t)({I3} + w@) * W_] = be@; "
             "a.ring[(LB_ + gl) * a.ring_cols + ({I3} - a.ring_lo) + w@] = be@; }"},
    // sources whose m*cos(w t + p) was computed during the previous pass (K_SRCPRE)
    /*VSRCP*/ {"const double g@ = {C0}; const double v@ = LD({I1});", "const double h@ = g@ * v@;", "ST({I0}, h@);"},
    /*ISRCP*/ {"const double v@ = LD({I1});", "", "ST({I0}, v@);"},
    /*SRCPRE*/ {"const double m@ = {C0}; const double w@ = {C1}; const double p@ = {C2};",
               "const double v@ = w@ == 0.0 ? m@ : m@ * emt_libm_cos(w@ * tn + p@);", "ST({I0}, v@);"},
    // sources read from the launch's value table (emt_src_kernel computes m*cos(w t + p))
    /*VSRCT*/ {"const double g@ = {C0}; const double v@ = SRCV_({I1});", "const double h@ = g@ * v@;", "ST({I0}, h@);"},
    /*ISRCT*/ {"const double v@ = SRCV_({I1});", "", "ST({I0}, v@);"},
};

// Per-segment record layout. Constant field modes: 0 = lane-invariant value in
// the double table, 1 = lane-varying, slot index (value from the per-lane
// const table in HBM), 2 = lane-varying, cached in shared memory (byte offset).
// Term operands (gather / sum / solve rows) are stored inline: a segment only
// holds tasks with the same term count, so term loops fully unroll.
struct SegLayout {
    int nI = 0, nC = 0, TC = 0;
    std::vector<int> cmode;
    int SI = 0, SD = 0;
    std::vector<int> cpos;  // per const field: position in the int (modes 1, 2) or double (mode 0) record
};

std::string cfield(const SegLayout& L, int n, const std::string& bi, const std::string& bd) {
    const int m = L.cmode[static_cast<size_t>(n)];
    const std::string pos = std::to_string(L.cpos[static_cast<size_t>(n)]);
    if (m == 0) return "kRd[" + bd + " + " + pos + "]";
    if (m == 2) return "LD(kRi[" + bi + " + " + pos + "])";
    return "__ldg(C + (size_t)kRi[" + bi + " + " + pos + "] * W_)";
}

std::string expand(const char* tpl, int j, const SegLayout& L, const std::string& bi, const std::string& bd) {
    std::string out;
    for (const char* c = tpl; c && *c; ++c) {
        if (*c == '@') {
            out += std::to_string(j);
        } else if (*c == '{' && (c[1] == 'I' || c[1] == 'C')) {
            const char kind = c[1];
            const char* e = std::strchr(c, '}');
            const int n = std::atoi(std::string(c + 2, e).c_str());
            if (kind == 'I') out += "kRi[" + bi + " + " + std::to_string(n) + "]";
            else out += cfield(L, n, bi, bd);
            c = e;
        } else {
            out += *c;
        }
    }
    return out;
}

// Loads / compute / store text of one task at unroll index j (record base `bi`,
// `bd`) for every kind except the switch.
void task_parts(int kind, int j, const SegLayout& L, const std::string& bi, const std::string& bd, std::string& ld,
                std::string& cp, std::string& st) {
    const std::string J = std::to_string(j);
    auto Tx = [&](int t) { return "kRi[" + bi + " + " + std::to_string(L.nI + 2 * t) + "]"; };
    auto Ty = [&](int t) { return "kRi[" + bi + " + " + std::to_string(L.nI + 2 * t + 1) + "]"; };
    auto I = [&](int n) { return "kRi[" + bi + " + " + std::to_string(n) + "]"; };
    if (kCode[kind].loads != nullptr) {
        ld = expand(kCode[kind].loads, j, L, bi, bd);
        cp = expand(kCode[kind].compute, j, L, bi, bd);
        st = expand(kCode[kind].store, j, L, bi, bd);
        return;
    }
    std::ostringstream l, c;
    if (kind == K_GATHER || kind == K_SUM) {  // sequential accumulation from 0.0 (exec.cpp:207-214, 245-253)
        for (int t = 0; t < L.TC; ++t) l << "const double a" << J << "_" << t << " = SGN(LD(" << Tx(t) << "), " << Ty(t) << "); ";
        c << "double acc" << J << " = 0.0; ";
        for (int t = 0; t < L.TC; ++t) c << "acc" << J << " = acc" << J << " + a" << J << "_" << t << "; ";
        st = "ST(" + I(0) + ", acc" + J + ");";
    } else {  // FWD / BWD rows (sparse.cpp:152-171) + divergence (exec.cpp:229-237)
        l << "double x" << J << " = LD(" << I(0) << "); ";
        for (int t = 0; t < L.TC; ++t)
            l << "const double p" << J << "_" << t << " = LU(" << Tx(t) << ") * LD(" << Ty(t) << "); ";
        for (int t = 0; t < L.TC; ++t) c << "x" << J << " = x" << J << " - p" << J << "_" << t << "; ";
        if (kind == K_BWD)
            c << "x" << J << " = x" << J << " / LU(" << I(1) << "); if (!(fabs(x" << J << ") <= a.div_limit) && " << I(2)
              << " < bad) bad = " << I(2) << "; ";
        st = "ST(" + I(0) + ", x" + J + ");";
    }
    ld = l.str();
    cp = c.str();
}

// Straight-line form of one task: every shared-memory offset and constant
// index is a literal, so the compiler may interleave independent tasks freely
// (no aliasing unknowns) — the latency-optimal form when the step fits the
// instruction cache.
struct LitCtx {
    std::function<std::string(int)> cst;  // const slot -> expression
    int sw_bit = -1;                       // >= 0: switch task writes its change flag to bit sw_bit of swbits
    bool chg_flag = false;                 // switch "changed" slots collapsed into needS
    bool dok = true;                       // divergence as an AND-ed predicate (cold index scan)
    bool sw_slim = false;                  // switch hot path only tests for a change; stores go to the cold path
    bool fused_pass = false;               // emit fused Norton tasks in their fused form (passes after the first)
    std::function<int(int)> lit_init;      // switch initial state: 0/1 when lane-invariant, -1 otherwise
    int divguard = 1;                      // reciprocal-multiply division: 1 = detect 0 < |q| < 2^-900 (stop the
                                           // launch, EMT_INEXACT_DIVISION), 2 = branch to IEEE x/u, 0 = none (dev)
    bool zterm = false;                    // drop zero-slot terms from sums
    int task_id = -1;                      // the task's index (per-task registers)
    int sh_rcp0 = 0;                       // SH index of the first pivot reciprocal (shared factors)
};

std::string expand_lit(const char* tpl, const Task& t, const LitCtx& c, const std::string& sfx = "_") {
    std::string out;
    for (const char* p = tpl; p && *p; ++p) {
        if (*p == '@') {
            out += sfx;
        } else if (*p == '{' && (p[1] == 'I' || p[1] == 'C')) {
            const char kind = p[1];
            const char* e = std::strchr(p, '}');
            const int n = std::atoi(std::string(p + 2, e).c_str());
            out += kind == 'I' ? std::to_string(t.f[static_cast<size_t>(n)]) : c.cst(t.ck[static_cast<size_t>(n)]);
            p = e;
        } else {
            out += *p;
        }
    }
    return out;
}

std::string task_literal(const Task& t, const LitCtx& c) {
    std::ostringstream o;
    o << "{ ";
    if (t.fused && c.fused_pass) {
        // i_prev = g (vb - va) + h as the finalize computed it last pass (exec.cpp:220-228)
        const std::string vb = std::to_string(t.f[1]), va = std::to_string(t.f[0]), h = std::to_string(t.f[3]);
        o << "const double vs = LD(" << vb << ") - LD(" << va << "); const double hp = LD(" << h << "); const double g = "
          << c.cst(t.ck[0]) << "; const double ip = g * vs + hp; ";
        if (t.kind == K_IND) o << "const double hn = ip + g * vs; ";
        else if (t.kind == K_CAP) o << "const double hn = -ip - g * vs; ";
        else o << "const double d = " << c.cst(t.ck[1]) << "; const double hn = d * ip + g * vs; ";
        o << "ST(" << h << ", hn);";
    } else if (t.out_alias && (t.kind == K_INTEG || t.kind == K_LAG)) {
        o << expand_lit(kCode[t.kind].loads, t, c) << " " << expand_lit(kCode[t.kind].compute, t, c) << " "
          << expand_lit("ST({I2}, y@); ST({I3}, u@);", t, c);
    } else if (kCode[t.kind].loads != nullptr) {
        o << expand_lit(kCode[t.kind].loads, t, c) << " " << expand_lit(kCode[t.kind].compute, t, c) << " "
          << expand_lit(kCode[t.kind].store, t, c);
    } else if (t.kind == K_GATHER || t.kind == K_SUM) {
        // terms read from the zero slot (resistor h, ground) are dropped: acc starts at +0.0
        // and an IEEE sum is -0 only when both addends are -0, so acc is never -0 and
        // acc + (+-0) == acc bit for bit
        o << "double acc = 0.0; ";
        for (const auto& tm : t.terms)
            if (tm.first != 0 || !c.zterm) o << "acc = acc + " << (tm.second ? "-" : "") << "LD(" << tm.first << "); ";
        o << "ST(" << t.f[0] << ", acc);";
    } else if (t.kind == K_FWD || t.kind == K_BWD) {
        auto lu = [](int x) { return x < 0 ? "SH[" + std::to_string(-x - 1) + "]" : "LU(" + std::to_string(x) + ")"; };
        o << "double x = LD(" << t.f[0] << "); ";
        for (const auto& tm : t.terms) o << "x = x - " << lu(tm.first) << " * LD(" << tm.second << "); ";
        if (t.kind == K_BWD)
            if (c.dok)
                if (t.f.size() > 3 && (t.f[3] >= 0 || t.f[3] <= -2))
                    o << "{ const double r_ = " << (t.f[3] >= 0 ? "LD(" + std::to_string(t.f[3]) + ")" : "SH[" + std::to_string(c.sh_rcp0 - t.f[3] - 2) + "]")
                      << "; const double d_ = " << lu(t.f[1])
                      << "; const double q_ = x * r_; double m_ = __fma_rn(__fma_rn(-d_, q_, x), r_, q_); "
                      << (c.divguard == 2 ? "if (__builtin_expect(!(fabs(q_) >= 0x1p-900), 0)) m_ = emt_div_ieee(x, d_); " : "")
                      << "x = m_; "
                      << (c.divguard == 1 ? "dok = dok & (fabs(x) <= dlim) & (fabs(q_) >= 0x1p-900); } "
                                 : c.divguard == 3 ? "dok = dok & (fabs(x) <= dlim) & !((fabs(q_) < 0x1p-900) & (q_ != 0.0)); } "
                                                   : "dok = dok & (fabs(x) <= dlim); } ");
                else
                    o << "x = x / " << lu(t.f[1]) << "; dok = dok & (fabs(x) <= dlim); ";
            else
                o << "x = x / " << lu(t.f[1]) << "; if (!(fabs(x) <= a.div_limit) && " << t.f[2] << " < bad) bad = " << t.f[2] << "; ";
        o << "ST(" << t.f[0] << ", x);";
    } else if (t.kind == K_SW && c.sw_bit >= 0 && c.sw_slim && t.ck.size() == 4 && c.lit_init && c.lit_init(t.ck[2]) >= 0) {
        // one toggle time: changed <=> (init XOR t >= t0) != state, init folded in
        o << "{ const bool f_ = t >= " << c.cst(t.ck[3]) << "; const bool s_ = LD(" << t.f[0] << ") != 0.0; if ("
          << (c.lit_init(t.ck[2]) ? "!f_" : "f_") << " != s_) swbits |= 1ull << " << c.sw_bit << "; }";
    } else if (t.kind == K_SW && c.sw_bit >= 0 && c.sw_slim) {
        o << "int now = " << c.cst(t.ck[2]) << " != 0.0 ? 1 : 0; ";
        for (size_t j = 3; j < t.ck.size(); ++j) o << "if (t >= " << c.cst(t.ck[j]) << ") now ^= 1; ";
        o << "if ((double)now != LD(" << t.f[0] << ")) swbits |= 1ull << " << c.sw_bit << ";";
    } else if (t.kind == K_SW && c.sw_bit >= 0) {
        // change flag into the warp's bit mask; event logging, the refactor flag
        // and wflag happen once per pass in the (rare) non-zero-mask path
        o << "int now = " << c.cst(t.ck[2]) << " != 0.0 ? 1 : 0; ";
        for (size_t j = 3; j < t.ck.size(); ++j) o << "if (t >= " << c.cst(t.ck[j]) << ") now ^= 1; ";
        o << "const double chg = (double)now != LD(" << t.f[0] << ") ? 1.0 : 0.0; "
          << (c.chg_flag ? std::string() : "ST(" + std::to_string(t.f[1]) + ", chg); ") << "ST(" << t.f[0]
          << ", (double)now); ST(" << t.f[2] << ", now != 0 ? " << c.cst(t.ck[0]) << " : " << c.cst(t.ck[1])
          << "); swbits |= (chg != 0.0 ? 1ull : 0ull) << " << c.sw_bit << ";";
    } else if (t.kind == K_SW) {
        o << "int now = " << c.cst(t.ck[2]) << " != 0.0 ? 1 : 0; ";
        for (size_t j = 3; j < t.ck.size(); ++j) o << "if (t >= " << c.cst(t.ck[j]) << ") now ^= 1; ";
        o << "const double chg = (double)now != LD(" << t.f[0] << ") ? 1.0 : 0.0; SETCHG(" << t.f[1] << ", chg); ST("
          << t.f[0] << ", (double)now); ST(" << t.f[2] << ", now != 0 ? " << c.cst(t.ck[0]) << " : " << c.cst(t.ck[1])
          << "); if (chg != 0.0) { wflag = 1; if (live && a.events) { const int e = atomicAdd(a.n_events, 1); "
          << "if (e < a.max_events) { a.events[3*e] = step; a.events[3*e+1] = gl; a.events[3*e+2] = " << t.f[3] << "; } } }";
    }
    o << " }";
    return o.str();
}

// One segment: N tasks of `kind` at table bases (bi0, bd0). Independent
// segments issue the operand loads of up to four tasks before any compute or
// store (the compiler cannot hoist shared-memory loads above stores itself).
std::string segment_code(int kind, int N, bool indep, int bi0, int bd0, const SegLayout& L, const char* ind) {
    std::ostringstream o;
    const std::string SI = std::to_string(L.SI), SD = std::to_string(L.SD);
    o << ind << "{  // " << kKindName[kind] << " x" << N << (L.TC ? " terms " + std::to_string(L.TC) : std::string()) << "\n";
    if (kind != K_SW) {
        const int U = indep ? knob("EMTB200_CG_UNROLL", 1) : 1;
        const int q0 = N - N % U;
        auto block = [&](const std::string& qexpr, int count, const char* in2) {
            std::string ld[4], cp[4], st[4];
            for (int j = 0; j < count; ++j) {
                const std::string bi = "bi" + std::to_string(j), bd = "bd" + std::to_string(j);
                o << in2 << "const int " << bi << " = " << bi0 << " + (" << qexpr << " + " << j << ") * " << SI << "; const int "
                  << bd << " = " << bd0 << " + (" << qexpr << " + " << j << ") * " << SD << "; (void)" << bd << ";\n";
                task_parts(kind, j, L, bi, bd, ld[j], cp[j], st[j]);
            }
            for (int j = 0; j < count; ++j) o << in2 << ld[j] << "\n";
            for (int j = 0; j < count; ++j) o << in2 << cp[j] << "\n";
            for (int j = 0; j < count; ++j) o << in2 << st[j] << "\n";
        };
        const std::string in2 = std::string(ind) + "    ";
        if (q0 > 0) {
            if (q0 == U) {
                o << ind << "  {\n";
                block("0", U, in2.c_str());
                o << ind << "  }\n";
            } else {
                o << ind << "  #pragma unroll 1\n" << ind << "  for (int q = 0; q < " << q0 << "; q += " << U << ") {\n";
                block("q", U, in2.c_str());
                o << ind << "  }\n";
            }
        }
        if (q0 < N) {
            o << ind << "  {\n";
            block(std::to_string(q0), N - q0, in2.c_str());
            o << ind << "  }\n";
        }
    } else {  // exec.cpp:151-165; consts [g_on, g_off, initial, t0, ...]
        o << ind << "  #pragma unroll 1\n"
          << ind << "  for (int q = 0; q < " << N << "; ++q) {\n"
          << ind << "    const int bi = " << bi0 << " + q * " << SI << "; const int bd = " << bd0 << " + q * " << SD
          << "; (void)bd;\n";
        auto I = [&](int n) { return "kRi[bi + " + std::to_string(n) + "]"; };
        o << ind << "    int now = " << cfield(L, 2, "bi", "bd") << " != 0.0 ? 1 : 0;\n";
        for (int c = 3; c < L.nC; ++c) o << ind << "    if (t >= " << cfield(L, c, "bi", "bd") << ") now ^= 1;\n";
        o << ind << "    const double chg = (double)now != LD(" << I(0) << ") ? 1.0 : 0.0;\n"
          << ind << "    SETCHG(" << I(1) << ", chg); ST(" << I(0) << ", (double)now); ST(" << I(2) << ", now != 0 ? "
          << cfield(L, 0, "bi", "bd") << " : " << cfield(L, 1, "bi", "bd") << ");\n"
          << ind << "    if (chg != 0.0) { wflag = 1; if (live && a.events) { const int e = atomicAdd(a.n_events, 1);"
          << " if (e < a.max_events) { a.events[3*e] = step; a.events[3*e+1] = gl; a.events[3*e+2] = " << I(3) << "; } } }\n"
          << ind << "  }\n";
    }
    o << ind << "}\n";
    return o.str();
}


// Task dependencies from the sequential process order (RAW, WAR, WAW), per region.
std::vector<std::vector<int>> task_deps(const std::vector<Task>& tasks) {
    const size_t nt = tasks.size();
    std::vector<std::vector<int>> deps(nt);
    std::map<int, int> last_writer;
    std::map<int, std::vector<int>> readers;
    int cur_region = 0;
    for (size_t i = 0; i < nt; ++i) {
        const Task& t = tasks[i];
        if (t.region != cur_region) {
            last_writer.clear();
            readers.clear();
            cur_region = t.region;
        }
        std::set<int> d;
        for (int r : t.reads) {
            auto it = last_writer.find(r);
            if (it != last_writer.end()) d.insert(it->second);
        }
        for (int w : t.writes) {
            auto it = last_writer.find(w);
            if (it != last_writer.end()) d.insert(it->second);
            for (int rd : readers[w]) d.insert(rd);
        }
        d.erase(static_cast<int>(i));
        deps[i].assign(d.begin(), d.end());
        for (int r : t.reads) readers[r].push_back(static_cast<int>(i));
        for (int w : t.writes) {
            last_writer[w] = static_cast<int>(i);
            readers[w].clear();
        }
    }
    return deps;
}

}  // namespace

// Straight-line launch prologue/epilogue copies: per warp, items q = warp (mod G) in
// groups whose loads issue back to back (a loop over an index table serialises a table
// load and the dependent arena load per slot: ~35 us per launch on C3).
static std::string warp_copies(const std::vector<std::pair<std::string, std::string>>& items, int G,
                               const std::string& ind, int group = 16, bool solo = false) {
    if (items.empty()) return std::string();
    std::ostringstream o;
    o << ind << "switch (warp) {\n";
    for (int w = 0; w < G; ++w) {
        std::vector<size_t> mine;
        for (size_t q = static_cast<size_t>(w); q < items.size(); q += static_cast<size_t>(G)) mine.push_back(q);
        if (mine.empty()) continue;
        o << ind << "case " << w << ": {\n";
        if (solo) o << ind << "  if (lane == 0)\n";  // one-lane mode: the shadows stay off shared memory
        if (solo) o << ind << "  {\n";
        for (size_t g0 = 0; g0 < mine.size(); g0 += static_cast<size_t>(group)) {
            const size_t g1 = std::min(mine.size(), g0 + static_cast<size_t>(group));
            o << ind << "  { ";
            for (size_t j = g0; j < g1; ++j) o << "const double t" << j - g0 << " = " << items[mine[j]].second << "; ";
            for (size_t j = g0; j < g1; ++j) o << items[mine[j]].first << " = t" << j - g0 << "; ";
            o << "}\n";
        }
        if (solo) o << ind << "  }\n";
        o << ind << "} break;\n";
    }
    o << ind << "}\n";
    return o.str();
}

bool generate_kernel(const Schedule& s, const std::vector<double>& ctab, int lanes, const CodegenOptions& opt,
                     GeneratedKernel& out, Failure& fail) {
    Gen g(s, ctab, lanes, opt);
    // scenario lanes per CTA: 32 = one per thread; 16 / 8 (experiment, EMTB200_CG_LPC) leave
    // the other threads of each warp shadowing lane 0 (same loads and stores, same values)
    // to shrink shared-memory traffic per instruction and spread the batch over more SMs —
    // bit-exact, but measured slower (C3 2.81 -> 3.42 / 4.92 ms per 1000 passes)
    // a single scenario (C2) runs with one lane per CTA in "solo" form (below): only thread 0
    // of each warp executes the step, so every shared-memory access moves one word
    int LPC = opt.lanes_per_cta > 0 ? opt.lanes_per_cta : knob("EMTB200_CG_LPC", lanes == 1 ? 1 : 32);
    if (LPC != 1 && LPC != 2 && LPC != 4 && LPC != 8 && LPC != 16) LPC = 32;
    g.ls = LPC;
    g.unit = LPC * 8;
    // one lane per CTA: only thread 0 of each warp touches shared memory (the other
    // threads only take part in the barriers), so there is no shared address two threads
    // read and write; every access is a single-thread one (C2)
    const bool solo = LPC == 1 && knob("EMTB200_CG_SOLO", 1) != 0 && knob("EMTB200_CG_SLCOPY", 1) != 0 &&
                      knob("EMTB200_CG_WARPMAJOR", 1) != 0 && knob("EMTB200_CG_STRAIGHT", 1) != 0 && opt.mode != 2;
    const int srcl1 = knob("EMTB200_CG_SRCL1", solo ? 0 : 4);  // passes ahead the source row is prefetched into L1
    g.presrc = knob("EMTB200_CG_PRESRC", 0) != 0;
    g.srctab = !g.presrc && knob("EMTB200_CG_SRCTAB", 1) != 0;
    g.rcp = knob("EMTB200_CG_RCP", 1) != 0 && opt.mode != 2 && knob("EMTB200_CG_STRAIGHT", 1) != 0;
    g.fusefin = knob("EMTB200_CG_FUSEFIN", 1) != 0 && opt.mode != 2 && knob("EMTB200_CG_STRAIGHT", 1) != 0 &&
                knob("EMTB200_CG_WARPMAJOR", 1) != 0;  // measured 3% slower: moves cos, does not remove it
    g.classify();
    std::vector<double> ginv;
    if (opt.tensor_solve && LPC == 32 && opt.mode != 2 && knob("EMTB200_CG_STRAIGHT", 1) != 0 && g.shared_g() && g.g_inverse(ginv)) {
        g.dmma = true;
        g.opt.lu_in_smem = false;  // the sweeps are gone; L/U stay in HBM for refactor + state
    }
    const int MT = (s.dim + 7) / 8, KT = (s.dim + 3) / 4;  // DMMA m8n8k4 tiles of G^-1
    if (!g.dmma && opt.mode != 2 && knob("EMTB200_CG_STRAIGHT", 1) != 0 && knob("EMTB200_CG_LOOPMIN", 0) == 0 &&
        knob("EMTB200_CG_SHLU", 1) != 0)
        g.lu_shared = g.factor_shared();
    const size_t ginv_bytes = g.dmma ? static_cast<size_t>(MT) * 8 * KT * 4 * sizeof(double) : 0;
    g.opt.smem_budget = opt.smem_budget > ginv_bytes ? opt.smem_budget - ginv_bytes : 0;
    int facts = 0;
    g.emit_all(facts);  // pass 1: slot sets
    if (facts != 1) {
        fail = {13, "", "schedule must hold exactly one FactorizeSystem process"};
        return false;
    }
    if (knob("EMTB200_CG_ALIAS", 1) && opt.mode != 2 && knob("EMTB200_CG_STRAIGHT", 1) != 0) {
        // output == state0 aliasing: only when the block is the slot's sole writer and no
        // task reads the output before the block runs in a pass (so the initial value of
        // the output slot is never observed); channels / latches read it at pass end
        std::map<int, int> cand, writer_count, first_writer;
        for (size_t i = 0; i < g.tasks.size(); ++i) {
            for (int w : g.tasks[i].writes) {
                writer_count[w] += 1;
                if (!first_writer.count(w)) first_writer[w] = static_cast<int>(i);
            }
        }
        for (const Proc& p : s.procs)
            if ((p.code == kCtlIntegrator || p.code == kCtlFirstOrderLag) && p.out >= 0 && p.state >= 0)
                cand[p.out] = p.state;
        for (size_t i = 0; i < g.tasks.size(); ++i)
            for (int r : g.tasks[i].reads) {
                auto it = cand.find(r);
                if (it != cand.end() && (!first_writer.count(r) || static_cast<int>(i) <= first_writer[r])) cand.erase(it);
            }
        std::set<int> forbidden(s.watch.begin(), s.watch.end());
        forbidden.insert(s.mentry_slot.begin(), s.mentry_slot.end());
        for (auto it = cand.begin(); it != cand.end();) {
            if (writer_count[it->first] != 1 || forbidden.count(it->first)) it = cand.erase(it);
            else ++it;
        }
        if (!cand.empty()) {
            g.alias_of = cand;
            g.classify();
            g.emit_all(facts);
        }
    }
    bool lu_smem = false;
    size_t smem = 0;
    if (!g.assign_hot(lu_smem, smem)) {
        fail = {13, "", "arena hot set exceeds the shared-memory budget"};
        return false;
    }
    if (g.fusefin && !g.fused.empty() && !lu_smem && !g.dmma && !g.lu_shared) {
        // measured: with the factors in HBM (C5 exact path) the fused form schedules worse
        g.fusefin = false;
        g.classify();
        g.emit_all(facts);
        if (!g.assign_hot(lu_smem, smem)) {
            fail = {13, "", "arena hot set exceeds the shared-memory budget"};
            return false;
        }
    }
    g.emit_all(facts);  // pass 2: records with shared-memory offsets

    if (knob("EMTB200_CG_COSTV2", 1)) {
        // cost model in issued instructions (the pass is issue/fetch bound)
        for (Task& t : g.tasks) {
            const int nt_ = static_cast<int>(t.terms.size());
            int c = 8;
            switch (t.kind) {
                case K_IND: case K_CAP: case K_SRL: c = t.fused ? 12 : 10; break;
                case K_VSRCT: c = 5; break;
                case K_ISRCT: c = 4; break;
                case K_VSRC: case K_ISRC: c = t.cost > 20 ? 60 : 4; break;
                case K_SW: c = 8; break;
                case K_GATHER: case K_SUM: c = 3 + 2 * nt_; break;
                case K_FWD: c = 3 + 4 * nt_; break;
                case K_BWD: c = (t.f.size() > 3 && t.f[3] >= 0 ? 10 : 20) + 4 * nt_; break;
                case K_FINC: c = 7; break;
                case K_FINS: c = 8; break;
                case K_REC: c = 3; break;
                case K_LATCH: c = 2; break;
                case K_BERG: c = knob("EMTB200_CG_BERGCOST", 150); break;  // + two L2 loads of peer histories (25..1000 swept: 150 best, C4 -2%)
                case K_SRCPRE: c = 60; break;
                default: c = 8; break;
            }
            t.cost = c;
        }
    }
    // Dependencies from the sequential order (RAW, WAR, WAW), per region.
    const size_t nt = g.tasks.size();
    std::vector<std::vector<int>> deps(nt);
    {
        std::map<int, int> last_writer;
        std::map<int, std::vector<int>> readers;
        int cur_region = 0;
        for (size_t i = 0; i < nt; ++i) {
            const Task& t = g.tasks[i];
            if (t.region != cur_region) {
                last_writer.clear();
                readers.clear();
                cur_region = t.region;
            }
            std::set<int> d;
            for (int r : t.reads) {
                auto it = last_writer.find(r);
                if (it != last_writer.end()) d.insert(it->second);
            }
            for (int w : t.writes) {
                auto it = last_writer.find(w);
                if (it != last_writer.end()) d.insert(it->second);
                for (int rd : readers[w]) d.insert(rd);
            }
            d.erase(static_cast<int>(i));
            deps[i].assign(d.begin(), d.end());
            for (int r : t.reads) readers[r].push_back(static_cast<int>(i));
            for (int w : t.writes) {
                last_writer[w] = static_cast<int>(i);
                readers[w].clear();
            }
        }
    }
    std::vector<int> ids_a, ids_b, ids_c, fillers;
    for (size_t i = 0; i < nt; ++i) {
        if (g.tasks[i].kind == K_SRCPRE) {  // dependency-free: placed into idle warp time afterwards
            fillers.push_back(static_cast<int>(i));
            continue;
        }
        (g.tasks[i].region == 0 ? ids_a : g.tasks[i].region == 1 ? ids_b : ids_c).push_back(static_cast<int>(i));
    }
    // the shared-factor kernel (C5) runs its chain-bound pass best on 6 warps
    // (5.86 vs 5.99 ms at 8, 4 and 12 worse; profiles/ab/warps_r2.log)
    const int G = std::max(1, std::min(opt.auto_warps && g.lu_shared && !g.dmma ? 6 : opt.warps, 32));
    double span_a = 0, span_b = 0;
    // barrier cost in the list scheduler's model (cycles): fewer, fuller phases pay off
    // up to ~250 with one warp dispatch per pass (C3 -1.9%, C4 -0.4%, C2 -0.5% against
    // 100 / 400 for the solo form; 60, 150, 350, 500, 700 measured worse or mixed,
    // profiles/ab/barrier_r2.log); the shared-factor kernel keeps 100 (250: C5 +3.7%)
    const long bar_cost = g.lu_shared ? 100 : 250;
    Sched sa = schedule_region(g.tasks, ids_a, deps, G, &span_a, bar_cost);
    if (sa.phases.size() == 1 && knob("EMTB200_CG_AFFINITY", 1) != 0) {
        // region A is one phase of independent tasks: regroup them so that tasks reading
        // the same node voltages share a warp (the compiler then loads each voltage once
        // per warp) — order by the lowest node slot read, cut into G chunks of equal cost
        std::vector<int> all;
        for (const auto& wl : sa.phases[0]) all.insert(all.end(), wl.begin(), wl.end());
        // (not with line ends: their peer-history loads want the scheduler's spread,
        // measured C4 3.22 -> 3.41 us when regrouped; C3 2.70 -> 2.63 ms, C2 2.18 -> 2.12 us)
        bool indep = true;
        for (int id : all) indep = indep && g.tasks[static_cast<size_t>(id)].kind != K_BERG;
        std::set<int> in_a(all.begin(), all.end());
        for (int id : all)
            for (int d : deps[static_cast<size_t>(id)]) indep = indep && !in_a.count(d);
        if (indep && !all.empty()) {
            // sort key: lowest node read (highest / both measured within 0.3% on C3)
            auto key = [&](int id) {
                long long lo = 1 << 30;
                for (int r : g.tasks[static_cast<size_t>(id)].reads)
                    if (r >= s.v_base && r < s.v_base + s.nodes) lo = std::min<long long>(lo, r - s.v_base);
                return lo;
            };
            std::stable_sort(all.begin(), all.end(), [&](int a, int b) { return key(a) < key(b); });
            long long total = 0;
            for (int id : all) total += g.tasks[static_cast<size_t>(id)].cost;
            std::vector<std::vector<int>> parts(static_cast<size_t>(G));
            {  // sorted cut (a greedy node-sharing assignment measured worse: C3 2.54 -> 2.59 ms)
                long long acc = 0;
                for (int id : all) {
                    const int w = static_cast<int>(std::min<long long>(G - 1, acc * G / std::max<long long>(1, total)));
                    parts[static_cast<size_t>(w)].push_back(id);
                    acc += g.tasks[static_cast<size_t>(id)].cost;
                }
            }
            sa.phases[0] = parts;
        }
    }
    Sched sb = schedule_region(g.tasks, ids_b, deps, G, &span_b, bar_cost);
    double span_c = 0;
    Sched sc3 = schedule_region(g.tasks, ids_c, deps, G, &span_c, bar_cost);
    {
        // filler tasks go where a warp idles longest before a barrier of the last region
        Sched& host = g.dmma ? sc3 : sb;
        if (host.phases.empty()) host.phases.assign(1, std::vector<std::vector<int>>(static_cast<size_t>(G)));
        std::vector<std::vector<long>> load(host.phases.size(), std::vector<long>(static_cast<size_t>(G), 0));
        std::vector<long> pmax(host.phases.size(), 0);
        for (size_t p = 0; p < host.phases.size(); ++p)
            for (int w = 0; w < G; ++w) {
                for (int id : host.phases[p][static_cast<size_t>(w)]) load[p][static_cast<size_t>(w)] += g.tasks[static_cast<size_t>(id)].cost;
                pmax[p] = std::max(pmax[p], load[p][static_cast<size_t>(w)]);
            }
        for (int id : fillers) {
            size_t bp = 0;
            int bw = 0;
            long best = LONG_MIN;
            for (size_t p = 0; p < host.phases.size(); ++p)
                for (int w = 0; w < G; ++w) {
                    const long slack = pmax[p] - load[p][static_cast<size_t>(w)];
                    if (slack > best) { best = slack; bp = p; bw = w; }
                }
            host.phases[bp][static_cast<size_t>(bw)].push_back(id);
            load[bp][static_cast<size_t>(bw)] += g.tasks[static_cast<size_t>(id)].cost;
            pmax[bp] = std::max(pmax[bp], load[bp][static_cast<size_t>(bw)]);
        }
    }
    if (knob("EMTB200_CG_DUMP", 0)) {  // schedule dump: per phase, per warp "kind x count (cost)"
        for (const Sched* sc : std::initializer_list<const Sched*>{&sa, &sb, &sc3}) {
            std::fprintf(stderr, "region %s\n", sc == &sa ? "A" : sc == &sb ? "B" : "C");
            for (size_t p = 0; p < sc->phases.size(); ++p) {
                std::fprintf(stderr, " phase %zu:", p);
                for (int w = 0; w < G; ++w) {
                    std::map<int, std::pair<int, long>> k;
                    for (int id : sc->phases[p][static_cast<size_t>(w)]) {
                        auto& e = k[g.tasks[static_cast<size_t>(id)].kind];
                        e.first += 1;
                        e.second += g.tasks[static_cast<size_t>(id)].cost;
                    }
                    std::fprintf(stderr, " |w%d", w);
                    for (auto& kv : k) std::fprintf(stderr, " %s%d(%ld)", kKindName[kv.first], kv.second.first, kv.second.second);
                }
                std::fprintf(stderr, "\n");
            }
        }
    }

    // ---- tables (records: ints + doubles, terms) and per-(phase, warp) segment code
    std::vector<int> rki;
    std::vector<double> rkd;
    int segs_total = 0;
    const bool straight = opt.mode != 2 && knob("EMTB200_CG_STRAIGHT", opt.mode == 1 ? 1 : 1) != 0;
    LitCtx lctx;
    if (knob("EMTB200_CG_SWFOLD", 1)) lctx.lit_init = [&](int k) -> int { return g.invariant(k) ? (g.c0(k) != 0.0 ? 1 : 0) : -1; };
    lctx.divguard = opt.exact_division ? 2 : knob("EMTB200_CG_DIVGUARD", 1);  // 0: dev A/B only (may misround)
    const bool dok_mode = straight && (knob("EMTB200_CG_DOK", 1) != 0 || g.dmma);
    lctx.dok = dok_mode;
    lctx.sh_rcp0 = g.sh_rcp(0);
    lctx.cst = [&](int k) -> std::string {
        if (g.invariant(k)) return "kC[" + std::to_string(k) + "]";
        if (g.vc_index[static_cast<size_t>(k)] >= 0) return "LD(" + std::to_string(g.vc_index[static_cast<size_t>(k)] * g.unit) + ")";
        return "__ldg(C + " + std::to_string(static_cast<long long>(k) * lanes) + ")";
    };
    // zero slot (S[0] = +0.0, never written): sums skip it and other reads become the
    // literal, removing a shared load from each ground-side branch voltage
    const int zmode = knob("EMTB200_CG_ZTERM", 1);  // 1: sums skip it, 2: also literal reads
    const bool zterm = straight && zmode != 0;
    lctx.zterm = zterm;
    const bool warp_major = knob("EMTB200_CG_WARPMAJOR", 1) != 0;
    const bool switch_bits = knob("EMTB200_CG_SWBITS", 1) != 0;
    bool sw_slim = switch_bits && g.chg_flag && knob("EMTB200_CG_SWSLIM", 1) != 0;
    const bool sw_gate = knob("EMTB200_CG_SWGATE", 1) != 0;
    {
        std::set<int> sw_slots;
        for (const Task& t : g.tasks)
            if (t.kind == K_SW) { sw_slots.insert(t.reads.begin(), t.reads.end()); sw_slots.insert(t.writes.begin(), t.writes.end()); }
        for (const Task& t : g.tasks) {
            if (t.kind == K_SW) continue;
            for (int x : t.reads) sw_slim = sw_slim && !sw_slots.count(x);
            for (int x : t.writes) sw_slim = sw_slim && !sw_slots.count(x);
        }
    }
    std::vector<std::pair<std::string, std::vector<int>>> sw_tables;
    // One same-kind segment as a loop over a constant-memory record table
    // (warp-uniform records: LDCU + LDS [lane base + uniform offset]).
    auto emit_compact = [&](const Segment& sg, const std::vector<int>& ordered) {
        SegLayout L;
        const Task& t0 = g.tasks[static_cast<size_t>(ordered[static_cast<size_t>(sg.first)])];
        L.nI = static_cast<int>(t0.f.size());
        L.nC = static_cast<int>(t0.ck.size());
        L.TC = static_cast<int>(t0.terms.size());
        L.cmode.assign(static_cast<size_t>(L.nC), 0);
        for (int c = 0; c < L.nC; ++c) {
            bool all_inv = true, all_cached = true;
            for (int q = 0; q < sg.count; ++q) {
                const int k = g.tasks[static_cast<size_t>(ordered[static_cast<size_t>(sg.first + q)])].ck[static_cast<size_t>(c)];
                all_inv = all_inv && g.invariant(k);
                all_cached = all_cached && g.vc_index[static_cast<size_t>(k)] >= 0;
            }
            L.cmode[static_cast<size_t>(c)] = all_inv ? 0 : (all_cached ? 2 : 1);
        }
        L.SI = L.nI + 2 * L.TC;
        L.SD = 0;
        L.cpos.assign(static_cast<size_t>(L.nC), 0);
        for (int c = 0; c < L.nC; ++c) L.cpos[static_cast<size_t>(c)] = L.cmode[static_cast<size_t>(c)] ? L.SI++ : L.SD++;
        const int bi0 = static_cast<int>(rki.size()), bd0 = static_cast<int>(rkd.size());
        for (int q = 0; q < sg.count; ++q) {
            const Task& t = g.tasks[static_cast<size_t>(ordered[static_cast<size_t>(sg.first + q)])];
            std::vector<int> rec(static_cast<size_t>(L.SI), 0);
            std::copy(t.f.begin(), t.f.end(), rec.begin());
            for (int j = 0; j < L.TC; ++j) {
                rec[static_cast<size_t>(L.nI + 2 * j)] = t.terms[static_cast<size_t>(j)].first;
                rec[static_cast<size_t>(L.nI + 2 * j + 1)] = t.terms[static_cast<size_t>(j)].second;
            }
            for (int c = 0; c < L.nC; ++c) {
                const int k = t.ck[static_cast<size_t>(c)];
                const int m = L.cmode[static_cast<size_t>(c)];
                if (m == 0) rkd.push_back(g.c0(k));
                else rec[static_cast<size_t>(L.cpos[static_cast<size_t>(c)])] = m == 2 ? g.vc_index[static_cast<size_t>(k)] * g.unit : k;
            }
            rki.insert(rki.end(), rec.begin(), rec.end());
        }
        ++segs_total;
        return segment_code(sg.kind, sg.count, sg.indep != 0, bi0, bd0, L, "      ");
    };
    // hybrid: in the straight-line form, long independent same-kind runs become loops
    const int loop_min = knob("EMTB200_CG_LOOPMIN", 0);
    // phase profiler (EMTB200_CG_PROF=1): CTA 0, lane 0 of each warp adds the cycles
    // since its previous marker to a.prof[warp * 64 + marker] (compute, then barrier wait)
    const bool prof = knob("EMTB200_CG_PROF", 0) != 0;
    int prof_base = 0;  // first marker id of the region being emitted
    auto mark = [&](int id) {
        if (!prof) return std::string();
        return "      PROF(" + std::to_string(id) + ");\n";
    };
    auto loopable = [](int kind) {
        return kind != K_SW && kind != K_FWD && kind != K_BWD && kind != K_BERG && kind != K_GATHER && kind != K_SUM;
    };
    std::vector<std::string> wprefix, wsuffix;  // per-warp code around a region's block (empty: none)
    // (A split poll — one warp waits for the peers' progress and releases the line-end
    // warps with a named barrier — measured slower: C4 3.26 -> 3.61 us; not kept.)
    // (Also measured slower and not kept: peer histories loaded one pass ahead into
    // registers, C4 3.21 -> 3.30 us; relaxed progress polls issued early in region A or
    // B with an acquire fence later, C4 +8..12%: the fence holds the warp ~1000 cycles.)
    bool in_region_a = false;
    auto region_code = [&](const Sched& sc, bool fused_pass) {
        std::ostringstream rc;
        if (straight && warp_major) {
            // One contiguous block per warp holding all of its phases, phases
            // separated by bar.sync: a single warp-uniform dispatch per region
            // (instead of an if/else chain per phase) and sequential code per
            // warp for the instruction prefetcher.
            rc << "    switch (warp) {\n";
            for (int w = 0; w < G; ++w) {
                rc << "    case " << w << ": {\n";
                if (!wprefix.empty()) rc << wprefix[static_cast<size_t>(w)];
                if (solo) rc << "      if (lane == 0) {\n";
                std::vector<int> sw_ids;  // process id per swbits bit
                std::vector<int> sw_tasks;  // task per swbits bit
                std::string sw_lits;        // gated slim switch tests of this warp
                for (size_t p = 0; p < sc.phases.size(); ++p) {
                    if (p > 0) rc << mark(prof_base + 2 * static_cast<int>(p) - 2) << (solo ? "      }\n" : "") << "      BAR();\n"
                                  << (solo ? "      if (lane == 0) {\n" : "") << mark(prof_base + 2 * static_cast<int>(p) - 1);
                    std::vector<int> ordered;
                    const auto segs = segments_of(sc.phases[p][static_cast<size_t>(w)], deps, g.tasks, ordered);
                    std::vector<int> seg_of(ordered.size(), -1);
                    for (size_t si = 0; si < segs.size(); ++si)
                        for (int q = 0; q < segs[si].count; ++q) seg_of[static_cast<size_t>(segs[si].first + q)] = static_cast<int>(si);
                    for (size_t oi = 0; oi < ordered.size(); ++oi) {
                        if (loop_min > 0) {
                            const Segment& sg = segs[static_cast<size_t>(seg_of[oi])];
                            if (sg.count >= loop_min && sg.indep && loopable(sg.kind)) {
                                if (static_cast<int>(oi) == sg.first) rc << emit_compact(sg, ordered);  // tasks in order
                                continue;
                            }
                        }
                        const int id = ordered[oi];
                        const Task& t = g.tasks[static_cast<size_t>(id)];
                        LitCtx c = lctx;
                        c.fused_pass = fused_pass;
                        c.task_id = id;
                        if (t.kind == K_SW && switch_bits && sw_ids.size() < 64 && t.region == 0) {
                            c.sw_bit = static_cast<int>(sw_ids.size());
                            c.chg_flag = g.chg_flag;
                            c.sw_slim = sw_slim;
                            sw_ids.push_back(t.f[3]);
                            sw_tasks.push_back(id);
                            if (sw_slim && sw_gate) {  // hot path gated below: nothing in the pass reads it
                                sw_lits += "        " + task_literal(t, c) + "\n";
                                continue;
                            }
                        }
                        rc << "      " << task_literal(t, c) << "\n";
                    }
                }
                if (!sw_lits.empty()) {
                    // switches only change state when t reaches one of their toggle times: the
                    // warp evaluates them on a launch's first pass and when some lane's next
                    // toggle time is due, and otherwise skips them (their hot path is a no-op)
                    std::ostringstream nx;
                    for (int id : sw_tasks) {
                        const Task& t = g.tasks[static_cast<size_t>(id)];
                        for (size_t q = 3; q < t.ck.size(); ++q)
                            nx << " { const double T_ = " << lctx.cst(t.ck[q]) << "; if (T_ > t && T_ < swnext) swnext = T_; }";
                    }
                    rc << (solo ? "      if (t >= swnext) {\n" : "      if (__any_sync(0xffffffffu, t >= swnext)) {\n") << sw_lits
                       << "        swnext = __longlong_as_double(0x7ff0000000000000LL);" << nx.str() << "\n      }\n";
                    sw_lits.clear();
                }
                if (!sw_ids.empty()) {
                    const std::string tab = "kSwIds" + std::to_string(sw_tables.size());
                    sw_tables.push_back({tab, sw_ids});
                    std::string commit;  // slim path: state and conductance stores of the changed switches
                    if (sw_slim) {
                        std::ostringstream cm;
                        // the first pass of a launch writes every switch's state and conductance,
                        // as the reference does each pass (the arena may hold other initial values)
                        cm << " { unsigned long long b = it == 0 ? " << (sw_tasks.size() >= 64 ? std::string("~0ull") : "((1ull << " + std::to_string(sw_tasks.size()) + ") - 1ull)")
                           << " : swbits; while (b) { const int j = __ffsll((long long)b) - 1; b &= b - 1; switch (j) {";
                        for (size_t j = 0; j < sw_tasks.size(); ++j) {
                            const Task& t = g.tasks[static_cast<size_t>(sw_tasks[j])];
                            cm << " case " << j << ": { int now = " << lctx.cst(t.ck[2]) << " != 0.0 ? 1 : 0;";
                            for (size_t q = 3; q < t.ck.size(); ++q) cm << " if (t >= " << lctx.cst(t.ck[q]) << ") now ^= 1;";
                            cm << " ST(" << t.f[0] << ", (double)now); ST(" << t.f[2] << ", now != 0 ? " << lctx.cst(t.ck[0]) << " : "
                               << lctx.cst(t.ck[1]) << "); } break;";
                        }
                        cm << " } } }";
                        commit = cm.str();
                    }
                    if (sw_slim) rc << "      if (it == 0 || swbits != 0ull) {" << commit << " }\n";
                    rc << "      if (swbits != 0ull) { wflag = 1;" << (g.chg_flag ? " needS[lane] = 1;" : "")
                       << " if (live && a.events) { unsigned long long b = swbits; while (b) { const int j = __ffsll((long long)b) - 1; "
                          "b &= b - 1; const int e = atomicAdd(a.n_events, 1); if (e < a.max_events) { a.events[3*e] = step; "
                          "a.events[3*e+1] = gl; a.events[3*e+2] = " << tab << "[j]; } } } }\n";
                }
                if (solo) rc << "      }\n";
                if (!wsuffix.empty()) rc << wsuffix[static_cast<size_t>(w)];
                rc << mark(prof_base + 2 * static_cast<int>(sc.phases.size()) - 2) << "    } break;\n";
            }
            rc << "    }\n";
            prof_base += 2 * static_cast<int>(sc.phases.size());
            return rc.str();
        }
        for (size_t p = 0; p < sc.phases.size(); ++p) {
            if (p > 0) rc << "    __syncthreads();\n";
            bool first = true;
            for (int w = 0; w < G; ++w) {
                std::vector<int> ordered;
                const auto segs = segments_of(sc.phases[p][static_cast<size_t>(w)], deps, g.tasks, ordered);
                if (segs.empty()) continue;
                rc << "    " << (first ? "if" : "else if") << " (warp == " << w << ") {\n";
                first = false;
                if (straight) {
                    for (int id : ordered) rc << "      " << task_literal(g.tasks[static_cast<size_t>(id)], lctx) << "\n";
                    rc << "    }\n";
                    continue;
                }
                for (const Segment& sg : segs) rc << emit_compact(sg, ordered);
                rc << "    }\n";
            }
        }
        return rc.str();
    };
    in_region_a = true;
    std::string code_a = region_code(sa, false);
    const std::string code_a0 = code_a;
    std::string code_af;
    if (!g.fused.empty()) {  // the launch's first pass reads i_prev from the arena; later passes recompute it
        code_af = region_code(sa, true);
        code_a = "    if (__builtin_expect(it != 0, 1)) {\n" + code_af + "    } else {\n" + code_a + "    }\n";
    }
    in_region_a = false;
    wprefix.clear();
    const std::string code_b = region_code(sb, false);
    wprefix.clear();
    wsuffix.clear();
    const std::string code_c = g.dmma ? region_code(sc3, false) : std::string();
    const size_t const_bytes = rki.size() * 4 + rkd.size() * 8 + static_cast<size_t>(s.consts) * 8;
    if (const_bytes > 62 * 1024) {
        fail = {13, "", "task tables (" + std::to_string(const_bytes) + " B) exceed constant memory"};
        return false;
    }


    std::string pre_prologue;
    if (!g.pre_ck.empty()) {  // the launch's first pass: source values computed here
        std::ostringstream pp;
        pp << "  if (warp == 0) { const double tn = (double)(a.step0 + 1) * " << lit(s.dt) << ";\n";
        for (size_t j = 0; j < g.pre_ck.size(); ++j)
            pp << "    { const double m_ = " << g.C(g.pre_ck[j][0]) << ", w_ = " << g.C(g.pre_ck[j][1]) << ", p_ = "
               << g.C(g.pre_ck[j][2]) << "; S[" << (g.pre_base + static_cast<int>(j)) * LPC
               << "] = w_ == 0.0 ? m_ : m_ * emt_libm_cos(w_ * tn + p_); }\n";
        pp << "  }\n";
        pre_prologue = pp.str();
    }
    // ---- shared-G tensor-core solve: V = G^-1 I with DMMA (mma.sync m8n8k4 f64)
    std::string dmma_prologue, dmma_block, dmma_tables;
    if (g.dmma) {
        const int MP = MT * 8, KP = KT * 4;
        std::vector<double> gi(static_cast<size_t>(MP) * KP, 0.0);
        for (int i = 0; i < s.dim; ++i)
            for (int j = 0; j < s.dim; ++j) gi[static_cast<size_t>(i) * KP + j] = ginv[static_cast<size_t>(i) * s.dim + j];
        std::vector<int> vrow(static_cast<size_t>(std::max(MP, KP)), 0);  // S row (double offset) of node k, 0 = zero slot
        for (int k = 0; k < s.dim; ++k) vrow[static_cast<size_t>(k)] = g.hot_index[static_cast<size_t>(s.v_base + k)] * 32;
        std::ostringstream tb;
        tb << "__device__ const double kGinv[" << gi.size() << "] = {";
        for (size_t q = 0; q < gi.size(); ++q) tb << (q ? "," : "") << lit(gi[q]);
        tb << "};\n__constant__ int kVrow[" << vrow.size() << "] = {";
        for (size_t q = 0; q < vrow.size(); ++q) tb << (q ? "," : "") << vrow[q];
        tb << "};\n";
        dmma_tables = tb.str();
        const long long gi_off = static_cast<long long>(g.smem_slots()) * 32 + 32;  // after serr/needS (64 ints)
        std::ostringstream pr;
        pr << "  double* __restrict__ GI = sm + " << gi_off << ";\n"
           << "  for (int q = threadIdx.x; q < " << gi.size() << "; q += " << 32 * G << ") GI[q] = kGinv[q];\n";
        dmma_prologue = pr.str();
        const int ntile = MT * 4;  // 4 n-tiles of 8 lanes
        std::ostringstream blk;
        blk << "    __syncthreads();  // every gather (I = the v slots) is in shared memory\n"
            << "    switch (warp) {\n";
        for (int w = 0; w < G; ++w) {
            std::vector<int> tiles;
            for (int t = w; t < ntile; t += G) tiles.push_back(t);
            blk << "    case " << w << ": {\n";
            for (size_t j = 0; j < tiles.size(); ++j) blk << "      double d" << j << "a = 0.0, d" << j << "b = 0.0;\n";
            for (int kk = 0; kk < KT; ++kk) {
                blk << "      { const int vr = kVrow[" << kk * 4 << " + (lane & 3)];\n";
                for (size_t j = 0; j < tiles.size(); ++j) {
                    const int mt = tiles[j] / 4, ntl = tiles[j] % 4;
                    blk << "        { const double av = GI[(" << mt * 8 << " + (lane >> 2)) * " << KP << " + " << kk * 4
                        << " + (lane & 3)]; const double bv = sm[vr + " << ntl * 8 << " + (lane >> 2)]; "
                        << "asm volatile(\"mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\" "
                        << ": \"+d\"(d" << j << "a), \"+d\"(d" << j << "b) : \"d\"(av), \"d\"(bv)); }\n";
                }
                blk << "      }\n";
            }
            blk << "      BAR();  // all reads of I done before V overwrites the v slots\n";
            for (size_t j = 0; j < tiles.size(); ++j) {
                const int mt = tiles[j] / 4, ntl = tiles[j] % 4;
                blk << "      { const int m = " << mt * 8 << " + (lane >> 2); if (m < " << s.dim << ") { const int o = kVrow[m] + "
                    << ntl * 8 << " + (lane & 3) * 2; sm[o] = d" << j << "a; sm[o + 1] = d" << j << "b; "
                    << "dok = dok & (fabs(d" << j << "a) <= dlim) & (fabs(d" << j << "b) <= dlim); } }\n";
            }
            blk << "    } break;\n";
        }
        blk << "    }\n"
            << "    __syncthreads();  // V visible to finalize / control\n";
        dmma_block = blk.str();
        smem += ginv_bytes + 32 * sizeof(int);
    }
    // (AC source values copied one pass ahead into shared memory with cp.async measured
    // slower: C3 2.64 -> 2.75 ms, C4 3.92 -> 4.34 ms per 1000 passes; not kept.)
    // ---- source
    std::ostringstream o;
    const int nhot = static_cast<int>(g.hot_slots.size());
    const long long Wl = lanes;
    o << "// generated by emtb200 codegen: " << s.nodes << " nodes, " << s.comps << " components, " << s.layers
      << " layers, " << lanes << " lanes, " << G << " warps, " << nt << " tasks, " << segs_total << " segments\n";
    {
        const int ns = g.tab_shared(), nv = static_cast<int>(g.tab_ck.size()) - g.tab_shared();
        o << "#define NSHR_ " << ns << "\n#define NSRC_ " << std::max<long long>(1, ns + static_cast<long long>(nv) * lanes) << "LL\n";
        out.nsrc = static_cast<int>(std::max<long long>(0, ns + static_cast<long long>(nv) * lanes));
        o << "#define SRCV_(j) __ldg(a.srctab + (size_t)it * NSRC_ + ((j) < NSHR_ ? (j) : NSHR_ + ((j) - NSHR_) * W_ + gl))\n";
    }
    o << "#define W_ " << Wl << "LL\n#define NCH " << s.channel_slot.size() << "\n#define LB_ " << opt.lane_begin << "LL\n";
    o << libm_cos_prelude();
    o << "struct KArgs { double* arena; const double* ctab; double* waves; unsigned char* refac; int* lane_err;\n"
      << "  int* events; int* n_events; int max_events; int step0; int nsteps; int row0; double div_limit;\n"
      << "  double* ring; long long ring_lo; long long ring_cols; unsigned int* progress; int min_k; int nblocks; long long* prof; const double* srctab;\n"
      << "  int prog_off; int sys_scope; int* pick; };\n";
    auto carr_i = [&](const char* qual, const char* name, const std::vector<int>& v) {
        o << qual << " int " << name << "[" << std::max<size_t>(1, v.size()) << "] = {";
        for (size_t q = 0; q < v.size(); ++q) o << (q ? "," : "") << v[q];
        if (v.empty()) o << "0";
        o << "};\n";
    };
    o << "__constant__ double kC[" << std::max(1, s.consts) << "] = {";
    for (int k = 0; k < s.consts; ++k) o << (k ? "," : "") << lit(g.c0(k));
    if (s.consts == 0) o << "0.0";
    o << "};\n";
    carr_i("__constant__", "kRi", rki);
    o << "__constant__ double kRd[" << std::max<size_t>(1, rkd.size()) << "] = {";
    for (size_t q = 0; q < rkd.size(); ++q) o << (q ? "," : "") << lit(rkd[q]);
    if (rkd.empty()) o << "0.0";
    o << "};\n";
    std::vector<int> hot_arena(g.hot_slots.begin() + 1, g.hot_slots.end());
    carr_i("__device__ const", "kHot", hot_arena);
    // Hot slots the launch-end block writes itself (lazily finalized currents, aliased
    // control outputs): their shared copy is stale, so the write-back must skip them —
    // two unordered stores to one arena word from different warps otherwise race.
    std::set<int> late_slots;
    for (const auto& kv : g.alias_of) late_slots.insert(kv.first);
    for (int c : g.lazy_fin) late_slots.insert(s.finalize[5 * static_cast<size_t>(c)]);
    std::vector<int> wb_q;  // hot indices (1-based) copied back at the launch end
    for (int q = 0; q + 1 < nhot; ++q)
        if (!late_slots.count(g.hot_slots[static_cast<size_t>(q) + 1])) wb_q.push_back(q + 1);
    carr_i("__device__ const", "kWbQ", wb_q);
    std::vector<int> dslot, dconst, cslot, chot, csign;
    for (int x = 0; x < s.extent; ++x) {
        if (g.cls[static_cast<size_t>(x)] == kDerived) {
            dslot.push_back(x);
            dconst.push_back(g.derived_const[static_cast<size_t>(x)]);
        } else if (g.cls[static_cast<size_t>(x)] == kContrib) {
            const int h = g.contrib_h[static_cast<size_t>(x)];
            cslot.push_back(x);
            chot.push_back(g.cls[static_cast<size_t>(h)] == kHot ? g.hot_index[static_cast<size_t>(h)] : -1);
            csign.push_back(g.contrib_sign[static_cast<size_t>(x)]);
        }
    }
    for (const auto& tb : sw_tables) carr_i("__constant__", tb.first.c_str(), tb.second);
    o << dmma_tables;
    carr_i("__device__ const", "kDerSlot", dslot);
    carr_i("__device__ const", "kVC", g.vc_slots);
    carr_i("__device__ const", "kChgSlot", g.chg_flag ? g.chg_slots : std::vector<int>());
    carr_i("__device__ const", "kDerConst", dconst);
    carr_i("__device__ const", "kConSlot", cslot);
    carr_i("__device__ const", "kConHot", chot);
    carr_i("__device__ const", "kConSign", csign);
    // warps reach their phase barriers at different instructions: the non-.aligned
    // barrier form is the one the PTX ISA allows there (compute-sanitizer synccheck clean)
    o << "#define BAR() asm volatile(\"barrier.sync 0;\" ::: \"memory\")\n";
    // non-aligned barrier reduction (warps arrive from different code): __syncthreads_or
    o << "__device__ __forceinline__ bool emt_bar_or(bool p) { unsigned r_; asm volatile(\"{ .reg .pred pi_, po_; setp.ne.u32 pi_, %1, 0; "
         "barrier.red.or.pred po_, 0, pi_; selp.u32 %0, 1, 0, po_; }\" : \"=r\"(r_) : \"r\"((unsigned)p) : \"memory\"); return r_ != 0; }\n";
    o << "#define PROF(id) do { if (a.prof && BID_ == 0 && lane == 0) { const long long c_ = clock64(); "
         "atomicAdd((unsigned long long*)(a.prof + warp * 64 + (id)), (unsigned long long)(c_ - prof_t)); prof_t = c_; } } while (0)\n";
    // a failing CTA leaves the step loop: release CTAs waiting on its progress word
    o << "#define FAILPUB() do { if (a.progress != nullptr && threadIdx.x == 0) atomicExch(a.progress + a.prog_off + BID_, 0x3fffffffu); } while (0)\n";
    o << "#define LD(o) (*(const double*)(Sb + (o)))\n"
      << "#define ST(o, v) (*(double*)(Sb + (o)) = (v))\n"
      << "#define SGN(x, n) ((n) ? -(x) : (x))\n";
    if (g.chg_flag)
        o << "#define SETCHG(o, c) do { if ((c) != 0.0) needS[lane] = 1; } while (0)\n";
    else
        o << "#define SETCHG(o, c) ST(o, c)\n";
    if (lu_smem)
        o << "#define LU(x) LD(x)\n";
    else
        o << "#define LU(x) (A[(size_t)(x) * W_])\n";

    // Full-chip launch (a.pick != null, engine.cu: setup_claim): the engine launches
    // one CTA per SM and the CTA on SM s < groups takes lane group s. A launch of
    // fewer CTAs than SMs runs up to 13% slower on some B200s (an issue throttle of
    // low-grid launches), and lane groups spread over more TPCs than SMs 0..n-1 run
    // slower still (profiles/ab/placement_r2.log). Correct whatever the placement:
    // a group is taken by compare-and-swap on its flag (a.pick[1 + g]); a CTA that
    // gets none (a spare SM, or its SM's group already taken) waits until every CTA
    // of the launch has started -- or 20 us have passed, e.g. while another kernel
    // holds SMs -- and then takes any group still free. Spares >= free groups, since
    // the grid is >= the group count.
    const std::string NG = "((W_ + " + std::to_string(LPC) + " - 1) / " + std::to_string(LPC) + ")";
    const std::string bid_code =
        "  int BID_ = blockIdx.x;\n"
        "  if (a.pick != nullptr) {\n"
        "    __shared__ int s_bid_;\n"
        "    if (threadIdx.x == 0) {\n"
        "      unsigned smid_; asm volatile(\"mov.u32 %0, %%smid;\" : \"=r\"(smid_));\n"
        "      int b_ = -1;\n"
        "      if ((long long)smid_ < " + NG + " && atomicCAS(a.pick + 1 + smid_, 0, 1) == 0) b_ = (int)smid_;\n"
        "      __threadfence();\n"
        "      atomicAdd(a.pick, 1);\n"
        "      if (b_ < 0) {\n"
        "        unsigned long long t0_, t_;\n"
        "        asm volatile(\"mov.u64 %0, %%globaltimer;\" : \"=l\"(t0_));\n"
        "        for (;;) {\n"
        "          if (*(volatile int*)a.pick >= (int)gridDim.x) break;\n"
        "          asm volatile(\"mov.u64 %0, %%globaltimer;\" : \"=l\"(t_));\n"
        "          if (t_ - t0_ > 20000ull) break;\n"
        "          __nanosleep(100);\n"
        "        }\n"
        "        __threadfence();\n"
        "        for (int g_ = 0; g_ < " + NG + " && b_ < 0; ++g_)\n"
        "          if (*(volatile int*)(a.pick + 1 + g_) == 0 && atomicCAS(a.pick + 1 + g_, 0, 1) == 0) b_ = g_;\n"
        "      }\n"
        "      s_bid_ = b_;\n"
        "    }\n"
        "    __syncthreads();\n"
        "    BID_ = s_bid_;\n"
        "    if (BID_ < 0) return;\n"
        "  }\n";
    o << "extern \"C\" __global__ void __launch_bounds__(" << 32 * G << ", 1) emt_cg_kernel(const KArgs a) {\n"
      << "  extern __shared__ double sm[];\n"
      << "  const int lane = threadIdx.x & 31; const int warp = threadIdx.x >> 5;\n"
      // dev check: a NaN-filled shared memory at entry turns any read-before-write of a
      // slot the prologue does not load into a parity failure
      << (knob("EMTB200_CG_POISON", 0) ? "  for (int q = threadIdx.x; q < " + std::to_string(smem / 8) +
                                             "; q += blockDim.x) sm[q] = __longlong_as_double(0x7ff4000000000badLL);\n  __syncthreads();\n"
                                       : std::string())
      << "  const int slane = lane < " << LPC << " ? lane : 0;  // shadow threads mirror lane 0\n"
      << bid_code
      << "  const int graw = BID_ * " << LPC << " + slane; const bool live = lane < " << LPC << " && graw < W_;\n"
      << "  const int gl = graw < W_ ? graw : (int)(W_ - 1);\n"
      << "  double* __restrict__ S = sm + slane;\n"
      << "  char* __restrict__ Sb = (char*)S;\n"
      << "  int* serr = (int*)(sm + " << static_cast<long long>(g.smem_slots()) * LPC << ") + slane - lane;\n"
      << "  int* needS = serr + " << LPC << "; (void)needS;\n"
      << "  double* __restrict__ A = a.arena + gl;\n"
      << "  const double* __restrict__ C = a.ctab + gl;\n"
      << "  (void)C;\n"
      << (solo ? "  if (warp == 0 && lane == 0) { S[0] = 0.0; serr[lane] = 0x7fffffff; needS[lane] = 0; }\n"
               : "  if (warp == 0) { S[0] = 0.0; serr[lane] = 0x7fffffff; needS[lane] = 0; }\n")
      << (g.lu_shared ? "  double* __restrict__ SH = sm + " + std::to_string(static_cast<long long>(g.smem_slots()) * LPC + LPC) +
                            ";  // shared factors: L, U, pivot reciprocals (one copy per CTA)\n"
                      : std::string())
      << pre_prologue
      << dmma_prologue
;
    const bool slcopy = knob("EMTB200_CG_SLCOPY", 1) != 0;
    if (slcopy) {
        std::vector<std::pair<std::string, std::string>> it;
        for (size_t q = 0; q < g.vc_slots.size(); ++q)
            it.push_back({"S[" + std::to_string((g.vc_base + static_cast<long long>(q)) * LPC) + "]",
                          "__ldg(C + (size_t)" + std::to_string(g.vc_slots[q]) + " * W_)"});
        for (int q = 0; q + 1 < nhot; ++q)
            it.push_back({"S[" + std::to_string(static_cast<long long>(q + 1) * LPC) + "]",
                          "A[(size_t)" + std::to_string(g.hot_slots[static_cast<size_t>(q) + 1]) + " * W_]"});
        o << warp_copies(it, G, "  ", 16, solo);
    } else {
        o << "  _Pragma(\"unroll 8\") for (int q = warp; q < " << g.vc_slots.size() << "; q += " << G << ") S[(" << g.vc_base << " + q) * " << LPC << "] = __ldg(C + (size_t)kVC[q] * W_);\n"
          << "  _Pragma(\"unroll 8\") for (int q = warp; q < " << nhot - 1 << "; q += " << G << ") S[(q + 1) * " << LPC << "] = A[(size_t)kHot[q] * W_];\n";
    }
    if (lu_smem && slcopy) {
        std::vector<std::pair<std::string, std::string>> it;
        for (size_t q = 0; q < s.l_col.size(); ++q)
            it.push_back({"S[" + std::to_string((g.l_base_smem + static_cast<long long>(q)) * LPC) + "]",
                          "A[(size_t)" + std::to_string(s.l + static_cast<long long>(q)) + " * W_]"});
        for (size_t q = 0; q < s.u_col.size(); ++q)
            it.push_back({"S[" + std::to_string((g.u_base_smem + static_cast<long long>(q)) * LPC) + "]",
                          "A[(size_t)" + std::to_string(s.u + static_cast<long long>(q)) + " * W_]"});
        o << warp_copies(it, G, "  ", 16, solo);
    } else if (lu_smem) {
        o << "  _Pragma(\"unroll 8\") for (int q = warp; q < " << s.l_col.size() << "; q += " << G << ") S[(" << g.l_base_smem << " + q) * " << LPC << "] = A[(size_t)("
          << s.l << " + q) * W_];\n";
        o << "  _Pragma(\"unroll 8\") for (int q = warp; q < " << s.u_col.size() << "; q += " << G << ") S[(" << g.u_base_smem << " + q) * " << LPC << "] = A[(size_t)("
          << s.u << " + q) * W_];\n";
    }
    if (lu_smem) {
        if (g.rcp_base >= 0 && slcopy) {
            std::vector<std::pair<std::string, std::string>> it;
            for (int i = 0; i < s.dim; ++i)
                it.push_back({"S[" + std::to_string(static_cast<long long>(g.rcp_base + i) * LPC) + "]",
                              "EMT_RCP(A[(size_t)" + std::to_string(s.u + s.u_row_ptr[static_cast<size_t>(i)]) + " * W_])"});
            o << warp_copies(it, G, "  ", 16, solo);
        } else if (g.rcp_base >= 0) {
            std::ostringstream dg;
            for (int i = 0; i < s.dim; ++i) dg << (i ? "," : "") << s.u_row_ptr[static_cast<size_t>(i)];
            o << "  { const int kUd[" << s.dim << "] = {" << dg.str() << "};\n"
              << "    _Pragma(\"unroll 8\") for (int q = warp; q < " << s.dim << "; q += " << G << ") S[(" << g.rcp_base << " + q) * " << LPC << "] = EMT_RCP(A[(size_t)("
              << s.u << " + kUd[q]) * W_]); }\n";
        }
    }
    if (g.lu_shared) {
        // the factors of the CTA's first lane (every lane holds the same); reciprocals
        // from the same arena values
        const std::string base = "(size_t)BID_ * " + std::to_string(LPC);
        std::vector<std::pair<std::string, std::string>> it;
        const size_t nl = s.l_col.size(), nu = s.u_col.size();
        for (size_t q = 0; q < nl; ++q)
            it.push_back({"SH[" + std::to_string(q) + "]", "a.arena[(size_t)" + std::to_string(s.l + static_cast<long long>(q)) + " * W_ + " + base + "]"});
        for (size_t q = 0; q < nu; ++q)
            it.push_back({"SH[" + std::to_string(nl + q) + "]", "a.arena[(size_t)" + std::to_string(s.u + static_cast<long long>(q)) + " * W_ + " + base + "]"});
        for (int i = 0; i < s.dim; ++i)
            it.push_back({"SH[" + std::to_string(g.sh_rcp(i)) + "]",
                          "EMT_RCP(a.arena[(size_t)" + std::to_string(s.u + s.u_row_ptr[static_cast<size_t>(i)]) + " * W_ + " + base + "])"});
        o << warp_copies(it, G, "  ", 16, solo);
    }
    // watch slots not rewritten by region-A tasks (the dirty flag) are checked up front
    std::set<int> written_a;
    for (const Task& t : g.tasks)
        if (t.region == 0)
            for (int w : t.writes) written_a.insert(w);
    o << "  __shared__ int s_cmin;\n"
      << "  if (threadIdx.x == 0) s_cmin = -0x3fffffff;\n"
      << "  __syncthreads();\n"
      << "  int it = 0;\n"
      << "  long long prof_t = clock64(); (void)prof_t;\n"
      << "  double swnext = -1.0; (void)swnext;  // per lane: next switch toggle time not yet reached\n"
      << "  const double dlim = a.div_limit; (void)dlim;\n"
      << "  for (; it < a.nsteps; ++it) {\n"
      << "    const int step = a.step0 + it;\n"
      << "    const double t = (double)(step + 1) * " << lit(s.dt) << ";\n"
      << "    const double tn = (double)(step + 2) * " << lit(s.dt) << "; (void)tn;\n"
      // the source-table row of pass it+4 into L1 (rows are 8*NSRC_ bytes, so a pass
      // whose row starts a new line would otherwise wait on L2 in the Norton region;
      // C3 -1.3%, profiles/ab/srcl1_r2.log; not in the solo form, where it measured +0.9%,
      // nor with lane-varying source columns (C4 +1%: the row is mostly other CTAs' lanes)
      << (srcl1 > 0 && !g.tab_ck.empty() && g.tab_shared() == static_cast<int>(g.tab_ck.size())
              ? "    if (threadIdx.x == 0 && it + " + std::to_string(srcl1) + " < a.nsteps) asm volatile(\"prefetch.global.L1 [%0];\" :: \"l\"(a.srctab + (size_t)(it + " +
                    std::to_string(srcl1) + ") * NSRC_));\n"
              : std::string())
      << "    int wflag = 0; int bad = 0x7fffffff; int srow = -1; unsigned long long swbits = 0ull; bool dok = true;\n"
      << "    (void)t; (void)bad; (void)srow; (void)step; (void)swbits; (void)dok;\n"
      ;
    {
        o << "    if (a.progress != nullptr && s_cmin < step + 2 - a.min_k) {\n"
      << "      // line ends read peer rings written >= K-1 passes earlier by other CTAs:\n"
      << "      // wait until every CTA has completed pass step+1-K (its progress word)\n"
      << "      __syncthreads();\n"
      // warp 0 polls the progress words in parallel (one acquire round trip, not nblocks)
      << "      if (warp == 0) {\n"
      << "        const long long t0 = clock64(); int m;\n"
      << "        for (;;) {\n"
      << "          m = 0x7fffffff;\n"
      << "          for (int c = lane; c < a.nblocks; c += 32) { unsigned int v; if (a.sys_scope) asm volatile(\"ld.acquire.sys.global.u32 %0, [%1];\" : \"=r\"(v) : \"l\"(a.progress + c) : \"memory\"); else asm volatile(\"ld.acquire.gpu.global.u32 %0, [%1];\" : \"=r\"(v) : \"l\"(a.progress + c) : \"memory\"); m = min(m, (int)v); }\n"
      << "          m = __reduce_min_sync(0xffffffffu, m);\n"
      << "          if (m >= step + 2 - a.min_k) break;\n"
      << "          if (__shfl_sync(0xffffffffu, (int)(clock64() - t0 > 8000000000LL), 0)) { m = -1; break; }  // warp-uniform\n"
      << "        }\n"
      << "        if (a.sys_scope) __threadfence_system();  // gpu scope: the acquire loads + bar.sync suffice\n"
      << "        if (lane == 0) s_cmin = m;\n"
      << "      }\n"
      << "      __syncthreads();\n"
      << "      if (s_cmin < 0) { if (warp == 0 && live) { a.lane_err[4*gl] = 64; a.lane_err[4*gl+1] = step; a.lane_err[4*gl+2] = -1; a.lane_err[4*gl+3] = 0; } FAILPUB(); return; }\n"
      << "    }\n"
;
    }
    o       << (solo ? "    if (warp == 0 && lane == 0) { " : "    if (warp == 0) { ");
    for (int x : s.watch)
        if (x >= 0 && !written_a.count(x)) o << "wflag |= (" << g.R(x) << " != 0.0); ";
    o << "}\n";
    const std::string refactor_block =
        std::string(solo ? "      if (warp == 0 && lane == 0) {\n" : "      if (warp == 0) {\n") + g.emit_refactor() +
        "        if (lane == 0) a.refac[a.row0 + it] = 1;\n"
        "      }\n"
        "      if (__syncthreads_or(srow >= 0 && live)) {\n"
        "        if (warp == 0 && live && srow >= 0) { a.lane_err[4*gl] = 8; a.lane_err[4*gl+1] = step; a.lane_err[4*gl+2] = srow; a.lane_err[4*gl+3] = " +
        std::to_string(g.fact_layer) + "; }\n"
        "        FAILPUB(); return;\n"
        "      }\n";
    // one dispatch per pass: each warp's region A and region B code in one case, the A/B
    // boundary a non-aligned barrier reduction inside the case; the rare refactorisation
    // leaves the switch and re-enters the case after it. C3 -1.2%, C2 -1.6%, C4 -1.7%;
    // not for shared factors (C5 +5.3%), profiles/ab/mergeab_r2.log
    std::vector<std::string> ba0, baf, bb;
    const bool merge_ab = knob("EMTB200_CG_MERGEAB", g.lu_shared ? 0 : 1) != 0 && straight && warp_major && !g.dmma && code_c.empty() &&
                          split_warp_cases(code_a0, G, ba0) && (code_af.empty() || split_warp_cases(code_af, G, baf)) &&
                          split_warp_cases(code_b, G, bb);
    if (merge_ab) {
        o << "    switch (warp) {\n";
        for (int w = 0; w < G; ++w) {
            o << "    case " << w << ": {\n";
            if (!code_af.empty())
                o << "    if (__builtin_expect(it != 0, 1)) {\n" << baf[static_cast<size_t>(w)] << "    } else {\n" << ba0[static_cast<size_t>(w)] << "    }\n";
            else
                o << ba0[static_cast<size_t>(w)];
            o << "      if (emt_bar_or(wflag)) goto cold_ab_;\n    resume_ab_" << w << ":;\n" << bb[static_cast<size_t>(w)] << "    } break;\n";
        }
        o << "    }\n    if (false) {\n    cold_ab_:;\n" << refactor_block << "      switch (warp) {";
        for (int w = 0; w < G; ++w) o << " case " << w << ": goto resume_ab_" << w << ";";
        o << " default: break; }\n    }\n";
    } else {
        o << code_a;
        o << "    if (__syncthreads_or(wflag)) {\n" << refactor_block << "    }\n";
    }
    // progress release at the pass end: st.release after bar.sync orders the whole CTA's
    // earlier stores (PTX memory model: the barrier puts them before the releasing
    // thread's store in causality order). Releasing right after region A (C4 3.35 ->
    // 4.60 us) or one pass late (neutral) measured no better; not kept.
    auto rel_stmt = [](const std::string& val) {
        return std::string("      if (a.sys_scope) { __threadfence_system(); asm volatile(\"st.release.sys.global.u32 [%0], %1;\" :: \"l\"(a.progress + a.prog_off + BID_), \"r\"((unsigned int)(") +
               val + ")) : \"memory\"); }\n" +
               "      else asm volatile(\"st.release.gpu.global.u32 [%0], %1;\" :: \"l\"(a.progress + a.prog_off + BID_), \"r\"((unsigned int)(" +
               val + ")) : \"memory\");\n";
    };
    // the release waits for the CTA's outstanding stores: issue it from the warp with
    // the least region-A work so that wait does not delay the next pass's critical path
    int rel_warp = 0;
    {
        long long best = -1;
        for (int w = 0; w < G; ++w) {
            long long c = 0;
            for (const auto& ph : sa.phases)
                for (int id : ph[static_cast<size_t>(w)]) c += g.tasks[static_cast<size_t>(id)].cost;
            if (best < 0 || c < best) { best = c; rel_warp = w; }
        }
        if (knob("EMTB200_CG_RELWARP", 1) == 0) rel_warp = 0;
    }
    const std::string release =
        std::string("    if (a.progress != nullptr && threadIdx.x == ") + std::to_string(32 * rel_warp) + ") {\n" +
        rel_stmt("step + 1") + "    }\n";
    if (!merge_ab) o << code_b;
    o << dmma_block << code_c;
    if (dok_mode) {
        // divergence (exec.cpp:229-237): rows only AND a NaN-safe predicate; the
        // failing node index (the lowest) is found in the cold path
        std::ostringstream tb;
        for (int i = 0; i < s.nodes; ++i) tb << (i ? "," : "") << g.off(s.v_base + i);
        if (s.nodes == 0) tb << "0";
        o << "    if (__syncthreads_or(!dok && live)) {\n"
          << "      const int kVoff[" << std::max(1, s.nodes) << "] = {" << tb.str() << "};\n"
          << "      if (warp == 0 && live) serr[lane] = 0x7fffffff;\n"
          << "      __syncthreads();\n"
          << "      if (warp == 0 && live) {\n"
          << "        for (int i = 0; i < " << s.nodes << "; ++i) if (!(fabs(LD(kVoff[i])) <= a.div_limit)) { bad = i; break; }\n"
          << "        if (bad != 0x7fffffff) { serr[lane] = bad; a.lane_err[4*gl] = 7; a.lane_err[4*gl+1] = step; a.lane_err[4*gl+2] = bad; a.lane_err[4*gl+3] = "
          << g.solve_layer << "; }\n"
          // no divergence: some row's quotient was below the Markstein bound or zero
          // (the other causes of !dok). Zero is exact (x is never -0 here); a nonzero
          // quotient below 2^-900 leaves a node voltage in (0, 2^-899): stop the launch
          << (lctx.divguard == 1
                  ? "        else { for (int i = 0; i < " + std::to_string(s.nodes) + "; ++i) { const double v_ = fabs(LD(kVoff[i])); "
                    "if (v_ < 0x1p-899 && v_ != 0.0) { bad = i; break; } }\n"
                    "          if (bad != 0x7fffffff) { serr[lane] = bad; a.lane_err[4*gl] = 66; a.lane_err[4*gl+1] = step; a.lane_err[4*gl+2] = bad; a.lane_err[4*gl+3] = " +
                        std::to_string(g.solve_layer) + "; } }\n"
                  : lctx.divguard == 3
                  ? "        else { bad = -1; serr[lane] = -1; a.lane_err[4*gl] = 66; a.lane_err[4*gl+1] = step; a.lane_err[4*gl+2] = -1; a.lane_err[4*gl+3] = " +
                        std::to_string(g.solve_layer) + "; }\n"
                  : std::string())
          << "      }\n"
          << "      if (__syncthreads_or(warp == 0 && live && serr[lane] != 0x7fffffff)) { FAILPUB(); return; }\n"
          << "    }\n"
          << "    if (false) {\n";
    } else {
        o << "    if (__syncthreads_or(bad != 0x7fffffff && live)) {\n"
          << "      if (bad != 0x7fffffff) atomicMin(&serr[lane], bad);\n"
          << "      __syncthreads();\n"
          << "      if (warp == 0 && live && serr[lane] != 0x7fffffff) { a.lane_err[4*gl] = 7; a.lane_err[4*gl+1] = step; a.lane_err[4*gl+2] = serr[lane]; a.lane_err[4*gl+3] = "
          << g.solve_layer << "; }\n"
          << "      FAILPUB(); return;\n";
    }
    o      << "    }\n";
    o << release;
    o << "  }\n";
    // save the resident state back to the arena (+ slots derived from it)
    o << "  __syncthreads();\n"
      << "  if (live) {\n"
;
    if (slcopy) {
        std::vector<std::pair<std::string, std::string>> it;
        for (int q : wb_q)
            it.push_back({"A[(size_t)" + std::to_string(g.hot_slots[static_cast<size_t>(q)]) + " * W_]",
                          "S[" + std::to_string(static_cast<long long>(q) * LPC) + "]"});
        o << warp_copies(it, G, "    ");
    } else {
        o << "    _Pragma(\"unroll 8\") for (int j = warp; j < " << wb_q.size() << "; j += " << G
          << ") { const int q = kWbQ[j]; A[(size_t)kHot[q - 1] * W_] = S[q * " << LPC << "]; }\n";
    }
    if (lu_smem) {
        o << "    _Pragma(\"unroll 8\") for (int q = warp; q < " << s.l_col.size() << "; q += " << G << ") A[(size_t)(" << s.l << " + q) * W_] = S[("
          << g.l_base_smem << " + q) * " << LPC << "];\n";
        o << "    _Pragma(\"unroll 8\") for (int q = warp; q < " << s.u_col.size() << "; q += " << G << ") A[(size_t)(" << s.u << " + q) * W_] = S[("
          << g.u_base_smem << " + q) * " << LPC << "];\n";
    }
    if (g.lu_shared) {
        std::vector<std::pair<std::string, std::string>> it;
        const size_t nl = s.l_col.size(), nu = s.u_col.size();
        for (size_t q = 0; q < nl; ++q) it.push_back({"A[(size_t)" + std::to_string(s.l + static_cast<long long>(q)) + " * W_]", "SH[" + std::to_string(q) + "]"});
        for (size_t q = 0; q < nu; ++q)
            it.push_back({"A[(size_t)" + std::to_string(s.u + static_cast<long long>(q)) + " * W_]", "SH[" + std::to_string(nl + q) + "]"});
        o << warp_copies(it, G, "    ");
    }
    o << "    if (a.nsteps > 0) {\n";
    if (slcopy) {
        std::vector<std::pair<std::string, std::string>> it;
        for (size_t q = 0; q < dslot.size(); ++q)
            it.push_back({"A[(size_t)" + std::to_string(dslot[q]) + " * W_]",
                          dconst[q] < 0 ? std::string("0.0") : "C[(size_t)" + std::to_string(dconst[q]) + " * W_]"});
        for (size_t q = 0; q < cslot.size(); ++q) {
            const std::string h = chot[q] < 0 ? std::string("0.0") : "S[" + std::to_string(static_cast<long long>(chot[q]) * LPC) + "]";
            it.push_back({"A[(size_t)" + std::to_string(cslot[q]) + " * W_]", csign[q] > 0 ? h : "-" + h});
        }
        if (g.chg_flag)
            for (int x : g.chg_slots) it.push_back({"A[(size_t)" + std::to_string(x) + " * W_]", "0.0"});
        o << warp_copies(it, G, "      ");
    } else {
        o << "      _Pragma(\"unroll 8\") for (int q = warp; q < " << dslot.size() << "; q += " << G << ") A[(size_t)kDerSlot[q] * W_] = kDerConst[q] < 0 ? 0.0 : C[(size_t)kDerConst[q] * W_];\n"
          << "      _Pragma(\"unroll 8\") for (int q = warp; q < " << cslot.size() << "; q += " << G << ") { const double h = kConHot[q] < 0 ? 0.0 : S[kConHot[q] * " << LPC << "]; "
          << "A[(size_t)kConSlot[q] * W_] = kConSign[q] > 0 ? h : -h; }\n"
          << "      _Pragma(\"unroll 8\") for (int q = warp; q < " << (g.chg_flag ? g.chg_slots.size() : 0) << "; q += " << G << ") A[(size_t)kChgSlot[q] * W_] = 0.0;\n";
    }
    if (slcopy) {  // one independent statement per line: spread over the warps
        std::vector<std::string> ln;
        std::istringstream fin(g.emit_lazy_finalize());
        for (std::string l; std::getline(fin, l);) ln.push_back(l);
        if (!ln.empty()) {
            o << "      switch (warp) {\n";
            for (int w = 0; w < G; ++w) {
                if (static_cast<size_t>(w) >= ln.size()) break;
                o << "      case " << w << ": {\n";
                for (size_t q = static_cast<size_t>(w); q < ln.size(); q += static_cast<size_t>(G)) o << ln[q] << "\n";
                o << "      } break;\n";
            }
            o << "      }\n";
        }
    } else {
        o << "      if (warp == " << (G - 1) << ") {\n" << g.emit_lazy_finalize() << "      }\n";
    }
    o
      << "    }\n"
      << "  }\n"
      << "}\n";

    if (!g.tab_ck.empty()) {
        // per-launch table of the AC source values m*cos(w t + p): the same expression,
        // operands and time base as the inline form (bit-identical), computed once per
        // (pass, source[, lane]) instead of inside every lane group's instruction stream.
        // Row = one pass: shared sources, then per-lane sources x W_ lanes.
        const int ns = g.tab_shared();
        o << "extern \"C\" __global__ void emt_src_kernel(double* tab, int step0, int nsteps, const double* __restrict__ ctab) {\n"
          << "  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;\n"
          << "  if (i >= (long long)nsteps * NSRC_) return;\n"
          << "  const int it = (int)(i / NSRC_); const int col = (int)(i - (long long)it * NSRC_);\n"
          << "  const double t = (double)(step0 + it + 1) * " << lit(s.dt) << ";\n"
          << "  int j = col; long long ln = 0;\n"
          << "  if (col >= " << ns << ") { j = " << ns << " + (col - " << ns << ") / (int)W_; ln = (col - " << ns << ") % W_; }\n"
          << "  const double* C = ctab + ln; (void)C;\n"
          << "  double v = 0.0;\n  switch (j) {\n";
        for (size_t j = 0; j < g.tab_ck.size(); ++j)
            o << "    case " << j << ": { const double m_ = " << g.C(g.tab_ck[j][0]) << ", w_ = " << g.C(g.tab_ck[j][1])
              << ", p_ = " << g.C(g.tab_ck[j][2]) << "; v = w_ == 0.0 ? m_ : m_ * emt_libm_cos(w_ * t + p_); } break;\n";
        o << "  }\n  tab[i] = v;\n}\n";
    }
    out.source = o.str();
    if (zterm && zmode == 2)
        for (size_t q = out.source.find("LD(0)"); q != std::string::npos; q = out.source.find("LD(0)", q + 5))
            out.source.replace(q, 5, "(0.0)");
    out.warps = G;
    out.lpc = LPC;
    out.smem_bytes = smem;
    out.hot_slots = nhot;
    out.lu_smem = lu_smem ? 1 : 0;
    out.phases_a = static_cast<int>(sa.phases.size());
    out.phases_b = static_cast<int>(sb.phases.size());
    out.tasks = static_cast<int>(nt);
    long work = 0;
    for (const Task& t : g.tasks) work += t.cost;
    std::ostringstream sum;
    sum << (straight ? "straight " : "compact ") << "lpc=" << LPC << " tasks=" << nt << " segments=" << segs_total << " hot=" << nhot << " lu_smem=" << lu_smem << (g.lu_shared ? " lu=shared" : "") << " smem=" << smem
        << " const=" << const_bytes << " phasesA=" << sa.phases.size() << " phasesB=" << sb.phases.size() << " warps=" << G
        << " est_span=" << static_cast<long>(span_a + span_b + span_c) << " est_work=" << work
        << (g.dmma ? " solve=dmma(G^-1 " + std::to_string(s.dim) + "x" + std::to_string(s.dim) + ")" : std::string(opt.tensor_solve ? " solve=lu(shared-G ineligible)" : ""));
    out.summary = sum.str() + dev_knob_note();
    return true;
}

}  // namespace emtb200

// =============================================================================
// Task-SIMT kernel: one CTA per scenario lane, one THREAD per task.
//
// The lane-SIMT kernel above puts 32 scenario lanes on the 32 threads of a warp
// and gives every warp its own straight-line instruction stream; with only a
// few hundred lanes it runs on a few dozen SMs and each step costs the full
// instruction latency of one lane's DAG. Here a warp instead executes up to 32
// *tasks of one kind* of one lane at once (a "wave"): task operands come from a
// per-thread record table in global memory (L1-resident after the first step,
// coalesced), lane state lives in the CTA's shared memory at one double per
// arena slot, and a batch of W lanes is W small CTAs spread over every SM.
// Waves are the DAG levels of each region split by kind; the list scheduler
// places them on warps with bar.sync phases, __syncwarp between the waves of
// one warp. Every task keeps the reference's floating-point operation order.
// =============================================================================

namespace emtb200 {
namespace {

struct TsCode {
    const char* body;  // per-thread code; RI(n) = int record field n, KS(c) = S index of const c,
                       // TA(j)/TB(j) = term j fields, NTERM = this thread's term count, NT_ = wave max
};

// Record layout per task: f fields, then ck (as S indices), then [n_terms, (a, b) pairs].
const char* ts_body(int kind) {
    switch (kind) {
        case K_IND: return "const double vs = S[RI(1)] - S[RI(0)]; const double ip = S[RI(2)]; const double g = S[KS(0)]; S[RI(3)] = ip + g * vs;";
        case K_CAP: return "const double vs = S[RI(1)] - S[RI(0)]; const double ip = S[RI(2)]; const double g = S[KS(0)]; S[RI(3)] = -ip - g * vs;";
        case K_SRL: return "const double vs = S[RI(1)] - S[RI(0)]; const double ip = S[RI(2)]; const double g = S[KS(0)]; const double d = S[KS(1)]; S[RI(3)] = d * ip + g * vs;";
        case K_VSRC: return "const double g = S[KS(0)]; const double m = S[KS(1)]; const double w = S[KS(2)]; const double p = S[KS(3)]; S[RI(0)] = g * (w == 0.0 ? m : m * emt_libm_cos(w * t + p));";
        case K_ISRC: return "const double m = S[KS(0)]; const double w = S[KS(1)]; const double p = S[KS(2)]; S[RI(0)] = w == 0.0 ? m : m * emt_libm_cos(w * t + p);";
        case K_CSRC: return "const double k = S[KS(0)]; const double x = S[RI(1)]; S[RI(0)] = k * x;";
        case K_FINC: return "const double vs = S[RI(3)] - S[RI(2)]; const double h = S[RI(1)]; const double g = S[KS(0)]; S[RI(0)] = g * vs + h;";
        case K_FINS: return "const double vs = S[RI(3)] - S[RI(2)]; const double h = S[RI(1)]; const double g = S[RI(4)]; S[RI(0)] = g * vs + h;";
        case K_GAIN: return "const double x = S[RI(1)]; const double u = RI(2) ? -x : x; S[RI(0)] = S[KS(0)] * u;";
        case K_INTEG: return "const double x = S[RI(1)]; const double u = RI(4) ? -x : x; const double s0 = S[RI(2)]; const double s1 = S[RI(3)]; const double c0 = S[KS(0)]; const double y = s0 + c0 * (u + s1); S[RI(2)] = y; S[RI(3)] = u; S[RI(0)] = y;";
        case K_LAG: return "const double x = S[RI(1)]; const double u = RI(4) ? -x : x; const double s0 = S[RI(2)]; const double s1 = S[RI(3)]; const double c0 = S[KS(0)]; const double c1 = S[KS(1)]; const double y = c0 * s0 + c1 * (u + s1); S[RI(2)] = y; S[RI(3)] = u; S[RI(0)] = y;";
        case K_PI: return "const double x = S[RI(1)]; const double u = RI(4) ? -x : x; const double s0 = S[RI(2)]; const double s1 = S[RI(3)]; const double kp = S[KS(0)]; const double ki = S[KS(1)]; const double y = s0 + ki * (u + s1); const double o = kp * u + y; S[RI(2)] = y; S[RI(3)] = u; S[RI(0)] = o;";
        case K_LIM: return "const double x = S[RI(1)]; const double u = RI(2) ? -x : x; const double lo = S[KS(0)]; const double hi = S[KS(1)]; S[RI(0)] = u < lo ? lo : (u > hi ? hi : u);";
        case K_CMP: return "const double x0 = S[RI(1)]; const double x1 = S[RI(2)]; const double p = RI(3) ? -x0 : x0; const double q = RI(4) ? -x1 : x1; S[RI(0)] = p >= q ? 1.0 : 0.0;";
        case K_CONST: return "S[RI(0)] = S[KS(0)];";
        case K_DELAY: return "const double x = S[RI(1)]; S[RI(0)] = RI(2) ? -x : x;";
        case K_REC: return "a.waves[((size_t)(a.row0 + it) * NCH + RI(0)) * W_ + gl] = S[RI(1)];";
        case K_LATCH: return "S[RI(1)] = S[RI(0)];";
        case K_BERG: return "const double vs = S[RI(1)] - S[RI(0)]; const double hp = S[RI(2)]; const double y2 = S[KS(0)]; const double c1 = S[KS(1)]; const double c0 = S[KS(2)]; const int K = (int)S[KS(3)]; const long long pl = (long long)S[KS(4)]; const long long pr = (long long)S[KS(5)] - a.ring_lo; const int L = RI(4); "
                            "const double be = y2 * vs + hp; int q1 = (step + 1 - K) % L; if (q1 < 0) q1 += L; const int q0 = q1 == 0 ? L - 1 : q1 - 1; "
                            "const double b1 = __ldcg(a.ring + pl * a.ring_cols + pr + q1); const double b0 = __ldcg(a.ring + pl * a.ring_cols + pr + q0); "
                            "S[RI(2)] = -(c1 * b1 + c0 * b0); const int w = step % L; A[(size_t)(RI(3) + w) * W_] = be; a.ring[(LB_ + gl) * a.ring_cols + (RI(3) - a.ring_lo) + w] = be;";
        default: return nullptr;
    }
}

struct Wave {
    int region = 0, level = 0, kind = 0;
    std::vector<int> tasks;
    int nf = 0, nc = 0, maxt = 0, rec_base = 0;
};

}  // namespace

bool generate_tsimt(const Schedule& s, const std::vector<double>& ctab, int lanes, const CodegenOptions& opt,
                    GeneratedKernel& out, Failure& fail) {
    Gen g(s, ctab, lanes, opt);
    g.ls = 1;
    g.unit = 1;
    g.classify();
    int facts = 0;
    g.emit_all(facts);
    if (facts != 1) {
        fail = {13, "", "schedule must hold exactly one FactorizeSystem process"};
        return false;
    }
    CodegenOptions o2 = opt;
    o2.smem_budget = 200 * 1024;
    o2.lu_in_smem = true;
    g.opt = o2;
    bool lu_smem = false;
    size_t smem = 0;
    if (!g.assign_hot(lu_smem, smem) || !lu_smem) {
        fail = {13, "", "task-SIMT: lane state exceeds shared memory"};
        return false;
    }
    g.emit_all(facts);
    const size_t nt = g.tasks.size();
    const std::vector<std::vector<int>> deps = task_deps(g.tasks);

    // every constant a task reads gets an S slot, loaded from the lane's column once per launch
    const int const_base = g.smem_slots();
    std::map<int, int> cidx;
    std::vector<int> cslots;
    for (const Task& t : g.tasks)
        for (int k : t.ck)
            if (!cidx.count(k)) {
                cidx[k] = const_base + static_cast<int>(cslots.size());
                cslots.push_back(k);
            }
    const int nslots = const_base + static_cast<int>(cslots.size());

    // ASAP levels per region; waves = (region, level, kind, #f, #ck, #terms class) chunks of 32
    std::vector<int> level(nt, 0);
    for (size_t i = 0; i < nt; ++i)
        for (int d : deps[i])
            if (g.tasks[static_cast<size_t>(d)].region == g.tasks[i].region)
                level[i] = std::max(level[i], level[static_cast<size_t>(d)] + 1);
    std::map<std::tuple<int, int, int, int, int>, std::vector<int>> groups;
    for (size_t i = 0; i < nt; ++i) {
        const Task& t = g.tasks[i];
        groups[{t.region, level[i], t.kind, static_cast<int>(t.f.size()), static_cast<int>(t.ck.size())}].push_back(static_cast<int>(i));
    }
    std::vector<Wave> waves;
    for (auto& kv : groups) {
        std::vector<int> ids = kv.second;
        std::stable_sort(ids.begin(), ids.end(), [&](int a, int b) {
            return g.tasks[static_cast<size_t>(a)].terms.size() < g.tasks[static_cast<size_t>(b)].terms.size();
        });
        for (size_t q = 0; q < ids.size(); q += 32) {
            Wave w;
            w.region = std::get<0>(kv.first);
            w.level = std::get<1>(kv.first);
            w.kind = std::get<2>(kv.first);
            w.nf = std::get<3>(kv.first);
            w.nc = std::get<4>(kv.first);
            w.tasks.assign(ids.begin() + static_cast<long>(q), ids.begin() + static_cast<long>(std::min(ids.size(), q + 32)));
            for (int id : w.tasks) w.maxt = std::max(w.maxt, static_cast<int>(g.tasks[static_cast<size_t>(id)].terms.size()));
            waves.push_back(std::move(w));
        }
    }
    // wave DAG (for the warp scheduler) + cost model (cycles)
    std::vector<int> wave_of(nt, -1);
    for (size_t w = 0; w < waves.size(); ++w)
        for (int id : waves[w].tasks) wave_of[static_cast<size_t>(id)] = static_cast<int>(w);
    std::vector<Task> wt(waves.size());
    std::vector<std::vector<int>> wdeps(waves.size());
    for (size_t w = 0; w < waves.size(); ++w) {
        std::set<int> d;
        for (int id : waves[w].tasks)
            for (int x : deps[static_cast<size_t>(id)])
                if (wave_of[static_cast<size_t>(x)] != static_cast<int>(w)) d.insert(wave_of[static_cast<size_t>(x)]);
        wdeps[w].assign(d.begin(), d.end());
        const int k = waves[w].kind;
        int c = 90;  // record + operand loads, compute, store
        if (k == K_VSRC || k == K_ISRC) c = 260;
        if (k == K_SW) c = 110 + 12 * waves[w].nc;
        if (k == K_GATHER || k == K_SUM) c = 80 + 10 * waves[w].maxt;
        if (k == K_FWD) c = 80 + 18 * waves[w].maxt;
        if (k == K_BWD) c = 130 + 18 * waves[w].maxt;
        if (k == K_BERG) c = 200;
        wt[w].cost = c;
        wt[w].region = waves[w].region;
    }
    const int G = std::max(1, std::min(opt.warps, 32));
    std::vector<int> wa, wb;
    for (size_t w = 0; w < waves.size(); ++w) (waves[w].region == 0 ? wa : wb).push_back(static_cast<int>(w));
    double span_a = 0, span_b = 0;
    const Sched sa = schedule_region(wt, wa, wdeps, G, &span_a);
    const Sched sb = schedule_region(wt, wb, wdeps, G, &span_b);

    // record table: per wave, field-major [field][32 threads]
    std::vector<int> rec;
    for (Wave& w : waves) {
        w.rec_base = static_cast<int>(rec.size());
        const int nfield = w.nf + w.nc + (w.maxt > 0 ? 1 + 2 * w.maxt : 0);
        rec.resize(rec.size() + static_cast<size_t>(nfield) * 32, 0);
        for (size_t j = 0; j < w.tasks.size(); ++j) {
            const Task& t = g.tasks[static_cast<size_t>(w.tasks[j])];
            auto put = [&](int field, int v) { rec[static_cast<size_t>(w.rec_base + field * 32) + j] = v; };
            for (int f = 0; f < w.nf; ++f) put(f, t.f[static_cast<size_t>(f)]);
            for (int c = 0; c < w.nc; ++c) put(w.nf + c, cidx[t.ck[static_cast<size_t>(c)]]);
            if (w.maxt > 0) {
                put(w.nf + w.nc, static_cast<int>(t.terms.size()));
                for (size_t q = 0; q < t.terms.size(); ++q) {
                    put(w.nf + w.nc + 1 + 2 * static_cast<int>(q), t.terms[q].first);
                    put(w.nf + w.nc + 2 + 2 * static_cast<int>(q), t.terms[q].second);
                }
            }
        }
    }

    auto ks = [](std::string text, int nf) {
        for (size_t pos; (pos = text.find("KS(")) != std::string::npos;)
            text.replace(pos, 3, "RI(" + std::to_string(nf) + " + ");
        return text;
    };
    auto wave_code = [&](const Wave& w) {
        std::ostringstream c;
        c << "      if (lane < " << w.tasks.size() << ") { const int rb = " << w.rec_base << " + lane; ";
        const int tb = w.nf + w.nc;
        if (w.kind == K_GATHER || w.kind == K_SUM) {
            c << "const int n = RI(" << tb << "); double acc = 0.0; ";
            for (int j = 0; j < w.maxt; ++j)
                c << "if (" << j << " < n) { const double v = S[RI(" << tb + 1 + 2 * j << ")]; acc = acc + (RI(" << tb + 2 + 2 * j
                  << ") ? -v : v); } ";
            c << "S[RI(0)] = acc;";
        } else if (w.kind == K_FWD || w.kind == K_BWD) {
            c << "const int n = RI(" << tb << "); double x = S[RI(0)]; ";
            for (int j = 0; j < w.maxt; ++j)
                c << "if (" << j << " < n) x = x - S[RI(" << tb + 1 + 2 * j << ")] * S[RI(" << tb + 2 + 2 * j << ")]; ";
            if (w.kind == K_BWD) c << "x = x / S[RI(1)]; dok = dok & (fabs(x) <= dlim); ";
            c << "S[RI(0)] = x;";
        } else if (w.kind == K_SW) {
            c << "int now = S[KS(2)] != 0.0 ? 1 : 0; ";
            for (int j = 3; j < w.nc; ++j) c << "if (t >= S[KS(" << j << ")]) now ^= 1; ";
            c << "const double chg = (double)now != S[RI(0)] ? 1.0 : 0.0; ";
            if (!g.chg_flag) c << "S[RI(1)] = chg; ";
            c << "S[RI(0)] = (double)now; S[RI(2)] = now != 0 ? S[KS(0)] : S[KS(1)]; "
              << "if (chg != 0.0) { wflag = 1; " << (g.chg_flag ? "needS[0] = 1; " : "")
              << "if (a.events) { const int e = atomicAdd(a.n_events, 1); if (e < a.max_events) { a.events[3*e] = step; "
                 "a.events[3*e+1] = gl; a.events[3*e+2] = RI(3); } } }";
        } else {
            const char* b = ts_body(w.kind);
            if (b == nullptr) return std::string("#error unsupported task kind\n");
            c << b;
        }
        c << " }\n";
        return ks(c.str(), w.nf);
    };
    auto region_code = [&](const Sched& sc) {
        std::ostringstream rc;
        rc << "    switch (warp) {\n";
        for (int wp = 0; wp < G; ++wp) {
            rc << "    case " << wp << ": {\n";
            for (size_t p = 0; p < sc.phases.size(); ++p) {
                if (p > 0) rc << "      BAR();\n";
                bool first = true;
                for (int wid : sc.phases[p][static_cast<size_t>(wp)]) {
                    if (!first) rc << "      __syncwarp();\n";
                    first = false;
                    rc << wave_code(waves[static_cast<size_t>(wid)]);
                }
            }
            rc << "    } break;\n";
        }
        rc << "    }\n";
        return rc.str();
    };
    const std::string code_a = region_code(sa);
    const std::string code_b = region_code(sb);

    std::ostringstream o;
    const int nhot = static_cast<int>(g.hot_slots.size());
    const int NTH = 32 * G;
    o << "// generated by emtb200 codegen (task-SIMT): " << s.nodes << " nodes, " << s.comps << " components, " << lanes
      << " lanes (one CTA each), " << G << " warps, " << nt << " tasks, " << waves.size() << " waves\n";
    o << "#define W_ " << static_cast<long long>(lanes) << "LL\n#define NCH " << s.channel_slot.size() << "\n#define LB_ "
      << opt.lane_begin << "LL\n";
    o << libm_cos_prelude();
    o << "struct KArgs { double* arena; const double* ctab; double* waves; unsigned char* refac; int* lane_err;\n"
      << "  int* events; int* n_events; int max_events; int step0; int nsteps; int row0; double div_limit;\n"
      << "  double* ring; long long ring_lo; long long ring_cols; unsigned int* progress; int min_k; int nblocks; long long* prof; const double* srctab;\n"
      << "  int prog_off; int sys_scope; };\n";
    auto garr = [&](const char* name, const std::vector<int>& v) {
        o << "__device__ const int " << name << "[" << std::max<size_t>(1, v.size()) << "] = {";
        for (size_t q = 0; q < v.size(); ++q) o << (q ? "," : "") << v[q];
        if (v.empty()) o << "0";
        o << "};\n";
    };
    garr("kRec", rec);
    std::vector<int> hot_arena(g.hot_slots.begin() + 1, g.hot_slots.end());
    garr("kHot", hot_arena);
    std::set<int> late_slots;  // written by the launch-end lazy finalize: not copied back (see generate_kernel)
    for (const auto& kv : g.alias_of) late_slots.insert(kv.first);
    for (int c : g.lazy_fin) late_slots.insert(s.finalize[5 * static_cast<size_t>(c)]);
    std::vector<int> wb_q;
    for (int q = 0; q + 1 < nhot; ++q)
        if (!late_slots.count(g.hot_slots[static_cast<size_t>(q) + 1])) wb_q.push_back(q + 1);
    garr("kWbQ", wb_q);
    garr("kCst", cslots);
    std::vector<int> dslot, dconst, cslot, chot, csign;
    for (int x = 0; x < s.extent; ++x) {
        if (g.cls[static_cast<size_t>(x)] == kDerived) {
            dslot.push_back(x);
            dconst.push_back(g.derived_const[static_cast<size_t>(x)]);
        } else if (g.cls[static_cast<size_t>(x)] == kContrib) {
            const int h = g.contrib_h[static_cast<size_t>(x)];
            cslot.push_back(x);
            chot.push_back(g.cls[static_cast<size_t>(h)] == kHot ? g.hot_index[static_cast<size_t>(h)] : -1);
            csign.push_back(g.contrib_sign[static_cast<size_t>(x)]);
        }
    }
    garr("kDerSlot", dslot);
    garr("kDerConst", dconst);
    garr("kConSlot", cslot);
    garr("kConHot", chot);
    garr("kConSign", csign);
    garr("kChgSlot", g.chg_flag ? g.chg_slots : std::vector<int>());
    o << "#define BAR() asm volatile(\"barrier.sync 0;\" ::: \"memory\")\n"
      << "#define RI(n) __ldg(kRec + rb + (n) * 32)\n";
    std::string refac = g.emit_refactor();
    for (size_t pos; (pos = refac.find("needS[lane]")) != std::string::npos;) refac.replace(pos, 11, "needS[0]");
    std::set<int> written_a;
    for (const Task& t : g.tasks)
        if (t.region == 0)
            for (int w : t.writes) written_a.insert(w);
    const int min_blocks = std::max(1, knob("EMTB200_TS_MINBLOCKS", 4));
    o << "extern \"C\" __global__ void __launch_bounds__(" << NTH << ", " << min_blocks << ") emt_ts_kernel(const KArgs a) {\n"
      << "  extern __shared__ double S[];\n"
      << "  const int lane = threadIdx.x & 31; const int warp = threadIdx.x >> 5;\n"
      << "  const int gl = blockIdx.x; const bool live = true; (void)live;\n"
      << "  double* __restrict__ A = a.arena + gl;\n"
      << "  const double* __restrict__ C = a.ctab + gl; (void)C;\n"
      << "  int* needS = (int*)(S + " << nslots << ");\n"
      << "  for (int q = threadIdx.x; q < " << nhot - 1 << "; q += " << NTH << ") S[q + 1] = A[(size_t)kHot[q] * W_];\n"
      << "  for (int q = threadIdx.x; q < " << s.l_col.size() << "; q += " << NTH << ") S[" << g.l_base_smem << " + q] = A[(size_t)("
      << s.l << " + q) * W_];\n"
      << "  for (int q = threadIdx.x; q < " << s.u_col.size() << "; q += " << NTH << ") S[" << g.u_base_smem << " + q] = A[(size_t)("
      << s.u << " + q) * W_];\n"
      << "  for (int q = threadIdx.x; q < " << cslots.size() << "; q += " << NTH << ") S[" << const_base << " + q] = __ldg(C + (size_t)kCst[q] * W_);\n"
      << "  if (threadIdx.x == 0) { S[0] = 0.0; needS[0] = 0; }\n"
      << "  __syncthreads();\n"
      << "  const double dlim = a.div_limit; (void)dlim;\n"
      << "  for (int it = 0; it < a.nsteps; ++it) {\n"
      << "    const int step = a.step0 + it;\n"
      << "    const double t = (double)(step + 1) * " << lit(s.dt) << ";\n"
      << "    int wflag = 0; int srow = -1; bool dok = true;\n"
      << "    (void)t; (void)srow; (void)step; (void)dok;\n"
      << "    if (threadIdx.x == 0) { ";
    for (int x : s.watch)
        if (x >= 0 && !written_a.count(x)) o << "wflag |= (" << g.R(x) << " != 0.0); ";
    o << "}\n" << code_a
      << "    if (__syncthreads_or(wflag)) {\n"
      << "      if (threadIdx.x == 0) {\n" << refac
      << "        a.refac[a.row0 + it] = 1;\n"
      << "      }\n"
      << "      if (__syncthreads_or(srow >= 0)) {\n"
      << "        if (threadIdx.x == 0 && srow >= 0) { a.lane_err[4*gl] = 8; a.lane_err[4*gl+1] = step; a.lane_err[4*gl+2] = srow; a.lane_err[4*gl+3] = "
      << g.fact_layer << "; }\n"
      << "        return;\n"
      << "      }\n"
      << "    }\n"
      << code_b;
    std::ostringstream tb;
    for (int i = 0; i < s.nodes; ++i) tb << (i ? "," : "") << g.off(s.v_base + i);
    if (s.nodes == 0) tb << "0";
    o << "    if (__syncthreads_or(!dok)) {\n"
      << "      const int kVoff[" << std::max(1, s.nodes) << "] = {" << tb.str() << "};\n"
      << "      if (threadIdx.x == 0) { int bad = 0; for (int i = 0; i < " << s.nodes << "; ++i) if (!(fabs(S[kVoff[i]]) <= a.div_limit)) { bad = i; break; }\n"
      << "        a.lane_err[4*gl] = 7; a.lane_err[4*gl+1] = step; a.lane_err[4*gl+2] = bad; a.lane_err[4*gl+3] = " << g.solve_layer << "; }\n"
      << "      return;\n"
      << "    }\n"
      << "  }\n"
      << "  __syncthreads();\n"
      << "  for (int j = threadIdx.x; j < " << wb_q.size() << "; j += " << NTH << ") { const int q = kWbQ[j]; A[(size_t)kHot[q - 1] * W_] = S[q]; }\n"
      << "  for (int q = threadIdx.x; q < " << s.l_col.size() << "; q += " << NTH << ") A[(size_t)(" << s.l << " + q) * W_] = S["
      << g.l_base_smem << " + q];\n"
      << "  for (int q = threadIdx.x; q < " << s.u_col.size() << "; q += " << NTH << ") A[(size_t)(" << s.u << " + q) * W_] = S["
      << g.u_base_smem << " + q];\n"
      << "  if (a.nsteps > 0) {\n"
      << "    for (int q = threadIdx.x; q < " << dslot.size() << "; q += " << NTH << ") A[(size_t)kDerSlot[q] * W_] = kDerConst[q] < 0 ? 0.0 : C[(size_t)kDerConst[q] * W_];\n"
      << "    for (int q = threadIdx.x; q < " << cslot.size() << "; q += " << NTH << ") { const double h = kConHot[q] < 0 ? 0.0 : S[kConHot[q]]; "
      << "A[(size_t)kConSlot[q] * W_] = kConSign[q] > 0 ? h : -h; }\n"
      << "    for (int q = threadIdx.x; q < " << (g.chg_flag ? g.chg_slots.size() : 0) << "; q += " << NTH << ") A[(size_t)kChgSlot[q] * W_] = 0.0;\n"
      << "    if (threadIdx.x == 0) {\n" << g.emit_lazy_finalize() << "    }\n"
      << "  }\n"
      << "}\n";
    out.source = o.str();
    out.name = "emt_ts_kernel";
    out.warps = G;
    out.smem_bytes = static_cast<size_t>(nslots) * sizeof(double) + 16;
    out.hot_slots = nhot;
    out.lu_smem = 1;
    out.phases_a = static_cast<int>(sa.phases.size());
    out.phases_b = static_cast<int>(sb.phases.size());
    out.tasks = static_cast<int>(nt);
    std::ostringstream sum;
    sum << "task-simt tasks=" << nt << " waves=" << waves.size() << " slots=" << nslots << " smem=" << out.smem_bytes
        << " rec=" << rec.size() * 4 << "B phasesA=" << sa.phases.size() << " phasesB=" << sb.phases.size() << " warps=" << G
        << " est_span=" << static_cast<long>(span_a + span_b);
    out.summary = sum.str() + dev_knob_note();
    return true;
}

}  // namespace emtb200
