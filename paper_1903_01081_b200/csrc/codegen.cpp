// Schedule -> specialised sm_100a kernel source. See codegen.hpp and DESIGN.md §4.
//
// Semantics are those of the reference's per-process kernels
// (Engine::run_proc, /root/reference/proj/src/exec.cpp:77-311, and the
// code-database templates proj/data/codedb/cpp/*.tpl); the generator turns the
// schedule's sequential process order into a dependency DAG of fine-grained
// tasks (one per Norton update, gather node, triangular-solve row, finalize
// component, control block, channel record, latch), then list-schedules the
// DAG onto the CTA's warps in barrier-separated phases. Within a task every
// floating-point operation keeps the reference's order (no FMA contraction:
// compiled with --fmad=false), so results stay bit-compatible.
#include "codegen.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <set>
#include <sstream>

namespace emtb200 {

namespace {

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

struct Task {
    std::string code;
    std::vector<int> reads, writes;  // arena slots (after contrib aliasing)
    int cost = 1;
    int region = 0;  // 0: before FactorizeSystem, 1: after
};

enum Cls { kNone = 0, kHot, kDerived, kContrib, kSolver, kGlobal };

struct Gen {
    const Schedule& s;
    const std::vector<double>& ct;
    int W;
    CodegenOptions opt;

    std::vector<int> cls;           // per arena slot
    std::vector<std::string> dexpr; // derived constant expression
    std::vector<int> derived_const; // const slot for derived g (-1: literal 0.0)
    std::vector<int> contrib_h, contrib_sign;
    std::vector<int> hot_index;
    std::vector<int> hot_slots;
    int l_base_smem = -1;  // hot index of L[0] when L/U are in smem
    int u_base_smem = -1;
    std::vector<Task> tasks;
    int fact_layer = 0, solve_layer = 0;

    Gen(const Schedule& sc, const std::vector<double>& c, int w, const CodegenOptions& o) : s(sc), ct(c), W(w), opt(o) {}

    bool invariant(int k) const {
        const double* row = ct.data() + static_cast<size_t>(k) * W;
        for (int l = 1; l < W; ++l)
            if (std::memcmp(&row[l], &row[0], sizeof(double)) != 0) return false;
        return true;
    }
    std::string C(int k) const {
        if (invariant(k)) return lit(ct[static_cast<size_t>(k) * W]);
        return "__ldg(C + " + std::to_string(static_cast<long long>(k) * W) + ")";
    }
    std::string R(int slot) const {
        if (slot < 0) return "(0.0)";
        switch (cls[static_cast<size_t>(slot)]) {
            case kDerived: return dexpr[static_cast<size_t>(slot)];
            case kContrib: {
                const std::string h = R(contrib_h[static_cast<size_t>(slot)]);
                return contrib_sign[static_cast<size_t>(slot)] > 0 ? h : "(-" + h + ")";
            }
            case kHot: return "S[" + std::to_string(hot_index[static_cast<size_t>(slot)] * 32) + "]";
            case kGlobal: return "A[" + std::to_string(static_cast<long long>(slot) * W) + "]";
            default: return "/*bad slot " + std::to_string(slot) + "*/(0.0)";
        }
    }
    // Writes to global-resident slots from clamped tail threads duplicate lane W-1
    // bit for bit (same inputs, same instruction), so they need no guard.
    std::string Wr(int slot) const {
        if (slot >= 0 && cls[static_cast<size_t>(slot)] == kGlobal)
            return "A[" + std::to_string(static_cast<long long>(slot) * W) + "]";
        return "S[" + std::to_string(hot_index[static_cast<size_t>(slot)] * 32) + "]";
    }
    int dep_slot(int slot) const {
        if (slot >= 0 && cls[static_cast<size_t>(slot)] == kContrib) return contrib_h[static_cast<size_t>(slot)];
        return slot;
    }
    std::string Lr(int k) const {
        if (l_base_smem >= 0) return "S[" + std::to_string((l_base_smem + k) * 32) + "]";
        return "A[" + std::to_string(static_cast<long long>(s.l + k) * W) + "]";
    }
    std::string Ur(int k) const {
        if (u_base_smem >= 0) return "S[" + std::to_string((u_base_smem + k) * 32) + "]";
        return "A[" + std::to_string(static_cast<long long>(s.u + k) * W) + "]";
    }
    std::string Lw(int k, const std::string& v) const {
        if (l_base_smem >= 0) return Lr(k) + " = " + v + ";";
        return "if (live) " + Lr(k) + " = " + v + ";";
    }
    std::string Uw(int k, const std::string& v) const {
        if (u_base_smem >= 0) return Ur(k) + " = " + v + ";";
        return "if (live) " + Ur(k) + " = " + v + ";";
    }

    // kern::source_value (proj/include/emtgrid/kernels.hpp:68-70)
    std::string source(int kmag, int kom, int kph) const {
        if (invariant(kom)) {
            if (ct[static_cast<size_t>(kom) * W] == 0.0) return C(kmag);
            return "(" + C(kmag) + " * cos(" + C(kom) + " * t + " + C(kph) + "))";
        }
        return "((" + C(kom) + ") == 0.0 ? " + C(kmag) + " : " + C(kmag) + " * cos(" + C(kom) + " * t + " + C(kph) + "))";
    }

    void classify() {
        const size_t n = static_cast<size_t>(s.extent);
        cls.assign(n, kNone);
        dexpr.assign(n, "");
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
        for (const Proc& p : s.procs) {
            if (p.code <= kNortonSwitch && p.code != kNortonSwitch && p.out >= 0) {
                cls[static_cast<size_t>(p.out)] = kDerived;
                if (p.code == kNortonCurrentSource || p.code == kNortonControlledSource) {
                    dexpr[static_cast<size_t>(p.out)] = "(0.0)";
                    derived_const[static_cast<size_t>(p.out)] = -1;
                } else {
                    dexpr[static_cast<size_t>(p.out)] = C(p.par);
                    derived_const[static_cast<size_t>(p.out)] = p.par;
                }
            }
            if ((p.code == kNortonResistor || p.code == kNortonSwitch) && p.out2 >= 0) {
                cls[static_cast<size_t>(p.out2)] = kDerived;
                dexpr[static_cast<size_t>(p.out2)] = "(0.0)";
                derived_const[static_cast<size_t>(p.out2)] = -1;
            }
            if (p.code == kInjectionPair && p.out >= 0 && p.in_count >= 1) {
                const int h = s.port_slot[static_cast<size_t>(p.in_base)];
                cls[static_cast<size_t>(p.out)] = kContrib;
                cls[static_cast<size_t>(p.out + 1)] = kContrib;
                contrib_h[static_cast<size_t>(p.out)] = h;
                contrib_sign[static_cast<size_t>(p.out)] = 1;
                contrib_h[static_cast<size_t>(p.out + 1)] = h;
                contrib_sign[static_cast<size_t>(p.out + 1)] = -1;
            }
        }
    }

    void add(Task&& t, int region) {
        t.region = region;
        tasks.push_back(std::move(t));
    }

    std::string sgn(double v) const { return lit(v); }

    // One non-singleton process: Engine::run_proc cases (exec.cpp:85-309).
    void emit_proc(const Proc& p, int region) {
        const int* in = s.port_slot.data() + p.in_base;
        const double* sg = s.port_sign.data() + p.in_base;
        auto IN = [&](int j) { return j < p.in_count ? in[j] : -1; };
        Task t;
        std::ostringstream o;
        auto reads = [&](std::initializer_list<int> sl) {
            for (int x : sl)
                if (x >= 0) t.reads.push_back(dep_slot(x));
        };
        switch (p.code) {
            case kNortonResistor:
                return;  // g, h are constants
            case kNortonInductor:
            case kNortonCapacitor:
            case kNortonSeriesRL: {
                reads({IN(0), IN(1), IN(2)});
                t.writes.push_back(p.out2);
                o << "{ const double vs = " << R(IN(1)) << " - " << R(IN(0)) << "; const double g = " << C(p.par) << "; ";
                if (p.code == kNortonInductor)
                    o << Wr(p.out2) << " = " << R(IN(2)) << " + g * vs; }";
                else if (p.code == kNortonCapacitor)
                    o << Wr(p.out2) << " = -" << R(IN(2)) << " - g * vs; }";
                else
                    o << Wr(p.out2) << " = " << C(p.par + 1) << " * " << R(IN(2)) << " + g * vs; }";
                t.cost = 8;
                break;
            }
            case kNortonVoltageSource: {
                t.writes.push_back(p.out2);
                o << "{ const double g = " << C(p.par) << "; " << Wr(p.out2) << " = g * "
                  << source(p.par + 1, p.par + 2, p.par + 3) << "; }";
                t.cost = invariant(p.par + 2) && ct[static_cast<size_t>(p.par + 2) * W] == 0.0 ? 3 : 90;
                break;
            }
            case kNortonCurrentSource: {
                t.writes.push_back(p.out2);
                o << Wr(p.out2) << " = " << source(p.par, p.par + 1, p.par + 2) << ";";
                t.cost = invariant(p.par + 1) && ct[static_cast<size_t>(p.par + 1) * W] == 0.0 ? 2 : 90;
                break;
            }
            case kNortonControlledSource: {
                if (p.in_count > 3) reads({IN(3)});
                t.writes.push_back(p.out2);
                o << Wr(p.out2) << " = " << C(p.par) << " * " << (p.in_count > 3 ? R(IN(3)) : std::string("(0.0)")) << ";";
                t.cost = 3;
                break;
            }
            case kNortonSwitch: {  // exec.cpp:151-165
                t.reads.push_back(p.state);
                t.writes.push_back(p.state);
                t.writes.push_back(p.state + 1);
                t.writes.push_back(p.out);
                o << "{ int now = " << C(p.par + 2) << " != 0.0 ? 1 : 0; ";
                for (int j = 3; j < p.par_len; ++j) o << "if (t >= " << C(p.par + j) << ") now ^= 1; ";
                o << "const double chg = (double)now != " << R(p.state) << " ? 1.0 : 0.0; "
                  << Wr(p.state + 1) << " = chg; " << Wr(p.state) << " = (double)now; " << Wr(p.out)
                  << " = now != 0 ? " << C(p.par) << " : " << C(p.par + 1) << "; "
                  << "if (chg != 0.0) { wflag = 1; if (live && a.events) { const int q = atomicAdd(a.n_events, 1); "
                  << "if (q < a.max_events) { a.events[3*q] = step; a.events[3*q+1] = gl; a.events[3*q+2] = " << p.id
                  << "; } } } }";
                t.cost = 8 + 2 * (p.par_len - 3);
                break;
            }
            case kInjectionPair:
                return;  // contrib slots alias +-h (exact negation)
            case kCtlGain:
                reads({IN(0)});
                t.writes.push_back(p.out);
                o << Wr(p.out) << " = " << C(p.par) << " * (" << sgn(sg[0]) << " * " << R(IN(0)) << ");";
                t.cost = 3;
                break;
            case kCtlSum: {
                o << "{ double acc = 0.0; ";
                for (int j = 0; j < p.in_count; ++j) {
                    reads({IN(j)});
                    o << "acc = acc + " << sgn(sg[j]) << " * " << R(IN(j)) << "; ";
                }
                t.writes.push_back(p.out);
                o << Wr(p.out) << " = acc; }";
                t.cost = 2 + 3 * p.in_count;
                break;
            }
            case kCtlIntegrator:
            case kCtlFirstOrderLag:
            case kCtlPiController: {
                reads({IN(0), p.state, p.state + 1});
                t.writes.push_back(p.state);
                t.writes.push_back(p.state + 1);
                t.writes.push_back(p.out);
                const std::string s0 = R(p.state), s1 = R(p.state + 1);
                o << "{ const double u = " << sgn(sg[0]) << " * " << R(IN(0)) << "; ";
                if (p.code == kCtlIntegrator) {
                    o << "const double y = " << s0 << " + " << C(p.par) << " * (u + " << s1 << "); " << Wr(p.state)
                      << " = y; " << Wr(p.state + 1) << " = u; " << Wr(p.out) << " = y; }";
                } else if (p.code == kCtlFirstOrderLag) {
                    o << "const double y = " << C(p.par) << " * " << s0 << " + " << C(p.par + 1) << " * (u + " << s1
                      << "); " << Wr(p.state) << " = y; " << Wr(p.state + 1) << " = u; " << Wr(p.out) << " = y; }";
                } else {
                    o << "const double y = " << s0 << " + " << C(p.par + 1) << " * (u + " << s1 << "); "
                      << Wr(p.state) << " = y; " << Wr(p.state + 1) << " = u; " << Wr(p.out) << " = " << C(p.par)
                      << " * u + y; }";
                }
                t.cost = 8;
                break;
            }
            case kCtlLimiter:
                reads({IN(0)});
                t.writes.push_back(p.out);
                o << "{ const double u = " << sgn(sg[0]) << " * " << R(IN(0)) << "; const double lo = " << C(p.par)
                  << ", hi = " << C(p.par + 1) << "; " << Wr(p.out) << " = u < lo ? lo : (u > hi ? hi : u); }";
                t.cost = 4;
                break;
            case kCtlComparator:
                reads({IN(0), IN(1)});
                t.writes.push_back(p.out);
                o << Wr(p.out) << " = " << sgn(sg[0]) << " * " << R(IN(0)) << " >= " << sgn(sg[1]) << " * " << R(IN(1))
                  << " ? 1.0 : 0.0;";
                t.cost = 4;
                break;
            case kCtlConstant:
                t.writes.push_back(p.out);
                o << Wr(p.out) << " = " << C(p.par) << ";";
                t.cost = 1;
                break;
            case kCtlDelay:
                reads({IN(0)});
                t.writes.push_back(p.out);
                o << Wr(p.out) << " = " << sgn(sg[0]) << " * " << R(IN(0)) << ";";
                t.cost = 2;
                break;
            default:
                return;
        }
        t.code = o.str();
        add(std::move(t), region);
    }

    // SolveSystem (exec.cpp:205-239): gather, lu_solve rows, finalize.
    void emit_solve(int region) {
        const int v = s.v_base;
        for (int node = 0; node < s.nodes; ++node) {
            Task t;
            std::ostringstream o;
            o << "{ double acc = 0.0; ";
            for (int q = s.gather_ptr[static_cast<size_t>(node)]; q < s.gather_ptr[static_cast<size_t>(node) + 1]; ++q) {
                const int slot = s.gather_slot[static_cast<size_t>(q)];
                t.reads.push_back(dep_slot(slot));
                o << "acc = acc + " << R(slot) << "; ";
            }
            o << Wr(v + node) << " = acc; }";
            t.writes.push_back(v + node);
            t.cost = 2 + 2 * static_cast<int>(t.reads.size());
            t.code = o.str();
            add(std::move(t), region);
        }
        if (s.nodes > 0) {
            for (int i = 0; i < s.dim; ++i) {  // forward, unit L (sparse.cpp:152-160)
                const int lb = s.l_row_ptr[static_cast<size_t>(i)], le = s.l_row_ptr[static_cast<size_t>(i) + 1];
                if (lb == le) continue;
                Task t;
                std::ostringstream o;
                o << "{ double x = " << R(v + i) << "; ";
                t.reads.push_back(v + i);
                for (int k = lb; k < le; ++k) {
                    const int c = s.l_col[static_cast<size_t>(k)];
                    t.reads.push_back(v + c);
                    o << "x = x - " << Lr(k) << " * " << R(v + c) << "; ";
                }
                o << Wr(v + i) << " = x; }";
                t.writes.push_back(v + i);
                t.cost = 2 + 3 * (le - lb);
                t.code = o.str();
                add(std::move(t), region);
            }
            for (int i = s.dim - 1; i >= 0; --i) {  // backward (sparse.cpp:161-171) + divergence (exec.cpp:229-237)
                const int ub = s.u_row_ptr[static_cast<size_t>(i)], ue = s.u_row_ptr[static_cast<size_t>(i) + 1];
                Task t;
                std::ostringstream o;
                o << "{ double x = " << R(v + i) << "; ";
                t.reads.push_back(v + i);
                for (int k = ub + 1; k < ue; ++k) {
                    const int c = s.u_col[static_cast<size_t>(k)];
                    t.reads.push_back(v + c);
                    o << "x = x - " << Ur(k) << " * " << R(v + c) << "; ";
                }
                o << "x = x / " << Ur(ub) << "; " << Wr(v + i) << " = x; "
                  << "if (!(fabs(x) <= a.div_limit) && " << i << " < bad) bad = " << i << "; }";
                t.writes.push_back(v + i);
                t.cost = 24 + 3 * (ue - ub - 1);
                t.code = o.str();
                add(std::move(t), region);
            }
        }
        for (int c = 0; c < s.comps; ++c) {  // i = g (v_b - v_a) + h
            const int* f = s.finalize.data() + 5 * c;
            Task t;
            t.reads = {dep_slot(f[1]), dep_slot(f[2])};
            if (f[3] >= 0) t.reads.push_back(f[3]);
            if (f[4] >= 0) t.reads.push_back(f[4]);
            t.writes.push_back(f[0]);
            std::ostringstream o;
            o << Wr(f[0]) << " = " << R(f[1]) << " * (" << R(f[4]) << " - " << R(f[3]) << ") + " << R(f[2]) << ";";
            t.cost = 6;
            t.code = o.str();
            add(std::move(t), region);
        }
    }

    // Classifies the arena slots the step loop touches: the most accessed go to
    // shared memory ([slot][32 lanes]) until the budget is spent, the rest stay
    // in the global arena ([slot][W], L2-resident, coalesced across lanes).
    void assign_hot(bool& lu_smem, size_t& smem_bytes) {
        std::map<int, long> uses;
        for (const Task& t : tasks) {
            for (int x : t.reads)
                if (x >= 0 && cls[static_cast<size_t>(x)] == kNone) uses[x] += 1;
            for (int x : t.writes)
                if (x >= 0 && cls[static_cast<size_t>(x)] == kNone) uses[x] += 1;
        }
        for (int x : s.watch)
            if (x >= 0 && cls[static_cast<size_t>(x)] == kNone) uses[x] += 0;
        for (int x : s.channel_slot)
            if (x >= 0 && cls[static_cast<size_t>(x)] == kNone) uses[x] += 1;
        for (size_t q = 0; q < s.latch_live.size(); ++q) {
            uses[s.latch_live[q]] += 1;
            uses[s.latch_shadow[q]] += 1;
        }
        for (int x : s.mentry_slot)
            if (x >= 0 && cls[static_cast<size_t>(x)] == kNone) uses[x] += 0;
        std::vector<std::pair<long, int>> order;
        for (const auto& kv : uses)
            if (cls[static_cast<size_t>(kv.first)] == kNone) order.push_back({-kv.second, kv.first});
        std::sort(order.begin(), order.end());
        const size_t per_slot = 32 * sizeof(double);
        const size_t fixed = 32 * sizeof(int);
        const size_t cap = opt.smem_budget > fixed ? (opt.smem_budget - fixed) / per_slot : 0;
        for (const auto& pr : order) {
            const int x = pr.second;
            if (hot_slots.size() < cap) {
                cls[static_cast<size_t>(x)] = kHot;
                hot_index[static_cast<size_t>(x)] = static_cast<int>(hot_slots.size());
                hot_slots.push_back(x);
            } else {
                cls[static_cast<size_t>(x)] = kGlobal;
            }
        }
        const size_t base = hot_slots.size() * per_slot + fixed;
        const size_t lu = (s.l_col.size() + s.u_col.size()) * per_slot;
        lu_smem = opt.lu_in_smem && base + lu <= opt.smem_budget;
        smem_bytes = base + (lu_smem ? lu : 0);
        if (lu_smem) {
            l_base_smem = static_cast<int>(hot_slots.size());
            u_base_smem = l_base_smem + static_cast<int>(s.l_col.size());
        }
    }

    // Refactorization (FactorizeSystem, exec.cpp:175-204; lu_factor, sparse.cpp:79-145)
    // as straight-line code for one lane per thread; lanes whose watch slots
    // are clear skip it (their factors would be recomputed bit-identically).
    std::string emit_refactor() const {
        std::ostringstream o;
        o << "      bool need = false;\n";
        for (int x : s.watch) o << "      need = need || (" << R(x) << " != 0.0);\n";
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
        // last row touching each scratch column (final scratch contents, sparse.cpp:92-131)
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
                o << "          u" << k << " = w" << c << "; " << Uw(k, "u" + std::to_string(k)) << "\n";
            }
            for (int c : cols)
                if (last_row[static_cast<size_t>(c)] == i)
                    o << "          if (live) A[" << static_cast<long long>(s.scratch + c) * W << "] = w" << c << ";\n";
            o << "          if (!(fabs(u" << ub << ") > " << lit(1e-12) << " * mx)) { srow = " << i << "; goto fact_done; }\n";
            o << "        }\n";
        }
        for (int x : s.watch) o << "        " << Wr(x) << " = 0.0;\n";
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
                      const std::vector<std::vector<int>>& deps, int G, double* makespan) {
    const long kBarrier = 60;
    Sched out;
    const size_t n = ids.size();
    if (n == 0) {
        if (makespan) *makespan = 0;
        return out;
    }
    std::map<int, int> local;  // task id -> position
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
    std::vector<long> finish(n, 0);
    for (size_t i = 0; i < n; ++i) missing[i] = static_cast<int>(pred[i].size());
    std::set<std::pair<long, int>> ready;  // (-bottom, i)
    for (size_t i = 0; i < n; ++i)
        if (missing[i] == 0) ready.insert({-bottom[i], static_cast<int>(i)});
    std::vector<long> T(static_cast<size_t>(G), 0);
    std::vector<std::vector<std::pair<int, int>>> plan(static_cast<size_t>(G));  // (task, phase)
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
            long waiting = 0;  // ready work only a barrier can expose to the idle warp
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
        long start = T[static_cast<size_t>(pick_w)];
        T[static_cast<size_t>(pick_w)] = start + cost[i];
        finish[i] = T[static_cast<size_t>(pick_w)];
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
    // drop empty trailing phases
    while (out.phases.size() > 1) {
        bool empty = true;
        for (const auto& v : out.phases.back()) empty = empty && v.empty();
        if (!empty) break;
        out.phases.pop_back();
    }
    if (makespan) *makespan = static_cast<double>(*std::max_element(T.begin(), T.end()));
    return out;
}

void emit_phases(std::ostringstream& o, const Sched& sc, const std::vector<Task>& tasks, const char* indent,
                 bool barrier_after_last) {
    for (size_t p = 0; p < sc.phases.size(); ++p) {
        bool first = true;
        for (size_t w = 0; w < sc.phases[p].size(); ++w) {
            if (sc.phases[p][w].empty()) continue;
            o << indent << (first ? "if" : "else if") << " (warp == " << w << ") {\n";
            for (int id : sc.phases[p][w]) o << indent << "  " << tasks[static_cast<size_t>(id)].code << "\n";
            o << indent << "}\n";
            first = false;
        }
        if (p + 1 < sc.phases.size() || barrier_after_last) o << indent << "__syncthreads();\n";
    }
}

}  // namespace

bool generate_kernel(const Schedule& s, const std::vector<double>& ctab, int lanes, const CodegenOptions& opt,
                     GeneratedKernel& out, Failure& fail) {
    Gen g(s, ctab, lanes, opt);
    g.classify();

    // Sequential process order -> tasks; the FactorizeSystem process splits regions.
    int region = 0;
    for (int L = 0; L < s.layers; ++L) {
        for (int k = s.layer_begin[static_cast<size_t>(L)]; k < s.layer_begin[static_cast<size_t>(L) + 1]; ++k) {
            const Proc& p = s.procs[static_cast<size_t>(k)];
            if (p.code == kFactorizeSystem) {
                if (region != 0) {
                    fail = {13, "", "schedule has more than one FactorizeSystem process"};
                    return false;
                }
                region = 1;
                g.fact_layer = L;
                continue;
            }
            if (p.code == kSolveSystem) {
                g.solve_layer = L;
                g.emit_solve(region);
                continue;
            }
            g.emit_proc(p, region);
        }
    }
    if (region == 0) {
        fail = {13, "", "schedule has no FactorizeSystem process"};
        return false;
    }
    // record (exec.cpp:313-321) then latch (exec.cpp:323-329)
    for (size_t ch = 0; ch < s.channel_slot.size(); ++ch) {
        Task t;
        const int slot = s.channel_slot[ch];
        if (slot >= 0) t.reads.push_back(g.dep_slot(slot));
        t.cost = 3;
        t.code = "if (live) a.waves[((size_t)(a.row0 + it) * " + std::to_string(s.channel_slot.size()) + " + " +
                 std::to_string(ch) + ") * " + std::to_string(lanes) + " + gl] = " + g.R(slot) + ";";
        // R() needs hot classification: patch after assign_hot (placeholder marker)
        t.code = "@REC" + std::to_string(ch) + "@";
        g.add(std::move(t), 1);
    }
    for (size_t q = 0; q < s.latch_live.size(); ++q) {
        Task t;
        t.reads.push_back(s.latch_live[q]);
        t.writes.push_back(s.latch_shadow[q]);
        t.cost = 2;
        t.code = "@LAT" + std::to_string(q) + "@";
        g.add(std::move(t), 1);
    }

    bool lu_smem = false;
    size_t smem = 0;
    // Hot classification needs every task's slot sets; codes emitted before it
    // referenced R()/Wr() of slots not yet indexed, so regenerate them now.
    g.assign_hot(lu_smem, smem);
    if (smem > opt.smem_budget) {
        fail = {13, "", "arena hot set (" + std::to_string(smem) + " B) exceeds shared memory budget"};
        return false;
    }
    {
        std::vector<Task> saved = std::move(g.tasks);
        g.tasks.clear();
        region = 0;
        for (int L = 0; L < s.layers; ++L) {
            for (int k = s.layer_begin[static_cast<size_t>(L)]; k < s.layer_begin[static_cast<size_t>(L) + 1]; ++k) {
                const Proc& p = s.procs[static_cast<size_t>(k)];
                if (p.code == kFactorizeSystem) { region = 1; continue; }
                if (p.code == kSolveSystem) { g.emit_solve(region); continue; }
                g.emit_proc(p, region);
            }
        }
        for (size_t ch = 0; ch < s.channel_slot.size(); ++ch) {
            Task t;
            const int slot = s.channel_slot[ch];
            if (slot >= 0) t.reads.push_back(g.dep_slot(slot));
            t.cost = 3;
            t.code = "if (live) a.waves[((size_t)(a.row0 + it) * " + std::to_string(s.channel_slot.size()) + " + " +
                     std::to_string(ch) + ") * " + std::to_string(lanes) + " + gl] = " + g.R(slot) + ";";
            g.add(std::move(t), 1);
        }
        for (size_t q = 0; q < s.latch_live.size(); ++q) {
            Task t;
            t.reads.push_back(s.latch_live[q]);
            t.writes.push_back(s.latch_shadow[q]);
            t.cost = 2;
            t.code = g.Wr(s.latch_shadow[q]) + " = " + g.R(s.latch_live[q]) + ";";
            g.add(std::move(t), 1);
        }
        (void)saved;
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
    std::vector<int> ids_a, ids_b;
    for (size_t i = 0; i < nt; ++i) (g.tasks[i].region == 0 ? ids_a : ids_b).push_back(static_cast<int>(i));
    const int G = std::max(1, std::min(opt.warps, 32));
    double span_a = 0, span_b = 0;
    const Sched sa = schedule_region(g.tasks, ids_a, deps, G, &span_a);
    const Sched sb = schedule_region(g.tasks, ids_b, deps, G, &span_b);

    // ---- source
    std::ostringstream o;
    const int nhot = static_cast<int>(g.hot_slots.size());
    o << "// generated by emtb200 codegen: " << s.nodes << " nodes, " << s.comps << " components, " << s.layers
      << " layers, " << lanes << " lanes, " << G << " warps\n";

    o << "struct KArgs { double* arena; const double* ctab; double* waves; unsigned char* refac; int* lane_err;\n"
      << "  int* events; int* n_events; int max_events; int step0; int nsteps; int row0; double div_limit; };\n";
    o << "__device__ const int kHot[" << std::max(1, nhot) << "] = {";
    for (int q = 0; q < nhot; ++q) o << (q ? "," : "") << g.hot_slots[static_cast<size_t>(q)];
    if (nhot == 0) o << "0";
    o << "};\n";
    // derived + contrib slots materialised at save time
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
    auto arr = [&](const char* name, const std::vector<int>& v) {
        o << "__device__ const int " << name << "[" << std::max<size_t>(1, v.size()) << "] = {";
        for (size_t q = 0; q < v.size(); ++q) o << (q ? "," : "") << v[q];
        if (v.empty()) o << "0";
        o << "};\n";
    };
    arr("kDerSlot", dslot);
    arr("kDerConst", dconst);
    arr("kConSlot", cslot);
    arr("kConHot", chot);
    arr("kConSign", csign);
    const long long Wl = lanes;
    o << "extern \"C\" __global__ void __launch_bounds__(" << 32 * G << ", 1) emt_cg_kernel(const KArgs a) {\n"
      << "  extern __shared__ double sm[];\n"
      << "  const int lane = threadIdx.x & 31; const int warp = threadIdx.x >> 5;\n"
      << "  const int graw = blockIdx.x * 32 + lane; const bool live = graw < " << Wl << ";\n"
      << "  const int gl = live ? graw : " << (Wl - 1) << ";\n"
      << "  double* __restrict__ S = sm + lane;\n"
      << "  int* serr = (int*)(sm + " << (static_cast<long long>(nhot) + (lu_smem ? static_cast<long long>(s.l_col.size() + s.u_col.size()) : 0)) * 32 << ");\n"
      << "  double* __restrict__ A = a.arena + gl;\n"
      << "  const double* __restrict__ C = a.ctab + gl;\n"
      << "  (void)C;\n"
      << "  for (int q = warp; q < " << nhot << "; q += " << G << ") S[q * 32] = A[(size_t)kHot[q] * " << Wl << "];\n";
    if (lu_smem) {
        o << "  for (int q = warp; q < " << s.l_col.size() << "; q += " << G << ") S[(" << g.l_base_smem << " + q) * 32] = A[(size_t)("
          << s.l << " + q) * " << Wl << "];\n";
        o << "  for (int q = warp; q < " << s.u_col.size() << "; q += " << G << ") S[(" << g.u_base_smem << " + q) * 32] = A[(size_t)("
          << s.u << " + q) * " << Wl << "];\n";
    }
    o << "  if (warp == 0) serr[lane] = 0x7fffffff;\n"
      << "  __syncthreads();\n"
      << "  int it = 0;\n"
      << "  for (; it < a.nsteps; ++it) {\n"
      << "    const int step = a.step0 + it;\n"
      << "    const double t = (double)(step + 1) * " << lit(s.dt) << ";\n"
      << "    int wflag = 0; int bad = 0x7fffffff; int srow = -1;\n"
      << "    (void)t; (void)bad; (void)srow;\n";
    // Watch slots not rewritten by region-A tasks this step (the dirty flag, or
    // slots set after the factorization point last step) are checked up front;
    // switch updates raise wflag inside their own tasks.
    {
        std::set<int> written_a;
        for (const Task& t : g.tasks)
            if (t.region == 0)
                for (int w : t.writes) written_a.insert(w);
        o << "    if (warp == 0) { ";
        for (int x : s.watch)
            if (x >= 0 && !written_a.count(x)) o << "wflag |= (" << g.R(x) << " != 0.0); ";
        o << "}\n";
    }
    emit_phases(o, sa, g.tasks, "    ", false);
    o << "    if (__syncthreads_or(wflag)) {\n"
      << "      if (warp == 0) {\n"
      << g.emit_refactor()
      << "        if (lane == 0) a.refac[a.row0 + it] = 1;\n"
      << "      }\n"
      << "      if (__syncthreads_or(srow >= 0 && live)) {\n"
      << "        if (warp == 0 && live && srow >= 0) { a.lane_err[4*gl] = 8; a.lane_err[4*gl+1] = step; a.lane_err[4*gl+2] = srow; a.lane_err[4*gl+3] = "
      << g.fact_layer << "; }\n"
      << "        return;\n"
      << "      }\n"
      << "    }\n";
    emit_phases(o, sb, g.tasks, "    ", false);
    o << "    if (__syncthreads_or(bad != 0x7fffffff && live)) {\n"
      << "      if (bad != 0x7fffffff) atomicMin(&serr[lane], bad);\n"
      << "      __syncthreads();\n"
      << "      if (warp == 0 && live && serr[lane] != 0x7fffffff) { a.lane_err[4*gl] = 7; a.lane_err[4*gl+1] = step; a.lane_err[4*gl+2] = serr[lane]; a.lane_err[4*gl+3] = "
      << g.solve_layer << "; }\n"
      << "      return;\n"
      << "    }\n"
      << "  }\n";
    // save
    o << "  __syncthreads();\n"
      << "  if (live) {\n"
      << "    for (int q = warp; q < " << nhot << "; q += " << G << ") A[(size_t)kHot[q] * " << Wl << "] = S[q * 32];\n";
    if (lu_smem) {
        o << "    for (int q = warp; q < " << s.l_col.size() << "; q += " << G << ") A[(size_t)(" << s.l << " + q) * " << Wl
          << "] = S[(" << g.l_base_smem << " + q) * 32];\n";
        o << "    for (int q = warp; q < " << s.u_col.size() << "; q += " << G << ") A[(size_t)(" << s.u << " + q) * " << Wl
          << "] = S[(" << g.u_base_smem << " + q) * 32];\n";
    }
    o << "    if (a.nsteps > 0) {\n"
      << "      for (int q = warp; q < " << dslot.size() << "; q += " << G << ") A[(size_t)kDerSlot[q] * " << Wl
      << "] = kDerConst[q] < 0 ? 0.0 : C[(size_t)kDerConst[q] * " << Wl << "];\n"
      << "      for (int q = warp; q < " << cslot.size() << "; q += " << G << ") { const double h = kConHot[q] < 0 ? 0.0 : S[kConHot[q] * 32]; "
      << "A[(size_t)kConSlot[q] * " << Wl << "] = kConSign[q] > 0 ? h : -h; }\n"
      << "    }\n"
      << "  }\n"
      << "}\n";

    out.source = o.str();
    out.warps = G;
    out.smem_bytes = smem;
    out.hot_slots = nhot;
    out.lu_smem = lu_smem ? 1 : 0;
    out.phases_a = static_cast<int>(sa.phases.size());
    out.phases_b = static_cast<int>(sb.phases.size());
    out.tasks = static_cast<int>(nt);
    std::ostringstream sum;
    long work = 0;
    for (const Task& t : g.tasks) work += t.cost;
    sum << "tasks=" << nt << " hot=" << nhot << " lu_smem=" << lu_smem << " smem=" << smem << " phasesA=" << sa.phases.size()
        << " phasesB=" << sb.phases.size() << " warps=" << G << " est_span=" << static_cast<long>(span_a + span_b)
        << " est_work=" << work;
    out.summary = sum.str();
    return true;
}

}  // namespace emtb200
