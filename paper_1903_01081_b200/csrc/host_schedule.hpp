// Host-side view of a compiled schedule (the boundary data of SURVEY.md §8(b))
// and the device planner's inputs: lu_symbolic fill and triangular level sets.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace emtb200 {

// KernelId (/root/reference/proj/include/emtgrid/kernels.hpp:36-59).
enum Kernel : int {
    kNortonResistor = 0,
    kNortonInductor,
    kNortonCapacitor,
    kNortonSeriesRL,
    kNortonVoltageSource,
    kNortonCurrentSource,
    kNortonControlledSource,
    kNortonSwitch,
    kInjectionPair,
    kFactorizeSystem,
    kSolveSystem,
    kCtlGain,
    kCtlSum,
    kCtlIntegrator,
    kCtlFirstOrderLag,
    kCtlLimiter,
    kCtlPiController,
    kCtlComparator,
    kCtlConstant,
    kCtlDelay,
    // Extension (no reference counterpart): lossless Bergeron
    // transmission-line end. par = [2/Zc, 1-f, f, K, peer_lane, peer_ring, L],
    // state = ring[L]; see oracle/emt_oracle.c case K_BERG for the semantics.
    kNortonBergeron,
    kKernelCount
};

struct Failure {
    int code = 0;  // 1 + emtgrid::ErrorCode
    std::string where, message;
};

struct Proc {
    int id = -1, kind = 0, code = 0, lane = 0;
    int out = -1, out_len = 0, out2 = -1, state = -1, state_len = 0, par = -1, par_len = 0;
    int in_base = 0, in_count = 0;
};

/// Parsed `.cgmsched` v1 text (record grammar: /root/reference/proj/docs/schedule_format.md).
struct Schedule {
    std::string profile;
    int width = 1, steps = 0, nodes = 0, comps = 0, blocks = 0, extent = 0, consts = 0, layers = 0;
    double dt = 0.0;
    std::vector<double> const_table;  // consts * width, slot-major
    std::vector<std::string> channel_names;
    std::vector<int> channel_slot;
    std::vector<int> latch_live, latch_shadow;

    // SolverTables (/root/reference/proj/include/emtgrid/schedule.hpp:22-39)
    int dim = 0, l_nnz = 0, u_nnz = 0, v_base = -1, matrix = -1, l = -1, u = -1, scratch = -1,
        dirty = -1, fcount = -1;
    std::vector<int> row_ptr{0}, col_idx;
    std::vector<int> mentry_ptr{0}, mentry_slot;
    std::vector<double> mentry_sign;
    std::vector<int> gather_ptr{0}, gather_slot;
    std::vector<int> finalize;  // 5 per component: i g h va vb
    std::vector<int> watch;

    // processes flattened layer-major, groups in order (decode, proj/src/exec.cpp:31-62)
    std::vector<Proc> procs;
    std::vector<int> layer_begin;  // layers + 1
    std::vector<int> port_slot;
    std::vector<double> port_sign;

    // lu_symbolic (/root/reference/proj/src/sparse.cpp:44-77)
    std::vector<int> l_row_ptr, l_col, u_row_ptr, u_col;
};

/// Parses the text; returns false and fills `fail` (MalformedDocument) on error.
bool parse_schedule(const char* text, Schedule& s, Failure& fail);

/// Identity-ordering symbolic LU exactly as the reference computes it.
void lu_symbolic(Schedule& s);

/// Level sets of the unit-lower forward sweep and the upper backward sweep:
/// rows in one level only depend on rows of earlier levels, so each level is
/// one parallel wave while every row keeps the reference's operation order.
void triangular_levels(const Schedule& s, std::vector<int>& fwd_ptr, std::vector<int>& fwd_rows,
                       std::vector<int>& bwd_ptr, std::vector<int>& bwd_rows);

}  // namespace emtb200
