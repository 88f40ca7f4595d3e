// Schedule -> specialised sm_100a kernel source (the code generator of
// SURVEY.md §8(f).1; the reference's C++ emitter is proj/src/codegen.cpp:84-230).
//
// The generated kernel runs 32 scenario lanes per CTA, one lane per thread
// (SIMT over scenarios: every thread executes the same straight-line code on
// its own lane's state), and splits the per-step work of those lanes across
// `warps` warps (warp-specialised partitions separated by CTA barriers).
// Every arena slot index, every lane-invariant constant and every sparse-LU
// index is baked into the instruction stream as an immediate.
#pragma once

#include <string>
#include <vector>

#include "host_schedule.hpp"

namespace emtb200 {

struct CodegenOptions {
    int warps = 4;                  // warps per CTA (work partitions of one 32-lane group)
    bool auto_warps = false;        // warps chosen by the engine: the generator may pick its own count
    size_t smem_budget = 227 * 1024;  // bytes of dynamic shared memory per CTA
    bool lu_in_smem = true;         // keep L/U factors on chip when they fit
    int mode = 0;                   // 0 auto, 1 straight-line tasks, 2 compact per-type loops
    long long lane_begin = 0;       // first batch lane of the engine (line-end peer lanes are batch indices)
    bool exact_division = false;    // IEEE fallback branch in every backward row (EMT_FLAG_EXACT_DIVISION)
    bool tensor_solve = false;      // shared-G batches: V = G^-1 I on the FP64 tensor cores (not bit-exact)
    int lanes_per_cta = 0;          // scenario lanes per CTA (32, 16 or 8; 0 = EMTB200_CG_LPC or 32)
};

struct GeneratedKernel {
    std::string source;
    std::string name = "emt_cg_kernel";
    int warps = 4;
    size_t smem_bytes = 0;
    int hot_slots = 0;      // arena slots resident in shared memory
    int lu_smem = 0;        // 1 when L/U live in shared memory
    int phases_a = 0, phases_b = 0;
    int tasks = 0;
    int nsrc = 0;           // AC source values tabulated per launch by emt_src_kernel (srctab)
    int lpc = 32;           // scenario lanes per CTA of the specialised kernel
    std::string summary;
};

/// `ctab` = consts x lanes constant table of the engine's lanes (slot-major);
/// a constant slot equal across all lanes becomes an immediate.
bool generate_kernel(const Schedule& s, const std::vector<double>& ctab, int lanes, const CodegenOptions& opt,
                     GeneratedKernel& out, Failure& fail);

/// Task-SIMT variant: one CTA per scenario lane, one thread per task of a
/// DAG wave (see codegen.cpp); `out.name` = "emt_ts_kernel", launch with
/// grid = lanes, block = 32 * out.warps, dynamic smem = out.smem_bytes.
bool generate_tsimt(const Schedule& s, const std::vector<double>& ctab, int lanes, const CodegenOptions& opt,
                    GeneratedKernel& out, Failure& fail);

/// The "sm100a" code-DB dialect (emit_program.cpp): a standalone CUDA program —
/// this schedule's specialised kernel plus a host main() with the "cpp" dialect's
/// CLI (--state --steps --out; exit 2 I/O, 3 singular, 4 divergence) and waveform text.
bool emit_program(const Schedule& s, const std::vector<double>& ctab, int lanes, std::string& out, Failure& fail);

}  // namespace emtb200
