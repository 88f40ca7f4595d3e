// emtgrid::execute_b200 — the reference-side binding of libemtb200.
//
// This is the translation unit a maintainer adds to emtgrid (proj/src/exec_b200.cpp),
// compiled here against the reference's own headers by `make -C oracle integ`
// together with reference_b200.patch (Strategy::Device, the "b200" profile,
// execute_task / run_vse dispatch). Contract: interpret()'s
// (/root/reference/proj/include/emtgrid/exec.hpp:27-30, proj/src/exec.cpp:350-383):
// same waveforms (bit for bit), same exceptions (code, where, message), ExecStats
// filled with the device-timed step loop.
#include <cstring>
#include <string>
#include <vector>

#include <cstdlib>

#include "emt_b200.h"
#include "emtgrid/codegen.hpp"
#include "emtgrid/exec.hpp"

namespace emtgrid {

namespace {

[[noreturn]] void rethrow(emt_status rc) {
    // status = 1 + ErrorCode for reference errors (include/emt_b200.h, common.hpp:11-33);
    // emt_last_error() = "<where>: <message>" ("row 1: zero pivot ...", "node index 3: ...")
    const std::string detail = emt_last_error();
    const std::size_t colon = detail.find(": ");
    const std::string where = colon == std::string::npos ? std::string() : detail.substr(0, colon);
    const std::string msg = colon == std::string::npos ? detail : detail.substr(colon + 2);
    if (rc >= 1 && rc <= static_cast<int>(ErrorCode::IoError) + 1) fail(static_cast<ErrorCode>(rc - 1), where, msg);
    fail(ErrorCode::ToolchainUnavailable, "b200", detail);  // CUDA / device failures
}

}  // namespace

WaveformSet execute_b200(const ScheduleProgram& s, const Eigen::VectorXd& initial, int steps,
                         const ExecOptions& options, int device) {
    if (steps < 0) fail(ErrorCode::NonPositiveInput, "steps", "negative step count");
    const std::string text = s.serialize();  // proj/src/schedule.cpp:335-411
    const int cols = static_cast<int>(s.channels.size()) * s.width;
    WaveformSet w;
    for (const auto& ch : s.channels) w.channels.push_back(ch.first);
    w.width = s.width;
    w.time.assign(static_cast<std::size_t>(steps), 0.0);
    std::vector<double> rows(static_cast<std::size_t>(steps) * static_cast<std::size_t>(cols));
    emt_exec_options o{};
    o.divergence_limit = options.divergence_limit;
    o.warmup_steps = options.warmup_steps;
    emt_config cfg{};
    cfg.device = device;
    emt_exec_stats st{};
    const emt_status rc = emt_interpret(text.c_str(), initial.data(), initial.size(), steps, &o, &cfg, rows.data(),
                                        w.time.data(), &st);
    if (rc != EMT_OK) rethrow(rc);
    w.values.resize(steps, cols);  // WaveformSet values: rows = steps, cols = channels*width
    for (int r = 0; r < steps; ++r)
        for (int c = 0; c < cols; ++c)
            w.values(r, c) = rows[static_cast<std::size_t>(r) * static_cast<std::size_t>(cols) + static_cast<std::size_t>(c)];
    if (options.stats != nullptr) {
        options.stats->factor_count = st.factor_count;
        options.stats->measured_seconds = st.measured_seconds;
        options.stats->measured_steps = st.measured_steps;
    }
    return w;
}

std::string emit_source_sm100a(const ScheduleProgram& s) {
    // emit_source's "sm100a" dialect (proj/src/codegen.cpp:84 + reference_b200.patch)
    const std::string text = s.serialize();
    char* src = nullptr;
    const emt_status rc = emt_emit_program(text.c_str(), &src);
    if (rc != EMT_OK) rethrow(rc);
    std::string out(src);
    emt_free(src);
    return out;
}

std::vector<std::string> sm100a_flags() {
    return {"-x", "cu", "-gencode", "arch=compute_100a,code=sm_100a", "-fmad=false", "-std=c++17", "-O3", "-w"};
}

}  // namespace emtgrid
