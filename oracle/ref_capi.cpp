// C entry points over the UNMODIFIED reference library (test infrastructure).
//
// oracle/Makefile compiles the reference sources where they lie under
// /root/reference/proj/src together with this file into
// oracle/_ref/libemtref.so. Only tests/, __graft_entry__.smoke() and the
// CPU-baseline leg of bench.py load it, as the checker / reference arm.
//
// Every function forwards to the reference's own public API:
//   compile_task      proj/src/pipeline.cpp:5-18   (+ ScheduleProgram::serialize,
//                                                   serialize_state; proj/src/schedule.cpp:335,582)
//   interpret         proj/src/exec.cpp:350-383
//   execute_parallel  proj/src/exec.cpp:385-500
//   run_serial        proj/src/kernels.cpp:687-902
//   gen_scale_case    proj/src/bench.cpp:54-117
// Status codes are 0 on success, else 1 + emtgrid::ErrorCode
// (proj/include/emtgrid/common.hpp:11-33).
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <json.hpp>

#include "emtgrid/bench.hpp"
#include "emtgrid/kernels.hpp"
#include "emtgrid/pipeline.hpp"

using namespace emtgrid;

namespace {

char* dup(const std::string& s) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.data(), s.size());
    p[s.size()] = '\0';
    return p;
}

void put_err(char* err, int err_len, const std::string& msg) {
    if (err == nullptr || err_len <= 0) return;
    std::snprintf(err, static_cast<std::size_t>(err_len), "%s", msg.c_str());
}

template <typename F>
int guarded(char* err, int err_len, F&& f) {
    try {
        f();
        return 0;
    } catch (const Error& e) {
        put_err(err, err_len, std::string(e.what()) + "|where=" + e.where());
        return 1 + static_cast<int>(e.code());
    } catch (const std::exception& e) {
        put_err(err, err_len, e.what());
        return 1000;
    }
}

void copy_waves(const WaveformSet& w, double* waves, double* time) {
    const Eigen::Index rows = w.values.rows();
    const Eigen::Index cols = w.values.cols();
    if (waves != nullptr) {
        for (Eigen::Index r = 0; r < rows; ++r) {
            for (Eigen::Index c = 0; c < cols; ++c) waves[r * cols + c] = w.values(r, c);
        }
    }
    if (time != nullptr) {
        for (std::size_t r = 0; r < w.time.size(); ++r) time[r] = w.time[r];
    }
}

}  // namespace

extern "C" {

void emtref_free(void* p) { std::free(p); }

/// parse_model -> compile_task(profile, optional scenario rows) -> text forms.
/// rows_json: null or [[{"component":..,"param":..,"value":..},...],...]
int emtref_compile(const char* document, const char* profile, const char* rows_json,
                   char** schedule_text, char** state_text, int* loop_insertions,
                   char* err, int err_len) {
    return guarded(err, err_len, [&] {
        const NetworkModel model = parse_model(document);
        ScenarioBatch batch;
        const ScenarioBatch* bp = nullptr;
        if (rows_json != nullptr && rows_json[0] != '\0') {
            const auto rows = nlohmann::json::parse(rows_json);
            batch.base_document = document;
            for (const auto& row : rows) {
                std::vector<ScenarioOverride> r;
                for (const auto& ov : row) {
                    r.push_back({ov.at("component").get<std::string>(),
                                 ov.at("param").get<std::string>(), ov.at("value").get<double>()});
                }
                batch.rows.push_back(std::move(r));
            }
            bp = &batch;
        }
        const CompiledTask task =
            compile_task(model, builtin_profile(profile ? profile : "cpu-serial"), bp);
        *schedule_text = dup(task.schedule.serialize());
        *state_text = dup(serialize_state(task.initial, task.schedule.arena_extent,
                                          task.schedule.width));
        if (loop_insertions != nullptr) *loop_insertions = task.loops.insertion_count();
    });
}

/// Shape of a schedule: width, channel count, extent, default steps.
int emtref_schedule_shape(const char* schedule_text, int* width, int* channels, int* extent,
                          int* steps, char* err, int err_len) {
    return guarded(err, err_len, [&] {
        const ScheduleProgram s = ScheduleProgram::parse(schedule_text);
        *width = s.width;
        *channels = static_cast<int>(s.channels.size());
        *extent = s.arena_extent;
        *steps = s.steps;
    });
}

/// interpret (workers == 0) or execute_parallel (workers >= 1) on a parsed
/// schedule + initial arena. waves: steps x (channels*width) row-major.
int emtref_execute(const char* schedule_text, const double* initial, int64_t initial_len,
                   int steps, int warmup, int workers, double* waves, double* time,
                   int* factor_count, double* measured_seconds, char* err, int err_len) {
    return guarded(err, err_len, [&] {
        const ScheduleProgram s = ScheduleProgram::parse(schedule_text);
        Eigen::VectorXd init(initial_len);
        for (int64_t k = 0; k < initial_len; ++k) init[k] = initial[k];
        ExecStats stats;
        ExecOptions opt;
        opt.warmup_steps = warmup;
        opt.stats = &stats;
        const WaveformSet w = workers > 0 ? execute_parallel(s, init, workers, steps, opt)
                                          : interpret(s, init, steps, opt);
        copy_waves(w, waves, time);
        if (factor_count) *factor_count = stats.factor_count;
        if (measured_seconds) *measured_seconds = stats.measured_seconds;
    });
}

/// parse_state: STATE v1 text -> flat arena (caller frees with emtref_free).
int emtref_parse_state(const char* state_text, double** arena, int64_t* len, int* width,
                       char* err, int err_len) {
    return guarded(err, err_len, [&] {
        const Eigen::VectorXd a = parse_state(state_text, width);
        *len = a.size();
        *arena = static_cast<double*>(std::malloc(sizeof(double) * static_cast<std::size_t>(a.size() + 1)));
        for (Eigen::Index k = 0; k < a.size(); ++k) (*arena)[k] = a[k];
    });
}

/// run_serial on a document; channels from the document's task.
int emtref_run_serial(const char* document, int steps, int warmup, double* waves,
                      double* time, int* channel_count, int* factor_count,
                      double* measured_seconds, char* err, int err_len) {
    return guarded(err, err_len, [&] {
        const NetworkModel model = parse_model(document);
        RunOptions opt;
        opt.steps_override = steps;
        opt.warmup_steps = warmup;
        int fc = 0;
        double secs = 0.0;
        opt.factor_count = &fc;
        opt.measured_seconds = &secs;
        const WaveformSet w = run_serial(model, model.task, opt);
        if (channel_count) *channel_count = static_cast<int>(w.channels.size());
        copy_waves(w, waves, time);
        if (factor_count) *factor_count = fc;
        if (measured_seconds) *measured_seconds = secs;
    });
}

/// Document's channel count and default step count (TaskConfig::steps).
int emtref_document_shape(const char* document, int* channels, int* steps, char* err,
                          int err_len) {
    return guarded(err, err_len, [&] {
        const NetworkModel model = parse_model(document);
        *channels = static_cast<int>(model.task.channels.size());
        *steps = model.task.steps();
    });
}

int emtref_gen_scale_case(const char* document, int k, char** out, char* err, int err_len) {
    return guarded(err, err_len, [&] { *out = dup(gen_scale_case(document, k)); });
}

int emtref_apply_overrides(const char* document, const char* row_json, char** out, char* err,
                           int err_len) {
    return guarded(err, err_len, [&] {
        std::vector<ScenarioOverride> r;
        for (const auto& ov : nlohmann::json::parse(row_json)) {
            r.push_back({ov.at("component").get<std::string>(), ov.at("param").get<std::string>(),
                         ov.at("value").get<double>()});
        }
        *out = dup(apply_overrides(document, r));
    });
}

/// WaveformSet::to_text of host rows (values: rows x (channels*width), row-major).
int emtref_waves_text(const char* const* names, int channels, int width, const double* time,
                      const double* values, int rows, char** out, char* err, int err_len) {
    return guarded(err, err_len, [&] {
        WaveformSet w;
        for (int c = 0; c < channels; ++c) w.channels.emplace_back(names[c]);
        w.width = width;
        w.time.assign(time, time + rows);
        const int cols = channels * width;
        w.values.resize(rows, cols);
        for (int r = 0; r < rows; ++r)
            for (int c = 0; c < cols; ++c) w.values(r, c) = values[static_cast<size_t>(r) * cols + c];
        *out = dup(w.to_text());
    });
}

}  // extern "C"
