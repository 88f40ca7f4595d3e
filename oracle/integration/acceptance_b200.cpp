// Acceptance criteria 3 and 4 of the reference (/root/reference/proj/tests/acceptance.cpp:96-146)
// with the B200 executor substituted, plus the paths reference_b200.patch opens:
// execute_task(Strategy::Device), the "b200" device profile, run_vse on a
// "device"-strategy package and orchestrator dispatch to a b200 worker slot.
// One PASS/FAIL line per check; exit status = number of failures (like acceptance.cpp).
//
//   acceptance_b200 <feeder33_pv3 document> <scratch dir>
//
// Test infrastructure (built by `make -C oracle integ`, run by tests/test_integration_b200.py).
#include <cstdio>
#include <exception>
#include <filesystem>
#include <string>

#include <cstdlib>
#include <sys/wait.h>

#include "emtgrid/bench.hpp"
#include "emtgrid/codegen.hpp"
#include "emtgrid/grid.hpp"

using namespace emtgrid;

namespace {

int failures = 0;

void report(const std::string& id, bool pass, const std::string& detail) {
    std::printf("[%s] %s -- %s\n", pass ? "PASS" : "FAIL", id.c_str(), detail.c_str());
    std::fflush(stdout);
    if (!pass) ++failures;
}

CompiledTask compile_document(const std::string& document, const ScenarioBatch* batch = nullptr,
                              const char* profile = "cpu-serial") {
    return compile_task(parse_model(document), builtin_profile(profile), batch);
}

// criterion 3: serial stepper, interpreter, parallel executor and the B200 executor are byte-identical
void criterion_backend_bitwise(const std::string& doc) {
    const int steps = 10000;
    const NetworkModel model = parse_model(doc);
    RunOptions serial_options;
    serial_options.steps_override = steps;
    const std::string serial_text = run_serial(model, model.task, serial_options).to_text();
    const CompiledTask task = compile_document(doc);
    bool pass = interpret(task.schedule, task.initial, steps).to_text() == serial_text;
    std::string mismatch = pass ? "" : " interpreter";
    for (int workers : {1, 2}) {
        if (execute_parallel(task.schedule, task.initial, workers, steps).to_text() != serial_text) {
            pass = false;
            mismatch += " parallel:" + std::to_string(workers);
        }
    }
    ExecStats stats;
    ExecOptions options;
    options.stats = &stats;
    if (execute_b200(task.schedule, task.initial, steps, options).to_text() != serial_text) {
        pass = false;
        mismatch += " b200";
    }
    // through the dispatch the patch adds: the b200 profile compiles, Strategy::Device executes
    const CompiledTask dtask = compile_document(doc, nullptr, "b200");
    if (execute_task(dtask, builtin_profile("b200").affinity, 0, steps).to_text() != serial_text) {
        pass = false;
        mismatch += " execute_task(device)";
    }
    report("criterion 3", pass,
           pass ? "33-node + 3-PV case, 10000 steps: run_serial == interpret == execute_parallel{1,2} == "
                  "execute_b200 == execute_task(Strategy::Device); factor_count " + std::to_string(stats.factor_count)
                : "mismatch in:" + mismatch);
}

// criterion 4: N=16 batch columns on the device == 16 independent serial runs
void criterion_vectorization(const std::string& doc) {
    const ScenarioBatch batch = gen_scenarios(doc, {700.0, 850.0, 1000.0, 1150.0}, {10.0, 20.0, 30.0, 40.0});
    const CompiledTask task = compile_document(doc, &batch);
    const int steps = 2000;
    const WaveformSet wide = execute_b200(task.schedule, task.initial, steps);
    bool pass = task.schedule.width == 16;
    int bad_lane = -1;
    for (int lane = 0; lane < 16 && pass; ++lane) {
        const NetworkModel lane_model = parse_model(apply_overrides(doc, batch.rows[static_cast<std::size_t>(lane)]));
        RunOptions options;
        options.steps_override = steps;
        if (wide.lane(lane).to_text() != run_serial(lane_model, lane_model.task, options).to_text()) {
            pass = false;
            bad_lane = lane;
        }
    }
    report("criterion 4", pass,
           pass ? "16-lane irradiance x temperature batch, 2000 steps: every execute_b200 lane byte-identical to "
                  "run_serial of its own document"
                : "first mismatching lane " + std::to_string(bad_lane));
}

std::string with_task(const std::string& doc, const char* profile, const char* strategy) {
    std::string out = doc;
    auto set = [&](const std::string& key, const std::string& value) {
        const std::size_t k = out.find("\"" + key + "\"");
        const std::size_t q0 = out.find('"', out.find(':', k) + 1);
        const std::size_t q1 = out.find('"', q0 + 1);
        out.replace(q0 + 1, q1 - q0 - 1, value);
    };
    set("device_profile", profile);
    set("strategy", strategy);
    return out;
}

// run_vse on a package whose manifest says strategy "device" (grid.cpp:113-140 + patch)
void vse_device_package(const std::string& doc, const std::string& scratch) {
    const std::string ddoc = with_task(doc, "b200", "device");
    const std::string sdoc = with_task(doc, "cpu-serial", "serial");
    const VsePackage dp = assemble_vse(ddoc, scratch + "/pkg_b200");
    const VsePackage sp = assemble_vse(sdoc, scratch + "/pkg_serial");
    run_vse(dp.dir, scratch + "/b200.txt");
    run_vse(sp.dir, scratch + "/serial.txt");
    const std::string a = read_file(scratch + "/b200.txt"), b = read_file(scratch + "/serial.txt");
    const bool manifest_ok = read_file(dp.dir + "/manifest.json").find("\"device\"") != std::string::npos;
    report("vse", a == b && manifest_ok && !a.empty(),
           "assemble_vse + run_vse of a b200/device package: waveform file byte-identical to the cpu-serial "
           "package's (" + std::to_string(a.size()) + " bytes)");
}

void profile_dispatch() {
    std::vector<WorkerSlot> slots = {{"cpu-0", "cpu-serial", 1, 0}, {"gpu-0", "b200", 2, 0}};
    const auto as = dispatch({{"t1", "b200"}, {"t2", "cpu-serial"}, {"t3", "b200"}, {"t4", "b200"}}, slots);
    bool pass = as.size() == 3 && as[0] == std::make_pair(std::string("t1"), std::string("gpu-0")) &&
                as[1].second == "cpu-0" && as[2] == std::make_pair(std::string("t3"), std::string("gpu-0"));
    const DeviceProfile p = builtin_profile("b200");
    pass = pass && p.affinity == Strategy::Device && to_string(p.affinity) == "device" &&
           strategy_from("device", "test") == Strategy::Device;
    report("dispatch", pass, "b200 tasks go to the b200 slot (capacity 2, third waits); profile affinity device");
}

// errors cross the boundary as the reference's: SingularMatrix at "row 1"
void singular_error() {
    const std::string doc = R"({"nodes": ["1", "2", "3", "4"], "components": [
      {"id": "la", "kind": "inductor", "params": {"inductance": 0.001}, "terminals": ["1", "2"]},
      {"id": "lb", "kind": "inductor", "params": {"inductance": 0.002}, "terminals": ["3", "4"]}],
     "control": [], "couplings": [],
     "task": {"dt": 1e-4, "duration": 1e-3, "channels": ["v:1"], "device_profile": "cpu-serial", "strategy": "serial"}})";
    const CompiledTask task = compile_document(doc);
    std::string ref_where, dev_where;
    int ref_code = -1, dev_code = -2;
    try {
        interpret(task.schedule, task.initial, 10);
    } catch (const Error& e) {
        ref_code = static_cast<int>(e.code());
        ref_where = e.where();
    }
    try {
        execute_b200(task.schedule, task.initial, 10);
    } catch (const Error& e) {
        dev_code = static_cast<int>(e.code());
        dev_where = e.where();
    }
    report("errors", ref_code == dev_code && ref_code == static_cast<int>(ErrorCode::SingularMatrix) &&
                         ref_where == dev_where,
           "ungrounded islands: interpret and execute_b200 both throw SingularMatrix at '" + ref_where + "' / '" +
               dev_where + "'");
}

// criterion 5 in the "sm100a" dialect (acceptance.cpp:150-187): the emitted program,
// built with nvcc, reproduces the interpreter — here byte for byte — with the "cpp"
// program's CLI; exit codes 3 (singular) and 4 (divergence); "cuda" stays unknown
int run_program(const std::string& bin, const std::string& dir, const CompiledTask& task, int steps) {
    write_file(dir + "/state.txt", serialize_state(task.initial, task.schedule.arena_extent, task.schedule.width));
    const std::string cmd = "\"" + bin + "\" --state \"" + dir + "/state.txt\" --steps " + std::to_string(steps) +
                            " --out \"" + dir + "/waves.txt\" 2> \"" + dir + "/stderr.txt\"";
    const int rc = std::system(cmd.c_str());
    return WIFEXITED(rc) ? WEXITSTATUS(rc) : -1;
}

void criterion_emitted_sm100a(const std::string& doc, const std::string& scratch) {
    const char* nv = std::getenv("EMTGRID_NVCC");
    const Toolchain tc{nv != nullptr && *nv != '\0' ? nv : "/usr/local/cuda/bin/nvcc", sm100a_flags()};
    const int steps = 1000;
    const CompiledTask task = compile_document(doc);
    const WaveformSet expected = interpret(task.schedule, task.initial, steps);
    const std::string dir = scratch + "/emit_feeder";
    const std::string bin = compile_emitted(emit_source(task.schedule, "sm100a"), tc, dir);
    const int rc = run_program(bin, dir, task, steps);
    const bool same = rc == 0 && WaveformSet::load(dir + "/waves.txt").to_text() == expected.to_text();

    bool cuda_unknown = false;
    try {
        emit_source(task.schedule, "cuda");
    } catch (const Error& e) {
        cuda_unknown = e.code() == ErrorCode::UnknownDialect;
    }
    const std::string islands = R"({"nodes": ["1", "2", "3", "4"], "components": [
      {"id": "la", "kind": "inductor", "params": {"inductance": 0.001}, "terminals": ["1", "2"]},
      {"id": "lb", "kind": "inductor", "params": {"inductance": 0.002}, "terminals": ["3", "4"]}],
     "control": [], "couplings": [],
     "task": {"dt": 1e-4, "duration": 1e-3, "channels": ["v:1"], "device_profile": "cpu-serial", "strategy": "serial"}})";
    const std::string diverging = R"({"nodes": ["1"], "components": [
      {"id": "r1", "kind": "resistor", "params": {"resistance": 1000.0}, "terminals": ["1", "0"]},
      {"id": "cs", "kind": "controlled_current_source", "params": {"gain": 1.0}, "terminals": ["1", "0"]}],
     "control": [{"id": "m2", "kind": "gain", "params": {"k": 4.0}, "inputs": ["v1"]},
                 {"id": "b1", "kind": "sum", "params": {}, "inputs": ["m2", "one"]},
                 {"id": "one", "kind": "constant", "params": {"value": 1.0}, "inputs": []}],
     "couplings": [{"direction": "meter", "electrical_ref": "1", "signal_ref": "v1"},
                   {"direction": "actuator", "electrical_ref": "cs", "signal_ref": "b1"}],
     "task": {"dt": 1e-3, "duration": 1.0, "channels": ["v:1"], "device_profile": "cpu-serial", "strategy": "serial"}})";
    const CompiledTask ti = compile_document(islands), td = compile_document(diverging);
    const int rc3 = run_program(compile_emitted(emit_source(ti.schedule, "sm100a"), tc, scratch + "/emit_islands"),
                                scratch + "/emit_islands", ti, 10);
    const int rc4 = run_program(compile_emitted(emit_source(td.schedule, "sm100a"), tc, scratch + "/emit_div"),
                                scratch + "/emit_div", td, 1000);
    // the rows before the divergence are written, like the cpp program's
    std::size_t div_rows = 0;
    try {
        interpret(td.schedule, td.initial, 1000);
    } catch (const Error&) {
    }
    const std::string div_text = read_file(scratch + "/emit_div/waves.txt");
    for (char ch : div_text) div_rows += ch == '\n' ? 1 : 0;
    const bool pass = same && cuda_unknown && rc3 == 3 && rc4 == 4 && div_rows > 1;
    report("criterion 5 (sm100a)", pass,
           "emit_source(feeder, \"sm100a\") built with nvcc: 1000 steps byte-identical to interpret (" +
               std::string(same ? "yes" : "NO") + "); exit codes singular " + std::to_string(rc3) + " (3), divergence " +
               std::to_string(rc4) + " (4) after " + std::to_string(div_rows - 1) + " rows; \"cuda\" " +
               (cuda_unknown ? "UnknownDialect" : "ACCEPTED"));
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: %s <feeder33_pv3.json> <scratch dir>\n", argv[0]);
        return 2;
    }
    const std::string doc = read_file(argv[1]);
    const std::string scratch = argv[2];
    std::filesystem::create_directories(scratch);
    for (auto* f : {criterion_backend_bitwise, criterion_vectorization}) {
        try {
            f(doc);
        } catch (const std::exception& e) {
            report("exception", false, e.what());
        }
    }
    try {
        criterion_emitted_sm100a(doc, scratch);
        vse_device_package(doc, scratch);
        profile_dispatch();
        singular_error();
    } catch (const std::exception& e) {
        report("exception", false, e.what());
    }
    return failures;
}
