// The "sm100a" code-database dialect: emit_source(schedule,
// "sm100a") for the reference's emitter (/root/reference/proj/src/codegen.cpp:84-230).
//
// The "cpp" dialect splices per-kernel templates into one C++ program whose CLI is
// `--state <file> --steps <n> --out <waveforms>` with exit codes 2 (usage / I/O),
// 3 (singular matrix) and 4 (divergence) (proj/data/codedb/cpp/prologue.tpl:87,
// :165, :198-224). The sm100a dialect emits the same program for a B200: the
// schedule-specialised step-loop kernel of codegen.cpp (straight-line, every slot
// and lane-invariant constant an immediate) plus a host main() with the same CLI,
// exit codes and waveform text (kHeader, then per step "%.17g" time and the
// channel values channel-major then lane, as prologue.tpl's main writes them).
// Build it with nvcc: -gencode arch=compute_100a,code=sm_100a -fmad=false.
//
// The program is exact everywhere (the backward sweep branches to IEEE division
// below the reciprocal-multiply's exact range, EMT_FLAG_EXACT_DIVISION), so its
// waveform file is byte-identical to the interpreter's. Schedules the specialised
// kernel cannot hold in shared memory, and line-coupled schedules (an extension
// the reference format has no process for), are rejected.
#include <cstdio>
#include <sstream>
#include <string>
#include <vector>

#include "codegen.hpp"

namespace emtb200 {

namespace {

std::string hexlit(double v) {
    char b[64];
    std::snprintf(b, sizeof b, "%a", v);
    return b;
}

const char* const kDriver = R"EMTDRV(
// ---- host driver (emt_emit_program): CLI and waveform text of the "cpp" dialect's program
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

static int load_state(const char* path, std::vector<double>& S) {
    FILE* f = fopen(path, "r");
    if (f == NULL) return 1;
    int extent = 0, width = 0;
    if (fscanf(f, "STATE v1 extent=%d width=%d", &extent, &width) != 2 || extent != EXTENT_ || width != (int)W_) {
        fclose(f);
        return 1;
    }
    S.assign((size_t)EXTENT_ * W_, 0.0);
    for (size_t k = 0; k < S.size(); ++k) {
        if (fscanf(f, "%lf", &S[k]) != 1) {
            fclose(f);
            return 1;
        }
    }
    fclose(f);
    return 0;
}

static void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        fprintf(stderr, "%s: %s\n", what, cudaGetErrorString(e));
        exit(2);
    }
}

int main(int argc, char** argv) {
    const char* state_path = NULL;
    const char* out_path = NULL;
    long steps = STEPS_;
    for (int i = 1; i + 1 < argc; i += 2) {
        if (strcmp(argv[i], "--state") == 0) state_path = argv[i + 1];
        else if (strcmp(argv[i], "--steps") == 0) steps = atol(argv[i + 1]);
        else if (strcmp(argv[i], "--out") == 0) out_path = argv[i + 1];
    }
    if (state_path == NULL || out_path == NULL) {
        fprintf(stderr, "usage: %s --state <file> --steps <n> --out <waveforms>\n", argv[0]);
        return 2;
    }
    std::vector<double> S;
    if (load_state(state_path, S) != 0) {
        fprintf(stderr, "cannot load state snapshot %s\n", state_path);
        return 2;
    }
    FILE* out = fopen(out_path, "w");
    if (out == NULL) {
        fprintf(stderr, "cannot open %s\n", out_path);
        return 2;
    }
    fputs(kHeader, out);
    const int chunk = CHUNK_;
    const size_t row = (size_t)NCH * W_;
    double *arena, *ctab, *waves, *srctab = NULL;
    unsigned char* refac;
    int *lane_err, *events, *n_events;
    check(cudaMalloc(&arena, S.size() * sizeof(double)), "cudaMalloc");
    check(cudaMalloc(&ctab, sizeof(kCtab)), "cudaMalloc");
    check(cudaMalloc(&waves, (size_t)chunk * row * sizeof(double) + 8), "cudaMalloc");
    check(cudaMalloc(&refac, (size_t)chunk), "cudaMalloc");
    check(cudaMalloc(&lane_err, 4 * sizeof(int) * (size_t)W_), "cudaMalloc");
    check(cudaMalloc(&events, 3 * sizeof(int) * (size_t)MAXEV_), "cudaMalloc");
    check(cudaMalloc(&n_events, sizeof(int)), "cudaMalloc");
#if NSRC > 0
    check(cudaMalloc(&srctab, (size_t)chunk * NSRC * sizeof(double)), "cudaMalloc");
#endif
    check(cudaMemcpy(arena, S.data(), S.size() * sizeof(double), cudaMemcpyHostToDevice), "H2D");
    check(cudaMemcpy(ctab, kCtab, sizeof(kCtab), cudaMemcpyHostToDevice), "H2D");
    check(cudaMemset(lane_err, 0, 4 * sizeof(int) * (size_t)W_), "memset");
    check(cudaMemset(n_events, 0, sizeof(int)), "memset");
    check(cudaFuncSetAttribute(emt_cg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_), "smem attribute");
    std::vector<double> host((size_t)chunk * row);
    std::vector<int> err(4 * (size_t)W_);
    for (long s0 = 0; s0 < steps; s0 += chunk) {
        const int n = (int)(steps - s0 < chunk ? steps - s0 : chunk);
        check(cudaMemset(refac, 0, (size_t)chunk), "memset");
#if NSRC > 0
        emt_src_kernel<<<(unsigned)(((long long)n * NSRC + 255) / 256), 256>>>(srctab, (int)s0, n, ctab);
#endif
        KArgs a = {arena, ctab, waves, refac, lane_err, events, n_events, MAXEV_, (int)s0, n, 0, 1e12,
                   NULL, 0, 0, NULL, 0, GRID_, NULL, srctab, 0, 0};
        emt_cg_kernel<<<GRID_, BLOCK_, SMEM_>>>(a);
        check(cudaGetLastError(), "launch");
        check(cudaDeviceSynchronize(), "step loop");
        check(cudaMemcpy(err.data(), lane_err, err.size() * sizeof(int), cudaMemcpyDeviceToHost), "D2H");
        int code = 0, fstep = 0x7fffffff;  // earliest failing step over the lanes
        for (long l = 0; l < W_; ++l)
            if (err[4 * l] != 0 && err[4 * l + 1] < fstep) { code = err[4 * l]; fstep = err[4 * l + 1]; }
        const int rows = code != 0 ? (int)(fstep - s0) : n;  // rows completed before the failing step
        if (rows > 0) check(cudaMemcpy(host.data(), waves, (size_t)rows * row * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
        for (int r = 0; r < rows; ++r) {
            const double t = (double)(s0 + r + 1) * DT_;
            fprintf(out, "%.17g", t);
            for (size_t c = 0; c < row; ++c) fprintf(out, " %.17g", host[(size_t)r * row + c]);
            fputc('\n', out);
        }
        if (code == 8) {
            fclose(out);
            fprintf(stderr, "singular matrix: zero pivot below tolerance\n");
            exit(3);
        }
        if (code == 7) {
            fclose(out);
            fprintf(stderr, "divergence: node voltage out of range\n");
            exit(4);
        }
        if (code != 0) {
            fclose(out);
            fprintf(stderr, "step loop failed (code %d)\n", code);
            exit(2);
        }
    }
    fclose(out);
    return 0;
}
)EMTDRV";

}  // namespace

bool emit_program(const Schedule& s, const std::vector<double>& ctab, int lanes, std::string& out, Failure& fail) {
    for (const Proc& p : s.procs)
        if (p.code == kNortonBergeron) {
            fail = {14, "sm100a", "line-coupled schedules have no emitted-program form"};  // UnknownKind
            return false;
        }
    CodegenOptions opt;
    opt.warps = 8;
    opt.exact_division = true;
    GeneratedKernel g;
    if (!generate_kernel(s, ctab, lanes, opt, g, fail)) return false;
    std::ostringstream o;
    o << "// emtb200 emit_source(schedule, \"sm100a\"): " << s.nodes << " nodes, " << s.comps << " components, "
      << lanes << " lanes; " << g.summary << "\n"
      << "// build: nvcc -gencode arch=compute_100a,code=sm_100a -fmad=false -std=c++17 -o program program.cu\n"
      << "// run:   ./program --state <STATE v1 file> --steps <n> --out <waveforms>  (exit 2 I/O, 3 singular, 4 divergence)\n";
    o << g.source << "\n";
    const int lpc = g.lpc > 0 ? g.lpc : 32;
    o << "#define EXTENT_ " << s.extent << "\n#define STEPS_ " << s.steps << "L\n#define DT_ (" << hexlit(s.dt) << ")\n"
      << "#define CHUNK_ 1000\n#define MAXEV_ 65536\n#define GRID_ " << (lanes + lpc - 1) / lpc << "\n#define BLOCK_ "
      << 32 * g.warps << "\n#define SMEM_ " << g.smem_bytes << "\n#define NSRC " << g.nsrc << "\n";
    o << "static const double kCtab[" << std::max<size_t>(1, ctab.size()) << "] = {";
    for (size_t k = 0; k < ctab.size(); ++k) o << (k ? (k % 8 ? "," : ",\n") : "") << hexlit(ctab[k]);
    if (ctab.empty()) o << "0.0";
    o << "};\n";
    std::string header = "time";
    for (const std::string& name : s.channel_names) {
        if (lanes == 1) header += " " + name;
        else
            for (int l = 0; l < lanes; ++l) header += " " + name + "#" + std::to_string(l);
    }
    o << "static const char kHeader[] = \"" << header << "\\n\";\n";
    o << kDriver;
    out = o.str();
    return true;
}

}  // namespace emtb200
