// NVRTC compilation + driver-API loading of generated kernels (sm_100a cubins),
// with an in-process and on-disk cache keyed by the source text.
#pragma once

#include <cuda.h>

#include <string>
#include <vector>

namespace emtb200 {

struct JitModule {
    CUmodule module = nullptr;
    CUfunction function = nullptr;
    CUfunction function2 = nullptr;  // optional "emt_src_kernel" of the same module
    double compile_seconds = 0.0;  // 0 when served from a cache
    bool cached = false;
};

/// Compiles `source` for the device's architecture (sm_100a on B200) with
/// --fmad=false and loads `entry`. Returns false with `log` on failure.
bool jit_load(const std::string& source, const std::string& entry, int device, JitModule& out, std::string& log);

/// Driver entry points resolved through cudaGetDriverEntryPoint (no link-time
/// dependency on libcuda, so the library also loads on GPU-less build hosts).
struct Driver {
    CUresult (*ModuleUnload)(CUmodule) = nullptr;
    CUresult (*FuncSetAttribute)(CUfunction, CUfunction_attribute, int) = nullptr;
    CUresult (*LaunchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                             CUstream, void**, void**) = nullptr;
    CUresult (*GetErrorString)(CUresult, const char**) = nullptr;
};
const Driver* driver();

/// Compile only (no device needed): returns the cubin; used by the build check.
bool jit_compile(const std::string& source, const std::string& arch, std::vector<char>& cubin, std::string& log);

}  // namespace emtb200
