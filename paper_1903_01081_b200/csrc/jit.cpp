// NVRTC JIT for the generated step-loop kernels (the paper's runtime
// code-generation step, CloudPSS §III.C; the reference shells out to the host
// C++ compiler instead, proj/src/codegen.cpp:232-258).
#include "jit.hpp"

#include <cuda_runtime.h>
#include <nvrtc.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <map>
#include <mutex>
#include <sstream>
#include <sys/stat.h>
#include <unistd.h>

namespace emtb200 {

namespace {

std::mutex g_mu;
std::map<std::string, std::vector<char>>& mem_cache() {
    static std::map<std::string, std::vector<char>> c;
    return c;
}

std::string cache_dir() {
    const char* env = std::getenv("EMTB200_CACHE");
    if (env && *env) return env;
    const char* home = std::getenv("HOME");
    return std::string(home && *home ? home : "/tmp") + "/.cache/emtb200";
}

std::string key_of(const std::string& src, const std::string& arch) {
    // FNV-1a 64 over source + arch + compiler version
    unsigned long long h = 1469598103934665603ULL;
    auto mix = [&h](const std::string& s) {
        for (unsigned char c : s) {
            h ^= c;
            h *= 1099511628211ULL;
        }
    };
    int maj = 0, min = 0;
    nvrtcVersion(&maj, &min);
    mix(src);
    mix(arch);
    mix(std::to_string(maj) + "." + std::to_string(min));
    char b[32];
    std::snprintf(b, sizeof b, "%016llx", h);
    return std::string(b) + "_" + arch + "_" + std::to_string(src.size());
}

template <typename F>
bool resolve(const char* name, F& fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || p == nullptr) return false;
    fn = reinterpret_cast<F>(p);
    return true;
}

struct FullDriver : Driver {
    CUresult (*DeviceGet)(CUdevice*, int) = nullptr;
    CUresult (*DeviceGetAttribute)(int*, CUdevice_attribute, CUdevice) = nullptr;
    CUresult (*ModuleLoadData)(CUmodule*, const void*) = nullptr;
    CUresult (*ModuleGetFunction)(CUfunction*, CUmodule, const char*) = nullptr;
    bool ok = false;
};

const FullDriver* full_driver() {
    static FullDriver d;
    static std::once_flag once;
    std::call_once(once, [] {
        d.ok = resolve("cuDeviceGet", d.DeviceGet) && resolve("cuDeviceGetAttribute", d.DeviceGetAttribute) &&
               resolve("cuModuleLoadData", d.ModuleLoadData) && resolve("cuModuleGetFunction", d.ModuleGetFunction) &&
               resolve("cuModuleUnload", d.ModuleUnload) && resolve("cuFuncSetAttribute", d.FuncSetAttribute) &&
               resolve("cuLaunchKernel", d.LaunchKernel) && resolve("cuGetErrorString", d.GetErrorString);
    });
    return d.ok ? &d : nullptr;
}

}  // namespace

const Driver* driver() { return full_driver(); }

bool jit_compile(const std::string& source, const std::string& arch, std::vector<char>& cubin, std::string& log) {
    nvrtcProgram prog;
    if (nvrtcCreateProgram(&prog, source.c_str(), "emt_generated.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
        log = "nvrtcCreateProgram failed";
        return false;
    }
    const std::string gpu = "--gpu-architecture=" + arch;
    const char* opts[] = {gpu.c_str(), "--fmad=false", "-std=c++17", "-default-device", "-lineinfo"};
    const nvrtcResult rc = nvrtcCompileProgram(prog, static_cast<int>(sizeof(opts) / sizeof(opts[0])), opts);
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    log.assign(n, '\0');
    if (n) nvrtcGetProgramLog(prog, &log[0]);
    if (rc != NVRTC_SUCCESS) {
        nvrtcDestroyProgram(&prog);
        log = std::string(nvrtcGetErrorString(rc)) + "\n" + log;
        return false;
    }
    size_t m = 0;
    nvrtcGetCUBINSize(prog, &m);
    cubin.resize(m);
    nvrtcGetCUBIN(prog, cubin.data());
    nvrtcDestroyProgram(&prog);
    return true;
}

bool jit_load(const std::string& source, const std::string& entry, int device, JitModule& out, std::string& log) {
    const FullDriver* d = full_driver();
    if (d == nullptr) {
        log = "CUDA driver entry points unavailable";
        return false;
    }
    CUdevice dev;
    if (d->DeviceGet(&dev, device) != CUDA_SUCCESS) {
        log = "cuDeviceGet failed";
        return false;
    }
    int major = 0, minor = 0;
    d->DeviceGetAttribute(&major, CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MAJOR, dev);
    d->DeviceGetAttribute(&minor, CU_DEVICE_ATTRIBUTE_COMPUTE_CAPABILITY_MINOR, dev);
    // arch-specific ("a") target: sm_100a on B200
    const std::string arch = "sm_" + std::to_string(major) + std::to_string(minor) + "a";
    const std::string key = key_of(source, arch);
    std::vector<char> cubin;
    bool have = false;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = mem_cache().find(key);
        if (it != mem_cache().end()) {
            cubin = it->second;
            have = true;
        }
    }
    const std::string path = cache_dir() + "/" + key + ".cubin";
    if (!have) {
        std::ifstream f(path, std::ios::binary);
        if (f) {
            cubin.assign(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
            have = !cubin.empty();
        }
    }
    out.cached = have;
    if (!have) {
        const auto t0 = std::chrono::steady_clock::now();
        if (!jit_compile(source, arch, cubin, log)) return false;
        out.compile_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        mkdir((cache_dir()).c_str(), 0755);
        std::string parent = cache_dir().substr(0, cache_dir().rfind('/'));
        mkdir(parent.c_str(), 0755);
        mkdir((cache_dir()).c_str(), 0755);
        // per-process temporary + rename: ranks of one job may compile the same kernel at once
        const std::string tmp = path + "." + std::to_string(static_cast<long>(getpid())) + ".tmp";
        std::ofstream f(tmp, std::ios::binary);
        if (f) {
            f.write(cubin.data(), static_cast<std::streamsize>(cubin.size()));
            f.close();
            std::rename(tmp.c_str(), path.c_str());
        }
    }
    {
        std::lock_guard<std::mutex> lk(g_mu);
        mem_cache()[key] = cubin;
    }
    if (d->ModuleLoadData(&out.module, cubin.data()) != CUDA_SUCCESS) {
        if (!out.cached) {
            log = "cuModuleLoadData failed";
            return false;
        }
        // unreadable cache entry: compile afresh
        const auto t0 = std::chrono::steady_clock::now();
        if (!jit_compile(source, arch, cubin, log)) return false;
        out.compile_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        out.cached = false;
        {
            std::lock_guard<std::mutex> lk(g_mu);
            mem_cache()[key] = cubin;
        }
        if (d->ModuleLoadData(&out.module, cubin.data()) != CUDA_SUCCESS) {
            log = "cuModuleLoadData failed";
            return false;
        }
    }
    out.function2 = nullptr;
    if (source.find("emt_src_kernel") != std::string::npos &&
        d->ModuleGetFunction(&out.function2, out.module, "emt_src_kernel") != CUDA_SUCCESS)
        out.function2 = nullptr;
    if (d->ModuleGetFunction(&out.function, out.module, entry.c_str()) != CUDA_SUCCESS) {
        log = "cuModuleGetFunction failed for " + entry;
        return false;
    }
    return true;
}

}  // namespace emtb200
