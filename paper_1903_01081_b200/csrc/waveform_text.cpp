// WaveformSet text output: the reference's
// WaveformSet::to_text (proj/src/waveform.cpp:22-42) — header "time" plus one
// name per channel ("name#lane" when width > 1), then one row per step of
// %.17g values (format_g17, proj/src/common.cpp:85-89) separated by single
// spaces — produced by several host threads over row blocks. Each value is
// formatted with std::to_chars(general, 17), which C++17 specifies as printf
// "%.*g" in the C locale, so the bytes equal the reference's snprintf output
// (tests/test_waveform_text.py checks both against the reference itself).
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/emt_b200.h"

namespace emtb200 {
emt_status set_error(int code, const std::string& msg);
}

namespace {

// "%.17g" of v appended at p (≤ 32 bytes): to_chars for finite values; printf's
// spellings for the rest ("nan"/"-nan", "inf"/"-inf", as glibc prints them)
char* g17(char* p, double v) {
    if (!std::isfinite(v)) {
        const int n = std::snprintf(p, 32, "%.17g", v);
        return p + n;
    }
    return std::to_chars(p, p + 32, v, std::chars_format::general, 17).ptr;
}

}  // namespace

extern "C" {

emt_status emt_waves_to_text(const char* const* channel_names, int32_t channels, int32_t width, const double* time,
                             const double* values, int64_t rows, int32_t threads, char** out, int64_t* out_len) {
    using emtb200::set_error;
    if (out == nullptr || (rows > 0 && (time == nullptr || (values == nullptr && channels > 0))) ||
        (channels > 0 && channel_names == nullptr))
        return set_error(EMT_INVALID_HANDLE, "null argument");
    if (channels < 0 || width < 1 || rows < 0) return set_error(EMT_NON_POSITIVE_INPUT, "channels/width/rows");
    std::string head = "time";
    for (int c = 0; c < channels; ++c) {
        if (width == 1) {
            head += " ";
            head += channel_names[c];
        } else {
            for (int l = 0; l < width; ++l) head += " " + std::string(channel_names[c]) + "#" + std::to_string(l);
        }
    }
    head += "\n";
    const int64_t cols = static_cast<int64_t>(channels) * width;
    const int nt = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(threads > 0 ? threads : 1, std::max<int64_t>(1, rows / 64))));
    // each thread formats a contiguous block of rows into its own buffer (≤ 32 bytes a value)
    std::vector<std::string> part(static_cast<size_t>(nt));
    auto work = [&](int k) {
        const int64_t r0 = rows * k / nt, r1 = rows * (k + 1) / nt;
        std::string& s = part[static_cast<size_t>(k)];
        s.resize(static_cast<size_t>((r1 - r0) * (cols + 1) * 32));
        char* p = s.data();
        for (int64_t r = r0; r < r1; ++r) {
            p = g17(p, time[r]);
            const double* row = values + r * cols;
            for (int64_t c = 0; c < cols; ++c) {
                *p++ = ' ';
                p = g17(p, row[c]);
            }
            *p++ = '\n';
        }
        s.resize(static_cast<size_t>(p - s.data()));
    };
    std::vector<std::thread> pool;
    for (int k = 1; k < nt; ++k) pool.emplace_back(work, k);
    work(0);
    for (auto& t : pool) t.join();
    size_t n = head.size();
    for (const auto& s : part) n += s.size();
    char* buf = static_cast<char*>(std::malloc(n + 1));
    if (buf == nullptr) return set_error(EMT_CAPACITY_EXCEEDED, "out of host memory");
    char* q = buf;
    std::memcpy(q, head.data(), head.size());
    q += head.size();
    for (const auto& s : part) {
        std::memcpy(q, s.data(), s.size());
        q += s.size();
    }
    *q = '\0';
    *out = buf;
    if (out_len != nullptr) *out_len = static_cast<int64_t>(n);
    return EMT_OK;
}

void emt_free(void* p) { std::free(p); }

}  // extern "C"
