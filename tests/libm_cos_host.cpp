// Host build of csrc/libmcos.cuh for tests/test_libm_cos.py (test infrastructure):
// the device cos replica against the live libm cos, compiled without contraction.
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstring>
using std::copysign;
using std::cos;
using std::fabs;
using std::fma;
static inline int emt_lo32(double d) {
    uint64_t b;
    std::memcpy(&b, &d, 8);
    return static_cast<int>(static_cast<uint32_t>(b));
}
#define EMT_LIBMCOS_TEXT(...) __VA_ARGS__
#define EMT_HD static inline
#define EMT_TABLE static const
#include "../paper_1903_01081_b200/csrc/libmcos.cuh"

extern "C" void replica_cos(const double* x, double* y, size_t n) {
    for (size_t i = 0; i < n; ++i) y[i] = emt_libm_cos(x[i]);
}
extern "C" void libm_cos(const double* x, double* y, size_t n) {
    for (size_t i = 0; i < n; ++i) y[i] = ::cos(x[i]);
}
