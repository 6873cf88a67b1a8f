// tests/cpp/fmt_harness.cpp — TEST INFRASTRUCTURE: host build of the device
// "%.17g" formatter (paper_1307_0491_b200/csrc/silt_csv.cuh) so the CPU test
// suite can check it against glibc's snprintf, the function the reference
// serialises with (src/snapshot.cpp:14-18).  Built by oracle/Makefile.
#include <cstdio>
#include <cstring>

#include "silt_csv.cuh"

namespace {
silt_csv::Pow5Table* table() {
    static silt_csv::Pow5Table* T = [] {
        auto* t = new silt_csv::Pow5Table;
        silt_csv::build_pow5(*t);
        return t;
    }();
    return T;
}
}  // namespace

extern "C" {

// out[k * stride ...]: NUL-terminated formatter output for v[k]
int fmt_g17_batch(const double* v, long long n, char* out, long long stride) {
    for (long long k = 0; k < n; ++k) {
        const int len = silt_csv::format_g17(v[k], out + k * stride, table());
        out[k * stride + len] = 0;
    }
    return 0;
}

// Compare with snprintf("%.17g") for v[0..n); returns the number of
// mismatches and the index of the first in *first (-1 if none).
long long fmt_g17_check(const double* v, long long n, long long* first) {
    long long bad = 0;
    *first = -1;
    char a[64], b[64];
    for (long long k = 0; k < n; ++k) {
        const int len = silt_csv::format_g17(v[k], a, table());
        a[len] = 0;
        std::snprintf(b, sizeof b, "%.17g", v[k]);
        if (std::strcmp(a, b) != 0) {
            if (*first < 0) *first = k;
            ++bad;
        }
    }
    return bad;
}
}
