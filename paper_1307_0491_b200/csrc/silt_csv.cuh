// silt_csv.cuh — "%.17g" formatting of doubles, exactly as glibc's printf
// prints them, usable on the device (snapshot writer) and on the host (the
// CPU test harness tests/cpp/fmt_harness.cpp compiles this same header).
//
// The reference serialises snapshots and reports with
// snprintf(buf, 40, "%.17g", v) (src/snapshot.cpp:14-18, src/report.cpp:11-15).
// glibc prints the correctly rounded (round-half-even) 17-significant-digit
// decimal value.  Here: v = m 2^e2 exactly; for the decimal exponent k the
// integer D = rhe(v 10^(16-k)) is computed EXACTLY — 128-bit arithmetic for
// 1e-11 <= |v| < 1e17 (every value of a physical snapshot), a small bigint
// (32-bit limbs, powers of five from a table) otherwise — and k is corrected
// until 10^16 <= D < 10^17.  The %g layout rules follow C99 7.19.6.1: fixed
// notation when -4 <= k < 17, else d.ddde±XX; trailing zeros and a bare
// decimal point removed.
#pragma once
#include <stdint.h>

#ifndef __CUDACC__
#include <cmath>
#ifndef __host__
#define __host__
#endif
#ifndef __device__
#define __device__
#endif
#ifndef __forceinline__
#define __forceinline__ inline
#endif
#endif

namespace silt_csv {

constexpr int kP5Max = 341;    // 5^0 .. 5^340
constexpr int kP5Limbs = 26;   // 5^340 < 2^790 -> 25 limbs (+1 spare)
constexpr int kBigLimbs = 36;  // numbers up to 2^1152
constexpr int kMaxNum = 25;    // longest "%.17g" output: -1.2345678901234567e-308

// Powers of five as little-endian 32-bit limbs: table[s][0..kP5Limbs).
struct Pow5Table {
    uint32_t limb[kP5Max][kP5Limbs];
    uint8_t used[kP5Max];  // significant limbs
    double approx[kP5Max]; // (double) 5^s (rounded; for quotient estimates)
};

// Host-side construction of the table (exact schoolbook products).
inline void build_pow5(Pow5Table& T) {
    uint32_t cur[kP5Limbs] = {1};
    int used = 1;
    double ap = 1.0;
    for (int s = 0; s < kP5Max; ++s) {
        for (int k = 0; k < kP5Limbs; ++k) T.limb[s][k] = cur[k];
        T.used[s] = (uint8_t)used;
        T.approx[s] = ap;
        uint64_t carry = 0;
        for (int k = 0; k < used; ++k) {
            const uint64_t x = (uint64_t)cur[k] * 5u + carry;
            cur[k] = (uint32_t)x;
            carry = x >> 32;
        }
        if (carry) cur[used++] = (uint32_t)carry;
        ap *= 5.0;
    }
}

struct Big {
    uint32_t l[kBigLimbs];
    int n;  // significant limbs
};

__host__ __device__ __forceinline__ void big_from_pow5_times(Big& b, const Pow5Table* T, int s,
                                                             uint64_t m) {
    // b = 5^s * m   (m < 2^64)
    const int u = T->used[s];
    const uint32_t m0 = (uint32_t)m, m1 = (uint32_t)(m >> 32);
    for (int k = 0; k < u + 2; ++k) b.l[k] = 0;
    uint64_t carry = 0;
    for (int k = 0; k < u; ++k) {
        const uint64_t x = (uint64_t)T->limb[s][k] * m0 + b.l[k] + carry;
        b.l[k] = (uint32_t)x;
        carry = x >> 32;
    }
    b.l[u] = (uint32_t)carry;
    carry = 0;
    for (int k = 0; k < u; ++k) {
        const uint64_t x = (uint64_t)T->limb[s][k] * m1 + b.l[k + 1] + carry;
        b.l[k + 1] = (uint32_t)x;
        carry = x >> 32;
    }
    b.l[u + 1] = (uint32_t)carry;
    b.n = u + 2;
    while (b.n > 1 && b.l[b.n - 1] == 0) --b.n;
}

// bit i of b
__host__ __device__ __forceinline__ uint32_t big_bit(const Big& b, int i) {
    const int w = i >> 5;
    return w < b.n ? (b.l[w] >> (i & 31)) & 1u : 0u;
}

// any bit below position i set?
__host__ __device__ __forceinline__ bool big_any_below(const Big& b, int i) {
    const int w = i >> 5;
    for (int k = 0; k < w && k < b.n; ++k)
        if (b.l[k]) return true;
    if (w < b.n && (b.l[w] & ((1u << (i & 31)) - 1u))) return true;
    return false;
}

// bits [i, i+64) of b
__host__ __device__ __forceinline__ uint64_t big_bits64(const Big& b, int i) {
    uint64_t r = 0;
    for (int q = 0; q < 64; q += 32) {
        const int pos = i + q;
        const int w = pos >> 5, o = pos & 31;
        uint64_t lo = w < b.n ? b.l[w] : 0u;
        uint64_t hi = (w + 1) < b.n ? b.l[w + 1] : 0u;
        const uint32_t part = (uint32_t)(o ? ((lo >> o) | (hi << (32 - o))) : lo);
        r |= (uint64_t)part << q;
    }
    return r;
}

__host__ __device__ __forceinline__ int big_bitlen(const Big& b) {
    int n = b.n;
    while (n > 1 && b.l[n - 1] == 0) --n;
    uint32_t top = b.l[n - 1];
    int bl = 0;
    while (top) {
        ++bl;
        top >>= 1;
    }
    return 32 * (n - 1) + bl;
}

__host__ __device__ __forceinline__ int big_cmp(const Big& a, const Big& b) {
    const int n = a.n > b.n ? a.n : b.n;
    for (int k = n - 1; k >= 0; --k) {
        const uint32_t x = k < a.n ? a.l[k] : 0u, y = k < b.n ? b.l[k] : 0u;
        if (x != y) return x < y ? -1 : 1;
    }
    return 0;
}

// r = a - b (a >= b); r may alias a
__host__ __device__ __forceinline__ void big_sub(const Big& a, const Big& b, Big& r) {
    int64_t borrow = 0;
    const int n = a.n;
    for (int k = 0; k < n; ++k) {
        int64_t x = (int64_t)a.l[k] - (k < b.n ? (int64_t)b.l[k] : 0) - borrow;
        borrow = x < 0;
        r.l[k] = (uint32_t)(x + (borrow ? ((int64_t)1 << 32) : 0));
    }
    r.n = n;
    while (r.n > 1 && r.l[r.n - 1] == 0) --r.n;
}

// D = round-half-even(|v| * 10^s) and F = floor(|v| * 10^s) for
// |v| = m 2^e2, m < 2^53.  Returns 0 on success, +1 if the result overflows
// 64 bits (s too large: the caller raises its decimal exponent), -1 if s is
// too small.
__host__ __device__ __forceinline__ int scaled_digits(uint64_t m, int e2, int s,
                                                      const Pow5Table* T, uint64_t& D,
                                                      uint64_t& F) {
    if (s >= 0) {
        if (s >= kP5Max) return 1;
        const int sh = e2 + s;  // |v| 10^s = m 5^s 2^sh
        if (s <= 27 && sh < 0 && sh > -128) {
            // 128-bit fast path: 5^27 < 2^63, so m 5^s < 2^116
            const uint64_t p5 = ((uint64_t)T->limb[s][1] << 32) | T->limb[s][0];
            const unsigned __int128 N = (unsigned __int128)m * p5;
            const int r = -sh;
            const unsigned __int128 q = N >> r;
            if ((uint64_t)(q >> 64)) return 1;
            const unsigned __int128 rem = N - (q << r);
            const unsigned __int128 half = (unsigned __int128)1 << (r - 1);
            uint64_t d = (uint64_t)q;
            F = d;
            if (rem > half || (rem == half && (d & 1u))) ++d;
            D = d;
            return 0;
        }
        Big N;
        big_from_pow5_times(N, T, s, m);
        if (sh >= 0) {  // exact integer
            if (big_bitlen(N) + sh > 64) return 1;
            const uint64_t x = ((uint64_t)(N.n > 1 ? N.l[1] : 0u) << 32) | N.l[0];
            D = F = x << sh;
            return 0;
        }
        const int r = -sh;
        if (big_bitlen(N) > r + 64) return 1;
        uint64_t d = big_bits64(N, r);
        F = d;
        if (big_bit(N, r - 1) && (big_any_below(N, r - 1) || (d & 1u))) ++d;
        D = d;
        return 0;
    }
    // s < 0: |v| 10^s = m 2^(e2 - t) / 5^t with t = -s
    const int t = -s;
    const int sh = e2 - t;
    if (t >= kP5Max) return -1;
    if (sh < 0) return -1;  // |v| < 10^(16 + t): exponent estimate too large
    Big N;
    {
        const int w = sh >> 5, o = sh & 31;
        if (w + 3 > kBigLimbs) return -1;
        for (int k = 0; k < w + 3; ++k) N.l[k] = 0;
        const uint64_t lo = (uint64_t)(uint32_t)m << o;
        const uint64_t hi = (m >> 32) << o;
        N.l[w] = (uint32_t)lo;
        const uint64_t mid = (lo >> 32) + (uint32_t)hi;
        N.l[w + 1] = (uint32_t)mid;
        N.l[w + 2] = (uint32_t)((hi >> 32) + (mid >> 32));
        N.n = w + 3;
        while (N.n > 1 && N.l[N.n - 1] == 0) --N.n;
    }
    // quotient estimate in floating point, then exact correction
#ifdef __CUDA_ARCH__
    const double qd = ldexp((double)m, sh) / T->approx[t];
#else
    const double qd = std::ldexp((double)m, sh) / T->approx[t];
#endif
    if (!(qd < 1.8e19)) return 1;
    uint64_t q = (uint64_t)qd;
    Big P, P5t;
    big_from_pow5_times(P5t, T, t, 1);
    big_from_pow5_times(P, T, t, q);
    while (big_cmp(P, N) > 0) {  // q too large (by a few units at most)
        --q;
        big_sub(P, P5t, P);
    }
    Big R;
    big_sub(N, P, R);
    while (big_cmp(R, P5t) >= 0) {  // q too small
        ++q;
        big_sub(R, P5t, R);
    }
    // rounding: compare 2R with 5^t
    Big R2;
    {
        uint32_t carry = 0;
        for (int k = 0; k < R.n; ++k) {
            const uint64_t x = ((uint64_t)R.l[k] << 1) | carry;
            R2.l[k] = (uint32_t)x;
            carry = (uint32_t)(x >> 32);
        }
        R2.l[R.n] = carry;
        R2.n = R.n + 1;
        while (R2.n > 1 && R2.l[R2.n - 1] == 0) --R2.n;
    }
    const int c = big_cmp(R2, P5t);
    F = q;
    if (c > 0 || (c == 0 && (q & 1u))) ++q;
    D = q;
    return 0;
}

__host__ __device__ __forceinline__ int put_uint(char* out, uint64_t x) {
    char tmp[24];
    int n = 0;
    do {
        tmp[n++] = (char)('0' + x % 10u);
        x /= 10u;
    } while (x);
    for (int k = 0; k < n; ++k) out[k] = tmp[n - 1 - k];
    return n;
}

// snprintf(out, 40, "%.17g", v) without the terminator; returns the length.
__host__ __device__ __forceinline__ int format_g17(double v, char* out, const Pow5Table* T) {
    uint64_t bits;
    {
        union {
            double d;
            uint64_t u;
        } cv;
        cv.d = v;
        bits = cv.u;
    }
    int n = 0;
    const bool neg = bits >> 63;
    const int be = (int)((bits >> 52) & 0x7ff);
    uint64_t frac = bits & ((1ull << 52) - 1);
    if (be == 0x7ff) {
        if (neg) out[n++] = '-';
        if (frac) {
            out[n++] = 'n', out[n++] = 'a', out[n++] = 'n';
        } else {
            out[n++] = 'i', out[n++] = 'n', out[n++] = 'f';
        }
        return n;
    }
    if (neg) out[n++] = '-';
    if (be == 0 && frac == 0) {
        out[n++] = '0';
        return n;
    }
    uint64_t m;
    int e2;
    if (be == 0) {
        m = frac;
        e2 = -1074;
    } else {
        m = frac | (1ull << 52);
        e2 = be - 1075;
    }
    // decimal exponent estimate from the binary one (exact correction below)
    const double av = v < 0 ? -v : v;
#ifdef __CUDA_ARCH__
    int k = (int)floor(log10(av));
#else
    int k = (int)std::floor(std::log10(av));
#endif
    // k = floor(log10 |v|) exactly: 10^16 <= floor(|v| 10^(16-k)) < 10^17
    uint64_t D = 0, Fl = 0;
    const uint64_t lo = 10000000000000000ull, hi = 100000000000000000ull;
    for (int it = 0; it < 16; ++it) {
        const int rc = scaled_digits(m, e2, 16 - k, T, D, Fl);
        if (rc) {  // estimate far off: move toward the right magnitude
            k += rc;
            continue;
        }
        if (Fl >= hi) {
            ++k;
            continue;
        }
        if (Fl < lo) {
            --k;
            continue;
        }
        break;
    }
    if (D == hi) {  // rounding carried into an 18th digit: 9.99..95 -> 1.0e(k+1)
        D = lo;
        ++k;
    }
    // D has 17 digits d0..d16; X = k
    char dig[17];
    {
        uint64_t x = D;
        for (int q = 16; q >= 0; --q) {
            dig[q] = (char)('0' + x % 10u);
            x /= 10u;
        }
    }
    int last = 16;  // last significant digit after stripping trailing zeros
    while (last > 0 && dig[last] == '0') --last;
    const int X = k;
    if (X < -4 || X >= 17) {
        out[n++] = dig[0];
        if (last >= 1) {
            out[n++] = '.';
            for (int q = 1; q <= last; ++q) out[n++] = dig[q];
        }
        out[n++] = 'e';
        int ex = X;
        if (ex < 0) {
            out[n++] = '-';
            ex = -ex;
        } else {
            out[n++] = '+';
        }
        if (ex < 10) out[n++] = '0';
        n += put_uint(out + n, (uint64_t)ex);
        return n;
    }
    if (X >= 0) {
        for (int q = 0; q <= X; ++q) out[n++] = dig[q];
        if (last > X) {
            out[n++] = '.';
            for (int q = X + 1; q <= last; ++q) out[n++] = dig[q];
        }
        return n;
    }
    out[n++] = '0';
    out[n++] = '.';
    for (int q = 0; q < -X - 1; ++q) out[n++] = '0';
    for (int q = 0; q <= last; ++q) out[n++] = dig[q];
    return n;
}

}  // namespace silt_csv
