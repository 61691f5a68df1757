/*
 * CPU ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of what the reference interpreter computes for the two
 * hot-path programs (minigpu.interp, /root/reference/pkg/src/minigpu/interp.py).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library, and only as the checker or as the
 * timed CPU baseline. The product (paper_2605_13864_b200/) never links it.
 *
 * Parity pinning: every function below is checked against the golden vectors
 * produced by the reference itself (tests/golden/gen_golden.py ->
 * tests/golden/golden.npz), see tests/test_oracle.py.
 *
 * Semantics restated:
 *  - transpose  : `out[x][y] = in[y][x]` over an H x W row-major `in`
 *                 (interp.py:282-300 loop nest, :259-277 Assign, Array.offset
 *                 row-major :61-70). A pure permutation: bit-exact for any cell
 *                 width (2/4/8 bytes), so bf16/fp64 bit patterns move untouched.
 *  - reduce f32 : `sum += arr[i]` for i ascending, each store rounded to
 *                 binary32 (interp.py:262-270 + f32() :43-44). Python adds the
 *                 two binary32 values in binary64 and rounds once more to
 *                 binary32; double rounding through binary64 is innocuous for
 *                 a binary32 add, so this equals a plain binary32 add.
 *  - reduce int : unbounded Python-int sum (interp.py:262-270, no f32 for int
 *                 cells). For int32 cells (CELL_BYTES = 4, intrinsics.py:35)
 *                 and N <= 2^32 the exact sum fits an int64.
 *  - reduce A.5 : per 512-element block b: s[t] = a[2t] + a[2t+1] (t < 256),
 *                 then for k = 0..7, h = 2^(7-k): s[t] = s[t] + s[t+h] for
 *                 t < h; partial p[b] = s[0]; then the host loop sums p[]
 *                 sequentially in binary32 (interp.py
 *                 :282-300 thread-for executed in ascending order).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <omp.h>

#define OR_EXPORT __attribute__((visibility("default")))

OR_EXPORT int or_max_threads(void) { return omp_get_max_threads(); }

/* Blocked transpose: out (cols x rows, pitch ld_out) = in^T (rows x cols, pitch ld_in). */
#define OR_BLK 64
#define OR_TRANSPOSE_BODY(T)                                                        \
    {                                                                               \
        const T *src = (const T *)in;                                               \
        T *dst = (T *)out;                                                          \
        int64_t nbr = (rows + OR_BLK - 1) / OR_BLK, nbc = (cols + OR_BLK - 1) / OR_BLK; \
        _Pragma("omp parallel for schedule(static) num_threads(nthreads)")          \
        for (int64_t b = 0; b < nbr * nbc; ++b) {                                   \
            int64_t r0 = (b / nbc) * OR_BLK, c0 = (b % nbc) * OR_BLK;               \
            int64_t r1 = r0 + OR_BLK < rows ? r0 + OR_BLK : rows;                   \
            int64_t c1 = c0 + OR_BLK < cols ? c0 + OR_BLK : cols;                   \
            for (int64_t c = c0; c < c1; ++c)                                       \
                for (int64_t r = r0; r < r1; ++r)                                   \
                    dst[c * ld_out + r] = src[r * ld_in + c];                       \
        }                                                                           \
    }

OR_EXPORT int or_transpose(const void *in, void *out, int64_t rows, int64_t cols,
                           int64_t ld_in, int64_t ld_out, int esize, int nthreads) {
    if (nthreads <= 0) nthreads = omp_get_max_threads();
    if (rows <= 0 || cols <= 0) return 0;
    switch (esize) {
    case 1: OR_TRANSPOSE_BODY(uint8_t); return 0;
    case 2: OR_TRANSPOSE_BODY(uint16_t); return 0;
    case 4: OR_TRANSPOSE_BODY(uint32_t); return 0;
    case 8: OR_TRANSPOSE_BODY(uint64_t); return 0;
    default: return -1;
    }
}

/* interp.py:262-270: sequential binary32 accumulation, i ascending. */
OR_EXPORT float or_reduce_f32_seq(const float *x, int64_t n) {
    volatile float s = 0.0f; /* volatile: forbid any reassociation/vectorisation */
    for (int64_t i = 0; i < n; ++i) s = s + x[i];
    return s;
}

/* Unbounded-int sum of int32 cells; exact in int64 for n <= 2^32. Integer
 * addition is associative, so the threaded split returns the same value. */
OR_EXPORT int64_t or_reduce_i32(const int32_t *x, int64_t n, int nthreads) {
    if (nthreads <= 0) nthreads = omp_get_max_threads();
    int64_t s = 0;
#pragma omp parallel for reduction(+ : s) schedule(static) num_threads(nthreads)
    for (int64_t i = 0; i < n; ++i) s += x[i];
    return s;
}

/* Appendix A.5 order: per-512 block tree partials, then sequential host sum.
 * Returns -1 if 512 does not divide n (exact_div, interp.py:209-214). */
OR_EXPORT int or_reduce_f32_tree512(const float *x, int64_t n, float *partials, float *result) {
    if (n % 512 != 0) return -1;
    int64_t nb = n / 512;
    for (int64_t b = 0; b < nb; ++b) {
        float s[256];
        const float *a = x + b * 512;
        for (int t = 0; t < 256; ++t) s[t] = a[2 * t] + a[2 * t + 1];
        for (int k = 0; k < 8; ++k) {
            int h = 1 << (7 - k);
            for (int t = 0; t < h; ++t) s[t] = s[t] + s[t + h];
        }
        partials[b] = s[0];
    }
    *result = or_reduce_f32_seq(partials, nb);
    return 0;
}

/* Reference value for tolerances: binary64 sum and sum of |x| (neumaier). */
OR_EXPORT void or_sum_f64(const float *x, int64_t n, double *sum, double *abssum) {
    double s = 0.0, c = 0.0, a = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double v = (double)x[i];
        double t = s + v;
        if ((s >= 0 ? s : -s) >= (v >= 0 ? v : -v)) c += (s - t) + v;
        else c += (v - t) + s;
        s = t;
        a += v >= 0 ? v : -v;
    }
    *sum = s + c;
    *abssum = a;
}

/* interp.py:262-270 for a float cell: `sum += v` is f32(old + v) with old and v
 * Python floats (binary64), i.e. a binary64 add rounded to binary32. Segmented
 * form for the vectorised interpreter (oracle/vinterp.py): segment g folds
 * v[ends[g-1] .. ends[g]) into acc[g] in order. Returns 1 if a finite sum
 * rounded to infinity (struct.pack("f") raises OverflowError there on older
 * CPythons and returns +-inf on 3.12+, :43-44; the caller applies the rule). */
OR_EXPORT int or_seg_f32_fold(const double *v, const int64_t *ends, int64_t nseg, double *acc) {
    int64_t b = 0;
    int ovf = 0;
    for (int64_t g = 0; g < nseg; ++g) {
        volatile double s = acc[g];
        for (int64_t i = b; i < ends[g]; ++i) {
            const double t = s + v[i];
            const float r = (float)t;
            if (isinf(r) && !isinf(t)) ovf = 1;
            s = (double)r;
        }
        acc[g] = s;
        b = ends[g];
    }
    return ovf;
}

/* Fast synthetic data (splitmix64) so the CPU legs do not spend minutes in numpy. */
static inline uint64_t or_splitmix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

OR_EXPORT void or_fill_u32(uint32_t *x, int64_t n, uint64_t seed, int nthreads) {
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(static) num_threads(nthreads)
    for (int64_t i = 0; i < n; ++i) x[i] = (uint32_t)(or_splitmix(seed * 0x100000001B3ull + (uint64_t)i) >> 32);
}
