/* Host-side widening of fp32 phase codes to the f64 phases the C ABI returns
 * (hs_phase_f64's rule: (double)p, except +-pi_f32 -> -+pi_f32 +- 2 pi), timed
 * for one 32-hologram config-3 step (33.4 M pixels) at 1..N threads, with
 * plain and non-temporal stores.  Measures whether shipping 4-byte phases
 * over PCIe and widening on the host beats shipping 8-byte phases.
 *   gcc -O3 -march=native -fopenmp -o tools/widen_probe tools/widen_probe.c */
#include <immintrin.h>
#include <omp.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static double now(void)
{
    struct timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return t.tv_sec + t.tv_nsec * 1e-9;
}

static inline double widen(float p)
{
    if (p == 3.14159274101257324f) return 3.14159274101257324 - 6.283185307179586;
    if (p == -3.14159274101257324f) return -3.14159274101257324 + 6.283185307179586;
    return (double)p;
}

int main(void)
{
    const size_t n = 32ull * 1042356;
    float *a = aligned_alloc(64, n * 4);
    double *b = aligned_alloc(64, n * 8);
    for (size_t i = 0; i < n; i++) a[i] = (float)(i % 1000) * 0.001f;
    memset(b, 0, n * 8);
    int maxth = omp_get_max_threads();
    printf("host threads available: %d\n", maxth);
    for (int th = 1; th <= maxth; th *= 2) {
        double best = 1e9, best_nt = 1e9;
        for (int r = 0; r < 5; r++) {
            double t0 = now();
#pragma omp parallel for num_threads(th) schedule(static)
            for (size_t i = 0; i < n; i++) b[i] = widen(a[i]);
            double t = now() - t0;
            if (t < best) best = t;
            t0 = now();
#pragma omp parallel for num_threads(th) schedule(static)
            for (size_t i = 0; i < n; i += 4) {
                __m256d v = _mm256_set_pd(widen(a[i + 3]), widen(a[i + 2]), widen(a[i + 1]), widen(a[i]));
                _mm256_stream_pd(b + i, v);
            }
            _mm_sfence();
            t = now() - t0;
            if (t < best_nt) best_nt = t;
        }
        printf("threads %3d: %.2f ms plain, %.2f ms streaming stores\n", th, best * 1e3, best_nt * 1e3);
    }
    return 0;
}
