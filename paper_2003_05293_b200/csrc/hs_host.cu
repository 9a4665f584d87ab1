// hs_host.cu -- host-side helpers of the C ABI (no device code).
//
// hs_widen_phases: the f64 phases of an fp32 solve from their 4-byte codes
// (hs_phase_code, csrc/hs_kernels.cuh): (double)p, except that the fp32
// atan2's +-pi_f32 wrap to -+pi_f32 +- 2 pi exactly as hs_phase_f64 does on
// the device, so the result is bit-identical to a device-side f64 store while
// the device->host copy moves 4 instead of 8 bytes per pixel.  Runs on all
// host threads with non-temporal stores (tools/widen_probe.c: 3.7 ms per
// 33.4 M pixels on the B200 box's 16 cores).
#include <immintrin.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#include <thread>
#include <vector>

namespace {

constexpr float kPiF = 3.14159274101257324f;
constexpr double kTwoPiD = 6.283185307179586;

inline double widen(float p)
{
    if (p == kPiF) return 3.14159274101257324 - kTwoPiD;
    if (p == -kPiF) return -3.14159274101257324 + kTwoPiD;
    return (double)p;
}

void widen_scalar(const float *src, double *dst, int64_t n)
{
    for (int64_t i = 0; i < n; ++i) dst[i] = widen(src[i]);
}

__attribute__((target("avx2"))) void widen_avx2(const float *src, double *dst, int64_t n)
{
    int64_t i = 0;
    // scalar head up to a 32-byte aligned destination
    while (i < n && (reinterpret_cast<uintptr_t>(dst + i) & 31)) {
        dst[i] = widen(src[i]);
        ++i;
    }
    const __m128 pi = _mm_set1_ps(kPiF), mpi = _mm_set1_ps(-kPiF);
    const __m256d fix_hi = _mm256_set1_pd(3.14159274101257324 - kTwoPiD);
    const __m256d fix_lo = _mm256_set1_pd(-3.14159274101257324 + kTwoPiD);
    for (; i + 4 <= n; i += 4) {
        const __m128 v = _mm_loadu_ps(src + i);
        __m256d d = _mm256_cvtps_pd(v);
        const __m256d is_hi = _mm256_castsi256_pd(_mm256_cvtepi32_epi64(_mm_castps_si128(_mm_cmpeq_ps(v, pi))));
        const __m256d is_lo = _mm256_castsi256_pd(_mm256_cvtepi32_epi64(_mm_castps_si128(_mm_cmpeq_ps(v, mpi))));
        d = _mm256_blendv_pd(d, fix_hi, is_hi);
        d = _mm256_blendv_pd(d, fix_lo, is_lo);
        _mm256_stream_pd(dst + i, d);
    }
    for (; i < n; ++i) dst[i] = widen(src[i]);
    _mm_sfence();
}

}  // namespace

extern "C" void hs_widen_phases(const float *src, double *dst, int64_t n)
{
    const bool avx2 = __builtin_cpu_supports("avx2");
    static const unsigned env_nt = getenv("HS_WIDEN_THREADS") ? (unsigned)atoi(getenv("HS_WIDEN_THREADS")) : 0;
    // all cores but two: the solve's host thread and the CUDA driver's own
    // threads keep running beside the widening (14 of 16 beat 16 of 16)
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    unsigned nt = env_nt ? env_nt : (hw > 4 ? hw - 2 : hw);
    const int64_t min_per = 1 << 18;
    nt = (unsigned)std::min<int64_t>(nt, std::max<int64_t>(1, n / min_per));
    auto run = [&](int64_t lo, int64_t hi) {
        if (avx2) widen_avx2(src + lo, dst + lo, hi - lo);
        else widen_scalar(src + lo, dst + lo, hi - lo);
    };
    if (nt <= 1) {
        run(0, n);
        return;
    }
    std::vector<std::thread> pool;
    pool.reserve(nt - 1);
    const int64_t per = (n + nt - 1) / nt;
    for (unsigned t = 1; t < nt; ++t) {
        const int64_t lo = std::min<int64_t>(n, t * per), hi = std::min<int64_t>(n, lo + per);
        pool.emplace_back(run, lo, hi);
    }
    run(0, std::min<int64_t>(n, per));
    for (auto &th : pool) th.join();
}
