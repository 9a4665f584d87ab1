// hs_host.cu -- host-side helpers of the C ABI (no device code).
//
// hs_widen_phases: the f64 phases of an fp32 solve from their 4-byte codes
// (hs_phase_code, csrc/hs_kernels.cuh): (double)p, except that the fp32
// atan2's +-pi_f32 wrap to -+pi_f32 +- 2 pi exactly as hs_phase_f64 does on
// the device, so the result is bit-identical to a device-side f64 store while
// the device->host copy moves 4 instead of 8 bytes per pixel.  Runs on all
// host threads (a persistent pool) with non-temporal stores
// (tools/widen_probe.c: 3.7 ms per 33.4 M pixels on the B200 box's 16 cores).
#include <immintrin.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#include <condition_variable>
#include <mutex>
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

// Persistent widening workers: one job at a time (the slot's widen stream
// runs its host functions in order), split into equal parts; the calling
// thread (the CUDA driver's host-function thread) takes part 0.  Spawning
// threads per call cost ~0.3 ms per chunk; waking parked workers costs a
// few microseconds, so a download can be widened in small chunks while they
// are still in the last-level cache.
class WidenPool {
  public:
    explicit WidenPool(unsigned nt) : nt_(nt)
    {
        for (unsigned t = 1; t < nt_; ++t) workers_.emplace_back([this, t] { loop(t); });
    }
    ~WidenPool()
    {
        {
            std::lock_guard<std::mutex> g(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto &w : workers_) w.join();
    }
    unsigned threads() const { return nt_; }
    void run(const float *src, double *dst, int64_t n, unsigned parts)
    {
        {
            std::lock_guard<std::mutex> g(mu_);
            src_ = src;
            dst_ = dst;
            n_ = n;
            parts_ = parts;
            pending_ = parts - 1;
            ++gen_;
        }
        cv_.notify_all();
        part(0);
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [this] { return pending_ == 0; });
    }

  private:
    void part(unsigned t)
    {
        const int64_t per = (n_ + parts_ - 1) / parts_;
        const int64_t lo = std::min<int64_t>(n_, (int64_t)t * per), hi = std::min<int64_t>(n_, lo + per);
        if (hi > lo) widen_run(src_ + lo, dst_ + lo, hi - lo);
    }
    void loop(unsigned t)
    {
        uint64_t seen = 0;
        for (;;) {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
            if (stop_) return;
            seen = gen_;
            const bool mine = t < parts_;
            lk.unlock();
            if (!mine) continue;
            part(t);
            lk.lock();
            if (--pending_ == 0) done_cv_.notify_one();
        }
    }
    static void widen_run(const float *src, double *dst, int64_t n)
    {
        static const bool avx2 = __builtin_cpu_supports("avx2");
        if (avx2) widen_avx2(src, dst, n);
        else widen_scalar(src, dst, n);
    }
    unsigned nt_;
    std::vector<std::thread> workers_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    uint64_t gen_ = 0;
    bool stop_ = false;
    const float *src_ = nullptr;
    double *dst_ = nullptr;
    int64_t n_ = 0;
    unsigned parts_ = 1, pending_ = 0;
};

unsigned widen_threads()
{
    static const unsigned env_nt = getenv("HS_WIDEN_THREADS") ? (unsigned)atoi(getenv("HS_WIDEN_THREADS")) : 0;
    // all cores but two: the solve's host thread and the CUDA driver's own
    // threads keep running beside the widening (14 of 16 beat 16 of 16)
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    return env_nt ? env_nt : (hw > 4 ? hw - 2 : hw);
}

}  // namespace

extern "C" void hs_widen_phases(const float *src, double *dst, int64_t n)
{
    static WidenPool pool(widen_threads());  // created on first use, lives for the process
    const int64_t min_per = 1 << 16;
    const unsigned parts = (unsigned)std::min<int64_t>(pool.threads(), std::max<int64_t>(1, n / min_per));
    if (parts <= 1) {
        if (__builtin_cpu_supports("avx2")) widen_avx2(src, dst, n);
        else widen_scalar(src, dst, n);
        return;
    }
    pool.run(src, dst, n, parts);
}
