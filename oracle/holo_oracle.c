/*
 * holo_oracle.c -- CPU restatement of the reference hot-path kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker (and the CPU
 * baseline timed by bench.py's cpu_baseline / --impl reference legs).  The
 * product path (paper_2003_05293_b200) never links, loads or calls it.
 *
 * It restates, in plain C with fp64 arithmetic and no FMA contraction
 * (built with -O2 -ffp-contract=off), the three numba @njit kernels of the
 * reference package `holospots`:
 *
 *   or_build_tables  <- holospots/kernels.py:78-96   (_build_tables)
 *   or_superpose     <- holospots/kernels.py:99-119  (_superpose_kernel)
 *   or_forward       <- holospots/kernels.py:122-144 (_forward_kernel)
 *
 * Operation order inside every expression follows the reference so that
 * the results reproduce numba/LLVM's output bit for bit (LLVM does not
 * contract fmul/fadd without fast-math, and both call glibc's cos/sin/
 * atan2).  Parallelism is OpenMP over the same independent units the
 * reference parallelises with prange (pixels for the backward pass, whole
 * chunks for the forward pass), so results never depend on thread count.
 *
 * Extra (not in the reference): or_superpose_mag also returns |S_p| so
 * the parity tests can mask ill-conditioned pixels.
 */
#include <math.h>
#include <stdint.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* kernels.py:78-96.  Tables are row-major [side][n]. */
void or_build_tables(int64_t side, const double *axis, double c1, double c2,
                     int64_t n, const double *sx, const double *sy,
                     const double *sz, double *gx_re, double *gx_im,
                     double *gy_re, double *gy_im)
{
    for (int64_t j = 0; j < side; ++j) {
        const double v = axis[j];
        const double v2 = v * v;
        for (int64_t k = 0; k < n; ++k) {
            const double tx = c1 * sx[k] * v + c2 * sz[k] * v2;
            gx_re[j * n + k] = cos(tx);
            gx_im[j * n + k] = sin(tx);
            const double ty = c1 * sy[k] * v + c2 * sz[k] * v2;
            gy_re[j * n + k] = cos(ty);
            gy_im[j * n + k] = sin(ty);
        }
    }
}

/* kernels.py:99-119.  u = gx * coef (formed by the caller, kernels.py:206-210),
 * v = gy.  out has stop-start entries.  mag (optional) receives |S_p|. */
void or_superpose_mag(const int64_t *cols, const int64_t *rows, int64_t start,
                      int64_t stop, int64_t n, const double *u_re,
                      const double *u_im, const double *v_re,
                      const double *v_im, double *out, double *mag,
                      int threads)
{
    const double pi = 3.141592653589793;
#ifdef _OPENMP
    if (threads < 1) threads = 1;
#pragma omp parallel for schedule(static) num_threads(threads)
#endif
    for (int64_t p = start; p < stop; ++p) {
        const int64_t c = cols[p];
        const int64_t r = rows[p];
        double sr = 0.0, si = 0.0;
        for (int64_t k = 0; k < n; ++k) {
            const double ar = u_re[c * n + k];
            const double ai = u_im[c * n + k];
            const double br = v_re[r * n + k];
            const double bi = v_im[r * n + k];
            sr += ar * br - ai * bi;
            si += ar * bi + ai * br;
        }
        if (sr == 0.0 && si == 0.0) {
            out[p - start] = 0.0;
        } else {
            const double ph = atan2(si, sr);
            out[p - start] = (ph == pi) ? -pi : ph;
        }
        if (mag) mag[p - start] = hypot(sr, si);
    }
}

void or_superpose(const int64_t *cols, const int64_t *rows, int64_t start,
                  int64_t stop, int64_t n, const double *u_re,
                  const double *u_im, const double *v_re, const double *v_im,
                  double *out, int threads)
{
    or_superpose_mag(cols, rows, start, stop, n, u_re, u_im, v_re, v_im, out,
                     (double *)0, threads);
}

/* kernels.py:122-144.  part_* are [nchunks][n]; chunk kc covers storage
 * pixels [start + kc*chunk, min(stop, start + (kc+1)*chunk)), summed left
 * to right. */
void or_forward(const int64_t *cols, const int64_t *rows, const double *amp,
                const double *phi, int64_t start, int64_t stop, int64_t chunk,
                int64_t n, const double *gx_re, const double *gx_im,
                const double *gy_re, const double *gy_im, int64_t nchunks,
                double *part_re, double *part_im, int threads)
{
#ifdef _OPENMP
    if (threads < 1) threads = 1;
#pragma omp parallel for schedule(static) num_threads(threads)
#endif
    for (int64_t kc = 0; kc < nchunks; ++kc) {
        const int64_t p0 = start + kc * chunk;
        const int64_t p1 = (stop < p0 + chunk) ? stop : p0 + chunk;
        double *pr = part_re + kc * n;
        double *pi_ = part_im + kc * n;
        for (int64_t k = 0; k < n; ++k) {
            pr[k] = 0.0;
            pi_[k] = 0.0;
        }
        for (int64_t p = p0; p < p1; ++p) {
            const int64_t c = cols[p];
            const int64_t r = rows[p];
            const double a = amp[p];
            const double br_ = a * cos(phi[p]);
            const double bi_ = -a * sin(phi[p]);
            for (int64_t k = 0; k < n; ++k) {
                const double gxr = gx_re[c * n + k], gxi = gx_im[c * n + k];
                const double gyr = gy_re[r * n + k], gyi = gy_im[r * n + k];
                const double tr = gxr * gyr - gxi * gyi;
                const double ti = gxr * gyi + gxi * gyr;
                pr[k] += br_ * tr - bi_ * ti;
                pi_[k] += br_ * ti + bi_ * tr;
            }
        }
    }
}

int or_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
