/* TEST INFRASTRUCTURE ONLY (oracle). See fftw3.h for scope.
 *
 * Stockham autosort, decimation in frequency, radices 4,2,3,5,7 plus a
 * generic O(p^2) butterfly for any other prime factor.  Stage with radix r
 * on a remaining length n_cur = r*m and stride s:
 *   y[q + s*(r*p + k)] = w_{n_cur}^{p*k} * sum_j x[q + s*(p + j*m)] w_r^{j*k}
 * which after all stages leaves X[k] in natural order.  All arithmetic is
 * double; twiddles come from one table w_n^i (i < n) built with cos/sin in
 * double, so the only fp32 rounding is the final store.
 */
#include "fftw3.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef struct { double re, im; } dcx;

struct fftwf_plan_s {
    int n;
    int sign;
    fftwf_complex* in;
    fftwf_complex* out;
    int nfac;
    int fac[64];
    dcx* tw;      /* tw[i] = exp(sign*2*pi*i*i/n), i < n */
    dcx* a;       /* work buffers */
    dcx* b;
    double c3[3], s3[3], c5[5], s5[5], c7[7], s7[7];
};

fftwf_complex* fftwf_alloc_complex(size_t n) {
    void* p = NULL;
    if (posix_memalign(&p, 64, (n ? n : 1) * sizeof(fftwf_complex)) != 0) return NULL;
    return (fftwf_complex*)p;
}

void fftwf_free(void* p) { free(p); }

fftwf_plan fftwf_plan_dft_1d(int n, fftwf_complex* in, fftwf_complex* out, int sign, unsigned flags) {
    (void)flags;
    if (n < 1) return NULL;
    struct fftwf_plan_s* p = (struct fftwf_plan_s*)calloc(1, sizeof(*p));
    p->n = n;
    p->sign = sign;
    p->in = in;
    p->out = out;
    int r = n;
    while (r % 4 == 0) { p->fac[p->nfac++] = 4; r /= 4; }
    while (r % 2 == 0) { p->fac[p->nfac++] = 2; r /= 2; }
    for (int f = 3; r > 1; f += 2)
        while (r % f == 0) { p->fac[p->nfac++] = f; r /= f; }
    p->tw = (dcx*)malloc(sizeof(dcx) * (size_t)n);
    for (int i = 0; i < n; ++i) {
        /* exact argument reduction: angle = 2*pi*i/n */
        double ang = 2.0 * M_PI * (double)i / (double)n;
        p->tw[i].re = cos(ang);
        p->tw[i].im = (double)sign * sin(ang);
    }
    for (int e = 0; e < 7; ++e) {
        if (e < 3) { p->c3[e] = cos(2.0 * M_PI * e / 3.0); p->s3[e] = sign * sin(2.0 * M_PI * e / 3.0); }
        if (e < 5) { p->c5[e] = cos(2.0 * M_PI * e / 5.0); p->s5[e] = sign * sin(2.0 * M_PI * e / 5.0); }
        p->c7[e] = cos(2.0 * M_PI * e / 7.0); p->s7[e] = sign * sin(2.0 * M_PI * e / 7.0);
    }
    p->a = (dcx*)malloc(sizeof(dcx) * (size_t)n);
    p->b = (dcx*)malloc(sizeof(dcx) * (size_t)n);
    return p;
}

void fftwf_destroy_plan(fftwf_plan p) {
    if (!p) return;
    free(p->tw);
    free(p->a);
    free(p->b);
    free(p);
}

static inline dcx cmul(dcx x, dcx y) {
    dcx r = {x.re * y.re - x.im * y.im, x.re * y.im + x.im * y.re};
    return r;
}

static void stage(const struct fftwf_plan_s* P, int r, int m, int s, const dcx* x, dcx* y) {
    const int n = P->n;
    const int ncur = r * m;
    const int twstep = n / ncur;          /* w_{ncur}^e = tw[e * twstep] */
    const double sg = (double)P->sign;
    for (int p = 0; p < m; ++p) {
        dcx w[r];
        for (int k = 0; k < r; ++k) w[k] = P->tw[(size_t)p * k * twstep];
        for (int q = 0; q < s; ++q) {
            dcx a[r];
            for (int j = 0; j < r; ++j) a[j] = x[q + (size_t)s * (p + (size_t)j * m)];
            dcx o[r];
            if (r == 2) {
                o[0].re = a[0].re + a[1].re; o[0].im = a[0].im + a[1].im;
                o[1].re = a[0].re - a[1].re; o[1].im = a[0].im - a[1].im;
            } else if (r == 4) {
                dcx t0 = {a[0].re + a[2].re, a[0].im + a[2].im};
                dcx t1 = {a[0].re - a[2].re, a[0].im - a[2].im};
                dcx t2 = {a[1].re + a[3].re, a[1].im + a[3].im};
                dcx t3 = {a[1].re - a[3].re, a[1].im - a[3].im};
                /* multiply t3 by sign*i */
                dcx t3i = {-sg * t3.im, sg * t3.re};
                o[0].re = t0.re + t2.re; o[0].im = t0.im + t2.im;
                o[2].re = t0.re - t2.re; o[2].im = t0.im - t2.im;
                o[1].re = t1.re + t3i.re; o[1].im = t1.im + t3i.im;
                o[3].re = t1.re - t3i.re; o[3].im = t1.im - t3i.im;
            } else if (r == 3 || r == 5 || r == 7) {
                /* odd prime: pair j with r-j (real cos part, imag sin part) */
                const int h = (r - 1) / 2;
                dcx sp[3], sm[3];
                o[0] = a[0];
                for (int j = 1; j <= h; ++j) {
                    sp[j - 1].re = a[j].re + a[r - j].re; sp[j - 1].im = a[j].im + a[r - j].im;
                    sm[j - 1].re = a[j].re - a[r - j].re; sm[j - 1].im = a[j].im - a[r - j].im;
                    o[0].re += sp[j - 1].re; o[0].im += sp[j - 1].im;
                }
                const double* C = (r == 3) ? P->c3 : (r == 5) ? P->c5 : P->c7;
                const double* S = (r == 3) ? P->s3 : (r == 5) ? P->s5 : P->s7;
                for (int k = 1; k <= h; ++k) {
                    double cr = a[0].re, ci = a[0].im, dr = 0.0, di = 0.0;
                    for (int j = 1; j <= h; ++j) {
                        int e = (j * k) % r;
                        cr += sp[j - 1].re * C[e]; ci += sp[j - 1].im * C[e];
                        dr += sm[j - 1].re * S[e]; di += sm[j - 1].im * S[e];
                    }
                    /* X_k = c + i*d_sin ; X_{r-k} = c - i*d_sin (S carries the sign) */
                    o[k].re = cr - di; o[k].im = ci + dr;
                    o[r - k].re = cr + di; o[r - k].im = ci - dr;
                }
            } else {
                /* generic DFT of length r (other primes) */
                for (int k = 0; k < r; ++k) {
                    double re = 0.0, im = 0.0;
                    for (int j = 0; j < r; ++j) {
                        dcx wj = P->tw[(size_t)((long long)j * k % r) * (n / r)];
                        re += a[j].re * wj.re - a[j].im * wj.im;
                        im += a[j].re * wj.im + a[j].im * wj.re;
                    }
                    o[k].re = re;
                    o[k].im = im;
                }
            }
            for (int k = 0; k < r; ++k) y[q + (size_t)s * ((size_t)r * p + k)] = k ? cmul(o[k], w[k]) : o[0];
        }
    }
}

static void run(const struct fftwf_plan_s* P, const fftwf_complex* in, fftwf_complex* out) {
    const int n = P->n;
    dcx* x = P->a;
    dcx* y = P->b;
    for (int i = 0; i < n; ++i) { x[i].re = in[i][0]; x[i].im = in[i][1]; }
    int s = 1, ncur = n;
    for (int f = 0; f < P->nfac; ++f) {
        int r = P->fac[f];
        int m = ncur / r;
        stage(P, r, m, s, x, y);
        dcx* t = x; x = y; y = t;
        s *= r;
        ncur = m;
    }
    for (int i = 0; i < n; ++i) { out[i][0] = (float)x[i].re; out[i][1] = (float)x[i].im; }
}

void fftwf_execute(const fftwf_plan p) { run(p, p->in, p->out); }

void fftwf_execute_dft(const fftwf_plan p, fftwf_complex* in, fftwf_complex* out) { run(p, in, out); }
