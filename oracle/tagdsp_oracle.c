/* TEST INFRASTRUCTURE ONLY (oracle) -- never linked into the product.
 *
 * Plain-C restatement of the reference tagdsp hot path
 * (/root/reference/proj, cited file:line), used by tests/ and bench.py's
 * cpu_baseline leg as the checker.  Arithmetic follows the reference
 * operation by operation (float where it uses float, double where it
 * accumulates in double, std::abs(complex<float>) == hypotf), and the FFT is
 * the same FFTW-API shim the compiled reference uses (oracle/fftw_shim), so
 * on identical inputs the restatement reproduces oracle/_ref bit for bit
 * (tests/test_oracle.py pins that, plus the reference's own golden values).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "fftw3.h"
#include "tagdsp_gpu_types.h"

typedef struct {
    float re, im;
} cf;

static inline cf cmulf(cf a, cf b) {
    cf r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
    return r;
}

/* ---- codegen.hpp:11-17 / codegen.cpp:10-38 ------------------------------ */
uint64_t tdo_splitmix64(uint64_t* state) {
    *state += 0x9E3779B97F4A7C15ULL;
    uint64_t z = *state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

typedef struct {
    uint64_t state;
    int have_spare;
    float spare;
} tdo_rng;

/* GaussianRng::next (codegen.cpp:10-24) */
static float rng_next(tdo_rng* g) {
    if (g->have_spare) {
        g->have_spare = 0;
        return g->spare;
    }
    double u1 = ((double)(tdo_splitmix64(&g->state) >> 11) + 1.0) * 0x1p-53;
    double u2 = (double)(tdo_splitmix64(&g->state) >> 11) * 0x1p-53;
    double r = sqrt(-2.0 * log(u1));
    double a = 2.0 * M_PI * u2;
    g->spare = (float)(r * sin(a));
    g->have_spare = 1;
    return (float)(r * cos(a));
}

void tdo_gaussian(uint64_t seed, uint64_t n, float* out) {
    tdo_rng g = {seed, 0, 0.0f};
    for (uint64_t i = 0; i < n; ++i) out[i] = rng_next(&g);
}

/* gen_code (codegen.cpp:26-38) */
void tdo_gen_code(uint64_t seed, uint64_t packet_bits, uint8_t* bits) {
    uint64_t state = seed, word = 0;
    for (uint64_t i = 0; i < packet_bits; ++i) {
        if (i % 64 == 0) word = tdo_splitmix64(&state);
        bits[i] = (uint8_t)((word >> (i % 64)) & 1);
    }
}

static size_t spb_of(const tdg_modulation* m) {
    double spb = m->sample_rate / m->bit_rate;
    size_t n = (size_t)(spb + 0.5);
    return n; /* types.hpp:32-38 (caller validated) */
}

/* synth_replica (codegen.cpp:40-60); out interleaved re,im */
void tdo_synth_replica(const uint8_t* bits, uint64_t nbits, const tdg_modulation* m, uint64_t padded_len,
                       float* out) {
    size_t spb = spb_of(m);
    memset(out, 0, sizeof(float) * 2 * padded_len);
    double phase = 0.0;
    size_t i = 0;
    for (uint64_t b = 0; b < nbits; ++b) {
        double step = 2.0 * M_PI * (bits[b] ? m->freq_one : m->freq_zero) / m->sample_rate;
        for (size_t k = 0; k < spb; ++k, ++i) {
            out[2 * i] = (float)cos(phase);
            out[2 * i + 1] = (float)sin(phase);
            phase += step;
            if (phase > 64.0 * M_PI) phase = remainder(phase, 2.0 * M_PI);
        }
    }
}

/* ---- fft.cpp:93-101 ------------------------------------------------------ */
uint64_t tdo_pad_length(uint64_t n) {
    if (n < 1) return 0;
    for (uint64_t m = n;; ++m) {
        uint64_t r = m;
        const uint64_t ps[4] = {2, 3, 5, 7};
        for (int k = 0; k < 4; ++k)
            while (r % ps[k] == 0) r /= ps[k];
        if (r == 1) return m;
    }
}

/* PlanCache::forward / inverse (fft.cpp:46-67): inverse scaled by 1/n in float */
static void fft_fwd(cf* in, cf* out, size_t n) {
    fftwf_plan p = fftwf_plan_dft_1d((int)n, (fftwf_complex*)in, (fftwf_complex*)out, FFTW_FORWARD, FFTW_ESTIMATE);
    fftwf_execute(p);
    fftwf_destroy_plan(p);
}

static void fft_inv(cf* in, cf* out, size_t n) {
    fftwf_plan p = fftwf_plan_dft_1d((int)n, (fftwf_complex*)in, (fftwf_complex*)out, FFTW_BACKWARD, FFTW_ESTIMATE);
    fftwf_execute(p);
    fftwf_destroy_plan(p);
    float inv = 1.0f / (float)n;
    for (size_t i = 0; i < n; ++i) {
        out[i].re *= inv;
        out[i].im *= inv;
    }
}

/* ---- dsp.cpp ------------------------------------------------------------- */
/* mix (dsp.cpp:18-33) */
static void mix(cf* x, size_t n, double lo, int64_t start, double fs) {
    if (lo == 0.0 || n == 0) return;
    double step = -2.0 * M_PI * lo / fs;
    double phase0 = step * (double)start;
    double wr = cos(step), wi = sin(step);
    double cr = cos(phase0), ci = sin(phase0);
    for (size_t i = 0; i < n; ++i) {
        cf w = {(float)cr, (float)ci};
        x[i] = cmulf(x[i], w);
        double nr = cr * wr - ci * wi, ni = cr * wi + ci * wr;
        cr = nr;
        ci = ni;
        if ((i & 255) == 255) {
            double ph = step * (double)(start + (int64_t)i + 1);
            cr = cos(ph);
            ci = sin(ph);
        }
    }
}

/* fill_bandpass (dsp.cpp:37-58) */
static void fill_bandpass(double center, double width, size_t taps, double fs, cf* out) {
    double fc = width / 2.0, mid = (double)(taps - 1) / 2.0, sum = 0.0;
    double* lp = (double*)malloc(sizeof(double) * taps);
    for (size_t k = 0; k < taps; ++k) {
        double t = (double)k - mid;
        double x = 2.0 * fc * t / fs;
        double sinc = (x == 0.0) ? 1.0 : sin(M_PI * x) / (M_PI * x);
        double w = (taps == 1) ? 1.0 : 0.54 - 0.46 * cos(2.0 * M_PI * (double)k / (double)(taps - 1));
        lp[k] = sinc * w;
        sum += lp[k];
    }
    for (size_t k = 0; k < taps; ++k) {
        double t = (double)k - mid;
        double a = 2.0 * M_PI * center * t / fs;
        double g = lp[k] / sum;
        out[k].re = (float)(g * cos(a));
        out[k].im = (float)(g * sin(a));
    }
    free(lp);
}

/* fill_matched (dsp.cpp:60-66) */
static void fill_matched(double freq, size_t spb, double fs, cf* out) {
    for (size_t k = 0; k < spb; ++k) {
        double a = 2.0 * M_PI * freq * (double)(spb - 1 - k) / fs;
        out[k].re = (float)cos(a);
        out[k].im = (float)-sin(a);
    }
}

/* convolve_into (dsp.cpp:68-73) */
static void convolve_into(const cf* a, size_t na, const cf* b, size_t nb, cf* out) {
    memset(out, 0, sizeof(cf) * (na + nb - 1));
    for (size_t i = 0; i < na; ++i)
        for (size_t j = 0; j < nb; ++j) {
            cf p = cmulf(a[i], b[j]);
            out[i + j].re += p.re;
            out[i + j].im += p.im;
        }
}

/* ola_into (dsp.cpp:77-104): FFT overlap-add into the full convolution */
static void ola_into(const cf* x, size_t n, const cf* h, size_t m, cf* out_full, size_t out_len) {
    size_t fft_n = (size_t)tdo_pad_length(4 * m);
    size_t block = fft_n - m + 1;
    cf* hbuf = (cf*)calloc(fft_n, sizeof(cf));
    cf* hspec = (cf*)malloc(sizeof(cf) * fft_n);
    cf* xbuf = (cf*)malloc(sizeof(cf) * fft_n);
    cf* xspec = (cf*)malloc(sizeof(cf) * fft_n);
    cf* ybuf = (cf*)malloc(sizeof(cf) * fft_n);
    memcpy(hbuf, h, sizeof(cf) * m);
    fft_fwd(hbuf, hspec, fft_n);
    memset(out_full, 0, sizeof(cf) * out_len);
    for (size_t start = 0; start < n; start += block) {
        size_t len = (block < n - start) ? block : n - start;
        memset(xbuf, 0, sizeof(cf) * fft_n);
        memcpy(xbuf, x + start, sizeof(cf) * len);
        fft_fwd(xbuf, xspec, fft_n);
        for (size_t k = 0; k < fft_n; ++k) xspec[k] = cmulf(xspec[k], hspec[k]);
        fft_inv(xspec, ybuf, fft_n);
        size_t tail = len + m - 1;
        if (tail > out_len - start) tail = out_len - start;
        for (size_t k = 0; k < tail; ++k) {
            out_full[start + k].re += ybuf[k].re;
            out_full[start + k].im += ybuf[k].im;
        }
    }
    free(hbuf);
    free(hspec);
    free(xbuf);
    free(xspec);
    free(ybuf);
}

/* demodulate (dsp.cpp:147-157) */
static void demodulate(const cf* f1, const cf* f0, size_t n, float eps, float* d, float* u) {
    for (size_t i = 0; i < n; ++i) {
        float a1 = hypotf(f1[i].re, f1[i].im);
        float a0 = hypotf(f0[i].re, f0[i].im);
        u[i] = a1 - a0;
        float den = a1 + a0;
        d[i] = u[i] / (den > eps ? den : eps);
    }
}

/* demodulate_signal (dsp.cpp:159-191) on complex input x (interleaved) */
int tdo_demodulate_signal(const float* xin, uint64_t n, int64_t start, double lo, const tdg_demod_config* cfg,
                          float* d, float* u) {
    if (n == 0) return 0;
    size_t spb = spb_of(&cfg->mod);
    size_t taps = (size_t)cfg->bandpass_taps, clen = taps + spb - 1;
    cf* y = (cf*)malloc(sizeof(cf) * n);
    memcpy(y, xin, sizeof(cf) * n);
    mix(y, n, lo, start, cfg->mod.sample_rate);
    cf* hbp = (cf*)malloc(sizeof(cf) * taps);
    cf* hm = (cf*)malloc(sizeof(cf) * spb);
    cf* h1c = (cf*)malloc(sizeof(cf) * clen);
    cf* h0c = (cf*)malloc(sizeof(cf) * clen);
    fill_bandpass(cfg->bandpass_center, cfg->bandpass_width, taps, cfg->mod.sample_rate, hbp);
    fill_matched(cfg->mod.freq_one, spb, cfg->mod.sample_rate, hm);
    convolve_into(hbp, taps, hm, spb, h1c);
    fill_matched(cfg->mod.freq_zero, spb, cfg->mod.sample_rate, hm);
    convolve_into(hbp, taps, hm, spb, h0c);
    size_t full = n + clen - 1;
    cf* f1 = (cf*)malloc(sizeof(cf) * full);
    cf* f0 = (cf*)malloc(sizeof(cf) * full);
    ola_into(y, n, h1c, clen, f1, full);
    ola_into(y, n, h0c, clen, f0, full);
    demodulate(f1, f0, n, cfg->eps, d, u);
    free(y);
    free(hbp);
    free(hm);
    free(h1c);
    free(h0c);
    free(f1);
    free(f0);
    return 0;
}

/* convert + demodulate_window (dsp.cpp:9-16, 193-197) */
int tdo_demodulate_window(const int16_t* iq, uint64_t n, int64_t start, const tdg_demod_config* cfg, float* d,
                          float* u) {
    float* x = (float*)malloc(sizeof(float) * 2 * (n ? n : 1));
    for (uint64_t i = 0; i < 2 * n; ++i) x[i] = (float)iq[i];
    int rc = tdo_demodulate_signal(x, n, start, cfg->lo_freq, cfg, d, u);
    free(x);
    return rc;
}

/* ---- detector.cpp -------------------------------------------------------- */
typedef struct {
    float* replica_d;
    cf* spectrum; /* conj(FFT(zero-padded replica_d)) */
    uint64_t nonzero_len, corr_len, window_len;
    float energy, abs_sum;
} tdo_code;

/* make_transformed (detector.cpp:11-48); returns 0 or 1 (invalid_argument) */
int tdo_make_transformed(const float* rd, const float* ru, uint64_t len, uint64_t window_len, uint64_t corr_len,
                         uint64_t* nonzero_len, float* energy, float* abs_sum, float* spectrum /* 2*corr_len */) {
    const float* sup = ru ? ru : rd;
    float peak = 0.0f;
    for (uint64_t i = 0; i < len; ++i) peak = fabsf(sup[i]) > peak ? fabsf(sup[i]) : peak;
    uint64_t n = 0;
    for (uint64_t i = 0; i < len; ++i)
        if (fabsf(sup[i]) > 1e-6f * peak) n = i + 1;
    *nonzero_len = n;
    if (window_len + n > corr_len + 1) return 1;
    double e = 0.0, a = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        e += (double)rd[i] * (double)rd[i];
        a += fabs((double)rd[i]);
    }
    *energy = (float)e;
    *abs_sum = (float)a;
    if (spectrum) {
        cf* buf = (cf*)calloc(corr_len, sizeof(cf));
        for (uint64_t i = 0; i < n; ++i) buf[i].re = rd[i];
        fft_fwd(buf, (cf*)spectrum, corr_len);
        for (uint64_t k = 0; k < corr_len; ++k) spectrum[2 * k + 1] = -spectrum[2 * k + 1];
        free(buf);
    }
    return 0;
}

/* prepare_code (detector.cpp:50-66): replica -> demod (lo = 0) -> make_transformed.
 * replica_d_out must hold window_len floats; returns 0, 1 (invalid_argument). */
int tdo_prepare_code(const uint8_t* bits, const tdg_demod_config* cfg, uint64_t window_len, uint64_t* nonzero_len,
                     float* energy, float* abs_sum, float* replica_d_out, float* spectrum, uint64_t* corr_len) {
    size_t spb = spb_of(&cfg->mod);
    uint64_t psamp = cfg->mod.packet_bits * spb;
    if (window_len < psamp) return 1;
    uint64_t clen = cfg->bandpass_taps + spb - 1;
    *corr_len = tdo_pad_length(window_len + psamp + clen);
    float* rep = (float*)malloc(sizeof(float) * 2 * window_len);
    tdo_synth_replica(bits, cfg->mod.packet_bits, &cfg->mod, window_len, rep);
    float* d = (float*)malloc(sizeof(float) * window_len);
    float* u = (float*)malloc(sizeof(float) * window_len);
    tdo_demodulate_signal(rep, window_len, 0, 0.0, cfg, d, u);
    int rc = tdo_make_transformed(d, u, window_len, window_len, *corr_len, nonzero_len, energy, abs_sum, spectrum);
    if (replica_d_out) memcpy(replica_d_out, d, sizeof(float) * (*nonzero_len));
    free(rep);
    free(d);
    free(u);
    return rc;
}

/* forward_window + correlate_spectrum (detector.cpp:70-88): xc[t], t < W */
static void xcorr_from_dspec(const cf* dspec, const float* spectrum, uint64_t N, uint64_t W, float* xc, cf* prod,
                             cf* time) {
    const cf* sp = (const cf*)spectrum;
    for (uint64_t k = 0; k < N; ++k) prod[k] = cmulf(dspec[k], sp[k]);
    fft_inv(prod, time, N);
    for (uint64_t t = 0; t < W; ++t) xc[t] = time[t].re;
}

/* batch_xcorr (detector.cpp:102-120): spectra n_codes x corr_len (interleaved),
 * out n_codes x W.  One forward transform for the batch. */
int tdo_batch_xcorr(const float* d, uint64_t W, const float* spectra, const uint64_t* nonzero_len, uint64_t n_codes,
                    uint64_t corr_len, float* out) {
    for (uint64_t c = 0; c < n_codes; ++c)
        if (W + nonzero_len[c] > corr_len + 1) return 1;
    cf* buf = (cf*)calloc(corr_len, sizeof(cf));
    cf* dspec = (cf*)malloc(sizeof(cf) * corr_len);
    cf* prod = (cf*)malloc(sizeof(cf) * corr_len);
    cf* time = (cf*)malloc(sizeof(cf) * corr_len);
    for (uint64_t i = 0; i < W; ++i) buf[i].re = d[i];
    fft_fwd(buf, dspec, corr_len);
    for (uint64_t c = 0; c < n_codes; ++c)
        xcorr_from_dspec(dspec, spectra + 2 * c * corr_len, corr_len, W, out + c * W, prod, time);
    free(buf);
    free(dspec);
    free(prod);
    free(time);
    return 0;
}

/* find_peak (detector.cpp:122-134): first index of max |xc| */
int tdo_find_peak(const float* xc, uint64_t n, uint64_t* j, float* value) {
    if (n == 0) return 1;
    uint64_t best = 0;
    float ba = fabsf(xc[0]);
    for (uint64_t i = 1; i < n; ++i) {
        float a = fabsf(xc[i]);
        if (a > ba) {
            ba = a;
            best = i;
        }
    }
    *j = best;
    *value = xc[best];
    return 0;
}

/* interpolate_peak (detector.cpp:136-145) */
float tdo_interpolate_peak(const float* xc, uint64_t n, uint64_t j) {
    if (j == 0 || j + 1 >= n) return 0.0f;
    float a = fabsf(xc[j - 1]), b = fabsf(xc[j]), c = fabsf(xc[j + 1]);
    float denom = a - 2.0f * b + c;
    if (denom >= 0.0f) return 0.0f;
    float delta = 0.5f * (a - c) / denom;
    return delta < -0.5f ? -0.5f : (delta > 0.5f ? 0.5f : delta);
}

/* statistics (detector.cpp:147-165) */
void tdo_statistics(const float* d, const float* u, uint64_t W, const float* rd, uint64_t n, uint64_t j, float* w_c,
                    float* q, float* p_c, int* partial) {
    uint64_t avail = j < W ? W - j : 0;
    uint64_t count = n < avail ? n : avail;
    *partial = count < n;
    double w = 0.0, qq = 0.0, p = 0.0;
    for (uint64_t i = 0; i < count; ++i) {
        double di = d[j + i];
        w += (double)rd[i] * di;
        qq += di * di;
        p += (double)rd[i] * (double)u[j + i];
    }
    *w_c = (float)w;
    *q = (float)qq;
    *p_c = (float)p;
}

/* detect (detector.cpp:167-206) for codes given by replica_d/spectrum. */
int tdo_detect(const float* d, const float* u, uint64_t W, const float* spectra, const float* const* replicas,
               const uint64_t* nonzero_len, const float* energy, uint64_t n_codes, uint64_t corr_len, float threshold,
               int64_t window_start, double fs, int32_t bin, tdg_detection* out) {
    float* xc = (float*)malloc(sizeof(float) * W * (n_codes ? n_codes : 1));
    int rc = tdo_batch_xcorr(d, W, spectra, nonzero_len, n_codes, corr_len, xc);
    if (rc) {
        free(xc);
        return rc;
    }
    for (uint64_t c = 0; c < n_codes; ++c) {
        const float* x = xc + c * W;
        uint64_t j;
        float value;
        tdo_find_peak(x, W, &j, &value);
        float delta = tdo_interpolate_peak(x, W, j);
        float wc, q, pc;
        int partial;
        tdo_statistics(d, u, W, replicas[c], nonzero_len[c], j, &wc, &q, &pc, &partial);
        tdg_detection* o = out + c;
        memset(o, 0, sizeof(*o));
        o->code_index = (int32_t)c;
        o->bin = bin;
        o->window_start = window_start;
        o->peak_index = j;
        o->subsample_offset = delta;
        o->peak_value = value;
        o->w_c = wc;
        o->q = q;
        o->p_c = pc;
        o->partial = (uint8_t)partial;
        float denom = sqrtf(q * energy[c]);
        o->score = (denom > 0.0f) ? wc / denom : 0.0f;
        o->toa_seconds = ((double)window_start + (double)j + (double)delta) / fs;
        o->accepted = !partial && o->score >= threshold;
    }
    free(xc);
    return 0;
}
