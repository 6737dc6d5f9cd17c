/* TEST INFRASTRUCTURE ONLY (oracle). Not part of the product path.
 *
 * Minimal FFTW3 single-precision API shim so the reference library
 * (/root/reference/proj/src/fft.cpp) can be compiled unmodified in an image
 * without libfftw3f.  Covers exactly the calls the reference makes:
 *   fftwf_alloc_complex   proj/src/fft.cpp:36-37
 *   fftwf_plan_dft_1d     proj/src/fft.cpp:39   (FFTW_ESTIMATE)
 *   fftwf_execute         proj/src/fft.cpp:51,62
 *   fftwf_destroy_plan    proj/src/fft.cpp:17
 *   fftwf_free            proj/src/fft.cpp:18-19
 * Semantics follow the published FFTW3 definition: unnormalised DFT,
 * FFTW_FORWARD = -1 (exp(-2*pi*i*jk/n)), FFTW_BACKWARD = +1.
 * Arithmetic is a mixed-radix Stockham FFT carried out in double precision
 * and rounded to float on output, i.e. at least as accurate as FFTW's fp32
 * codelets.  FFTW version is unpinned by the reference (proj/README.md:10-11);
 * the paper used 3.3.8.
 */
#ifndef TAGDSP_ORACLE_FFTW3_SHIM_H
#define TAGDSP_ORACLE_FFTW3_SHIM_H
#include <stddef.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef float fftwf_complex[2];
typedef struct fftwf_plan_s* fftwf_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_ESTIMATE (1U << 6)

fftwf_complex* fftwf_alloc_complex(size_t n);
void fftwf_free(void* p);
fftwf_plan fftwf_plan_dft_1d(int n, fftwf_complex* in, fftwf_complex* out, int sign, unsigned flags);
void fftwf_execute(const fftwf_plan plan);
void fftwf_destroy_plan(fftwf_plan plan);

/* Shim extension (oracle restatement + tests): transform explicit buffers
 * with a plan's size and sign (FFTW's new-array execute). */
void fftwf_execute_dft(const fftwf_plan plan, fftwf_complex* in, fftwf_complex* out);

#ifdef __cplusplus
}
#endif
#endif
