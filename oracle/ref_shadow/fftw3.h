/* TEST INFRASTRUCTURE ONLY - lets the reference's FFTW-based SQG model
 * (proj/src/{spectral,sqg}.cpp) compile unmodified against NVIDIA's cuFFTW
 * (option i).  cuFFTW implements the FFTW3 API on top of
 * cuFFT but lacks fftw_alloc_real / fftw_alloc_complex, which the reference
 * uses (proj/src/spectral.cpp:25-26, proj/src/sqg.cpp:106-109). */
#pragma once
#include <cufftw.h>
static inline double* fftw_alloc_real(size_t n) {
    return (double*)fftw_malloc(n * sizeof(double));
}
static inline fftw_complex* fftw_alloc_complex(size_t n) {
    return (fftw_complex*)fftw_malloc(n * sizeof(fftw_complex));
}
