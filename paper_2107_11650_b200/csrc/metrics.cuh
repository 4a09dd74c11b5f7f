// Image-quality metrics on the device (metrics.cu): host buffers in, FP64.
#pragma once
#include <cstddef>

namespace shlr_b200 {

// ssos (proj/src/io.cpp:105-117): x is m x n x j interleaved complex, out m x n.
void ssos_host(const double* x, size_t m, size_t n, size_t j, double* out);
// rlne (proj/src/metrics.cpp:9-21) over `count` pixels; throws InvalidArg for
// an identically zero reference.
double rlne_host(const double* ref, const double* rec, size_t count);
// mssim (proj/src/metrics.cpp:23-75): mean SSIM over 11 x 11 Gaussian windows.
double mssim_host(const double* ref, const double* rec, size_t rows, size_t cols);

}  // namespace shlr_b200
