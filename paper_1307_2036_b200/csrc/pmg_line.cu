// Batched tridiagonal line solves on the device (paper Alg. 3, the scalar
// utility of reference tridiag.py:59-100 as a library entry point).
//
// The smoother's own column solves live inside the half-sweep kernels; this
// entry point solves arbitrary independent systems T_s x_s = f_s, one thread
// per system, with the arrays stored system-fastest (element k of system s at
// k * nsys + s) so every step of the elimination is one coalesced load per
// warp.  The elimination keeps the reciprocal pivots in the output array
// (x is the forward sweep's workspace) and reports the first row whose pivot
// fell below PIVOT_FLOOR in any system: the reference raises ZeroPivotError
// there (tridiag.py:79-90), the host wrapper does the same.
#include <atomic>
#include <cmath>
#include <string>

#include <cuda_runtime.h>

#include "../../include/pmg.h"

namespace pmg {
extern std::atomic<long long> g_launches;
int set_error(int code, const char *msg);
}

namespace {

constexpr double PIVOT_FLOOR = 1e-300;   // tridiag.py:17

// forward: piv_0 = a_0, w_0 = b_0 / piv_0, y_0 = f_0 / piv_0;
//          piv_k = a_k - c_{k-1} w_{k-1}, w_k = b_k / piv_k,
//          y_k = (f_k - c_{k-1} y_{k-1}) / piv_k
// backward: x_{n-1} = y_{n-1}, x_k = y_k - w_k x_{k+1}.
// w is kept in registers only for the current row: it is rebuilt on the way
// back from the stored y and the stored reciprocal pivot (ws), so the kernel
// needs one n-long scratch besides x.
__global__ void k_thomas_batch(int n, long long nsys, const double *__restrict__ a,
                               const double *__restrict__ b, const double *__restrict__ c,
                               const double *__restrict__ f, double *__restrict__ x,
                               double *__restrict__ ws, int *__restrict__ bad) {
    const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (s >= nsys) return;
    double wprev = 0.0, yprev = 0.0;
    for (int k = 0; k < n; ++k) {
        const long long q = (long long)k * nsys + s;
        const double piv = (k > 0) ? a[q] - wprev * c[q - nsys] : a[q];
        if (fabs(piv) < PIVOT_FLOOR) {
            atomicMin(bad, k);
            return;
        }
        // row 0 divides, later rows multiply by the reciprocal: the
        // reference's roundings (tridiag.py:84-96)
        double y, w;
        if (k == 0) {
            y = f[q] / piv;
            w = (n > 1) ? b[q] / piv : 0.0;
        } else {
            const double inv = 1.0 / piv;
            y = (f[q] - yprev * c[q - nsys]) * inv;
            w = (k + 1 < n) ? b[q] * inv : 0.0;
        }
        x[q] = y;
        ws[q] = w;
        wprev = w;
        yprev = y;
    }
    double xn = x[(long long)(n - 1) * nsys + s];
    for (int k = n - 2; k >= 0; --k) {
        const long long q = (long long)k * nsys + s;
        xn = x[q] - ws[q] * xn;
        x[q] = xn;
    }
}

}  // namespace

extern "C" int pmg_thomas_batch(int n, long long nsys, const double *a, const double *b,
                                const double *c, const double *f, double *x, double *work,
                                int *bad_row, void *stream) {
    if (n < 1 || nsys < 0 || !a || !f || !x || !work || !bad_row || (n > 1 && (!b || !c)))
        return pmg::set_error(PMG_ERR_VALUE, "thomas_batch: bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    // the device word the kernel lowers to the first failing row; work holds
    // n * nsys doubles of scratch followed by that word
    int *dbad = reinterpret_cast<int *>(work + (long long)n * nsys);
    const int big = 0x7fffffff;
    cudaError_t e = cudaMemcpyAsync(dbad, &big, sizeof(int), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess && nsys > 0) {
        const int T = 128;
        k_thomas_batch<<<(unsigned)((nsys + T - 1) / T), T, 0, st>>>(n, nsys, a, b, c, f, x, work,
                                                                     dbad);
        pmg::g_launches.fetch_add(1, std::memory_order_relaxed);
        e = cudaGetLastError();
    }
    int h = big;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h, dbad, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess)
        return pmg::set_error(PMG_ERR_CUDA, (std::string("thomas_batch: ") +
                                             cudaGetErrorString(e)).c_str());
    *bad_row = (h == big) ? -1 : h;
    if (h != big)
        return pmg::set_error(PMG_ERR_PIVOT,
                              ("zero pivot at row " + std::to_string(h)).c_str());
    return PMG_OK;
}

extern "C" long long pmg_thomas_work_doubles(int n, long long nsys) {
    return (long long)n * nsys + 1;
}
