// Analytic two-mode solutions and the numeric-vs-analytic error report for
// batches of 2-DOF systems (modal.py:98-162; see osc_modal.cuh).  The fused
// form -- the error accumulated inside the K1 time loop at every retained
// sample, with no samples written -- lives in k_batch2.cu.
#include "osc_kernels.h"
#include "osc_modal.cuh"

namespace osc {
namespace {

__global__ void modal_batch2_kernel(const double *__restrict__ m, const double *__restrict__ C,
                                    const double *__restrict__ x0, const double *__restrict__ v0,
                                    int64_t B, double *__restrict__ sol)
{
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < B;
         i += int64_t(gridDim.x) * blockDim.x) {
        const Modal2 s = analytic2(m[i], m[B + i], C[i], C[B + i], x0[i], x0[B + i], v0[i],
                                   v0[B + i]);
#pragma unroll
        for (int f = 0; f < kModalFields; ++f)
            sol[f * B + i] = s.f[f];
    }
}

// One system per thread, samples in order: xs is [nsamp][2][B], ts [nsamp].
__global__ void compare_batch2_kernel(const double *__restrict__ sol,
                                      const double *__restrict__ xs,
                                      const double *__restrict__ ts, int64_t nsamp, int64_t B,
                                      double *__restrict__ out)
{
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < B;
         i += int64_t(gridDim.x) * blockDim.x) {
        const Modal2 s = load_modal(sol, B, i);
        ErrAcc acc;
        for (int64_t k = 0; k < nsamp; ++k)
            acc.add_sample(s, ts[k], xs[k * 2 * B + i], xs[k * 2 * B + B + i]);
        out[i] = acc.max_err;
        out[B + i] = acc.rmse();
        out[2 * B + i] = acc.at_time;
    }
}

unsigned grid_for(int64_t B, int threads)
{
    const int64_t g = (B + threads - 1) / threads;
    return static_cast<unsigned>(g < 148 * 64 ? (g > 0 ? g : 1) : 148 * 64);
}

}  // namespace

cudaError_t launch_modal_batch2(const double *m, const double *C, const double *x0,
                                const double *v0, int64_t B, double *sol, cudaStream_t stream)
{
    modal_batch2_kernel<<<grid_for(B, 256), 256, 0, stream>>>(m, C, x0, v0, B, sol);
    return cudaGetLastError();
}

cudaError_t launch_compare_batch2(const double *sol, const double *xs, const double *ts,
                                  int64_t nsamp, int64_t B, double *out, cudaStream_t stream)
{
    compare_batch2_kernel<<<grid_for(B, 256), 256, 0, stream>>>(sol, xs, ts, nsamp, B, out);
    return cudaGetLastError();
}

}  // namespace osc
