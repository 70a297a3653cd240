// K1's throughput builds (two or four systems per thread; C2): the kernel
// template of k_batch2_impl.cuh instantiated in a translation unit of its own,
// compiled with ptxas register-usage level 2 (build.py PER_SOURCE_FLAGS).
#include "k_batch2_impl.cuh"

namespace osc {

cudaError_t launch_batch2_wide(int ns, const double *m, const double *C, double *x, double *v,
                               int64_t B, StepConsts k, int64_t nsteps, int64_t stride,
                               double *xs, double *vs, double *es, int64_t *first_bad,
                               int threads, bool fma, cudaStream_t stream, const CmpArgs *cmp,
                               Div2Plan plan)
{
    if (ns == 2)
        return launch_ns<2>(m, C, x, v, B, k, nsteps, stride, xs, vs, es, first_bad, threads, fma,
                            stream, cmp, plan);
    return launch_ns<4>(m, C, x, v, B, k, nsteps, stride, xs, vs, es, first_bad, threads, fma,
                        stream, cmp, plan);
}

}  // namespace osc
