/*
 * Plain-C use of the B200 RK4 library through include/osc_b200.h only:
 * no Python, no torch.  Integrates a batch of independent 2-DOF systems
 * (BASELINE configs[1] shape, smaller B) twice -- through the synchronous
 * host-pointer entry point and through the device-pointer one on a CUDA
 * stream -- checks the two agree bit for bit, shows the error contract
 * (OSC_INVALID for a bad dt, OSC_NONFINITE + first_bad for a divergent system)
 * and runs one chain sharded over the GPUs of the process (osc_rk4_chain_sharded)
 * against the single-GPU chain.
 *
 * build:  gcc -O2 -I include examples/c_abi_demo.c -o c_abi_demo \
 *           -L paper_1702_02207_b200 -l:libosc_b200.so -L/usr/local/cuda/lib64 -lcudart \
 *           -Wl,-rpath,$PWD/paper_1702_02207_b200
 * run:    ./c_abi_demo [dump.bin]   (prints "ok" and exits 0; with a path, also
 *         writes m, C, x0, v0, x, v as raw float64 [2][B] each, so a checker can
 *         compare the result with the CPU oracle)
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "osc_b200.h"

#define B 4096
#define NSTEPS 2000

static double urand(uint64_t *s)
{
    *s = *s * 6364136223846793005ull + 1442695040888963407ull;
    return (double)(*s >> 11) * (1.0 / 9007199254740992.0);
}

int main(int argc, char **argv)
{
    static double m[2 * B], C[2 * B], x[2 * B], v[2 * B], x2[2 * B], v2[2 * B], x0[2 * B],
        v0[2 * B];
    static int64_t fb[B], fb2[B];
    uint64_t seed = 1702;
    for (int i = 0; i < 2 * B; ++i) {
        m[i] = 0.5 + 1.5 * urand(&seed);
        C[i] = 500.0 + 1500.0 * urand(&seed);
        x[i] = 2.0 * urand(&seed) - 1.0;
        v[i] = 0.0;
    }
    memcpy(x0, x, sizeof x);
    memcpy(v0, v, sizeof v);
    memcpy(x2, x, sizeof x);
    memcpy(v2, v, sizeof v);

    if (osc_abi_version() != OSC_ABI_VERSION) {
        fprintf(stderr, "ABI mismatch\n");
        return 1;
    }
    /* 1. host-pointer form: synchronous, copies inside */
    int rc = osc_rk4_batch2_host(m, C, x, v, B, 1e-4, NSTEPS, NSTEPS, NULL, NULL, fb);
    if (rc != OSC_OK) {
        fprintf(stderr, "host call failed: %s\n", osc_last_error());
        return 1;
    }

    /* 2. device-pointer form on a stream */
    double *dm, *dC, *dx, *dv;
    int64_t *dfb;
    cudaStream_t st;
    cudaStreamCreate(&st);
    cudaMalloc((void **)&dm, sizeof m);
    cudaMalloc((void **)&dC, sizeof C);
    cudaMalloc((void **)&dx, sizeof x2);
    cudaMalloc((void **)&dv, sizeof v2);
    cudaMalloc((void **)&dfb, sizeof fb2);
    cudaMemcpyAsync(dm, m, sizeof m, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(dC, C, sizeof C, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(dx, x2, sizeof x2, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(dv, v2, sizeof v2, cudaMemcpyHostToDevice, st);
    rc = osc_rk4_batch2(dm, dC, dx, dv, B, 1e-4, NSTEPS, NSTEPS, NULL, NULL, NULL, dfb, 0, st);
    if (rc != OSC_OK) {
        fprintf(stderr, "device call failed: %s\n", osc_last_error());
        return 1;
    }
    cudaMemcpyAsync(x2, dx, sizeof x2, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(v2, dv, sizeof v2, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(fb2, dfb, sizeof fb2, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if (memcmp(x, x2, sizeof x) || memcmp(v, v2, sizeof v) || memcmp(fb, fb2, sizeof fb)) {
        fprintf(stderr, "host and device forms differ\n");
        return 1;
    }
    for (int i = 0; i < 2 * B; ++i)
        if (!isfinite(x[i]) || !isfinite(v[i])) {
            fprintf(stderr, "non-finite state\n");
            return 1;
        }

    if (argc > 1) {
        FILE *f = fopen(argv[1], "wb");
        if (!f) {
            perror(argv[1]);
            return 1;
        }
        fwrite(m, sizeof m, 1, f);
        fwrite(C, sizeof C, 1, f);
        fwrite(x0, sizeof x0, 1, f);
        fwrite(v0, sizeof v0, 1, f);
        fwrite(x, sizeof x, 1, f);
        fwrite(v, sizeof v, 1, f);
        fclose(f);
    }

    /* 3. the error contract */
    if (osc_rk4_batch2_host(m, C, x, v, B, -1.0, 10, 1, NULL, NULL, fb) != OSC_INVALID) {
        fprintf(stderr, "bad dt not rejected\n");
        return 1;
    }
    {
        /* the reference's parameter rule (oscillator.py:66-80): a zero mass is
         * rejected before anything runs, the offender named, x untouched */
        double m0 = m[B + 5], x5 = x[B + 5];
        m[B + 5] = 0.0;
        int which = -1;
        int64_t idx = -1;
        if (osc_rk4_batch2_host(m, C, x, v, B, 1e-4, 10, 10, NULL, NULL, fb) != OSC_INVALID ||
            !osc_last_invalid_parameter(&which, &idx) || which != 0 || idx != B + 5 ||
            x[B + 5] != x5) {
            fprintf(stderr, "zero mass not rejected (%s)\n", osc_last_error());
            return 1;
        }
        m[B + 5] = m0;
    }
    double mm[2] = {0.002, 0.002}, cc[2] = {20250.0, 20250.0}, xx[2] = {2.0, -3.0},
           vv[2] = {0.0, 0.0};
    int64_t bad = 0;
    rc = osc_rk4_batch2_host(mm, cc, xx, vv, 1, 2e-2, 1000, 1000, NULL, NULL, &bad);
    if (rc != OSC_NONFINITE || bad < 1) {
        fprintf(stderr, "divergence not reported (rc=%d, step=%lld)\n", rc, (long long)bad);
        return 1;
    }
    /* 4. one chain sharded over the GPUs of this process (here: device 0
     *    twice) == the single-GPU chain, byte for byte */
    {
        enum { S = 20000, STEPS = 100 };
        static double cm[S], cc[S], cx[S], cv[S], cx2[S], cv2[S];
        for (int i = 0; i < S; ++i) {
            cm[i] = 0.5 + 1.5 * urand(&seed);
            cc[i] = 500.0 + 1500.0 * urand(&seed);
            cx[i] = cx2[i] = 2.0 * urand(&seed) - 1.0;
            cv[i] = cv2[i] = 0.0;
        }
        int64_t fb1 = 0, fb2 = 0;
        const int devs[2] = {0, 0};
        if (osc_rk4_chains_host(cm, cc, cx, cv, 1, S, 1e-3, STEPS, STEPS, NULL, NULL, &fb1) != OSC_OK ||
            osc_rk4_chain_sharded(2, devs, cm, cc, cx2, cv2, S, 1e-3, STEPS, 0, &fb2, 0) != OSC_OK) {
            fprintf(stderr, "chain calls failed: %s\n", osc_last_error());
            return 1;
        }
        if (memcmp(cx, cx2, sizeof cx) || memcmp(cv, cv2, sizeof cv)) {
            fprintf(stderr, "sharded chain differs from the single-GPU chain\n");
            return 1;
        }
    }
    printf("ok: %d systems x %d steps, host == device form, sharded chain == single chain, "
           "diverging system tagged at step %lld (%s)\n", B, NSTEPS, (long long)bad,
           osc_last_error());
    cudaFree(dm);
    cudaFree(dC);
    cudaFree(dx);
    cudaFree(dv);
    cudaFree(dfb);
    cudaStreamDestroy(st);
    return 0;
}
