/* vfmm_c_example.c -- the C ABI used from plain C (no CUDA headers, no Python): one periodic
 * FMM evaluation of N = n^3 lattice vortex particles through vfmm_evaluate_host (host buffers).
 *
 *   gcc -O2 -I include examples/vfmm_c_example.c -L paper_1110_2921_b200/lib -lvfmm \
 *       -Wl,-rpath,$PWD/paper_1110_2921_b200/lib -lm -o examples/vfmm_c_example
 *   ./examples/vfmm_c_example [n] > out.txt
 *
 * Writes "n p depth ms_total" and then the velocity and stretching of particle 0 and
 * particle N-1 (tests/test_gpu_parity.py compares them with the Python binding). */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "vfmm.h"

static int check(vfmm_ctx* ctx, vfmm_status s, const char* what) {
    if (s == VFMM_OK) return 0;
    fprintf(stderr, "%s: %s (%s)\n", what, vfmm_strerror(s),
            ctx ? vfmm_last_error_message(ctx) : "");
    return 1;
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 16;
    const int64_t N = (int64_t)n * n * n;
    vfmm_params prm;
    vfmm_params_default(&prm);            /* p = 10, 27^3 images, classical scheme, box 2 pi */
    prm.p = 6;
    prm.depth = 2;
    const float h = prm.box_len / (float)n;
    prm.sigma = h;                        /* overlap h / sigma = 1 */
    float* buf = (float*)malloc(sizeof(float) * 12 * (size_t)N);
    float *pos = buf, *gam = buf + 3 * N, *vel = buf + 6 * N, *dg = buf + 9 * N;
    for (int64_t i = 0; i < N; ++i) {     /* cell-centre lattice, x fastest; Taylor-Green-like */
        const float x = prm.box_lo + h * ((float)(i % n) + 0.5f);
        const float y = prm.box_lo + h * ((float)((i / n) % n) + 0.5f);
        const float z = prm.box_lo + h * ((float)(i / ((int64_t)n * n)) + 0.5f);
        pos[i] = x;
        pos[N + i] = y;
        pos[2 * N + i] = z;
        const float v3 = h * h * h;
        gam[i] = -cosf(x) * sinf(y) * sinf(z) * v3;
        gam[N + i] = -sinf(x) * cosf(y) * sinf(z) * v3;
        gam[2 * N + i] = 2.f * sinf(x) * sinf(y) * cosf(z) * v3;
    }
    vfmm_ctx* ctx = NULL;
    if (check(NULL, vfmm_create(&ctx, &prm, 0), "vfmm_create")) return 1;
    if (check(ctx, vfmm_evaluate_host(ctx, N, pos, gam, vel, dg), "vfmm_evaluate_host")) return 1;
    vfmm_stats st;
    if (check(ctx, vfmm_get_stats(ctx, &st), "vfmm_get_stats")) return 1;
    printf("%d %d %d %.6f\n", n, prm.p, st.depth_used, st.ms_total);
    const int64_t idx[2] = {0, N - 1};
    for (int k = 0; k < 2; ++k) {
        const int64_t i = idx[k];
        printf("%.9e %.9e %.9e %.9e %.9e %.9e\n", vel[i], vel[N + i], vel[2 * N + i], dg[i],
               dg[N + i], dg[2 * N + i]);
    }
    vfmm_destroy(ctx);
    free(buf);
    return 0;
}
