/* Plain-C use of libconebeam_b200 (include/conebeam_b200.h): a small seeded
 * scan reconstructed with cbb_reconstruct, with the reference's error model.
 * Build (from the repo root):
 *   gcc -std=c99 -O2 -Iinclude examples/reconstruct_c.c \
 *       -Lpaper_1401_3615_b200 -lconebeam_b200 \
 *       -Wl,-rpath,$PWD/paper_1401_3615_b200 -lm -o reconstruct_c
 * Run with "--abi-only" to print the library version and exit without a GPU. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "conebeam_b200.h"

int main(int argc, char** argv) {
    printf("libconebeam_b200 %s, status 5 = \"%s\"\n", cbb_version(), cbb_status_name(5));
    if (argc > 1 && strcmp(argv[1], "--abi-only") == 0)
        return 0;
    if (cbb_device_count() < 1) {
        fprintf(stderr, "no CUDA device\n");
        return 1;
    }
    /* 64^3 volume at 1 mm, 32 views of a 160x160 detector (SID 200 mm,
     * SDD 400 mm, 1 mm pixels), matrices in the reference's column-major
     * convention (u = a0 x + a3 y + a6 z + a9, ...), w(0) = 1. */
    const int L = 64, W = 160, H = 160, N = 32;
    const double sid = 200.0, sdd = 400.0, pix = 1.0, pi = 3.14159265358979323846;
    cbb_volume_geometry g = {L, 1.0, -0.5 * (L - 1)};
    double* mats = malloc(sizeof(double) * 12 * N);
    float* imgs = malloc(sizeof(float) * (size_t)N * W * H);
    float* vol = calloc((size_t)L * L * L, sizeof(float));
    for (int i = 0; i < N; ++i) {
        const double th = 2.0 * pi * i / N, c = cos(th), s = sin(th), f = sdd / pix;
        const double cu = 0.5 * (W - 1), cv = 0.5 * (H - 1);
        double* a = mats + 12 * i;
        /* rows: u = f*(e_u . X) + cu*w, v = f*(e_v . X) + cv*w, w = (R - d . X)/R */
        const double wx = -c / sid, wy = -s / sid, w0 = 1.0;
        a[0] = f * -s / sid + cu * wx; a[1] = cv * wx; a[2] = wx;
        a[3] = f * c / sid + cu * wy;  a[4] = cv * wy; a[5] = wy;
        a[6] = 0.0;                    a[7] = f / sid; a[8] = 0.0;
        a[9] = cu * w0;                a[10] = cv * w0; a[11] = w0;
        for (int y = 0; y < H; ++y)
            for (int x = 0; x < W; ++x)
                imgs[((size_t)i * H + y) * W + x] = (float)(x + 2 * y);
    }
    cbb_options opt;
    cbb_options_defaults(&opt);
    opt.num_gpus = 1;
    cbb_run_stats st;
    const cbb_status rc = cbb_reconstruct(vol, &g, imgs, W, H, N, mats, &opt, &st);
    if (rc != CBB_OK) {
        fprintf(stderr, "cbb_reconstruct: %s: %s\n", cbb_status_name(rc), cbb_last_error());
        return 1;
    }
    double sum = 0.0;
    for (size_t k = 0; k < (size_t)L * L * L; ++k)
        sum += vol[k];
    printf("%.3g voxel updates in %.3f ms, volume sum %.6g\n", (double)st.voxel_updates,
           st.total_seconds * 1e3, sum);
    /* Volume::validate semantics (proj/src/dataset.cpp:146-151): a non-finite
     * voxel is rejected with CBB_ERR_INVALID and the volume is not touched */
    const float keep = vol[1234];
    vol[4321] = NAN;
    const cbb_status bad = cbb_reconstruct(vol, &g, imgs, W, H, N, mats, &opt, NULL);
    printf("nan voxel: status %d \"%s\" (%s)\n", (int)bad, cbb_last_error(),
           vol[1234] == keep && isnan(vol[4321]) ? "volume unchanged" : "VOLUME CHANGED");
    if (bad != CBB_ERR_INVALID || vol[1234] != keep)
        return 1;
    free(mats);
    free(imgs);
    free(vol);
    return 0;
}
