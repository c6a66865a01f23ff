/*
 * fdk_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference's scalar back-projection oracle, used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
 * CHECKER. It is never linked into, loaded by, or called from the product
 * library (paper_1401_3615_b200/); the product fails loudly without its CUDA
 * library instead of falling back to this file.
 *
 * Parity pin: tests/test_oracle.py checks this restatement against
 *   - the golden FNV-1a hash 0xab67551f9fba3780 of the reference test
 *     proj/tests/test_kernel_ref.cpp:236-269,
 *   - the hand-evaluated sampler examples proj/tests/test_kernel_ref.cpp:42-49,
 *   - and, when oracle/_ref was built from /root/reference, bitwise equality
 *     with the reference's own reconstruct_reference on seeded inputs.
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off; NO -ffast-math, the
 * reference's CMake sets -ffp-contract=off at proj/CMakeLists.txt:13-15 and
 * the golden hash depends on it).
 *
 * Every float operation below is written in the reference's evaluation order;
 * C evaluates a*b + c*d + e*f + g left to right, so the sums are
 * ((a*b + c*d) + e*f) + g exactly as in proj/include/conebeam/kernel_ref.hpp:61-63.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_OK 0
#define ORACLE_ERR_INVALID 1
#define ORACLE_ERR_GEOMETRY 5

/* proj/include/conebeam/kernel_ref.hpp:19-49 (bilinear_sample_guarded):
 * |ix|,|iy| < 1e9 guard, C truncation toward zero, per-tap bounds guards
 * (width/height matched per axis), two-stage lerp, all in float. */
float oracle_bilinear_sample_guarded(const float *img, int width, int height,
                                     float ix, float iy) {
    if (!(fabsf(ix) < 1.0e9f) || !(fabsf(iy) < 1.0e9f))
        return 0.0f;
    const int iix = (int)ix;
    const int iiy = (int)iy;
    const float scalex = ix - (float)iix;
    const float scaley = iy - (float)iiy;
    float valbl = 0.0f, valbr = 0.0f, valtl = 0.0f, valtr = 0.0f;
    if (iiy >= 0 && iiy < height && iix >= 0 && iix < width)
        valbl = img[iiy * width + iix];
    if (iiy >= 0 && iiy < height && iix + 1 >= 0 && iix + 1 < width)
        valbr = img[iiy * width + iix + 1];
    if (iiy + 1 >= 0 && iiy + 1 < height && iix >= 0 && iix < width)
        valtl = img[(iiy + 1) * width + iix];
    if (iiy + 1 >= 0 && iiy + 1 < height && iix + 1 >= 0 && iix + 1 < width)
        valtr = img[(iiy + 1) * width + iix + 1];
    const float valb = (1 - scalex) * valbl + scalex * valbr;
    const float valt = (1 - scalex) * valtl + scalex * valtr;
    return (1 - scaley) * valb + scaley * valt;
}

/* proj/include/conebeam/kernel_ref.hpp:59-70 (detail::reference_sample) for
 * an unpadded image (pad offsets are 0 and leave the arithmetic unchanged).
 * Returns 0 and sets *zero_w when w == 0 (the reference throws
 * geometry_error there). */
static inline float sample_one(const float *img, int width, int height,
                               const float a[12], float wx, float wy, float wz,
                               int *zero_w) {
    const float u = wx * a[0] + wy * a[3] + wz * a[6] + a[9];
    const float v = wx * a[1] + wy * a[4] + wz * a[7] + a[10];
    const float w = wx * a[2] + wy * a[5] + wz * a[8] + a[11];
    if (w == 0.0f) {
        *zero_w = 1;
        return 0.0f;
    }
    const float ix = u / w;
    const float iy = v / w;
    const float val = oracle_bilinear_sample_guarded(img, width, height, ix, iy);
    return val / (w * w);
}

/* proj/src/kernel_ref.cpp:5-30 (backproject_reference) restricted to z-planes
 * [z0, z1): matrix and geometry are cast double->float exactly as at :11-15,
 * world coordinates are O + idx*MM in float (:21,23,25), voxels are updated
 * z -> y -> x with "+=" in place (:20-29). */
static int backproject_planes(float *vol, int L, float O, float MM,
                              const float *img, int width, int height,
                              const float a[12], int z0, int z1) {
    int zero_w = 0;
    for (int z = z0; z < z1; ++z) {
        const float wz = O + z * MM;
        float *plane = vol + (size_t)z * L * L;
        for (int y = 0; y < L; ++y) {
            const float wy = O + y * MM;
            float *line = plane + (size_t)y * L;
            for (int x = 0; x < L; ++x) {
                const float wx = O + x * MM;
                line[x] += sample_one(img, width, height, a, wx, wy, wz, &zero_w);
                if (zero_w)
                    return ORACLE_ERR_GEOMETRY;
            }
        }
    }
    return ORACLE_OK;
}

static void cast_matrix(const double *m, float a[12]) {
    for (int i = 0; i < 12; ++i)
        a[i] = (float)m[i];
}

/* One projection into the whole volume (backproject_reference). */
int oracle_backproject(float *vol, int L, double voxel_mm, double origin_mm,
                       const float *img, int width, int height, const double *mat) {
    if (!vol || !img || !mat || L < 1 || width < 1 || height < 1)
        return ORACLE_ERR_INVALID;
    float a[12];
    cast_matrix(mat, a);
    return backproject_planes(vol, L, (float)origin_mm, (float)voxel_mm, img, width,
                              height, a, 0, L);
}

struct recon_job {
    float *vol;
    int L;
    float O, MM;
    const float *imgs;
    int width, height, count;
    const double *mats;
    int z0, z1;
    int status;
};

/* All projections in order over the job's z-planes. Voxels of different
 * planes are independent and each voxel still sees its projections in
 * ascending order, so the result is bitwise that of reconstruct_reference
 * (proj/src/kernel_ref.cpp:32-38) regardless of how planes are split. */
static void *recon_worker(void *arg) {
    struct recon_job *j = (struct recon_job *)arg;
    const size_t pix = (size_t)j->width * j->height;
    j->status = ORACLE_OK;
    for (int p = 0; p < j->count; ++p) {
        float a[12];
        cast_matrix(j->mats + 12 * (size_t)p, a);
        int s = backproject_planes(j->vol, j->L, j->O, j->MM, j->imgs + pix * p,
                                   j->width, j->height, a, j->z0, j->z1);
        if (s != ORACLE_OK) {
            j->status = s;
            break;
        }
    }
    return NULL;
}

/* reconstruct_reference over a stack: imgs = count x height x width floats,
 * mats = count x 12 doubles (column-major 3x4, proj/include/conebeam/geometry.hpp:47-65).
 * threads <= 0 selects 1. */
int oracle_reconstruct(float *vol, int L, double voxel_mm, double origin_mm,
                       const float *imgs, int width, int height, int count,
                       const double *mats, int threads) {
    if (!vol || !imgs || !mats || L < 1 || width < 1 || height < 1 || count < 1)
        return ORACLE_ERR_INVALID;
    if (threads < 1)
        threads = 1;
    if (threads > L)
        threads = L;
    struct recon_job *jobs = (struct recon_job *)calloc((size_t)threads, sizeof *jobs);
    pthread_t *tids = (pthread_t *)calloc((size_t)threads, sizeof *tids);
    if (!jobs || !tids) {
        free(jobs);
        free(tids);
        return ORACLE_ERR_INVALID;
    }
    for (int t = 0; t < threads; ++t) {
        struct recon_job *j = &jobs[t];
        j->vol = vol;
        j->L = L;
        j->O = (float)origin_mm;
        j->MM = (float)voxel_mm;
        j->imgs = imgs;
        j->width = width;
        j->height = height;
        j->count = count;
        j->mats = mats;
        j->z0 = (int)((long long)L * t / threads);
        j->z1 = (int)((long long)L * (t + 1) / threads);
    }
    int status = ORACLE_OK;
    if (threads == 1) {
        recon_worker(&jobs[0]);
    } else {
        for (int t = 0; t < threads; ++t)
            pthread_create(&tids[t], NULL, recon_worker, &jobs[t]);
        for (int t = 0; t < threads; ++t)
            pthread_join(tids[t], NULL);
    }
    for (int t = 0; t < threads; ++t)
        if (jobs[t].status != ORACLE_OK)
            status = jobs[t].status;
    free(jobs);
    free(tids);
    return status;
}

struct slab_job {
    float *vol_slab;
    int L, z_begin, nz;
    float O, MM;
    const float *imgs;
    int width, height, count;
    const double *mats;
    int row0, row1; /* rows of the flattened (z, y) line space */
    int status;
};

/* Lines [row0, row1) of the slab's (z, y) line space, all projections in
 * order per line: each voxel sees its projections in ascending order. */
static void *slab_worker(void *arg) {
    struct slab_job *j = (struct slab_job *)arg;
    const size_t pix = (size_t)j->width * j->height;
    const int L = j->L;
    j->status = ORACLE_OK;
    for (int row = j->row0; row < j->row1; ++row) {
        const int z = j->z_begin + row / L;
        const int y = row % L;
        const float wz = j->O + z * j->MM;
        const float wy = j->O + y * j->MM;
        float *line = j->vol_slab + (size_t)row * L;
        for (int p = 0; p < j->count; ++p) {
            float a[12];
            cast_matrix(j->mats + 12 * (size_t)p, a);
            int zero_w = 0;
            for (int x = 0; x < L; ++x) {
                const float wx = j->O + x * j->MM;
                line[x] += sample_one(j->imgs + pix * p, j->width, j->height, a, wx, wy, wz,
                                      &zero_w);
                if (zero_w) {
                    j->status = ORACLE_ERR_GEOMETRY;
                    return NULL;
                }
            }
        }
    }
    return NULL;
}

/* reconstruct_reference restricted to the z-slab [z_begin, z_end) of an
 * L^3 volume: vol_slab holds (z_end - z_begin) planes of L*L floats. Voxels
 * are independent, so this equals the matching planes of the full run. */
int oracle_reconstruct_slab(float *vol_slab, int L, double voxel_mm, double origin_mm,
                            int z_begin, int z_end, const float *imgs, int width, int height,
                            int count, const double *mats, int threads) {
    if (!vol_slab || !imgs || !mats || L < 1 || z_begin < 0 || z_end > L || z_begin >= z_end ||
        width < 1 || height < 1 || count < 1)
        return ORACLE_ERR_INVALID;
    const int rows = (z_end - z_begin) * L;
    if (threads < 1)
        threads = 1;
    if (threads > rows)
        threads = rows;
    struct slab_job *jobs = (struct slab_job *)calloc((size_t)threads, sizeof *jobs);
    pthread_t *tids = (pthread_t *)calloc((size_t)threads, sizeof *tids);
    if (!jobs || !tids) {
        free(jobs);
        free(tids);
        return ORACLE_ERR_INVALID;
    }
    for (int t = 0; t < threads; ++t) {
        struct slab_job *j = &jobs[t];
        j->vol_slab = vol_slab;
        j->L = L;
        j->z_begin = z_begin;
        j->nz = z_end - z_begin;
        j->O = (float)origin_mm;
        j->MM = (float)voxel_mm;
        j->imgs = imgs;
        j->width = width;
        j->height = height;
        j->count = count;
        j->mats = mats;
        j->row0 = (int)((long long)rows * t / threads);
        j->row1 = (int)((long long)rows * (t + 1) / threads);
        pthread_create(&tids[t], NULL, slab_worker, j);
    }
    int status = ORACLE_OK;
    for (int t = 0; t < threads; ++t) {
        pthread_join(tids[t], NULL);
        if (jobs[t].status != ORACLE_OK)
            status = jobs[t].status;
    }
    free(jobs);
    free(tids);
    return status;
}

/* ---- arbitrary z-planes, cache-tiled (large-volume parity checks) --------
 * reconstruct_reference restricted to a list of z-planes. Work units are
 * tiles of TILE_LINES consecutive y-lines of one plane; a unit applies every
 * projection in order to all its lines before the next projection, so the
 * detector footprint of the tile stays in cache across its lines. Each voxel
 * still receives its projections one by one in ascending order with the
 * arithmetic of sample_one, so the result is bitwise that of the reference
 * for every tiling and thread count. Units are handed out dynamically. */
#define TILE_LINES 8

struct planes_job {
    float *out;            /* nplanes x L x L */
    const int *planes;
    int nplanes, L;
    float O, MM;
    const float *imgs;
    int width, height, count;
    const double *mats;
    int units;
    int *next;             /* shared unit counter */
    int *status;           /* shared status */
};

static void *planes_worker(void *arg) {
    struct planes_job *j = (struct planes_job *)arg;
    const size_t pix = (size_t)j->width * j->height;
    const int L = j->L;
    const int tiles_per_plane = (L + TILE_LINES - 1) / TILE_LINES;
    for (;;) {
        const int u = __atomic_fetch_add(j->next, 1, __ATOMIC_RELAXED);
        if (u >= j->units || __atomic_load_n(j->status, __ATOMIC_RELAXED) != ORACLE_OK)
            break;
        const int pi = u / tiles_per_plane;
        const int y0 = (u % tiles_per_plane) * TILE_LINES;
        const int y1 = y0 + TILE_LINES < L ? y0 + TILE_LINES : L;
        const int z = j->planes[pi];
        const float wz = j->O + z * j->MM;
        for (int p = 0; p < j->count; ++p) {
            float a[12];
            cast_matrix(j->mats + 12 * (size_t)p, a);
            const float *img = j->imgs + pix * p;
            int zero_w = 0;
            for (int y = y0; y < y1; ++y) {
                const float wy = j->O + y * j->MM;
                float *line = j->out + ((size_t)pi * L + y) * L;
                for (int x = 0; x < L; ++x) {
                    const float wx = j->O + x * j->MM;
                    line[x] += sample_one(img, j->width, j->height, a, wx, wy, wz, &zero_w);
                    if (zero_w) {
                        __atomic_store_n(j->status, ORACLE_ERR_GEOMETRY, __ATOMIC_RELAXED);
                        return NULL;
                    }
                }
            }
        }
    }
    return NULL;
}

/* out: nplanes x L x L floats, accumulated (+=) like the volume planes
 * planes[0..nplanes) of reconstruct_reference. */
int oracle_reconstruct_planes(float *out, int L, double voxel_mm, double origin_mm,
                              const int *planes, int nplanes, const float *imgs, int width,
                              int height, int count, const double *mats, int threads) {
    if (!out || !planes || !imgs || !mats || L < 1 || nplanes < 1 || width < 1 || height < 1 ||
        count < 1)
        return ORACLE_ERR_INVALID;
    for (int i = 0; i < nplanes; ++i)
        if (planes[i] < 0 || planes[i] >= L)
            return ORACLE_ERR_INVALID;
    if (threads < 1)
        threads = 1;
    int next = 0, status = ORACLE_OK;
    struct planes_job job = {out, planes, nplanes, L, (float)origin_mm, (float)voxel_mm, imgs,
                             width, height, count, mats,
                             nplanes * ((L + TILE_LINES - 1) / TILE_LINES), &next, &status};
    pthread_t *tids = (pthread_t *)calloc((size_t)threads, sizeof *tids);
    if (!tids)
        return ORACLE_ERR_INVALID;
    for (int t = 0; t < threads; ++t)
        pthread_create(&tids[t], NULL, planes_worker, &job);
    for (int t = 0; t < threads; ++t)
        pthread_join(tids[t], NULL);
    free(tids);
    return status;
}

/* ---- content hash for the oracle-volume cache ------------------------------
 * The reference's bench caches its reference volume under the FNV-1a hash of
 * the stack file (proj/src/bench.cpp:194-214). Stacks here are up to 13.6 GB,
 * so the key is FNV-1a over 64-bit words of fixed 64 MiB chunks (hashed in
 * parallel), folded in chunk order with the total length: a different, but
 * equally deterministic, content key. */
#define HASH_CHUNK (64ull << 20)

struct hash_job {
    const unsigned char *data;
    size_t n, nchunks;
    uint64_t *out;
    int *next;
};

static uint64_t fnv_words(const unsigned char *p, size_t n) {
    uint64_t h = 1469598103934665603ull;
    size_t i = 0;
    for (; i + 8 <= n; i += 8) {
        uint64_t w;
        memcpy(&w, p + i, 8);
        h ^= w;
        h *= 1099511628211ull;
    }
    for (; i < n; ++i) {
        h ^= p[i];
        h *= 1099511628211ull;
    }
    return h;
}

static void *hash_worker(void *arg) {
    struct hash_job *j = (struct hash_job *)arg;
    for (;;) {
        const size_t c = (size_t)__atomic_fetch_add(j->next, 1, __ATOMIC_RELAXED);
        if (c >= j->nchunks)
            break;
        const size_t off = c * HASH_CHUNK;
        const size_t len = j->n - off < HASH_CHUNK ? j->n - off : HASH_CHUNK;
        j->out[c] = fnv_words(j->data + off, len);
    }
    return NULL;
}

uint64_t oracle_content_hash(const void *data, size_t n, int threads) {
    const size_t nchunks = (n + HASH_CHUNK - 1) / HASH_CHUNK;
    uint64_t *part = (uint64_t *)calloc(nchunks ? nchunks : 1, sizeof *part);
    if (!part)
        return 0;
    int next = 0;
    struct hash_job job = {(const unsigned char *)data, n, nchunks, part, &next};
    if (threads < 1)
        threads = 1;
    if ((size_t)threads > nchunks)
        threads = nchunks ? (int)nchunks : 1;
    pthread_t *tids = (pthread_t *)calloc((size_t)threads, sizeof *tids);
    for (int t = 0; tids && t < threads; ++t)
        pthread_create(&tids[t], NULL, hash_worker, &job);
    for (int t = 0; tids && t < threads; ++t)
        pthread_join(tids[t], NULL);
    uint64_t h = fnv_words((const unsigned char *)part, nchunks * sizeof *part);
    h ^= (uint64_t)n;
    h *= 1099511628211ull;
    free(tids);
    free(part);
    return h;
}

/* FNV-1a 64 over raw bytes (proj/tests/helpers.hpp:41-49). */
uint64_t oracle_fnv1a64(const void *data, size_t n) {
    const unsigned char *p = (const unsigned char *)data;
    uint64_t hash = 1469598103934665603ull;
    for (size_t i = 0; i < n; ++i) {
        hash ^= p[i];
        hash *= 1099511628211ull;
    }
    return hash;
}
