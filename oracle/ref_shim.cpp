// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern-"C" shim, written for this repo, that is compiled together with
// the reference's OWN sources where they lie under /root/reference/proj/src
// (geometry.cpp, dataset.cpp, kernel_ref.cpp, kernel_opt.cpp) by
// oracle/Makefile into oracle/_ref/libconebeam_ref.so. It lets tests and the
// bench's CPU baseline call the unmodified reference implementation with
// plain pointers. Nothing in the product links or loads it.
//
// Entry points wrap, respectively:
//   reconstruct_reference   proj/src/kernel_ref.cpp:32-38
//   backproject_reference   proj/src/kernel_ref.cpp:5-30
//   reconstruct_optimized   proj/src/kernel_opt.cpp:658-716
//   make_circular_trajectory proj/src/geometry.cpp:79-116
//   bilinear_sample_guarded proj/include/conebeam/kernel_ref.hpp:19-49
// Error mapping follows proj/src/capi.cpp:30-60 (cb_status values).
#include <cstdint>
#include <cstring>
#include <new>
#include <string>
#include <thread>

#include "conebeam/dataset.hpp"
#include "conebeam/kernel_opt.hpp"
#include "conebeam/kernel_ref.hpp"

namespace {

thread_local std::string g_err;

template <typename Fn>
int guarded(Fn&& fn) noexcept {
    try {
        fn();
        return 0;
    } catch (const conebeam::truncated_error& e) {
        g_err = e.what();
        return 4;
    } catch (const conebeam::format_error& e) {
        g_err = e.what();
        return 3;
    } catch (const conebeam::io_error& e) {
        g_err = e.what();
        return 2;
    } catch (const conebeam::geometry_error& e) {
        g_err = e.what();
        return 5;
    } catch (const conebeam::validation_error& e) {
        g_err = e.what();
        return 1;
    } catch (const std::bad_alloc&) {
        g_err = "out of memory";
        return 6;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 7;
    }
}

conebeam::VolumeGeometry make_geometry(int L, double voxel_mm, double origin_mm) {
    conebeam::VolumeGeometry g;
    g.edge_voxels = L;
    g.voxel_mm = voxel_mm;
    g.origin_mm = origin_mm;
    return g;
}

conebeam::ProjectionStack make_stack(int L, double voxel_mm, double origin_mm,
                                     const float* imgs, int W, int H, int N,
                                     const double* mats) {
    conebeam::ProjectionStack s;
    s.geometry = make_geometry(L, voxel_mm, origin_mm);
    s.matrices.resize(N);
    s.images.resize(N);
    const std::size_t pix = static_cast<std::size_t>(W) * H;
    for (int i = 0; i < N; ++i) {
        std::memcpy(s.matrices[i].a.data(), mats + 12 * static_cast<std::size_t>(i),
                    12 * sizeof(double));
        s.images[i].width = W;
        s.images[i].height = H;
        s.images[i].data.assign(imgs + pix * i, imgs + pix * (i + 1));
    }
    return s;
}

conebeam::Volume make_volume(int L, double voxel_mm, double origin_mm, const float* vol) {
    conebeam::Volume v(make_geometry(L, voxel_mm, origin_mm));
    std::memcpy(v.voxels.data(), vol, v.voxels.size() * sizeof(float));
    return v;
}

} // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

unsigned ref_hardware_concurrency(void) { return std::thread::hardware_concurrency(); }

int ref_reconstruct_reference(float* vol, int L, double voxel_mm, double origin_mm,
                              const float* imgs, int W, int H, int N, const double* mats) {
    return guarded([&] {
        auto v = make_volume(L, voxel_mm, origin_mm, vol);
        const auto s = make_stack(L, voxel_mm, origin_mm, imgs, W, H, N, mats);
        conebeam::reconstruct_reference(v, s);
        std::memcpy(vol, v.voxels.data(), v.voxels.size() * sizeof(float));
    });
}

int ref_backproject_reference(float* vol, int L, double voxel_mm, double origin_mm,
                              const float* img, int W, int H, const double* mat) {
    return guarded([&] {
        auto v = make_volume(L, voxel_mm, origin_mm, vol);
        conebeam::ProjectionImage im;
        im.width = W;
        im.height = H;
        im.data.assign(img, img + static_cast<std::size_t>(W) * H);
        conebeam::ProjectionMatrix m;
        std::memcpy(m.a.data(), mat, 12 * sizeof(double));
        conebeam::backproject_reference(v, im, m);
        std::memcpy(vol, v.voxels.data(), v.voxels.size() * sizeof(float));
    });
}

// Optimized CPU path with the reference's options (lanes 1/4/8/16, chunk,
// workers 0=all, clip, pad). Timings come from its own ReconstructStats.
int ref_reconstruct_optimized(float* vol, int L, double voxel_mm, double origin_mm,
                              const float* imgs, int W, int H, int N, const double* mats,
                              int lanes, int chunk, int workers, int use_clip, int use_pad,
                              double* precompute_s, double* kernel_s, uint64_t* updates) {
    return guarded([&] {
        auto v = make_volume(L, voxel_mm, origin_mm, vol);
        const auto s = make_stack(L, voxel_mm, origin_mm, imgs, W, H, N, mats);
        conebeam::OptOptions o;
        o.lanes = lanes;
        o.chunk_size = chunk;
        o.workers = workers;
        o.use_clip = use_clip != 0;
        o.use_pad = use_pad != 0;
        conebeam::ReconstructStats st;
        conebeam::reconstruct_optimized(v, s, o, &st);
        std::memcpy(vol, v.voxels.data(), v.voxels.size() * sizeof(float));
        if (precompute_s)
            *precompute_s = st.precompute_seconds;
        if (kernel_s)
            *kernel_s = st.kernel_seconds;
        if (updates)
            *updates = st.voxel_updates;
    });
}

int ref_make_circular_trajectory(int n, double sid, double sdd, int W, int H, double px,
                                 double range_rad, double* out) {
    return guarded([&] {
        conebeam::TrajectoryConfig c;
        c.num_projections = n;
        c.source_isocenter_mm = sid;
        c.source_detector_mm = sdd;
        c.detector_width = W;
        c.detector_height = H;
        c.pixel_size_mm = px;
        c.angular_range_rad = range_rad;
        const auto ms = conebeam::make_circular_trajectory(c);
        for (int i = 0; i < n; ++i)
            std::memcpy(out + 12 * static_cast<std::size_t>(i), ms[i].a.data(),
                        12 * sizeof(double));
    });
}

float ref_bilinear_sample_guarded(const float* img, int W, int H, float ix, float iy) {
    conebeam::ProjectionImage im;
    im.width = W;
    im.height = H;
    im.data.assign(img, img + static_cast<std::size_t>(W) * H);
    return conebeam::bilinear_sample_guarded(im, ix, iy);
}

} // extern "C"
