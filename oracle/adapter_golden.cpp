// adapter_golden.cpp -- TEST INFRASTRUCTURE: the reference's own golden case
// (proj/tests/test_kernel_ref.cpp:236-269), built with the reference's types
// and generators, run through the C++ drop-in adapter include/conebeam_b200.hpp
// (-> libconebeam_b200.so on the GPU) and through the reference oracle, and
// compared. Built by oracle/Makefile into oracle/_ref/ (needs /root/reference);
// executed by tests/test_gpu_parity.py on the GPU box.
#include <cmath>
#include <cstdint>
#include <cstdio>

#include "conebeam/kernel_ref.hpp"
#include "conebeam_b200.hpp"

static uint64_t fnv1a64(const void* data, std::size_t n) {
    const auto* p = static_cast<const unsigned char*>(data);
    uint64_t h = 1469598103934665603ull;
    for (std::size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 1099511628211ull;
    }
    return h;
}

int main() {
    using namespace conebeam;
    TrajectoryConfig cfg;
    cfg.num_projections = 32;
    cfg.source_isocenter_mm = 200.0;
    cfg.source_detector_mm = 400.0;
    cfg.detector_width = 160;
    cfg.detector_height = 160;
    cfg.pixel_size_mm = 1.0;
    auto matrices = make_circular_trajectory(cfg);
    for (auto& m : matrices)
        for (auto& c : m.a)
            c = std::round(c * 1e6) / 1e6;
    const auto geometry = VolumeGeometry::centered(64, 1.0);
    ProjectionStack stack;
    stack.geometry = geometry;
    stack.matrices = matrices;
    stack.images.assign(matrices.size(), synth_projection_image(160, 160, parse_field_spec("ramp")));

    Volume ref(geometry);
    reconstruct_reference(ref, stack);
    Volume gpu(geometry);
    conebeam_b200::reconstruct(gpu, stack);
    Volume gpu1(geometry);
    for (std::size_t i = 0; i < stack.count(); ++i)
        conebeam_b200::backproject(gpu1, stack.images[i], stack.matrices[i]);

    const uint64_t hr = fnv1a64(ref.voxels.data(), ref.voxels.size() * 4);
    const uint64_t hg = fnv1a64(gpu.voxels.data(), gpu.voxels.size() * 4);
    const uint64_t h1 = fnv1a64(gpu1.voxels.data(), gpu1.voxels.size() * 4);
    std::printf("reference %016llx b200 %016llx b200-per-projection %016llx\n",
                (unsigned long long)hr, (unsigned long long)hg, (unsigned long long)h1);

    // w == 0 maps back to the reference's geometry_error
    Volume small(VolumeGeometry::centered(4, 1.0));
    ProjectionImage img;
    img.width = 8;
    img.height = 8;
    img.data.assign(64, 1.0f);
    ProjectionMatrix m;
    m.a[0] = 1.0;
    m.a[4] = 1.0;
    bool threw = false;
    try {
        conebeam_b200::backproject(small, img, m);
    } catch (const geometry_error&) {
        threw = true;
    }
    std::printf("w0_geometry_error %d\n", threw ? 1 : 0);

    // backproject_reference's validation (kernel_ref.cpp:6-9) through the
    // adapter: a non-finite voxel, a short voxel buffer and a padded image each
    // raise validation_error and leave the volume untouched
    auto raises_validation = [&](auto&& fn) {
        try {
            fn();
        } catch (const validation_error&) {
            return true;
        } catch (...) {
        }
        return false;
    };
    ProjectionStack tiny;
    tiny.geometry = VolumeGeometry::centered(8, 1.0);
    tiny.matrices.assign(1, stack.matrices[0]);
    tiny.images.assign(1, synth_projection_image(16, 16, parse_field_spec("ramp")));
    Volume nanvol(tiny.geometry);
    nanvol.voxels[37] = std::nanf("");
    const bool v_nan = raises_validation([&] { conebeam_b200::reconstruct(nanvol, tiny); }) &&
                       raises_validation([&] {
                           conebeam_b200::backproject(nanvol, tiny.images[0], tiny.matrices[0]);
                       }) &&
                       std::isnan(nanvol.voxels[37]) && nanvol.voxels[36] == 0.0f;
    Volume shortvol(tiny.geometry);
    shortvol.voxels.resize(100);
    const bool v_short = raises_validation([&] { conebeam_b200::reconstruct(shortvol, tiny); });
    ProjectionStack padded = tiny;
    padded.images[0].pad_du = -2;
    Volume pv(tiny.geometry);
    const bool v_pad = raises_validation([&] { conebeam_b200::reconstruct(pv, padded); }) &&
                       raises_validation([&] {
                           conebeam_b200::backproject(pv, padded.images[0], padded.matrices[0]);
                       });
    std::printf("validation nan %d short %d padded %d\n", v_nan, v_short, v_pad);
    return (hr == 0xab67551f9fba3780ull && hg == hr && h1 == hr && threw && v_nan && v_short &&
            v_pad)
               ? 0
               : 1;
}
