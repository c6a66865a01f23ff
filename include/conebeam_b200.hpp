// conebeam_b200.hpp -- header-only C++ drop-in adapter for the reference
// library's types (proj/include/conebeam/{geometry,dataset,errors}.hpp).
//
// A maintainer of the reference adds this header to the reference build and
// links libconebeam_b200.so; the functions below have the signatures and the
// error behaviour of
//   conebeam::backproject_reference   (proj/include/conebeam/kernel_ref.hpp:77)
//   conebeam::reconstruct_reference   (proj/include/conebeam/kernel_ref.hpp:80)
// and throw the reference's exception types for the matching C statuses
// (inverse of proj/src/capi.cpp:30-60).
#pragma once

#include <string>

#include "conebeam/dataset.hpp"
#include "conebeam/errors.hpp"
#include "conebeam_b200.h"

namespace conebeam_b200 {

inline void throw_on(cbb_status s) {
    if (s == CBB_OK)
        return;
    const std::string msg = cbb_last_error();
    switch (s) {
    case CBB_ERR_INVALID: throw conebeam::validation_error(msg);
    case CBB_ERR_IO: throw conebeam::io_error(msg);
    case CBB_ERR_TRUNCATED: throw conebeam::truncated_error(msg);
    case CBB_ERR_FORMAT: throw conebeam::format_error(msg);
    case CBB_ERR_GEOMETRY: throw conebeam::geometry_error(msg);
    default: throw conebeam::error(std::string(cbb_status_name(s)) + ": " + msg);
    }
}

inline cbb_volume_geometry to_c(const conebeam::VolumeGeometry& g) {
    return cbb_volume_geometry{g.edge_voxels, g.voxel_mm, g.origin_mm};
}

/// backproject_reference on the B200: validates like the reference
/// (kernel_ref.cpp:6-9), accumulates one projection into vol (bitwise equal
/// in the default exact mode).
inline void backproject(conebeam::Volume& vol, const conebeam::ProjectionImage& img,
                        const conebeam::ProjectionMatrix& m) {
    img.validate();
    vol.validate();
    if (img.padded())
        throw conebeam::validation_error("backproject_reference requires an unpadded image");
    const cbb_volume_geometry g = to_c(vol.geometry);
    throw_on(cbb_backproject(vol.voxels.data(), &g, img.data.data(), img.width, img.height,
                             m.a.data()));
}

/// reconstruct_reference on the B200 (all projections, in order). Options
/// (GPU count, batch, exact/fast) default to cbb_options_defaults.
inline void reconstruct(conebeam::Volume& vol, const conebeam::ProjectionStack& stack,
                        const cbb_options* options = nullptr, cbb_run_stats* stats = nullptr) {
    stack.validate();
    if (vol.geometry != stack.geometry)
        throw conebeam::geometry_error("reconstruct_reference: volume and stack geometries differ");
    // backproject_reference's checks for every projection (kernel_ref.cpp:6-9),
    // made once up front: the volume (finite, L^3 voxels -- the library reads
    // and writes L^3 floats through vol.voxels) and unpadded images. Unlike
    // the reference, nothing has been accumulated when one of them throws.
    vol.validate();
    for (const auto& img : stack.images)
        if (img.padded())
            throw conebeam::validation_error("backproject_reference requires an unpadded image");
    const int W = stack.images.front().width, H = stack.images.front().height;
    // the images stay where they are (one buffer each); only the 96-byte
    // matrices are gathered
    std::vector<const float*> imgs(stack.count());
    std::vector<double> mats(12 * stack.count());
    for (std::size_t i = 0; i < stack.count(); ++i) {
        imgs[i] = stack.images[i].data.data();
        std::copy(stack.matrices[i].a.begin(), stack.matrices[i].a.end(), mats.begin() + 12 * i);
    }
    const cbb_volume_geometry g = to_c(vol.geometry);
    throw_on(cbb_reconstruct_images(vol.voxels.data(), &g, imgs.data(), W, H,
                                    static_cast<int32_t>(stack.count()), mats.data(), options,
                                    stats));
}

} // namespace conebeam_b200
