// dropin_correlation.cpp — the operators of proj/include/pvo/correlation.hpp on
// the GPU.
//
// Replaces proj/src/correlation.cpp.  correlate (correlation.cpp:37-71) runs
// pvo_correlate: the 3x3 production kernel (Gram-form, FP32 dots, with the
// FP64 re-evaluation of cancelling outputs) or, for other patch widths, the
// direct FP64 form; correlate_at / correlate_at_cubic (correlation.cpp:8-35)
// run pvo_correlate_points (FP64, the reference's per-channel sampler
// expressions).  The pyramid / grid arguments are provider-owned host grids;
// the C-ABI keeps them on the device between calls (grid cache keyed by
// address + shape + a content fingerprint), so each frame's pyramid crosses
// PCIe once, not once per patch.
#include <cmath>
#include <stdexcept>

#include "dropin_runtime.hpp"
#include "pvo/correlation.hpp"

namespace pvo {

namespace {
void require_channels(int channels, const FeatureGrid& grid) {
    // the kernels address the grid with the query's channel count as its stride
    if (grid.channels != channels && grid.width * grid.height > 0) {
        throw std::invalid_argument("correlate: feature channels differ from the grid's");
    }
}
}  // namespace

double correlate_at(const float* feature, int channels, const FeatureGrid& grid, double x, double y) {
    require_channels(channels, grid);
    const double xy[2] = {x, y};
    double out = 0.0;
    dropin::check(pvo_correlate_points(dropin::context(), 1, channels, feature, grid.data.data(), grid.width,
                                       grid.height, xy, 0, &out));
    return out;
}

double correlate_at_cubic(const float* feature, int channels, const FeatureGrid& grid, double x, double y) {
    require_channels(channels, grid);
    const double xy[2] = {x, y};
    double out = 0.0;
    dropin::check(pvo_correlate_points(dropin::context(), 1, channels, feature, grid.data.data(), grid.width,
                                       grid.height, xy, 1, &out));
    return out;
}

CorrelationGrid correlate(const PatchFeatures& patch_features, const FeaturePyramid& pyramid,
                          const std::vector<Vec2>& reprojection) {
    const int p = patch_features.width;
    const int pp = p * p;
    if ((int)reprojection.size() != pp) throw std::invalid_argument("correlate: reprojection size mismatch");
    std::vector<double> coords(2 * (size_t)pp);
    for (int k = 0; k < pp; ++k) {
        coords[2 * k] = reprojection[k].x();
        coords[2 * k + 1] = reprojection[k].y();
        if (!std::isfinite(coords[2 * k]) || !std::isfinite(coords[2 * k + 1]))
            throw std::invalid_argument("correlate: non-finite reprojection");
    }
    CorrelationGrid grid;
    grid.patch_width = p;
    const size_t per_level = (size_t)pp * kCorrSize * kCorrSize;
    grid.values[0].resize(per_level);
    grid.values[1].resize(per_level);
    if (pp == 0) return grid;
    const int C = patch_features.channels;
    require_channels(C, pyramid.level0);
    require_channels(C, pyramid.level1);
    if (patch_features.level0.size() < (size_t)pp * C || patch_features.level1.size() < (size_t)pp * C)
        throw std::invalid_argument("correlate: patch features smaller than p * p * channels");
    std::vector<float> out(2 * per_level);
    dropin::check(pvo_correlate(dropin::context(), p, C, patch_features.level0.data(), patch_features.level1.data(),
                                pyramid.level0.data.data(), pyramid.level0.width, pyramid.level0.height,
                                pyramid.level1.data.data(), pyramid.level1.width, pyramid.level1.height, coords.data(),
                                out.data()));
    std::copy(out.begin(), out.begin() + per_level, grid.values[0].begin());
    std::copy(out.begin() + per_level, out.end(), grid.values[1].begin());
    return grid;
}

}  // namespace pvo
