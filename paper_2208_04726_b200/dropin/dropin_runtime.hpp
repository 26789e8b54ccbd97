// dropin_runtime.hpp — shared plumbing of the drop-in operator layer.
//
// The drop-in sources (dropin_*.cpp) implement the functions the reference
// DECLARES in proj/include/pvo/{camera,correlation,bundle_adjust}.hpp, with the
// reference's own signatures and Eigen types, on top of the C-ABI
// (include/pvo_capi.h).  A maintainer builds them in place of
// proj/src/{camera,correlation,bundle_adjust}.cpp and links libpvo_b200.so
// (INTEGRATION.md); every other reference source and test compiles unchanged.
//
// This header supplies the per-thread device context (the reference operators
// are free functions without a context argument: SPEC threading model = one
// context per host thread, device from PVO_DEVICE, default 0) and the mapping
// of pvo_status codes back onto the reference's exception types.
#pragma once

#include <array>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pvo_capi.h"
#include "pvo/se3.hpp"

namespace pvo {
struct DegenerateProblem;  // bundle_adjust.hpp:54-56 (thrown from dropin_bundle_adjust.cpp)

namespace dropin {

// Context of the calling thread, created on first use, destroyed at thread exit.
pvo_ctx* context();

// Status -> exception (std::invalid_argument, std::domain_error,
// std::out_of_range; DEGENERATE is rethrown as pvo::DegenerateProblem by the
// BA translation unit through `degenerate`).
[[noreturn]] void raise(int status, void (*degenerate)(const std::string&) = nullptr);

inline void check(int status, void (*degenerate)(const std::string&) = nullptr) {
    if (status != PVO_OK) raise(status, degenerate);
}

// Pose <-> 7 doubles (qx qy qz qw tx ty tz, Eigen coefficient order).
inline std::array<double, 7> flat(const Pose& p) {
    const Quat& q = p.rotation();
    const Vec3& t = p.translation();
    return {q.x(), q.y(), q.z(), q.w(), t.x(), t.y(), t.z()};
}
inline void flat_into(const Pose& p, double* out) {
    const std::array<double, 7> f = flat(p);
    for (int i = 0; i < 7; ++i) out[i] = f[i];
}
// A device result as a Pose.  When the 7 doubles equal `original`'s bit for
// bit the original object is returned (the Pose constructor renormalises,
// which could move an unchanged pose by an ulp; fixed and skipped poses must
// stay bit-identical, bundle_adjust.hpp:44).
inline Pose unflat(const double* v, const Pose* original = nullptr) {
    if (original) {
        const std::array<double, 7> o = flat(*original);
        bool same = true;
        for (int i = 0; i < 7; ++i) same = same && o[i] == v[i];
        if (same) return *original;
    }
    return Pose(Quat(v[3], v[0], v[1], v[2]), Vec3(v[4], v[5], v[6]));
}

}  // namespace dropin
}  // namespace pvo
