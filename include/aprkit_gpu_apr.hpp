// Device implementation of the apr.hpp drop-in (include/aprkit_gpu/aprkit/apr.hpp);
// included once the runtime in aprkit_gpu.hpp is complete.
#pragma once

namespace aprkit {

// Structural invariants and the domain partition (apr.hpp:61-134), on the device.
// The reference's two O(1) shape checks (apr.hpp:62-64) are answered here with
// its messages; every other check runs in aprgpu_validate_access.  Structures
// the device layout cannot hold -- more than APRGPU_MAX_LEVELS levels, a
// level_offset shorter than the level range, or a level wider than kMaxYDim
// (linear_access.hpp:17) -- raise CapabilityError: there is no CPU path.
inline ValidationReport validate(const LinearAccess& a, const std::array<int, 3>& source_dims) {
    if (a.l_min > a.l_max) return ValidationReport::violation("l_min > l_max");
    if ((int)a.z_dim.size() <= a.l_max || (int)a.x_dim.size() <= a.l_max || (int)a.y_dim.size() <= a.l_max)
        return ValidationReport::violation("per-level dim arrays too short");
    if (a.l_min < 0 || a.l_max >= APRGPU_MAX_LEVELS)
        throw CapabilityError("validate: levels outside [0, " + std::to_string(APRGPU_MAX_LEVELS) +
                              ") are not supported by the device structure");
    if (!gpu::well_formed(a)) throw CapabilityError("validate: level_offset shorter than the level range");
    for (int l = a.l_min; l <= a.l_max; ++l)
        if (a.y_dim[l] > kMaxYDim)
            throw CapabilityError("validate: y_dim above kMaxYDim (" + std::to_string(kMaxYDim) + ")");
    const aprgpu_access_desc d = gpu::describe(a);
    const int32_t dims[3] = {source_dims[0], source_dims[1], source_dims[2]};
    int ok = 0;
    char msg[512];
    gpu::check(aprgpu_validate_access(gpu::Runtime::get().ctx(), &d, dims, &ok, msg, sizeof(msg)));
    return ok ? ValidationReport::success() : ValidationReport::violation(msg);
}

inline ValidationReport validate(const APR& apr) { return validate(apr.access, apr.source_dims); }

}  // namespace aprkit
