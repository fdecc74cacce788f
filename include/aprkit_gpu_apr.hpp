// Device implementation of the apr.hpp drop-in (include/aprkit_gpu/aprkit/apr.hpp);
// included once the runtime in aprkit_gpu.hpp is complete.
#pragma once

namespace aprkit {

// Structural invariants and the domain partition (apr.hpp:61-134), on the device.
inline ValidationReport validate(const LinearAccess& a, const std::array<int, 3>& source_dims) {
    if (!gpu::well_formed(a) || a.l_max >= APRGPU_MAX_LEVELS) return validate_reference_cpu_(a, source_dims);
    for (int l = a.l_min; l <= a.l_max; ++l)
        if (a.y_dim[l] > 65536) return validate_reference_cpu_(a, source_dims);
    const aprgpu_access_desc d = gpu::describe(a);
    const int32_t dims[3] = {source_dims[0], source_dims[1], source_dims[2]};
    int ok = 0;
    char msg[512];
    gpu::check(aprgpu_validate_access(gpu::Runtime::get().ctx(), &d, dims, &ok, msg, sizeof(msg)));
    return ok ? ValidationReport::success() : ValidationReport::violation(msg);
}

inline ValidationReport validate(const APR& apr) { return validate(apr.access, apr.source_dims); }

}  // namespace aprkit
