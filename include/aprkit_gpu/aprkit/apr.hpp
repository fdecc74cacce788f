// Drop-in for aprkit/apr.hpp (reference: proj/include/aprkit/apr.hpp).
//
// Found ahead of the reference header (see convolve.hpp here); keeps the APR
// types, computational_ratio and resolution_level_at from the reference and
// replaces the structure validator:
//   validate  apr.hpp:61-136  -> aprgpu_validate_access: the same checks, in the
//             same order, with the same messages, in O(particles + rows) on the
//             device instead of an O(pixels) cover map (load_apr / read_apr,
//             io.hpp:165, use it through this header).
// Structures the device cannot hold (more than 20 levels, y beyond 65536)
// raise CapabilityError; the reference's validate (renamed below) is never
// called -- there is no CPU path.
#pragma once

#define validate validate_reference_cpu_
#include_next "aprkit/apr.hpp"
#undef validate

#define APRKIT_GPU_APR_OVERLAY 1
#include "aprkit_gpu.hpp"
#ifdef APRKIT_GPU_RUNTIME_DONE
#include "aprkit_gpu_apr.hpp"
#endif
