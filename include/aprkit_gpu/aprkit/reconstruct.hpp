// Drop-in for aprkit/reconstruct.hpp (reference: proj/include/aprkit/reconstruct.hpp).
//
// Found ahead of the reference header (see convolve.hpp here); keeps PadMode,
// reflect_index, PatchSpec and fill_level_row from the reference and replaces
// the dense reconstructions with the device kernels (csrc/reconstruct.cu):
//   reconstruct_level  reconstruct.hpp:73-84   -> aprgpu_reconstruct_level
//   reconstruct_full   reconstruct.hpp:87-90   -> aprgpu_reconstruct_level (l_max, no tree)
//   reconstruct_patch  reconstruct.hpp:94-129  -> aprgpu_reconstruct_patch
// Outputs are bit-identical (values are copied, never combined).  One edge
// case differs: a cell no source covers (interior-node cells when tree values
// are omitted below l_max, or a malformed APR) is 0 in a device patch, where
// the reference's reused row buffer (:108) leaves the previous row's value.
#pragma once

#define reconstruct_level reconstruct_level_reference_cpu_
#define reconstruct_full reconstruct_full_reference_cpu_
#define reconstruct_patch reconstruct_patch_reference_cpu_
#include_next "aprkit/reconstruct.hpp"
#undef reconstruct_level
#undef reconstruct_full
#undef reconstruct_patch

#define APRKIT_GPU_RECONSTRUCT_OVERLAY 1
#include "aprkit_gpu.hpp"
#ifdef APRKIT_GPU_RUNTIME_DONE
#include "aprkit_gpu_reconstruct.hpp"
#endif
