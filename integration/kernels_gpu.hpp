// Factory of the drop-in GPU kernel (kernels_gpu.cpp).  In lbmbench itself
// make_kernel (kernels.cpp:95-109) would route to it for a GPU descriptor;
// here the check program calls it directly.
#pragma once

#include <memory>

#include "lbm/kernels.hpp"

namespace lbm::gpu {

std::unique_ptr<Kernel> make_gpu_kernel(const KernelDescriptor& d, const FlagField& ff,
                                        const PaddingPolicy& pad, int row_pad = 0);

}  // namespace lbm::gpu
