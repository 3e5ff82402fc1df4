// Host interface of the non-GEMM sm_100a kernels.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace pbk {}  // namespace pbk
