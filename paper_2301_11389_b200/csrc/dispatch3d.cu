// dispatch3d.cu — host launchers of the 3-D kernels (k3d.cuh).
#include "internal.h"

namespace stb200 {

cudaError_t dispatch_3d(stencil_s*, const void* const*, void* const*, cudaStream_t, int64_t,
                        int64_t) {
    return cudaErrorNotSupported;
}

}  // namespace stb200
