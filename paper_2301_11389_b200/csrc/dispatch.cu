// dispatch.cu — kind/dtype/variant -> kernel launcher.
#include "internal.h"

namespace stb200 {

cudaError_t dispatch_2d(stencil_s* h, const void* const* in, void* const* out, cudaStream_t s,
                        int64_t a, int64_t b);
cudaError_t dispatch_3d(stencil_s* h, const void* const* in, void* const* out, cudaStream_t s,
                        int64_t a, int64_t b);

cudaError_t dispatch_kernel(stencil_s* h, const void* const* in, void* const* out, cudaStream_t s,
                            int64_t a, int64_t b) {
    return h->ndims == 2 ? dispatch_2d(h, in, out, s, a, b) : dispatch_3d(h, in, out, s, a, b);
}

}  // namespace stb200
