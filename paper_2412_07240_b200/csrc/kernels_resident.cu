// kernels_resident.cu -- one CTA per filter, the whole half spectrum resident in
// shared memory: regrid (gather) -> forward 2-D real DFT -> s*Psi -> inverse ->
// likelihood, normaliser and moments, in ONE launch per filter epoch.
#include "device_common.cuh"

namespace pmf {

bool resident_supported(const Dims& d, int dtype) {
    (void)d; (void)dtype;
    return false;
}

cudaError_t launch_resident(const Dims& d, int dtype, PencilBufs& b, const Twiddles& tw, const ModelParams* mp,
                            const LikParams* lp, double ks, cudaStream_t s, int64_t* launches) {
    (void)d; (void)dtype; (void)b; (void)tw; (void)mp; (void)lp; (void)ks; (void)s; (void)launches;
    return cudaErrorNotSupported;
}

}  // namespace pmf
