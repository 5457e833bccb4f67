// Explicit instantiations of the equal-width kernels for Q = 33..48
// (split across translation units so nvcc builds them in parallel).
#include "bx_launch.cuh"

namespace bx {
template cudaError_t launch_eq<33>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<34>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<35>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<36>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<37>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<38>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<39>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<40>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<41>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<42>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<43>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<44>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<45>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<46>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<47>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<48>(const EqArgs&, const LaunchCfg&, cudaStream_t);
}  // namespace bx
