// Explicit instantiations of the equal-width kernels for Q = 65..80
// (split across translation units so nvcc builds them in parallel).
#include "bx_launch.cuh"

namespace bx {
template cudaError_t launch_eq<65>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<66>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<67>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<68>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<69>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<70>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<71>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<72>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<73>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<74>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<75>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<76>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<77>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<78>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<79>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<80>(const EqArgs&, const LaunchCfg&, cudaStream_t);
}  // namespace bx
