// Explicit instantiations of the equal-width kernels for Q = 81..96
// (split across translation units so nvcc builds them in parallel).
#include "bx_launch.cuh"

namespace bx {
template cudaError_t launch_eq<81>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<82>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<83>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<84>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<85>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<86>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<87>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<88>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<89>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<90>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<91>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<92>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<93>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<94>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<95>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<96>(const EqArgs&, const LaunchCfg&, cudaStream_t);
}  // namespace bx
