// Explicit instantiations of the equal-width kernels for Q = 97..112
// (split across translation units so nvcc builds them in parallel).
#include "bx_launch.cuh"

namespace bx {
template cudaError_t launch_eq<97>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<98>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<99>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<100>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<101>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<102>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<103>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<104>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<105>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<106>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<107>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<108>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<109>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<110>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<111>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<112>(const EqArgs&, const LaunchCfg&, cudaStream_t);
}  // namespace bx
