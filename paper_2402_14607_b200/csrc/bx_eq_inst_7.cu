// Explicit instantiations of the equal-width kernels for Q = 113..128
// (split across translation units so nvcc builds them in parallel).
#include "bx_launch.cuh"

namespace bx {
template cudaError_t launch_eq<113>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<114>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<115>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<116>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<117>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<118>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<119>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<120>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<121>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<122>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<123>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<124>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<125>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<126>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<127>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<128>(const EqArgs&, const LaunchCfg&, cudaStream_t);
}  // namespace bx
