// Explicit instantiations of the equal-width kernels for Q = 49..64
// (split across translation units so nvcc builds them in parallel).
#include "bx_launch.cuh"

namespace bx {
template cudaError_t launch_eq<49>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<50>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<51>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<52>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<53>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<54>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<55>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<56>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<57>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<58>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<59>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<60>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<61>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<62>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<63>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<64>(const EqArgs&, const LaunchCfg&, cudaStream_t);
}  // namespace bx
