// Explicit instantiations of the equal-width kernels for Q = 1..16
// (split across translation units so nvcc builds them in parallel).
#include "bx_launch.cuh"

namespace bx {
template cudaError_t launch_eq<1>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<2>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<3>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<4>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<5>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<6>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<7>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<8>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<9>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<10>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<11>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<12>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<13>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<14>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<15>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<16>(const EqArgs&, const LaunchCfg&, cudaStream_t);
}  // namespace bx
