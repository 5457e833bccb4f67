// Explicit instantiations of the equal-width kernels for Q = 17..32
// (split across translation units so nvcc builds them in parallel).
#include "bx_launch.cuh"

namespace bx {
template cudaError_t launch_eq<17>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<18>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<19>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<20>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<21>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<22>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<23>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<24>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<25>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<26>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<27>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<28>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<29>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<30>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<31>(const EqArgs&, const LaunchCfg&, cudaStream_t);
template cudaError_t launch_eq<32>(const EqArgs&, const LaunchCfg&, cudaStream_t);
}  // namespace bx
