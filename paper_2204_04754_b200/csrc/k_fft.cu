// k_fft.cu — batched polyphase FFT-correlation E/M path (SRMRA_PATH_FFT).  (stub)
#include "srmra_internal.cuh"
namespace srmra {
bool fft_supported(int, int, int) { return false; }
cudaError_t launch_fft_init(srmra_ctx*) { return cudaErrorNotSupported; }
cudaError_t launch_fft_prep(srmra_ctx*) { return cudaErrorNotSupported; }
cudaError_t launch_fft_em(srmra_ctx*) { return cudaErrorNotSupported; }
cudaError_t launch_fft_fold(srmra_ctx*) { return cudaErrorNotSupported; }
int fft_launches_per_iter(const srmra_ctx*) { return 0; }
}  // namespace srmra
