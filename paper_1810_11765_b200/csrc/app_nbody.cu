// app_nbody.cu -- placeholder (filled in later)
#include "dsr_host.h"
namespace dsr {
bool nb_method_info(uint32_t, MethodInfo*) { return false; }
bool nb_method_launch(uint32_t, const LaunchCtx&, uint32_t, int, const void*) { return false; }
bool nb_kernel_launch(uint32_t, const LaunchCtx&, uint64_t, const void*, size_t, int*) { return false; }
bool nb_ctor_launch(uint32_t, const LaunchCtx&, uint32_t, uint64_t, const void*, size_t, int*) { return false; }
}  // namespace dsr
