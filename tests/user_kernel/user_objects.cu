// A user kernel compiled OUTSIDE libdsr.so against the device header: it
// creates and destroys objects of a heap that libdsr created, through the
// descriptor from dsr_device_view (new / destroy from any GPU code).
// Built by tests/test_gpu_user_kernel.py with nvcc for sm_100a.
#include "dsr_device.cuh"

// type 0 = Item{id: u32, twice: u64}; thread i creates Item(i, 2i) and, when
// i % 3 == 0, destroys the object it created in the previous call (handles[i]).
__global__ void user_items(dsr::DevHeap h, uint32_t n, uint64_t* handles, int destroy_pass) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (destroy_pass) {
    if (i % 3 == 0) {
      dsr::dsr_destroy(h, handles[i]);
      handles[i] = 0;
    }
    return;
  }
  const uint64_t hd = dsr::dsr_new(h, 0);
  if (hd) {
    *dsr::field_ptr<uint32_t>(h, hd, 0) = i;
    *dsr::field_ptr<uint64_t>(h, hd, 1) = 2ull * i;
  }
  handles[i] = hd;
}

extern "C" int user_launch(const void* view, size_t bytes, uint32_t n, uint64_t* handles, int destroy_pass,
                           void* stream) {
  if (bytes != sizeof(dsr::DevHeap)) return 1;
  dsr::DevHeap h;
  memcpy(&h, view, sizeof(h));
  user_items<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(h, n, handles, destroy_pass);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
