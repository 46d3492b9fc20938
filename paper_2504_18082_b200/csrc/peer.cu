// peer.cu -- NEXT-1 plumbing: share a feature shard with the other processes of the node
// (CUDA IPC; on an NVLink/NVSwitch box the mapped peer memory is read over NVLink by
// cmb_gather_aggregate_sharded).  Host code only.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "common.cuh"

using namespace cmb;

namespace {

// base address of the allocation holding p (the caching allocator sub-allocates, and an IPC
// handle names the whole allocation)
cmb_status allocation_base(const void* p, uintptr_t* base) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CMB_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
  CMB_ARG(fn != nullptr, "cmb_ipc_export: cuMemGetAddressRange unavailable");
  auto range = reinterpret_cast<CUresult(CUDAAPI*)(CUdeviceptr*, size_t*, CUdeviceptr)>(fn);
  CUdeviceptr b = 0;
  size_t sz = 0;
  CMB_ARG(range(&b, &sz, reinterpret_cast<CUdeviceptr>(p)) == CUDA_SUCCESS,
          "cmb_ipc_export: pointer is not device memory");
  *base = static_cast<uintptr_t>(b);
  return CMB_OK;
}

}  // namespace

extern "C" {

cmb_status cmb_ipc_export(const void* dev_ptr, void* handle, uint64_t* offset) {
  CMB_ARG(dev_ptr && handle && offset, "cmb_ipc_export: null argument");
  uintptr_t base = 0;
  const cmb_status st = allocation_base(dev_ptr, &base);
  if (st != CMB_OK) return st;
  cudaIpcMemHandle_t h;
  CMB_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  std::memcpy(handle, &h, sizeof(h));
  *offset = reinterpret_cast<uintptr_t>(dev_ptr) - base;
  return CMB_OK;
}

cmb_status cmb_ipc_open(const void* handle, uint64_t offset, void** dev_ptr, void** base) {
  CMB_ARG(handle && dev_ptr && base, "cmb_ipc_open: null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* b = nullptr;
  CMB_CUDA(cudaIpcOpenMemHandle(&b, h, cudaIpcMemLazyEnablePeerAccess));
  *base = b;
  *dev_ptr = static_cast<char*>(b) + offset;
  return CMB_OK;
}

cmb_status cmb_ipc_close(void* base) {
  CMB_ARG(base, "cmb_ipc_close: null base");
  CMB_CUDA(cudaIpcCloseMemHandle(base));
  return CMB_OK;
}

}  // extern "C"
