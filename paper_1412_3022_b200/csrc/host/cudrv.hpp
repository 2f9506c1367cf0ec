// Driver-API entry points resolved at run time (dlopen of libcuda.so.1), so libpmrc.so loads on a
// machine without a GPU driver (the CPU test tier checks its exported symbols) and fails loudly
// with PMRC_ECUDA only when a GPU call is made.
#pragma once
#include <cuda.h>

namespace pmrc {
struct Drv {
  bool ok = false;
  CUresult (*GetErrorString)(CUresult, const char **) = nullptr;
  CUresult (*ModuleLoadData)(CUmodule *, const void *) = nullptr;
  CUresult (*ModuleUnload)(CUmodule) = nullptr;
  CUresult (*ModuleGetFunction)(CUfunction *, CUmodule, const char *) = nullptr;
  CUresult (*FuncGetAttribute)(int *, CUfunction_attribute, CUfunction) = nullptr;
  CUresult (*FuncSetAttribute)(CUfunction, CUfunction_attribute, int) = nullptr;
  CUresult (*OccupancyMaxActiveBlocksPerMultiprocessor)(int *, CUfunction, int, size_t) = nullptr;
  CUresult (*CtxGetDevice)(CUdevice *) = nullptr;
  CUresult (*DeviceGetAttribute)(int *, CUdevice_attribute, CUdevice) = nullptr;
  CUresult (*LaunchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                           CUstream, void **, void **) = nullptr;
  CUresult (*LaunchKernelEx)(const CUlaunchConfig *, CUfunction, void **, void **) = nullptr;  // optional (PDL)
};
const Drv &drv();
}  // namespace pmrc
