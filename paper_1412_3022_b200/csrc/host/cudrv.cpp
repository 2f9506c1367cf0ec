#include "cudrv.hpp"

#include <dlfcn.h>

namespace pmrc {
const Drv &drv() {
  static Drv d = [] {
    Drv x;
    void *h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return x;
#define PM_SYM(field, name) x.field = reinterpret_cast<decltype(x.field)>(dlsym(h, name))
    PM_SYM(GetErrorString, "cuGetErrorString");
    PM_SYM(ModuleLoadData, "cuModuleLoadData");
    PM_SYM(ModuleUnload, "cuModuleUnload");
    PM_SYM(ModuleGetFunction, "cuModuleGetFunction");
    PM_SYM(FuncGetAttribute, "cuFuncGetAttribute");
    PM_SYM(FuncSetAttribute, "cuFuncSetAttribute");
    PM_SYM(OccupancyMaxActiveBlocksPerMultiprocessor, "cuOccupancyMaxActiveBlocksPerMultiprocessor");
    PM_SYM(CtxGetDevice, "cuCtxGetDevice");
    PM_SYM(DeviceGetAttribute, "cuDeviceGetAttribute");
    PM_SYM(LaunchKernel, "cuLaunchKernel");
    PM_SYM(LaunchKernelEx, "cuLaunchKernelEx");
#undef PM_SYM
    x.ok = x.GetErrorString && x.ModuleLoadData && x.ModuleUnload && x.ModuleGetFunction && x.FuncGetAttribute && x.FuncSetAttribute &&
           x.OccupancyMaxActiveBlocksPerMultiprocessor && x.CtxGetDevice && x.DeviceGetAttribute && x.LaunchKernel;
    return x;
  }();
  return d;
}
}  // namespace pmrc
