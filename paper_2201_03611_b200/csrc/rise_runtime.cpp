// rise_runtime.cpp — native runtime behind include/rise_b200.h.
//
// NVRTC compiles kernel text to sm_100a CUBIN; the CUDA driver API (loaded
// with dlopen so the library also loads on GPU-less build hosts) loads the
// module and launches it with cuLaunchKernelEx (thread-block clusters, large
// dynamic shared memory).  Runs in the primary context so device buffers are
// interchangeable with any other primary-context user.
//
// Reference counterpart: cexec.py (the Python evaluator of emitted C text),
// cexec.py:97 parse_kernel -> rs_compile, cexec.py:509 execute_kernel ->
// rs_launch, cexec.py:533-552 flatten/unflatten -> rs_memcpy_*.

#include "../../include/rise_b200.h"

#include <cuda.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err = "";

int fail(const char* fmt, ...) {
  char buf[4096];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return 1;
}

// ---- driver API table (dlopen'd) ----------------------------------------
struct Driver {
  bool loaded = false;
  void* handle = nullptr;
  CUresult (*Init)(unsigned);
  CUresult (*DeviceGet)(CUdevice*, int);
  CUresult (*DeviceGetCount)(int*);
  CUresult (*DeviceGetAttribute)(int*, CUdevice_attribute, CUdevice);
  CUresult (*DevicePrimaryCtxRetain)(CUcontext*, CUdevice);
  CUresult (*CtxSetCurrent)(CUcontext);
  CUresult (*CtxSynchronize)(void);
  CUresult (*ModuleLoadData)(CUmodule*, const void*);
  CUresult (*ModuleUnload)(CUmodule);
  CUresult (*ModuleGetFunction)(CUfunction*, CUmodule, const char*);
  CUresult (*FuncSetAttribute)(CUfunction, CUfunction_attribute, int);
  CUresult (*FuncGetAttribute)(int*, CUfunction_attribute, CUfunction);
  CUresult (*LaunchKernelEx)(const CUlaunchConfig*, CUfunction, void**, void**);
  CUresult (*MemAlloc)(CUdeviceptr*, size_t);
  CUresult (*MemFree)(CUdeviceptr);
  CUresult (*MemcpyHtoDAsync)(CUdeviceptr, const void*, size_t, CUstream);
  CUresult (*MemcpyDtoHAsync)(void*, CUdeviceptr, size_t, CUstream);
  CUresult (*MemcpyDtoDAsync)(CUdeviceptr, CUdeviceptr, size_t, CUstream);
  CUresult (*MemsetD8Async)(CUdeviceptr, unsigned char, size_t, CUstream);
  CUresult (*StreamCreate)(CUstream*, unsigned);
  CUresult (*StreamDestroy)(CUstream);
  CUresult (*StreamSynchronize)(CUstream);
  CUresult (*EventCreate)(CUevent*, unsigned);
  CUresult (*EventDestroy)(CUevent);
  CUresult (*EventRecord)(CUevent, CUstream);
  CUresult (*EventSynchronize)(CUevent);
  CUresult (*EventElapsedTime)(float*, CUevent, CUevent);
  CUresult (*StreamWaitEvent)(CUstream, CUevent, unsigned);
  CUresult (*TensorMapEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  CUresult (*GetErrorString)(CUresult, const char**);
  CUresult (*StreamBeginCapture)(CUstream, CUstreamCaptureMode);
  CUresult (*StreamEndCapture)(CUstream, CUgraph*);
  CUresult (*GraphInstantiate)(CUgraphExec*, CUgraph, unsigned long long);
  CUresult (*GraphLaunch)(CUgraphExec, CUstream);
  CUresult (*GraphUpload)(CUgraphExec, CUstream);
  CUresult (*GraphExecDestroy)(CUgraphExec);
  CUresult (*GraphDestroy)(CUgraph);
  CUresult (*IpcGetMemHandle)(CUipcMemHandle*, CUdeviceptr);
  CUresult (*IpcOpenMemHandle)(CUdeviceptr*, CUipcMemHandle, unsigned);
  CUresult (*IpcCloseMemHandle)(CUdeviceptr);
  CUresult (*MemGetAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr);
  CUresult (*MemcpyPeerAsync)(CUdeviceptr, CUcontext, CUdeviceptr, CUcontext, size_t, CUstream);
};

Driver g_drv;
std::mutex g_mu;
CUcontext g_ctx = nullptr;
CUdevice g_dev = 0;
bool g_inited = false;

template <typename F>
bool sym(F& fn, const char* name) {
  fn = reinterpret_cast<F>(dlsym(g_drv.handle, name));
  return fn != nullptr;
}

int load_driver() {
  if (g_drv.loaded) return 0;
  g_drv.handle = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
  if (!g_drv.handle) g_drv.handle = dlopen("libcuda.so", RTLD_NOW | RTLD_GLOBAL);
  if (!g_drv.handle) return fail("rs_init: cannot load the CUDA driver (libcuda.so.1): %s", dlerror());
  bool ok = true;
  ok &= sym(g_drv.Init, "cuInit");
  ok &= sym(g_drv.DeviceGet, "cuDeviceGet");
  ok &= sym(g_drv.DeviceGetCount, "cuDeviceGetCount");
  ok &= sym(g_drv.DeviceGetAttribute, "cuDeviceGetAttribute");
  ok &= sym(g_drv.DevicePrimaryCtxRetain, "cuDevicePrimaryCtxRetain");
  ok &= sym(g_drv.CtxSetCurrent, "cuCtxSetCurrent");
  ok &= sym(g_drv.CtxSynchronize, "cuCtxSynchronize");
  ok &= sym(g_drv.ModuleLoadData, "cuModuleLoadData");
  ok &= sym(g_drv.ModuleUnload, "cuModuleUnload");
  ok &= sym(g_drv.ModuleGetFunction, "cuModuleGetFunction");
  ok &= sym(g_drv.FuncSetAttribute, "cuFuncSetAttribute");
  ok &= sym(g_drv.FuncGetAttribute, "cuFuncGetAttribute");
  ok &= sym(g_drv.LaunchKernelEx, "cuLaunchKernelEx");
  ok &= sym(g_drv.MemAlloc, "cuMemAlloc_v2");
  ok &= sym(g_drv.MemFree, "cuMemFree_v2");
  ok &= sym(g_drv.MemcpyHtoDAsync, "cuMemcpyHtoDAsync_v2");
  ok &= sym(g_drv.MemcpyDtoHAsync, "cuMemcpyDtoHAsync_v2");
  ok &= sym(g_drv.MemcpyDtoDAsync, "cuMemcpyDtoDAsync_v2");
  ok &= sym(g_drv.MemsetD8Async, "cuMemsetD8Async");
  ok &= sym(g_drv.StreamCreate, "cuStreamCreate");
  ok &= sym(g_drv.StreamDestroy, "cuStreamDestroy_v2");
  ok &= sym(g_drv.StreamSynchronize, "cuStreamSynchronize");
  ok &= sym(g_drv.EventCreate, "cuEventCreate");
  ok &= sym(g_drv.EventDestroy, "cuEventDestroy_v2");
  ok &= sym(g_drv.EventRecord, "cuEventRecord");
  ok &= sym(g_drv.EventSynchronize, "cuEventSynchronize");
  ok &= sym(g_drv.EventElapsedTime, "cuEventElapsedTime");
  ok &= sym(g_drv.StreamWaitEvent, "cuStreamWaitEvent");
  ok &= sym(g_drv.TensorMapEncodeTiled, "cuTensorMapEncodeTiled");
  ok &= sym(g_drv.GetErrorString, "cuGetErrorString");
  ok &= sym(g_drv.StreamBeginCapture, "cuStreamBeginCapture_v2");
  ok &= sym(g_drv.StreamEndCapture, "cuStreamEndCapture");
  ok &= sym(g_drv.GraphInstantiate, "cuGraphInstantiateWithFlags");
  ok &= sym(g_drv.GraphLaunch, "cuGraphLaunch");
  ok &= sym(g_drv.GraphUpload, "cuGraphUpload");
  ok &= sym(g_drv.GraphExecDestroy, "cuGraphExecDestroy");
  ok &= sym(g_drv.GraphDestroy, "cuGraphDestroy");
  ok &= sym(g_drv.IpcGetMemHandle, "cuIpcGetMemHandle");
  ok &= sym(g_drv.IpcOpenMemHandle, "cuIpcOpenMemHandle_v2");
  ok &= sym(g_drv.IpcCloseMemHandle, "cuIpcCloseMemHandle");
  ok &= sym(g_drv.MemGetAddressRange, "cuMemGetAddressRange_v2");
  ok &= sym(g_drv.MemcpyPeerAsync, "cuMemcpyPeerAsync");
  if (!ok) return fail("rs_init: the CUDA driver lacks a required entry point");
  g_drv.loaded = true;
  return 0;
}

int cu_check(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return 0;
  const char* s = "unknown";
  if (g_drv.GetErrorString) g_drv.GetErrorString(r, &s);
  return fail("%s failed: %s (CUresult %d)", what, s, (int)r);
}

#define CU(call, what)                         \
  do {                                         \
    if (int _e = cu_check((call), (what))) return _e; \
  } while (0)

// ---- NCCL (dlopen'd; the soname resolves to the copy already loaded by
// the process, e.g. torch's, or the system one) ----------------------------
struct NcclId {
  char internal[128];
};
struct Nccl {
  bool loaded = false;
  void* handle = nullptr;
  int (*GetUniqueId)(NcclId*);
  int (*CommInitRank)(void**, int, NcclId, int);
  int (*CommDestroy)(void*);
  int (*AllGather)(const void*, void*, size_t, int, void*, CUstream);
  const char* (*GetErrorString)(int);
};
Nccl g_nccl;
constexpr int kNcclUint8 = 1;

int load_nccl() {
  if (g_nccl.loaded) return 0;
  const char* env = getenv("RISE_NCCL_LIB");
  const char* names[] = {env ? env : "libnccl.so.2", "libnccl.so.2", "libnccl.so"};
  for (const char* n : names) {
    g_nccl.handle = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
    if (g_nccl.handle) break;
  }
  if (!g_nccl.handle) return fail("rs_comm: cannot load NCCL (libnccl.so.2): %s", dlerror());
  auto get = [](const char* name) { return dlsym(g_nccl.handle, name); };
  g_nccl.GetUniqueId = reinterpret_cast<int (*)(NcclId*)>(get("ncclGetUniqueId"));
  g_nccl.CommInitRank = reinterpret_cast<int (*)(void**, int, NcclId, int)>(get("ncclCommInitRank"));
  g_nccl.CommDestroy = reinterpret_cast<int (*)(void*)>(get("ncclCommDestroy"));
  g_nccl.AllGather = reinterpret_cast<int (*)(const void*, void*, size_t, int, void*, CUstream)>(get("ncclAllGather"));
  g_nccl.GetErrorString = reinterpret_cast<const char* (*)(int)>(get("ncclGetErrorString"));
  if (!g_nccl.GetUniqueId || !g_nccl.CommInitRank || !g_nccl.CommDestroy || !g_nccl.AllGather ||
      !g_nccl.GetErrorString)
    return fail("rs_comm: the NCCL library lacks a required entry point");
  g_nccl.loaded = true;
  return 0;
}

int nccl_check(int r, const char* what) {
  if (r == 0) return 0;
  return fail("%s failed: %s (ncclResult %d)", what, g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?", r);
}

int ensure_ctx() {
  if (!g_inited) return fail("rs_init has not been called");
  return cu_check(g_drv.CtxSetCurrent(g_ctx), "cuCtxSetCurrent");
}

}  // namespace

struct rs_module_s {
  CUmodule mod = nullptr;
  std::vector<std::string> lowered;
};

struct rs_function_s {
  CUfunction fn = nullptr;
  int smem_optin = 0;  // dynamic smem bytes already enabled via attribute
};

extern "C" {

const char* rs_last_error(void) { return g_err.c_str(); }

int rs_abi_version(void) { return 1; }

int rs_init(int device) {
  std::lock_guard<std::mutex> lock(g_mu);
  if (int e = load_driver()) return e;
  if (g_inited) {
    if (device != (int)g_dev) return fail("rs_init: already initialised on device %d", (int)g_dev);
    return cu_check(g_drv.CtxSetCurrent(g_ctx), "cuCtxSetCurrent");
  }
  CU(g_drv.Init(0), "cuInit");
  int count = 0;
  CU(g_drv.DeviceGetCount(&count), "cuDeviceGetCount");
  if (device < 0 || device >= count) return fail("rs_init: device %d out of range (%d devices)", device, count);
  CU(g_drv.DeviceGet(&g_dev, device), "cuDeviceGet");
  CU(g_drv.DevicePrimaryCtxRetain(&g_ctx, g_dev), "cuDevicePrimaryCtxRetain");
  CU(g_drv.CtxSetCurrent(g_ctx), "cuCtxSetCurrent");
  g_inited = true;
  return 0;
}

int rs_device_count(int* count) {
  if (int e = load_driver()) return e;
  CU(g_drv.Init(0), "cuInit");
  CU(g_drv.DeviceGetCount(count), "cuDeviceGetCount");
  return 0;
}

int rs_device_attribute(int attribute, int* value) {
  if (int e = ensure_ctx()) return e;
  CU(g_drv.DeviceGetAttribute(value, (CUdevice_attribute)attribute, g_dev), "cuDeviceGetAttribute");
  return 0;
}

int rs_nvrtc_version(int* major, int* minor) {
  if (nvrtcVersion(major, minor) != NVRTC_SUCCESS) return fail("nvrtcVersion failed");
  return 0;
}

void rs_free_host(void* p) { free(p); }

int rs_compile_cubin(const char* source, const char* program_name, const char* const* opts, int nopts,
                     const char* const* name_exprs, int nexprs, void** out_image, size_t* out_size,
                     char** out_lowered_names, char** out_log) {
  *out_image = nullptr;
  *out_size = 0;
  if (out_lowered_names) *out_lowered_names = nullptr;
  if (out_log) *out_log = nullptr;
  nvrtcProgram prog;
  nvrtcResult r = nvrtcCreateProgram(&prog, source, program_name ? program_name : "rise.cu", 0, nullptr, nullptr);
  if (r != NVRTC_SUCCESS) return fail("nvrtcCreateProgram: %s", nvrtcGetErrorString(r));
  for (int i = 0; i < nexprs; ++i) {
    r = nvrtcAddNameExpression(prog, name_exprs[i]);
    if (r != NVRTC_SUCCESS) {
      nvrtcDestroyProgram(&prog);
      return fail("nvrtcAddNameExpression(%s): %s", name_exprs[i], nvrtcGetErrorString(r));
    }
  }
  std::vector<const char*> all;
  bool has_arch = false;
  for (int i = 0; i < nopts; ++i) {
    all.push_back(opts[i]);
    if (strstr(opts[i], "arch") != nullptr) has_arch = true;
  }
  if (!has_arch) all.push_back("--gpu-architecture=sm_100a");
  nvrtcResult cr = nvrtcCompileProgram(prog, (int)all.size(), all.data());
  size_t log_size = 0;
  nvrtcGetProgramLogSize(prog, &log_size);
  std::string log(log_size, '\0');
  if (log_size) nvrtcGetProgramLog(prog, &log[0]);
  if (out_log) {
    *out_log = (char*)malloc(log.size() + 1);
    memcpy(*out_log, log.c_str(), log.size() + 1);
  }
  if (cr != NVRTC_SUCCESS) {
    nvrtcDestroyProgram(&prog);
    return fail("NVRTC compilation of %s failed (%s):\n%s", program_name ? program_name : "rise.cu",
                nvrtcGetErrorString(cr), log.c_str());
  }
  std::string names;
  for (int i = 0; i < nexprs; ++i) {
    const char* lowered = nullptr;
    r = nvrtcGetLoweredName(prog, name_exprs[i], &lowered);
    if (r != NVRTC_SUCCESS || !lowered) {
      nvrtcDestroyProgram(&prog);
      return fail("nvrtcGetLoweredName(%s): %s", name_exprs[i], nvrtcGetErrorString(r));
    }
    names += lowered;
    names += '\n';
  }
  size_t size = 0;
  r = nvrtcGetCUBINSize(prog, &size);
  if (r != NVRTC_SUCCESS || size == 0) {
    nvrtcDestroyProgram(&prog);
    return fail("nvrtcGetCUBINSize: %s (compile with a real sm_ architecture)", nvrtcGetErrorString(r));
  }
  void* image = malloc(size);
  r = nvrtcGetCUBIN(prog, (char*)image);
  nvrtcDestroyProgram(&prog);
  if (r != NVRTC_SUCCESS) {
    free(image);
    return fail("nvrtcGetCUBIN: %s", nvrtcGetErrorString(r));
  }
  *out_image = image;
  *out_size = size;
  if (out_lowered_names) {
    *out_lowered_names = (char*)malloc(names.size() + 1);
    memcpy(*out_lowered_names, names.c_str(), names.size() + 1);
  }
  return 0;
}

int rs_module_load(const void* image, size_t size, rs_module* out_module) {
  (void)size;
  if (int e = ensure_ctx()) return e;
  CUmodule mod;
  CU(g_drv.ModuleLoadData(&mod, image), "cuModuleLoadData");
  auto* m = new rs_module_s();
  m->mod = mod;
  *out_module = m;
  return 0;
}

int rs_compile(const char* source, const char* program_name, const char* const* opts, int nopts,
               const char* const* name_exprs, int nexprs, rs_module* out_module) {
  void* image = nullptr;
  size_t size = 0;
  char* names = nullptr;
  if (int e = rs_compile_cubin(source, program_name, opts, nopts, name_exprs, nexprs, &image, &size, &names,
                               nullptr))
    return e;
  rs_module m = nullptr;
  int e = rs_module_load(image, size, &m);
  free(image);
  if (e) {
    free(names);
    return e;
  }
  std::string all(names ? names : "");
  free(names);
  size_t pos = 0;
  while (pos < all.size()) {
    size_t nl = all.find('\n', pos);
    if (nl == std::string::npos) nl = all.size();
    m->lowered.push_back(all.substr(pos, nl - pos));
    pos = nl + 1;
  }
  *out_module = m;
  return 0;
}

int rs_module_lowered_name(rs_module m, int index, const char** out_name) {
  if (!m || index < 0 || index >= (int)m->lowered.size()) return fail("rs_module_lowered_name: bad index %d", index);
  *out_name = m->lowered[index].c_str();
  return 0;
}

int rs_module_get_function(rs_module m, const char* lowered_name, rs_function* out_fn) {
  if (int e = ensure_ctx()) return e;
  CUfunction fn;
  CU(g_drv.ModuleGetFunction(&fn, m->mod, lowered_name), "cuModuleGetFunction");
  auto* f = new rs_function_s();
  f->fn = fn;
  *out_fn = f;
  return 0;
}

int rs_module_unload(rs_module m) {
  if (!m) return 0;
  if (g_inited && m->mod) g_drv.ModuleUnload(m->mod);
  delete m;
  return 0;
}

int rs_function_attribute(rs_function f, int attribute, int* value) {
  if (int e = ensure_ctx()) return e;
  CU(g_drv.FuncGetAttribute(value, (CUfunction_attribute)attribute, f->fn), "cuFuncGetAttribute");
  return 0;
}

int rs_launch(rs_function f, const unsigned grid[3], const unsigned block[3], const unsigned cluster[3],
              unsigned smem, void* stream, void** args) {
  return rs_launch_ex(f, grid, block, cluster, smem, stream, args, 0u);
}

int rs_launch_ex(rs_function f, const unsigned grid[3], const unsigned block[3], const unsigned cluster[3],
                 unsigned smem, void* stream, void** args, unsigned flags) {
  if (int e = ensure_ctx()) return e;
  if (smem > 48 * 1024 && (int)smem > f->smem_optin) {
    CU(g_drv.FuncSetAttribute(f->fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)smem),
       "cuFuncSetAttribute(MAX_DYNAMIC_SHARED_SIZE_BYTES)");
    f->smem_optin = (int)smem;
  }
  CUlaunchConfig cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDimX = grid[0];
  cfg.gridDimY = grid[1];
  cfg.gridDimZ = grid[2];
  cfg.blockDimX = block[0];
  cfg.blockDimY = block[1];
  cfg.blockDimZ = block[2];
  cfg.sharedMemBytes = smem;
  cfg.hStream = (CUstream)stream;
  CUlaunchAttribute attr[3];
  unsigned na = 0;
  if (cluster && (cluster[0] * cluster[1] * cluster[2]) > 1) {
    attr[na].id = CU_LAUNCH_ATTRIBUTE_CLUSTER_DIMENSION;
    attr[na].value.clusterDim.x = cluster[0];
    attr[na].value.clusterDim.y = cluster[1];
    attr[na].value.clusterDim.z = cluster[2];
    ++na;
  }
  if (flags & RS_LAUNCH_COOPERATIVE) {  // every block co-resident (grid-wide barriers), or the launch fails
    attr[na].id = CU_LAUNCH_ATTRIBUTE_COOPERATIVE;
    attr[na].value.cooperative = 1;
    ++na;
  }
  if (flags & RS_LAUNCH_PDL) {
    attr[na].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
    attr[na].value.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (na) {
    cfg.attrs = attr;
    cfg.numAttrs = na;
  }
  CU(g_drv.LaunchKernelEx(&cfg, f->fn, args, nullptr), "cuLaunchKernelEx");
  return 0;
}

int rs_malloc(void** dptr, size_t bytes) {
  if (int e = ensure_ctx()) return e;
  CUdeviceptr p = 0;
  CU(g_drv.MemAlloc(&p, bytes ? bytes : 1), "cuMemAlloc");
  *dptr = (void*)p;
  return 0;
}

int rs_free(void* dptr) {
  if (int e = ensure_ctx()) return e;
  CU(g_drv.MemFree((CUdeviceptr)dptr), "cuMemFree");
  return 0;
}

int rs_memcpy_htod(void* dst, const void* src, size_t bytes, void* stream) {
  if (int e = ensure_ctx()) return e;
  CU(g_drv.MemcpyHtoDAsync((CUdeviceptr)dst, src, bytes, (CUstream)stream), "cuMemcpyHtoDAsync");
  return 0;
}

int rs_memcpy_dtoh(void* dst, const void* src, size_t bytes, void* stream) {
  if (int e = ensure_ctx()) return e;
  CU(g_drv.MemcpyDtoHAsync(dst, (CUdeviceptr)src, bytes, (CUstream)stream), "cuMemcpyDtoHAsync");
  return 0;
}

int rs_memcpy_dtod(void* dst, const void* src, size_t bytes, void* stream) {
  if (int e = ensure_ctx()) return e;
  CU(g_drv.MemcpyDtoDAsync((CUdeviceptr)dst, (CUdeviceptr)src, bytes, (CUstream)stream), "cuMemcpyDtoDAsync");
  return 0;
}

// primary contexts of the other devices a peer copy names (retained once,
// kept for the process: a copy may still be in flight when the call returns)
CUcontext g_peer_ctx[64] = {};

int rs_memcpy_peer(void* dst, int dst_device, const void* src, int src_device, size_t bytes, void* stream) {
  if (int e = ensure_ctx()) return e;
  int n = 0;
  CU(g_drv.DeviceGetCount(&n), "cuDeviceGetCount");
  if (dst_device < 0 || src_device < 0 || dst_device >= n || src_device >= n || n > 64)
    return fail("rs_memcpy_peer: device %d -> %d out of range (%d devices)", src_device, dst_device, n);
  CUcontext ctx[2] = {nullptr, nullptr};
  const int devs[2] = {dst_device, src_device};
  {
    std::lock_guard<std::mutex> lock(g_mu);
    for (int i = 0; i < 2; ++i) {
      if (!g_peer_ctx[devs[i]]) {
        CUdevice d;
        CU(g_drv.DeviceGet(&d, devs[i]), "cuDeviceGet");
        CU(g_drv.DevicePrimaryCtxRetain(&g_peer_ctx[devs[i]], d), "cuDevicePrimaryCtxRetain");
      }
      ctx[i] = g_peer_ctx[devs[i]];
    }
  }
  CU(g_drv.MemcpyPeerAsync((CUdeviceptr)dst, ctx[0], (CUdeviceptr)src, ctx[1], bytes, (CUstream)stream),
     "cuMemcpyPeerAsync");
  return 0;
}

int rs_memset_d8(void* dst, unsigned char value, size_t bytes, void* stream) {
  if (int e = ensure_ctx()) return e;
  CU(g_drv.MemsetD8Async((CUdeviceptr)dst, value, bytes, (CUstream)stream), "cuMemsetD8Async");
  return 0;
}

int rs_stream_create(void** stream) {
  if (int e = ensure_ctx()) return e;
  CUstream s;
  CU(g_drv.StreamCreate(&s, CU_STREAM_NON_BLOCKING), "cuStreamCreate");
  *stream = (void*)s;
  return 0;
}

int rs_stream_destroy(void* stream) {
  if (int e = ensure_ctx()) return e;
  CU(g_drv.StreamDestroy((CUstream)stream), "cuStreamDestroy");
  return 0;
}

int rs_stream_synchronize(void* stream) {
  if (int e = ensure_ctx()) return e;
  CU(g_drv.StreamSynchronize((CUstream)stream), "cuStreamSynchronize");
  return 0;
}

int rs_device_synchronize(void) {
  if (int e = ensure_ctx()) return e;
  CU(g_drv.CtxSynchronize(), "cuCtxSynchronize");
  return 0;
}

int rs_event_create(void** event) {
  if (int e = ensure_ctx()) return e;
  CUevent ev;
  CU(g_drv.EventCreate(&ev, CU_EVENT_DEFAULT), "cuEventCreate");
  *event = (void*)ev;
  return 0;
}

int rs_event_destroy(void* event) {
  if (int e = ensure_ctx()) return e;
  CU(g_drv.EventDestroy((CUevent)event), "cuEventDestroy");
  return 0;
}

int rs_event_record(void* event, void* stream) {
  if (int e = ensure_ctx()) return e;
  CU(g_drv.EventRecord((CUevent)event, (CUstream)stream), "cuEventRecord");
  return 0;
}

int rs_stream_wait_event(void* stream, void* event) {
  if (int e = ensure_ctx()) return e;
  CU(g_drv.StreamWaitEvent((CUstream)stream, (CUevent)event, 0), "cuStreamWaitEvent");
  return 0;
}

int rs_event_synchronize(void* event) {
  if (int e = ensure_ctx()) return e;
  CU(g_drv.EventSynchronize((CUevent)event), "cuEventSynchronize");
  return 0;
}

int rs_event_elapsed_ms(float* ms, void* start, void* end) {
  if (int e = ensure_ctx()) return e;
  CU(g_drv.EventElapsedTime(ms, (CUevent)start, (CUevent)end), "cuEventElapsedTime");
  return 0;
}

int rs_graph_capture_begin(void* stream) {
  if (int e = ensure_ctx()) return e;
  if (!stream) return fail("rs_graph_capture_begin: capture needs a non-default stream");
  CU(g_drv.StreamBeginCapture((CUstream)stream, CU_STREAM_CAPTURE_MODE_THREAD_LOCAL), "cuStreamBeginCapture");
  return 0;
}

int rs_graph_capture_end(void* stream, void** graph_exec) {
  if (int e = ensure_ctx()) return e;
  CUgraph g = nullptr;
  CU(g_drv.StreamEndCapture((CUstream)stream, &g), "cuStreamEndCapture");
  CUgraphExec x = nullptr;
  CUresult r = g_drv.GraphInstantiate(&x, g, 0);
  g_drv.GraphDestroy(g);
  CU(r, "cuGraphInstantiate");
  *graph_exec = (void*)x;
  return 0;
}

int rs_graph_launch(void* graph_exec, void* stream) {
  if (int e = ensure_ctx()) return e;
  CU(g_drv.GraphLaunch((CUgraphExec)graph_exec, (CUstream)stream), "cuGraphLaunch");
  return 0;
}

int rs_graph_upload(void* graph_exec, void* stream) {
  if (int e = ensure_ctx()) return e;
  CU(g_drv.GraphUpload((CUgraphExec)graph_exec, (CUstream)stream), "cuGraphUpload");
  return 0;
}

int rs_graph_destroy(void* graph_exec) {
  if (!graph_exec) return 0;
  if (int e = ensure_ctx()) return e;
  CU(g_drv.GraphExecDestroy((CUgraphExec)graph_exec), "cuGraphExecDestroy");
  return 0;
}

int rs_tma_desc_2d_f32(void* desc, const void* base, uint64_t dim0, uint64_t dim1, uint64_t row_stride_bytes,
                       uint32_t box0, uint32_t box1, int swizzle) {
  if (int e = load_driver()) return e;
  cuuint64_t dims[2] = {dim0, dim1};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box0, box1};
  cuuint32_t estr[2] = {1, 1};
  CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_NONE;
  if (swizzle == 1) sw = CU_TENSOR_MAP_SWIZZLE_32B;
  if (swizzle == 2) sw = CU_TENSOR_MAP_SWIZZLE_64B;
  if (swizzle == 3) sw = CU_TENSOR_MAP_SWIZZLE_128B;
  if (swizzle == 4) sw = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;  // MN-major tf32 UMMA operands
  CU(g_drv.TensorMapEncodeTiled((CUtensorMap*)desc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base),
                                dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
     "cuTensorMapEncodeTiled");
  return 0;
}

// ---- multi-GPU ------------------------------------------------------------

struct rs_comm_s {
  void* nccl = nullptr;
  int nranks = 0, rank = 0;
};

namespace {
std::mutex g_ipc_mu;
std::vector<std::pair<CUdeviceptr, CUdeviceptr>> g_ipc_open;  // (returned pointer, mapped base)
}  // namespace

int rs_ipc_handle(void* handle_out, size_t* offset_out, const void* dptr) {
  if (int e = ensure_ctx()) return e;
  CUdeviceptr base = 0;
  size_t size = 0;
  CU(g_drv.MemGetAddressRange(&base, &size, (CUdeviceptr)dptr), "cuMemGetAddressRange");
  CUipcMemHandle h;
  CU(g_drv.IpcGetMemHandle(&h, base), "cuIpcGetMemHandle");
  static_assert(sizeof(CUipcMemHandle) == 64, "CUipcMemHandle is 64 bytes");
  memcpy(handle_out, &h, sizeof(h));
  *offset_out = (size_t)((CUdeviceptr)dptr - base);
  return 0;
}

int rs_ipc_open(void** dptr_out, const void* handle, size_t offset) {
  if (int e = ensure_ctx()) return e;
  CUipcMemHandle h;
  memcpy(&h, handle, sizeof(h));
  CUdeviceptr base = 0;
  CU(g_drv.IpcOpenMemHandle(&base, h, CU_IPC_MEM_LAZY_ENABLE_PEER_ACCESS), "cuIpcOpenMemHandle");
  std::lock_guard<std::mutex> lock(g_ipc_mu);
  g_ipc_open.emplace_back(base + offset, base);
  *dptr_out = (void*)(base + offset);
  return 0;
}

int rs_ipc_close(void* dptr) {
  if (int e = ensure_ctx()) return e;
  CUdeviceptr base = 0;
  {
    std::lock_guard<std::mutex> lock(g_ipc_mu);
    for (size_t i = 0; i < g_ipc_open.size(); ++i) {
      if (g_ipc_open[i].first == (CUdeviceptr)dptr) {
        base = g_ipc_open[i].second;
        g_ipc_open.erase(g_ipc_open.begin() + (long)i);
        break;
      }
    }
  }
  if (!base) return fail("rs_ipc_close: %p was not returned by rs_ipc_open", dptr);
  CU(g_drv.IpcCloseMemHandle(base), "cuIpcCloseMemHandle");
  return 0;
}

int rs_halo_exchange(void* band, size_t row_bytes, size_t rows, const void* above, size_t above_rows,
                     const void* below, void* stream) {
  if (int e = ensure_ctx()) return e;
  if (rows == 0) return fail("rs_halo_exchange: empty band");
  if (above && above_rows == 0) return fail("rs_halo_exchange: the band above owns no rows");
  const CUdeviceptr b = (CUdeviceptr)band;
  const CUstream st = (CUstream)stream;
  // row 0 <- last owned row of the band above (or this band's row 1)
  const CUdeviceptr top_src = above ? (CUdeviceptr)above + above_rows * row_bytes : b + row_bytes;
  CU(g_drv.MemcpyDtoDAsync(b, top_src, row_bytes, st), "cuMemcpyDtoDAsync (halo above)");
  // row rows+1 <- first owned row of the band below (or this band's row `rows`)
  const CUdeviceptr bot_src = below ? (CUdeviceptr)below + row_bytes : b + rows * row_bytes;
  CU(g_drv.MemcpyDtoDAsync(b + (rows + 1) * row_bytes, bot_src, row_bytes, st), "cuMemcpyDtoDAsync (halo below)");
  return 0;
}

int rs_comm_unique_id(void* id_out) {
  if (int e = load_nccl()) return e;
  NcclId id;
  if (int e = nccl_check(g_nccl.GetUniqueId(&id), "ncclGetUniqueId")) return e;
  memcpy(id_out, &id, sizeof(id));
  return 0;
}

int rs_comm_init(rs_comm* out, int nranks, int rank, const void* id) {
  if (int e = ensure_ctx()) return e;
  if (int e = load_nccl()) return e;
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail("rs_comm_init: rank %d of %d", rank, nranks);
  NcclId nid;
  memcpy(&nid, id, sizeof(nid));
  void* c = nullptr;
  if (int e = nccl_check(g_nccl.CommInitRank(&c, nranks, nid, rank), "ncclCommInitRank")) return e;
  rs_comm h = new rs_comm_s;
  h->nccl = c;
  h->nranks = nranks;
  h->rank = rank;
  *out = h;
  return 0;
}

int rs_comm_destroy(rs_comm comm) {
  if (!comm) return 0;
  if (int e = ensure_ctx()) return e;
  int r = g_nccl.CommDestroy(comm->nccl);
  delete comm;
  return nccl_check(r, "ncclCommDestroy");
}

int rs_allgather(rs_comm comm, const void* send, void* recv, size_t bytes_per_rank, void* stream) {
  if (!comm) return fail("rs_allgather: no communicator");
  if (int e = ensure_ctx()) return e;
  return nccl_check(g_nccl.AllGather(send, recv, bytes_per_rank, kNcclUint8, comm->nccl, (CUstream)stream),
                    "ncclAllGather");
}

}  // extern "C"
