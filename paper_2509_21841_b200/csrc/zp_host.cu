// Error state, device gate, tensor-map encoding and CUDA-IPC helpers.
#include "zp_host.h"
#include "../../include/zeppelin_b200.h"

#include <cstdio>
#include <cstring>
#include <mutex>

namespace {
thread_local char g_err[512] = "ok";
constexpr int kMaxDevices = 64;
int g_dev_checked[kMaxDevices] = {};  // per device ordinal: 0 unknown / failed, 1 good
std::mutex g_mu;

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PFN_encodeTiled g_encode = nullptr;
}  // namespace

int zp_fail(int code, const char* msg) {
  std::snprintf(g_err, sizeof(g_err), "%s", msg);
  return code;
}

int zp_fail_cuda(cudaError_t e, const char* where) {
  std::snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
  return ZP_ECUDA;
}

int zp_check_device() {
  std::lock_guard<std::mutex> lk(g_mu);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) {
    cudaGetLastError();
    return zp_fail(ZP_ENODEV, "no CUDA device visible");
  }
  if (g_dev_checked[dev] == 1) return ZP_OK;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) {
    cudaGetLastError();
    return zp_fail(ZP_ENODEV, "no CUDA device visible");
  }
  if (prop.major != 10 || prop.minor != 0) {
    std::snprintf(g_err, sizeof(g_err), "device sm_%d%d is not sm_100 (B200); no fallback exists",
                  prop.major, prop.minor);
    return ZP_ENODEV;
  }
  if (!g_encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      cudaGetLastError();
      return zp_fail(ZP_ENODEV, "cuTensorMapEncodeTiled entry point unavailable");
    }
    g_encode = reinterpret_cast<PFN_encodeTiled>(fn);
  }
  g_dev_checked[dev] = 1;
  return ZP_OK;
}

int zp_make_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows,
                         uint64_t row_pitch_bytes, uint32_t box_cols, uint32_t box_rows) {
  if ((reinterpret_cast<uintptr_t>(base) & 15u) || (row_pitch_bytes & 15u))
    return zp_fail(ZP_EINVAL, "tensor map: base and row pitch must be 16-byte aligned");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_pitch_bytes};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    std::snprintf(g_err, sizeof(g_err), "cuTensorMapEncodeTiled failed (CUresult %d)", int(r));
    return ZP_ETMA;
  }
  return ZP_OK;
}

int zp_make_tmap_2d_f32(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows,
                        uint64_t row_pitch_bytes, uint32_t box_cols, uint32_t box_rows) {
  if ((reinterpret_cast<uintptr_t>(base) & 15u) || (row_pitch_bytes & 15u))
    return zp_fail(ZP_EINVAL, "tensor map: base and row pitch must be 16-byte aligned");
  if (zp_check_device() != ZP_OK) return ZP_ENODEV;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_pitch_bytes};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    std::snprintf(g_err, sizeof(g_err), "cuTensorMapEncodeTiled (f32) failed (CUresult %d)", int(r));
    return ZP_ETMA;
  }
  return ZP_OK;
}

extern "C" const char* zp_last_error(void) { return g_err; }

extern "C" int zp_version(void) { return 2; }  // 2: parity kernel, ring hops, phased remap, spin bound

extern "C" int zp_device_sm_count(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    return zp_fail(ZP_ENODEV, "no CUDA device visible");
  }
  return n;
}

extern "C" int zp_ipc_get_handle(void* dev_ptr, void* handle_out64, int64_t* offset_out) {
  typedef CUresult (*PFN_range)(CUdeviceptr*, size_t*, CUdeviceptr);
  static PFN_range range_fn = nullptr;
  if (!range_fn) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      cudaGetLastError();
      return zp_fail(ZP_ENODEV, "cuMemGetAddressRange entry point unavailable");
    }
    range_fn = reinterpret_cast<PFN_range>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range_fn(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return zp_fail(ZP_ECUDA, "cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return zp_fail_cuda(e, "cudaIpcGetMemHandle");
  std::memcpy(handle_out64, &h, sizeof(h));
  *offset_out = int64_t(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
  return ZP_OK;
}

extern "C" int zp_ipc_open_handle(const void* handle64, void** dev_ptr_out) {
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return zp_fail_cuda(e, "cudaIpcOpenMemHandle");
  return ZP_OK;
}

extern "C" int zp_ipc_close_handle(void* dev_ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
  if (e != cudaSuccess) return zp_fail_cuda(e, "cudaIpcCloseMemHandle");
  return ZP_OK;
}
