// Ring KV exchange without SMs: copy-engine pulls between IPC-mapped ring
// buffers, ordered by epoch flags that the GPUs' stream front-ends wait on and
// write (CUDA stream memory operations).  A hop therefore overlaps a ring
// round's persistent attention kernel completely — it needs no CTA, so the
// round keeps all 148 SMs.
//
// Reference semantics: after round r, ring position i forwards the KV set it
// holds to position i+1 (attention_engine.py:247-251, src of round r is
// (i - r) mod g, :237).  Here position i+1 PULLS it: the receiver copies from
// its predecessor's buffer once the predecessor announced the set ("full"),
// and announces back when it finished reading ("consumed") so the buffer can
// be refilled.  Flags are int32 epochs compared with wrap-around GEQ.
#include "zp_host.h"
#include "../../include/zeppelin_b200.h"

namespace {

typedef CUresult (*PFN_waitValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PFN_writeValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PFN_waitValue32 g_wait = nullptr;
PFN_writeValue32 g_write = nullptr;

int load_memops() {
  if (g_wait && g_write) return ZP_OK;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn) {
    cudaGetLastError();
    return zp_fail(ZP_ENODEV, "cuStreamWaitValue32 entry point unavailable");
  }
  g_wait = reinterpret_cast<PFN_waitValue32>(fn);
  fn = nullptr;
  if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn) {
    cudaGetLastError();
    return zp_fail(ZP_ENODEV, "cuStreamWriteValue32 entry point unavailable");
  }
  g_write = reinterpret_cast<PFN_writeValue32>(fn);
  return ZP_OK;
}

int wait_geq(const int32_t* flag, int32_t epoch, cudaStream_t s) {
  CUresult r = g_wait(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(flag), cuuint32_t(epoch),
                      CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) return zp_fail(ZP_ECUDA, "cuStreamWaitValue32 failed");
  return ZP_OK;
}

// The default write carries a memory barrier: every preceding operation of
// the stream (the hop's copy) is visible before the flag.
int write_flag(int32_t* flag, int32_t epoch, cudaStream_t s) {
  CUresult r = g_write(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(flag), cuuint32_t(epoch),
                       CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r != CUDA_SUCCESS) return zp_fail(ZP_ECUDA, "cuStreamWriteValue32 failed");
  return ZP_OK;
}

}  // namespace

extern "C" int zp_stream_wait_flag(const int32_t* flag, int32_t epoch, void* stream) {
  if (!flag) return zp_fail(ZP_EINVAL, "zp_stream_wait_flag: null flag");
  if (zp_check_device() != ZP_OK || load_memops() != ZP_OK) return ZP_ENODEV;
  return wait_geq(flag, epoch, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int zp_stream_write_flag(int32_t* flag, int32_t epoch, void* stream) {
  if (!flag) return zp_fail(ZP_EINVAL, "zp_stream_write_flag: null flag");
  if (zp_check_device() != ZP_OK || load_memops() != ZP_OK) return ZP_ENODEV;
  return write_flag(flag, epoch, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int zp_ring_hop(void* dst, const void* src, int64_t bytes, const int32_t* full_flag,
                           int32_t full_epoch, const int32_t* free_flag, int32_t free_epoch,
                           int32_t* consumed_flag, int32_t consumed_epoch, int32_t* next_full_flag,
                           int32_t next_full_epoch, void* stream) {
  if (bytes < 0 || (bytes > 0 && (!dst || !src)) || !full_flag || !consumed_flag)
    return zp_fail(ZP_EINVAL, "zp_ring_hop: bad arguments");
  if (zp_check_device() != ZP_OK || load_memops() != ZP_OK) return ZP_ENODEV;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int rc;
  // 1. the predecessor's set is in its buffer
  if ((rc = wait_geq(full_flag, full_epoch, s)) != ZP_OK) return rc;
  // 2. my successor finished reading what my destination buffer held before
  if (free_flag && (rc = wait_geq(free_flag, free_epoch, s)) != ZP_OK) return rc;
  // 3. the pull itself: one copy-engine transfer over NVLink
  if (bytes > 0) {
    cudaError_t e = cudaMemcpyAsync(dst, src, size_t(bytes), cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return zp_fail_cuda(e, "zp_ring_hop: copy");
  }
  // 4. tell the predecessor its buffer may be refilled
  if ((rc = write_flag(consumed_flag, consumed_epoch, s)) != ZP_OK) return rc;
  // 5. tell the successor my buffer holds the set it pulls next
  if (next_full_flag && (rc = write_flag(next_full_flag, next_full_epoch, s)) != ZP_OK) return rc;
  return ZP_OK;
}

extern "C" int zp_memcpy_async(void* dst, const void* src, int64_t bytes, void* stream) {
  if (bytes < 0 || (bytes > 0 && (!dst || !src))) return zp_fail(ZP_EINVAL, "zp_memcpy_async: bad arguments");
  if (bytes == 0) return ZP_OK;
  if (zp_check_device() != ZP_OK) return ZP_ENODEV;
  cudaError_t e = cudaMemcpyAsync(dst, src, size_t(bytes), cudaMemcpyDeviceToDevice,
                                  reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return zp_fail_cuda(e, "zp_memcpy_async");
  return ZP_OK;
}

extern "C" int zp_memset_async(void* dst, int value, int64_t bytes, void* stream) {
  if (bytes < 0 || (bytes > 0 && !dst)) return zp_fail(ZP_EINVAL, "zp_memset_async: bad arguments");
  if (bytes == 0) return ZP_OK;
  if (zp_check_device() != ZP_OK) return ZP_ENODEV;
  cudaError_t e = cudaMemsetAsync(dst, value, size_t(bytes), reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return zp_fail_cuda(e, "zp_memset_async");
  return ZP_OK;
}
