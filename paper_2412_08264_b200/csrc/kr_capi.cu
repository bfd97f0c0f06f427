// kr_capi.cu -- ABI version, error state, operator validation, device queries.
#include <cstring>
#include <map>
#include <mutex>
#include <utility>
#include <string>

#include <cudaTypedefs.h>
#include <cstdlib>

#include "kr_common.cuh"
#include "kr_internal.h"

namespace kr {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(KR_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return KR_OK;
}

int validate_op(const kr_op& op) {
  if (op.rows <= 0 || op.cols <= 0) return fail(KR_EINVAL, "image shape must be positive");
  if (op.batch < 0) return fail(KR_EINVAL, "batch must be nonnegative");
  switch (op.data_kind) {
    case KR_DATA_NONE:
      break;
    case KR_DATA_MASK:
      if (!op.mask) return fail(KR_EINVAL, "mask data term without a mask");
      break;
    case KR_DATA_BLUR:
      if (op.blur_size < 1 || op.blur_size % 2 == 0 || op.blur_size > KR_MAX_BLUR)
        return fail(KR_EINVAL, "blur size must be odd and <= 31");
      break;
    case KR_DATA_DENSE:
      if (!op.dense) return fail(KR_EINVAL, "dense operator without a matrix");
      if (op.rows != 1) return fail(KR_EINVAL, "dense operators use rows = 1, cols = n");
      return KR_OK;
    default:
      return fail(KR_EINVAL, "unknown data kind");
  }
  if (!(op.ridge >= 0.0)) return fail(KR_EINVAL, "ridge must be nonnegative");
  switch (op.reg_kind) {
    case KR_REG_NONE:
      break;
    case KR_REG_FILTERS:
      if (op.num_filters < 1 || op.num_filters > KR_MAX_FILTERS) return fail(KR_EINVAL, "1 <= num_filters <= 64");
      if (op.ksize < 1 || op.ksize % 2 == 0 || op.ksize > KR_MAX_KSIZE)
        return fail(KR_EINVAL, "kernel size must be odd and <= 9");
      if (!op.kernels || !op.fweights) return fail(KR_EINVAL, "filters without kernels / weights");
      if (op.potential != KR_POT_QUADRATIC && op.potential != KR_POT_SMOOTH_ABS)
        return fail(KR_EINVAL, "unknown potential");
      if (op.potential == KR_POT_SMOOTH_ABS && !(op.eps > 0.0)) return fail(KR_EINVAL, "eps must be positive");
      break;
    case KR_REG_TV:
      if (!op.fweights) return fail(KR_EINVAL, "TV without a weight");
      if (!(op.eps > 0.0)) return fail(KR_EINVAL, "eps must be positive");
      break;
    default:
      return fail(KR_EINVAL, "unknown regulariser kind");
  }
  return KR_OK;
}

// The opt-in cap only ever grows (per kernel and device): host threads launching
// the same kernel with different sizes must not lower it under each other.
int ensure_smem(const void* kernel, size_t bytes) {
  if (bytes > 227 * 1024) return fail(KR_EINVAL, "tile needs more than 227 KB of shared memory");
  if (bytes > 48 * 1024) {
    // Opt in ONCE per (device, kernel) to the largest dynamic size the device allows: the
    // launch's own smem request still sets the occupancy, and raising the attribute again
    // later (e.g. as the candidate width t grows) would be a cudaFuncSetAttribute on a
    // kernel that another host thread's stream may be running -- the driver serialises
    // that call behind the running launch (measured: ~1 ms stalls of the recycle update).
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> cap;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    size_t& c = cap[{dev, kernel}];
    if (bytes > c) {
      int optin = 0;
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
      cudaFuncAttributes fa{};
      cudaFuncGetAttributes(&fa, kernel);
      size_t lim = optin > 0 ? (size_t)optin - fa.sharedSizeBytes : bytes;
      if (lim < bytes) lim = bytes;
      cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lim);
      if (e != cudaSuccess)
        return fail(KR_ECUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e) + " (dynamic " +
                                  std::to_string(bytes) + " B + static " + std::to_string(fa.sharedSizeBytes) +
                                  " B > opt-in " + std::to_string(optin) + " B)");
      c = lim;
    }
  }
  return KR_OK;
}

bool make_region_tmap(CUtensorMap* map, const double* base, int cols, int rows, int64_t ncols, int64_t batch,
                      int64_t ld, int64_t bs, int box_w, int box_h) {
  static const bool off = getenv("KR_TMA") && getenv("KR_TMA")[0] == '0';
  if (off || !base || ((uintptr_t)base & 15) || cols % 2 || ld % 2 || bs % 2 || box_w % 2 || box_w > 256 ||
      box_h > 256 || cols < 2 || rows < 1 || ncols < 1 || batch < 1)
    return false;
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      enc = nullptr;
  }
  if (!enc) return false;
  const cuuint64_t dims[4] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)ncols, (cuuint64_t)batch};
  const cuuint64_t strides[3] = {(cuuint64_t)cols * 8, (cuuint64_t)ld * 8, (cuuint64_t)bs * 8};
  const cuuint32_t box[4] = {(cuuint32_t)box_w, (cuuint32_t)box_h, 1, 1};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int device_sms() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

}  // namespace kr

extern "C" int kr_abi_version(void) { return KR_ABI_VERSION; }

extern "C" const char* kr_last_error(void) { return kr::g_last_error.c_str(); }

extern "C" int kr_device_info(int32_t* num_sms, int32_t* cc_major, int32_t* cc_minor) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return kr::fail(KR_ECUDA, std::string("cudaGetDevice: ") + cudaGetErrorString(e));
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  if (num_sms) *num_sms = v;
  cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMajor, dev);
  if (cc_major) *cc_major = v;
  cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMinor, dev);
  if (cc_minor) *cc_minor = v;
  return KR_OK;
}

extern "C" int kr_struct_sizes(int64_t* op_size, int64_t* args_size) {
  if (op_size) *op_size = (int64_t)sizeof(kr_op);
  if (args_size) *args_size = (int64_t)sizeof(kr_solve_args);
  return KR_OK;
}

namespace kr {

// One cuSOLVER handle per (host thread, device); the stream is rebound per call.
int cusolver_handle(cusolverDnHandle_t* out, cudaStream_t st) {
  static thread_local cusolverDnHandle_t handles[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return fail(KR_ECUDA, "device index out of range");
  if (!handles[dev] && cusolverDnCreate(&handles[dev]) != CUSOLVER_STATUS_SUCCESS)
    return fail(KR_ECUDA, "cusolverDnCreate failed");
  if (cusolverDnSetStream(handles[dev], st) != CUSOLVER_STATUS_SUCCESS)
    return fail(KR_ECUDA, "cusolverDnSetStream failed");
  *out = handles[dev];
  return KR_OK;
}


}  // namespace kr
