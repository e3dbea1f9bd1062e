// Multi-GPU statistics reduction for cs_sweep_random_multi: NCCL
// communicators over this process's devices 0..n-1 (ncclCommInitAll), one
// SUM all-reduce of a packed int64 buffer per round. NCCL is loaded at run
// time (libnccl.so.2), so single-GPU users of the library never need it.
//
// Packed layout (n devices): four per-device key slots each — [0, n) min
// keys, [n, 2n) max keys, [2n, 3n) iteration-time min keys, [3n, 4n)
// iteration-time max keys (each device writes only its own slots, the
// others stay 0) — then words 2..2007 of the statistics (counters and
// histograms, summed; the key words among them are zeroed), then n pairs of
// float64 bit patterns (per-device slots; summed in device order on the
// host, so the result is deterministic). Keys are (m << key_bits) |
// (seed - round base), as in the single-device statistics
// (include/commsched.h CS_DSTATS_*).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <cstdlib>
#include <nccl.h>

#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "core.hpp"
#include "sweep.hpp"

namespace tictac {

namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string why;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // An NCCL already in the process (e.g. torch's) first; then the one
    // TICTAC_NCCL_LIB names (the Python binding points it at torch's
    // bundled copy, so a later `import torch` finds the same, newer library
    // under the shared soname); then the system's. Loaded RTLD_LOCAL: its
    // symbols never interpose on other libraries.
    api.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    const char* env = std::getenv("TICTAC_NCCL_LIB");
    if (!api.h && env && *env) api.h = dlopen(env, RTLD_NOW | RTLD_LOCAL);
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      if (api.h) break;
      api.h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
    }
    if (!api.h) {
      api.why = std::string("NCCL unavailable: ") + dlerror();
      return;
    }
    api.comm_init_all = reinterpret_cast<decltype(api.comm_init_all)>(dlsym(api.h, "ncclCommInitAll"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(api.h, "ncclAllReduce"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(api.h, "ncclGetErrorString"));
    if (!api.comm_init_all || !api.all_reduce || !api.error_string) api.why = "NCCL symbols missing";
  });
  return api;
}

void nccheck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(kInternal, std::string(what) + ": " + nccl().error_string(r));
}

void ck(cudaError_t e) {
  if (e != cudaSuccess) fail(kInternal, std::string("CUDA error: ") + cudaGetErrorString(e));
}

class NcclReducer final : public DeviceReducer {
 public:
  explicit NcclReducer(int n) : n_(n), comms_(n) {
    const NcclApi& api = nccl();
    if (!api.why.empty()) fail(kInternal, api.why);
    std::vector<int> devs(n);
    for (int d = 0; d < n; ++d) devs[d] = d;
    nccheck(api.comm_init_all(comms_.data(), n, devs.data()), "ncclCommInitAll");
  }
  // Communicators stay alive for the process (like the reference's
  // thread-local error string, they are process-lifetime state).
  void reduce(int d, const int64_t* d_i64, const double* d_f64, int64_t* h_i64, double* h_f64) const override {
    const size_t kw = 4 * static_cast<size_t>(n_), cw = CS_DSTATS_I64 - 2;
    const size_t words = kw + cw + CS_DSTATS_F64 * static_cast<size_t>(n_);
    int64_t* buf = nullptr;
    ck(cudaMallocAsync(&buf, 8 * words, 0));
    struct Free {
      int64_t* p;
      ~Free() { cudaFreeAsync(p, 0); }
    } guard{buf};
    ck(cudaMemsetAsync(buf, 0, 8 * words, 0));
    ck(cudaMemcpyAsync(buf + d, d_i64, 8, cudaMemcpyDeviceToDevice, 0));
    ck(cudaMemcpyAsync(buf + n_ + d, d_i64 + 1, 8, cudaMemcpyDeviceToDevice, 0));
    ck(cudaMemcpyAsync(buf + 2 * n_ + d, d_i64 + 4, 8, cudaMemcpyDeviceToDevice, 0));
    ck(cudaMemcpyAsync(buf + 3 * n_ + d, d_i64 + 5, 8, cudaMemcpyDeviceToDevice, 0));
    ck(cudaMemcpyAsync(buf + kw, d_i64 + 2, 8 * cw, cudaMemcpyDeviceToDevice, 0));
    ck(cudaMemsetAsync(buf + kw + 2, 0, 16, 0));  // words 4, 5 travel in the key slots
    const size_t fo = kw + cw;
    ck(cudaMemcpyAsync(buf + fo + CS_DSTATS_F64 * static_cast<size_t>(d), d_f64, 8 * CS_DSTATS_F64,
                       cudaMemcpyDeviceToDevice, 0));
    nccheck(nccl().all_reduce(buf, buf, words, ncclInt64, ncclSum, comms_[d], 0), "ncclAllReduce");
    if (!h_i64) {
      ck(cudaStreamSynchronize(0));
      return;
    }
    std::vector<int64_t> h(words);
    ck(cudaMemcpyAsync(h.data(), buf, 8 * words, cudaMemcpyDeviceToHost, 0));
    ck(cudaStreamSynchronize(0));
    uint64_t kmin = ~0ULL, kmax = 0, ikmin = ~0ULL, ikmax = 0;  // an idle device's min keys are all ones
    for (int k = 0; k < n_; ++k) {
      kmin = std::min(kmin, static_cast<uint64_t>(h[k]));
      kmax = std::max(kmax, static_cast<uint64_t>(h[n_ + k]));
      ikmin = std::min(ikmin, static_cast<uint64_t>(h[2 * n_ + k]));
      ikmax = std::max(ikmax, static_cast<uint64_t>(h[3 * n_ + k]));
    }
    std::memcpy(h_i64 + 2, h.data() + kw, 8 * cw);
    h_i64[0] = static_cast<int64_t>(kmin);
    h_i64[1] = static_cast<int64_t>(kmax);
    h_i64[4] = static_cast<int64_t>(ikmin);
    h_i64[5] = static_cast<int64_t>(ikmax);
    for (int f = 0; f < CS_DSTATS_F64; ++f) {
      double acc = 0.0;
      for (int k = 0; k < n_; ++k) {
        double x;
        std::memcpy(&x, &h[fo + CS_DSTATS_F64 * static_cast<size_t>(k) + f], 8);
        acc += x;
      }
      h_f64[f] = acc;
    }
  }

 private:
  int n_;
  mutable std::vector<ncclComm_t> comms_;
};

}  // namespace

const DeviceReducer& nccl_reducer(int n_devices, std::unique_lock<std::mutex>& hold) {
  static std::mutex mu;  // one multi-GPU sweep at a time per communicator set
  static std::vector<std::unique_ptr<NcclReducer>> cache(65);
  hold = std::unique_lock<std::mutex>(mu);
  if (n_devices < 2 || n_devices > 64) fail(kParameter, "n_devices must be within [2, 64]");
  if (!cache[n_devices]) cache[n_devices] = std::make_unique<NcclReducer>(n_devices);
  return *cache[n_devices];
}

}  // namespace tictac
