// Device-resident graph structure: CSR adjacency in the reference's index
// model plus per-resource op lists and ready-bitset offsets for the event
// simulator. Uploaded once per cs_graph (lazily) and reused by every call.
#include <mutex>
#include <vector>

#include "common.cuh"
#include "csk.h"
#include "devgraph.cuh"

namespace tictac_dev {

std::atomic<int64_t> g_launches{0};

int ensure_device(char* err) {
  static int ok = -1;
  static char msg[256];
  static std::once_flag once;  // first calls may come from several threads
  std::call_once(once, [] {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
      std::snprintf(msg, sizeof msg, "CUDA device unavailable: %s",
                    e != cudaSuccess ? cudaGetErrorString(e) : "no devices");
      ok = 0;
    } else {
      e = cudaFree(nullptr);  // create the primary context
      if (e != cudaSuccess) {
        std::snprintf(msg, sizeof msg, "CUDA context creation failed: %s", cudaGetErrorString(e));
        ok = 0;
      } else {
        ok = 1;
        // per-call buffers come from the stream-ordered allocator; keep what
        // it has reserved instead of returning it to the driver at each sync
        int dev = 0;
        cudaMemPool_t pool;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
          uint64_t keep = UINT64_MAX;
          cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        cudaGetLastError();
      }
    }
  });
  if (!ok) std::snprintf(err, 256, "%s", msg);
  return ok ? 0 : 1;
}

template <typename T>
static int upload(T** dst, const T* src, size_t count, char* err) {
  CK(cudaMalloc(reinterpret_cast<void**>(dst), sizeof(T) * (count ? count : 1)));
  if (count) CK(cudaMemcpy(*dst, src, sizeof(T) * count, cudaMemcpyHostToDevice));
  return 0;
}

}  // namespace tictac_dev

using namespace tictac_dev;

extern "C" DeviceGraph* csk_graph_upload(int32_t n, const int32_t* pred_off, const int32_t* pred_idx,
                                         const int32_t* succ_off, const int32_t* succ_idx,
                                         const int8_t* kind, const int32_t* res, int32_t n_res,
                                         const int8_t* res_channel, const int32_t* res_device,
                                         int32_t n_dev, char* err) {
  if (ensure_device(err)) return nullptr;
  auto* g = new DeviceGraph();
  g->n = n;
  g->nres = n_res;
  g->ndev = n_dev;
  g->h_pred_off.assign(pred_off, pred_off + n + 1);
  g->h_pred_idx.assign(pred_idx, pred_idx + pred_off[n]);
  g->h_succ_off.assign(succ_off, succ_off + n + 1);
  g->h_succ_idx.assign(succ_idx, succ_idx + succ_off[n]);
  g->h_kind.assign(kind, kind + n);
  g->h_res.assign(res, res + n);
  g->h_chan.assign(res_channel, res_channel + n_res);
  g->h_res_dev.assign(res_device, res_device + n_res);
  // per-resource op lists (ascending op index) and local indices
  std::vector<int32_t> rops_off(n_res + 1, 0), rops(n), lidx(n), rb_off(n_res + 1, 0);
  for (int32_t i = 0; i < n; ++i) rops_off[res[i] + 1]++;
  for (int32_t r = 0; r < n_res; ++r) rops_off[r + 1] += rops_off[r];
  std::vector<int32_t> fill(rops_off.begin(), rops_off.end() - 1);
  for (int32_t i = 0; i < n; ++i) {
    lidx[i] = fill[res[i]] - rops_off[res[i]];
    rops[fill[res[i]]++] = i;
  }
  for (int32_t r = 0; r < n_res; ++r)
    rb_off[r + 1] = rb_off[r] + (rops_off[r + 1] - rops_off[r] + 31) / 32;
  std::vector<int32_t> col(n, -1), recv_ops;
  for (int32_t i = 0; i < n; ++i)
    if (kind[i] == 1) {
      col[i] = static_cast<int32_t>(recv_ops.size());
      recv_ops.push_back(i);
    }
  g->R = static_cast<int32_t>(recv_ops.size());
  g->rb_words = rb_off[n_res];
  g->h_recv_ops = recv_ops;
  g->h_col = col;
  if (upload(&g->pred_off, pred_off, n + 1, err) || upload(&g->pred_idx, pred_idx, pred_off[n], err) ||
      upload(&g->succ_off, succ_off, n + 1, err) || upload(&g->succ_idx, succ_idx, succ_off[n], err) ||
      upload(&g->kind, kind, n, err) || upload(&g->res, res, n, err) ||
      upload(&g->chan, res_channel, n_res, err) || upload(&g->res_dev, res_device, n_res, err) ||
      upload(&g->rops_off, rops_off.data(), n_res + 1, err) || upload(&g->rops, rops.data(), n, err) ||
      upload(&g->lidx, lidx.data(), n, err) || upload(&g->rb_off, rb_off.data(), n_res + 1, err) ||
      upload(&g->recv_ops, recv_ops.data(), recv_ops.size(), err) ||
      upload(&g->col, col.data(), n, err)) {
    csk_graph_free(g);
    return nullptr;
  }
  return g;
}

extern "C" void csk_graph_free(DeviceGraph* g) {
  if (!g) return;
  void* ptrs[] = {g->pred_off, g->pred_idx, g->succ_off, g->succ_idx, g->kind, g->res,
                  g->chan,     g->res_dev,  g->rops_off, g->rops,     g->lidx, g->rb_off,
                  g->recv_ops, g->col};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (g->rows) {
    const Rows& r = *g->rows;
    const void* rp[] = {r.d_self, r.d_preoff, r.d_pre,    r.d_rowof,   r.d_succoff, r.d_succ,
                        r.d_ntrow, r.d_ntoff, r.d_ntterm, r.d_ntchunk, r.d_hasrows, r.d_g1};
    for (const void* p : rp)
      if (p) cudaFree(const_cast<void*>(p));
  }
  delete g;
}

extern "C" int64_t csk_launches(void) { return g_launches.load(); }
