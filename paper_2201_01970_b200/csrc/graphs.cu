// CUDA-graph cache for the CPR application: the ~300 colour-sweep / transfer
// launches of one preconditioner application are captured once per (plan,
// input, output) triple and replayed with a single cudaGraphLaunch, so the
// GPU runs them back to back without host launch gaps.
#include <list>
#include <map>
#include <tuple>

#include "engine.h"

namespace {

struct GraphCache {
  using Key = std::tuple<const void*, const void*, const void*>;
  std::map<Key, cudaGraphExec_t> map;
  std::list<Key> lru;
  cudaStream_t cap = nullptr;
  size_t cap_limit = 64;
  ~GraphCache() {
    for (auto& kv : map) cudaGraphExecDestroy(kv.second);
    if (cap) cudaStreamDestroy(cap);
  }
};

}  // namespace

using namespace cprb;

extern "C" {

int cprb_cpr_apply(const cprb_cpr* P, const double* r, double* z, void* stream);

int cprb_graph_cache_create(void** out) {
  auto* c = new GraphCache();
  if (cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return check_launch("graph cache stream");
  }
  *out = c;
  return CPRB_OK;
}

int cprb_graph_cache_destroy(void* h) {
  delete static_cast<GraphCache*>(h);
  return CPRB_OK;
}

int cprb_amg_cycle(const cprb_amg* h, const double* r, double* z, void* stream);

static int graph_run(void* h, int op, const void* P, const double* r, double* z, void* stream);

int cprb_cpr_apply_graph(void* h, const cprb_cpr* P, const double* r, double* z, void* stream) {
  return graph_run(h, 0, P, r, z, stream);
}

int cprb_amg_cycle_graph(void* h, const cprb_amg* A, const double* r, double* z, void* stream) {
  return graph_run(h, 1, A, r, z, stream);
}

static int graph_run(void* h, int op, const void* P, const double* r, double* z, void* stream) {
  auto* c = static_cast<GraphCache*>(h);
  GraphCache::Key key{(const char*)P + op, r, z};
  auto it = c->map.find(key);
  cudaGraphExec_t exec = nullptr;
  if (it == c->map.end()) {
    cudaGraph_t g = nullptr;
    if (cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
      return check_launch("begin capture");
    int rc = op == 0 ? cprb_cpr_apply((const cprb_cpr*)P, r, z, c->cap)
                     : cprb_amg_cycle((const cprb_amg*)P, r, z, c->cap);
    cudaError_t e = cudaStreamEndCapture(c->cap, &g);
    if (rc) return rc;
    if (e != cudaSuccess) return set_error(CPRB_EDEVICE, std::string("end capture: ") + cudaGetErrorString(e));
    e = cudaGraphInstantiate(&exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return set_error(CPRB_EDEVICE, std::string("instantiate: ") + cudaGetErrorString(e));
    if (c->map.size() >= c->cap_limit) {
      auto old = c->lru.front();
      c->lru.pop_front();
      cudaGraphExecDestroy(c->map[old]);
      c->map.erase(old);
    }
    c->map[key] = exec;
    c->lru.push_back(key);
  } else {
    exec = it->second;
  }
  if (cudaGraphLaunch(exec, (cudaStream_t)stream) != cudaSuccess) return check_launch("graph launch");
  return CPRB_OK;
}

}  // extern "C"
