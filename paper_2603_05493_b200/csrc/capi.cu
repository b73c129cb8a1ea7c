// Library-level pieces of the C ABI: error text, streams, CUDA-graph helpers.
#include <cstdlib>
#include <string>

#include "common.cuh"

namespace ksb {

static thread_local std::string g_error;
std::atomic<int64_t> g_kernel_launches{0};

void set_error(const std::string& message) { g_error = message; }
int fail(int status, const std::string& message) {
  g_error = message;
  return status;
}
int cuda_fail(cudaError_t err, const char* what) {
  g_error = std::string("cuda: ") + cudaGetErrorString(err) + " in " + what;
  return KS_ERR_CUDA;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* off = std::getenv("KS_B200_NO_PDL");
    return !(off && off[0] == '1');
  }();
  return on;
}

}  // namespace ksb

using namespace ksb;

struct ks_graph {
  cudaGraph_t graph;
  cudaGraphExec_t exec;
};

extern "C" {

const char* ks_last_error(void) { return g_error.c_str(); }
const char* ks_version(void) { return "ks_b200 0.1 (sm_100a)"; }

int ks_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int64_t ks_kernel_launch_count(void) { return g_kernel_launches.load(); }

int ks_stream_create(ks_stream* out) {
  if (!out) return fail(KS_ERR_INVALID, "null argument");
  cudaStream_t s;
  KS_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  *out = s;
  return KS_OK;
}
int ks_stream_destroy(ks_stream s) {
  KS_CUDA(cudaStreamDestroy(static_cast<cudaStream_t>(s)));
  return KS_OK;
}
int ks_stream_sync(ks_stream s) {
  KS_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(s)));
  return KS_OK;
}

int ks_graph_begin_capture(ks_stream s) {
  KS_CUDA(cudaStreamBeginCapture(static_cast<cudaStream_t>(s), cudaStreamCaptureModeThreadLocal));
  return KS_OK;
}
int ks_graph_end_capture(ks_stream s, ks_graph** out) {
  if (!out) return fail(KS_ERR_INVALID, "null argument");
  ks_graph* g = new ks_graph{nullptr, nullptr};
  cudaError_t err = cudaStreamEndCapture(static_cast<cudaStream_t>(s), &g->graph);
  if (err == cudaSuccess) err = cudaGraphInstantiate(&g->exec, g->graph, 0);
  if (err != cudaSuccess) {
    if (g->graph) cudaGraphDestroy(g->graph);
    delete g;
    return cuda_fail(err, "graph capture");
  }
  *out = g;
  return KS_OK;
}
int ks_graph_launch(ks_graph* g, ks_stream s) {
  if (!g) return fail(KS_ERR_INVALID, "null graph");
  KS_CUDA(cudaGraphLaunch(g->exec, static_cast<cudaStream_t>(s)));
  return KS_OK;
}
int ks_graph_node_count(ks_graph* g, int64_t* kernel_nodes, int64_t* all_nodes) {
  if (!g) return fail(KS_ERR_INVALID, "null graph");
  size_t n = 0;
  KS_CUDA(cudaGraphGetNodes(g->graph, nullptr, &n));
  std::string unused;
  cudaGraphNode_t* nodes = new cudaGraphNode_t[n ? n : 1];
  cudaError_t err = cudaGraphGetNodes(g->graph, nodes, &n);
  int64_t kernels = 0;
  for (size_t i = 0; err == cudaSuccess && i < n; ++i) {
    cudaGraphNodeType type;
    err = cudaGraphNodeGetType(nodes[i], &type);
    kernels += type == cudaGraphNodeTypeKernel;
  }
  delete[] nodes;
  if (err != cudaSuccess) return cuda_fail(err, "graph nodes");
  if (kernel_nodes) *kernel_nodes = kernels;
  if (all_nodes) *all_nodes = static_cast<int64_t>(n);
  return KS_OK;
}
void ks_graph_destroy(ks_graph* g) {
  if (!g) return;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  delete g;
}

}  // extern "C"
