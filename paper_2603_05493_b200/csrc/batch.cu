// Batched environments (BASELINE.json configs[4]; the reference has no batch API).
//
// A ks_batch owns n independent worlds -- one SparseTsdf + one DenseEsdf each, same configuration -- and runs one update
// of all of them (upload staged frames -> integrate_depth per camera -> stamp_primitive for the environment's primitives
// and meshes -> build_esdf -> a 32-byte collision summary) as ONE enqueue, ONE captured graph.  Nothing is shared between
// environments, so there is no data-path collective; the only exchange is an ncclAllGather of the summaries, enqueued
// on the same stream (a node of the same graph) when a communicator is attached.
//
// Execution: the environments are dealt round-robin onto `lanes` streams that fork from and join into the batch's main
// stream.  Inside one lane an environment's kernels keep their programmatic-launch chain; across lanes the short,
// latency-bound kernels of one environment (discovery, allocation, directory, seeding) run beside the sweeps of
// another, which is what "environment as the outer grid dimension" buys for kernels that do not fill the GPU.
//
// This file is a composition layer: it only calls the C ABI of tsdf.cu / esdf.cu, so a batch update leaves every world
// exactly as the per-handle calls would (tests/test_gpu_env_batch.py compares each environment with its own oracle world).
#include <dlfcn.h>

#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

using namespace ksb;

namespace {

// ---- NCCL, resolved at run time (the library itself links only the static CUDA runtime) -----------------------------
struct UniqueId {
  char bytes[128];  // NCCL_UNIQUE_ID_BYTES
};
struct NcclApi {
  void* lib = nullptr;
  int (*GetUniqueId)(void*) = nullptr;
  int (*CommInitRank)(void**, int, UniqueId /* ncclUniqueId, by value */, int) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  int (*CommDestroy)(void*) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  std::string why;
};
constexpr int kNcclFloat64 = 8;  // ncclDouble

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    const char* names[] = {std::getenv("KS_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
    for (const char* name : names) {
      if (!name || !*name) continue;
      a.lib = dlopen(name, RTLD_NOW | RTLD_NOLOAD);  // the copy the host process already mapped (torch bundles one)
      if (!a.lib) a.lib = dlopen(name, RTLD_NOW | RTLD_LOCAL);
      if (a.lib) break;
    }
    if (!a.lib) {
      a.why = "nccl: libnccl.so.2 not found (set KS_NCCL_LIB)";
      return a;
    }
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(a.lib, "ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(a.lib, "ncclCommInitRank"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(a.lib, "ncclAllGather"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(a.lib, "ncclCommDestroy"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(a.lib, "ncclGetErrorString"));
    if (!a.GetUniqueId || !a.CommInitRank || !a.AllGather || !a.CommDestroy) a.why = "nccl: symbols missing in libnccl", a.lib = nullptr;
    return a;
  }();
  return api;
}

int nccl_fail(int rc, const char* what) {
  NcclApi& a = nccl();
  return fail(KS_ERR_CUDA, std::string("nccl: ") + (a.GetErrorString ? a.GetErrorString(rc) : "error") + " in " + what);
}

struct EnvInputs {
  int cameras = 1;
  std::vector<ks_primitive> prims;
  std::vector<const ks_mesh*> meshes;
  double* probes_dev = nullptr;
  int64_t n_probes = 0;
  double near_distance = 0.0;
};

}  // namespace

struct ks_batch {
  int n = 0, lanes = 1;
  std::vector<ks_tsdf*> tsdf;
  std::vector<ks_esdf*> esdf;
  std::vector<EnvInputs> in;
  cudaStream_t main = nullptr;
  std::vector<cudaStream_t> lane;  // lane[0] == main
  cudaEvent_t fork = nullptr;
  std::vector<cudaEvent_t> join;
  int first_env = 0;               // global id of environment 0 (the tag of its summary row)
  double* summary_dev = nullptr;   // [n][4]  {env id, min probe distance, probes within near_distance, seed count}
  double* gathered_dev = nullptr;  // [world][max_local][4]
  int world = 1, rank = 0, max_local = 0;
  void* comm = nullptr;
  bool own_comm = false;
  cudaGraphExec_t exec[2] = {nullptr, nullptr};  // private graphs of one update: [0] frames resident, [1] frames uploaded first
  int64_t exec_nodes[2] = {0, 0};
  bool dirty = true;                             // inputs changed since the captures
};

namespace {

int enqueue_env(ks_batch* b, int i, bool upload) {
  int rc;
  ks_tsdf* t = b->tsdf[i];
  ks_esdf* e = b->esdf[i];
  const EnvInputs& in = b->in[i];
  for (int slot = 0; slot < in.cameras; ++slot) {
    if (upload && (rc = ks_tsdf_upload_frame_slot_async(t, slot)) != KS_OK) return rc;
    if ((rc = ks_tsdf_integrate_slot_async(t, slot)) != KS_OK) return rc;
  }
  if (!in.prims.empty() && (rc = ks_tsdf_stamp_batch_async(t, in.prims.data(), static_cast<int32_t>(in.prims.size()))) != KS_OK) return rc;
  for (const ks_mesh* m : in.meshes)
    if ((rc = ks_tsdf_stamp_mesh_async(t, m)) != KS_OK) return rc;
  if ((rc = ks_esdf_build_async(e, t)) != KS_OK) return rc;
  if (in.n_probes > 0)
    rc = ks_esdf_probe_summary_device_async(e, in.probes_dev, in.n_probes, in.near_distance, static_cast<double>(b->first_env + i),
                                            b->summary_dev + 4 * static_cast<size_t>(i));
  return rc;
}

int enqueue_update(ks_batch* b, bool upload) {
  int rc = KS_OK;
  if (b->lanes > 1) {
    KS_CUDA(cudaEventRecord(b->fork, b->main));
    for (int l = 1; l < b->lanes; ++l) KS_CUDA(cudaStreamWaitEvent(b->lane[l], b->fork, 0));
  }
  for (int i = 0; i < b->n && rc == KS_OK; ++i) rc = enqueue_env(b, i, upload);
  if (b->lanes > 1) {  // join even after a failed enqueue: a capture must not be left with dangling branches
    for (int l = 1; l < b->lanes; ++l) {
      cudaEventRecord(b->join[l], b->lane[l]);
      cudaStreamWaitEvent(b->main, b->join[l], 0);
    }
  }
  if (rc != KS_OK) return rc;
  if (b->comm) {
    const int nrc = nccl().AllGather(b->summary_dev, b->gathered_dev, 4 * static_cast<size_t>(b->max_local), kNcclFloat64, b->comm, b->main);
    if (nrc != 0) return nccl_fail(nrc, "ncclAllGather");
  }
  KS_CUDA(cudaGetLastError());
  return KS_OK;
}

void drop_graphs(ks_batch* b) {
  for (int k = 0; k < 2; ++k) {
    if (b->exec[k]) cudaGraphExecDestroy(b->exec[k]);
    b->exec[k] = nullptr;
  }
}

}  // namespace

extern "C" {

int ks_partition_envs(int32_t n_envs, int32_t world, int32_t rank, int32_t* lo, int32_t* hi) {
  if (n_envs < 0 || world < 1 || rank < 0 || rank >= world || !lo || !hi) return fail(KS_ERR_INVALID, "bad partition arguments");
  const int base = n_envs / world, extra = n_envs % world;  // contiguous ranges; earlier ranks take the remainder
  *lo = rank * base + (rank < extra ? rank : extra);
  *hi = *lo + base + (rank < extra ? 1 : 0);
  return KS_OK;
}

int ks_batch_create(int32_t n_envs, const ks_tsdf_config* tsdf_cfg, const ks_esdf_config* esdf_cfg, int32_t lanes, ks_batch** out) {
  if (!out || !tsdf_cfg || !esdf_cfg) return fail(KS_ERR_INVALID, "null argument");
  if (n_envs < 1 || n_envs > 4096) return fail(KS_ERR_INVALID, "batch: n_envs must be in [1, 4096]");
  if (lanes < 1) lanes = 1;
  if (lanes > 8) lanes = 8;
  if (lanes > n_envs) lanes = n_envs;
  ks_batch* b = new ks_batch();
  b->n = n_envs, b->lanes = lanes, b->max_local = n_envs;
  b->in.resize(n_envs);
  auto bail = [&](int rc) {
    const std::string why = ks_last_error();
    ks_batch_destroy(b);
    set_error(why);
    return rc;
  };
  cudaError_t err = cudaStreamCreateWithFlags(&b->main, cudaStreamNonBlocking);
  if (err != cudaSuccess) {
    cuda_fail(err, "batch stream");
    return bail(KS_ERR_CUDA);
  }
  b->lane.assign(lanes, nullptr), b->join.assign(lanes, nullptr);
  b->lane[0] = b->main;
  for (int l = 1; l < lanes && err == cudaSuccess; ++l) {
    err = cudaStreamCreateWithFlags(&b->lane[l], cudaStreamNonBlocking);
    if (err == cudaSuccess) err = cudaEventCreateWithFlags(&b->join[l], cudaEventDisableTiming);
  }
  if (err == cudaSuccess) err = cudaEventCreateWithFlags(&b->fork, cudaEventDisableTiming);
  if (err == cudaSuccess) err = cudaMalloc(&b->summary_dev, sizeof(double) * 4 * n_envs);
  if (err == cudaSuccess) err = cudaMemset(b->summary_dev, 0xFF, sizeof(double) * 4 * n_envs);  // NaN until an update wrote the row
  if (err != cudaSuccess) {
    cuda_fail(err, "batch buffers");
    return bail(KS_ERR_CUDA);
  }
  b->gathered_dev = b->summary_dev;  // one rank: the gathered view is the local one
  for (int i = 0; i < n_envs; ++i) {
    ks_tsdf* t = nullptr;
    ks_esdf* e = nullptr;
    int rc = ks_tsdf_create(tsdf_cfg, &t);
    if (rc != KS_OK) return bail(rc);
    b->tsdf.push_back(t);
    if ((rc = ks_esdf_create(esdf_cfg, &e)) != KS_OK) return bail(rc);
    b->esdf.push_back(e);
    if ((rc = ks_tsdf_set_stream(t, b->lane[i % lanes])) != KS_OK) return bail(rc);
    if ((rc = ks_esdf_set_stream(e, b->lane[i % lanes])) != KS_OK) return bail(rc);
  }
  *out = b;
  return KS_OK;
}

void ks_batch_destroy(ks_batch* b) {
  if (!b) return;
  if (b->main) cudaStreamSynchronize(b->main);
  for (size_t l = 1; l < b->lane.size(); ++l)
    if (b->lane[l]) cudaStreamSynchronize(b->lane[l]);
  drop_graphs(b);
  if (b->comm && b->own_comm && nccl().CommDestroy) nccl().CommDestroy(b->comm);
  for (ks_esdf* e : b->esdf) ks_esdf_destroy(e);
  for (ks_tsdf* t : b->tsdf) ks_tsdf_destroy(t);
  for (EnvInputs& in : b->in)
    if (in.probes_dev) cudaFree(in.probes_dev);
  if (b->gathered_dev && b->gathered_dev != b->summary_dev) cudaFree(b->gathered_dev);
  if (b->summary_dev) cudaFree(b->summary_dev);
  for (size_t l = 1; l < b->lane.size(); ++l) {
    if (b->join[l]) cudaEventDestroy(b->join[l]);
    if (b->lane[l]) cudaStreamDestroy(b->lane[l]);
  }
  if (b->fork) cudaEventDestroy(b->fork);
  if (b->main) cudaStreamDestroy(b->main);
  cudaGetLastError();
  delete b;
}

int32_t ks_batch_size(const ks_batch* b) { return b ? b->n : 0; }
int32_t ks_batch_lanes(const ks_batch* b) { return b ? b->lanes : 0; }
ks_tsdf* ks_batch_tsdf(ks_batch* b, int32_t env) { return b && env >= 0 && env < b->n ? b->tsdf[env] : nullptr; }
ks_esdf* ks_batch_esdf(ks_batch* b, int32_t env) { return b && env >= 0 && env < b->n ? b->esdf[env] : nullptr; }
ks_stream ks_batch_stream(ks_batch* b) { return b ? static_cast<ks_stream>(b->main) : nullptr; }

int ks_batch_set_first_env(ks_batch* b, int32_t first_env) {
  if (!b) return fail(KS_ERR_INVALID, "null batch");
  b->first_env = first_env, b->dirty = true;
  return KS_OK;
}

int ks_batch_set_inputs(ks_batch* b, int32_t env, int32_t n_cameras, const ks_primitive* prims, int32_t n_prims,
                        const ks_mesh* const* meshes, int32_t n_meshes) {
  if (!b || env < 0 || env >= b->n) return fail(KS_ERR_INVALID, "batch: environment out of range");
  if (n_cameras < 0 || n_cameras > KS_MAX_FRAME_SLOTS) return fail(KS_ERR_INVALID, "batch: camera count out of range");
  if ((n_prims > 0 && !prims) || (n_meshes > 0 && !meshes) || n_prims < 0 || n_meshes < 0) return fail(KS_ERR_INVALID, "null argument");
  EnvInputs& in = b->in[env];
  in.cameras = n_cameras;
  in.prims.assign(prims, prims + n_prims);
  in.meshes.assign(meshes, meshes + n_meshes);
  b->dirty = true;
  return KS_OK;
}

int ks_batch_set_probes(ks_batch* b, int32_t env, const double* points_host, int64_t n, double near_distance) {
  if (!b || env < 0 || env >= b->n) return fail(KS_ERR_INVALID, "batch: environment out of range");
  if (n < 0 || (n > 0 && !points_host)) return fail(KS_ERR_INVALID, "null argument");
  EnvInputs& in = b->in[env];
  KS_CUDA(cudaStreamSynchronize(b->lane[env % b->lanes]));  // an update in flight may still read the old points
  if (n != in.n_probes) {
    if (in.probes_dev) cudaFree(in.probes_dev);
    in.probes_dev = nullptr, in.n_probes = 0;
    if (n > 0) KS_CUDA(cudaMalloc(&in.probes_dev, sizeof(double) * 3 * n));
    b->dirty = true;  // the pointer is baked into the captured launch
  }
  if (n > 0) KS_CUDA(cudaMemcpy(in.probes_dev, points_host, sizeof(double) * 3 * n, cudaMemcpyHostToDevice));
  if (in.near_distance != near_distance) b->dirty = true;
  in.n_probes = n, in.near_distance = near_distance;
  return KS_OK;
}

int ks_batch_update_async(ks_batch* b, int32_t upload_frames) {
  if (!b) return fail(KS_ERR_INVALID, "null batch");
  return enqueue_update(b, upload_frames != 0);
}

// the same update through the batch's private graph: captured at the first call (and again after the inputs changed),
// replayed afterwards -- one launch call for n environments
int ks_batch_update(ks_batch* b, int32_t upload_frames) {
  if (!b) return fail(KS_ERR_INVALID, "null batch");
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(b->main, &cap);
  if (cap != cudaStreamCaptureStatusNone) return enqueue_update(b, upload_frames != 0);  // inside the caller's own capture
  const int up = upload_frames != 0;
  if (b->dirty) drop_graphs(b), b->dirty = false;
  if (!b->exec[up]) {
    // first bring every world to its steady shape outside the capture (directory binding, list growth, per-handle
    // attribute setup happen at the first enqueue and are not capturable)
    int rc = enqueue_update(b, up != 0);
    if (rc != KS_OK) return rc;
    KS_CUDA(cudaStreamSynchronize(b->main));
    const int64_t before = g_kernel_launches.load();
    cudaGraph_t graph = nullptr;
    KS_CUDA(cudaStreamBeginCapture(b->main, cudaStreamCaptureModeThreadLocal));
    rc = enqueue_update(b, up != 0);
    const cudaError_t end = cudaStreamEndCapture(b->main, &graph);
    if (rc != KS_OK || end != cudaSuccess || !graph) {
      if (graph) cudaGraphDestroy(graph);
      cudaGetLastError();
      return rc != KS_OK ? rc : cuda_fail(end, "batch capture");
    }
    b->exec_nodes[up] = g_kernel_launches.load() - before;
    const cudaError_t inst = cudaGraphInstantiate(&b->exec[up], graph, 0);
    cudaGraphDestroy(graph);
    if (inst != cudaSuccess) {
      b->exec[up] = nullptr;
      return cuda_fail(inst, "batch graph instantiate");
    }
    return KS_OK;  // the warm-up enqueue above was this call's update
  }
  KS_CUDA(cudaGraphLaunch(b->exec[up], b->main));
  g_kernel_launches.fetch_add(b->exec_nodes[up], std::memory_order_relaxed);
  return KS_OK;
}

int64_t ks_batch_graph_kernels(const ks_batch* b) { return !b ? 0 : b->exec[0] ? b->exec_nodes[0] : b->exec[1] ? b->exec_nodes[1] : 0; }

int ks_batch_sync(ks_batch* b, ks_tsdf_report* reports, ks_esdf_report* esdf_reports, double* summaries_host) {
  if (!b) return fail(KS_ERR_INVALID, "null batch");
  // every environment's control blocks are requested first (each on its own lane), then the lanes are waited for once:
  // one round trip for the whole batch instead of two per environment
  if (b->lanes > 1) {  // a replayed update ran on the batch stream: the lanes' copies must come after it
    KS_CUDA(cudaEventRecord(b->fork, b->main));
    for (int l = 1; l < b->lanes; ++l) KS_CUDA(cudaStreamWaitEvent(b->lane[l], b->fork, 0));
  }
  for (int i = 0; i < b->n; ++i) {
    int rc = tsdf_report_enqueue(b->tsdf[i]);
    if (rc == KS_OK) rc = esdf_report_enqueue(b->esdf[i]);
    if (rc != KS_OK) return rc;
  }
  for (cudaStream_t lane : b->lane) KS_CUDA(cudaStreamSynchronize(lane));
  int first = KS_OK;
  std::string why;
  for (int i = 0; i < b->n; ++i) {
    ks_tsdf_report r;
    ks_esdf_report er;
    int rc = tsdf_report_collect(b->tsdf[i], &r);
    if (rc != KS_OK && first == KS_OK) first = rc, why = "environment " + std::to_string(b->first_env + i) + ": " + ks_last_error();
    rc = esdf_report_collect(b->esdf[i], &er);
    if (rc != KS_OK && first == KS_OK) first = rc, why = "environment " + std::to_string(b->first_env + i) + ": " + ks_last_error();
    if (reports) reports[i] = r;
    if (esdf_reports) esdf_reports[i] = er;
  }
  if (summaries_host) KS_CUDA(cudaMemcpy(summaries_host, b->summary_dev, sizeof(double) * 4 * b->n, cudaMemcpyDeviceToHost));
  if (first != KS_OK) return fail(first, why);
  return KS_OK;
}

double* ks_batch_summary_device(ks_batch* b) { return b ? b->summary_dev : nullptr; }
double* ks_batch_gathered_device(ks_batch* b) { return b ? b->gathered_dev : nullptr; }
int32_t ks_batch_gathered_rows(const ks_batch* b) { return b ? b->world * b->max_local : 0; }

int ks_batch_gathered(ks_batch* b, double* host_out) {
  if (!b || !host_out) return fail(KS_ERR_INVALID, "null argument");
  KS_CUDA(cudaStreamSynchronize(b->main));
  KS_CUDA(cudaMemcpy(host_out, b->gathered_dev, sizeof(double) * 4 * b->world * b->max_local, cudaMemcpyDeviceToHost));
  return KS_OK;
}

int ks_nccl_unique_id(void* out128) {
  if (!out128) return fail(KS_ERR_INVALID, "null argument");
  NcclApi& a = nccl();
  if (!a.lib) return fail(KS_ERR_UNSUPPORTED, a.why);
  const int rc = a.GetUniqueId(out128);
  return rc == 0 ? KS_OK : nccl_fail(rc, "ncclGetUniqueId");
}

static int attach(ks_batch* b, void* comm, bool own, int world, int rank, int max_local) {
  if (world < 1 || rank < 0 || rank >= world || max_local < b->n) return fail(KS_ERR_INVALID, "batch: bad communicator shape");
  KS_CUDA(cudaStreamSynchronize(b->main));
  // every rank contributes max_local rows (ranks with fewer environments pad with NaN rows), so the local buffer is regrown
  double* local = nullptr;
  double* all = nullptr;
  cudaError_t err = cudaMalloc(&local, sizeof(double) * 4 * max_local);
  if (err == cudaSuccess) err = cudaMemset(local, 0xFF, sizeof(double) * 4 * max_local);
  if (err == cudaSuccess) err = cudaMalloc(&all, sizeof(double) * 4 * max_local * world);
  if (err == cudaSuccess) err = cudaMemset(all, 0xFF, sizeof(double) * 4 * max_local * world);
  if (err != cudaSuccess) {
    cudaFree(local), cudaFree(all);
    return cuda_fail(err, "batch gather buffers");
  }
  if (b->gathered_dev && b->gathered_dev != b->summary_dev) cudaFree(b->gathered_dev);
  cudaFree(b->summary_dev);
  b->summary_dev = local, b->gathered_dev = all;
  b->comm = comm, b->own_comm = own, b->world = world, b->rank = rank, b->max_local = max_local;
  b->dirty = true;
  return KS_OK;
}

int ks_batch_attach_nccl_comm(ks_batch* b, void* nccl_comm, int32_t world, int32_t rank, int32_t max_local_envs) {
  if (!b || !nccl_comm) return fail(KS_ERR_INVALID, "null argument");
  NcclApi& a = nccl();
  if (!a.lib) return fail(KS_ERR_UNSUPPORTED, a.why);
  return attach(b, nccl_comm, false, world, rank, max_local_envs);
}

int ks_batch_attach_nccl(ks_batch* b, const void* unique_id128, int32_t world, int32_t rank, int32_t max_local_envs) {
  if (!b || !unique_id128) return fail(KS_ERR_INVALID, "null argument");
  NcclApi& a = nccl();
  if (!a.lib) return fail(KS_ERR_UNSUPPORTED, a.why);
  UniqueId id;
  std::memcpy(id.bytes, unique_id128, sizeof id.bytes);
  void* comm = nullptr;
  const int rc = a.CommInitRank(&comm, world, id, rank);
  if (rc != 0) return nccl_fail(rc, "ncclCommInitRank");
  const int arc = attach(b, comm, true, world, rank, max_local_envs);
  if (arc != KS_OK) a.CommDestroy(comm);
  return arc;
}

}  // extern "C"
