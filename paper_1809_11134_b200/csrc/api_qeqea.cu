// C ABI of the QEQEA engine handle (QeqeaEngine, engine.py:266-384).
#include <cstring>
#include <string>
#include <vector>

#include "qeqea_internal.h"

namespace isq {

struct QeqeaHandle {
  QeqeaArgs a;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int rank = 0, world = 1;
  int64_t shard = 0;  // circuits per rank (padded)
  int max_batch = 0;
  GenRecord* h_records = nullptr;  // pinned
  QeqeaDevState* h_state = nullptr;  // pinned
  GenGraph graph;                    // isq_qeqea_step on small populations
  int launch_mode = ISQ_LAUNCH_AUTO;
  PeerTable* d_peers = nullptr;      // peer transport table (device)
  std::vector<void*> ipc_opened;     // peer buffers mapped by isq_qeqea_ipc_open
};

static void close_peers(QeqeaHandle* h) {
  for (void* p : h->ipc_opened) cudaIpcCloseMemHandle(p);
  h->ipc_opened.clear();
  cudaFree(h->d_peers);
  h->d_peers = nullptr;
  h->a.peers = nullptr;
}

static void free_handle(QeqeaHandle* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  QeqeaArgs& a = h->a;
  const bool sharded = a.world > 1;
  void* bufs[] = {a.rot, a.inter, a.qlive, a.fitness, a.flats, a.gate_codes, a.gate_thetas,
                  a.touch_fbefore, a.touch_mutated, a.st, a.records, a.best_codes, a.best_thetas,
                  (void*)a.target, a.part_max, a.part_sum, a.part_arg, a.send_flats, a.recv_codes,
                  a.recv_thetas, a.elite};
  for (void* b : bufs) cudaFree(b);
  if (sharded) {  // world 1: the owner-side arrays alias the circuit-side ones
    cudaFree(a.owner_flats);
    cudaFree(a.owner_codes);
    cudaFree(a.owner_thetas);
  }
  h->graph.reset();
  close_peers(h);
  if (h->h_records) cudaFreeHost(h->h_records);
  if (h->h_state) cudaFreeHost(h->h_state);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

static isq_status validate(const isq_qeqea_config* c) {
  auto bad = [](const std::string& m) {
    set_error(m);
    return ISQ_ERR_CONFIG;
  };
  if (c->number_of_wires < 2) return bad("numberOfWires must be ≥ 2");
  if (c->size_of_individual < 1 || c->size_of_population < 1)
    return bad("sizeOfIndividual and sizeOfPopulation must be ≥ 1");
  if (!(c->probability_of_mutation >= 0.0 && c->probability_of_mutation <= 1.0))
    return bad("probabilityOfMutation must be in [0, 1]");
  if (!(c->mutation_range > 0.0)) return bad("mutationRange must be > 0");
  if (c->n_meas < 1) return bad("nMeas must be ≥ 1");
  if (c->max_generations < 1) return bad("maxGenerations must be ≥ 1");
  if (!(c->target_fitness > 0.0 && c->target_fitness <= 1.0))
    return bad("targetFitness must be in (0, 1]");
  if (c->number_of_wires > ISQ_MAX_WIRES) {
    set_error("numberOfWires=" + std::to_string(c->number_of_wires) +
              " exceeds the device kernels (2..13 wires, the reference's default 4^n <= 2^26 cap)");
    return ISQ_ERR_UNSUPPORTED;
  }
  if (c->size_of_individual > 4096) {
    set_error("sizeOfIndividual > 4096 is not supported by the device engine");
    return ISQ_ERR_UNSUPPORTED;
  }
  const int64_t n = c->number_of_wires;
  const int64_t K = n + n * (n - 1) / 2;
  const int64_t Q = K * c->size_of_population * c->size_of_individual;
  if (Q >= (1LL << 32) - 1) {
    set_error("qubit_count = K*P*L must stay below 2^32 for the device engine");
    return ISQ_ERR_UNSUPPORTED;
  }
  if (c->world < 1 || c->rank < 0 || c->rank >= c->world) return bad("invalid rank/world");
  if (c->world > kMaxWorld) return bad("world exceeds " + std::to_string(kMaxWorld) + " ranks");
  if (c->precision != ISQ_PRECISION_FP64 && c->precision != ISQ_PRECISION_FP32)
    return bad("precision must be ISQ_PRECISION_FP64 or ISQ_PRECISION_FP32");
  if (c->world > c->size_of_individual)
    return bad("population sharding needs sizeOfIndividual >= world (each rank owns positions)");
  return ISQ_OK;
}

#define TRYA(expr)                                                   \
  do {                                                               \
    cudaError_t _e = (expr);                                         \
    if (_e != cudaSuccess) {                                         \
      set_error(std::string(#expr) + ": " + cudaGetErrorString(_e)); \
      free_handle(h);                                                \
      return ISQ_ERR_CUDA;                                           \
    }                                                                \
  } while (0)

static isq_status null_handle() {
  set_error("null engine handle");
  return ISQ_ERR_CONFIG;
}

}  // namespace isq

using namespace isq;

extern "C" {

isq_status isq_qeqea_create(const isq_qeqea_config* cfg, const double* target, int32_t device,
                            int32_t max_batch, void** out) {
  *out = nullptr;
  isq_status st = validate(cfg);
  if (st != ISQ_OK) return st;
  QeqeaHandle* h = new QeqeaHandle();
  h->device = device;
  h->rank = cfg->rank;
  h->world = cfg->world;
  h->max_batch = max_batch < 1 ? 1 : max_batch;
  QeqeaArgs& a = h->a;
  std::memset(&a, 0, sizeof(a));
  a.n = cfg->number_of_wires;
  a.L = cfg->size_of_individual;
  a.P = cfg->size_of_population;
  a.K = a.n + a.n * (a.n - 1) / 2;
  a.Q = a.K * a.P * a.L;
  a.Qt = (int64_t)a.n * a.P * a.L;
  a.p_mut = cfg->probability_of_mutation;
  a.mutation_range = cfg->mutation_range;
  a.target_fitness = cfg->target_fitness;
  a.n_meas = cfg->n_meas;
  a.max_generations = (uint64_t)cfg->max_generations;
  a.seed = cfg->seed;
  a.precision = cfg->precision;
  a.rec_cap = h->max_batch;
  h->shard = (a.P + h->world - 1) / h->world;
  // sharding (engine_common.cuh QeqeaArgs): circuits [c0, c0 + S), positions [p_lo, p_lo + Lr)
  a.world = h->world;
  a.rank = h->rank;
  a.S = h->shard;
  a.c0 = (int64_t)h->rank * a.S;
  for (int o = 0; o <= a.world; ++o) a.p_bounds[o] = (int)((int64_t)o * a.L / a.world);
  a.p_lo = a.p_bounds[a.rank];
  a.Lr = a.p_bounds[a.rank + 1] - a.p_lo;
  a.div_L.init((uint32_t)a.L);
  a.div_LP.init((uint32_t)(a.L * a.P));
  a.div_Lr.init((uint32_t)(a.Lr > 0 ? a.Lr : 1));
  a.div_S.init((uint32_t)a.S);
  a.Qloc = a.K * a.P * a.Lr;
  a.Qtloc = (int64_t)a.n * a.P * a.Lr;
  a.elite_len = 2 + a.L + (a.L + 7) / 8;
  const int64_t D = 1LL << a.n;
  const int64_t nc = a.S * a.L;                  // circuit-side touches
  const int64_t no = (int64_t)a.world * a.S * a.Lr;  // owner-side touches
  TRYA(cudaSetDevice(device));
  {  // the bank and the per-touch arrays must fit: a clear error instead of a failed allocation
    const double need = (double)a.Qtloc * sizeof(RotRec) + (double)(a.Qloc - a.Qtloc) * sizeof(IntRec) +
                        (double)nc * (4 + 1 + 8) + (double)no * (8 + 1 + 48) +
                        (a.world > 1 ? (double)no * 13 + (double)nc * 13 : 0.0) + (double)D * D * 16;
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess && need > (double)free_b) {
      set_error("this configuration needs " + std::to_string((int64_t)(need / 1e9)) + " GB of device memory, " +
                std::to_string((int64_t)(free_b / 1000000000ull)) + " GB are free (shard it over more GPUs)");
      free_handle(h);
      return ISQ_ERR_UNSUPPORTED;
    }
  }
  if (qeqea_configure_device() != ISQ_OK) {
    free_handle(h);
    return ISQ_ERR_CUDA;
  }
  TRYA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  h->own_stream = true;
  TRYA(cudaMalloc((void**)&a.rot, a.Qtloc * sizeof(RotRec)));
  TRYA(cudaMalloc((void**)&a.inter, (a.Qloc - a.Qtloc) * sizeof(IntRec)));
  TRYA(cudaMalloc((void**)&a.fitness, a.S * a.world * 8));
  TRYA(cudaMalloc((void**)&a.flats, nc * 4));
  TRYA(cudaMalloc((void**)&a.gate_codes, nc));
  TRYA(cudaMalloc((void**)&a.gate_thetas, nc * 8));
  TRYA(cudaMalloc((void**)&a.touch_fbefore, no * 8));
  TRYA(cudaMalloc((void**)&a.touch_mutated, no));
  TRYA(cudaMalloc((void**)&a.qlive, no * 48));
  if (a.world > 1) {
    TRYA(cudaMalloc((void**)&a.owner_flats, no * 4));
    TRYA(cudaMalloc((void**)&a.owner_codes, no));
    TRYA(cudaMalloc((void**)&a.owner_thetas, no * 8));
    TRYA(cudaMalloc((void**)&a.send_flats, nc * 4));
    TRYA(cudaMalloc((void**)&a.recv_codes, nc));
    TRYA(cudaMalloc((void**)&a.recv_thetas, nc * 8));
    TRYA(cudaMalloc((void**)&a.elite, (int64_t)a.world * a.elite_len * 8));
  } else {
    a.owner_flats = a.flats;
    a.owner_codes = a.gate_codes;
    a.owner_thetas = a.gate_thetas;
  }
  TRYA(cudaMalloc((void**)&a.st, sizeof(QeqeaDevState)));
  TRYA(cudaMalloc((void**)&a.records, sizeof(GenRecord) * h->max_batch));
  TRYA(cudaMalloc((void**)&a.best_codes, a.L));
  TRYA(cudaMalloc((void**)&a.best_thetas, a.L * 8));
  TRYA(cudaMalloc((void**)&a.target, D * D * 16));
  a.n_parts = (int)((a.P + 4095) / 4096);
  if (a.n_parts > 1024) a.n_parts = 1024;
  if (a.n_parts < 1) a.n_parts = 1;
  TRYA(cudaMalloc((void**)&a.part_max, a.n_parts * 8));
  TRYA(cudaMalloc((void**)&a.part_sum, a.n_parts * 8));
  TRYA(cudaMalloc((void**)&a.part_arg, a.n_parts * 8));
  TRYA(cudaMallocHost((void**)&h->h_records, sizeof(GenRecord) * h->max_batch));
  TRYA(cudaMallocHost((void**)&h->h_state, sizeof(QeqeaDevState)));
  TRYA(cudaMemcpyAsync((void*)a.target, target, D * D * 16, cudaMemcpyHostToDevice, h->stream));
  QeqeaDevState s0;
  std::memset(&s0, 0, sizeof(s0));
  s0.best_circuit = -1;
  *h->h_state = s0;
  TRYA(cudaMemcpyAsync(a.st, h->h_state, sizeof(s0), cudaMemcpyHostToDevice, h->stream));
  TRYA(cudaMemsetAsync(a.best_codes, 0, a.L, h->stream));
  TRYA(cudaMemsetAsync(a.best_thetas, 0, a.L * 8, h->stream));
  TRYA(cudaMemsetAsync(a.fitness, 0, h->shard * h->world * 8, h->stream));
  if (qeqea_launch_init(a, h->stream) != ISQ_OK) {
    free_handle(h);
    return ISQ_ERR_CUDA;
  }
  TRYA(cudaStreamSynchronize(h->stream));
  *out = h;
  return ISQ_OK;
}

isq_status isq_qeqea_destroy(void* handle) {
  free_handle(static_cast<QeqeaHandle*>(handle));
  return ISQ_OK;
}

isq_status isq_qeqea_set_stream(void* handle, void* stream) {
  QeqeaHandle* h = static_cast<QeqeaHandle*>(handle);
  if (!h) return null_handle();
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  ISQ_CUDA_TRY(cudaStreamSynchronize(h->stream));
  if (h->own_stream) cudaStreamDestroy(h->stream);
  h->own_stream = false;
  h->stream = (cudaStream_t)stream;
  return ISQ_OK;
}

isq_status isq_qeqea_begin_batch(void* handle) {
  QeqeaHandle* h = static_cast<QeqeaHandle*>(handle);
  if (!h) return null_handle();
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  // rec_base := generation (device-side copy, stream ordered)
  ISQ_CUDA_TRY(cudaMemcpyAsync(&h->a.st->rec_base, &h->a.st->generation, 8,
                               cudaMemcpyDeviceToDevice, h->stream));
  return ISQ_OK;
}

static isq_status need_world1(const QeqeaHandle* h, const char* what) {
  if (h->world == 1) return ISQ_OK;
  set_error(std::string(what) + " drives a single rank; at world > 1 use prepare / values / score / finish");
  return ISQ_ERR_CONFIG;
}

isq_status isq_qeqea_eval(void* handle) {
  QeqeaHandle* h = static_cast<QeqeaHandle*>(handle);
  if (!h) return null_handle();
  isq_status st = need_world1(h, "isq_qeqea_eval");
  if (st != ISQ_OK) return st;
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  return qeqea_launch_eval(h->a, h->stream);
}

isq_status isq_qeqea_prepare(void* handle) {
  QeqeaHandle* h = static_cast<QeqeaHandle*>(handle);
  if (!h) return null_handle();
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  return qeqea_launch_prepare(h->a, h->stream);
}

isq_status isq_qeqea_values(void* handle) {
  QeqeaHandle* h = static_cast<QeqeaHandle*>(handle);
  if (!h) return null_handle();
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  return qeqea_launch_values(h->a, h->stream);
}

isq_status isq_qeqea_score(void* handle) {
  QeqeaHandle* h = static_cast<QeqeaHandle*>(handle);
  if (!h) return null_handle();
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  return qeqea_launch_score(h->a, h->stream);
}

isq_status isq_qeqea_finish(void* handle) {
  QeqeaHandle* h = static_cast<QeqeaHandle*>(handle);
  if (!h) return null_handle();
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  return qeqea_launch_finish(h->a, h->stream);
}

isq_status isq_qeqea_set_peers(void* handle, const isq_qeqea_peer_buffers* peers) {
  QeqeaHandle* h = static_cast<QeqeaHandle*>(handle);
  if (!h) return null_handle();
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  ISQ_CUDA_TRY(cudaStreamSynchronize(h->stream));
  if (peers == nullptr) {
    close_peers(h);
    return ISQ_OK;
  }
  if (h->world < 2) {
    set_error("the peer transport needs world > 1");
    return ISQ_ERR_CONFIG;
  }
  PeerTable t;
  std::memset(&t, 0, sizeof(t));
  for (int r = 0; r < h->world; ++r) {
    const isq_qeqea_peer_buffers& b = peers[r];
    if (!b.recv_flats || !b.recv_codes || !b.recv_thetas || !b.fitness || !b.elite) {
      set_error("peer buffers of rank " + std::to_string(r) + " incomplete");
      return ISQ_ERR_CONFIG;
    }
    t.recv_flats[r] = static_cast<uint32_t*>(b.recv_flats);
    t.recv_codes[r] = static_cast<uint8_t*>(b.recv_codes);
    t.recv_thetas[r] = static_cast<double*>(b.recv_thetas);
    t.fitness[r] = static_cast<double*>(b.fitness);
    t.elite[r] = static_cast<double*>(b.elite);
  }
  if (t.recv_flats[h->rank] != h->a.owner_flats || t.fitness[h->rank] != h->a.fitness) {
    set_error("peers[rank] must be this handle's own exchange buffers");
    return ISQ_ERR_CONFIG;
  }
  if (!h->d_peers) ISQ_CUDA_TRY(cudaMalloc((void**)&h->d_peers, sizeof(PeerTable)));
  ISQ_CUDA_TRY(cudaMemcpy(h->d_peers, &t, sizeof(t), cudaMemcpyHostToDevice));
  h->a.peers = h->d_peers;
  return ISQ_OK;
}

isq_status isq_qeqea_ipc_export(void* handle, isq_ipc_handle* out) {
  QeqeaHandle* h = static_cast<QeqeaHandle*>(handle);
  if (!h) return null_handle();
  const QeqeaArgs& a = h->a;
  if (h->world < 2) {
    set_error("the peer transport needs world > 1");
    return ISQ_ERR_CONFIG;
  }
  static_assert(sizeof(cudaIpcMemHandle_t) == sizeof(isq_ipc_handle), "IPC handle size");
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  void* bufs[ISQ_PEER_BUFFERS] = {a.owner_flats, a.recv_codes, a.recv_thetas, a.fitness, a.elite};
  for (int k = 0; k < ISQ_PEER_BUFFERS; ++k) {
    cudaIpcMemHandle_t m;
    ISQ_CUDA_TRY(cudaIpcGetMemHandle(&m, bufs[k]));
    std::memcpy(&out[k], &m, sizeof(m));
  }
  return ISQ_OK;
}

isq_status isq_qeqea_ipc_open(void* handle, const isq_ipc_handle* all) {
  QeqeaHandle* h = static_cast<QeqeaHandle*>(handle);
  if (!h) return null_handle();
  const QeqeaArgs& a = h->a;
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  close_peers(h);
  std::vector<isq_qeqea_peer_buffers> peers(h->world);
  for (int r = 0; r < h->world; ++r) {
    void* p[ISQ_PEER_BUFFERS];
    if (r == h->rank) {
      p[0] = a.owner_flats;
      p[1] = a.recv_codes;
      p[2] = a.recv_thetas;
      p[3] = a.fitness;
      p[4] = a.elite;
    } else {
      for (int k = 0; k < ISQ_PEER_BUFFERS; ++k) {
        cudaIpcMemHandle_t m;
        std::memcpy(&m, &all[r * ISQ_PEER_BUFFERS + k], sizeof(m));
        cudaError_t e = cudaIpcOpenMemHandle(&p[k], m, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
          set_error(std::string("cudaIpcOpenMemHandle (rank ") + std::to_string(r) + "): " +
                    cudaGetErrorString(e));
          close_peers(h);
          return ISQ_ERR_CUDA;
        }
        h->ipc_opened.push_back(p[k]);
      }
    }
    peers[r] = isq_qeqea_peer_buffers{p[0], p[1], p[2], p[3], p[4]};
  }
  return isq_qeqea_set_peers(handle, peers.data());
}

isq_status isq_qeqea_exchange(void* handle, isq_qeqea_exchange_buffers* x) {
  QeqeaHandle* h = static_cast<QeqeaHandle*>(handle);
  if (!h) return null_handle();
  const QeqeaArgs& a = h->a;
  std::memset(x, 0, sizeof(*x));
  x->world = a.world;
  x->rank = a.rank;
  x->shard = a.S;
  x->elite_len = a.elite_len;
  for (int o = 0; o <= a.world; ++o) x->position_bounds[o] = a.p_bounds[o];
  x->send_flats = a.send_flats;
  x->recv_flats = a.world > 1 ? a.owner_flats : nullptr;
  x->send_codes = a.world > 1 ? a.owner_codes : nullptr;
  x->recv_codes = a.recv_codes;
  x->send_thetas = a.world > 1 ? a.owner_thetas : nullptr;
  x->recv_thetas = a.recv_thetas;
  x->fitness = a.fitness;
  x->elite = a.elite;
  x->stream = h->stream;
  return ISQ_OK;
}

isq_status isq_qeqea_read_batch(void* handle, isq_generation_record* records, int32_t* n_done,
                                int32_t* stop_reason, uint64_t* generation, double* best_fitness) {
  QeqeaHandle* h = static_cast<QeqeaHandle*>(handle);
  if (!h) return null_handle();
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  ISQ_CUDA_TRY(cudaMemcpyAsync(h->h_state, h->a.st, sizeof(QeqeaDevState), cudaMemcpyDeviceToHost,
                               h->stream));
  ISQ_CUDA_TRY(cudaStreamSynchronize(h->stream));
  const QeqeaDevState s = *h->h_state;
  int64_t done = (int64_t)(s.generation - s.rec_base);
  if (done > h->max_batch) done = h->max_batch;
  if (done > 0 && records) {
    ISQ_CUDA_TRY(cudaMemcpy(h->h_records, h->a.records, sizeof(GenRecord) * done,
                            cudaMemcpyDeviceToHost));
    std::memcpy(records, h->h_records, sizeof(GenRecord) * done);
  }
  if (n_done) *n_done = (int32_t)done;
  if (stop_reason) *stop_reason = s.stop;
  if (generation) *generation = s.generation;
  if (best_fitness) *best_fitness = s.best_fitness;
  return ISQ_OK;
}

isq_status isq_qeqea_step(void* handle, int32_t n_generations, isq_generation_record* records,
                          int32_t* n_done, int32_t* stop_reason) {
  QeqeaHandle* h = static_cast<QeqeaHandle*>(handle);
  if (!h) return null_handle();
  isq_status st0 = need_world1(h, "isq_qeqea_step");
  if (st0 != ISQ_OK) return st0;
  if (n_generations > h->max_batch) {
    set_error("n_generations exceeds the handle's record capacity (max_batch)");
    return ISQ_ERR_CONFIG;
  }
  isq_status st = isq_qeqea_begin_batch(handle);
  if (st != ISQ_OK) return st;
  const QeqeaArgs& a = h->a;
  const int mode = h->launch_mode;
  if (mode == ISQ_LAUNCH_FUSED || (mode == ISQ_LAUNCH_AUTO && qeqea_small(a))) {
    st = n_generations > 0 ? qeqea_launch_small(a, n_generations, h->stream) : ISQ_OK;
    if (st != ISQ_OK) return st;
    return isq_qeqea_read_batch(handle, records, n_done, stop_reason, nullptr, nullptr);
  }
  // n > 5 runs the generic fitness kernel, whose scratch is allocated on
  // first use: plain launches only (a capture would record the allocation)
  const int per_graph = (mode == ISQ_LAUNCH_KERNELS || a.n > ISQ_MAX_FAST_WIRES) ? 0
                        : mode == ISQ_LAUNCH_GRAPH                              ? 16
                                                                                : graph_generations(a.P * a.L);
  st = run_generations(h->graph, h->stream, n_generations, per_graph,
                       [&a](cudaStream_t s) {
                         isq_status r = qeqea_launch_eval(a, s);
                         return r != ISQ_OK ? r : qeqea_launch_finish(a, s);
                       });
  if (st != ISQ_OK) return st;
  return isq_qeqea_read_batch(handle, records, n_done, stop_reason, nullptr, nullptr);
}

isq_status isq_qeqea_set_launch_mode(void* handle, int32_t mode) {
  QeqeaHandle* h = static_cast<QeqeaHandle*>(handle);
  if (!h) return null_handle();
  if (mode < ISQ_LAUNCH_AUTO || mode > ISQ_LAUNCH_FUSED) {
    set_error("unknown launch mode");
    return ISQ_ERR_CONFIG;
  }
  h->launch_mode = mode;
  return ISQ_OK;
}

isq_status isq_qeqea_set_limits(void* handle, int64_t max_generations, double target_fitness,
                                int32_t stop) {
  QeqeaHandle* h = static_cast<QeqeaHandle*>(handle);
  if (!h) return null_handle();
  if (max_generations < 1) {
    set_error("maxGenerations must be ≥ 1");
    return ISQ_ERR_CONFIG;
  }
  if (!(target_fitness > 0.0 && target_fitness <= 1.0)) {
    set_error("targetFitness must be in (0, 1]");
    return ISQ_ERR_CONFIG;
  }
  if (stop < 0 || stop > 2) {
    set_error("stop must be 0 (running), 1 (target-reached) or 2 (generation-limit)");
    return ISQ_ERR_CONFIG;
  }
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  ISQ_CUDA_TRY(cudaStreamSynchronize(h->stream));
  h->a.max_generations = (uint64_t)max_generations;
  h->a.target_fitness = target_fitness;
  h->graph.reset();  // captured launches carry the old limits by value
  ISQ_CUDA_TRY(cudaMemcpy(&h->a.st->stop, &stop, sizeof(stop), cudaMemcpyHostToDevice));
  return ISQ_OK;
}

isq_status isq_qeqea_buffers(void* handle, void** fitness_dev, int64_t* shard_len,
                             void** stream) {
  QeqeaHandle* h = static_cast<QeqeaHandle*>(handle);
  if (!h) return null_handle();
  if (fitness_dev) *fitness_dev = h->a.fitness;
  if (shard_len) *shard_len = h->shard;
  if (stream) *stream = h->stream;
  return ISQ_OK;
}

isq_status isq_qeqea_best(void* handle, uint8_t* codes, double* thetas, double* fitness) {
  QeqeaHandle* h = static_cast<QeqeaHandle*>(handle);
  if (!h) return null_handle();
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  ISQ_CUDA_TRY(cudaStreamSynchronize(h->stream));
  ISQ_CUDA_TRY(cudaMemcpy(codes, h->a.best_codes, h->a.L, cudaMemcpyDeviceToHost));
  ISQ_CUDA_TRY(cudaMemcpy(thetas, h->a.best_thetas, h->a.L * 8, cudaMemcpyDeviceToHost));
  QeqeaDevState s;
  ISQ_CUDA_TRY(cudaMemcpy(&s, h->a.st, sizeof(s), cudaMemcpyDeviceToHost));
  *fitness = s.best_fitness;
  return ISQ_OK;
}

// Device temporaries for the reference's array layout.
struct SoaTemps {
  double *theta = nullptr, *qamp = nullptr, *smax = nullptr;
  ~SoaTemps() {
    cudaFree(theta);
    cudaFree(qamp);
    cudaFree(smax);
  }
  cudaError_t alloc(const QeqeaArgs& a) {
    cudaError_t e = cudaMalloc((void**)&theta, a.Qloc * 8);
    if (e == cudaSuccess) e = cudaMalloc((void**)&qamp, a.Qtloc * 48 + 16);
    if (e == cudaSuccess) e = cudaMalloc((void**)&smax, a.Qloc * 8);
    return e;
  }
};

isq_status isq_qeqea_get_state(void* handle, double* theta, double* qamp, double* slot_max,
                               uint64_t* generation, double* best_fitness, int32_t* stop) {
  QeqeaHandle* h = static_cast<QeqeaHandle*>(handle);
  if (!h) return null_handle();
  const QeqeaArgs& a = h->a;
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  ISQ_CUDA_TRY(cudaStreamSynchronize(h->stream));
  if (theta || qamp || slot_max) {
    SoaTemps t;
    ISQ_CUDA_TRY(t.alloc(a));
    isq_status st = qeqea_launch_pack(a, t.theta, t.qamp, t.smax, h->stream);
    if (st != ISQ_OK) return st;
    ISQ_CUDA_TRY(cudaStreamSynchronize(h->stream));
    if (theta) ISQ_CUDA_TRY(cudaMemcpy(theta, t.theta, a.Qloc * 8, cudaMemcpyDeviceToHost));
    if (qamp) ISQ_CUDA_TRY(cudaMemcpy(qamp, t.qamp, a.Qtloc * 48, cudaMemcpyDeviceToHost));
    if (slot_max) ISQ_CUDA_TRY(cudaMemcpy(slot_max, t.smax, a.Qloc * 8, cudaMemcpyDeviceToHost));
  }
  QeqeaDevState s;
  ISQ_CUDA_TRY(cudaMemcpy(&s, a.st, sizeof(s), cudaMemcpyDeviceToHost));
  if (generation) *generation = s.generation;
  if (best_fitness) *best_fitness = s.best_fitness;
  if (stop) *stop = s.stop;
  return ISQ_OK;
}

isq_status isq_qeqea_set_state(void* handle, const double* theta, const double* qamp,
                               const double* slot_max, uint64_t generation, double best_fitness,
                               int32_t stop, const uint8_t* best_codes, const double* best_thetas) {
  QeqeaHandle* h = static_cast<QeqeaHandle*>(handle);
  if (!h) return null_handle();
  const QeqeaArgs& a = h->a;
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  ISQ_CUDA_TRY(cudaStreamSynchronize(h->stream));
  if (theta && qamp) {
    SoaTemps t;
    ISQ_CUDA_TRY(t.alloc(a));
    ISQ_CUDA_TRY(cudaMemcpy(t.theta, theta, a.Qloc * 8, cudaMemcpyHostToDevice));
    ISQ_CUDA_TRY(cudaMemcpy(t.qamp, qamp, a.Qtloc * 48, cudaMemcpyHostToDevice));
    if (slot_max) ISQ_CUDA_TRY(cudaMemcpy(t.smax, slot_max, a.Qloc * 8, cudaMemcpyHostToDevice));
    isq_status st = qeqea_launch_unpack(a, t.theta, t.qamp, slot_max ? t.smax : nullptr, h->stream);
    if (st != ISQ_OK) return st;
    ISQ_CUDA_TRY(cudaStreamSynchronize(h->stream));
  } else if (theta || qamp || slot_max) {
    set_error("set_state needs both theta and qamp");
    return ISQ_ERR_CONFIG;
  }
  if (best_codes) ISQ_CUDA_TRY(cudaMemcpy(a.best_codes, best_codes, a.L, cudaMemcpyHostToDevice));
  if (best_thetas)
    ISQ_CUDA_TRY(cudaMemcpy(a.best_thetas, best_thetas, a.L * 8, cudaMemcpyHostToDevice));
  QeqeaDevState s;
  std::memset(&s, 0, sizeof(s));
  s.generation = generation;
  s.rec_base = generation;
  s.best_fitness = best_fitness;
  s.best_circuit = -1;
  s.stop = stop;
  ISQ_CUDA_TRY(cudaMemcpy(a.st, &s, sizeof(s), cudaMemcpyHostToDevice));
  return ISQ_OK;
}

isq_status isq_qeqea_live_population(void* handle, double* theta, double* qutrits) {
  QeqeaHandle* h = static_cast<QeqeaHandle*>(handle);
  if (!h) return null_handle();
  const QeqeaArgs& a = h->a;
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  double *d_t = nullptr, *d_q = nullptr;
  ISQ_CUDA_TRY(cudaMalloc((void**)&d_t, a.Qloc * 8));
  cudaError_t e = cudaMalloc((void**)&d_q, a.Qtloc * 48 + 16);
  if (e != cudaSuccess) {
    cudaFree(d_t);
    set_error(std::string("cudaMalloc: ") + cudaGetErrorString(e));
    return ISQ_ERR_CUDA;
  }
  isq_status st = qeqea_launch_live(a, d_t, d_q, h->stream);
  if (st == ISQ_OK) {
    e = cudaStreamSynchronize(h->stream);
    if (e == cudaSuccess) e = cudaMemcpy(theta, d_t, a.Qloc * 8, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && qutrits) e = cudaMemcpy(qutrits, d_q, a.Qtloc * 48, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
      set_error(std::string("live population: ") + cudaGetErrorString(e));
      st = ISQ_ERR_CUDA;
    }
  }
  cudaFree(d_t);
  cudaFree(d_q);
  return st;
}

isq_status isq_qeqea_sample(void* handle, int64_t c0, int64_t c1, int64_t* flats, uint8_t* codes,
                            double* thetas) {
  QeqeaHandle* h = static_cast<QeqeaHandle*>(handle);
  if (!h) return null_handle();
  const QeqeaArgs& a = h->a;
  isq_status st0 = need_world1(h, "isq_qeqea_sample");
  if (st0 != ISQ_OK) return st0;
  if (c0 < 0 || c1 > a.P || c1 < c0) {
    set_error("circuit range out of bounds");
    return ISQ_ERR_CONFIG;
  }
  if (c1 == c0) return ISQ_OK;
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  const int64_t n = (c1 - c0) * a.L;
  int64_t* d_f = nullptr;
  uint8_t* d_c = nullptr;
  double* d_t = nullptr;
  ISQ_CUDA_TRY(cudaMalloc((void**)&d_f, n * 8));
  ISQ_CUDA_TRY(cudaMalloc((void**)&d_c, n));
  ISQ_CUDA_TRY(cudaMalloc((void**)&d_t, n * 8));
  isq_status st = qeqea_launch_sample(a, c0, c1, d_f, d_c, d_t, h->stream);
  cudaError_t e = cudaStreamSynchronize(h->stream);
  if (st == ISQ_OK && e == cudaSuccess) {
    cudaMemcpy(flats, d_f, n * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(codes, d_c, n, cudaMemcpyDeviceToHost);
    e = cudaMemcpy(thetas, d_t, n * 8, cudaMemcpyDeviceToHost);
  }
  cudaFree(d_f);
  cudaFree(d_c);
  cudaFree(d_t);
  if (st == ISQ_OK && e != cudaSuccess) {
    set_error(std::string("sample: ") + cudaGetErrorString(e));
    st = ISQ_ERR_CUDA;
  }
  return st;
}

isq_status isq_qeqea_fitness(void* handle, double* out) {
  QeqeaHandle* h = static_cast<QeqeaHandle*>(handle);
  if (!h) return null_handle();
  ISQ_CUDA_TRY(cudaSetDevice(h->device));
  ISQ_CUDA_TRY(cudaStreamSynchronize(h->stream));
  ISQ_CUDA_TRY(cudaMemcpy(out, h->a.fitness, h->a.P * 8, cudaMemcpyDeviceToHost));
  return ISQ_OK;
}

}  // extern "C"
