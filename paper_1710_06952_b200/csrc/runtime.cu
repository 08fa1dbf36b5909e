// runtime.cu -- host runtime behind the C ABI (include/adpsgd.h).
//
// Owns placement, device memory, CUDA IPC peer mapping over NVLink, the NCCL
// communicator, the host executor (stream-ordered replay / step / gossip) and
// the launch of the persistent engine.  No exception crosses the ABI.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include <nccl.h>
#include <nvtx3/nvToolsExt.h>
#include <unistd.h>

#include "../../include/adpsgd.h"
#include "comm.h"
#include "internal.h"

using namespace adp;

static_assert(sizeof(adpsgd_log_entry) == sizeof(LogEntry), "log entry layout");

namespace {

thread_local std::string g_err;

adpsgd_status fail(adpsgd_status s, const std::string& m) {
  g_err = m;
  return s;
}

#define CU(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess)                                                             \
      return fail(ADPSGD_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));     \
  } while (0)
#define NC(x)                                                                          \
  do {                                                                                 \
    ncclResult_t r_ = (x);                                                             \
    if (r_ != ncclSuccess)                                                             \
      return fail(ADPSGD_E_NCCL, std::string(#x) + ": " + ncclGetErrorString(r_));     \
  } while (0)
#define CO(x)                                                                          \
  do {                                                                                 \
    std::string m_;                                                                    \
    const int r_ = (x);                                                                \
    if (r_ != 0) return fail((adpsgd_status)r_, m_.empty() ? std::string(#x) : m_);    \
  } while (0)
#define ST(x)                                                                          \
  do {                                                                                 \
    adpsgd_status s_ = (x);                                                            \
    if (s_ != ADPSGD_OK) return s_;                                                    \
  } while (0)

constexpr uint32_t kBlobMagic = 0xADB5D200u;
constexpr int kPoolStreams = 8;     // replay DAG stream lanes
constexpr int kEventRing = 4096;    // recycled cudaEvents for the replay DAG

struct PeerBlob {
  uint32_t magic, version;
  int32_t rank, n_local;
  int64_t d_pad;
  int64_t gctl_offset, log_offset, log_cap, slots_offset;
  int32_t engine_grid, pad0;
  cudaIpcMemHandle_t models, ctl;
  // in-process ranks (cfg.comm_local): raw device addresses, valid in this process
  int32_t local, device;
  uint64_t pid, models_ptr, ctl_ptr;
};

uint64_t splitmix64(uint64_t& s) {
  uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

}  // namespace

struct adpsgd_ctx {
  // ---- configuration (owned copies) ----
  int rank = 0, world = 1, device = 0;
  int n = 0;
  long long d = 0, d_pad = 0, n4 = 0;
  adpsgd_model_kind model = ADPSGD_MODEL_NONE;
  float gamma = 0.f;
  int M = 1, T = 0;
  uint64_t seed = 0;
  QuadParams q{};
  long long compute_ns = 0;
  int engine_cps = 0, engine_threads = 512;
  int wait_free = 0;                 // App. A runtime for adpsgd_run (reading R20)
  int engine_fuse = 1;               // fuse due passive steps into pair passes
  int engine_coop = 0;               // cooperative cross-GPU events: 0 auto, 1 on, -1 off
  long long fuse_wait_ns = 0;        // how long a due passive stays absorbable
  std::vector<float> link;           // link slowdown per worker (reading R21)
  long long link_ns = 0;
  float link_max() const { return link.empty() ? 1.0f : *std::max_element(link.begin(), link.end()); }
  long long log_cap = 1 << 20;
  std::vector<int32_t> edges;
  std::vector<int8_t> role;
  std::vector<std::vector<int>> nb;
  std::vector<int> nb_flat, nb_off;
  std::vector<int> worker_rank, worker_local;
  std::vector<float> straggle;
  std::vector<int> local_ids;
  int n_local = 0;
  int S = 0, feat = 0;
  MlpShape mlp{0, 0, 0};
  // ---- device state ----
  cudaStream_t stream = nullptr;
  float* models = nullptr;
  char* ctl_arena = nullptr;
  size_t ctl_bytes = 0, gctl_offset = 0, log_offset = 0, slots_offset = 0;
  float* rrows = nullptr;            // engine replay stale reads: [n_local][T+1][d_pad] gradient rows
  int rrows_n = 0;
  std::vector<size_t> peer_slots_off;
  int engine_grid = 0;
  WorkerCtl* ctl = nullptr;
  GlobalCtl* gctl = nullptr;
  LogEntry* log = nullptr;           // rank 0 only (local)
  GlobalCtl* gctl0 = nullptr;        // rank 0's (local or peer)
  LogEntry* log0 = nullptr;
  std::vector<float*> peer_models;
  std::vector<char*> peer_ctl;
  std::vector<bool> peer_imported;
  WorkerDesc* d_workers = nullptr;
  int* d_nbrs = nullptr;
  int* d_local_ids = nullptr;
  Slot* d_slots = nullptr;
  ReplayEv* d_rev = nullptr;
  size_t rev_cap = 0;
  float* dx0 = nullptr;
  float *dA = nullptr, *db = nullptr;
  int* dy = nullptr;
  float* gslots = nullptr;
  unsigned char* lin_buf = nullptr;   // config-1 replay op list (k_lin_replay)
  size_t lin_cap = 0;
  int gslot_n = 0;
  float* gstep = nullptr;            // per-local-worker gradient buffers (adpsgd_step)
  float* wf_g = nullptr;             // App. A: [n_local][2][d_pad] gradient rows (wait_free)
  float* comp_row = nullptr;         // host replay: compensated pulled model (COMPENSATE events)
  float* mlp_scratch = nullptr;
  size_t mlp_scratch_n = 0;
  std::vector<MlpWork> mlp_work;     // one per replay stream lane
  std::vector<cudaStream_t> pool;    // replay DAG streams
  std::vector<cudaEvent_t> evring;
  size_t evnext = 0;
  int* d_batch = nullptr;
  size_t batch_cap = 0;
  double* sum64 = nullptr;
  double* mk_acc = nullptr;
  float *xr = nullptr, *gsum = nullptr;
  unsigned long long ar_k = 0;
  // D-PSGD baseline (double-buffered rows + halo of remote neighbour rows)
  float* dp_x[2] = {nullptr, nullptr};
  float* dp_halo = nullptr;
  const float** d_dp_nbr[2] = {nullptr, nullptr};
  int* d_dp_deg = nullptr;
  float* d_dp_wself = nullptr;
  float dp_wnb = 0.f;
  int dp_cur = 0;
  unsigned long long dp_k = 0;
  std::vector<int> dp_halo_w;                     // remote rows received each round (ascending id)
  std::vector<std::pair<int, int>> dp_send;       // (local worker, destination rank), ascending id
  Comm* comm = nullptr;              // NCCL (processes) or in-process (threads), comm.h
  bool comm_local = false;           // ranks are host threads of this process (cfg.comm_local)
  bool connected = false;
  // super-learner mode (reading R22): this rank's group communicator and buffers
  Comm* super_comm = nullptr;
  int super_R = 0;
  float* super_g = nullptr;                        // learner gradient, then the group's sum
  unsigned long long* super_k = nullptr;           // ticket broadcast by the group leader
  unsigned long long* k_host = nullptr;            // pinned: step_multi reads its ticket here
  int* super_bar = nullptr;                        // group barrier word
  long long super_c = 0;                           // gradient events of this rank's super-learner
  std::vector<std::vector<int>> super_nb;          // super-learner ring neighbours
  // ---- host executor state ----
  std::mutex mu;
  std::vector<cudaEvent_t> last_evt;
  std::vector<uint64_t> step_ctr;
  unsigned long long host_k = 0;
  bool ticket_dirty = false;         // multi-GPU adpsgd_step moved the device counter
  unsigned long long* agree64 = nullptr;   // ticket agreement scratch (collective calls, world > 1)
  std::vector<unsigned int> epochs;  // per-worker committed-replay-event counts (mirror)
  long long launches = 0;
  unsigned int run_counter = 0;
  std::vector<Slot> h_slots;
  std::vector<ReplayEv> h_rev;

  cudaStream_t use(adpsgd_stream s) const { return s ? (cudaStream_t)s : stream; }
  float* row(int w) const { return models + (long long)worker_local[w] * d_pad; }
  bool is_local(int w) const { return worker_rank[w] == rank; }
  uint2 seed2() const { return make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)); }
};

namespace {

// ------------------------------------------------------------ graph checks --
adpsgd_status check_graph(adpsgd_ctx* c, const adpsgd_graph* g) {
  const int n = g->n;
  if (n < 1 || g->n_edges < 0 || (g->n_edges > 0 && !g->edges))
    return fail(ADPSGD_E_INVALID, "graph: n < 1 or null edges");
  c->nb.assign(n, {});
  for (int e = 0; e < g->n_edges; ++e) {
    const int a = g->edges[2 * e], b = g->edges[2 * e + 1];
    if (a < 0 || a >= n || b < 0 || b >= n || a == b)
      return fail(ADPSGD_E_INVALID, "graph: edge out of range or self-loop (S:80)");
    if (std::find(c->nb[a].begin(), c->nb[a].end(), b) != c->nb[a].end())
      return fail(ADPSGD_E_INVALID, "graph: duplicate edge");
    c->nb[a].push_back(b);
    c->nb[b].push_back(a);
  }
  for (auto& v : c->nb) std::sort(v.begin(), v.end());
  // connectivity + 2-colouring (BFS per component, each started as active)
  std::vector<int> col(n, -1), q;
  bool bip = true;
  int comps = 0;
  for (int s0 = 0; s0 < n; ++s0) {
    if (col[s0] >= 0) continue;
    ++comps;
    col[s0] = 0;
    q.assign(1, s0);
    for (size_t h = 0; h < q.size(); ++h) {
      const int u = q[h];
      for (int w : c->nb[u]) {
        if (col[w] < 0) { col[w] = 1 - col[u]; q.push_back(w); }
        else if (col[w] == col[u]) bip = false;
      }
    }
  }
  if (c->super_R > 1) {
    // super-learner context (R22): the learners' graph is R copies of the
    // super-learners' graph; that contracted graph must be connected
    const int R = c->super_R;
    if (n % R) return fail(ADPSGD_E_INVALID, "super_R must divide n");
    const int S = n / R;
    std::vector<int> seen(S, 0), sq(1, 0);
    seen[0] = 1;
    for (size_t h = 0; h < sq.size(); ++h)
      for (int r = 0; r < R; ++r)
        for (int v : c->nb[sq[h] * R + r])
          if (!seen[v / R]) { seen[v / R] = 1; sq.push_back(v / R); }
    if ((int)sq.size() != S) return fail(ADPSGD_E_DISCONNECTED, "super-learner graph is not connected (rho = 1)");
  } else if (comps != 1) {
    return fail(ADPSGD_E_DISCONNECTED, "graph is not connected (rho = 1)");
  }
  c->role.assign(n, 0);
  if (g->role) {
    for (int v = 0; v < n; ++v) {
      if (g->role[v] != 0 && g->role[v] != 1) return fail(ADPSGD_E_INVALID, "role must be 0/1");
      c->role[v] = g->role[v];
    }
    for (int e = 0; e < g->n_edges; ++e)
      if (c->role[g->edges[2 * e]] == c->role[g->edges[2 * e + 1]])
        return fail(ADPSGD_E_NOT_BIPARTITE, "edge joins two workers of the same role (P:469-476)");
  } else {
    if (!bip) return fail(ADPSGD_E_NOT_BIPARTITE, "graph has an odd cycle: no active/passive split");
    for (int v = 0; v < n; ++v) c->role[v] = (int8_t)col[v];
  }
  c->edges.assign(g->edges, g->edges + 2 * g->n_edges);
  c->nb_flat.clear();
  c->nb_off.assign(n + 1, 0);
  for (int v = 0; v < n; ++v) {
    c->nb_off[v] = (int)c->nb_flat.size();
    c->nb_flat.insert(c->nb_flat.end(), c->nb[v].begin(), c->nb[v].end());
  }
  c->nb_off[n] = (int)c->nb_flat.size();
  return ADPSGD_OK;
}

bool is_neighbour(const adpsgd_ctx* c, int i, int j) {
  return std::binary_search(c->nb[i].begin(), c->nb[i].end(), j);
}

adpsgd_status upload_workers(adpsgd_ctx* c) {
  std::vector<WorkerDesc> wd(c->n);
  for (int w = 0; w < c->n; ++w) {
    const int r = c->worker_rank[w];
    WorkerDesc& x = wd[w];
    const long long l = c->worker_local[w];
    if (r == c->rank) {
      x.x = c->row(w);
      x.ctl = c->ctl + l;
    } else {
      x.x = c->peer_models[r] ? c->peer_models[r] + l * c->d_pad : nullptr;
      x.ctl = c->peer_ctl[r] ? reinterpret_cast<WorkerCtl*>(c->peer_ctl[r]) + l : nullptr;
    }
    x.rank = r;
    x.role = c->role[w];
    x.nb_off = c->nb_off[w];
    x.nb_cnt = c->nb_off[w + 1] - c->nb_off[w];
    x.straggle = c->straggle[w];
    x.local = r == c->rank ? c->worker_local[w] : -1;
    x.gb = (r == c->rank && c->wf_g) ? c->wf_g + l * 2 * c->d_pad : nullptr;
    x.gr = (r == c->rank && c->rrows) ? c->rrows + l * (long long)c->rrows_n * c->d_pad : nullptr;
    x.link = c->link[w];
    x.slot = c->peer_ctl[r] ? reinterpret_cast<Slot*>(c->peer_ctl[r] + c->peer_slots_off[r]) + l : nullptr;
  }
  CU(cudaMemcpy(c->d_workers, wd.data(), sizeof(WorkerDesc) * c->n, cudaMemcpyHostToDevice));
  CU(cudaDeviceSynchronize());   // pageable H2D may still be in flight; kernels use non-blocking streams
  return ADPSGD_OK;
}

adpsgd_status read_ticket(adpsgd_ctx* c, unsigned long long* k) {
  CU(cudaStreamSynchronize(c->stream));
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpy(k, &c->gctl0->ticket, sizeof(*k), cudaMemcpyDeviceToHost));
  return ADPSGD_OK;
}

// Multi-GPU adpsgd_step moves the device counter under every rank, so at the
// start of a collective call (world > 1) the ranks agree on it: each reads the
// device ticket after its own work has drained, then an all-reduce (MAX).  A
// rank's read follows all of its own steps, so the latest read -- the maximum
// -- covers every ticket taken; no rank can launch the collective's engine
// before every rank has contributed its read.  The read is a stream-ordered
// copy on c->stream, the stream the all-reduce runs on.
adpsgd_status settle_ticket(adpsgd_ctx* c) {
  if (c->world == 1 || !c->comm) return ADPSGD_OK;
  CU(cudaStreamSynchronize(c->stream));
  CU(cudaDeviceSynchronize());
  if (!c->agree64) CU(cudaMalloc(&c->agree64, sizeof(unsigned long long)));
  CU(cudaMemcpyAsync(c->agree64, &c->gctl0->ticket, sizeof(unsigned long long), cudaMemcpyDeviceToDevice,
                     c->stream));
  CO(c->comm->allreduce(c->agree64, c->agree64, 1, DType::U64, ROp::Max, c->stream, m_));
  unsigned long long t = 0;
  CU(cudaMemcpyAsync(&t, c->agree64, sizeof t, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  c->host_k = t;
  c->ticket_dirty = false;
  return ADPSGD_OK;
}

adpsgd_status host_ticket(adpsgd_ctx* c, unsigned long long* k) {
  ST(settle_ticket(c));
  *k = c->host_k;          // authoritative on every rank (see replay_engine)
  return ADPSGD_OK;
}

adpsgd_status ensure_gslots(adpsgd_ctx* c, int count) {
  if (c->gslot_n >= count) return ADPSGD_OK;
  if (c->gslots) cudaFree(c->gslots);
  c->gslots = nullptr;
  CU(cudaMalloc(&c->gslots, sizeof(float) * c->d_pad * count));
  // legacy-stream memset: finish it before any kernel on a non-blocking stream
  CU(cudaMemset(c->gslots, 0, sizeof(float) * c->d_pad * count));
  CU(cudaDeviceSynchronize());
  c->gslot_n = count;
  return ADPSGD_OK;
}

void release_mlp_work(MlpWork& w) { w = MlpWork{}; }

// one MLP scratch (gathered batch, partial planes, tensor maps, side stream) per stream lane
adpsgd_status ensure_mlp_scratch(adpsgd_ctx* c, int lanes = 1) {
  const size_t per = (mlp_scratch_floats(c->mlp, c->M) + 255) / 256 * 256;
  if ((int)c->mlp_work.size() >= lanes) return ADPSGD_OK;
  CU(cudaDeviceSynchronize());
  if (c->mlp_scratch) cudaFree(c->mlp_scratch);
  c->mlp_scratch = nullptr;
  CU(cudaMalloc(&c->mlp_scratch, sizeof(float) * per * lanes));
  c->mlp_scratch_n = per * lanes;
  for (MlpWork& w : c->mlp_work) release_mlp_work(w);
  c->mlp_work.assign(lanes, MlpWork{});
  for (int l = 0; l < lanes; ++l)                                 // tensor maps over each lane's planes
    CU(mlp_plan(c->mlp_work[l], c->mlp, c->M, c->mlp_scratch + per * l));
  return ADPSGD_OK;
}

// ------------------------------------------------------ replay stream DAG --
adpsgd_status ensure_pool(adpsgd_ctx* c, int ns) {
  while ((int)c->pool.size() < ns) {
    cudaStream_t st;
    CU(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    c->pool.push_back(st);
  }
  if (ns > 1 && c->evring.empty()) {
    c->evring.assign(kEventRing, nullptr);
    for (auto& e : c->evring) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  return ADPSGD_OK;
}

struct DagState {
  std::vector<cudaEvent_t> w_evt;                 // last op that wrote worker w's row
  std::vector<std::vector<cudaEvent_t>> r_evts;   // gradient reads of the row since that write
  std::vector<cudaEvent_t> g_evt, gready;         // slot consumer / slot producer
  DagState(int n, int slots) : w_evt(n, nullptr), r_evts(n), g_evt(slots, nullptr), gready(slots, nullptr) {}
};

adpsgd_status dag_wait(cudaStream_t st, cudaEvent_t e) {
  if (e) CU(cudaStreamWaitEvent(st, e, 0));
  return ADPSGD_OK;
}

// events are recycled from a ring: a recycled event stands for a LATER op
// enqueued earlier in host order, so a wait on it is conservative, never cyclic
adpsgd_status dag_record(adpsgd_ctx* c, cudaStream_t st, cudaEvent_t* out) {
  cudaEvent_t e = c->evring[c->evnext++ % c->evring.size()];
  CU(cudaEventRecord(e, st));
  *out = e;
  return ADPSGD_OK;
}

adpsgd_status dag_fork(adpsgd_ctx* c, cudaStream_t s, int ns) {
  cudaEvent_t e;
  ST(dag_record(c, s, &e));
  for (int l = 0; l < ns; ++l) CU(cudaStreamWaitEvent(c->pool[l], e, 0));
  return ADPSGD_OK;
}

adpsgd_status dag_join(adpsgd_ctx* c, cudaStream_t s, int ns) {
  for (int l = 0; l < ns; ++l) {
    cudaEvent_t e;
    ST(dag_record(c, c->pool[l], &e));
    CU(cudaStreamWaitEvent(s, e, 0));
  }
  return ADPSGD_OK;
}

// gradient of the built-in model at xhat into g (minibatch of event k)
adpsgd_status model_grad(adpsgd_ctx* c, const float* xhat, float* g, unsigned long long k,
                         const int* idx_dev, cudaStream_t s, int lane = 0) {
  switch (c->model) {
    case ADPSGD_MODEL_QUADRATIC:
      CU(launch_quad_grad(xhat, g, c->d, c->n4, c->q, k, s));
      break;
    case ADPSGD_MODEL_LSQ:
    case ADPSGD_MODEL_LOGREG:
      CU(launch_linear_grad((int)c->model, c->dA, c->db, c->S, idx_dev, c->M, c->seed2(), k, xhat, g,
                            c->d, s));
      break;
    case ADPSGD_MODEL_MLP:
      ST(ensure_mlp_scratch(c, lane + 1));
      CU(launch_mlp_grad(c->mlp_work[lane], c->dA, c->dy, c->S, idx_dev, c->seed2(), k, xhat, g, s));
      break;
    default:
      return fail(ADPSGD_E_UNSUPPORTED, "model has no built-in gradient");
  }
  c->launches += (c->model == ADPSGD_MODEL_MLP) ? kMlpLaunches : 1;
  return ADPSGD_OK;
}

adpsgd_status validate_events(adpsgd_ctx* c, const adpsgd_event* ev, int64_t K, bool need_local) {
  for (int64_t e = 0; e < K; ++e) {
    const int i = ev[e].i, j = ev[e].j, tau = ev[e].tau;
    char buf[160];
    if (i < 0 || i >= c->n || j < -1 || j >= c->n || i == j) {
      snprintf(buf, sizeof buf, "event %lld: invalid (i=%d, j=%d)", (long long)e, i, j);
      return fail(ADPSGD_E_INVALID, buf);
    }
    if (j >= 0 && !is_neighbour(c, i, j)) {
      snprintf(buf, sizeof buf, "event %lld: (%d,%d) is not an edge", (long long)e, i, j);
      return fail(ADPSGD_E_NOT_NEIGHBOURS, buf);
    }
    if (j >= 0 && c->role[i] == c->role[j]) return fail(ADPSGD_E_NOT_BIPARTITE, "event pairs same roles");
    if (tau < 0 || tau > c->T || tau > e) {
      snprintf(buf, sizeof buf, "event %lld: tau=%d exceeds min(k, T=%d) (P:601-602)", (long long)e, tau, c->T);
      return fail(ADPSGD_E_STALENESS, buf);
    }
    if (need_local && (!c->is_local(i) || (j >= 0 && !c->is_local(j))))
      return fail(ADPSGD_E_UNSUPPORTED, "host executor needs every worker local (world_size 1)");
  }
  return ADPSGD_OK;
}

// ----------------------------------------------------------- host replay ----
adpsgd_status replay_host(adpsgd_ctx* c, const adpsgd_event* ev, int64_t K, const int32_t* bidx,
                          cudaStream_t s) {
  ST(validate_events(c, ev, K, true));
  const bool has_model = c->model != ADPSGD_MODEL_NONE && c->model != ADPSGD_MODEL_EXTERNAL;
  for (int64_t e = 0; e < K; ++e)
    if (!(ev[e].flags & ADPSGD_EV_NO_GRAD) && !has_model && c->model == ADPSGD_MODEL_EXTERNAL)
      return fail(ADPSGD_E_UNSUPPORTED, "replay with gradients needs a built-in model");
  unsigned long long k0;
  ST(host_ticket(c, &k0));
  // App. A compensation (reading R20): comp_src[e] = worker i's previous
  // gradient event when it was still buffered at e's read point.  Its gradient
  // is in slot comp_src mod (T+1) at that point: it was computed at its own
  // read point (<= e's, checked) and that slot is reused only by the read of
  // event comp_src + T + 1, which comes later.
  std::vector<int64_t> comp_src(K, -1);
  bool any_comp = false;
  {
    std::vector<int64_t> last(c->n, -1);
    for (int64_t e = 0; e < K; ++e) {
      if (!has_model || (ev[e].flags & ADPSGD_EV_NO_GRAD)) continue;
      const int i = ev[e].i;
      const int64_t t = e - ev[e].tau;
      if ((ev[e].flags & ADPSGD_EV_COMPENSATE) && last[i] >= t) {
        if (last[i] - ev[last[i]].tau > t) {
          char buf[160];
          snprintf(buf, sizeof buf, "event %lld: compensated read precedes the previous gradient's read (App. A)",
                   (long long)e);
          return fail(ADPSGD_E_STALENESS, buf);
        }
        comp_src[e] = last[i];
        any_comp = true;
      }
      last[i] = e;
    }
  }
  // Events on disjoint workers commute (every coordinate sees the same op
  // sequence), so large-d / heavy-gradient replays run as a DAG over a pool of
  // streams: each op waits (cudaEvent) only for the last writer of the rows it
  // reads, the readers of the rows it writes, and its gradient slot.  The
  // result is bitwise the serial one.
  const int ns =
      (!any_comp && (c->model == ADPSGD_MODEL_MLP || c->d >= (1 << 16))) ? std::min(kPoolStreams, c->n) : 1;
  // gradient slots: event e's gradient lives in slot e mod `slots` from its read
  // to its event; T + 1 suffice in stream order, and in the DAG more slots let
  // more gradients be in flight (a slot's next read waits for its previous
  // event): up to 32, within 1 GB
  constexpr int kDagSlots = 32;
  const int slots = ns > 1 ? std::max(c->T + 1, (int)std::min<long long>(kDagSlots, (1LL << 30) / (4 * c->d_pad)))
                           : c->T + 1;
  bool need_slots = false;
  std::vector<std::vector<int64_t>> reads(K);
  for (int64_t e = 0; e < K; ++e) {
    const bool grad = has_model && !(ev[e].flags & ADPSGD_EV_NO_GRAD);
    if (!grad) continue;
    if (c->model == ADPSGD_MODEL_QUADRATIC && ev[e].tau == 0 && !any_comp) continue;   // fused inline
    need_slots = true;
    reads[e - ev[e].tau].push_back(e);   // gradient at X_{e - tau}
  }
  if (need_slots) ST(ensure_gslots(c, slots));
  if (any_comp && !c->comp_row) CU(cudaMalloc(&c->comp_row, sizeof(float) * c->d_pad));
  const bool sampled = c->model == ADPSGD_MODEL_LSQ || c->model == ADPSGD_MODEL_LOGREG ||
                       c->model == ADPSGD_MODEL_MLP;
  if (sampled && bidx) {
    const size_t need = (size_t)K * c->M;
    if (c->batch_cap < need) {
      if (c->d_batch) cudaFree(c->d_batch);
      c->d_batch = nullptr;
      CU(cudaMalloc(&c->d_batch, sizeof(int) * need));
      c->batch_cap = need;
    }
    for (size_t t = 0; t < need; ++t)
      if (bidx[t] < 0 || bidx[t] >= c->S) return fail(ADPSGD_E_INVALID, "batch index out of range");
    CU(cudaMemcpyAsync(c->d_batch, bidx, sizeof(int) * need, cudaMemcpyHostToDevice, s));
  }
  ST(ensure_pool(c, ns));
  if (c->model == ADPSGD_MODEL_MLP && need_slots) ST(ensure_mlp_scratch(c, ns));
  DagState dag(c->n, slots);
  if (ns > 1) ST(dag_fork(c, s, ns));
  // config 1 (lsq / logreg, one lane): the whole schedule -- at each event e the gradients read
  // at X_e, then event e -- in ONE launch of k_lin_replay
  const bool fuse_lin = (c->model == ADPSGD_MODEL_LSQ || c->model == ADPSGD_MODEL_LOGREG) && ns == 1 && !any_comp &&
                        c->d % 4 == 0 && c->M <= 1024;
  if (fuse_lin && K > 0) {
    std::vector<LinRead> lr;
    std::vector<LinEventOp> lo((size_t)K);
    for (int64_t e = 0; e < K; ++e) {
      LinEventOp& op = lo[(size_t)e];
      op.r0 = (int)lr.size();
      for (int64_t kp : reads[e]) {
        LinRead r{};
        const int i = ev[kp].i;
        r.x = c->row(i);
        r.g = c->gslots + (long long)(kp % slots) * c->d_pad;
        r.idx = bidx ? c->d_batch + kp * c->M : nullptr;
        r.k = (ev[kp].flags & ADPSGD_EV_FLUSH_FIRST) ? read_key(k0 + kp - ev[kp].tau, i) : k0 + kp;
        lr.push_back(r);
      }
      op.r1 = (int)lr.size();
      const int i = ev[e].i, j = ev[e].j;
      const bool grad = !(ev[e].flags & ADPSGD_EV_NO_GRAD);
      if (j >= 0 || grad) {
        op.xi = c->row(i);
        op.xj = j >= 0 ? c->row(j) : nullptr;
        op.g = grad ? c->gslots + (long long)(e % slots) * c->d_pad : nullptr;
        op.ff = grad && (ev[e].flags & ADPSGD_EV_FLUSH_FIRST) ? 1 : 0;
      }
    }
    const size_t bytes = lo.size() * sizeof(LinEventOp) + lr.size() * sizeof(LinRead);
    if (c->lin_cap < bytes) {
      if (c->lin_buf) cudaFree(c->lin_buf);
      c->lin_buf = nullptr;
      CU(cudaMalloc(&c->lin_buf, bytes));
      c->lin_cap = bytes;
    }
    // lin_buf may still feed the previous replay, and the host vectors die with this call:
    // stage them in stream order and wait (a few tens of KB)
    CU(cudaStreamSynchronize(s));
    CU(cudaMemcpyAsync(c->lin_buf, lo.data(), lo.size() * sizeof(LinEventOp), cudaMemcpyHostToDevice, s));
    if (!lr.empty())
      CU(cudaMemcpyAsync(c->lin_buf + lo.size() * sizeof(LinEventOp), lr.data(), lr.size() * sizeof(LinRead),
                         cudaMemcpyHostToDevice, s));
    CU(cudaStreamSynchronize(s));
    LinReplayParams lp{};
    lp.kind = (int)c->model; lp.S = c->S; lp.M = c->M; lp.A = c->dA; lp.b = c->db; lp.key = c->seed2();
    lp.gamma = c->gamma; lp.d = c->d; lp.n4 = c->n4; lp.nops = (int)K;
    lp.ops = reinterpret_cast<const LinEventOp*>(c->lin_buf);
    lp.reads = reinterpret_cast<const LinRead*>(c->lin_buf + lo.size() * sizeof(LinEventOp));
    CU(launch_lin_replay(lp, s));
    ++c->launches;
  }
  for (int64_t e = 0; e < K && !fuse_lin; ++e) {
    for (int64_t kp : reads[e]) {     // stale reads that happen before event e
      const int i = ev[kp].i;
      const int lane = ns > 1 ? i % ns : 0;
      cudaStream_t st = ns > 1 ? c->pool[lane] : s;
      const int sl = (int)(kp % slots);
      if (ns > 1) { ST(dag_wait(st, dag.w_evt[i])); ST(dag_wait(st, dag.g_evt[sl])); }
      float* slot = c->gslots + (long long)sl * c->d_pad;
      const int* idx = (sampled && bidx) ? c->d_batch + kp * c->M : nullptr;
      const unsigned long long key =
          (ev[kp].flags & ADPSGD_EV_FLUSH_FIRST) ? read_key(k0 + kp - ev[kp].tau, i) : k0 + kp;
      const float* src = c->row(i);
      if (comp_src[kp] >= 0) {            // pulled while g_p was buffered: x - gamma g_p
        CU(launch_comp_row(src, c->gslots + (long long)(comp_src[kp] % slots) * c->d_pad, c->gamma, c->comp_row,
                           c->n4, st));
        ++c->launches;
        src = c->comp_row;
      }
      ST(model_grad(c, src, slot, key, idx, st, lane));
      if (ns > 1) {
        cudaEvent_t done;
        ST(dag_record(c, st, &done));
        dag.r_evts[i].push_back(done);
        dag.gready[sl] = done;
      }
    }
    const int i = ev[e].i, j = ev[e].j;
    const bool grad = has_model && !(ev[e].flags & ADPSGD_EV_NO_GRAD);
    int mode = kGradNone;
    const float* g = nullptr;
    const int sl = (int)(e % slots);
    unsigned long long key = k0 + e;
    if (grad) {
      if (c->model == ADPSGD_MODEL_QUADRATIC && ev[e].tau == 0 && !any_comp) mode = kGradQuadInline;
      else { mode = kGradExternal; g = c->gslots + (long long)sl * c->d_pad; }
      if (ev[e].flags & ADPSGD_EV_FLUSH_FIRST) {
        key = read_key(k0 + e, i);           // tau = 0 here when inline
        mode |= kModeFlushFirst;
      }
    }
    if (j >= 0 || mode != kGradNone) {
      cudaStream_t st = ns > 1 ? c->pool[i % ns] : s;
      if (ns > 1) {
        ST(dag_wait(st, dag.w_evt[i]));
        for (cudaEvent_t r : dag.r_evts[i]) ST(dag_wait(st, r));
        if (j >= 0) {
          ST(dag_wait(st, dag.w_evt[j]));
          for (cudaEvent_t r : dag.r_evts[j]) ST(dag_wait(st, r));
        }
        if ((mode & 0xf) == kGradExternal) ST(dag_wait(st, dag.gready[sl]));
      }
      CU(launch_event(c->row(i), j >= 0 ? c->row(j) : nullptr, g, nullptr, c->d, c->n4, c->gamma,
                      c->q, key, mode, st));
      ++c->launches;
      if (ns > 1) {
        cudaEvent_t done;
        ST(dag_record(c, st, &done));
        dag.w_evt[i] = done;
        dag.r_evts[i].clear();
        if (j >= 0) { dag.w_evt[j] = done; dag.r_evts[j].clear(); }
        if ((mode & 0xf) == kGradExternal) dag.g_evt[sl] = done;
      }
    }
  }
  if (ns > 1) ST(dag_join(c, s, ns));
  c->host_k = k0 + K;
  CU(launch_set_u64(&c->gctl0->ticket, c->host_k, s));
  CU(launch_set_u64(&c->gctl0->committed, c->host_k, s));
  c->launches += 2;
  return ADPSGD_OK;
}

// --------------------------------------------------------- engine helpers --
adpsgd_status engine_launch(adpsgd_ctx* c, int mode, unsigned long long target, cudaStream_t s) {
  EngineParams p{};
  p.workers = c->d_workers;
  p.nbrs = c->d_nbrs;
  p.n = c->n;
  p.n_local = c->n_local;
  p.slots = c->d_slots;
  p.local_ids = c->d_local_ids;
  p.gctl0 = c->gctl0;
  p.gctl = c->gctl;
  p.log = c->log0;
  p.log_cap = c->log_cap;
  p.target = target;
  p.mode = mode;
  p.model = (int)c->model == ADPSGD_MODEL_QUADRATIC ? 2 : 0;
  p.my_rank = c->rank;
  p.rev = c->d_rev;
  p.q = c->q;
  p.gamma = c->gamma;
  p.d = c->d;
  p.n4 = c->n4;
  p.compute_ns = c->compute_ns;
  p.seed = make_uint2((uint32_t)(c->seed ^ 0x5bd1e995u), (uint32_t)(c->seed >> 32) ^ c->run_counter);
  p.watchdog_ns = 60ull * 1000000000ull;
  p.wait_free = mode == 0 ? c->wait_free : 0;
  p.link_ns = c->link_ns;
  p.fuse = c->engine_fuse;
  p.fuse_wait_ns = (unsigned long long)c->fuse_wait_ns;
  // cooperative cross-GPU events: the partner GPU's CTAs claim half of the tiles;
  // not in the wait-free loop (its gradient rows are not peer-mapped)
  bool coop = c->engine_coop > 0;
  if (c->engine_coop == 0 && c->world > 1) {
    // auto: on at two GPUs (measured: N=2 all-cross 455 -> 624 GB/s free-running,
    // 599 -> 644 replay; bench block placement +1.8%), when at most half of the
    // edges cross GPUs (bench at N=4, block placement: +1.9%), or when some GPU
    // starts fewer than half the cross events another one starts (free-running:
    // only actives start events).  Off when nearly every edge crosses and the
    // initiators are spread evenly (N=4 xor placement: 535 -> 457 GB/s, every
    // event then waits for its second half queued behind the partner's own work).
    std::vector<int> init(c->world, 0);
    int cross = 0;
    for (size_t e = 0; e + 1 < c->edges.size(); e += 2) {
      const int a = c->edges[e], b = c->edges[e + 1];
      if (c->worker_rank[a] == c->worker_rank[b]) continue;
      ++cross;
      const int act = c->role[a] == 0 ? a : b;
      init[c->worker_rank[act]]++;
    }
    const int mx = *std::max_element(init.begin(), init.end()), mn = *std::min_element(init.begin(), init.end());
    const bool few_cross = 2 * (size_t)cross <= c->edges.size() / 2;
    coop = c->world == 2 || few_cross || (mode == 0 && mx > 2 * mn);
  }
  p.coop = (c->world > 1 && coop && !(mode == 0 && c->wait_free)) ? 1 : 0;
  // the grid is fixed at init (and checked equal across ranks at import: the
  // per-GPU cap on a cross event's CTAs is grid / 8 on both sides)
  if (c->engine_grid < 1) return fail(ADPSGD_E_CUDA, "engine kernel cannot be resident");
  CU(cudaMemsetAsync(&c->gctl->abort_flag, 0, sizeof(unsigned int), s));
  // processes: a cooperative launch guarantees co-residency of the grid; in-process
  // ranks sharing a device launch normally (their grids together fit the device)
  CU(launch_engine(p, c->engine_grid, c->engine_threads, !c->comm_local, s));
  ++c->launches;
  ++c->run_counter;
  return ADPSGD_OK;
}

adpsgd_status reset_slots(adpsgd_ctx* c, cudaStream_t s) {
  c->h_slots.assign(c->n_local, Slot{});
  for (int l = 0; l < c->n_local; ++l) {
    Slot& x = c->h_slots[l];
    x.tag = 0;
    x.pending_j = -2;
    x.absorb = -1;
    x.nb_ctr = c->run_counter << 20;
    x.j = -1;
  }
  CU(cudaMemcpyAsync(c->d_slots, c->h_slots.data(), sizeof(Slot) * c->n_local, cudaMemcpyHostToDevice, s));
  CU(cudaStreamSynchronize(s));
  return ADPSGD_OK;
}

// ---------------------------------------------------------- host planning --
// worker -> rank (0 block: contiguous ring segments; 1 interleave; 2 explicit)
adpsgd_status compute_placement(int n, int world, int placement, const int32_t* explicit_rank,
                                std::vector<int>& wr, std::vector<int>& wl) {
  if (n < 1 || world < 1) return fail(ADPSGD_E_INVALID, "n / world_size");
  wr.assign(n, 0);
  for (int w = 0; w < n; ++w) {
    if (placement == 0) wr[w] = (int)((long long)w * world / n);
    else if (placement == 1) wr[w] = w % world;
    else if (placement == 2) {
      if (!explicit_rank) return fail(ADPSGD_E_INVALID, "explicit placement needs worker_rank");
      wr[w] = explicit_rank[w];
      if (wr[w] < 0 || wr[w] >= world) return fail(ADPSGD_E_INVALID, "worker_rank out of range");
    } else return fail(ADPSGD_E_INVALID, "placement");
  }
  wl.assign(n, 0);
  std::vector<int> cnt(world, 0);
  for (int w = 0; w < n; ++w) wl[w] = cnt[wr[w]]++;
  return ADPSGD_OK;
}

// Engine-replay plan.  Every worker w has a sequence of ops: the schedule's
// events touching w (as i or j) and the stale reads of w's own gradient events
// (tau > 0: the gradient at X_{k - tau}, is computed by a read op placed
// in w's sequence right before the first event >= k - tau that touches w, into
// one of w's T + 1 read rows -- w's m-th stale event uses row m mod (T + 1),
// which no later read can overwrite before the event ran, since that read's
// point is after it).  An op waits until epoch[i] (and epoch[j] for a pair)
// equals the number of earlier ops in that worker's sequence, and bumps them
// when it commits, so every worker sees the schedule's order.  Every rank runs
// this on the same schedule and epoch mirror and keeps the ops whose worker i
// is local.  A read op's k holds its gradient's random-draw key.
void plan_replay(const std::vector<int>& wr, const std::vector<int>& wl, int rank, int n_local,
                 const adpsgd_event* ev, int64_t K, unsigned long long k0, int T, bool stale_reads,
                 std::vector<unsigned int>& ep, std::vector<std::vector<ReplayEv>>& per) {
  per.assign(n_local, {});
  const int n = (int)ep.size();
  std::vector<std::vector<int64_t>> reads_at(stale_reads ? K : 0);   // stale events read before event e
  if (stale_reads)
    for (int64_t e = 0; e < K; ++e)
      if (ev[e].tau > 0 && !(ev[e].flags & ADPSGD_EV_NO_GRAD)) reads_at[e - ev[e].tau].push_back(e);
  std::vector<int> row(n, 0);
  std::vector<int> row_of(stale_reads ? K : 0, -1);
  for (int64_t e = 0; e < K; ++e) {
    if (stale_reads)
      for (int64_t f : reads_at[e]) {
        const int i = ev[f].i;
        row_of[f] = row[i]++ % (T + 1);
        ReplayEv r{};
        r.kind = kKindRead;
        r.k = (long long)((ev[f].flags & ADPSGD_EV_FLUSH_FIRST) ? read_key(k0 + e, i) : k0 + f);
        r.j = -1;
        r.flags = ev[f].flags;
        r.e_i = ep[i]++;
        r.grow = row_of[f];
        if (wr[i] == rank) per[wl[i]].push_back(r);
      }
    const int i = ev[e].i, j = ev[e].j;
    ReplayEv r{};
    r.kind = kKindEvent;
    r.k = (long long)(k0 + e);
    r.j = j;
    r.flags = ev[e].flags;
    r.e_i = ep[i];
    r.e_j = j >= 0 ? ep[j] : 0;
    r.grow = stale_reads ? row_of[e] : -1;
    ep[i]++;
    if (j >= 0) ep[j]++;
    if (wr[i] == rank) per[wl[i]].push_back(r);
  }
}

adpsgd_status replay_engine(adpsgd_ctx* c, const adpsgd_event* ev, int64_t K, cudaStream_t s) {
  if (!c->connected) return fail(ADPSGD_E_STATE, "not connected");
  if (c->model != ADPSGD_MODEL_NONE && c->model != ADPSGD_MODEL_QUADRATIC)
    return fail(ADPSGD_E_UNSUPPORTED, "engine replay supports models NONE and QUADRATIC");
  ST(validate_events(c, ev, K, false));
  bool stale = false;
  for (int64_t e = 0; e < K; ++e) {
    // with tau = 0 the previous gradient is always applied before the read: COMPENSATE is a no-op
    if ((ev[e].flags & ADPSGD_EV_COMPENSATE) && ev[e].tau > 0)
      return fail(ADPSGD_E_UNSUPPORTED, "engine replay does not run stale COMPENSATE events (use HOST)");
    stale |= ev[e].tau > 0 && !(ev[e].flags & ADPSGD_EV_NO_GRAD) && c->model == ADPSGD_MODEL_QUADRATIC;
  }
  // read rows for stale reads (T + 1 per local worker), allocated before any
  // engine of this call runs (the peers' engines never touch them)
  if (stale && c->rrows_n < c->T + 1 && c->n_local) {
    CU(cudaDeviceSynchronize());
    if (c->rrows) cudaFree(c->rrows);
    c->rrows = nullptr;
    CU(cudaMalloc(&c->rrows, sizeof(float) * c->d_pad * (size_t)(c->T + 1) * c->n_local));
    CU(cudaMemset(c->rrows, 0, sizeof(float) * c->d_pad * (size_t)(c->T + 1) * c->n_local));
    c->rrows_n = c->T + 1;
    ST(upload_workers(c));
  }
  // the op list (<= one op per endpoint of each event + one read per event), sized before the
  // collective below: after it a peer's engine may already run, and with ranks sharing a GPU
  // (comm_local) a cudaMalloc / cudaFree that synchronises the device would wait for it
  {
    const size_t cap = (size_t)3 * (size_t)K + (size_t)c->n_local + 1;
    if (c->rev_cap < cap) {
      CU(cudaDeviceSynchronize());
      if (c->d_rev) cudaFree(c->d_rev);
      c->d_rev = nullptr;
      CU(cudaMalloc(&c->d_rev, sizeof(ReplayEv) * cap));
      c->rev_cap = cap;
    }
  }
  // k and the epochs are tracked identically on every rank (they only change
  // through collective calls whose effect is known: a replay advances k by K
  // and the epochs by the schedule, a run ends at exactly its target), so no
  // rank reads device state that another rank's engine may already be moving.
  ST(settle_ticket(c));
  const unsigned long long k0 = c->host_k;
  std::vector<std::vector<ReplayEv>> per;
  plan_replay(c->worker_rank, c->worker_local, c->rank, c->n_local, ev, K, k0, c->T, stale, c->epochs, per);
  c->h_rev.clear();
  ST(reset_slots(c, s));
  for (int l = 0; l < c->n_local; ++l) {
    c->h_slots[l].ev_cur = (long long)c->h_rev.size();
    c->h_rev.insert(c->h_rev.end(), per[l].begin(), per[l].end());
    c->h_slots[l].ev_end = (long long)c->h_rev.size();
  }
  if (c->rev_cap < c->h_rev.size() + 1) return fail(ADPSGD_E_STATE, "replay op list exceeds its bound");
  if (!c->h_rev.empty())
    CU(cudaMemcpyAsync(c->d_rev, c->h_rev.data(), sizeof(ReplayEv) * c->h_rev.size(), cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(c->d_slots, c->h_slots.data(), sizeof(Slot) * c->n_local, cudaMemcpyHostToDevice, s));
  ST(engine_launch(c, 1, k0 + (unsigned long long)K, s));
  c->host_k = k0 + (unsigned long long)K;
  return ADPSGD_OK;
}

adpsgd_status destroy_impl(adpsgd_ctx* c) {
  if (!c) return ADPSGD_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  delete c->super_comm;
  delete c->comm;
  for (size_t r = 0; r < c->peer_models.size() && !c->comm_local; ++r) {
    if ((int)r == c->rank) continue;
    if (c->peer_models[r]) cudaIpcCloseMemHandle(c->peer_models[r]);
    if (c->peer_ctl[r]) cudaIpcCloseMemHandle(c->peer_ctl[r]);
  }
  for (MlpWork& w : c->mlp_work) release_mlp_work(w);
  for (auto e : c->last_evt) if (e) cudaEventDestroy(e);
  for (auto e : c->evring) if (e) cudaEventDestroy(e);
  for (auto st : c->pool) if (st) cudaStreamDestroy(st);
  void* bufs[] = {c->models, c->ctl_arena, c->d_workers, c->d_nbrs, c->d_local_ids,
                  c->d_rev, c->dx0, c->dA, c->db, c->dy, c->gslots, c->gstep, c->mlp_scratch, c->lin_buf,
                  c->d_batch, c->sum64, c->mk_acc, c->xr, c->gsum, c->rrows,
                  c->dp_x[0], c->dp_x[1], c->dp_halo, c->d_dp_nbr[0], c->d_dp_nbr[1], c->d_dp_deg,
                  c->d_dp_wself, c->wf_g, c->comp_row, c->super_g, c->super_k, c->super_bar, c->agree64};
  for (void* b : bufs) if (b) cudaFree(b);
  if (c->k_host) cudaFreeHost(c->k_host);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return ADPSGD_OK;
}

// Load every kernel of the library on the current device now.  Under lazy
// module loading (the CUDA 12 default) a kernel's first launch loads it, and
// loading can wait for the device to drain -- which never happens while another
// rank's kernel on the same device spins on work this launch belongs to (a peer
// lock kernel waiting for our commit, a cooperative engine).  Each translation
// unit is one module: enumerate its functions from one anchor kernel.
adpsgd_status preload_modules(int device) {
  static std::mutex mu;
  static std::vector<int> done;
  std::lock_guard<std::mutex> lk(mu);
  if (std::find(done.begin(), done.end(), device) != done.end()) return ADPSGD_OK;
  using FnGetModule = CUresult (*)(CUmodule*, CUfunction);
  using FnCount = CUresult (*)(unsigned int*, CUmodule);
  using FnEnum = CUresult (*)(CUfunction*, unsigned int, CUmodule);
  using FnLoad = CUresult (*)(CUfunction);
  void *p_mod = nullptr, *p_cnt = nullptr, *p_enum = nullptr, *p_load = nullptr;
  cudaDriverEntryPointQueryResult q;
  CU(cudaGetDriverEntryPointByVersion("cuFuncGetModule", &p_mod, 12040, cudaEnableDefault, &q));
  CU(cudaGetDriverEntryPointByVersion("cuModuleGetFunctionCount", &p_cnt, 12040, cudaEnableDefault, &q));
  CU(cudaGetDriverEntryPointByVersion("cuModuleEnumerateFunctions", &p_enum, 12040, cudaEnableDefault, &q));
  CU(cudaGetDriverEntryPointByVersion("cuFuncLoad", &p_load, 12040, cudaEnableDefault, &q));
  if (!p_mod || !p_cnt || !p_enum || !p_load) return fail(ADPSGD_E_UNSUPPORTED, "driver lacks module enumeration");
  const void* anchors[] = {kernels_module_anchor(), engine_module_anchor(), gemm_module_anchor(),
                           mlp_module_anchor(), comm_module_anchor()};
  for (const void* a : anchors) {
    cudaFunction_t f = nullptr;
    CU(cudaGetFuncBySymbol(&f, a));          // loads the anchor, yields its module
    CUmodule mod = nullptr;
    unsigned int cnt = 0;
    if (((FnGetModule)p_mod)(&mod, (CUfunction)f) != CUDA_SUCCESS || ((FnCount)p_cnt)(&cnt, mod) != CUDA_SUCCESS)
      return fail(ADPSGD_E_CUDA, "module enumeration failed");
    std::vector<CUfunction> fns(cnt);
    if (cnt && ((FnEnum)p_enum)(fns.data(), cnt, mod) != CUDA_SUCCESS)
      return fail(ADPSGD_E_CUDA, "module enumeration failed");
    for (CUfunction fn : fns)
      if (((FnLoad)p_load)(fn) != CUDA_SUCCESS) return fail(ADPSGD_E_CUDA, "cuFuncLoad failed");
  }
  done.push_back(device);
  return ADPSGD_OK;
}

adpsgd_status init_impl(const adpsgd_graph* g, int32_t n_workers, int64_t d,
                        const adpsgd_config* cfg, adpsgd_ctx** out) {
  if (!g || !cfg || !out) return fail(ADPSGD_E_INVALID, "null argument");
  if (n_workers != g->n) return fail(ADPSGD_E_INVALID, "n_workers != graph.n");
  if (d < 1 || d > (1LL << 31) - 64) return fail(ADPSGD_E_INVALID, "d out of range");   // engine: < 2^16 claim chunks
  if (cfg->world_size < 1 || cfg->rank < 0 || cfg->rank >= cfg->world_size)
    return fail(ADPSGD_E_INVALID, "rank/world_size");
  if (cfg->batch_M < 0 || cfg->staleness_cap_T < 0) return fail(ADPSGD_E_INVALID, "M/T < 0");
  std::unique_ptr<adpsgd_ctx> c(new adpsgd_ctx());
  c->rank = cfg->rank;
  c->world = cfg->world_size;
  c->device = cfg->device;
  c->n = n_workers;
  c->d = d;
  c->d_pad = (d + 63) / 64 * 64;
  c->n4 = c->d_pad / 4;
  c->model = cfg->model;
  c->gamma = cfg->gamma;
  c->M = cfg->batch_M > 0 ? cfg->batch_M : 1;
  c->T = cfg->staleness_cap_T;
  c->seed = cfg->seed;
  c->q.data_key = cfg->quad_data_key;
  c->q.noise_key = cfg->quad_noise_key;
  c->q.Mf = (float)c->M;
  c->q.s = cfg->quad_noise_s;
  c->compute_ns = cfg->compute_ns;
  c->engine_cps = cfg->engine_ctas_per_sm;
  c->engine_threads = 512;
  // engine_variant: the round-1 A/B variants (register slices, per-warp barriers,
  // two-sided push protocol) were measured slower and removed; 0 is the engine
  if (cfg->engine_variant != 0) return fail(ADPSGD_E_UNSUPPORTED, "engine_variant must be 0 (the A/B variants "
                                                                  "1-3 were removed)");
  if (cfg->log_capacity > 0) c->log_cap = cfg->log_capacity;
  if (c->model < ADPSGD_MODEL_NONE || c->model > ADPSGD_MODEL_MLP) return fail(ADPSGD_E_INVALID, "model");
  c->wait_free = cfg->wait_free;
  c->super_R = cfg->super_R > 1 ? cfg->super_R : 0;
  c->engine_fuse = cfg->engine_no_fuse ? 0 : 1;
  c->engine_coop = cfg->engine_coop;
  c->comm_local = cfg->comm_local != 0;
  if (cfg->engine_grid < 0) return fail(ADPSGD_E_INVALID, "engine_grid < 0");
  if (c->engine_coop < -1 || c->engine_coop > 1) return fail(ADPSGD_E_INVALID, "engine_coop must be -1, 0 or 1");
  c->fuse_wait_ns = cfg->engine_fuse_wait_ns;
  if (c->fuse_wait_ns < 0) return fail(ADPSGD_E_INVALID, "engine_fuse_wait_ns < 0");
  if (c->wait_free < 0 || c->wait_free > 2) return fail(ADPSGD_E_INVALID, "wait_free must be 0, 1 or 2");
  if (c->wait_free && c->model != ADPSGD_MODEL_QUADRATIC)
    return fail(ADPSGD_E_UNSUPPORTED, "the wait-free (App. A) engine loop supports the QUADRATIC model");
  ST(check_graph(c.get(), g));
  // placement
  ST(compute_placement(c->n, c->world, cfg->placement, cfg->worker_rank, c->worker_rank, c->worker_local));
  for (int w = 0; w < c->n; ++w)
    if (c->worker_rank[w] == c->rank) c->local_ids.push_back(w);
  c->n_local = (int)c->local_ids.size();
  if (c->n_local > kMaxLocal) return fail(ADPSGD_E_UNSUPPORTED, "more than 128 workers on one GPU");
  c->straggle.assign(c->n, 1.0f);
  if (cfg->straggler)
    for (int w = 0; w < c->n; ++w) {
      if (!(cfg->straggler[w] >= 1.0f)) return fail(ADPSGD_E_INVALID, "straggler factors must be >= 1");
      c->straggle[w] = cfg->straggler[w];
    }
  c->link.assign(c->n, 1.0f);
  c->link_ns = cfg->link_ns;
  if (c->link_ns < 0) return fail(ADPSGD_E_INVALID, "link_ns < 0");
  if (cfg->link_slow)
    for (int w = 0; w < c->n; ++w) {
      if (!(cfg->link_slow[w] >= 1.0f)) return fail(ADPSGD_E_INVALID, "link_slow factors must be >= 1");
      c->link[w] = cfg->link_slow[w];
    }
  // model data
  if (c->model == ADPSGD_MODEL_LSQ || c->model == ADPSGD_MODEL_LOGREG || c->model == ADPSGD_MODEL_MLP) {
    if (cfg->n_samples < 1 || !cfg->data_A) return fail(ADPSGD_E_INVALID, "dataset required");
    c->S = cfg->n_samples;
    if (c->model == ADPSGD_MODEL_MLP) {
      c->mlp = MlpShape{cfg->mlp_in, cfg->mlp_hid, cfg->mlp_out};
      const long long dim = (long long)c->mlp.n_hid * c->mlp.n_in + c->mlp.n_hid +
                            (long long)c->mlp.n_out * c->mlp.n_hid + c->mlp.n_out;
      if (dim != d || !cfg->data_y) return fail(ADPSGD_E_INVALID, "mlp dims do not match d / labels missing");
      if (!mlp_supported(c->mlp, c->M))
        return fail(ADPSGD_E_UNSUPPORTED, "MLP tensor-core path needs batch_M, mlp_in, mlp_hid multiples of 128, "
                                          "mlp_hid <= 1024 and mlp_out <= 32");
      c->feat = c->mlp.n_in;
    } else {
      if (!cfg->data_b) return fail(ADPSGD_E_INVALID, "data_b required");
      c->feat = (int)d;
    }
    if (c->M > 1024) return fail(ADPSGD_E_UNSUPPORTED, "batch_M > 1024");
  }
  CU(cudaSetDevice(c->device));
  ST(preload_modules(c->device));
  CU(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  // the ticket slot host-driven steps and super-learners read back, allocated here and never
  // lazily: a cudaMalloc while another rank's lock kernel spins can stall until that rank's
  // commit -- which may be waiting to be launched by the thread inside cudaMalloc
  CU(cudaMalloc(&c->super_k, sizeof(unsigned long long)));
  CU(cudaMallocHost(&c->k_host, sizeof(unsigned long long)));
  // models
  CU(cudaMalloc(&c->models, sizeof(float) * c->d_pad * std::max(1, c->n_local)));
  CU(cudaMemset(c->models, 0, sizeof(float) * c->d_pad * std::max(1, c->n_local)));
  CU(cudaMalloc(&c->dx0, sizeof(float) * c->d_pad));
  CU(cudaMemset(c->dx0, 0, sizeof(float) * c->d_pad));
  if (cfg->x0) CU(cudaMemcpy(c->dx0, cfg->x0, sizeof(float) * d, cudaMemcpyHostToDevice));
  if (cfg->x0_per_worker) {
    for (int l = 0; l < c->n_local; ++l)
      CU(cudaMemcpy(c->models + (long long)l * c->d_pad, cfg->x0_per_worker + (long long)c->local_ids[l] * d,
                    sizeof(float) * d, cudaMemcpyHostToDevice));
  } else if (c->n_local) {
    // the memsets / copies above ran on the legacy stream, which a non-blocking
    // stream does not wait for: settle them before the first kernel
    CU(cudaDeviceSynchronize());
    CU(launch_init_rows(c->models, c->n_local, c->d_pad, c->d, c->dx0, c->stream));
  }
  // control arena (peer-mapped): WorkerCtl[n_local] | GlobalCtl | push counters [n_local][kMaxGrid] |
  // engine Slots[n_local] | (rank 0) log
  c->gctl_offset = sizeof(WorkerCtl) * std::max(1, c->n_local);
  c->slots_offset = (c->gctl_offset + sizeof(GlobalCtl) + 127) / 128 * 128;
  c->log_offset = (c->slots_offset + sizeof(Slot) * std::max(1, c->n_local) + 255) / 256 * 256;
  c->ctl_bytes = c->log_offset + (c->rank == 0 ? sizeof(LogEntry) * c->log_cap : 0);
  CU(cudaMalloc(&c->ctl_arena, c->ctl_bytes));
  CU(cudaMemset(c->ctl_arena, 0, c->ctl_bytes));
  c->ctl = reinterpret_cast<WorkerCtl*>(c->ctl_arena);
  c->gctl = reinterpret_cast<GlobalCtl*>(c->ctl_arena + c->gctl_offset);
  c->log = c->rank == 0 ? reinterpret_cast<LogEntry*>(c->ctl_arena + c->log_offset) : nullptr;
  if (c->rank == 0) { c->gctl0 = c->gctl; c->log0 = c->log; }
  // datasets (every rank: Strategy-1)
  if (c->S) {
    CU(cudaMalloc(&c->dA, sizeof(float) * (size_t)c->S * c->feat));
    CU(cudaMemcpy(c->dA, cfg->data_A, sizeof(float) * (size_t)c->S * c->feat, cudaMemcpyHostToDevice));
    if (cfg->data_b) {
      CU(cudaMalloc(&c->db, sizeof(float) * c->S));
      CU(cudaMemcpy(c->db, cfg->data_b, sizeof(float) * c->S, cudaMemcpyHostToDevice));
    }
    if (cfg->data_y) {
      for (int s = 0; s < c->S; ++s)
        if (cfg->data_y[s] < 0 || cfg->data_y[s] >= c->mlp.n_out) return fail(ADPSGD_E_INVALID, "label range");
      CU(cudaMalloc(&c->dy, sizeof(int) * c->S));
      CU(cudaMemcpy(c->dy, cfg->data_y, sizeof(int) * c->S, cudaMemcpyHostToDevice));
    }
  }
  // tables
  CU(cudaMalloc(&c->d_workers, sizeof(WorkerDesc) * c->n));
  CU(cudaMalloc(&c->d_nbrs, sizeof(int) * std::max<size_t>(1, c->nb_flat.size())));
  if (!c->nb_flat.empty())
    CU(cudaMemcpy(c->d_nbrs, c->nb_flat.data(), sizeof(int) * c->nb_flat.size(), cudaMemcpyHostToDevice));
  CU(cudaMalloc(&c->d_local_ids, sizeof(int) * std::max(1, c->n_local)));
  if (c->n_local)
    CU(cudaMemcpy(c->d_local_ids, c->local_ids.data(), sizeof(int) * c->n_local, cudaMemcpyHostToDevice));
  c->d_slots = reinterpret_cast<Slot*>(c->ctl_arena + c->slots_offset);   // zeroed with the arena
  if (c->wait_free && c->n_local) {          // App. A gradient rows: buffer + computing gradient
    CU(cudaMalloc(&c->wf_g, sizeof(float) * 2 * c->d_pad * c->n_local));
    CU(cudaMemset(c->wf_g, 0, sizeof(float) * 2 * c->d_pad * c->n_local));
  }
  CU(cudaMalloc(&c->sum64, sizeof(double) * c->d_pad));
  CU(cudaMalloc(&c->mk_acc, sizeof(double)));
  c->peer_models.assign(c->world, nullptr);
  c->peer_ctl.assign(c->world, nullptr);
  c->peer_slots_off.assign(c->world, 0);
  c->peer_imported.assign(c->world, false);
  {
    int sms = 0;
    CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
    const int occ = engine_max_ctas_per_sm(c->engine_threads);
    const int cps = c->engine_cps > 0 ? std::min(c->engine_cps, occ) : std::min(2, occ);
    const int full = cps * sms;
    // in-process ranks may share one device: by default each takes 1/world of it
    // so that every rank's persistent engine is resident at once
    c->engine_grid = cfg->engine_grid > 0 ? std::min(full, (int)cfg->engine_grid)
                                          : ((c->comm_local && c->world > 1) ? std::max(1, full / c->world) : full);
    if (c->engine_grid > kMaxGrid) c->engine_grid = kMaxGrid;
  }
  c->peer_models[c->rank] = c->models;
  c->peer_ctl[c->rank] = c->ctl_arena;
  c->peer_slots_off[c->rank] = c->slots_offset;
  c->peer_imported[c->rank] = true;
  c->last_evt.assign(c->n, nullptr);
  for (auto& e : c->last_evt) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  c->step_ctr.assign(c->n, 0);
  c->epochs.assign(c->n, 0u);
  c->launches += 1;
  if (c->world == 1) {
    ST(upload_workers(c.get()));
    c->connected = true;
  }
  CU(cudaDeviceSynchronize());
  *out = c.release();
  return ADPSGD_OK;
}

}  // namespace

#define GUARD(...)                                                                    \
  try {                                                                               \
    __VA_ARGS__                                                                       \
  } catch (const std::bad_alloc&) {                                                   \
    return fail(ADPSGD_E_OOM, "host allocation failed");                              \
  } catch (...) {                                                                     \
    return fail(ADPSGD_E_INVALID, "internal exception");                              \
  }

// NVTX range over a public call (header-only NVTX 3: no cost unless a tool attaches)
struct NvtxScope {
  explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
  ~NvtxScope() { nvtxRangePop(); }
};

#define CTX_CHECK(c)                                                                  \
  NvtxScope nvtx_scope_(__func__);                                                    \
  if (!(c)) return fail(ADPSGD_E_INVALID, "null context");                           \
  CU(cudaSetDevice((c)->device));

extern "C" {

int32_t adpsgd_abi_version(void) { return ADPSGD_ABI_VERSION; }
const char* adpsgd_last_error(void) { return g_err.c_str(); }

adpsgd_status adpsgd_init(const adpsgd_graph* g, int32_t n_workers, int64_t d,
                          const adpsgd_config* cfg, adpsgd_ctx** out) {
  GUARD(return init_impl(g, n_workers, d, cfg, out);)
}

adpsgd_status adpsgd_destroy(adpsgd_ctx* ctx) { GUARD(return destroy_impl(ctx);) }

adpsgd_status adpsgd_peer_info_size(int64_t* bytes) {
  if (!bytes) return fail(ADPSGD_E_INVALID, "null");
  *bytes = (int64_t)sizeof(PeerBlob);
  return ADPSGD_OK;
}

adpsgd_status adpsgd_export_peer_info(adpsgd_ctx* c, void* buf, int64_t cap, int64_t* n_out) {
  GUARD({
    CTX_CHECK(c);
    if (!buf || cap < (int64_t)sizeof(PeerBlob)) return fail(ADPSGD_E_INVALID, "buffer too small");
    PeerBlob b{};
    b.magic = kBlobMagic;
    b.version = ADPSGD_ABI_VERSION;
    b.rank = c->rank;
    b.n_local = c->n_local;
    b.d_pad = c->d_pad;
    b.gctl_offset = (int64_t)c->gctl_offset;
    b.log_offset = (int64_t)c->log_offset;
    b.log_cap = c->log_cap;
    b.slots_offset = (int64_t)c->slots_offset;
    b.engine_grid = c->engine_grid;
    CU(cudaIpcGetMemHandle(&b.models, c->models));
    CU(cudaIpcGetMemHandle(&b.ctl, c->ctl_arena));
    b.local = c->comm_local ? 1 : 0;
    b.device = c->device;
    b.pid = (uint64_t)getpid();
    b.models_ptr = (uint64_t)(uintptr_t)c->models;
    b.ctl_ptr = (uint64_t)(uintptr_t)c->ctl_arena;
    memcpy(buf, &b, sizeof b);
    if (n_out) *n_out = (int64_t)sizeof b;
    return ADPSGD_OK;
  })
}

adpsgd_status adpsgd_import_peer_info(adpsgd_ctx* c, int32_t rank, const void* buf, int64_t n) {
  GUARD({
    CTX_CHECK(c);
    if (!buf || n < (int64_t)sizeof(PeerBlob) || rank < 0 || rank >= c->world)
      return fail(ADPSGD_E_INVALID, "bad peer blob");
    if (rank == c->rank) return ADPSGD_OK;
    PeerBlob b;
    memcpy(&b, buf, sizeof b);
    if (b.magic != kBlobMagic || b.rank != rank || b.d_pad != c->d_pad)
      return fail(ADPSGD_E_INVALID, "peer blob mismatch (magic/rank/d)");
    if (b.engine_grid != c->engine_grid)
      return fail(ADPSGD_E_UNSUPPORTED, "engine grid differs across ranks (different GPU models?)");
    if (c->comm_local) {
      // in-process rank: its memory is addressable here as is (same device, or a
      // peer device once peer access is enabled)
      if (!b.local || b.pid != (uint64_t)getpid())
        return fail(ADPSGD_E_INVALID, "comm_local: peer blob is not from an in-process rank");
      if (b.device != c->device) {
        cudaError_t pe = cudaDeviceEnablePeerAccess(b.device, 0);
        if (pe == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else if (pe != cudaSuccess)
          return fail(ADPSGD_E_UNSUPPORTED, std::string("peer access: ") + cudaGetErrorString(pe));
      }
      c->peer_models[rank] = reinterpret_cast<float*>((uintptr_t)b.models_ptr);
      c->peer_ctl[rank] = reinterpret_cast<char*>((uintptr_t)b.ctl_ptr);
      c->peer_slots_off[rank] = (size_t)b.slots_offset;
      c->peer_imported[rank] = true;
      if (rank == 0) {
        c->gctl0 = reinterpret_cast<GlobalCtl*>(c->peer_ctl[0] + b.gctl_offset);
        c->log0 = reinterpret_cast<LogEntry*>(c->peer_ctl[0] + b.log_offset);
        c->log_cap = b.log_cap;
      }
      return ADPSGD_OK;
    }
    if (b.local) return fail(ADPSGD_E_INVALID, "peer blob is from an in-process rank (set comm_local)");
    void* pm = nullptr;
    void* pc = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&pm, b.models, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess)
      return fail(ADPSGD_E_UNSUPPORTED, std::string("cannot map peer models over NVLink: ") + cudaGetErrorString(e));
    e = cudaIpcOpenMemHandle(&pc, b.ctl, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess)
      return fail(ADPSGD_E_UNSUPPORTED, std::string("cannot map peer control: ") + cudaGetErrorString(e));
    c->peer_models[rank] = static_cast<float*>(pm);
    c->peer_ctl[rank] = static_cast<char*>(pc);
    c->peer_slots_off[rank] = (size_t)b.slots_offset;
    c->peer_imported[rank] = true;
    if (rank == 0) {
      c->gctl0 = reinterpret_cast<GlobalCtl*>(c->peer_ctl[0] + b.gctl_offset);
      c->log0 = reinterpret_cast<LogEntry*>(c->peer_ctl[0] + b.log_offset);
      c->log_cap = b.log_cap;
    }
    return ADPSGD_OK;
  })
}

adpsgd_status adpsgd_nccl_unique_id(void* buf128) {
  if (!buf128) return fail(ADPSGD_E_INVALID, "null");
  ncclUniqueId id;
  NC(ncclGetUniqueId(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  memcpy(buf128, &id, sizeof id);
  return ADPSGD_OK;
}

adpsgd_status adpsgd_connect(adpsgd_ctx* c, const void* nccl_id) {
  GUARD({
    CTX_CHECK(c);
    for (int r = 0; r < c->world; ++r)
      if (!c->peer_imported[r]) return fail(ADPSGD_E_STATE, "peer info of some rank not imported");
    ST(upload_workers(c));
    if (c->world > 1) {
      if (!nccl_id) return fail(ADPSGD_E_INVALID, "nccl_id required when world_size > 1");
      if (c->comm_local) CO(make_local_comm(nccl_id, c->world, c->rank, c->device, &c->comm, m_));
      else CO(make_nccl_comm(nccl_id, c->world, c->rank, &c->comm, m_));
      // adpsgd_step's built-in gradient buffers, now rather than under another rank's lock wait
      if (c->model == ADPSGD_MODEL_LSQ || c->model == ADPSGD_MODEL_LOGREG || c->model == ADPSGD_MODEL_MLP) {
        if (!c->gstep) CU(cudaMalloc(&c->gstep, sizeof(float) * c->d_pad * std::max(1, c->n_local)));
        if (c->model == ADPSGD_MODEL_MLP) ST(ensure_mlp_scratch(c, 1));
      }
    }
    c->connected = true;
    return ADPSGD_OK;
  })
}

static adpsgd_status step_multi(adpsgd_ctx* c, int w, const float* grad, adpsgd_stream s, int64_t* ticket_out,
                                int gossip_j);

adpsgd_status adpsgd_gossip(adpsgd_ctx* c, int32_t i, int32_t j, adpsgd_stream s) {
  GUARD({
    CTX_CHECK(c);
    if (i < 0 || j < 0 || i >= c->n || j >= c->n || i == j) return fail(ADPSGD_E_INVALID, "i/j");
    if (!is_neighbour(c, i, j)) return fail(ADPSGD_E_NOT_NEIGHBOURS, "not an edge");
    if (c->role[i] == c->role[j]) return fail(ADPSGD_E_NOT_BIPARTITE, "gossip pairs two workers of the same role");
    // a pure average is an event of the log like any other (reading R23): it
    // takes the next ticket k and is logged with NO_GRAD, so the event log
    // replays every change of X; the paper's k (gradient updates) is
    // the subsequence of events without NO_GRAD
    if (c->world > 1) {
      if (!c->is_local(i)) return fail(ADPSGD_E_INVALID, "adpsgd_gossip: worker i must live on this rank");
      return step_multi(c, i, nullptr, s, nullptr, j);
    }
    std::lock_guard<std::mutex> lk(c->mu);
    unsigned long long k;
    ST(host_ticket(c, &k));
    cudaStream_t st = c->use(s);
    CU(cudaStreamWaitEvent(st, c->last_evt[i], 0));
    CU(cudaStreamWaitEvent(st, c->last_evt[j], 0));
    CU(launch_event(c->row(i), c->row(j), nullptr, nullptr, c->d, c->n4, c->gamma, c->q, 0, kGradNone, st));
    CU(launch_step_commit(c->gctl0, c->ctl + c->worker_local[i], c->log0, c->log_cap, (long long)k, i, j,
                          ADPSGD_EV_NO_GRAD, 0, st));
    c->launches += 2;
    CU(cudaEventRecord(c->last_evt[i], st));
    CU(cudaEventRecord(c->last_evt[j], st));
    c->host_k = k + 1;
    return ADPSGD_OK;
  })
}

// adpsgd_step at world_size > 1: the passive side's lock (the partner's when w
// is active, w's own when it steps alone) and the ticket k are taken on the
// device -- the lock may live on a peer GPU and other ranks step concurrently --
// k is read back (a built-in gradient's draws are keyed by k), then gradient,
// fused pass over NVLink, and a commit kernel that logs and unlocks.
// gossip_j >= 0: adpsgd_gossip(w, gossip_j) -- the pair average alone, a NO_GRAD event.
static adpsgd_status step_multi(adpsgd_ctx* c, int w, const float* grad, adpsgd_stream s, int64_t* ticket_out,
                                int gossip_j) {
  if (!c->connected) return fail(ADPSGD_E_STATE, "not connected");
  if (!c->is_local(w)) return fail(ADPSGD_E_INVALID, "adpsgd_step: worker w must live on this rank");
  std::lock_guard<std::mutex> lk(c->mu);
  const bool gossip = gossip_j >= 0;
  int j = gossip ? gossip_j : -1;
  if (!gossip && c->role[w] == 0 && !c->nb[w].empty()) {
    uint64_t st = c->seed ^ (0x9E3779B97F4A7C15ull * (uint64_t)(w + 1)) ^ (c->step_ctr[w]++ << 20);
    const uint64_t r = splitmix64(st);
    j = c->nb[w][(size_t)((r >> 32) * c->nb[w].size() >> 32)];
  }
  auto ctl_of = [&](int v) {
    return reinterpret_cast<WorkerCtl*>(c->peer_ctl[c->worker_rank[v]]) + c->worker_local[v];
  };
  auto row_of = [&](int v) {
    return c->peer_models[c->worker_rank[v]] + (long long)c->worker_local[v] * c->d_pad;
  };
  // every buffer was allocated at connect: nothing here may synchronise the device (which
  // would wait for a peer's lock kernel spinning on a lock whose release this thread launches)
  if (!gossip && !grad && c->model != ADPSGD_MODEL_QUADRATIC && !c->gstep)
    return fail(ADPSGD_E_STATE, "adpsgd_step: gradient buffers missing (allocated by adpsgd_connect)");
  cudaStream_t st = c->use(s);
  // rows of local workers stay ordered with this context's other streams (as
  // the single-GPU adpsgd_step / adpsgd_gossip order them)
  const bool j_local = j >= 0 && c->is_local(j);
  CU(cudaStreamWaitEvent(st, c->last_evt[w], 0));
  if (j_local) CU(cudaStreamWaitEvent(st, c->last_evt[j], 0));
  // the passive endpoint's lock (bipartite order): the partner of an
  // active, or the worker itself when it is passive (a local step, or a gossip
  // call naming the passive first)
  unsigned int* lock = &ctl_of((j >= 0 && c->role[w] == 0) ? j : w)->lock;
  CU(launch_super_lock(lock, &c->gctl0->ticket, c->super_k, &c->gctl->error, 20ull * 1000000000ull, st));
  CU(cudaMemcpyAsync(c->k_host, c->super_k, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  const unsigned long long k = *c->k_host;
  if (k == ~0ull) return fail(ADPSGD_E_TIMEOUT, "adpsgd_step: lock wait exceeded the watchdog");
  int mode = gossip ? kGradNone : kGradExternal;
  const float* g = grad;
  if (!gossip && !grad) {
    if (c->model == ADPSGD_MODEL_QUADRATIC) {
      mode = kGradQuadInline;
    } else {
      float* gb = c->gstep + (long long)c->worker_local[w] * c->d_pad;
      ST(model_grad(c, c->row(w), gb, k, nullptr, st));
      g = gb;
    }
  }
  CU(launch_event(c->row(w), j >= 0 ? row_of(j) : nullptr, g, nullptr, c->d, c->n4, c->gamma, c->q, k, mode, st));
  CU(launch_super_commit(c->log0, c->log_cap, c->super_k, w, j, gossip ? (unsigned)ADPSGD_EV_NO_GRAD : 0u,
                         c->ctl + c->worker_local[w], &c->gctl0->committed, lock, st));
  CU(cudaEventRecord(c->last_evt[w], st));
  if (j_local) CU(cudaEventRecord(c->last_evt[j], st));
  c->launches += 3;
  c->ticket_dirty = true;                 // other ranks move the counter too: re-read before the next run
  if (ticket_out) *ticket_out = (int64_t)k;
  return ADPSGD_OK;
}

adpsgd_status adpsgd_step(adpsgd_ctx* c, int32_t w, const float* grad, adpsgd_stream s,
                          int64_t* ticket_out) {
  GUARD({
    CTX_CHECK(c);
    if (w < 0 || w >= c->n) return fail(ADPSGD_E_INVALID, "worker");
    if (!grad && (c->model == ADPSGD_MODEL_NONE || c->model == ADPSGD_MODEL_EXTERNAL))
      return fail(ADPSGD_E_INVALID, "no gradient: pass grad or configure a built-in model");
    if (c->world > 1) return step_multi(c, w, grad, s, ticket_out, -1);
    std::lock_guard<std::mutex> lk(c->mu);
    int j = -1;
    if (c->role[w] == 0 && !c->nb[w].empty()) {
      uint64_t st = c->seed ^ (0x9E3779B97F4A7C15ull * (uint64_t)(w + 1)) ^ (c->step_ctr[w]++ << 20);
      const uint64_t r = splitmix64(st);
      j = c->nb[w][(size_t)((r >> 32) * c->nb[w].size() >> 32)];
    }
    unsigned long long k;
    ST(host_ticket(c, &k));
    cudaStream_t st = c->use(s);
    CU(cudaStreamWaitEvent(st, c->last_evt[w], 0));
    if (j >= 0) CU(cudaStreamWaitEvent(st, c->last_evt[j], 0));
    int mode = kGradExternal;
    const float* g = grad;
    if (!grad) {
      if (c->model == ADPSGD_MODEL_QUADRATIC) mode = kGradQuadInline;
      else {
        if (!c->gstep) CU(cudaMalloc(&c->gstep, sizeof(float) * c->d_pad * std::max(1, c->n_local)));
        float* gb = c->gstep + (long long)c->worker_local[w] * c->d_pad;
        ST(model_grad(c, c->row(w), gb, k, nullptr, st));
        g = gb;
      }
    }
    CU(launch_event(c->row(w), j >= 0 ? c->row(j) : nullptr, g, nullptr, c->d, c->n4, c->gamma, c->q,
                    k, mode, st));
    CU(launch_step_commit(c->gctl0, c->ctl + c->worker_local[w], c->log0, c->log_cap, (long long)k, w, j,
                          0u, 1, st));
    c->launches += 2;
    CU(cudaEventRecord(c->last_evt[w], st));
    if (j >= 0) CU(cudaEventRecord(c->last_evt[j], st));
    c->host_k = k + 1;
    if (ticket_out) *ticket_out = (int64_t)k;
    return ADPSGD_OK;
  })
}

adpsgd_status adpsgd_replay(adpsgd_ctx* c, const adpsgd_event* ev, int64_t K, const int32_t* bidx,
                            uint32_t flags, adpsgd_stream s) {
  GUARD({
    CTX_CHECK(c);
    if (K < 0 || (K > 0 && !ev)) return fail(ADPSGD_E_INVALID, "schedule");
    if (!c->connected) return fail(ADPSGD_E_STATE, "not connected");
    if (K == 0) return ADPSGD_OK;
    const bool engine = (flags & ADPSGD_REPLAY_ENGINE) || (!(flags & ADPSGD_REPLAY_HOST) && c->world > 1);
    std::lock_guard<std::mutex> lk(c->mu);
    if (engine) return replay_engine(c, ev, K, c->use(s));
    return replay_host(c, ev, K, bidx, c->use(s));
  })
}

adpsgd_status adpsgd_run(adpsgd_ctx* c, int64_t n_updates, adpsgd_stream s) {
  GUARD({
    CTX_CHECK(c);
    if (!c->connected) return fail(ADPSGD_E_STATE, "not connected");
    if (c->model != ADPSGD_MODEL_NONE && c->model != ADPSGD_MODEL_QUADRATIC)
      return fail(ADPSGD_E_UNSUPPORTED, "free-running engine supports models NONE and QUADRATIC");
    if (n_updates < 0) return fail(ADPSGD_E_INVALID, "n_updates");
    std::lock_guard<std::mutex> lk(c->mu);
    // the run ends with the ticket at exactly k0 + n_updates on every rank
    ST(settle_ticket(c));
    const unsigned long long k0 = c->host_k;
    cudaStream_t st = c->use(s);
    ST(reset_slots(c, st));
    ST(engine_launch(c, 0, k0 + (unsigned long long)n_updates, st));
    c->host_k = k0 + (unsigned long long)n_updates;
    return ADPSGD_OK;
  })
}

adpsgd_status adpsgd_consensus_mean(adpsgd_ctx* c, float* out, double* mk_out, adpsgd_stream s) {
  GUARD({
    CTX_CHECK(c);
    if (!out) return fail(ADPSGD_E_INVALID, "out");
    if (!c->connected) return fail(ADPSGD_E_STATE, "not connected");
    cudaStream_t st = c->use(s);
    // quiesce: every rank's engine (and its P2P stores into our rows) has
    // finished once this tiny all-reduce completes on our stream
    if (c->world == 1) {               // one pass over the rows: x_bar (+ M_k)
      if (mk_out) CU(cudaMemsetAsync(c->mk_acc, 0, sizeof(double), st));
      CU(launch_consensus_fused(c->models, c->n_local, c->d_pad, c->d, c->n, out, mk_out ? c->mk_acc : nullptr,
                                &c->gctl->error, st));
      ++c->launches;
      if (mk_out) {
        double acc = 0.0;
        CU(cudaMemcpyAsync(&acc, c->mk_acc, sizeof(double), cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        if (!std::isfinite(acc)) {
          char buf[96];
          snprintf(buf, sizeof buf, "non-finite model value at the consensus after event %llu (S:289)",
                   (unsigned long long)c->host_k);
          return fail(ADPSGD_E_DIVERGED, buf);
        }
        *mk_out = acc / (double)c->n;
      }
      return ADPSGD_OK;
    }
    if (c->world > 1) CO(c->comm->allreduce(c->mk_acc, c->mk_acc, 1, DType::F64, ROp::Sum, st, m_));
    CU(launch_consensus_sum(c->models, c->n_local, c->d_pad, c->d, c->sum64, st));
    ++c->launches;
    if (c->world > 1) CO(c->comm->allreduce(c->sum64, c->sum64, (size_t)c->d, DType::F64, ROp::Sum, st, m_));
    CU(launch_consensus_finalize(c->sum64, c->n, c->d, out, &c->gctl->error, st));
    ++c->launches;
    if (mk_out) {
      CU(cudaMemsetAsync(c->mk_acc, 0, sizeof(double), st));
      CU(launch_consensus_mk(c->models, c->n_local, c->d_pad, c->d, c->sum64, c->n, c->mk_acc, st));
      ++c->launches;
      if (c->world > 1) CO(c->comm->allreduce(c->mk_acc, c->mk_acc, 1, DType::F64, ROp::Sum, st, m_));
      double acc = 0.0;
      CU(cudaMemcpyAsync(&acc, c->mk_acc, sizeof(double), cudaMemcpyDeviceToHost, st));
      CU(cudaStreamSynchronize(st));
      if (!std::isfinite(acc)) {
        char buf[96];
        snprintf(buf, sizeof buf, "non-finite model value at the consensus after event %llu (S:289)",
                 (unsigned long long)c->host_k);
        return fail(ADPSGD_E_DIVERGED, buf);
      }
      *mk_out = acc / (double)c->n;
    }
    return ADPSGD_OK;
  })
}

adpsgd_status adpsgd_allreduce_reset(adpsgd_ctx* c, const float* host_x) {
  GUARD({
    CTX_CHECK(c);
    if (!c->xr) {
      CU(cudaMalloc(&c->xr, sizeof(float) * c->d_pad));
      CU(cudaMalloc(&c->gsum, sizeof(float) * c->d_pad));
    }
    CU(cudaDeviceSynchronize());
    CU(cudaMemcpy(c->xr, c->dx0, sizeof(float) * c->d_pad, cudaMemcpyDeviceToDevice));
    if (host_x) CU(cudaMemcpy(c->xr, host_x, sizeof(float) * c->d, cudaMemcpyHostToDevice));
    CU(cudaDeviceSynchronize());
    c->ar_k = 0;
    return ADPSGD_OK;
  })
}

adpsgd_status adpsgd_allreduce_sgd(adpsgd_ctx* c, int64_t n_rounds, adpsgd_stream s) {
  GUARD({
    CTX_CHECK(c);
    if (c->model != ADPSGD_MODEL_QUADRATIC) return fail(ADPSGD_E_UNSUPPORTED, "baseline uses the quadratic");
    if (!c->connected) return fail(ADPSGD_E_STATE, "not connected");
    if (!c->xr) ST(adpsgd_allreduce_reset(c, nullptr));
    cudaStream_t st = c->use(s);
    float smax = 1.0f;
    for (int w : c->local_ids) smax = std::max(smax, c->straggle[w]);
    // slow link (R21): a ring all-reduce moves ~2 models over every link per
    // round, so the round waits 2 (L_max - 1) link_ns for its slowest link
    const unsigned long long delay = (unsigned long long)((double)smax * (double)c->compute_ns) +
                                     (unsigned long long)(2.0 * ((double)c->link_max() - 1.0) * (double)c->link_ns);
    for (int64_t r = 0; r < n_rounds; ++r) {
      if (delay) { CU(launch_delay(delay, st)); ++c->launches; }
      CU(launch_ar_grad_sum(c->xr, c->gsum, c->d, c->n4, c->q, c->ar_k, c->n_local, c->d_local_ids, st));
      if (c->world > 1)
        CO(c->comm->allreduce(c->gsum, c->gsum, (size_t)c->d_pad, DType::F32, ROp::Sum, st, m_));
      CU(launch_ar_update(c->xr, c->gsum, c->gamma, c->n, c->d, c->n4, st));
      c->launches += 2;
      c->ar_k += (unsigned long long)c->n;
    }
    return ADPSGD_OK;
  })
}

adpsgd_status adpsgd_allreduce_read_model(adpsgd_ctx* c, float* host_out) {
  GUARD({
    CTX_CHECK(c);
    if (!host_out || !c->xr) return fail(ADPSGD_E_STATE, "no baseline replica");
    CU(cudaStreamSynchronize(c->stream));
    CU(cudaDeviceSynchronize());
    CU(cudaMemcpy(host_out, c->xr, sizeof(float) * c->d, cudaMemcpyDeviceToHost));
    return ADPSGD_OK;
  })
}

static adpsgd_status dpsgd_setup(adpsgd_ctx* c) {
  if (c->dp_x[0]) return ADPSGD_OK;
  const size_t rows = (size_t)std::max(1, c->n_local);
  CU(cudaMalloc(&c->dp_x[0], sizeof(float) * c->d_pad * rows));
  CU(cudaMalloc(&c->dp_x[1], sizeof(float) * c->d_pad * rows));
  int dmax = 0;
  for (int w = 0; w < c->n; ++w) dmax = std::max(dmax, (int)c->nb[w].size());
  if (dmax > kDpMaxDeg) return fail(ADPSGD_E_UNSUPPORTED, "D-PSGD baseline supports degree <= 16");
  c->dp_wnb = (float)(1.0 / (double)(dmax + 1));
  // halo: remote neighbours of local workers (received), local workers needed remotely (sent)
  std::vector<char> need(c->n, 0);
  std::vector<std::vector<char>> sendto(c->n, std::vector<char>(c->world, 0));
  for (int w : c->local_ids)
    for (int j : c->nb[w])
      if (!c->is_local(j)) need[j] = 1;
  for (int w = 0; w < c->n; ++w)
    if (!c->is_local(w))
      for (int j : c->nb[w])
        if (c->is_local(j)) sendto[j][c->worker_rank[w]] = 1;
  c->dp_halo_w.clear();
  c->dp_send.clear();
  std::vector<int> halo_idx(c->n, -1);
  for (int w = 0; w < c->n; ++w) {
    if (need[w]) { halo_idx[w] = (int)c->dp_halo_w.size(); c->dp_halo_w.push_back(w); }
    if (c->is_local(w))
      for (int r = 0; r < c->world; ++r)
        if (sendto[w][r]) c->dp_send.emplace_back(w, r);
  }
  if (!c->dp_halo_w.empty()) CU(cudaMalloc(&c->dp_halo, sizeof(float) * c->d_pad * c->dp_halo_w.size()));
  std::vector<int> deg(rows, 0);
  std::vector<float> wself(rows, 1.f);
  for (int par = 0; par < 2; ++par) {
    std::vector<const float*> tab(rows * kDpMaxDeg, nullptr);
    for (int l = 0; l < c->n_local; ++l) {
      const int w = c->local_ids[l];
      deg[l] = (int)c->nb[w].size();
      wself[l] = (float)(1.0 - (double)deg[l] / (double)(dmax + 1));
      for (int t = 0; t < deg[l]; ++t) {            // ascending neighbour order (c->nb is sorted)
        const int j = c->nb[w][t];
        tab[l * kDpMaxDeg + t] = c->is_local(j) ? c->dp_x[par] + (long long)c->worker_local[j] * c->d_pad
                                                : c->dp_halo + (long long)halo_idx[j] * c->d_pad;
      }
    }
    CU(cudaMalloc(&c->d_dp_nbr[par], sizeof(const float*) * tab.size()));
    CU(cudaMemcpy(c->d_dp_nbr[par], tab.data(), sizeof(const float*) * tab.size(), cudaMemcpyHostToDevice));
  }
  CU(cudaMalloc(&c->d_dp_deg, sizeof(int) * rows));
  CU(cudaMemcpy(c->d_dp_deg, deg.data(), sizeof(int) * rows, cudaMemcpyHostToDevice));
  CU(cudaMalloc(&c->d_dp_wself, sizeof(float) * rows));
  CU(cudaMemcpy(c->d_dp_wself, wself.data(), sizeof(float) * rows, cudaMemcpyHostToDevice));
  CU(cudaDeviceSynchronize());
  return ADPSGD_OK;
}

adpsgd_status adpsgd_dpsgd_reset(adpsgd_ctx* c, const float* x0_per_worker) {
  GUARD({
    CTX_CHECK(c);
    if (c->model != ADPSGD_MODEL_QUADRATIC && c->model != ADPSGD_MODEL_NONE)
      return fail(ADPSGD_E_UNSUPPORTED, "D-PSGD baseline uses the quadratic (or no gradient)");
    ST(dpsgd_setup(c));
    CU(cudaDeviceSynchronize());
    for (int l = 0; l < c->n_local; ++l) {
      float* row = c->dp_x[0] + (long long)l * c->d_pad;
      CU(cudaMemcpy(row, c->dx0, sizeof(float) * c->d_pad, cudaMemcpyDeviceToDevice));
      if (x0_per_worker)
        CU(cudaMemcpy(row, x0_per_worker + (long long)c->local_ids[l] * c->d, sizeof(float) * c->d,
                      cudaMemcpyHostToDevice));
    }
    CU(cudaDeviceSynchronize());
    c->dp_cur = 0;
    c->dp_k = 0;
    return ADPSGD_OK;
  })
}

adpsgd_status adpsgd_dpsgd(adpsgd_ctx* c, int64_t n_rounds, adpsgd_stream s) {
  GUARD({
    CTX_CHECK(c);
    if (!c->connected) return fail(ADPSGD_E_STATE, "not connected");
    if (!c->dp_x[0]) ST(adpsgd_dpsgd_reset(c, nullptr));
    cudaStream_t st = c->use(s);
    float smax = 1.0f;
    for (int w : c->local_ids) smax = std::max(smax, c->straggle[w]);
    // slow link (R21): every worker exchanges one model with each neighbour per
    // round (in parallel, full duplex), so the round waits (L_max - 1) link_ns
    const unsigned long long delay = (unsigned long long)((double)smax * (double)c->compute_ns) +
                                     (unsigned long long)(((double)c->link_max() - 1.0) * (double)c->link_ns);
    const int model = c->model == ADPSGD_MODEL_QUADRATIC ? 1 : 0;
    for (int64_t r = 0; r < n_rounds; ++r) {
      if (delay) { CU(launch_delay(delay, st)); ++c->launches; }     // the round waits for its slowest worker
      float* xin = c->dp_x[c->dp_cur];
      if (c->world > 1) {                                            // halo exchange (synchronous round)
        std::vector<P2POp> sends, recvs;
        for (size_t h = 0; h < c->dp_halo_w.size(); ++h)
          recvs.push_back({c->dp_halo + (long long)h * c->d_pad, (size_t)c->d_pad, c->worker_rank[c->dp_halo_w[h]]});
        for (auto& ps : c->dp_send)
          sends.push_back({xin + (long long)c->worker_local[ps.first] * c->d_pad, (size_t)c->d_pad, ps.second});
        CO(c->comm->exchange(sends, recvs, st, m_));
      }
      if (c->n_local) {
        CU(launch_dpsgd(c->d_dp_nbr[c->dp_cur], c->d_dp_deg, c->d_dp_wself, c->dp_wnb, xin, c->dp_x[1 - c->dp_cur],
                        c->n_local, c->d_pad, c->d, c->q, model, c->gamma, c->dp_k, c->d_local_ids, st));
        ++c->launches;
      }
      c->dp_cur ^= 1;
      c->dp_k += (unsigned long long)c->n;
    }
    return ADPSGD_OK;
  })
}

adpsgd_status adpsgd_dpsgd_read_model(adpsgd_ctx* c, int32_t w, float* host_out) {
  GUARD({
    CTX_CHECK(c);
    if (w < 0 || w >= c->n || !host_out || !c->is_local(w) || !c->dp_x[0])
      return fail(ADPSGD_E_INVALID, "worker / no D-PSGD state");
    CU(cudaDeviceSynchronize());
    CU(cudaMemcpy(host_out, c->dp_x[c->dp_cur] + (long long)c->worker_local[w] * c->d_pad, sizeof(float) * c->d,
                  cudaMemcpyDeviceToHost));
    return ADPSGD_OK;
  })
}

// --------------------------------------------------------- super-learner --
// P:952-956, reading R22.  Learner w lives on rank w (explicit placement); the
// learner graph is R copies of the super-learners' graph, learner (s, r) = s*R + r.
static adpsgd_status super_setup(adpsgd_ctx* c) {
  const int R = c->super_R > 1 ? c->super_R : 1;
  if (c->world % R || c->n != c->world) return fail(ADPSGD_E_INVALID, "super_run: n == world_size, super_R | world");
  for (int w = 0; w < c->n; ++w)
    if (c->worker_rank[w] != w) return fail(ADPSGD_E_INVALID, "super_run: learner w must live on rank w");
  const int S = c->n / R;
  c->super_nb.assign(S, {});
  for (int w = 0; w < c->n; ++w) {
    const int s = w / R, r = w % R;
    if (c->role[w] != c->role[s * R]) return fail(ADPSGD_E_INVALID, "super_run: a super-learner's learners differ in role");
    std::vector<int> nb;
    for (int v : c->nb[w]) {
      if (v % R != r) return fail(ADPSGD_E_INVALID, "super_run: learner (s, r) may only neighbour learners (s', r)");
      nb.push_back(v / R);
    }
    std::sort(nb.begin(), nb.end());
    if (r == 0) c->super_nb[s] = nb;
    else if (nb != c->super_nb[s]) return fail(ADPSGD_E_INVALID, "super_run: learner graphs differ across r");
  }
  if (R > 1 && !c->super_comm) CO(c->comm->split(c->rank / R, c->rank % R, &c->super_comm, m_));
  if (!c->super_g) {
    CU(cudaMalloc(&c->super_g, sizeof(float) * c->d_pad));
    // MLP scratch now: its first allocation synchronises the device, which must
    // not happen under a lock (in-process ranks share the device with the
    // lock kernels spinning on it)
    if (c->model == ADPSGD_MODEL_MLP) ST(ensure_mlp_scratch(c, 1));
    CU(cudaMalloc(&c->super_bar, sizeof(int)));
    CU(cudaMemset(c->super_bar, 0, sizeof(int)));
    CU(cudaDeviceSynchronize());
  }
  return ADPSGD_OK;
}

static uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

adpsgd_status adpsgd_super_run(adpsgd_ctx* c, int64_t n_steps, adpsgd_stream strm) {
  GUARD({
    CTX_CHECK(c);
    if (!c->connected) return fail(ADPSGD_E_STATE, "not connected");
    if (c->model == ADPSGD_MODEL_NONE || c->model == ADPSGD_MODEL_EXTERNAL)
      return fail(ADPSGD_E_UNSUPPORTED, "super_run needs a built-in model (quadratic, lsq, logreg, mlp)");
    if (n_steps < 0) return fail(ADPSGD_E_INVALID, "n_steps < 0");
    ST(super_setup(c));
    ST(settle_ticket(c));
    const int R = c->super_R > 1 ? c->super_R : 1;
    cudaStream_t st = c->use(strm);
    const int w = c->rank, s = w / R, r = w % R, S = c->n / R;
    const bool active = c->role[w] == 0 && !c->super_nb[s].empty();
    float* row = c->row(w);
    auto ctl_of = [&](int v) { return reinterpret_cast<WorkerCtl*>(c->peer_ctl[v]) + c->worker_local[v]; };
    auto row_of = [&](int v) { return c->peer_models[v] + (long long)c->worker_local[v] * c->d_pad; };
    const unsigned long long watchdog = 20ull * 1000000000ull;
    for (int64_t step = 0; step < n_steps; ++step) {
      const long long cs = c->super_c;
      const unsigned long long key = (1ull << 61) | ((unsigned long long)s << 44) | ((unsigned long long)cs << 8) |
                                     (unsigned long long)r;
      int js = -1;
      if (active) {                     // the group's shared neighbour choice (uniform over N(s))
        const auto& nb = c->super_nb[s];
        js = nb[splitmix64(c->seed ^ ((uint64_t)s << 40) ^ (uint64_t)cs) % nb.size()];
      }
      unsigned int* lock = &ctl_of((active ? js : s) * R)->lock;   // the passive side's leader lock
      auto gradient = [&]() -> adpsgd_status {   // learner r's minibatch gradient (device Philox batches)
        ST(model_grad(c, row, c->super_g, key, nullptr, st));
        if (R > 1) CO(c->super_comm->allreduce(c->super_g, c->super_g, (size_t)c->d_pad, DType::F32, ROp::Sum, st, m_));
        return ADPSGD_OK;
      };
      auto lock_and_share_k = [&]() -> adpsgd_status {
        if (r == 0) {
          CU(launch_super_lock(lock, &c->gctl0->ticket, c->super_k, &c->gctl->error, watchdog, st));
          // in-process ranks share the device's hardware queues: nothing that
          // depends on a spinning lock kernel may be queued behind it, where it
          // could block the release another rank has queued (as step_multi does)
          if (c->comm_local) CU(cudaStreamSynchronize(st));
        }
        if (R > 1) CO(c->super_comm->broadcast(c->super_k, 1, DType::U64, 0, st, m_));
        return ADPSGD_OK;
      };
      if (active) {                     // gradient first: x_s changes only through s's own events
        ST(gradient());
        ST(lock_and_share_k());
        CU(launch_event(row, row_of(js * R + r), c->super_g, nullptr, c->d, c->n4, c->gamma, c->q, 0, kGradExternal, st,
                        c->super_k));   // skipped if the leader's lock wait timed out
      } else {                          // a passive reads its model under its own lock
        ST(lock_and_share_k());
        ST(gradient());
        CU(launch_event(row, nullptr, c->super_g, nullptr, c->d, c->n4, c->gamma, c->q, 0, kGradExternal, st, c->super_k));
      }
      if (R > 1) CO(c->super_comm->allreduce(c->super_bar, c->super_bar, 1, DType::I32, ROp::Sum, st, m_));
      if (r == 0)
        CU(launch_super_commit(c->log0, c->log_cap, c->super_k, s, js, 0u, ctl_of(s * R), &c->gctl0->committed, lock,
                               st));
      c->launches += 3;                 // lock, event, commit (model_grad counts its own)
      c->super_c += 1;
    }
    c->host_k += (unsigned long long)S * (unsigned long long)n_steps;
    return ADPSGD_OK;
  })
}

adpsgd_status adpsgd_sync(adpsgd_ctx* c) {
  GUARD({
    CTX_CHECK(c);
    CU(cudaDeviceSynchronize());
    unsigned int err = 0;
    CU(cudaMemcpy(&err, &c->gctl->error, sizeof err, cudaMemcpyDeviceToHost));
    if (err) {
      CU(cudaMemset(&c->gctl->error, 0, sizeof err));
      CU(cudaDeviceSynchronize());
      return fail((adpsgd_status)err, "device-side error latched (e.g. watchdog timeout)");
    }
    return ADPSGD_OK;
  })
}

adpsgd_status adpsgd_read_model(adpsgd_ctx* c, int32_t w, float* host_out) {
  GUARD({
    CTX_CHECK(c);
    if (w < 0 || w >= c->n || !host_out) return fail(ADPSGD_E_INVALID, "worker/out");
    if (!c->is_local(w)) return fail(ADPSGD_E_INVALID, "worker not local to this rank");
    CU(cudaDeviceSynchronize());
    CU(cudaMemcpy(host_out, c->row(w), sizeof(float) * c->d, cudaMemcpyDeviceToHost));
    return ADPSGD_OK;
  })
}

adpsgd_status adpsgd_write_model(adpsgd_ctx* c, int32_t w, const float* host_in) {
  GUARD({
    CTX_CHECK(c);
    if (w < 0 || w >= c->n || !host_in) return fail(ADPSGD_E_INVALID, "worker/in");
    if (!c->is_local(w)) return fail(ADPSGD_E_INVALID, "worker not local to this rank");
    CU(cudaDeviceSynchronize());
    CU(cudaMemcpy(c->row(w), host_in, sizeof(float) * c->d, cudaMemcpyHostToDevice));
    CU(cudaDeviceSynchronize());
    return ADPSGD_OK;
  })
}

adpsgd_status adpsgd_model_device_ptr(adpsgd_ctx* c, int32_t w, float** p) {
  if (!c || !p || w < 0 || w >= c->n || !c->is_local(w)) return fail(ADPSGD_E_INVALID, "worker");
  *p = c->row(w);
  return ADPSGD_OK;
}

adpsgd_status adpsgd_worker_rank(adpsgd_ctx* c, int32_t w, int32_t* r) {
  if (!c || !r || w < 0 || w >= c->n) return fail(ADPSGD_E_INVALID, "worker");
  *r = c->worker_rank[w];
  return ADPSGD_OK;
}

adpsgd_status adpsgd_get_ticket(adpsgd_ctx* c, int64_t* k) {
  GUARD({
    CTX_CHECK(c);
    if (!k || !c->gctl0) return fail(ADPSGD_E_STATE, "not connected");
    unsigned long long v;
    ST(read_ticket(c, &v));
    *k = (int64_t)v;
    return ADPSGD_OK;
  })
}

adpsgd_status adpsgd_read_log(adpsgd_ctx* c, int64_t k_from, adpsgd_log_entry* out, int64_t cap,
                              int64_t* n_out) {
  GUARD({
    CTX_CHECK(c);
    if (!out || cap < 0 || k_from < 0 || !c->log0) return fail(ADPSGD_E_INVALID, "args / no log");
    unsigned long long kt;
    ST(read_ticket(c, &kt));
    long long avail = (long long)kt - k_from;
    if (avail < 0) avail = 0;
    long long n = std::min<long long>(std::min<long long>(avail, cap), c->log_cap);
    for (long long t = 0; t < n;) {
      const long long pos = (k_from + t) % c->log_cap;
      const long long run = std::min(n - t, c->log_cap - pos);
      CU(cudaMemcpy(out + t, c->log0 + pos, sizeof(LogEntry) * run, cudaMemcpyDeviceToHost));
      t += run;
    }
    if (n_out) *n_out = n;
    return ADPSGD_OK;
  })
}

adpsgd_status adpsgd_read_update_counts(adpsgd_ctx* c, int64_t* out_n) {
  GUARD({
    CTX_CHECK(c);
    if (!out_n) return fail(ADPSGD_E_INVALID, "out");
    CU(cudaDeviceSynchronize());
    std::vector<WorkerCtl> h(std::max(1, c->n_local));
    CU(cudaMemcpy(h.data(), c->ctl, sizeof(WorkerCtl) * c->n_local, cudaMemcpyDeviceToHost));
    for (int l = 0; l < c->n_local; ++l) out_n[l] = (int64_t)h[l].updates;
    return ADPSGD_OK;
  })
}

adpsgd_status adpsgd_get_stats(adpsgd_ctx* c, adpsgd_stats* o) {
  GUARD({
    CTX_CHECK(c);
    if (!o) return fail(ADPSGD_E_INVALID, "out");
    CU(cudaDeviceSynchronize());
    GlobalCtl g;
    CU(cudaMemcpy(&g, c->gctl, sizeof g, cudaMemcpyDeviceToHost));
    unsigned long long kt = 0;
    if (c->gctl0) CU(cudaMemcpy(&kt, &c->gctl0->ticket, sizeof kt, cudaMemcpyDeviceToHost));
    o->ticket = (int64_t)kt;
    o->local_events = (int64_t)g.st_events;
    o->local_pair_events = (int64_t)g.st_pair;
    o->local_cross_events = (int64_t)g.st_cross;
    o->local_bytes = g.st_bytes;
    if (c->n_local > 0) {                  // this GPU's share of cross pairs committed by peers
      std::vector<WorkerCtl> h(c->n_local);
      CU(cudaMemcpy(h.data(), c->ctl, sizeof(WorkerCtl) * c->n_local, cudaMemcpyDeviceToHost));
      for (const WorkerCtl& w : h) o->local_bytes += w.peer_bytes;
    }
    o->local_nvlink_bytes = g.st_nvl_bytes;
    o->engine_busy_ns = (double)g.st_busy_ns;
    o->engine_busy_cross_ns = (double)g.st_busy_cross_ns;
    return ADPSGD_OK;
  })
}

adpsgd_status adpsgd_reset_stats(adpsgd_ctx* c) {
  GUARD({
    CTX_CHECK(c);
    CU(cudaDeviceSynchronize());
    // zero the statistics fields only: ticket, committed, error and abort_flag
    // live in the same struct and peers may advance rank 0's ticket / committed
    // (system-scope atomics over NVLink) at any time
    char* base = reinterpret_cast<char*>(c->gctl);
    CU(cudaMemset(base + offsetof(GlobalCtl, st_events), 0,
                  offsetof(GlobalCtl, abort_flag) - offsetof(GlobalCtl, st_events)));
    CU(cudaMemset(base + offsetof(GlobalCtl, st_busy_cross_ns), 0, sizeof(unsigned long long)));
    for (int l = 0; l < c->n_local; ++l) CU(cudaMemset(&c->ctl[l].peer_bytes, 0, sizeof(double)));
    CU(cudaDeviceSynchronize());
    return ADPSGD_OK;
  })
}

adpsgd_status adpsgd_launch_count(adpsgd_ctx* c, int64_t* out) {
  if (!c || !out) return fail(ADPSGD_E_INVALID, "null");
  *out = c->launches;
  return ADPSGD_OK;
}

adpsgd_status adpsgd_plan_placement(int32_t n, int32_t world_size, int32_t placement,
                                    const int32_t* worker_rank_in, int32_t* worker_rank_out,
                                    int32_t* local_index_out) {
  GUARD({
    if (!worker_rank_out || !local_index_out) return fail(ADPSGD_E_INVALID, "null output");
    std::vector<int> wr, wl;
    ST(compute_placement(n, world_size, placement, worker_rank_in, wr, wl));
    for (int w = 0; w < n; ++w) { worker_rank_out[w] = wr[w]; local_index_out[w] = wl[w]; }
    return ADPSGD_OK;
  })
}

adpsgd_status adpsgd_plan_replay(int32_t n, const int32_t* worker_rank, int32_t rank, const adpsgd_event* schedule,
                                 int64_t K, int64_t k0, int32_t T, int32_t stale_reads, uint32_t* epochs,
                                 int64_t* out, int64_t cap, int64_t* n_out) {
  GUARD({
    if (n < 1 || !worker_rank || !epochs || K < 0 || (K > 0 && !schedule) || k0 < 0 || !n_out || T < 0)
      return fail(ADPSGD_E_INVALID, "plan_replay args");
    std::vector<int> wr(worker_rank, worker_rank + n), wl(n, 0);
    int world = 0;
    for (int w = 0; w < n; ++w) world = std::max(world, wr[w] + 1);
    std::vector<int> cnt(std::max(world, 1), 0);
    for (int w = 0; w < n; ++w) {
      if (wr[w] < 0) return fail(ADPSGD_E_INVALID, "worker_rank");
      wl[w] = cnt[wr[w]]++;
    }
    for (int64_t e = 0; e < K; ++e) {
      if (schedule[e].i < 0 || schedule[e].i >= n || schedule[e].j < -1 || schedule[e].j >= n)
        return fail(ADPSGD_E_INVALID, "event index");
      if (schedule[e].tau < 0 || schedule[e].tau > T || schedule[e].tau > e)
        return fail(ADPSGD_E_STALENESS, "tau exceeds min(k, T)");
    }
    const int n_local = rank >= 0 && rank < (int)cnt.size() ? cnt[rank] : 0;
    std::vector<unsigned int> ep(epochs, epochs + n);
    std::vector<std::vector<ReplayEv>> per;
    plan_replay(wr, wl, rank, n_local, schedule, K, (unsigned long long)k0, T, stale_reads != 0, ep, per);
    int64_t m = 0;
    for (auto& lst : per) m += (int64_t)lst.size();
    if (out && cap < m) return fail(ADPSGD_E_INVALID, "output capacity");
    int64_t t = 0;
    if (out)
      for (int l = 0; l < n_local; ++l) {
        int w = 0;
        while (!(wr[w] == rank && wl[w] == l)) ++w;
        for (const ReplayEv& r : per[l]) {
          int64_t* o = out + 8 * t++;
          o[0] = r.k; o[1] = w; o[2] = r.j; o[3] = r.flags; o[4] = r.e_i; o[5] = r.e_j;
          o[6] = r.kind; o[7] = r.grow;
        }
      }
    for (int w = 0; w < n; ++w) epochs[w] = ep[w];
    *n_out = m;
    return ADPSGD_OK;
  })
}

// split-K partials of a tile are reduced in DSMEM across a cluster of CTAs when splits is a
// power of two <= 16 (one pass, no partial planes); otherwise planes + a fixed-order sum
static int gemm_cluster(int splits) {
  return (splits >= 2 && splits <= 16 && (splits & (splits - 1)) == 0) ? splits : 1;
}

adpsgd_status adpsgd_gemm_tf32x3(const float* A, const float* B, float* C, int32_t M, int32_t N, int32_t K,
                                 int32_t splits) {
  GUARD({
    if (!A || !B || !C || M <= 0 || N <= 0 || K <= 0 || splits < 1) return fail(ADPSGD_E_INVALID, "gemm args");
    if (M % 128 || N % 64 || K % (32 * splits)) return fail(ADPSGD_E_INVALID, "gemm shape");
    const int bn = N % 128 == 0 ? 128 : 64;
    const int cl = gemm_cluster(splits);
    float* part = nullptr;
    if (cl < splits) CU(cudaMalloc(&part, sizeof(float) * (size_t)splits * M * N));
    CUtensorMap ta, tb;
    adpsgd_status st = ADPSGD_OK;
    cudaError_t e = make_tmap_k_major(&ta, A, M, K, 128);
    if (e == cudaSuccess) e = make_tmap_k_major(&tb, B, N, K, bn);
    if (e == cudaSuccess) e = launch_gemm_tf32x3(ta, tb, cl < splits ? part : C, M, N, K, splits, bn, nullptr, cl);
    if (e == cudaSuccess && cl < splits) e = launch_sum_planes(part, C, splits / cl, (long long)M * N, nullptr);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) st = fail(ADPSGD_E_CUDA, std::string("gemm: ") + cudaGetErrorString(e));
    if (part) cudaFree(part);
    return st;
  })
}

adpsgd_status adpsgd_gemm_tf32x3_bench(int32_t M, int32_t N, int32_t K, int32_t splits, int32_t bn, int32_t reps,
                                       double* ms_out) {
  GUARD({
    if (!ms_out || M <= 0 || N <= 0 || K <= 0 || splits < 1 || reps < 1 || (bn != 64 && bn != 128))
      return fail(ADPSGD_E_INVALID, "gemm bench args");
    if (M % 128 || N % bn || K % (32 * splits)) return fail(ADPSGD_E_INVALID, "gemm shape");
    const size_t na = (size_t)M * K, nb = (size_t)N * K;
    float* buf = nullptr;
    CU(cudaMalloc(&buf, sizeof(float) * (na + nb + (size_t)(splits + 1) * M * N)));
    float *a = buf, *b = a + na, *part = b + nb;
    float* c = part + (size_t)splits * M * N;
    CUtensorMap ta, tb;
    adpsgd_status st = ADPSGD_OK;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    cudaError_t e = launch_fill_hash(a, (long long)na, 1u, nullptr);
    if (e == cudaSuccess) e = launch_fill_hash(b, (long long)nb, 2u, nullptr);
    if (e == cudaSuccess) e = make_tmap_k_major(&ta, a, M, K, 128);
    if (e == cudaSuccess) e = make_tmap_k_major(&tb, b, N, K, bn);
    const int cl = gemm_cluster(splits);
    auto once = [&]() {
      cudaError_t r = launch_gemm_tf32x3(ta, tb, cl < splits ? part : c, M, N, K, splits, bn, nullptr, cl);
      if (r == cudaSuccess && cl < splits) r = launch_sum_planes(part, c, splits / cl, (long long)M * N, nullptr);
      return r;
    };
    for (int w = 0; w < 2 && e == cudaSuccess; ++w) e = once();
    if (e == cudaSuccess) e = cudaEventCreate(&e0);
    if (e == cudaSuccess) e = cudaEventCreate(&e1);
    if (e == cudaSuccess) e = cudaEventRecord(e0, nullptr);
    for (int r = 0; r < reps && e == cudaSuccess; ++r) e = once();
    if (e == cudaSuccess) e = cudaEventRecord(e1, nullptr);
    if (e == cudaSuccess) e = cudaEventSynchronize(e1);
    float ms = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
    if (e != cudaSuccess) st = fail(ADPSGD_E_CUDA, std::string("gemm bench: ") + cudaGetErrorString(e));
    else *ms_out = (double)ms / reps;
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    cudaFree(buf);
    return st;
  })
}

}  // extern "C"
