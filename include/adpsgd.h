/*
 * adpsgd.h -- C ABI of the B200-native AD-PSGD hot path (arXiv 1710.06952).
 * ABI version 3.  Implemented by paper_1710_06952_b200/libadpsgd.so (sm_100a).
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n.
 *
 * The method (Alg. 1; matrix form P:546-561):
 *     X_{k+1} = X_k W_k - gamma * dg(Xhat_k; xi_k, i_k),   Xhat_k = X_{k - tau_k}
 * Each gradient update, on any worker, advances the virtual counter k
 * (P:429-432).  W_k is the pair average x_i, x_j <- (x_i + x_j)/2 of a worker and
 * a neighbour on a bipartite graph (actives initiate, passives serve).
 * Problem statement: min_x f(x) = sum_i p_i f_i(x), f_i = E_xi F_i(x; xi)
 * (Eq. 1); all workers see all data (Strategy-1).
 *
 * PROCESS MODEL.  One context per rank, one GPU per context (cfg.device).  n
 * workers are placed on world_size ranks (cfg.placement).  With world_size > 1
 * the ranks exchange opaque peer blobs (adpsgd_export_peer_info -> any
 * transport -> adpsgd_import_peer_info) and call adpsgd_connect; peers' model
 * and control memory is then mapped over NVLink (CUDA IPC) and the fused
 * kernels read/write neighbours' models directly.  Production: one process per
 * GPU, NCCL collectives.  cfg.comm_local = 1: the ranks are host threads of one
 * process (e.g. several virtual ranks on ONE GPU, which runs the same
 * cross-rank protocol -- remote locks, mailboxes, tickets -- with local
 * pointers); collectives are in-process fixed-order reductions.
 *
 * ERRORS.  Every call returns adpsgd_status; nothing throws, aborts or exits
 * across the ABI.  Out-params are written only on ADPSGD_OK.  Asynchronous
 * calls (gossip/step/replay/run/consensus_mean/allreduce_sgd) latch
 * device-detected errors into a device error word, reported by the next
 * adpsgd_sync / adpsgd_read_*.  adpsgd_last_error() gives a thread-local text.
 *
 * OWNERSHIP.  All memory the library allocates (models, gradient slots, control
 * words, event log) belongs to the context and is freed by adpsgd_destroy.  Host
 * inputs (graph, config arrays, schedules, batch indices, datasets) are copied
 * before the call returns.  Device pointers passed in (grad, out) are borrowed
 * and must stay valid until the enqueued work on `stream` completes.
 *
 * LAYOUT.  Each worker's model x_i is a row of d_pad = roundup(d, 64) fp32,
 * 256-byte aligned, in its home GPU's HBM; padding entries are kept at 0.
 *
 * STREAMS.  adpsgd_stream is a cudaStream_t on the context's device; NULL means
 * the context's internal stream.
 */
#ifndef ADPSGD_H_
#define ADPSGD_H_
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ADPSGD_ABI_VERSION 3

typedef struct adpsgd_ctx adpsgd_ctx;
typedef void* adpsgd_stream;

typedef enum {
  ADPSGD_OK = 0,
  ADPSGD_E_INVALID = 1,        /* null pointer, n < 1, d < 1, index out of range, i == j  */
  ADPSGD_E_NOT_BIPARTITE = 2,  /* an edge joins two workers of the same role         */
  ADPSGD_E_DISCONNECTED = 3,   /* graph not connected, rho = 1                       */
  ADPSGD_E_NOT_NEIGHBOURS = 4, /* event (i, j) is not an edge of the graph                        */
  ADPSGD_E_STALENESS = 5,      /* tau > min(k, T) (Assumption 1.7)               */
  ADPSGD_E_DIVERGED = 6,       /* non-finite model value detected                                  */
  ADPSGD_E_TIMEOUT = 7,        /* device-side wait exceeded the watchdog                           */
  ADPSGD_E_CUDA = 8,
  ADPSGD_E_NCCL = 9,
  ADPSGD_E_OOM = 10,
  ADPSGD_E_STATE = 11,         /* call not valid in the current state (e.g. not connected)         */
  ADPSGD_E_UNSUPPORTED = 12    /* combination not supported (message says which)                   */
} adpsgd_status;

/* Undirected communication graph (V, E) with the active/passive
 * split of P:469-473.  Caller-owned, copied by adpsgd_init.                    */
typedef struct {
  int32_t n;                /* number of workers                                              */
  int32_t n_edges;
  const int32_t* edges;     /* 2*n_edges endpoints; undirected; no self-loops, no duplicates  */
  const int8_t* role;       /* n entries, 0 = active, 1 = passive; NULL = BFS 2-colouring     */
} adpsgd_graph;

typedef enum {
  ADPSGD_MODEL_NONE = 0,      /* pure averaging (W_k only)                                    */
  ADPSGD_MODEL_EXTERNAL = 1,  /* gradients supplied by the caller (adpsgd_step grad pointer)  */
  ADPSGD_MODEL_QUADRATIC = 2, /* synthetic quadratic, procedural data             */
  ADPSGD_MODEL_LSQ = 3,       /* least squares F = 1/2 (a.x - b)^2                            */
  ADPSGD_MODEL_LOGREG = 4,    /* logistic F = log(1 + exp(-y a.x)), y in {-1,+1}             */
  ADPSGD_MODEL_MLP = 5        /* 2-layer tanh MLP + softmax cross-entropy (R18)     */
} adpsgd_model_kind;

typedef struct {
  /* --- process / placement --- */
  int32_t rank;               /* this process's rank in [0, world_size)                       */
  int32_t world_size;         /* number of processes (one GPU each)                           */
  int32_t device;             /* CUDA device ordinal this context drives                      */
  int32_t placement;          /* 0 block (contiguous ring segments), 1 interleave (w mod G),  */
                              /* 2 explicit (worker_rank)                                     */
  const int32_t* worker_rank; /* n entries when placement == 2                                */
  /* --- method hyper-parameters --- */
  float gamma;                /* learning rate; multiplies the batch SUM (reading R2)         */
  int32_t batch_M;            /* minibatch size M                                 */
  int32_t staleness_cap_T;    /* T of Assumption 1.7; replay rejects tau > T      */
  uint64_t seed;              /* device RNG seed (neighbour choice, Philox batch sampling)     */
  adpsgd_model_kind model;
  /* --- synthetic quadratic (model == QUADRATIC) --- */
  uint32_t quad_data_key;     /* data landscape key                                           */
  uint32_t quad_noise_key;    /* gradient-noise key                                           */
  float quad_noise_s;         /* s = sigma * sqrt(3 M)                                        */
  /* --- datasets for LSQ / LOGREG / MLP (host pointers, copied to every GPU) --- */
  int32_t n_samples;          /* S                                                            */
  const float* data_A;        /* S x feat fp32 row-major (feat = d for LSQ/LOGREG, mlp_in)   */
  const float* data_b;        /* S targets (LSQ) or labels +-1 (LOGREG)                       */
  const int32_t* data_y;      /* S class labels (MLP)                                         */
  int32_t mlp_in, mlp_hid, mlp_out;
  /* --- initial models --- */
  const float* x0;            /* d floats, same for every worker; NULL = zeros        */
  const float* x0_per_worker; /* n*d floats (pure-gossip tests); overrides x0                 */
  /* --- scheduler (free-running engine) --- */
  const float* straggler;     /* n slowdown factors >= 1; NULL = all 1          */
  int64_t compute_ns;         /* emulated per-gradient compute time t_c of a 1x worker        */
  int32_t engine_ctas_per_sm; /* 0 = default                                                  */
  int32_t engine_variant;     /* reserved (the round-1 A/B variants are gone): must be 0;     */
                              /* anything else fails with ADPSGD_E_UNSUPPORTED                */
  int64_t log_capacity;       /* event-log ring entries on rank 0; 0 = default (1<<20)        */
  int32_t wait_free;          /* adpsgd_run loop: 0 = Alg. 1 (gradient fused into the event); */
                              /* 1 = App. A wait-free runtime: a worker pulls   */
                              /* its model, computes g into a buffer during s_w*t_c, and its  */
                              /* communication loop flushes it (FLUSH_FIRST events) while     */
                              /* actives keep averaging (NO_GRAD events) in between;          */
                              /* 2 = as 1 plus local-update compensation (COMPENSATE).        */
                              /* QUADRATIC model only; one-sided NVLink access.               */
  int32_t reserved0;
  /* --- heterogeneous communication (Fig. loss-link), reading R21 --- */
  const float* link_slow;     /* n factors L_w >= 1: worker w's network link is L_w x slower;  */
                              /* NULL = all 1.  Emulated: a model transfer over a link of     */
                              /* factor L takes L * link_ns, so a pair event holds both        */
                              /* workers (and the passive's lock) (max(L_i, L_j) - 1) * link_ns */
                              /* after its pass; the synchronous baselines wait for their     */
                              /* slowest link every round (adpsgd_allreduce_sgd, adpsgd_dpsgd)*/
  int64_t link_ns;            /* nominal time of one model transfer over a 1x link            */
  int32_t engine_no_fuse;     /* 0 (default): when an active holds a passive's lock and the   */
                              /* passive's own local step is due, run both events (tickets    */
                              /* k, k+1) in one pass -- same result and log, 16d bytes instead */
                              /* of 24d; 1: never fuse                                        */
  int32_t reserved1;
  int64_t engine_fuse_wait_ns;/* a due passive waits up to this long for an active to take    */
                              /* its lock (and fuse its step) before stepping alone; 0 = never */
                              /* waits.  Scheduling only: any interleaving is an AD-PSGD run.  */
  int32_t super_R;            /* > 1: super-learner context (adpsgd_super_run, reading R22):  */
                              /* the graph is R copies of the super-learners' graph and only  */
                              /* that contracted graph must be connected                      */
  int32_t engine_coop;        /* cooperative cross-GPU events (world > 1): both GPUs' engines */
                              /* process half of a cross event's tiles, so both drive NVLink. */
                              /* 0 = auto (on at world 2, when at most half the edges cross,  */
                              /* or when GPUs start cross events unevenly; off when nearly     */
                              /* every edge crosses with initiators spread evenly), 1 = on,    */
                              /* -1 = off                                                      */
  /* --- in-process ranks (appended in ABI version 3) --- */
  int32_t comm_local;         /* 0: one process per rank -- peers mapped with CUDA IPC, NCCL    */
                              /*    collectives (the production path);                          */
                              /* 1: the world_size ranks are host threads of ONE process (any   */
                              /*    devices, several ranks may share one GPU): peers' memory is */
                              /*    addressed directly and collectives are fixed-order device   */
                              /*    reductions between host barriers (comm.h).  adpsgd_connect's*/
                              /*    id is then any 128-byte token common to the group, and each */
                              /*    rank's calls must come from its own host thread.            */
  int32_t engine_grid;        /* engine CTAs per rank; 0 = ctas_per_sm x SMs, divided by        */
                              /* world_size when comm_local (ranks sharing a GPU must all be    */
                              /* resident).  Must be equal on every rank.                       */
} adpsgd_config;

/* A schedule event (reading R5): worker i makes the gradient update; j is its
 * averaging partner (must be a neighbour of the other role) or -1 (W_k = I);
 * tau is the staleness of the read, Xhat = X_{k - tau}.                         */
typedef struct { int32_t i, j, tau; uint32_t flags; } adpsgd_event;
#define ADPSGD_EV_NO_GRAD 1u   /* pure averaging: W_k only, no gradient update (takes a ticket, R23) */
/* App. A, the wait-free runtime, reading R20:
 * FLUSH_FIRST  the communication thread flushes g into x_i BEFORE averaging
 *              (Alg. 2 order): x_i <- fl(x_i - fl(gamma g));
 *              m = fl(fl(x_i + x_j) * 0.5); x_i = x_j = m.  The gradient exists
 *              before its flush event, so its random draws (noise, Philox batch)
 *              are keyed by the read point: key = 2^62 | (k - tau) << 20 | i.
 * COMPENSATE   local-update compensation (footnote at P:1265-1268): if worker
 *              i's previous gradient event k_p (same schedule) has k_p >= k - tau,
 *              i.e. it was still in the buffer when the model was pulled, the
 *              gradient is evaluated at fl(xhat - fl(gamma g_p)).  Requires
 *              k_p - tau_p <= k - tau (one gradient at a time per worker), else
 *              ADPSGD_E_STALENESS.                                              */
#define ADPSGD_EV_FLUSH_FIRST 2u
#define ADPSGD_EV_COMPENSATE 4u

/* Committed-event record written by the device (event log ring on rank 0).   */
typedef struct {
  int64_t k;          /* virtual counter value of this update                 */
  int32_t i, j, tau;  /* as adpsgd_event                                                  */
  uint32_t flags;
  uint64_t t_start_ns, t_end_ns;   /* %globaltimer at pass start / commit                 */
} adpsgd_log_entry;

typedef struct {
  int64_t ticket;            /* committed events system-wide (the virtual counter k)       */
  int64_t local_events;      /* events committed by this rank's engine/executor            */
  int64_t local_pair_events; /* of which pair averages                                     */
  int64_t local_cross_events;/* of which the partner lives on another rank (NVLink)       */
  double  local_bytes;       /* algorithmic HBM bytes of this GPU: rows resident here that
                                committed events read + wrote (a cross pair credits each GPU
                                its own row: 8d bytes, the initiator's g row extra)          */
  double  local_nvlink_bytes;/* algorithmic bytes that crossed NVLink (both directions)    */
  double  engine_busy_ns;    /* sum over events of (t_end - t_start)                       */
  double  engine_busy_cross_ns; /* the part of engine_busy_ns spent in cross-GPU events    */
} adpsgd_stats;

/* ---------------------------------------------------------------- lifecycle -- */

/* Validate the graph, place workers, allocate
 * models, gradient slots, control words and the event log on cfg->device, and
 * write x_i <- x0 for every local worker (Alg. 1 Require).  With
 * world_size == 1 the context is ready on return; otherwise call
 * export/import_peer_info and adpsgd_connect first.                            */
adpsgd_status adpsgd_init(const adpsgd_graph* g, int32_t n_workers, int64_t d,
                          const adpsgd_config* cfg, adpsgd_ctx** out);
adpsgd_status adpsgd_destroy(adpsgd_ctx* ctx);
const char* adpsgd_last_error(void);
int32_t adpsgd_abi_version(void);

/* Multi-process wiring (world_size > 1).  The blob holds CUDA IPC handles of
 * this rank's model arena and control arena.  import for every other rank,
 * then connect (collective: every rank must call it; nccl_id is the 128-byte
 * ncclUniqueId produced by adpsgd_nccl_unique_id on rank 0).                   */
adpsgd_status adpsgd_peer_info_size(int64_t* bytes);
adpsgd_status adpsgd_export_peer_info(adpsgd_ctx* ctx, void* buf, int64_t cap, int64_t* n_out);
adpsgd_status adpsgd_import_peer_info(adpsgd_ctx* ctx, int32_t rank, const void* buf, int64_t n);
adpsgd_status adpsgd_nccl_unique_id(void* buf128);
adpsgd_status adpsgd_connect(adpsgd_ctx* ctx, const void* nccl_id /* 128 B, NULL if world 1 */);

/* ------------------------------------------------------------- hot path ---- */

/* Pairwise averaging alone (W_k): x_i, x_j <- fl(fl(x_i + x_j)*0.5).
 * i and j must be neighbours of different roles; i lives on this rank (j may
 * be remote when world_size > 1: the passive endpoint's lock and the ticket are
 * then taken on the device, as adpsgd_step does).  Like every pure average
 * (NO_GRAD events of replays and runs) it takes the next ticket k and is
 * logged with flags = ADPSGD_EV_NO_GRAD (reading R23: the ticket
 * counts committed events; the paper's k of P:429-432 counts the events
 * without NO_GRAD, and staleness tau is measured in ticket units).             */
adpsgd_status adpsgd_gossip(adpsgd_ctx* ctx, int32_t i, int32_t j, adpsgd_stream s);

/* One AD-PSGD worker iteration for local worker w: gradient at the
 * current model (tau = 0) -- the caller's `grad` (device, d floats) or the
 * built-in model when grad == NULL -- then, if w is active, average with a
 * neighbour j drawn uniformly from N(w) and apply x_w <- m - gamma g (Alg. 1
 * order, reading R1); if w is passive, x_w <- x_w - gamma g (W_k = I).
 * Serialised against other adpsgd_step calls of the same context by stream
 * order.  world_size > 1: w must live on this rank; the passive side's lock
 * (the partner's, or w's own for a passive step) and the ticket k are taken
 * on the device -- other ranks may step concurrently -- then the fused pass
 * runs over NVLink and a commit kernel logs and unlocks.  Collective calls
 * (run/replay/super_run) made after such steps first agree on the device
 * counter across ranks (a small NCCL all-reduce), so every rank must have
 * finished its steps before any rank enters one (e.g. a barrier).
 * *ticket_out (nullable) receives k.                                           */
adpsgd_status adpsgd_step(adpsgd_ctx* ctx, int32_t w, const float* grad, adpsgd_stream s,
                          int64_t* ticket_out);

/* Deterministic replay of a schedule (events k = k0 .. k0+n_events-1, where k0
 * is the current ticket).  Result is bitwise independent of interleaving.
 * batch_idx: n_events*M sample indices (host), or NULL for device Philox
 *  sampling (idx = (u32*S)>>32, u32 = Philox4x32-10(key=seed, ctr=(lo32(k), m, BATCH, hi32(k)))).
 * flags: 0 = auto, ADPSGD_REPLAY_HOST = stream-ordered per-event kernels (all
 * models, any tau <= T; world 1), ADPSGD_REPLAY_ENGINE = the persistent NVLink
 * engine with device epoch flags (models NONE/QUADRATIC, any tau <= T: a stale
 * read is an op of the worker's sequence computing the gradient at X_{k-tau}
 * into one of its T + 1 read rows, see adpsgd_plan_replay; no COMPENSATE
 * events; any world; collective: every rank passes the same schedule).         */
#define ADPSGD_REPLAY_HOST 1u
#define ADPSGD_REPLAY_ENGINE 2u
adpsgd_status adpsgd_replay(adpsgd_ctx* ctx, const adpsgd_event* schedule, int64_t n_events,
                            const int32_t* batch_idx, uint32_t flags, adpsgd_stream s);

/* Super-learners (reading R22): "combining learners on the same
 * computing node as a super-learner (via NCCL AllReduce)".  Learner w lives on
 * rank w (n == world_size, placement 2 with worker_rank[w] = w); learner (s, r)
 * = s*R + r belongs to super-learner s, and the graph must be R copies of the
 * super-learners' bipartite graph (learner (s, r) neighbours (s', r) only).
 * Every rank runs n_steps iterations of its super-learner's loop: its learner
 * gradient at its replica (any built-in model; its noise / Philox minibatch keyed
 * by 2^61 | s<<44 | c<<8 | r, c = the super-learner's gradient count), NCCL
 * all-reduce SUM over the group; the
 * group leader takes the passive super-learner's lock (active: a neighbour drawn
 * uniformly; passive: its own) and the ticket k; every replica r averages with
 * replica r of the partner over NVLink and applies x <- m - gamma g (Alg. 1
 * order; a passive only updates); group barrier; the leader logs {k, s, j} and
 * unlocks.  R = cfg.super_R (1 if unset).  Collective over all ranks; the
 * replicas of a super-learner stay bitwise equal.                            */
adpsgd_status adpsgd_super_run(adpsgd_ctx* ctx, int64_t n_steps, adpsgd_stream s);

/* Free-running asynchronous AD-PSGD (the wait-free runtime of App. A,
 * P:1235-1314, realised on the device): one persistent kernel per GPU runs
 * every local worker's loop -- emulated compute (s_w * t_c), neighbour choice,
 * device try-lock of the passive (bipartite order: one lock per event, so no
 * wait cycle), fused average + gradient update over NVLink, ticket,
 * log, release -- until the system-wide counter has advanced by n_updates.
 * Collective: every rank calls it with the same n_updates.  Models:
 * QUADRATIC (tau = 0 fused gradient) or NONE (actives gossip continuously).   */
adpsgd_status adpsgd_run(adpsgd_ctx* ctx, int64_t n_updates, adpsgd_stream s);

/* Consensus output: out = fl32( (sum_i x_i)/n ) with an fp64 sum over all
 * workers on all ranks (NCCL AllReduce fp64 when world > 1); mk_out (nullable)
 * receives M_k = (1/n) sum_i ||xbar - x_i||^2 (p_i = 1/n).
 * out_device: d floats on this context's device (every rank gets the result).
 * Synchronous w.r.t. the host when mk_out != NULL.  A non-finite model value
 * (a diverged run) latches ADPSGD_E_DIVERGED for the next adpsgd_sync,
 * and is returned at once when mk_out != NULL.                               */
adpsgd_status adpsgd_consensus_mean(adpsgd_ctx* ctx, float* out_device, double* mk_out,
                                    adpsgd_stream s);

/* AllReduce-SGD comparison baseline (reading R12), on a separate
 * replica: per round every worker computes its minibatch gradient at the common
 * model (straggler: the round waits for max_w s_w * t_c), gradients are summed
 * locally and across ranks (ncclAllReduce fp32 over NVLink), and every replica
 * applies x <- x - gamma * (sum g)/n.  Collective.  Model QUADRATIC.          */
adpsgd_status adpsgd_allreduce_sgd(adpsgd_ctx* ctx, int64_t n_rounds, adpsgd_stream s);
adpsgd_status adpsgd_allreduce_read_model(adpsgd_ctx* ctx, float* host_out);
adpsgd_status adpsgd_allreduce_reset(adpsgd_ctx* ctx, const float* host_x /* d or NULL=x0 */);

/* D-PSGD comparison baseline (Table 4's second column), reading R19:
 * synchronous rounds X <- X W - gamma G with W = I - L/(deg_max + 1) on the
 * graph, gradients at each worker's own pre-round model (quadratic, event key
 * round_base + w).  Runs on its own double-buffered replica of all rows; remote
 * neighbour rows arrive each round by NCCL send/recv (a halo exchange); every
 * round waits for its slowest worker (max_w s_w * t_c).  Collective.  fp32 op
 * order as in the header comment of oracle_dpsgd_round (bit-exact).           */
adpsgd_status adpsgd_dpsgd(adpsgd_ctx* ctx, int64_t n_rounds, adpsgd_stream s);
adpsgd_status adpsgd_dpsgd_reset(adpsgd_ctx* ctx, const float* x0_per_worker /* n*d host or NULL = x0 */);
adpsgd_status adpsgd_dpsgd_read_model(adpsgd_ctx* ctx, int32_t w, float* host_out);

/* -------------------------------------------------------- state access ---- */
adpsgd_status adpsgd_sync(adpsgd_ctx* ctx);   /* wait for all work; return latched device error */
adpsgd_status adpsgd_read_model(adpsgd_ctx* ctx, int32_t w, float* host_out);   /* local w */
adpsgd_status adpsgd_write_model(adpsgd_ctx* ctx, int32_t w, const float* host_in);
adpsgd_status adpsgd_model_device_ptr(adpsgd_ctx* ctx, int32_t w, float** dev_ptr);
adpsgd_status adpsgd_worker_rank(adpsgd_ctx* ctx, int32_t w, int32_t* rank);
adpsgd_status adpsgd_get_ticket(adpsgd_ctx* ctx, int64_t* k);
/* Event log (rank 0 holds it): entries with k in [k_from, k_from + cap).       */
adpsgd_status adpsgd_read_log(adpsgd_ctx* ctx, int64_t k_from, adpsgd_log_entry* out, int64_t cap,
                              int64_t* n_out);
/* Per-worker committed gradient updates (the empirical p_i), local workers. */
adpsgd_status adpsgd_read_update_counts(adpsgd_ctx* ctx, int64_t* out_n);
adpsgd_status adpsgd_get_stats(adpsgd_ctx* ctx, adpsgd_stats* out);
adpsgd_status adpsgd_reset_stats(adpsgd_ctx* ctx);
/* Number of kernels this context launched since creation (bench gpu_launches). */
adpsgd_status adpsgd_launch_count(adpsgd_ctx* ctx, int64_t* out);

/* ------------------------------------------------ host-only planning ------
 * Pure host functions (no device work, usable without a GPU) that expose the
 * multi-rank planning adpsgd_init / adpsgd_replay perform internally.       */
/* Worker -> rank placement and each worker's index among its rank's workers
 * (placement 0 block, 1 interleave, 2 explicit from worker_rank_in).          */
adpsgd_status adpsgd_plan_placement(int32_t n, int32_t world_size, int32_t placement,
                                    const int32_t* worker_rank_in, int32_t* worker_rank_out,
                                    int32_t* local_index_out);
/* The engine-replay plan of `rank`: the ops whose worker i lives on `rank`,
 * grouped by local worker in execution order, each as int64[8]
 * {k, i, j, flags, e_i, e_j, kind, row}.  kind 0 = an event (k = its index);
 * kind 2 = a stale read (stale_reads != 0 and tau > 0): the gradient of
 * event f at X_{f - tau} computed into worker i's read row `row` (f's m-th such
 * event of i uses row m mod (T + 1)), placed before the first event >= f - tau
 * touching i; its k is the gradient's random-draw key.  An event with row >= 0
 * applies that row.  e_i / e_j are the epochs (counts of earlier ops of i / j,
 * starting from `epochs`) the device waits for; `epochs` (n entries) is
 * advanced in place exactly as on every rank.  out may be NULL to query n_out. */
adpsgd_status adpsgd_plan_replay(int32_t n, const int32_t* worker_rank, int32_t rank, const adpsgd_event* schedule,
                                 int64_t K, int64_t k0, int32_t T, int32_t stale_reads, uint32_t* epochs,
                                 int64_t* out, int64_t cap, int64_t* n_out);

/* Diagnostics: the MLP's tensor-core GEMM on its own.
 * C[M x N] = A[M x K] . B[N x K]^T, fp32 row-major DEVICE pointers on the current
 * device, computed as 3xTF32 (hi*hi + hi*lo + lo*hi, the split done in shared
 * memory) with tcgen05.mma into TMEM, split-K over `splits` CTAs per tile
 * (partials summed in a fixed order: in distributed shared memory across a
 * thread-block cluster when splits is a power of two <= 16, else through
 * partial planes).  Requires M % 128 == 0, N % 64 == 0, K % (32 * splits) == 0.
 * Synchronous.                                                                  */
adpsgd_status adpsgd_gemm_tf32x3(const float* A, const float* B, float* C, int32_t M, int32_t N, int32_t K,
                                 int32_t splits);

/* Diagnostics: device time of that GEMM alone (tcgen05 utilisation
 * of the MLP GEMMs swept over M).  Allocates operands of the given shape on the
 * current device, then times `reps` launches
 * of the GEMM kernel (+ the split-K partial sum when splits > 1) with CUDA
 * events after 2 warm-up launches; *ms_out = mean milliseconds per GEMM.
 * bn = 64 or 128 (N tile).  Shape rules as adpsgd_gemm_tf32x3.  Synchronous.  */
adpsgd_status adpsgd_gemm_tf32x3_bench(int32_t M, int32_t N, int32_t K, int32_t splits, int32_t bn, int32_t reps,
                                       double* ms_out);

#ifdef __cplusplus
}
#endif
#endif /* ADPSGD_H_ */
