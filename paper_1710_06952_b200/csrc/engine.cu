// engine.cu -- the persistent AD-PSGD engine: one cooperative kernel per GPU
// runs every local worker's loop of the wait-free runtime (App. A)
// on the device, with no host round trip per event.
//
// Per local worker w, in free-running mode (mode 0):
//   1. compute phase: emulated gradient time s_w * t_c (timer; no SM spinning)
//   2. w active : pick j ~ U(N(w)), try-lock(j) at system scope
//      w passive: try-lock(w)     (its local gradient flush)
//      Only passives carry locks and every event takes exactly one, so no
//      wait cycle can form -- the device form of the bipartite argument
//      (P:458-479).  A failed try-lock leaves the worker pending; no CTA
//      ever blocks on it.
//   3. take ticket k (CAS on rank 0's counter, bounded by the run's target):
//      the virtual counter of P:429-432, taken while holding the lock so the
//      ticket order is the serialisation order (log replay).
//   4. fused pass over d, split across ALL CTAs of the grid (interleaved tiles):
//      m = fl(fl(x_w + x_j)*0.5); x_j <- m; x_w <- fl(m - fl(gamma g)),
//      g = quadratic gradient at the pre-average x_w (tau = 0) -- Alg. 1 steps
//      4-6, reading R1.
//   5. the CTA finishing the last slice commits: log {k,i,j,0}, counters,
//      release fence (sys), unlock, schedule the next compute phase.
// Replay mode (mode 1): the event list of each local worker is consumed in
// order; event k starts when epoch[i] == e_i(k) and epoch[j] == e_j(k) (device
// epoch flags, system scope), and commits by bumping both epochs.
//
// Cross-GPU pairs (world > 1), two-sided: the GPU computing the event posts a
// push request on the partner's home GPU, whose engine copies x_j tile by tile
// into the computing GPU's landing row (NVLink writes) and publishes per-CTA
// progress counters; the computing CTAs consume tiles as they land (never
// blocking: they return to the scheduler when nothing has landed) and write the
// average back into x_j (NVLink writes).  NVLink then carries writes only, in
// both directions: tools/membench measured 672 GB/s per direction for
// bidirectional pushes vs 476 GB/s when one GPU both reads and writes its peer.
#include "internal.h"

namespace adp {

namespace {

constexpr int kEngineThreads = 512;
constexpr int kEngineUnroll = 2;
constexpr int kExit = -2;
constexpr int kPickPush = 1 << 20;      // pick codes >= kPickPush: push request of local worker
constexpr int kPickGuest = kPickPush - 1; // a peer's cooperative event posted in a local mailbox

struct SmemSlot {                  // tid 0 copies the running event here for the CTA
  float* xi;
  float* xj;
  float* land;
  long long k;
  int grad;
  int pair;
  int cross;                       // partner row lives on another GPU (P2P stores)
  long long t0, t1;                // tile sub-range (two-sided cross consume)
  // push request
  const float* src;
  float* dst;
  unsigned int* cnt;
  unsigned int tag16;
  // App. A: flush-first order, pulls, buffered gradients
  int ff;
  int kind;
  unsigned long long key;
  const float* g;
  float* gout;
  int absorb;                      // fused passive local step (event k-1) before the pair
  // tile split and arrival: own events use (blockIdx, grid) or, when
  // cooperative, (blockIdx, 2 grid); a guest (a peer's cooperative event) uses
  // (grid + blockIdx, 2 grid) and arrives on the initiator's slot
  long long first, step;
  int ncta;                        // CTAs that arrive on the event's counter
  int coop;
  int guest;
  int gl;                          // local worker whose mailbox carried the guest event
  unsigned int* gdone;             // initiator's slot->done (peer)
  unsigned int* gready;            // initiator's slot->commit_ready (peer)
};

__device__ __forceinline__ unsigned int tag_of(unsigned int seq, unsigned int st) { return (seq << 2) | st; }

__device__ void latch_error(const EngineParams& p, unsigned int code) {
  atomicCAS(&p.gctl->error, 0u, code);
  atomicExch(&p.gctl->abort_flag, 1u);
}

// tickets k, k+1, ..: up to `want` consecutive values of rank 0's counter below
// the target (free-running).  Returns how many were taken (0 = run is over).
__device__ __noinline__ int take_tickets(const EngineParams& p, unsigned long long* k, int want) {
  unsigned long long t = ld_relaxed_sys64(&p.gctl0->ticket);
  while (true) {
    if (t >= p.target) return 0;
    const int got = (t + (unsigned long long)want <= p.target) ? want : (int)(p.target - t);
    const unsigned long long old = atomicCAS_system(&p.gctl0->ticket, t, t + (unsigned long long)got);
    if (old == t) { *k = t; return got; }
    t = old;
  }
}
__device__ __forceinline__ bool take_ticket(const EngineParams& p, unsigned long long* k) {
  return take_tickets(p, k, 1) == 1;
}

__device__ void publish_running(Slot* sl, unsigned int seq) {
  __threadfence();                                   // fields before the tag
  st_release_gpu(&sl->tag, tag_of(seq + 1, kStateRunning));
}

// Cooperative cross-GPU event: after publishing event seq+1 in worker w's slot,
// post it in partner j's guest mailbox (j's home GPU) so that GPU's CTAs take
// half of the tiles -- both GPUs then drive NVLink (reads of the other row and
// writes of the results in both directions) instead of one.
// The mailbox has its own sequence (a partner serves events of several
// initiators, whose slot sequences may coincide); the poster holds the partner
// exclusively (its lock or its epoch), so read-increment is race-free.
__device__ void post_guest(const EngineParams& p, Slot* sl, int w, int j) {
  WorkerCtl* cj = p.workers[j].ctl;                   // peer memory
  __threadfence_system();                             // the slot's fields, system-wide
  *(volatile int*)&cj->guest_i = w;
  st_release_sys(&cj->guest_tag, tag_of(sl->gseq, kStateRunning));
}

// cross-GPU event (two-sided): ask j's home GPU to push x_j into our landing row
__device__ void post_push_request(const EngineParams& p, Slot* sl, int w, int j, unsigned int seq) {
  const WorkerDesc& dw = p.workers[w];
  const unsigned int tag16 = (seq + 1) & 0xffffu;    // the seq this event is published with
  sl->tag16 = tag16;
  sl->land = dw.land;
  sl->pcnt = dw.pcnt;
  WorkerCtl* cj = p.workers[j].ctl;                   // peer memory
  const unsigned int rq = ld_acquire_sys(&cj->req_tag) >> 2;
  *(volatile int*)&cj->req_consumer = w;
  *(volatile unsigned int*)&cj->req_tag16 = tag16;
  st_release_sys(&cj->req_tag, ((rq + 1u) << 2) | kStateRunning);
}

// App. A wait-free runtime, reading R20.  A worker runs two
// threads that share the gradient buffer g (one of its two gradient rows):
//  * computation thread (App. A Alg. 1): pull x^w -- a consistent copy, so a
//    passive holds its own lock; the read point t is the ticket counter at that
//    moment -- and compute g' at x^w (compensated by the buffered g when
//    wait_free == 2) into the other row; after s_w * t_c, when the buffer is
//    empty, g' becomes the buffer;
//  * communication thread (Alg. 2 / Alg. 3): an active flushes the buffer (if
//    any) and averages with a random neighbour, continuously (NO_GRAD events
//    when the buffer is empty); a passive flushes its buffer when it fills and
//    otherwise only serves the actives' averages.
// Both run as events of the worker's slot, so the pull is serialised with the
// worker's own averages.  Pulls take no ticket (X does not change); flushes log
// tau = k - t and the flags FLUSH_FIRST | COMPENSATE, which is all the oracle
// needs to replay the run.
__device__ __noinline__ bool start_wait_free(const EngineParams& p, Slot* sl, unsigned int tag, int w,
                                             unsigned long long now) {
  const unsigned int seq = tag >> 2;
  const WorkerDesc dw = p.workers[w];
  volatile WorkerCtl* cw = dw.ctl;                     // home GPU control word
  const bool active = dw.role == 0 && dw.nb_cnt > 0;
  const long long dpad = p.n4 * 4;
  if (cw->wf_state == 1u && now >= cw->wf_ready_ns && cw->wf_pub == 0u) {   // g' -> buffer
    cw->wf_buf ^= 1u;
    cw->wf_tread_pub = cw->wf_tread_cur;
    cw->wf_comp_pub = cw->wf_comp_cur;
    cw->wf_pub = 1u;
    cw->wf_state = 0u;
  }
  if (cw->wf_state == 0u) {                            // computation thread: pull
    unsigned int* lock = nullptr;
    if (!active) {
      lock = &dw.ctl->lock;
      if (atomicCAS_system(lock, 0u, 1u) != 0u) { st_release_gpu(&sl->tag, tag); return false; }
      __threadfence_system();
    }
    const unsigned long long t = ld_relaxed_sys64(&p.gctl0->ticket);
    const bool comp = p.wait_free == 2 && cw->wf_pub != 0u;
    cw->wf_tread_cur = t;
    cw->wf_comp_cur = comp ? 1u : 0u;
    sl->kind = kKindPull;
    sl->absorb = -1;
    sl->coop = 0;
    sl->i = w; sl->j = -1; sl->tau = 0; sl->flags = 0u; sl->k = -1;
    sl->key = read_key(t, w);
    sl->xi = dw.x; sl->xj = nullptr;
    sl->g = comp ? dw.gb + (long long)cw->wf_buf * dpad : nullptr;
    sl->gout = dw.gb + (long long)(cw->wf_buf ^ 1u) * dpad;
    sl->ctl_i = dw.ctl; sl->ctl_j = nullptr; sl->lock = lock; sl->cross = 0;
    sl->t0 = now;
    sl->done = 0;
    publish_running(sl, seq);
    return true;
  }
  const bool flush = cw->wf_pub != 0u;                 // communication thread
  int j = -1;
  unsigned int* lock;
  if (active) {
    j = sl->pending_j;
    if (j < -1) {
      const uint4 r = philox4x32_10(make_uint4((uint32_t)w, sl->nb_ctr, 0x4E424F52u, 0u), p.seed);
      j = p.nbrs[dw.nb_off + (int)(((unsigned long long)r.x * (unsigned)dw.nb_cnt) >> 32)];
      sl->pending_j = j;
    }
    lock = &p.workers[j].ctl->lock;
  } else {
    if (!flush) { st_release_gpu(&sl->tag, tag); return false; }
    lock = &dw.ctl->lock;
  }
  if (atomicCAS_system(lock, 0u, 1u) != 0u) { st_release_gpu(&sl->tag, tag); return false; }
  __threadfence_system();
  unsigned long long k;
  if (!take_ticket(p, &k)) {
    __threadfence_system();
    atomicExch_system(lock, 0u);
    st_release_gpu(&sl->tag, tag_of(seq, kStateFinished));
    return true;
  }
  sl->kind = kKindEvent;
  sl->absorb = -1;
  sl->coop = 0;
  sl->i = w; sl->j = j; sl->k = (long long)k; sl->key = k;
  sl->tau = flush ? (int)(k - cw->wf_tread_pub) : 0;
  sl->flags = flush ? (2u | (cw->wf_comp_pub ? 4u : 0u)) : 1u;
  sl->g = flush ? dw.gb + (long long)cw->wf_buf * dpad : nullptr;
  sl->xi = dw.x; sl->xj = j >= 0 ? p.workers[j].x : nullptr;
  sl->ctl_i = dw.ctl; sl->ctl_j = j >= 0 ? p.workers[j].ctl : nullptr; sl->lock = lock;
  sl->cross = j >= 0 && p.workers[j].rank != p.my_rank;
  if (j >= 0) { sl->pending_j = -2; sl->nb_ctr += 1; }
  sl->t0 = now;
  sl->done = 0;
  publish_running(sl, seq);
  return true;
}

// Called by tid 0 of some CTA that found no slice to do.  Returns true if it
// started or finished a worker (progress).
__device__ __noinline__ bool try_start(const EngineParams& p, int s, unsigned int tag, unsigned long long now) {
  Slot* sl = p.slots + s;
  const unsigned int seq = tag >> 2;
  bool done = false;
  if (p.mode == 0) {
    // stop early if the system-wide budget is exhausted (straggler in compute),
    // once a slow-link transfer still in progress has ended
    done = ld_relaxed_sys64(&p.gctl0->ticket) >= p.target;
    if (done) {
      if (*(unsigned int* volatile*)&sl->held_lock && now < *(volatile unsigned long long*)&sl->unlock_at)
        return false;
    } else if (now < *(volatile unsigned long long*)&sl->ready_ns) {
      return false;
    }
  }
  if (atomicCAS(&sl->tag, tag, tag_of(seq, kStateClaimed)) != tag) return false;   // claim
  if (p.mode == 0) {
    if (sl->held_lock) {                    // release the partner held by the slow transfer (R21)
      __threadfence_system();
      atomicExch_system(sl->held_lock, 0u);
      sl->held_lock = nullptr;
    }
    if (done) {
      st_release_gpu(&sl->tag, tag_of(seq, kStateFinished));
      return true;
    }
  }

  const int w = p.local_ids[s];
  const WorkerDesc dw = p.workers[w];
  if (p.mode == 1) {
    // ---------------------------------------------------------- replay ----
    const long long cur = *(volatile long long*)&sl->ev_cur;
    if (cur >= *(volatile long long*)&sl->ev_end) {
      st_release_gpu(&sl->tag, tag_of(seq, kStateFinished));
      return true;
    }
    const ReplayEv e = p.rev[cur];
    const unsigned int ei = ld_acquire_sys(&dw.ctl->epoch);
    unsigned int ej = 0;
    WorkerCtl* cj = nullptr;
    if (e.j >= 0) { cj = p.workers[e.j].ctl; ej = ld_acquire_sys(&cj->epoch); }
    if (ei != e.e_i || (e.j >= 0 && ej != e.e_j)) {        // predecessors not committed yet
      st_release_gpu(&sl->tag, tag);
      return false;
    }
    __threadfence_system();                                 // acquire their data
    sl->i = w; sl->j = e.j; sl->tau = 0; sl->flags = e.flags; sl->k = e.k;
    sl->kind = kKindEvent; sl->g = nullptr; sl->absorb = -1;
    sl->key = (e.flags & 2u) ? read_key((unsigned long long)e.k, w) : (unsigned long long)e.k;   // R20
    sl->xi = dw.x; sl->xj = e.j >= 0 ? p.workers[e.j].x : nullptr;
    sl->ctl_i = dw.ctl; sl->ctl_j = cj; sl->lock = nullptr;
    sl->cross = e.j >= 0 && p.workers[e.j].rank != p.my_rank;
    if (sl->cross && p.two_sided) post_push_request(p, sl, w, e.j, seq);
    sl->coop = sl->cross && p.coop;
    sl->commit_ready = 0u;
    if (sl->coop) sl->gseq = (ld_acquire_sys(&p.workers[e.j].ctl->guest_tag) >> 2) + 1u;
    sl->ev_cur = cur + 1;
    sl->t0 = now;
    sl->done = 0;
    publish_running(sl, seq);
    if (sl->coop) post_guest(p, sl, w, e.j);
    return true;
  }
  // ------------------------------------------------------- free-running ----
  if (p.wait_free) return start_wait_free(p, sl, tag, w, now);
  int j = -1;
  unsigned int* lock;
  if (dw.role == 0 && dw.nb_cnt > 0) {
    j = sl->pending_j;
    if (j < -1) {
      const uint4 r = philox4x32_10(make_uint4((uint32_t)w, sl->nb_ctr, 0x4E424F52u, 0u), p.seed);
      j = p.nbrs[dw.nb_off + (int)(((unsigned long long)r.x * (unsigned)dw.nb_cnt) >> 32)];
      sl->pending_j = j;
    }
    lock = &p.workers[j].ctl->lock;
  } else {                                                  // passive (or isolated): local update
    if (p.model == 0) {                                     // pure gossip: passives only serve
      st_release_gpu(&sl->tag, tag_of(seq, kStateFinished));
      return true;
    }
    if (p.fuse && p.fuse_wait_ns && now < *(volatile unsigned long long*)&sl->ready_ns + p.fuse_wait_ns) {
      // stay due but idle for a while: an active that takes our lock now runs
      // this step inside its pair pass (only if some neighbour lives on this GPU)
      bool local_nb = false;
      for (int t = 0; t < dw.nb_cnt && !local_nb; ++t) local_nb = p.workers[p.nbrs[dw.nb_off + t]].local >= 0;
      if (local_nb) {
        st_release_gpu(&sl->tag, tag);
        return false;
      }
    }
    lock = &dw.ctl->lock;
  }
  if (atomicCAS_system(lock, 0u, 1u) != 0u) {              // busy: stay pending, never block
    st_release_gpu(&sl->tag, tag);
    return false;
  }
  __threadfence_system();                                   // acquire the previous holder's data
  // Fusion: holding the passive's lock, take over the passive's own pending
  // local step if it is due (its slot idle and its compute phase over): event
  // k is x_j's local update, event k+1 this pair, both in ONE pass (16d bytes
  // instead of 8d + 16d).  Ticket order = lock order, so the log replays as is.
  int absorb = -1;
  unsigned int tj = 0u;
  if (p.fuse && j >= 0 && p.model != 0) {
    const int lj = p.workers[j].local;
    if (lj >= 0) {
      Slot* sj = p.slots + lj;
      tj = ld_acquire_gpu(&sj->tag);
      if ((tj & 3u) == kStateIdle && now >= *(volatile unsigned long long*)&sj->ready_ns &&
          atomicCAS(&sj->tag, tj, tag_of(tj >> 2, kStateClaimed)) == tj)
        absorb = lj;
    }
  }
  unsigned long long k;
  const int got = take_tickets(p, &k, absorb >= 0 ? 2 : 1);
  if (absorb >= 0 && got < 2) {                             // one ticket left: the pair runs alone
    st_release_gpu(&p.slots[absorb].tag, tj);
    absorb = -1;
  }
  if (got == 0) {
    __threadfence_system();
    atomicExch_system(lock, 0u);
    st_release_gpu(&sl->tag, tag_of(seq, kStateFinished));
    return true;
  }
  if (absorb >= 0) ++k;                                     // the pair is the second event
  sl->absorb = absorb;
  sl->i = w; sl->j = j; sl->tau = 0; sl->flags = p.model == 0 ? 1u : 0u; sl->k = (long long)k;
  sl->kind = kKindEvent; sl->key = k; sl->g = nullptr;
  sl->xi = dw.x; sl->xj = j >= 0 ? p.workers[j].x : nullptr;
  sl->ctl_i = dw.ctl; sl->ctl_j = j >= 0 ? p.workers[j].ctl : nullptr; sl->lock = lock;
  sl->cross = j >= 0 && p.workers[j].rank != p.my_rank;
  if (sl->cross && p.two_sided) post_push_request(p, sl, w, j, seq);
  sl->coop = sl->cross && p.coop;
  sl->commit_ready = 0u;
  if (sl->coop) sl->gseq = (ld_acquire_sys(&p.workers[j].ctl->guest_tag) >> 2) + 1u;
  sl->pending_j = -2;
  sl->nb_ctr += 1;
  sl->t0 = now;
  sl->done = 0;
  publish_running(sl, seq);
  if (sl->coop) post_guest(p, sl, w, j);
  return true;
}

// Called by tid 0 of the CTA that finished the last slice of slot s.
__device__ __noinline__ void commit(const EngineParams& p, int s) {
  Slot* sl = p.slots + s;
  __threadfence_system();                 // every slice's stores (fenced by their CTAs) first
  const unsigned long long now = globaltimer();
  const double d4 = 4.0 * (double)p.d;
  if (sl->kind == kKindPull) {            // App. A: g' computed; its compute phase starts now
    volatile WorkerCtl* cw = sl->ctl_i;
    cw->wf_ready_ns = now + (unsigned long long)((double)p.workers[sl->i].straggle * (double)p.compute_ns);
    cw->wf_state = 1u;
    atomicAdd(&p.gctl->st_bytes, (sl->g ? 3.0 : 2.0) * d4);
    atomicAdd(&p.gctl->st_busy_ns, now - sl->t0);
    if (sl->lock) { __threadfence_system(); atomicExch_system(sl->lock, 0u); }
    const unsigned int seq = sl->tag >> 2;
    st_release_gpu(&sl->tag, tag_of(seq, kStateIdle));
    return;
  }
  const int i = sl->i, j = sl->j;
  const unsigned int flags = sl->flags;
  const long long k = sl->k;
  const bool grad = !(flags & 1u) && p.model != 0;
  if (p.wait_free && grad) ((volatile WorkerCtl*)sl->ctl_i)->wf_pub = 0u;   // buffer flushed (g <- 0)
  if (grad) atomicAdd(&sl->ctl_i->updates, 1ull);
  if (j >= 0) atomicAdd(&sl->ctl_i->gossips, 1ull);
  // event log (rank 0's ring; a P2P store when this rank is not 0)
  LogEntry* le = p.log + (k % p.log_cap);
  le->k = k; le->i = i; le->j = j; le->tau = sl->tau; le->flags = flags;
  le->t0 = sl->t0; le->t1 = now;
  const int ab = sl->absorb;
  if (ab >= 0) {                          // the fused passive step: event k-1 = (j, -1), W = I
    atomicAdd(&sl->ctl_j->updates, 1ull);
    LogEntry* lj = p.log + ((k - 1) % p.log_cap);
    lj->k = k - 1; lj->i = j; lj->j = -1; lj->tau = 0; lj->flags = 0u;
    lj->t0 = sl->t0; lj->t1 = now;
    atomicAdd(&p.gctl->st_events, 1ull);
    atomicAdd_system(&p.gctl0->committed, 1ull);
    Slot* sj = p.slots + ab;              // the passive's next compute phase starts now
    sj->ready_ns = now + (unsigned long long)((double)p.workers[j].straggle * (double)p.compute_ns);
    sl->absorb = -1;
    __threadfence();
    st_release_gpu(&sj->tag, tag_of(sj->tag >> 2, kStateIdle));
  }
  // stats: algorithmic bytes: pair 16d, local 8d; NVLink 8d per cross
  // pair; a flushed App. A buffer adds its 4d read; a fused passive step adds
  // nothing (its row is already read and written by the pair)
  atomicAdd(&p.gctl->st_events, 1ull);
  if (j >= 0) atomicAdd(&p.gctl->st_pair, 1ull);
  // a cross pair's rows live on two GPUs: each HBM moves its own row (2 rows of
  // the 4), the partner's share is credited to the partner's WorkerCtl
  if (sl->cross) {
    atomicAdd(&p.gctl->st_cross, 1ull);
    atomicAdd(&p.gctl->st_nvl_bytes, 2.0 * d4);
    atomicAdd_system(&p.workers[j].ctl->peer_bytes, 2.0 * d4);
  }
  atomicAdd(&p.gctl->st_bytes,
            ((j >= 0 ? (sl->cross ? 2.0 : 4.0) : (grad ? 2.0 : 0.0)) + (sl->g && grad ? 1.0 : 0.0)) * d4);
  atomicAdd(&p.gctl->st_busy_ns, now - sl->t0);
  if (sl->cross) atomicAdd(&p.gctl->st_busy_cross_ns, now - sl->t0);
  __threadfence_system();                 // log + data before the release below
  if (sl->coop) {
    // every tile of both GPUs is done: clear the partner's mailbox BEFORE the
    // partner is released (epoch / lock), or the next initiator's post -- maybe
    // from another GPU -- could be overwritten by this clear
    st_release_sys(&p.workers[j].ctl->guest_tag, tag_of(sl->gseq, kStateIdle));
    sl->coop = 0;
    __threadfence_system();   // the clear must be visible before the release below (a relaxed
                              // unlock / epoch bump is not ordered after a release store)
  }
  if (p.mode == 1) {
    atomicAdd_system(&sl->ctl_i->epoch, 1u);
    if (j >= 0) atomicAdd_system(&sl->ctl_j->epoch, 1u);
    atomicAdd_system(&p.gctl0->ticket, 1ull);
  } else {
    // slow link (R21): the transfer over the slower endpoint's link takes L x
    // link_ns; both workers stay busy and the passive stays locked until then
    float L = 1.0f;
    if (j >= 0) L = fmaxf(p.workers[i].link, p.workers[j].link);
    const unsigned long long hold = L > 1.0f ? (unsigned long long)((double)(L - 1.0f) * (double)p.link_ns) : 0ull;
    if (hold) {
      sl->held_lock = sl->lock;
      sl->unlock_at = now + hold;
    } else {
      atomicExch_system(sl->lock, 0u);
    }
    const float sw = p.workers[i].straggle;
    // Alg. 1 loop: the next gradient is computed before the next event; in the
    // App. A runtime the communication thread never waits for it
    sl->ready_ns = now + hold + (p.wait_free ? 0ull : (unsigned long long)((double)sw * (double)p.compute_ns));
  }
  atomicAdd_system(&p.gctl0->committed, 1ull);
  const unsigned int seq = sl->tag >> 2;
  st_release_gpu(&sl->tag, tag_of(seq, kStateIdle));
}

// tile x stages, fixed-mix A/B (tools/ab_engine.py, mixed / local-only GB/s):
// 512x4 5356/4774, 1024x3 5488/5129, 1536x2 5589/5109, 2048x2 5491/5010 (2048x2
// needs 128 KB: one CTA per SM).  Whole bench (tools/ab_build.py + bench.py
// --no-extras, 3 runs each): 1536x2 0.869-0.871 of the HBM peak, 1024x3
// 0.863-0.867, 512x6 0.819-0.824.
#ifndef ADPSGD_TILE4
#define ADPSGD_TILE4 1536
#endif
#ifndef ADPSGD_STAGES
#define ADPSGD_STAGES 2
#endif
constexpr int kTile4 = ADPSGD_TILE4;     // float4 per stream per stage (24 KB)
constexpr int kStages = ADPSGD_STAGES;
constexpr size_t kTmaSmem = (size_t)kStages * 2 * kTile4 * sizeof(float4) + 2 * kStages * sizeof(uint64_t);

// engine variants: 0 = bulk-copy staged, CTA barrier per tile (default);
// 1 = register slices (no staging, one-sided cross access); 2 = bulk-copy
// staged, per-warp empty mbarriers.  tools/ab_engine.py on a fixed 512-event
// mix at d = 25.6M: 5404 / 4996 / 5324 GB/s (variant 0 / 1 / 2).
template <int kVar>
using EngineStager = Stager<kTile4, kStages, kVar == 2>;

template <int kVar, bool kPair, int kGrad, bool kFF = false, bool kPreJ = false>
__device__ __forceinline__ void slice(const EngineParams& p, const SmemSlot& e, EngineStager<kVar>& stg) {
  const uint32_t kk = quad_event_key_h(p.q.noise_key, e.key);
  const uint32_t kkj = kPreJ ? quad_event_key_h(p.q.noise_key, e.key - 1ull) : 0u;   // the passive's event k-1
  float4* xi4 = reinterpret_cast<float4*>(e.xi);
  float4* xj4 = reinterpret_cast<float4*>(e.xj);
  const float4* g4 = reinterpret_cast<const float4*>(e.g);
  if (kVar != 1) {
    if (e.cross && p.two_sided)             // consume landed tiles [t0, t1); average back to x_j
      stg.template run_range<kPair, kGrad, kFF>(xi4, reinterpret_cast<const float4*>(e.land), xj4, blockIdx.x,
                                                gridDim.x, p.n4, e.t0, e.t1, p.d, p.gamma, p.q, kk, g4);
    else
      stg.template run<kPair, kGrad, kFF, kPreJ>(xi4, xj4, e.first, e.step, p.n4, p.d, p.gamma, p.q, kk, g4, kkj);
  } else {
    const long long per = (p.n4 + gridDim.x - 1) / gridDim.x;
    const long long lo = (long long)blockIdx.x * per;
    const long long hi = lo + per < p.n4 ? lo + per : p.n4;
    event_range<kPair, kGrad, kEngineUnroll, kFF>(xi4, xj4, g4, nullptr, lo, hi, threadIdx.x, blockDim.x, p.d,
                                                  p.gamma, p.q, kk);
  }
}

template <int kVar>
__global__ void __launch_bounds__(kEngineThreads, 2) k_engine(const __grid_constant__ EngineParams p) {
  extern __shared__ __align__(128) unsigned char dyn_smem[];
  __shared__ unsigned int done_seq[kMaxLocal];   // last event seq this CTA finished, per slot
  __shared__ unsigned int push_seq[kMaxLocal];   // last push request seq this CTA served, per worker
  __shared__ unsigned int cons_seq[kMaxLocal];   // event seq cons_cnt refers to
  __shared__ unsigned int cons_cnt[kMaxLocal];   // tiles of a cross event consumed so far
  __shared__ unsigned int gdone_seq[kMaxLocal];  // last guest event seq this CTA finished, per mailbox
  __shared__ int s_pick;
  __shared__ unsigned int s_seq;
  __shared__ SmemSlot s_ev;
  EngineStager<kVar> stg;
  stg.buf = reinterpret_cast<float4*>(dyn_smem);
  stg.bar = reinterpret_cast<uint64_t*>(dyn_smem + (size_t)kStages * 2 * kTile4 * sizeof(float4));
  stg.empty = stg.bar + kStages;
  stg.consumed = 0;
  if (kVar != 1 && threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(stg.bar + s, 1);
      mbar_init(stg.empty + s, kEngineThreads / 32);
    }
    mbar_fence_init();
  }
  for (int s = threadIdx.x; s < kMaxLocal; s += blockDim.x) {
    done_seq[s] = 0u;
    cons_seq[s] = 0u;
    cons_cnt[s] = 0u;
    gdone_seq[s] = 0u;
    push_seq[s] = 0xffffffffu;
  }
  __syncthreads();
  if (p.two_sided)                           // push requests this CTA served in earlier launches
    for (int l = threadIdx.x; l < p.n_local; l += blockDim.x) push_seq[l] = p.served[l * kMaxGrid + blockIdx.x];
  __syncthreads();
  const int L = p.n_local;
#ifdef ADPSGD_ROT0
  const int rot = 0;                         // A/B: every CTA prefers the same running event
#else
  const int rot = L ? (int)(blockIdx.x % (unsigned)L) : 0;
#endif
  const long long my_tiles = EngineStager<kVar>::tiles_of(blockIdx.x, gridDim.x, p.n4);
  // An event of fewer tiles than CTAs (small d) is taken by `part` CTAs only,
  // rotated by the slot index so that concurrent small events use disjoint CTAs;
  // the others neither pick it up nor arrive on its counter.
#ifndef ADPSGD_MIN_TILES_PER_CTA
#define ADPSGD_MIN_TILES_PER_CTA 4   // config 2 A/B (d = 2^20): 1 -> 79k, 2 -> 91k, 4 -> 96k, 8 -> 92k replay events/s
#endif
  const int tiles_ev = (int)((p.n4 + kTile4 - 1) / kTile4);
  const int want = (tiles_ev + ADPSGD_MIN_TILES_PER_CTA - 1) / ADPSGD_MIN_TILES_PER_CTA;
  const int part = (kVar == 1 || want >= (int)gridDim.x) ? (int)gridDim.x : (want > 0 ? want : 1);
  // A cross-GPU event is bound by NVLink (~1/8 of HBM), so it is given a
  // fraction of the CTAs (rotated by slot, like small events): the rest keep
  // streaming local events from HBM meanwhile instead of every CTA stalling on
  // its share of the remote tiles.  Both GPUs of a cooperative event use the same
  // fraction (same grid), so the arrival count is 2 * xpart.
#ifndef ADPSGD_CROSS_RESERVE
#define ADPSGD_CROSS_RESERVE 0   // A/B (tools/ab_reserve.sh): 1 -> N=2 13.5k vs 14.5k, N=4 26.5k vs 28.4k (dropped)
#endif
  constexpr bool kReserve = ADPSGD_CROSS_RESERVE != 0;
#ifndef ADPSGD_CROSS_DIV
#define ADPSGD_CROSS_DIV 4   // N=2 A/B (bench --no-extras, coop auto): 1 -> 14.17k, 2 -> 14.44k, 4 -> 14.58k, 8 -> 14.05k gossip-steps/s
#endif
  const int xpart = kVar == 1 ? (int)gridDim.x
                    : max(1, min(part, (int)gridDim.x / (ADPSGD_CROSS_DIV > 1 ? ADPSGD_CROSS_DIV : 1)));
  unsigned long long last_progress = globaltimer();
  while (true) {
    if (threadIdx.x == 0) {
      int pick = -1;
      if (ld_acquire_gpu(&p.gctl->abort_flag)) pick = kExit;
      // 1. push requests from other GPUs (they unblock remote consumers; never wait)
      if (p.two_sided)
        for (int t = 0; t < L && pick == -1; ++t) {
          const int l = (t + rot) % L;
          WorkerCtl* c = p.workers[p.local_ids[l]].ctl;
          const unsigned int tag = ld_acquire_sys(&c->req_tag);
          if ((tag & 3u) == kStateRunning && (tag >> 2) != push_seq[l]) {
            const int ci = *(volatile int*)&c->req_consumer;
            s_ev.src = p.workers[p.local_ids[l]].x;
            s_ev.dst = p.workers[ci].land;
            s_ev.cnt = p.workers[ci].pcnt + blockIdx.x;
            s_ev.tag16 = *(volatile unsigned int*)&c->req_tag16;
            s_seq = tag >> 2;
            pick = kPickPush + l;
          }
        }
      auto scan_guests = [&]() {
        // 2b. cooperative events of peer GPUs posted in our workers' mailboxes
        if (p.coop)
          for (int t = 0; t < L && pick == -1; ++t) {
            const int l = (t + rot) % L;
            const int wl = p.local_ids[l];
            WorkerCtl* cl = p.workers[wl].ctl;
            const unsigned int gt = ld_acquire_sys(&cl->guest_tag);
            if ((gt & 3u) != kStateRunning || (gt >> 2) == gdone_seq[l]) continue;
            int grb = (int)blockIdx.x;
            if (xpart < (int)gridDim.x) {
              const int base = kReserve && p.reserve ? (int)gridDim.x - xpart
                                                     : (int)(((unsigned int)l * (unsigned int)xpart) % gridDim.x);
              grb = (int)((blockIdx.x + gridDim.x - base) % gridDim.x);
              if (grb >= xpart) { gdone_seq[l] = gt >> 2; continue; }  // not one of this event's CTAs
            }
            const int gi = *(volatile int*)&cl->guest_i;
            Slot* sa = p.workers[gi].slot;                 // the initiator's slot (peer memory)
            const unsigned int fl = *(volatile unsigned int*)&sa->flags;
            s_ev.xi = p.workers[gi].x;
            s_ev.xj = p.workers[wl].x;
            s_ev.k = *(volatile long long*)&sa->k;
            s_ev.key = *(volatile unsigned long long*)&sa->key;
            s_ev.grad = (!(fl & 1u) && p.model != 0) ? 1 : 0;
            s_ev.ff = (fl & 2u) ? 1 : 0;
            s_ev.kind = kKindEvent;
            s_ev.g = nullptr;
            s_ev.gout = nullptr;
            s_ev.absorb = 0;
            s_ev.pair = 1;
            s_ev.cross = 1;
            s_ev.t0 = s_ev.t1 = 0;
            s_ev.coop = 1;
            s_ev.first = (long long)xpart + grb;
            s_ev.step = 2ll * xpart;
            s_ev.ncta = 2 * xpart;
            s_ev.guest = 1;
            s_ev.gl = l;
            s_ev.gdone = &sa->done;
            s_ev.gready = &sa->commit_ready;
            s_seq = gt >> 2;
            pick = kPickGuest;
          }
      };
#ifdef ADPSGD_GUEST_FIRST
      scan_guests();
#endif
      // 2. running events with work for this CTA
      for (int t = 0; t < L && pick == -1; ++t) {
        const int s = (t + rot) % L;
        const unsigned int tag = ld_acquire_gpu(&p.slots[s].tag);
        if (p.coop && (tag & 3u) == kStateRunning && *(volatile int*)&p.slots[s].coop) {
          const unsigned int g = *(volatile unsigned int*)&p.slots[s].gseq;
          if (ld_acquire_sys(&p.slots[s].commit_ready) == g && atomicCAS(&p.slots[s].commit_ready, g, 0u) == g) {
            commit(p, s);                                   // last arrival was on the partner GPU
            continue;
          }
        }
        if ((tag & 3u) != kStateRunning || (tag >> 2) == done_seq[s]) continue;
        Slot* sl = p.slots + s;
        int rb = (int)blockIdx.x;
        const int cross = *(volatile int*)&sl->cross;
        const int coop = *(volatile int*)&sl->coop;
        // CTAs that take this event: all, `part` (small d) or `xpart` (cross-GPU, one-sided or cooperative)
        int evp = (cross && !p.two_sided) ? xpart : ((!coop && !(p.two_sided && cross)) ? part : (int)gridDim.x);
        int base = (int)(((unsigned int)s * (unsigned int)evp) % gridDim.x);
        if (kReserve && p.reserve && xpart < (int)gridDim.x) {
          // cross events keep to the last xpart CTAs and large local events to the
          // others, so a CTA busy on NVLink never holds up a local event's arrival
          if (cross) base = (int)gridDim.x - xpart;
          else if (evp == (int)gridDim.x) { evp = (int)gridDim.x - xpart; base = 0; }
        }
        if (evp < (int)gridDim.x) {
          rb = (int)((blockIdx.x + gridDim.x - base) % gridDim.x);
          if (rb >= evp) { done_seq[s] = tag >> 2; continue; }    // not one of this event's CTAs
        }
        long long t0 = 0, t1 = 0;
        if (cross && p.two_sided && kVar != 1) {
          if (cons_seq[s] != (tag >> 2)) { cons_seq[s] = tag >> 2; cons_cnt[s] = 0u; }
          const unsigned int tag16 = *(volatile unsigned int*)&sl->tag16;
          unsigned int avail = 0;
          if (my_tiles > 0) {
            const unsigned int v = ld_acquire_sys(*(unsigned int* volatile*)&sl->pcnt + blockIdx.x);
            avail = (v >> 16) == tag16 ? (v & 0xffffu) : 0u;
            if (avail <= cons_cnt[s]) continue;              // nothing landed yet: look elsewhere
          }
          t0 = cons_cnt[s];
          t1 = avail;
          s_ev.land = *(float* volatile*)&sl->land;
        }
        pick = s;
        s_seq = tag >> 2;
        s_ev.xi = *(float* volatile*)&sl->xi;
        s_ev.xj = *(float* volatile*)&sl->xj;
        s_ev.k = *(volatile long long*)&sl->k;
        const unsigned int fl = *(volatile unsigned int*)&sl->flags;
        s_ev.grad = (!(fl & 1u) && p.model != 0) ? 1 : 0;
        s_ev.ff = (fl & 2u) ? 1 : 0;
        s_ev.kind = *(volatile int*)&sl->kind;
        s_ev.key = *(volatile unsigned long long*)&sl->key;
        s_ev.g = *(float* volatile*)&sl->g;
        s_ev.gout = *(float* volatile*)&sl->gout;
        s_ev.absorb = *(volatile int*)&sl->absorb >= 0 ? 1 : 0;
        s_ev.pair = s_ev.xj != nullptr;
        s_ev.cross = cross;
        s_ev.t0 = t0;
        s_ev.t1 = t1;
        s_ev.coop = coop;
        s_ev.first = rb;
        s_ev.step = coop ? 2ll * evp : (long long)evp;
        s_ev.ncta = coop ? 2 * evp : evp;
        s_ev.guest = 0;
      }
#ifndef ADPSGD_GUEST_FIRST
      scan_guests();
#endif
      // 3. scheduler duty
      if (pick == -1) {
        const unsigned long long now = globaltimer();
        int n_fin = 0;
        bool progress = false;
        for (int t = 0; t < L; ++t) {
          const int s = (t + rot) % L;
          const unsigned int tag = ld_acquire_gpu(&p.slots[s].tag);
          const unsigned int st = tag & 3u;
          if (st == kStateFinished) ++n_fin;
          else if (st == kStateIdle) progress |= try_start(p, s, tag, now);
        }
        // local work done; with cross-GPU partners stay to serve push requests
        // until every event of the run is committed system-wide
        if (n_fin == L && (!(p.two_sided || p.coop) || ld_relaxed_sys64(&p.gctl0->committed) >= p.target))
          pick = kExit;
        if (progress) last_progress = now;
        else if (now - last_progress > p.watchdog_ns) { latch_error(p, 7u); pick = kExit; }
      } else {
        last_progress = globaltimer();
      }
      s_pick = pick;
    }
    __syncthreads();
    const int pick = s_pick;
    if (pick == kExit) break;
    if (pick >= kPickPush) {
      const SmemSlot& e = s_ev;      // stable until the trailing barrier
      if (kVar != 1)
        stg.push(reinterpret_cast<const float4*>(e.src), reinterpret_cast<float4*>(e.dst), e.cnt, e.tag16,
                 blockIdx.x, gridDim.x, p.n4);
      __syncthreads();
      if (threadIdx.x == 0) push_seq[pick - kPickPush] = s_seq;
    } else if (pick >= 0) {
      const SmemSlot& e = s_ev;      // stable until the trailing barrier
      if (e.kind == kKindPull) {
        if (kVar != 1)
          stg.pull(reinterpret_cast<const float4*>(e.xi), reinterpret_cast<const float4*>(e.g),
                   reinterpret_cast<float4*>(e.gout), e.first, e.step, p.n4, p.d, p.gamma, p.q,
                   quad_event_key_h(p.q.noise_key, e.key));
      } else if (kVar != 1 && e.g) {        // App. A flush of the buffered gradient (staged variants)
        if (e.pair) slice<kVar, true, kGradExternal, true>(p, e, stg);
        else slice<kVar, false, kGradExternal>(p, e, stg);
      } else if (e.pair) {
        if (e.grad) {
          if (kVar != 1 && e.ff) slice<kVar, true, kGradQuadInline, true>(p, e, stg);
          else if (kVar != 1 && e.absorb) slice<kVar, true, kGradQuadInline, false, true>(p, e, stg);
          else slice<kVar, true, kGradQuadInline>(p, e, stg);
        } else {
          slice<kVar, true, kGradNone>(p, e, stg);
        }
      } else if (e.grad) {
        slice<kVar, false, kGradQuadInline>(p, e, stg);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        bool finished = true;
        if (e.cross && p.two_sided && kVar != 1) {
          cons_cnt[pick] = (unsigned int)e.t1;
          finished = e.t1 >= my_tiles;
        }
        if (finished && e.guest) {          // our half of a peer's cooperative event
          gdone_seq[e.gl] = s_seq;
          __threadfence_system();
          if (atomicAdd_system(e.gdone, 1u) == (unsigned int)e.ncta - 1u) st_release_sys(e.gready, s_seq);
        } else if (finished) {
          done_seq[pick] = s_seq;
          // this CTA's slice is visible before its arrival; P2P stores need the
          // system-scope fence, local ones only gpu scope (the committing CTA
          // issues fence.sys before the cross-GPU release, which is cumulative)
          if (e.cross) __threadfence_system();
          else __threadfence();
          if (e.coop) {
            if (atomicAdd_system(&p.slots[pick].done, 1u) == (unsigned int)e.ncta - 1u) commit(p, pick);
          } else if (atomicAdd(&p.slots[pick].done, 1u) == (unsigned int)e.ncta - 1u) {
            commit(p, pick);
          }
        }
      }
    } else if (threadIdx.x == 0) {
      __nanosleep(256);
    }
    __syncthreads();
  }
  if (p.two_sided)
    for (int l = threadIdx.x; l < p.n_local; l += blockDim.x) p.served[l * kMaxGrid + blockIdx.x] = push_seq[l];
}

const void* engine_fn(int variant, size_t* smem) {
  switch (variant) {
    case 1: *smem = 0; return (const void*)k_engine<1>;
    case 2: *smem = kTmaSmem; return (const void*)k_engine<2>;
    default: *smem = kTmaSmem; return (const void*)k_engine<0>;
  }
}

}  // namespace

int engine_max_ctas_per_sm(int threads, int variant) {
  int n = 0;
  size_t smem = 0;
  const void* fn = engine_fn(variant, &smem);
  if (smem) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, threads, smem);
  return n;
}

cudaError_t launch_engine(const EngineParams& p, int grid, int threads, bool cooperative, cudaStream_t s) {
  EngineParams pp = p;
  void* args[] = {&pp};
  if (threads != kEngineThreads || grid > kMaxGrid) return cudaErrorInvalidValue;
  size_t smem = 0;
  const void* fn = engine_fn(p.variant, &smem);
  if (smem) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (cooperative) return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(threads), args, smem, s);
  return cudaLaunchKernel(fn, dim3(grid), dim3(threads), args, smem, s);
}

const void* engine_module_anchor() { return (const void*)k_engine<0>; }

}  // namespace adp
