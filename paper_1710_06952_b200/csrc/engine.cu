// engine.cu -- the persistent AD-PSGD engine: one persistent kernel per GPU
// runs every local worker's loop of the asynchronous runtime on the device,
// with no host round trip per event.
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
//      the virtual counter of P:429-432 (reading R23), taken while holding the
//      lock so the ticket order is the serialisation order (log replay).
//   4. fused pass over d: m = fl(fl(x_w + x_j)*0.5); x_j <- m;
//      x_w <- fl(m - fl(gamma g)), g = the quadratic gradient at the pre-average
//      x_w (tau = 0) -- Alg. 1 steps 4-6, reading R1.
//   5. the CTA whose leave finishes the event commits: log {k,i,j,0}, counters,
//      release fence (sys), unlock, schedule the next compute phase.
// Replay mode (mode 1): the op list of each local worker is consumed in order;
// an op starts when epoch[i] == e_i and epoch[j] == e_j (device epoch flags,
// system scope) and bumps both epochs at commit.  A stale read (tau > 0,
// X_hat = X_{k - tau}) is its own op, placed in worker i's sequence
// where X_{k - tau} holds: it computes the gradient into one of the worker's
// T + 1 read rows, which the event applies later.
//
// Work distribution: an event's float4 range is cut into tiles of kTile4; the
// CTAs that join an event claim tile chunks from its claim word until none is
// left (TileClaim), so a CTA held up on NVLink never delays a local event's
// tiles.  A claim is one atomicAdd that also names the event (sequence tag):
// owning an uncredited chunk pins the event -- it cannot commit, nor its slot
// be reused, while the CTA still reads its fields -- and the CTA whose credit
// brings the event's remaining tiles to zero commits.  (A CAS-based join pin
// cost 0.80 vs 0.93 of the HBM peak: 296 CTAs retrying one word per event.)
// A cross-GPU event is joined by at most grid / kCrossDiv CTAs per GPU (it is
// NVLink-bound); with cooperative events the partner GPU claims the odd tiles
// (its half) from its own mailbox claim word.
#include "internal.h"

namespace adp {

namespace {

constexpr int kEngineThreads = 512;
constexpr int kExit = -2;
constexpr int kPickGuest = 1 << 20;     // a peer's cooperative event posted in a local mailbox
constexpr int kTile4 = 1536;            // float4 per stream per stage (24 KB); round-1 A/B: 1536x2 stages
                                        // 0.869-0.871 of the HBM peak vs 1024x3 0.863-0.867, 512x6 0.82
constexpr int kStages = 2;
constexpr int kClaimChunk = 8;          // tiles per claimed chunk, at most (A/B at N=1: 4 -> 0.907, 8 -> 0.930,
                                        // 16 -> 0.928 of peak); small events use smaller chunks so that up to
                                        // one chunk per CTA spreads them over the whole grid
constexpr bool kRotate = true;          // CTA b scans slots from b mod L (else every CTA from slot 0)
constexpr int kCrossDiv = 8;            // CTAs per GPU on one cross-GPU event: grid / 8 (round-2 A/B, claim engine,
                                        // bench --no-extras: 2 / 4 / 8 -> N=2 0.835 / 0.864 / 0.890, N=4 0.815 /
                                        // 0.849 / 0.881 of the HBM peak; round-1 static engine at
                                        // N=2: 1 -> 14.17k, 2 -> 14.44k, 4 -> 14.58k, 8 -> 14.05k steps/s)
constexpr size_t kTmaSmem = (size_t)kStages * 2 * kTile4 * sizeof(float4) + kStages * sizeof(uint64_t);
using EngineStager = Stager<kTile4, kStages>;
using Claim = TileClaim;
constexpr int kPer = kTile4 / 512;

struct SmemSlot {                  // tid 0 copies the joined event here for the CTA
  float* xi;
  float* xj;
  int grad;
  int pair;
  int cross;                       // partner row lives on another GPU (peer loads / stores)
  int ff;                          // App. A order (flush first)
  int kind;
  unsigned long long key;
  const float* g;
  float* gout;
  int absorb;                      // fused passive local step (event k-1) before the pair
  // this CTA's claim on the event: tile c of its share is c * stride + off
  unsigned long long* ctr;
  unsigned int n, stride, off;
  unsigned int first;              // the chunk the join's claim returned
  unsigned int nc;                 // the claim word's chunk count
  unsigned int* rem;               // the initiator slot's remaining tiles (peer memory for a guest)
  int guest;                       // a peer's cooperative event (our half)
  int slot;                        // local slot (own events) or mailbox index (guest)
  unsigned int seq;                // the slot's / mailbox's sequence
  unsigned int* gready;            // initiator's slot->commit_ready (peer; guest events)
};

__device__ __forceinline__ unsigned int tag_of(unsigned int seq, unsigned int st) { return (seq << 2) | st; }

__device__ void latch_error(const EngineParams& p, unsigned int code) {
  atomicCAS(&p.gctl->error, 0u, code);
  atomicExch(&p.gctl->abort_flag, 1u);
}

__device__ __forceinline__ unsigned int event_tiles(const EngineParams& p) {
  return (unsigned int)((p.n4 + kTile4 - 1) / kTile4);
}

// Credit `tiles` finished tiles to an event; true if they were its last ones.
// System scope: a partner GPU credits its half of a cooperative event too.
__device__ __forceinline__ bool credit(unsigned int* rem, unsigned int tiles) {
  return atomicAdd_system(rem, 0u - tiles) == tiles;
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

// Make the slot's event (fields already written) visible as running: fresh
// claim word (new seq, chunk count), remaining tiles, then the tag.
// chunks a share of `share` tiles is dealt in: chunk = clamp(T / grid, 1, kClaimChunk)
__device__ __forceinline__ unsigned int share_chunks(const EngineParams& p, unsigned int share) {
  const unsigned int per = event_tiles(p) / gridDim.x;
  const unsigned int chunk = per < 1u ? 1u : (per > (unsigned)kClaimChunk ? (unsigned)kClaimChunk : per);
  return (share + chunk - 1) / chunk;
}

__device__ void publish_running(const EngineParams& p, Slot* sl, unsigned int seq) {
  const unsigned int T = event_tiles(p);
  const unsigned int share = sl->coop ? (T + 1u) / 2u : T;
  sl->nwork = 0u;
  sl->ntiles = T;
  sl->commit_ready = 0u;
  sl->rem = T;
  __threadfence();                                   // fields before the claim word (a claim reads them)
  *(volatile unsigned long long*)&sl->next = claim_word(seq + 1, share_chunks(p, share));
  __threadfence_system();                            // ... and before the tag (a guest reads them)
  st_release_gpu(&sl->tag, tag_of(seq + 1, kStateRunning));
}

// Cooperative cross-GPU event: after publishing event seq+1 in worker w's slot,
// post it in partner j's guest mailbox (j's home GPU) so that GPU's CTAs claim
// the odd tiles -- both GPUs then drive NVLink (reads of the other row and
// writes of the results in both directions) instead of one.  The mailbox has
// its own sequence (a partner serves events of several initiators); the poster
// holds the partner exclusively (its lock or its epoch), so read-increment is
// race-free.
__device__ void post_guest(Slot* sl, const EngineParams& p, int w, int j) {
  WorkerCtl* cj = p.workers[j].ctl;                   // peer memory
  *(volatile int*)&cj->guest_i = w;
  *(volatile unsigned int*)&cj->guest_nwork = 0u;
  __threadfence_system();                             // guest_i before the claim word
  *(volatile unsigned long long*)&cj->guest_next =
      claim_word(sl->gseq, share_chunks(p, event_tiles(p) / 2u));
  __threadfence_system();
  st_release_sys(&cj->guest_tag, tag_of(sl->gseq, kStateRunning));
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
    publish_running(p, sl, seq);
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
  sl->gout = nullptr;
  sl->xi = dw.x; sl->xj = j >= 0 ? p.workers[j].x : nullptr;
  sl->ctl_i = dw.ctl; sl->ctl_j = j >= 0 ? p.workers[j].ctl : nullptr; sl->lock = lock;
  sl->cross = j >= 0 && p.workers[j].rank != p.my_rank;
  if (j >= 0) { sl->pending_j = -2; sl->nb_ctr += 1; }
  sl->t0 = now;
  publish_running(p, sl, seq);
  return true;
}

// Called by tid 0 of some CTA that found no tile to work on.  Returns true if
// it started or finished a worker (progress).
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
    const long long dpad = p.n4 * 4;
    sl->i = w; sl->j = e.j; sl->tau = 0; sl->flags = e.flags; sl->k = e.k;
    sl->absorb = -1; sl->lock = nullptr;
    sl->xi = dw.x; sl->xj = e.j >= 0 ? p.workers[e.j].x : nullptr;
    sl->ctl_i = dw.ctl; sl->ctl_j = cj;
    sl->key = (e.flags & 2u) ? read_key((unsigned long long)e.k, w) : (unsigned long long)e.k;   // R20
    if (e.kind == kKindRead) {                              // stale read: g at X_{k - tau}
      sl->kind = kKindRead;
      sl->key = (unsigned long long)e.k;                    // e.k holds the read's key (plan_replay)
      sl->g = nullptr;
      sl->gout = dw.gr + (long long)e.grow * dpad;
      sl->xj = nullptr; sl->ctl_j = nullptr; sl->j = -1;
      sl->cross = 0; sl->coop = 0;
    } else {
      sl->kind = kKindEvent;
      sl->g = e.grow >= 0 ? dw.gr + (long long)e.grow * dpad : nullptr;   // read earlier by a kKindRead op
      sl->gout = nullptr;
      sl->cross = e.j >= 0 && p.workers[e.j].rank != p.my_rank;
      // a guest cannot read a gradient row (not peer-mapped): such events stay one-sided
      sl->coop = sl->cross && p.coop && !sl->g;
    }
    if (sl->coop) sl->gseq = (ld_acquire_sys(&p.workers[e.j].ctl->guest_tag) >> 2) + 1u;
    sl->ev_cur = cur + 1;
    sl->t0 = now;
    publish_running(p, sl, seq);
    if (sl->coop) post_guest(sl, p, w, e.j);
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
  sl->kind = kKindEvent; sl->key = k; sl->g = nullptr; sl->gout = nullptr;
  sl->xi = dw.x; sl->xj = j >= 0 ? p.workers[j].x : nullptr;
  sl->ctl_i = dw.ctl; sl->ctl_j = j >= 0 ? p.workers[j].ctl : nullptr; sl->lock = lock;
  sl->cross = j >= 0 && p.workers[j].rank != p.my_rank;
  sl->coop = sl->cross && p.coop;
  if (sl->coop) sl->gseq = (ld_acquire_sys(&p.workers[j].ctl->guest_tag) >> 2) + 1u;
  sl->pending_j = -2;
  sl->nb_ctr += 1;
  sl->t0 = now;
  publish_running(p, sl, seq);
  if (sl->coop) post_guest(sl, p, w, j);
  return true;
}

// Called by tid 0 of the CTA whose leave finished the event of slot s.
__device__ __noinline__ void commit(const EngineParams& p, int s) {
  Slot* sl = p.slots + s;
  __threadfence_system();                 // every tile's stores (fenced by their CTAs) first
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
  if (sl->kind == kKindRead) {            // replay stale read done: the worker's next op may run
    atomicAdd(&p.gctl->st_bytes, 2.0 * d4);
    atomicAdd(&p.gctl->st_busy_ns, now - sl->t0);
    __threadfence_system();
    atomicAdd_system(&sl->ctl_i->epoch, 1u);
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
  // pair; an applied gradient row adds its 4d read; a fused passive step adds
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

// The staged pass of one joined event over the tiles this CTA claims.
template <bool kPair, int kGrad, bool kFF = false, bool kPreJ = false>
__device__ __forceinline__ unsigned int event_pass(const EngineParams& p, const SmemSlot& e, EngineStager& stg,
                                                   Claim& cl) {
  EventBody<kPer, kPair, kGrad, kFF, kPreJ> body;
  body.xi4 = reinterpret_cast<float4*>(e.xi);
  body.xj4 = reinterpret_cast<float4*>(e.xj);
  body.g4 = reinterpret_cast<const float4*>(e.g);
  body.hi = p.n4;
  body.d = p.d;
  body.gamma = p.gamma;
  body.q = p.q;
  body.kk = quad_event_key_h(p.q.noise_key, e.key);
  body.kkj = kPreJ ? quad_event_key_h(p.q.noise_key, e.key - 1ull) : 0u;   // the passive's event k-1
  return stg.drive(cl, body.xi4, kPair ? body.xj4 : nullptr, p.n4, body);
}

__global__ void __launch_bounds__(kEngineThreads, 2) k_engine(const __grid_constant__ EngineParams p) {
  extern __shared__ __align__(128) unsigned char dyn_smem[];
  __shared__ unsigned int done_seq[kMaxLocal];   // last event seq this CTA is done with, per slot
  __shared__ unsigned int gdone_seq[kMaxLocal];  // last guest event seq this CTA is done with, per mailbox
  __shared__ int s_pick;
  __shared__ int s_stile[kStages];
  __shared__ SmemSlot s_ev;
  EngineStager stg;
  stg.buf = reinterpret_cast<float4*>(dyn_smem);
  stg.bar = reinterpret_cast<uint64_t*>(dyn_smem + (size_t)kStages * 2 * kTile4 * sizeof(float4));
  stg.stile = s_stile;
  stg.consumed = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(stg.bar + s, 1);
    mbar_fence_init();
  }
  for (int s = threadIdx.x; s < kMaxLocal; s += blockDim.x) {
    done_seq[s] = 0u;
    gdone_seq[s] = 0u;
  }
  __syncthreads();
  const int L = p.n_local;
  const int rot = (kRotate && L) ? (int)(blockIdx.x % (unsigned)L) : 0;
  const unsigned int T = event_tiles(p);
  const unsigned int xpart = max(1u, gridDim.x / (unsigned)kCrossDiv);
  Claim cl;                                     // thread 0's claim on the joined event
  unsigned long long last_progress = globaltimer();
  while (true) {
    if (threadIdx.x == 0) {
      int pick = -1;
      if (ld_acquire_gpu(&p.gctl->abort_flag)) pick = kExit;
      // 1. running events of local workers with tiles left to claim
      for (int t = 0; t < L && pick == -1; ++t) {
        const int s = (t + rot) % L;
        Slot* sl = p.slots + s;
        const unsigned int tag = ld_acquire_gpu(&sl->tag);
        if (p.coop && (tag & 3u) == kStateRunning && *(volatile int*)&sl->coop) {
          const unsigned int g = *(volatile unsigned int*)&sl->gseq;
          if (ld_acquire_sys(&sl->commit_ready) == g && atomicCAS(&sl->commit_ready, g, 0u) == g) {
            commit(p, s);                                   // the last leave was on the partner GPU
            continue;
          }
        }
        unsigned int seq = tag >> 2;
        if ((tag & 3u) != kStateRunning || seq == done_seq[s]) continue;
        const unsigned long long w0 = *(volatile unsigned long long*)&sl->next;
        if (claim_seq(w0) != (seq & kClaimSeqMask) || claim_idx(w0) >= claim_nc(w0)) { done_seq[s] = seq; continue; }
        if (*(volatile int*)&sl->cross && atomicAdd(&sl->nwork, 1u) >= xpart) { done_seq[s] = seq; continue; }
        const unsigned long long w = atomicAdd(&sl->next, 1ull);          // join = claim a chunk
        if (claim_idx(w) >= claim_nc(w)) { done_seq[s] = seq; continue; }
        // we own a chunk of event claim_seq(w): it is pinned and its fields are
        // stable until we credit the chunk (a newer event than `seq` if the slot
        // moved on meanwhile -- then the tag already shows it)
        __threadfence();
        if (claim_seq(w) != (seq & kClaimSeqMask)) seq = ld_acquire_gpu(&sl->tag) >> 2;
        const int coop = *(volatile int*)&sl->coop;
        const unsigned int share = coop ? (T + 1u) / 2u : T;
        s_ev.xi = *(float* volatile*)&sl->xi;
        s_ev.xj = *(float* volatile*)&sl->xj;
        const unsigned int fl = *(volatile unsigned int*)&sl->flags;
        s_ev.kind = *(volatile int*)&sl->kind;
        s_ev.grad = (!(fl & 1u) && p.model != 0) ? 1 : 0;
        s_ev.ff = (fl & 2u) ? 1 : 0;
        s_ev.key = *(volatile unsigned long long*)&sl->key;
        s_ev.g = *(float* volatile*)&sl->g;
        s_ev.gout = *(float* volatile*)&sl->gout;
        s_ev.absorb = *(volatile int*)&sl->absorb >= 0 ? 1 : 0;
        s_ev.pair = s_ev.xj != nullptr;
        s_ev.cross = *(volatile int*)&sl->cross;
        s_ev.ctr = &sl->next;
        s_ev.n = share;
        s_ev.stride = coop ? 2u : 1u;
        s_ev.off = 0u;
        s_ev.first = claim_idx(w);
        s_ev.nc = claim_nc(w);
        s_ev.rem = &sl->rem;
        s_ev.guest = 0;
        s_ev.slot = s;
        s_ev.seq = seq;
        pick = s;
      }
      // 2. cooperative events of peer GPUs posted in our workers' mailboxes
      if (p.coop)
        for (int t = 0; t < L && pick == -1; ++t) {
          const int l = (t + rot) % L;
          const int wl = p.local_ids[l];
          WorkerCtl* mb = p.workers[wl].ctl;
          const unsigned int gt = ld_acquire_sys(&mb->guest_tag);
          unsigned int gseq = gt >> 2;
          if ((gt & 3u) != kStateRunning || gseq == gdone_seq[l]) continue;
          const unsigned int share = T / 2u;
          const unsigned long long w0 = *(volatile unsigned long long*)&mb->guest_next;
          if (claim_seq(w0) != (gseq & kClaimSeqMask) || claim_idx(w0) >= claim_nc(w0)) { gdone_seq[l] = gseq; continue; }
          if (atomicAdd(&mb->guest_nwork, 1u) >= xpart) { gdone_seq[l] = gseq; continue; }
          const unsigned long long w = atomicAdd(&mb->guest_next, 1ull);
          if (claim_idx(w) >= claim_nc(w)) { gdone_seq[l] = gseq; continue; }
          __threadfence_system();                         // the poster's guest_i / slot fields
          if (claim_seq(w) != (gseq & kClaimSeqMask)) gseq = ld_acquire_sys(&mb->guest_tag) >> 2;
          const int gi = *(volatile int*)&mb->guest_i;
          Slot* sa = p.workers[gi].slot;                 // the initiator's slot (peer memory)
          const unsigned int fl = *(volatile unsigned int*)&sa->flags;
          s_ev.xi = p.workers[gi].x;
          s_ev.xj = p.workers[wl].x;
          s_ev.key = *(volatile unsigned long long*)&sa->key;
          s_ev.grad = (!(fl & 1u) && p.model != 0) ? 1 : 0;
          s_ev.ff = (fl & 2u) ? 1 : 0;
          s_ev.kind = kKindEvent;
          s_ev.g = nullptr;
          s_ev.gout = nullptr;
          s_ev.absorb = 0;
          s_ev.pair = 1;
          s_ev.cross = 1;
          s_ev.ctr = &mb->guest_next;
          s_ev.n = share;
          s_ev.stride = 2u;
          s_ev.off = 1u;
          s_ev.first = claim_idx(w);
          s_ev.nc = claim_nc(w);
          s_ev.rem = &sa->rem;
          s_ev.guest = 1;
          s_ev.slot = l;
          s_ev.seq = gseq;
          s_ev.gready = &sa->commit_ready;
          pick = kPickGuest;
        }
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
        // local work done; with cooperative partners stay to serve their
        // events until every event of the run is committed system-wide
        if (n_fin == L && (!p.coop || ld_relaxed_sys64(&p.gctl0->committed) >= p.target)) pick = kExit;
        if (progress) last_progress = now;
        else if (now - last_progress > p.watchdog_ns) { latch_error(p, 7u); pick = kExit; }
      } else if (pick != kExit) {
        last_progress = globaltimer();
        cl.init(s_ev.ctr, s_ev.n, s_ev.stride, s_ev.off, s_ev.first, s_ev.nc);
      }
      s_pick = pick;
    }
    __syncthreads();
    const int pick = s_pick;
    if (pick == kExit) break;
    if (pick >= 0) {                 // a joined event (own slot or, kPickGuest, a peer's half)
      const SmemSlot& e = s_ev;      // stable until the trailing barrier
      unsigned int tiles = 0;
      if (e.kind != kKindEvent) {    // App. A pull / replay stale read: gradient at x_i into gout
        ReadBody body;
        body.gout = reinterpret_cast<float4*>(e.gout);
        body.hi = p.n4;
        body.d = p.d;
        body.gamma = p.gamma;
        body.q = p.q;
        body.kk = quad_event_key_h(p.q.noise_key, e.key);
        body.comp = e.g != nullptr;
        tiles = stg.drive(cl, reinterpret_cast<const float4*>(e.xi), reinterpret_cast<const float4*>(e.g), p.n4,
                          body);
      } else if (e.g) {              // a gradient row: App. A flush (FF) or a replayed stale read (Alg. 1)
        if (e.pair) tiles = e.ff ? event_pass<true, kGradExternal, true>(p, e, stg, cl)
                                 : event_pass<true, kGradExternal>(p, e, stg, cl);
        else tiles = event_pass<false, kGradExternal>(p, e, stg, cl);
      } else if (e.pair) {
        if (e.grad) {
          if (e.ff) tiles = event_pass<true, kGradQuadInline, true>(p, e, stg, cl);
          else if (e.absorb) tiles = event_pass<true, kGradQuadInline, false, true>(p, e, stg, cl);
          else tiles = event_pass<true, kGradQuadInline>(p, e, stg, cl);
        } else {
          tiles = event_pass<true, kGradNone>(p, e, stg, cl);
        }
      } else if (e.grad) {
        tiles = event_pass<false, kGradQuadInline>(p, e, stg, cl);
      } else {                       // a partner-less NO_GRAD event: W = I, nothing to stream
        if (threadIdx.x == 0) while (cl.next() >= 0) ++tiles;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        // this CTA's tiles are visible before its leave; peer stores need the
        // system-scope fence, local ones gpu scope (the committing CTA issues
        // fence.sys before the cross-GPU release, which is cumulative)
        if (e.cross) __threadfence_system();
        else __threadfence();
        if (e.guest) gdone_seq[e.slot] = e.seq;
        else done_seq[e.slot] = e.seq;
        if (tiles && credit(e.rem, tiles)) {
          if (e.guest) st_release_sys(e.gready, e.seq);   // the initiator's scheduler commits
          else commit(p, e.slot);
        }
      }
    } else if (threadIdx.x == 0) {
      __nanosleep(256);
    }
    __syncthreads();
  }
}

}  // namespace

int engine_max_ctas_per_sm(int threads) {
  int n = 0;
  cudaFuncSetAttribute((const void*)k_engine, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, (const void*)k_engine, threads, kTmaSmem);
  return n;
}

cudaError_t launch_engine(const EngineParams& p, int grid, int threads, bool cooperative, cudaStream_t s) {
  EngineParams pp = p;
  void* args[] = {&pp};
  if (threads != kEngineThreads || grid > kMaxGrid) return cudaErrorInvalidValue;
  cudaFuncSetAttribute((const void*)k_engine, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmem);
  if (cooperative) return cudaLaunchCooperativeKernel((const void*)k_engine, dim3(grid), dim3(threads), args,
                                                      kTmaSmem, s);
  return cudaLaunchKernel((const void*)k_engine, dim3(grid), dim3(threads), args, kTmaSmem, s);
}

const void* engine_module_anchor() { return (const void*)k_engine; }

}  // namespace adp
