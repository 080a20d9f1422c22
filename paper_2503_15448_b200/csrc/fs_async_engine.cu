// Host event engine of the buffered asynchronous federation (f2).
//
// Behavioural contract: FederationEngine.run_async, pkg/src/fedsim/server.py
// :485-637 (handle 530-624, flush 516-528, AsyncBuffer 58-69), on the
// discrete-event clock of simnet.py:18-103 -- events delivered in (time,
// insertion counter) order, one log record per handled event. The Python
// mirror is paper_2503_15448_b200/server.py (run_async); this engine runs the
// same state machine over plain arrays and never touches parameters.
//
// Training is deferred exactly as in the Python engine: a cycle records the
// model version it fetched at broadcast_arrive; the first train_done whose
// cycle has no outcome yet suspends the engine (fs_async_run returns
// FS_ASYNC_NEED_EVAL) with every not-yet-evaluated cycle listed; the caller
// trains + scores that batch on the GPU and hands the accept flags back with
// fs_async_provide. Aggregations never suspend: each one is queued as a job
// (new version <- mean of the listed cycles' updates) for the caller to
// launch, in order, before the next training batch. Window reports are
// queued the same way. The processed-event log is kept columnar.
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <map>
#include <queue>
#include <mutex>
#include <vector>

#include "fs_common.cuh"
#include "../../include/fedsim_b200.h"

namespace {

enum Kind : int8_t {
  K_BROADCAST = 0, K_FAIL = 1, K_DONE = 2, K_UPLOAD = 3, K_RECOVER = 4, K_CHECKPOINT = 5,
  K_TIMEOUT = 6, K_AGGREGATE = 7, K_RUN_END = 8
};

struct Ev {
  double t;
  int64_t seq;
  int8_t kind;
  int32_t ci, cycle;
  int64_t a, b;  // kind-specific payload
};
struct EvLater {
  bool operator()(const Ev& x, const Ev& y) const { return x.t > y.t || (x.t == y.t && x.seq > y.seq); }
};

struct Deferred {
  int32_t ci, cycle, version;
  int8_t evaluated, accepted;
  double relevance;  // NaN = None
};

}  // namespace

struct fs_async_engine {
  // ---- world (copied)
  int32_t N, C, rounds, k_min;
  int64_t budget;
  double timeout_s, agg_cost, horizon, recovery_s;
  bool plan_per_cycle;
  std::vector<int32_t> cid, steps;
  std::vector<double> down, up;
  std::vector<uint8_t> trains, failed, recovered;
  std::vector<double> fail_off, span;
  std::vector<int32_t> n_captures, cap_ptr;
  std::vector<double> cap_off;
  // ---- state
  std::priority_queue<Ev, std::vector<Ev>, EvLater> heap;
  int64_t seq = 0;
  double now = 0.0;
  bool stopped = false, started = false, finished = false, in_hand = false;
  Ev hand{};
  int32_t agg_count = 0, aggs_reported = 0;
  int64_t applied = 0;
  double server_free = 0.0, transfer = 0.0;
  int64_t buf_epoch = 0;
  std::vector<std::pair<int32_t, int32_t>> pending;               // (deferred id, fetched)
  std::vector<std::vector<std::pair<int32_t, int32_t>>> batches;  // aggregate event payloads
  std::vector<int32_t> cycles;                                    // cycles started per client
  std::vector<int32_t> active;                                    // deferred id per client (-1)
  std::vector<Deferred> deferred;
  std::vector<int32_t> unevaluated;
  std::vector<int32_t> window_stale;
  int64_t w_acc = 0, w_rej = 0, w_fail = 0, w_steps = 0, trainings = 0;
  int32_t phase = 0;  // 0 = first run with horizon, 1 = after the horizon/cycle-cap run_end
  // ---- outputs since the last yield
  std::vector<int32_t> ev_id, ev_ci, ev_cycle, ev_version;
  std::vector<int32_t> job_version, job_member, job_stale;
  std::vector<int64_t> job_off{0};
  std::vector<int64_t> rep_i;
  std::vector<double> rep_d;
  std::vector<int64_t> rep_off{0};
  std::vector<int32_t> rep_stale;
  // ---- columnar log
  std::vector<int8_t> lk;
  std::vector<double> lt, lx;
  std::vector<int32_t> lci, lcy;
  std::vector<int64_t> la, lb, ll;
  std::vector<int32_t> list_cid, list_stale;

  size_t plan_ix(int32_t ci, int32_t cycle) const { return plan_per_cycle ? (size_t)ci * C + cycle : (size_t)ci; }

  void schedule(double t, int8_t kind, int32_t ci, int32_t cycle, int64_t a = 0, int64_t b = 0) {
    heap.push(Ev{t, seq++, kind, ci, cycle, a, b});
  }
  void log(const Ev& e, int64_t a, int64_t b, double x, int64_t l = -1) {
    lk.push_back(e.kind); lt.push_back(e.t); lci.push_back(e.ci); lcy.push_back(e.cycle);
    la.push_back(a); lb.push_back(b); lx.push_back(x); ll.push_back(l);
  }

  void start_cycle(int32_t ci, double t_request) {  // server.py start_cycle
    const int32_t cyc = cycles[ci];
    if (cyc >= C) return;
    cycles[ci] += 1;
    const double depart = std::max(t_request, server_free);
    schedule(depart + down[ci], K_BROADCAST, ci, cyc);
    transfer += down[ci];
  }

  void flush(double t_now, int trigger) {
    batches.push_back(pending);
    const int64_t count = (int64_t)pending.size();
    pending.clear();
    buf_epoch += 1;
    const double start = std::max(t_now, server_free);
    const double cost = agg_cost * (double)count;
    const double done = start + cost;
    server_free = done;
    // a = batch slot, b = (trigger << 32) | window; round = agg_count at flush
    const int64_t window = applied / N;
    Ev e{done, seq++, K_AGGREGATE, trigger, agg_count, (int64_t)batches.size() - 1, window};
    heap.push(e);
  }

  void report(int64_t window, double t_s) {
    const int64_t ri[9] = {window, agg_count, N, agg_count - aggs_reported, w_acc, w_rej, w_fail, w_steps, 0};
    rep_i.insert(rep_i.end(), ri, ri + 9);
    rep_d.push_back(t_s);
    rep_d.push_back(transfer);
    rep_stale.insert(rep_stale.end(), window_stale.begin(), window_stale.end());
    rep_off.push_back((int64_t)rep_stale.size());
    w_acc = w_rej = w_fail = w_steps = 0;
  }

  // returns false when the event must wait for an evaluation
  bool handle(const Ev& e) {
    switch (e.kind) {
      case K_BROADCAST: {
        const int32_t ci = e.ci, cyc = e.cycle;
        const size_t p = plan_ix(ci, cyc);
        for (int32_t q = 0; q < n_captures[p]; ++q)
          schedule(e.t + cap_off[cap_ptr[ci] + q], K_CHECKPOINT, ci, cyc);
        if (failed[p]) {
          schedule(e.t + fail_off[p], K_FAIL, ci, cyc, recovered[p]);
          if (recovered[p]) schedule(e.t + fail_off[p] + recovery_s, K_RECOVER, ci, cyc);
        }
        if (!trains[p]) {
          w_fail += 1;
          start_cycle(ci, e.t + span[p]);
        } else {
          const int32_t id = (int32_t)deferred.size();
          deferred.push_back(Deferred{ci, cyc, agg_count, 0, 0, NAN});
          unevaluated.push_back(id);
          schedule(e.t + span[p], K_DONE, ci, cyc, id);
          if (failed[p]) w_fail += 1;
          active[ci] = id;
        }
        log(e, 0, 0, 0.0);
        return true;
      }
      case K_DONE: {
        const int32_t id = (int32_t)e.a;
        Deferred& d = deferred[id];
        if (!d.evaluated) return false;
        trainings += 1;
        w_steps += steps[e.ci];
        if (d.accepted) {
          w_acc += 1;
          schedule(e.t + up[e.ci], K_UPLOAD, e.ci, e.cycle, id, d.version);
          transfer += up[e.ci];
        } else {
          w_rej += 1;
          start_cycle(e.ci, e.t);
        }
        log(e, d.accepted, 0, d.relevance);
        return true;
      }
      case K_UPLOAD: {
        pending.emplace_back((int32_t)e.a, (int32_t)e.b);
        if (pending.size() == 1) schedule(e.t + timeout_s, K_TIMEOUT, -1, -1, buf_epoch, 1);
        if ((int64_t)pending.size() >= k_min) flush(e.t, 0);
        start_cycle(e.ci, e.t);
        log(e, agg_count - e.b, 0, 0.0);
        return true;
      }
      case K_TIMEOUT: {
        if (e.a != buf_epoch) return true;  // stale timer: no record
        if (!pending.empty()) flush(e.t, 1);
        log(e, e.a, e.b, 0.0);
        return true;
      }
      case K_AGGREGATE: {
        const auto& batch = batches[e.a];
        const int64_t l0 = (int64_t)list_cid.size();
        for (const auto& m : batch) {
          list_cid.push_back(cid[deferred[m.first].ci]);
          list_stale.push_back(agg_count - m.second);
          window_stale.push_back(agg_count - m.second);
        }
        // job: version agg_count+1 = mean of the batch's updates (server.py:590-594)
        for (const auto& m : batch) {
          job_member.push_back(m.first);
          job_stale.push_back(agg_count - m.second);
        }
        job_version.push_back(agg_count + 1);
        job_off.push_back((int64_t)job_member.size());
        agg_count += 1;
        const int64_t before = applied;
        applied += (int64_t)batch.size();
        // record: a = round, b = window, x = cost, ci = trigger, cycle = count, l = list offset
        Ev rec = e;
        rec.cycle = (int32_t)batch.size();
        log(rec, e.cycle, e.b, agg_cost * (double)batch.size(), l0);
        const int64_t w_hi = std::min<int64_t>(applied / N, rounds);
        for (int64_t w = before / N; w < w_hi; ++w) {
          report(w, e.t);
          aggs_reported = agg_count;
          window_stale.clear();
        }
        if (applied >= budget) schedule(e.t, K_RUN_END, -1, -1, 0);
        return true;
      }
      case K_RUN_END:
        stopped = true;
        log(e, e.a, 0, 0.0);
        return true;
      default:  // client_fail, client_recover, checkpoint
        log(e, e.a, 0, 0.0);
        return true;
    }
  }

  void clear_outputs() {
    ev_id.clear(); ev_ci.clear(); ev_cycle.clear(); ev_version.clear();
    job_version.clear(); job_member.clear(); job_stale.clear(); job_off.assign(1, 0);
    rep_i.clear(); rep_d.clear(); rep_off.assign(1, 0); rep_stale.clear();
  }

  // Timeline.run(handler, horizon): deliver until empty / stopped / beyond the
  // horizon. Returns 1 when an event waits for an evaluation, 2 (device mode)
  // when window reports are ready.
  int drain(double limit) {
    if (in_hand) {
      if (!handle(hand)) return 1;
      in_hand = false;
      if (dx && !rep_d.empty()) return 2;
    }
    while (!heap.empty() && !stopped && heap.top().t <= limit) {
      Ev e = heap.top();
      heap.pop();
      now = e.t;
      if (!handle(e)) {
        hand = e;
        in_hand = true;
        return 1;
      }
      if (dx && !rep_d.empty()) return 2;
    }
    return 0;
  }

  int step() {
    if (!started) {
      started = true;
      for (int32_t ci = 0; ci < N; ++ci) start_cycle(ci, 0.0);
    }
    if (phase == 0) {
      const double limit = horizon >= 0.0 ? horizon : INFINITY;
      if (int r = drain(limit)) return r;
      if (horizon >= 0.0 && !stopped && now < horizon) now = horizon;
      if (!stopped) {
        const int64_t reason = (horizon >= 0.0 && now >= horizon) ? 1 : 2;
        schedule(now, K_RUN_END, -1, -1, reason);
      }
      phase = 1;
    }
    if (!stopped) {
      if (int r = drain(INFINITY)) return r;
    }
    finished = true;
    return 0;
  }

  struct DeviceExec* dx = nullptr;
  int run();

  int yield_eval() {
    for (int32_t id : unevaluated) {
      ev_id.push_back(id);
      ev_ci.push_back(deferred[id].ci);
      ev_cycle.push_back(deferred[id].cycle);
      ev_version.push_back(deferred[id].version);
    }
    return FS_ASYNC_NEED_EVAL;
  }

  void provide(int32_t n, const uint8_t* accepted, const double* relevance) {
    for (int32_t i = 0; i < n; ++i) {
      Deferred& d = deferred[unevaluated[i]];
      d.evaluated = 1;
      d.accepted = accepted[i] ? 1 : 0;
      d.relevance = relevance[i];
    }
    unevaluated.clear();
  }
};

// ------------------------------------------------------------------ device mode
// The engine's own executor: the per-flush work of server.DeviceAsyncExecutor
// (TrainPlan + run_trainer + align + one host read) without a Python round trip.
namespace {

struct DevBlock {
  void* ptr;
  int64_t refs;
};

}  // namespace

// Page-locked host buffers outlive an engine: cudaFreeHost unpins pages and
// took up to 0.9 s at engine teardown, so freed buffers go back to a
// process-wide cache (one per allocation flag set) and later engines reuse them.
struct PinnedCache {
  std::mutex mu;
  std::vector<std::pair<void*, size_t>> free_default, free_mapped;
};
static PinnedCache& pinned_cache() {
  static PinnedCache c;
  return c;
}
static int pinned_get(size_t bytes, unsigned flags, void** out, size_t* got) {
  PinnedCache& c = pinned_cache();
  {
    std::lock_guard<std::mutex> lk(c.mu);
    auto& v = flags & cudaHostAllocMapped ? c.free_mapped : c.free_default;
    size_t best = v.size();
    for (size_t i = 0; i < v.size(); ++i)
      if (v[i].second >= bytes && (best == v.size() || v[i].second < v[best].second)) best = i;
    if (best < v.size()) {
      *out = v[best].first;
      *got = v[best].second;
      v.erase(v.begin() + best);
      return FS_OK;
    }
  }
  if (cudaHostAlloc(out, bytes, flags) != cudaSuccess) return FS_ECUDA;
  *got = bytes;
  return FS_OK;
}
static void pinned_put(void* p, size_t bytes, unsigned flags) {
  if (!p) return;
  PinnedCache& c = pinned_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  (flags & cudaHostAllocMapped ? c.free_mapped : c.free_default).push_back({p, bytes});
}

struct DeviceExec {
  fs_async_device d;
  cudaStream_t st;
  int64_t M = 0, ldw = 0, esz = 8;
  int32_t sum_hidden = 0;
  std::vector<int64_t> row_off;
  std::vector<int32_t> n_rows, batch;
  // pinned staging + device mirror (one copy per flush)
  uint8_t* h_stage = nullptr;
  size_t h_stage_bytes = 0;
  uint8_t* d_stage = nullptr;
  size_t stage_cap = 0, stage_off = 0, stage_done = 0;  // [stage_done, stage_off) not yet copied
  // pooled device buffers
  void* d_perm = nullptr; size_t perm_cap = 0;
  void* d_bits = nullptr; size_t bits_cap = 0;
  void* d_ws = nullptr; size_t ws_cap = 0;
  void* d_sorted = nullptr; size_t sorted_cap = 0;
  int64_t* d_res = nullptr; size_t res_cap = 0;
  int64_t* h_res = nullptr;
  // model versions and trained rows (stream-ordered allocations)
  std::vector<DevBlock> blocks;                 // block id -> allocation + live references
  std::vector<std::pair<uint64_t, int64_t>> version;  // version -> (ptr, block id; -1 = caller-owned)
  std::vector<uint64_t> row_ptr;                // deferred id -> trained row (accepted only)
  std::vector<int64_t> row_block;
  std::vector<uint64_t> rep_w;
  int64_t flushes = 0, launches = 0;
  int32_t div_client = -1, div_cycle = -1;
  double t_prep = 0, t_wait = 0, t_post = 0;  // host seconds: before the sync, in it, after it
  // K2/K3 lookahead: every client owns two plan slots (shuffles + keep bits);
  // after a flush trains cycle c of a client from slot p, its cycle c+1 is
  // generated into slot 1-p on a side stream while the trainer runs, so the
  // next flush's trainer starts without waiting for K2/K3.
  cudaStream_t side = nullptr;
  cudaEvent_t side_copy = nullptr, side_done = nullptr;
  bool side_used = false;
  int32_t E = 0, C = 0;
  std::vector<int64_t> perm_pre, mask_pre;   // per-client slot offsets
  int64_t perm_sum = 0, mask_sum = 0;
  int32_t* d_perm_all = nullptr;
  uint32_t* d_bits_all = nullptr;
  std::vector<int32_t> gen_cycle;            // [client][slot] cycle held (-1 none)
  std::vector<int32_t> cid_of;
  int64_t misses = 0;
  // ---- per-client completion mode (bf16 unit-major trainer): every flush
  // launches its new cycles as one trainer kernel on a stream of its own; a
  // client's CTA publishes {aligned, status} to a mapped host record the
  // moment its row is written, and the event loop waits only for the cycle it
  // needs, not for the launch's longest client.
  bool percycle = false;
  static constexpr int kRecChunk = 1 << 16;
  std::vector<fs_client_done*> rec_host;      // chunks of mapped records, by deferred id
  std::vector<uint64_t> rec_dev;
  std::vector<uint8_t> launched;
  std::vector<int32_t> vref;                  // launched-not-collected cycles reading a version
  struct Batch {
    cudaStream_t s;
    std::vector<int32_t> ids;
    int32_t left;
  };
  std::vector<Batch> inflight;
  std::vector<cudaStream_t> stream_pool;
  size_t next_stream = 0;
  std::vector<std::pair<void*, cudaEvent_t>> deferred_free;  // freed once the event completes
  int32_t low_version = 0;                    // versions below are released
  // ---- client sharding (fs_async_device.world_size > 1): this rank trains
  // the cycles of the clients it owns; outcomes and aggregation partials are
  // summed over the ranks through d.exchange (ShardedAsyncExecutor's scheme)
  bool sharded = false;
  std::vector<int32_t> owner;
  std::vector<uint8_t> row_owned;             // deferred id -> this rank holds its accepted row
  double* d_x = nullptr;                      // exchange buffer
  size_t x_cap = 0;
  double t_poll = 0, t_jobs = 0, t_batch = 0, t_look = 0, t_alloc = 0, t_copy = 0, t_launch = 0;
  int64_t perm_at(int32_t ci, int32_t p) const { return p * perm_sum + perm_pre[ci]; }
  int64_t mask_at(int32_t ci, int32_t p) const { return p * mask_sum + mask_pre[ci]; }
  static double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
  }

  ~DeviceExec() {
    for (cudaStream_t ps : stream_pool) {
      cudaStreamSynchronize(ps);
      cudaStreamDestroy(ps);
    }
    for (auto& f : deferred_free) {
      cudaEventSynchronize(f.second);
      cudaFree(f.first);
      cudaEventDestroy(f.second);
    }
    for (auto* h : rec_host) pinned_put(h, sizeof(fs_client_done) * kRecChunk, cudaHostAllocMapped);
    if (main_ev) cudaEventDestroy(main_ev);
    cudaStreamSynchronize(st);
    for (auto& b : arena_pending) {  // every release is complete after the syncs above
      cudaEventDestroy(b.ready);
      arena_free.push_back(ArenaBlock{b.p, b.cls, nullptr});
    }
    for (auto& bm : batch_mem) {  // blocks of launches whose rows were never all dropped
      cudaEventDestroy(bm.end);
      arena_free.push_back(ArenaBlock{bm.mem, arena_cls[bm.mem], nullptr});
    }
    for (auto ev : event_pool) cudaEventDestroy(ev);
    for (auto& b : blocks)
      if (b.ptr) cudaFreeAsync(b.ptr, st);
    if (d_perm) cudaFreeAsync(d_perm, st);
    if (d_bits) cudaFreeAsync(d_bits, st);
    if (d_ws) cudaFreeAsync(d_ws, st);
    if (d_sorted) cudaFreeAsync(d_sorted, st);
    if (d_res) cudaFreeAsync(d_res, st);
    if (d_x) cudaFreeAsync(d_x, st);
    if (d_stage) cudaFreeAsync(d_stage, st);
    if (side) {
      cudaStreamSynchronize(side);
      cudaStreamDestroy(side);
    }
    if (side_copy) cudaEventDestroy(side_copy);
    if (side_done) cudaEventDestroy(side_done);
    if (d_perm_all) cudaFreeAsync(d_perm_all, st);
    if (d_bits_all) cudaFreeAsync(d_bits_all, st);
    cudaStreamSynchronize(st);
    pinned_put(h_stage, h_stage_bytes, cudaHostAllocDefault);
    pinned_put(h_res, 1 << 20, cudaHostAllocDefault);
  }

  static int cuda(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return FS_OK;
    fs::set_error("async device: %s: %s", what, cudaGetErrorString(e));
    return FS_ECUDA;
  }
  int grow(void** p, size_t* cap, size_t need, const char* what) {
    if (need <= *cap) return FS_OK;
    if (*p) cudaFreeAsync(*p, st);
    size_t n = need + need / 4 + 256;
    *p = nullptr;
    *cap = 0;
    if (int rc = cuda(cudaMallocAsync(p, n, st), what)) return rc;
    *cap = n;
    return FS_OK;
  }
  int alloc_block(size_t bytes, int64_t refs, int64_t* id, void** out) {
    void* p = nullptr;
    if (int rc = cuda(cudaMallocAsync(&p, bytes, st), "row block")) return rc;
    blocks.push_back(DevBlock{p, refs});
    *id = (int64_t)blocks.size() - 1;
    *out = p;
    return FS_OK;
  }
  void unref(int64_t b) {
    if (b < 0) return;
    if (--blocks[b].refs == 0) {
      cudaFreeAsync(blocks[b].ptr, st);
      blocks[b].ptr = nullptr;
    }
  }
  // staging: pack on the host, one H2D per commit
  uint64_t put(const void* src, size_t bytes) {
    stage_off = (stage_off + 15) & ~(size_t)15;
    const uint64_t dptr = (uint64_t)(d_stage + stage_off);
    memcpy(h_stage + stage_off, src, bytes);
    stage_off += bytes;
    return dptr;
  }
  // room for `more` bytes; growing waits for the stream (earlier regions were
  // copied by then) and restarts the arena
  int stage_reserve(size_t more) {
    if (((stage_off + 15) & ~(size_t)15) + more <= stage_cap) return FS_OK;
    if (int rc = cuda(cudaStreamSynchronize(st), "staging grow")) return rc;
    if (side)
      if (int rc = cuda(cudaStreamSynchronize(side), "staging grow")) return rc;
    pinned_put(h_stage, h_stage_bytes, cudaHostAllocDefault);
    if (d_stage) cudaFreeAsync(d_stage, st);
    h_stage = nullptr;
    d_stage = nullptr;
    stage_cap = stage_off = stage_done = 0;
    const size_t n = 2 * more + 4096;
    if (pinned_get(n, cudaHostAllocDefault, (void**)&h_stage, &h_stage_bytes) != FS_OK) {
      fs::set_error("fs_async: pinned staging allocation failed");
      return FS_ECUDA;
    }
    if (int rc = cuda(cudaMallocAsync((void**)&d_stage, n, st), "device staging")) return rc;
    stage_cap = n;
    return FS_OK;
  }
  int commit(cudaStream_t s = nullptr) {
    if (stage_off == stage_done) return FS_OK;
    // the side stream's kernels may still read staged arguments of an earlier
    // lookahead: main-stream copies into the arena wait for them
    if ((!s || s == st) && side_used)
      if (int rc = cuda(cudaStreamWaitEvent(st, side_done, 0), "event")) return rc;
    const size_t lo = stage_done;
    stage_done = stage_off;
    return cuda(cudaMemcpyAsync(d_stage + lo, h_stage + lo, stage_off - lo, cudaMemcpyHostToDevice, s ? s : st),
                "stage copy");
  }
  // after a host synchronisation every staged copy has run: reuse the arena
  void stage_reset() {
    if (side_used) cudaEventSynchronize(side_copy);  // the side stream's staged copy ran too
    stage_off = stage_done = 0;
  }

  int init(const fs_async_device* dev, const fs_async_engine* e) {
    const int32_t n_clients = e->N;
    d = *dev;
    st = (cudaStream_t)dev->stream;
    M = 0;
    for (int l = 0; l + 1 < d.n_dims; ++l) M += (int64_t)(d.dims[l] + 1) * d.dims[l + 1];
    for (int l = 1; l + 1 < d.n_dims; ++l) sum_hidden += d.dims[l];
    esz = d.bf16 ? 4 : 8;
    ldw = (M * esz + 127) / 128 * 128 / esz;
    row_off.assign(dev->row_off_host, dev->row_off_host + n_clients);
    n_rows.assign(dev->n_rows_host, dev->n_rows_host + n_clients);
    batch.assign(dev->batch_host, dev->batch_host + n_clients);
    version.push_back({(uint64_t)dev->w0, -1});
    cudaMemPool_t pool;
    int device = 0;
    cudaGetDevice(&device);
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;  // keep freed blocks cached across synchronisations
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    size_t h_res_got = 0;
    if (pinned_get(1 << 20, cudaHostAllocDefault, (void**)&h_res, &h_res_got) != FS_OK) {
      fs::set_error("fs_async: pinned results allocation failed");
      return FS_ECUDA;
    }
    if (int rc = stage_reserve(1 << 19)) return rc;
    // lookahead plan slots
    E = d.epochs;
    C = e->C;
    cid_of = e->cid;
    perm_pre.resize(n_clients);
    mask_pre.resize(n_clients);
    for (int32_t i = 0; i < n_clients; ++i) {
      const int64_t nr = n_rows[i], b = batch[i];
      const int64_t spe = (nr + b - 1) / b;
      perm_pre[i] = perm_sum;
      mask_pre[i] = mask_sum;
      perm_sum += (int64_t)E * nr;
      if (d.dropout_rate > 0.0) mask_sum += (int64_t)E * spe * ((b * sum_hidden + 31) / 32);
    }
    gen_cycle.assign(2 * (size_t)n_clients, -1);
    if (int rc = cuda(cudaMallocAsync((void**)&d_perm_all, 8 * (size_t)std::max<int64_t>(perm_sum, 1), st), "perm slots"))
      return rc;
    if (mask_sum > 0)
      if (int rc = cuda(cudaMallocAsync((void**)&d_bits_all, 8 * (size_t)mask_sum, st), "mask slots")) return rc;
    if (int rc = cuda(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking), "side stream")) return rc;
    if (int rc = cuda(cudaEventCreateWithFlags(&side_copy, cudaEventDisableTiming), "event")) return rc;
    if (int rc = cuda(cudaEventCreateWithFlags(&side_done, cudaEventDisableTiming), "event")) return rc;
    // the side stream may only touch the slots once they are allocated
    if (int rc = cuda(cudaEventRecord(side_done, st), "event")) return rc;
    if (int rc = cuda(cudaStreamWaitEvent(side, side_done, 0), "event")) return rc;
    sharded = d.world_size > 1;
    if (sharded) {
      if (!d.owner_host || !d.exchange || d.rank < 0 || d.rank >= d.world_size || d.staleness_alpha >= 0.0) {
        fs::set_error("async device: sharding needs owner_host, exchange and 0 <= rank < world_size "
                      "(staleness weighting runs unsharded)");
        return FS_EINVAL;
      }
      owner.assign(d.owner_host, d.owner_host + n_clients);
    }
    percycle = !sharded && d.bf16 && d.n_dims == 5 && (d.dims[1] == 128 || d.dims[1] == 256) &&
               d.dims[2] == 128 && d.dims[3] == 64 && d.dims[0] <= 64;
    if (percycle) {
      stream_pool.resize(8);
      for (auto& ps : stream_pool)
        if (int rc = cuda(cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking), "pool stream")) return rc;
    }
    // cycle 0 of every client, in bulk, while the caller still prepares
    std::vector<int32_t> all, zero, slot;
    for (int32_t i = 0; i < n_clients; ++i)
      if (mine(i)) {
        all.push_back(i);
        zero.push_back(0);
        slot.push_back(0);
      }
    if (C > 0 && !all.empty())
      if (int rc = generate(all.data(), zero.data(), slot.data(), (int32_t)all.size(), side)) return rc;
    return FS_OK;
  }

  bool mine(int32_t ci) const { return !sharded || owner[ci] == d.rank; }
  // sum n doubles at d_x over the ranks (the callback runs the collective)
  int exchange(int64_t n) {
    if (int rc = cuda(cudaStreamSynchronize(st), "exchange")) return rc;
    if (d.exchange(d.exchange_ctx, d_x, n, st) != 0) {
      fs::set_error("async device: exchange callback failed");
      return FS_EINVAL;
    }
    return FS_OK;
  }

  // K2 shuffles + K3 keep bits of (client ci[j], cycle cyc[j]) into slot par[j],
  // on stream s (the main stream for misses, the side stream for lookahead)
  int generate(const int32_t* ci, const int32_t* cyc, const int32_t* par, int32_t n, cudaStream_t s) {
    if (n == 0 || E == 0) return FS_OK;
    std::vector<uint64_t> seeds(n);
    std::vector<int32_t> cid(n), i32(2 * (size_t)n);
    std::vector<int64_t> i64(2 * (size_t)n);
    int64_t max_rows = 1;
    for (int32_t j = 0; j < n; ++j) cid[j] = cid_of[ci[j]];
    fs_train_seeds_host(d.master_seed, cid.data(), cyc, n, seeds.data());
    for (int32_t j = 0; j < n; ++j) {
      i32[j] = n_rows[ci[j]];
      i32[n + j] = batch[ci[j]];
      i64[j] = perm_at(ci[j], par[j]);
      i64[n + j] = mask_at(ci[j], par[j]);
      max_rows = std::max<int64_t>(max_rows, n_rows[ci[j]]);
      gen_cycle[2 * (size_t)ci[j] + par[j]] = cyc[j];
    }
    uint64_t p_seed, p64, p32;
    void* tmp = nullptr;
    if (percycle) {  // no per-flush host sync in this mode: a stream-ordered temporary
      const size_t b_seed = 8 * (size_t)n, b64 = 8 * i64.size(), b32 = 4 * i32.size();
      std::vector<uint8_t> h(b_seed + b64 + b32);
      memcpy(h.data(), seeds.data(), b_seed);
      memcpy(h.data() + b_seed, i64.data(), b64);
      memcpy(h.data() + b_seed + b64, i32.data(), b32);
      if (int rc = cuda(cudaMallocAsync(&tmp, h.size(), s), "plan args")) return rc;
      if (int rc = cuda(cudaMemcpyAsync(tmp, h.data(), h.size(), cudaMemcpyHostToDevice, s), "plan args")) return rc;
      p_seed = (uint64_t)tmp;
      p64 = p_seed + b_seed;
      p32 = p64 + b64;
      if (s == side) side_used = true;
    } else {
      if (int rc = stage_reserve(16 * (size_t)n + 64 + 8 * (size_t)n * 3)) return rc;
      p_seed = put(seeds.data(), 8 * (size_t)n);
      p64 = put(i64.data(), 8 * i64.size());
      p32 = put(i32.data(), 4 * i32.size());
      if (int rc = commit(s)) return rc;
      if (s == side) {
        side_used = true;
        if (int rc = cuda(cudaEventRecord(side_copy, side), "event")) return rc;
      }
    }
    launches += 1;
    if (int rc = fs_shuffle_perms((const uint64_t*)p_seed, (const int32_t*)p32, (const int64_t*)p64, n, E,
                                  (int32_t)max_rows, d_perm_all, s))
      return rc;
    if (d.dropout_rate > 0.0) {
      launches += 1;
      if (int rc = fs_dropout_bits((const uint64_t*)p_seed, (const int32_t*)p32, (const int32_t*)(p32 + 4 * n),
                                   (const int64_t*)(p64 + 8 * n), n, E, sum_hidden, 1.0 - d.dropout_rate,
                                   d_bits_all, s))
        return rc;
    }
    if (tmp) cudaFreeAsync(tmp, s);
    if (s == side) return cuda(cudaEventRecord(side_done, side), "event");
    return FS_OK;
  }

  uint64_t prev_of(int32_t v) const {
    return v > 0 ? version[v - 1].first : (uint64_t)d.w0_prev;
  }

  // aggregation jobs queued by the event loop, one launch pair
  // sharded aggregation jobs: this rank's members of every job summed in
  // canonical order into float64 partials, one exchange, means on every rank
  // (model versions stay replicated; the sum re-associates across ranks, so
  // they are tolerance-matched to one GPU like the sync path)
  int launch_jobs_sharded(fs_async_engine* e) {
    const int32_t nj = (int32_t)e->job_version.size();
    int64_t blk;
    void* base;
    if (int rc = alloc_block((size_t)nj * ldw * esz, nj, &blk, &base)) return rc;
    std::vector<uint64_t> outs(nj);
    for (int32_t j = 0; j < nj; ++j) {
      outs[j] = (uint64_t)base + (uint64_t)j * ldw * esz;
      if ((int32_t)version.size() != e->job_version[j]) {
        fs::set_error("async device: versions out of order");
        return FS_EINVAL;
      }
      version.push_back({outs[j], blk});
    }
    if (int rc = grow((void**)&d_x, &x_cap, 8 * (size_t)nj * M, "exchange buffer")) return rc;
    if (int rc = cuda(cudaMemsetAsync(d_x, 0, 8 * (size_t)nj * M, st), "partials")) return rc;
    std::vector<std::vector<uint64_t>> own(nj);
    size_t staged = 0, max_own = 1;
    for (int32_t j = 0; j < nj; ++j) {
      for (int64_t i = e->job_off[j]; i < e->job_off[j + 1]; ++i) {
        const int32_t m = e->job_member[i];
        if (m < (int32_t)row_owned.size() && row_owned[m]) own[j].push_back(row_ptr[m]);
      }
      staged += 16 * own[j].size() + 16;
      max_own = std::max(max_own, own[j].size());
    }
    if (int rc = stage_reserve(staged + 64)) return rc;
    std::vector<uint64_t> p_rows(nj, 0);
    for (int32_t j = 0; j < nj; ++j)
      if (!own[j].empty()) p_rows[j] = put(own[j].data(), 8 * own[j].size());
    if (int rc = commit()) return rc;
    if (int rc = grow(&d_sorted, &sorted_cap, 8 * max_own, "sorted rows")) return rc;
    for (int32_t j = 0; j < nj; ++j) {
      const int32_t k = (int32_t)own[j].size();
      if (k == 0) continue;
      const uint64_t* rows = (const uint64_t*)p_rows[j];
      if (k > 1) {
        launches += 1;
        if (int rc = fs_canonical_order(rows, k, M, (int32_t)esz, (uint64_t*)d_sorted, st)) return rc;
        rows = (const uint64_t*)d_sorted;
      }
      launches += 1;
      if (int rc = fs_sum_rows(rows, k, M, (int32_t)esz, d_x + (size_t)j * M, st)) return rc;
    }
    if (int rc = exchange((int64_t)nj * M)) return rc;
    for (int32_t j = 0; j < nj; ++j) {
      launches += 1;
      if (int rc = fs_mean_finish(d_x + (size_t)j * M, e->job_off[j + 1] - e->job_off[j], M, (int32_t)esz,
                                  (void*)outs[j], st))
        return rc;
    }
    for (int64_t i = 0; i < e->job_off[nj]; ++i) {
      const int32_t m = e->job_member[i];
      if (m < (int32_t)row_owned.size() && row_owned[m]) {
        row_owned[m] = 0;
        unref(row_block[m]);
      }
    }
    e->job_version.clear();
    e->job_member.clear();
    e->job_stale.clear();
    e->job_off.assign(1, 0);
    return FS_OK;
  }

  int launch_jobs(fs_async_engine* e) {
    const int32_t nj = (int32_t)e->job_version.size();
    if (nj == 0) return FS_OK;
    if (sharded) return launch_jobs_sharded(e);
    struct Acc {
      double& t;
      double t0;
      ~Acc() { t += now_s() - t0; }
    } acc_{t_jobs, now_s()};
    const int64_t nrows = e->job_off[nj];
    int32_t max_k = 1;
    for (int32_t j = 0; j < nj; ++j) max_k = std::max<int32_t>(max_k, (int32_t)(e->job_off[j + 1] - e->job_off[j]));
    int64_t blk;
    void* base;
    if (int rc = alloc_block((size_t)nj * ldw * esz, nj, &blk, &base)) return rc;
    std::vector<uint64_t> rows(nrows), outs(nj);
    for (int64_t i = 0; i < nrows; ++i) rows[i] = row_ptr[e->job_member[i]];
    for (int32_t j = 0; j < nj; ++j) {
      outs[j] = (uint64_t)base + (uint64_t)j * ldw * esz;
      if ((int32_t)version.size() != e->job_version[j]) {
        fs::set_error("async device: versions out of order");
        return FS_EINVAL;
      }
      version.push_back({outs[j], blk});
    }
    // opt-in staleness weights (1 + s) ** -alpha, s = versions since the member fetched its model
    const bool weighted = d.staleness_alpha >= 0.0;
    std::vector<double> wts(weighted ? nrows : 0);
    for (int64_t i = 0; i < (int64_t)wts.size(); ++i) wts[i] = std::pow(1.0 + (double)e->job_stale[i], -d.staleness_alpha);
    const int64_t nw = weighted ? nrows : 0;
    uint64_t p_rows, p_off, p_out, p_w = 0;
    void* tmp = nullptr;
    if (percycle) {  // no per-flush host sync in this mode: a stream-ordered temporary
      std::vector<uint64_t> h(nrows + nj + 1 + nj + nw);
      memcpy(h.data(), rows.data(), 8 * nrows);
      memcpy(h.data() + nrows, e->job_off.data(), 8 * (nj + 1));
      memcpy(h.data() + nrows + nj + 1, outs.data(), 8 * nj);
      if (nw) memcpy(h.data() + nrows + 2 * nj + 1, wts.data(), 8 * nw);
      if (int rc = cuda(cudaMallocAsync(&tmp, 8 * h.size(), st), "jobs args")) return rc;
      if (int rc = cuda(cudaMemcpyAsync(tmp, h.data(), 8 * h.size(), cudaMemcpyHostToDevice, st), "jobs args"))
        return rc;
      p_rows = (uint64_t)tmp;
      p_off = p_rows + 8 * nrows;
      p_out = p_off + 8 * (nj + 1);
      p_w = p_out + 8 * nj;
    } else {
      if (int rc = stage_reserve(16 * (size_t)(2 * nrows + 2 * nj + 8 + nw))) return rc;
      p_rows = put(rows.data(), 8 * nrows);
      p_off = put(e->job_off.data(), 8 * (nj + 1));
      p_out = put(outs.data(), 8 * nj);
      if (nw) p_w = put(wts.data(), 8 * nw);
      if (int rc = commit()) return rc;
    }
    if (int rc = grow(&d_sorted, &sorted_cap, (weighted ? 16 : 8) * nrows, "sorted rows")) return rc;
    launches += 1;
    if (weighted) {
      if (int rc = fs_aggregate_jobs_weighted((const uint64_t*)p_rows, (const double*)p_w, (const int64_t*)p_off, nj,
                                              max_k, M, (int32_t)esz, (uint64_t*)d_sorted,
                                              (double*)d_sorted + nrows, (const uint64_t*)p_out, st))
        return rc;
    } else if (int rc = fs_aggregate_jobs((const uint64_t*)p_rows, (const int64_t*)p_off, nj, max_k, M, (int32_t)esz,
                                          (uint64_t*)d_sorted, (const uint64_t*)p_out, st)) {
      return rc;
    }
    if (tmp) cudaFreeAsync(tmp, st);
    for (int64_t i = 0; i < nrows; ++i) {
      if (percycle) drop_row(e->job_member[i]);
      else unref(row_block[e->job_member[i]]);
    }
    e->job_version.clear();
    e->job_member.clear();
    e->job_stale.clear();
    e->job_off.assign(1, 0);
    return FS_OK;
  }

  // one deferred flush: train + score every pending cycle, hand outcomes back
  // (sharded: this rank's cycles, then one exchange of every outcome)
  int flush(fs_async_engine* e) {
    const double t0 = now_s();
    if (int rc = launch_jobs(e)) return rc;
    const std::vector<int32_t>& pending = e->unevaluated;
    const int32_t K = (int32_t)pending.size();
    std::vector<int32_t> ids, pos;  // this rank's pending cycles and their index in `pending`
    for (int32_t i = 0; i < K; ++i)
      if (mine(e->deferred[pending[i]].ci)) {
        ids.push_back(pending[i]);
        pos.push_back(i);
      }
    const int32_t k = (int32_t)ids.size();
    const int32_t E = d.epochs;
    std::vector<int32_t> ci(k), cyc(k), ver(k);
    for (int32_t i = 0; i < k; ++i) {
      const Deferred& q = e->deferred[ids[i]];
      ci[i] = q.ci; cyc[i] = q.cycle; ver[i] = q.version;
    }
    int64_t blk = -1;
    void* wout = nullptr;
    std::vector<int32_t> scored_ix;
    if (k > 0) {
      // ---- TrainPlan (device.TrainPlan): slots, offsets, LPT order
      std::vector<int64_t> i64(3 * (size_t)k);
      std::vector<int32_t> i32(5 * (size_t)k), slot(k);
      std::vector<uint64_t> wst(k);
      std::vector<double> lr((size_t)k * std::max(E, 1));
      int64_t max_b = 1;
      std::vector<int64_t> work(k);
      std::vector<int32_t> miss_ci, miss_cyc, miss_slot;
      for (int32_t i = 0; i < k; ++i) {
        const int32_t c = ci[i];
        if (gen_cycle[2 * (size_t)c] == cyc[i]) slot[i] = 0;
        else if (gen_cycle[2 * (size_t)c + 1] == cyc[i]) slot[i] = 1;
        else {  // not generated ahead (first use after a skipped cycle): now, on the main stream
          slot[i] = gen_cycle[2 * (size_t)c] < gen_cycle[2 * (size_t)c + 1] ? 0 : 1;
          miss_ci.push_back(c);
          miss_cyc.push_back(cyc[i]);
          miss_slot.push_back(slot[i]);
        }
      }
      if (side_used)  // lookahead of earlier flushes: ordered before this trainer (and any miss writes)
        if (int rc = cuda(cudaStreamWaitEvent(st, side_done, 0), "event")) return rc;
      if (!miss_ci.empty()) {
        misses += (int64_t)miss_ci.size();
        if (int rc = generate(miss_ci.data(), miss_cyc.data(), miss_slot.data(), (int32_t)miss_ci.size(), st))
          return rc;
      }
      for (int32_t i = 0; i < k; ++i) {
        const int64_t nr = n_rows[ci[i]], b = batch[ci[i]];
        const int64_t spe = (nr + b - 1) / b, total = (int64_t)E * spe;
        i64[i] = row_off[ci[i]];
        i64[k + i] = perm_at(ci[i], slot[i]);
        i64[2 * k + i] = mask_at(ci[i], slot[i]);
        i32[i] = (int32_t)nr;
        i32[k + i] = (int32_t)b;
        i32[2 * k + i] = 0;
        i32[3 * k + i] = (int32_t)total;
        work[i] = total * b;
        max_b = std::max(max_b, b);
        const int32_t r = std::min(cyc[i], e->rounds - 1);
        const double l = d.base_lr * std::pow(d.lr_decay, (double)r);  // lr_schedule (model.py:224-230)
        for (int32_t ep = 0; ep < std::max(E, 1); ++ep) lr[(size_t)i * std::max(E, 1) + ep] = l;
        wst[i] = version[ver[i]].first;
      }
      std::vector<int32_t> order(k);  // longest client first (LPT)
      for (int32_t i = 0; i < k; ++i) order[i] = i;
      std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return work[a] > work[b]; });
      for (int32_t i = 0; i < k; ++i) i32[4 * k + i] = order[i];
      // ---- rows + alignment requests
      if (int rc = alloc_block((size_t)k * ldw * esz, 1, &blk, &wout)) return rc;
      std::vector<uint64_t> pc, pg, pp;
      for (int32_t i = 0; i < k; ++i) {
        const uint64_t prev = prev_of(ver[i]);
        if (d.align_mode == FS_ALIGN_DELTA_SIGN && prev == 0) continue;  // no movement history: accept
        scored_ix.push_back(i);
        pc.push_back((uint64_t)wout + (uint64_t)i * ldw * esz);
        pg.push_back(wst[i]);
        pp.push_back(prev);
      }
      const int32_t ns = (int32_t)scored_ix.size();
      if (int rc = stage_reserve(64 * (size_t)k * (8 + std::max(E, 1)) + 4096)) return rc;
      const uint64_t p64 = put(i64.data(), 8 * i64.size());
      const uint64_t p32 = put(i32.data(), 4 * i32.size());
      const uint64_t plr = put(lr.data(), 8 * lr.size());
      const uint64_t pws = put(wst.data(), 8 * (size_t)k);
      uint64_t palign = 0;
      if (ns) {
        std::vector<uint64_t> ap(pc);
        ap.insert(ap.end(), pg.begin(), pg.end());
        ap.insert(ap.end(), pp.begin(), pp.end());
        palign = put(ap.data(), 8 * ap.size());
      }
      if (int rc = commit()) return rc;
      const uint64_t row_off_p = p64, perm_off_p = p64 + 8 * k, mask_off_p = p64 + 16 * k;
      const uint64_t n_rows_p = p32, batch_p = p32 + 4 * k, start_p = p32 + 8 * k, end_p = p32 + 12 * k,
                     order_p = p32 + 16 * k;
      const bool masks = d.dropout_rate > 0.0 && E > 0;
      // ---- K5
      if (int rc = grow((void**)&d_res, &res_cap, 8 * (size_t)(2 * k + 2), "results")) return rc;
      int32_t* status = (int32_t*)(d_res + k);
      if (int rc = cuda(cudaMemsetAsync(status, 0, 4 * (size_t)k, st), "status")) return rc;
      fs_train_desc t;
      memset(&t, 0, sizeof(t));
      t.n_dims = d.n_dims;
      for (int l = 0; l < d.n_dims; ++l) t.dims[l] = d.dims[l];
      t.n_req = k;
      t.epochs = E;
      t.max_batch = (int32_t)max_b;
      for (int32_t i = 0; i < k; ++i) t.max_rows = std::max(t.max_rows, n_rows[ci[i]]);
      t.mask_mode = masks ? FS_MASK_BITS : FS_MASK_NONE;
      t.scale = masks ? 1.0 / (1.0 - d.dropout_rate) : 1.0;
      t.features = (const double*)d.features;
      t.labels = (const double*)d.labels;
      t.row_off = (const int64_t*)row_off_p;
      t.n_rows = (const int32_t*)n_rows_p;
      t.batch = (const int32_t*)batch_p;
      t.lr = (const double*)plr;
      t.w_start = (const uint64_t*)pws;
      t.w_out = (double*)wout;
      t.ldw = ldw;
      t.perm = (const int32_t*)d_perm_all;
      t.perm_off = (const int64_t*)perm_off_p;
      t.mask_bits = masks ? (const uint32_t*)d_bits_all : nullptr;
      t.mask_off = (const int64_t*)mask_off_p;
      t.start_step = (const int32_t*)start_p;
      t.end_step = (const int32_t*)end_p;
      t.order = (const int32_t*)order_p;
      t.status = status;
      t.grid = d.grid;
      const size_t need = d.bf16 ? fs_train_bf16_workspace_bytes(&t) : fs_train_workspace_bytes(&t);
      if (need == 0) {
        fs::set_error("async device: layer dims not supported by the trainer");
        return FS_EINVAL;
      }
      if (int rc = grow(&d_ws, &ws_cap, need, "trainer workspace")) return rc;
      t.workspace = d_ws;
      t.workspace_bytes = ws_cap;
      launches += 1;
      if (int rc = d.bf16 ? fs_train_bf16(&t, d.features, (const float*)d.labels, st) : fs_train_f64(&t, st))
        return rc;
      // ---- lookahead: K2/K3 of every trained client's next cycle, on the side stream
      {
        std::vector<int32_t> nci, ncy, nsl;
        for (int32_t i = 0; i < k; ++i)
          if (cyc[i] + 1 < C) {
            nci.push_back(ci[i]);
            ncy.push_back(cyc[i] + 1);
            nsl.push_back(1 - slot[i]);
          }
        if (!nci.empty())
          if (int rc = generate(nci.data(), ncy.data(), nsl.data(), (int32_t)nci.size(), side)) return rc;
      }
      // ---- K6
      if (ns) {
        launches += 1;
        const uint64_t* a = (const uint64_t*)palign;
        const int rc = d.bf16 ? fs_sign_align_f32(a, a + ns, a + 2 * ns, ns, M, d.align_mode, d_res, st)
                              : fs_sign_align_f64(a, a + ns, a + 2 * ns, ns, M, d.align_mode, d_res, st);
        if (rc) return rc;
      }
      if (int rc = cuda(cudaMemcpyAsync(h_res, d_res, 8 * (size_t)k + 4 * (size_t)k, cudaMemcpyDeviceToHost, st),
                        "results D2H"))
        return rc;
    }
    const double t1 = now_s();
    if (int rc = cuda(cudaStreamSynchronize(st), "flush")) return rc;
    const double t2 = now_s();
    t_prep += t1 - t0;
    t_wait += t2 - t1;
    stage_reset();
    flushes += 1;
    // ---- outcomes of every pending cycle: [aligned | status] by position in `pending`
    std::vector<int64_t> aligned(K, 0), stat(K, 0);
    {
      const int32_t* h_status = (const int32_t*)(h_res + k);
      for (int32_t s = 0; s < (int32_t)scored_ix.size(); ++s) aligned[pos[scored_ix[s]]] = h_res[s];
      for (int32_t i = 0; i < k; ++i) stat[pos[i]] = h_status[i];
    }
    if (sharded) {  // every rank's outcomes (counts < 2^53: exact in float64)
      if (int rc = grow((void**)&d_x, &x_cap, 16 * (size_t)std::max(K, 1), "exchange buffer")) return rc;
      std::vector<double> hx(2 * (size_t)K);
      for (int32_t i = 0; i < K; ++i) {
        hx[i] = (double)aligned[i];
        hx[K + i] = (double)stat[i];
      }
      if (K > 0) {
        if (int rc = cuda(cudaMemcpyAsync(d_x, hx.data(), 16 * (size_t)K, cudaMemcpyHostToDevice, st), "outcomes"))
          return rc;
        if (int rc = exchange(2 * (int64_t)K)) return rc;
        if (int rc = cuda(cudaMemcpyAsync(hx.data(), d_x, 16 * (size_t)K, cudaMemcpyDeviceToHost, st), "outcomes"))
          return rc;
        if (int rc = cuda(cudaStreamSynchronize(st), "outcomes")) return rc;
      }
      for (int32_t i = 0; i < K; ++i) {
        aligned[i] = (int64_t)hx[i];
        stat[i] = (int64_t)hx[K + i];
      }
    }
    for (int32_t i = 0; i < K; ++i)
      if (stat[i]) {  // lowest pending index, as the serial reference would meet it
        const Deferred& q = e->deferred[pending[i]];
        div_client = e->cid[q.ci];
        div_cycle = q.cycle;
        fs::set_error("loss became non-finite training client %d cycle %d", div_client, div_cycle);
        return FS_EDIVERGED;
      }
    // ---- outcomes (selection.filter_update: ratio >= theta, inclusive)
    std::vector<uint8_t> acc(K, 1);
    std::vector<double> rel(K, NAN);
    for (int32_t i = 0; i < K; ++i) {
      const Deferred& q = e->deferred[pending[i]];
      if (d.align_mode == FS_ALIGN_DELTA_SIGN && prev_of(q.version) == 0) continue;  // unscored: accepted
      const double r = (double)aligned[i] / (double)M;
      rel[i] = r;
      acc[i] = r >= d.theta;
    }
    if ((int64_t)row_ptr.size() < (int64_t)e->deferred.size()) {
      row_ptr.resize(e->deferred.size() * 2 + 16, 0);
      row_block.resize(e->deferred.size() * 2 + 16, -1);
    }
    if (sharded && row_owned.size() < row_ptr.size()) row_owned.resize(row_ptr.size(), 0);
    int64_t n_acc = 0;
    for (int32_t i = 0; i < k; ++i)
      if (acc[pos[i]]) {
        row_ptr[ids[i]] = (uint64_t)wout + (uint64_t)i * ldw * esz;
        row_block[ids[i]] = blk;
        if (sharded) row_owned[ids[i]] = 1;
        ++n_acc;
      }
    if (blk >= 0) {
      blocks[blk].refs = n_acc;
      if (n_acc == 0) {  // nothing to aggregate from this flush
        cudaFreeAsync(blocks[blk].ptr, st);
        blocks[blk].ptr = nullptr;
      }
    }
    e->provide(K, acc.data(), rel.data());
    t_post += now_s() - t2;
    // every deferred cycle is trained: later ones fetch the newest version
    const int32_t latest = (int32_t)version.size() - 1;
    for (int32_t v = 0; v < latest - 1; ++v)
      if (version[v].second >= 0) {
        unref(version[v].second);
        version[v].second = -2;  // released
      }
    return FS_OK;
  }

  // ================================================================ per-client completion mode
  fs_client_done* rec(int32_t id, uint64_t* dev_addr) {
    const size_t c = (size_t)id / kRecChunk, o = (size_t)id % kRecChunk;
    while (rec_host.size() <= c) {
      void* h = nullptr;
      size_t got = 0;
      if (pinned_get(sizeof(fs_client_done) * kRecChunk, cudaHostAllocMapped, &h, &got) != FS_OK) return nullptr;
      memset(h, 0, sizeof(fs_client_done) * kRecChunk);
      void* dv = nullptr;
      cudaHostGetDevicePointer(&dv, h, 0);
      rec_host.push_back((fs_client_done*)h);
      rec_dev.push_back((uint64_t)dv);
    }
    if (dev_addr) *dev_addr = rec_dev[c] + o * sizeof(fs_client_done);
    return rec_host[c] + o;
  }

  void free_after(void* p, cudaStream_t s) {  // device memory read by work queued on s
    cudaEvent_t ev;
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    cudaEventRecord(ev, s);
    deferred_free.push_back({p, ev});
  }
  void reap() {
    size_t w = 0;
    for (size_t i = 0; i < deferred_free.size(); ++i) {
      if (cudaEventQuery(deferred_free[i].second) == cudaSuccess) {
        cudaFreeAsync(deferred_free[i].first, st);
        cudaEventDestroy(deferred_free[i].second);
      } else {
        deferred_free[w++] = deferred_free[i];
      }
    }
    deferred_free.resize(w);
  }

  // free model versions no launched cycle reads and no later cycle can fetch
  void release_versions(const fs_async_engine* e) {
    const int32_t latest = (int32_t)version.size() - 1;
    if ((int32_t)vref.size() < latest + 1) vref.resize(latest + 1, 0);
    // every deferred cycle not collected yet (launched or not) reads its
    // fetched version and the one before it
    int32_t keep = latest - 1;
    for (int32_t id : e->unevaluated) keep = std::min(keep, std::max(e->deferred[id].version - 1, 0));
    while (low_version < keep && vref[low_version] == 0) {
      if (version[low_version].second >= 0) {
        unref(version[low_version].second);
        version[low_version].second = -2;
      }
      ++low_version;
    }
  }

  // one trainer launch for every pending cycle not launched yet, on its own stream
  int launch_batch(fs_async_engine* e) {
    struct Acc {
      double& t;
      double t0;
      ~Acc() { t += now_s() - t0; }
    } acc_{t_batch, now_s()};
    if ((int64_t)launched.size() < (int64_t)e->deferred.size()) {
      const size_t n = e->deferred.size() * 2 + 16;
      row_ptr.resize(n, 0);
      row_block.resize(n, -1);
      launched.resize(n, 0);
    }
    std::vector<int32_t> ids;
    for (int32_t id : e->unevaluated)
      if (!launched[id]) ids.push_back(id);
    const int32_t k = (int32_t)ids.size();
    if (k == 0) return FS_OK;
    // an idle stream, so this launch never queues behind an older long one
    cudaStream_t bs = nullptr;
    for (size_t q = 0; q < stream_pool.size() && !bs; ++q) {
      cudaStream_t cand = stream_pool[(next_stream + q) % stream_pool.size()];
      if (cudaStreamQuery(cand) == cudaSuccess) bs = cand;
    }
    if (!bs) {
      if (stream_pool.size() < 64) {
        if (int rc = cuda(cudaStreamCreateWithFlags(&bs, cudaStreamNonBlocking), "pool stream")) return rc;
        stream_pool.push_back(bs);
      } else {
        bs = stream_pool[next_stream % stream_pool.size()];
      }
    }
    ++next_stream;
    std::vector<int32_t> ci(k), cyc(k), ver(k), slot(k);
    for (int32_t i = 0; i < k; ++i) {
      const Deferred& q = e->deferred[ids[i]];
      ci[i] = q.ci; cyc[i] = q.cycle; ver[i] = q.version;
    }
    // K2/K3 slots (lookahead on the side stream, misses generated on the batch stream)
    std::vector<int32_t> miss_ci, miss_cyc, miss_slot;
    for (int32_t i = 0; i < k; ++i) {
      const int32_t c = ci[i];
      if (gen_cycle[2 * (size_t)c] == cyc[i]) slot[i] = 0;
      else if (gen_cycle[2 * (size_t)c + 1] == cyc[i]) slot[i] = 1;
      else {
        slot[i] = gen_cycle[2 * (size_t)c] < gen_cycle[2 * (size_t)c + 1] ? 0 : 1;
        miss_ci.push_back(c); miss_cyc.push_back(cyc[i]); miss_slot.push_back(slot[i]);
      }
    }
    if (side_used)
      if (int rc = cuda(cudaStreamWaitEvent(bs, side_done, 0), "event")) return rc;
    if (!miss_ci.empty()) {
      misses += (int64_t)miss_ci.size();
      // generate() stages through the shared arena; copies go on the batch stream
      if (int rc = generate(miss_ci.data(), miss_cyc.data(), miss_slot.data(), (int32_t)miss_ci.size(), bs))
        return rc;
    }
    const int32_t E = d.epochs;
    const int32_t EL = std::max(E, 1);
    std::vector<int64_t> i64(3 * (size_t)k);
    std::vector<int32_t> i32(5 * (size_t)k);
    std::vector<double> lr((size_t)k * EL);
    std::vector<uint64_t> wst(k), wpv(k), dn(k);
    std::vector<int64_t> work(k);
    int64_t max_b = 1;
    for (int32_t i = 0; i < k; ++i) {
      const int64_t nr = n_rows[ci[i]], b = batch[ci[i]];
      const int64_t spe = (nr + b - 1) / b, total = (int64_t)E * spe;
      i64[i] = row_off[ci[i]];
      i64[k + i] = perm_at(ci[i], slot[i]);
      i64[2 * k + i] = mask_at(ci[i], slot[i]);
      i32[i] = (int32_t)nr;
      i32[k + i] = (int32_t)b;
      i32[2 * k + i] = 0;
      i32[3 * k + i] = (int32_t)total;
      work[i] = total * b;
      max_b = std::max(max_b, b);
      const int32_t r = std::min(cyc[i], e->rounds - 1);
      const double l = d.base_lr * std::pow(d.lr_decay, (double)r);  // lr_schedule (model.py:224-230)
      for (int32_t ep = 0; ep < EL; ++ep) lr[(size_t)i * EL + ep] = l;
      wst[i] = version[ver[i]].first;
      wpv[i] = prev_of(ver[i]);
      if (!rec(ids[i], &dn[i])) return cuda(cudaErrorMemoryAllocation, "completion records");
      if ((int32_t)vref.size() <= ver[i]) vref.resize(ver[i] + 1, 0);
      vref[ver[i]] += 1;
      if (ver[i] > 0) vref[ver[i] - 1] += 1;
    }
    std::vector<int32_t> order(k);
    for (int32_t i = 0; i < k; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return work[a] > work[b]; });
    for (int32_t i = 0; i < k; ++i) i32[4 * k + i] = order[i];
    // one stream-ordered allocation: metadata | trainer workspace | rows
    const size_t meta = ((8 * i64.size() + 4 * i32.size() + 8 * lr.size() + 8 * 3 * (size_t)k) + 255) / 256 * 256;
    fs_train_desc t;
    memset(&t, 0, sizeof(t));
    t.n_dims = d.n_dims;
    for (int l = 0; l < d.n_dims; ++l) t.dims[l] = d.dims[l];
    t.n_req = k;
    t.epochs = E;
    t.max_batch = (int32_t)max_b;
    t.grid = d.grid;
    const size_t wsb = (fs_train_bf16_workspace_bytes(&t) + 255) / 256 * 256;
    const size_t rows_b = (size_t)k * ldw * esz;
    const size_t status_b = (4 * (size_t)k + 255) / 256 * 256;
    uint8_t* mem = nullptr;
    double ta = now_s();
    // allocated (and later freed) on the main stream: the pool then reuses
    // memory without cross-stream dependencies (allocating on the batch
    // streams cost ~50-100 us per launch); the batch stream waits for main,
    // which also orders it after the versions the aggregation jobs wrote
    if (int rc = arena_get(meta + wsb + status_b + rows_b, &mem)) return rc;
    if (!main_ev) cudaEventCreateWithFlags(&main_ev, cudaEventDisableTiming);
    cudaEventRecord(main_ev, st);
    cudaStreamWaitEvent(bs, main_ev, 0);
    t_alloc += now_s() - ta;
    std::vector<uint8_t> h(meta);
    size_t o = 0;
    auto put_h = [&](const void* src, size_t n) {
      const size_t at = o;
      memcpy(h.data() + o, src, n);
      o += n;
      return (uint64_t)(mem + at);
    };
    const uint64_t p64 = put_h(i64.data(), 8 * i64.size());
    const uint64_t plr = put_h(lr.data(), 8 * lr.size());
    const uint64_t pws = put_h(wst.data(), 8 * (size_t)k);
    const uint64_t ppv = put_h(wpv.data(), 8 * (size_t)k);
    const uint64_t pdn = put_h(dn.data(), 8 * (size_t)k);
    const uint64_t p32 = put_h(i32.data(), 4 * i32.size());
    ta = now_s();
    if (int rc = cuda(cudaMemcpyAsync(mem, h.data(), meta, cudaMemcpyHostToDevice, bs), "batch metadata")) return rc;
    t_copy += now_s() - ta;
    int32_t* status = (int32_t*)(mem + meta + wsb);
    if (int rc = cuda(cudaMemsetAsync(status, 0, 4 * (size_t)k, bs), "status")) return rc;
    uint8_t* rows = mem + meta + wsb + status_b;
    const bool masks = d.dropout_rate > 0.0 && E > 0;
    t.mask_mode = masks ? FS_MASK_BITS : FS_MASK_NONE;
    t.scale = masks ? 1.0 / (1.0 - d.dropout_rate) : 1.0;
    t.row_off = (const int64_t*)p64;
    t.perm_off = (const int64_t*)(p64 + 8 * k);
    t.mask_off = (const int64_t*)(p64 + 16 * k);
    t.n_rows = (const int32_t*)p32;
    t.batch = (const int32_t*)(p32 + 4 * k);
    t.start_step = (const int32_t*)(p32 + 8 * k);
    t.end_step = (const int32_t*)(p32 + 12 * k);
    t.order = (const int32_t*)(p32 + 16 * k);
    t.lr = (const double*)plr;
    t.w_start = (const uint64_t*)pws;
    t.w_out = (double*)rows;
    t.ldw = ldw;
    t.perm = (const int32_t*)d_perm_all;
    t.mask_bits = masks ? (const uint32_t*)d_bits_all : nullptr;
    t.status = status;
    t.workspace = mem + meta;
    t.workspace_bytes = wsb;
    t.done = (const uint64_t*)pdn;
    t.w_prev = (const uint64_t*)ppv;
    t.align_mode = d.align_mode;
    t.done_tag = 1;
    launches += 1;
    ta = now_s();
    if (int rc = fs_train_bf16(&t, d.features, (const float*)d.labels, bs)) return rc;
    t_launch += now_s() - ta;
    // rows stay until aggregated (accepted) or collected (rejected); one block per batch
    blocks.push_back(DevBlock{nullptr, k});
    const int64_t blk = (int64_t)blocks.size() - 1;
    for (int32_t i = 0; i < k; ++i) {
      row_ptr[ids[i]] = (uint64_t)rows + (uint64_t)i * ldw * esz;
      row_block[ids[i]] = blk;
      launched[ids[i]] = 1;
    }
    cudaEvent_t end_ev = get_event();
    cudaEventRecord(end_ev, bs);
    batch_mem.push_back({blk, mem, end_ev});
    // lookahead: K2/K3 of every launched client's next cycle
    std::vector<int32_t> nci, ncy, nsl;
    for (int32_t i = 0; i < k; ++i)
      if (cyc[i] + 1 < C) {
        nci.push_back(ci[i]);
        ncy.push_back(cyc[i] + 1);
        nsl.push_back(1 - slot[i]);
      }
    ta = now_s();
    if (!nci.empty())
      if (int rc = generate(nci.data(), ncy.data(), nsl.data(), (int32_t)nci.size(), side)) return rc;
    t_look += now_s() - ta;
    inflight.push_back(Batch{bs, ids, k});
    flushes += 1;
    return FS_OK;
  }

  struct BatchMem {
    int64_t blk;
    uint8_t* mem;
    cudaEvent_t end;  // recorded right behind the batch's trainer kernel
  };
  std::vector<BatchMem> batch_mem;
  cudaEvent_t main_ev = nullptr;
  // batch memory arena: power-of-two blocks (>= 1 MB) recycled by the host
  // once the event recorded at their release has completed (stream-ordered
  // allocations cost ~45 us per launch here)
  struct ArenaBlock {
    uint8_t* p;
    int cls;
    cudaEvent_t ready;  // null: free now
  };
  // process-wide (one device per process): blocks outlive an engine, so a new
  // run starts warm; the pending list is per engine and drains at destroy
  static std::vector<ArenaBlock>& arena_free_list() {
    static std::vector<ArenaBlock> v;
    return v;
  }
  static std::map<uint8_t*, int>& arena_classes() {
    static std::map<uint8_t*, int> m;
    return m;
  }
  std::vector<ArenaBlock>& arena_free = arena_free_list();
  std::vector<ArenaBlock> arena_pending;
  std::vector<cudaEvent_t> event_pool;
  cudaEvent_t get_event() {
    if (!event_pool.empty()) {
      cudaEvent_t ev = event_pool.back();
      event_pool.pop_back();
      return ev;
    }
    cudaEvent_t ev;
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    return ev;
  }
  static int arena_class(size_t bytes) {
    int c = 20;
    while (((size_t)1 << c) < bytes) ++c;
    return c;
  }
  int arena_get(size_t bytes, uint8_t** out) {
    const int cls = arena_class(bytes);
    for (size_t i = 0; i < arena_pending.size();) {  // recycle completed releases
      if (cudaEventQuery(arena_pending[i].ready) == cudaSuccess) {
        event_pool.push_back(arena_pending[i].ready);
        arena_pending[i].ready = nullptr;
        arena_free.push_back(arena_pending[i]);
        arena_pending[i] = arena_pending.back();
        arena_pending.pop_back();
      } else {
        ++i;
      }
    }
    // the smallest free block that fits (at most 4x the request): a fresh
    // cudaMalloc costs ~0.1-1 ms and synchronises with the device
    size_t best = arena_free.size();
    for (size_t i = 0; i < arena_free.size(); ++i)
      if (arena_free[i].cls >= cls && arena_free[i].cls <= cls + 2 &&
          (best == arena_free.size() || arena_free[i].cls < arena_free[best].cls))
        best = i;
    if (best < arena_free.size()) {
      *out = arena_free[best].p;
      arena_free[best] = arena_free.back();
      arena_free.pop_back();
      return FS_OK;
    }
    ++arena_mallocs;
    if (int rc = cuda(cudaMalloc((void**)out, (size_t)1 << cls), "batch arena")) return rc;
    arena_cls[*out] = cls;
    return FS_OK;
  }
  std::map<uint8_t*, int>& arena_cls = arena_classes();
  int64_t arena_mallocs = 0;
  void arena_release(uint8_t* p) {  // after everything queued on the main stream so far
    cudaEvent_t ev = get_event();
    cudaEventRecord(ev, st);
    arena_pending.push_back(ArenaBlock{p, arena_cls[p], ev});
  }

  void drop_row(int32_t id) {  // the row of a collected cycle is no longer needed
    const int64_t b = row_block[id];
    if (b < 0) return;
    row_block[id] = -1;
    if (--blocks[b].refs == 0)
      for (size_t i = 0; i < batch_mem.size(); ++i)
        if (batch_mem[i].blk == b) {
          // after the aggregations queued on the main stream and the batch's own kernel
          // (whose CTAs still claim work items from the workspace after their last client)
          cudaStreamWaitEvent(st, batch_mem[i].end, 0);
          event_pool.push_back(batch_mem[i].end);  // re-recorded only after this wait was queued
          arena_release(batch_mem[i].mem);
          batch_mem.erase(batch_mem.begin() + i);
          break;
        }
  }

  // collect every finished client of the in-flight launches
  int poll(fs_async_engine* e) {
    for (size_t bi = 0; bi < inflight.size();) {
      Batch& b = inflight[bi];
      for (int32_t& id : b.ids) {
        if (id < 0) continue;
        fs_client_done* r = rec(id, nullptr);
        if (r->tag == 0) continue;
        std::atomic_thread_fence(std::memory_order_acquire);
        Deferred& q = e->deferred[id];
        if (r->status) {
          div_client = e->cid[q.ci];
          div_cycle = q.cycle;
          fs::set_error("loss became non-finite training client %d cycle %d", div_client, div_cycle);
          return FS_EDIVERGED;
        }
        const uint64_t prev = prev_of(q.version);
        const bool scored = !(d.align_mode == FS_ALIGN_DELTA_SIGN && prev == 0);
        q.evaluated = 1;
        if (scored) {
          const double ratio = (double)r->aligned / (double)M;  // filter_update: ratio >= theta
          q.relevance = ratio;
          q.accepted = ratio >= d.theta;
        } else {
          q.relevance = NAN;
          q.accepted = 1;
        }
        vref[q.version] -= 1;
        if (q.version > 0) vref[q.version - 1] -= 1;
        if (!q.accepted) drop_row(id);
        auto it = std::find(e->unevaluated.begin(), e->unevaluated.end(), id);
        if (it != e->unevaluated.end()) e->unevaluated.erase(it);
        id = -1;
        --b.left;
      }
      if (b.left == 0) inflight.erase(inflight.begin() + bi);
      else ++bi;
    }
    return FS_OK;
  }

  int flush_percycle(fs_async_engine* e) {
    const double t0 = now_s();
    const int32_t X = (int32_t)e->hand.a;  // the train_done waiting for its outcome
    if (int rc = launch_jobs(e)) return rc;
    if (int rc = launch_batch(e)) return rc;  // every pending cycle not launched yet (X among them if new)
    const double t1 = now_s();
    uint32_t spins = 0;
    while (!e->deferred[X].evaluated) {
      if (int rc = poll(e)) return rc;
      if (e->deferred[X].evaluated) break;
      if ((++spins & 255) == 0) {  // a faulted launch never publishes: surface its error
        for (const Batch& b : inflight) {
          const cudaError_t err = cudaStreamQuery(b.s);
          if (err != cudaSuccess && err != cudaErrorNotReady) return cuda(err, "in-flight trainer");
        }
        if (now_s() - t1 > 60.0) {
          fs::set_error("async device: client %d did not complete within 60 s", X);
          return FS_ECUDA;
        }
      }
    }
    const double t2 = now_s();
    t_prep += t1 - t0;
    t_wait += t2 - t1;
    release_versions(e);
    return FS_OK;
  }
};

int fs_async_engine::run() {
  clear_outputs();
  if (finished) return 0;
  for (;;) {
    const int r = step();
    if (r == 1) {
      if (!dx) return yield_eval();
      if (int rc = dx->percycle ? dx->flush_percycle(this) : dx->flush(this)) return rc;
      continue;
    }
    if (r == 2) {  // device mode: reports need their versions to exist
      if (int rc = dx->launch_jobs(this)) return rc;
      dx->rep_w.clear();
      for (size_t i = 0; i < rep_i.size() / 9; ++i) dx->rep_w.push_back(dx->version[rep_i[9 * i + 1]].first);
      return FS_ASYNC_REPORT;
    }
    if (dx)
      if (int rc = dx->launch_jobs(this)) return rc;
    return 0;
  }
}

extern "C" {

fs_async_engine* fs_async_create(const fs_async_world* w) {
  if (!w || w->n_clients < 1 || w->max_cycles < 0 || w->k_min < 1) return nullptr;
  auto* e = new fs_async_engine();
  const int32_t N = w->n_clients;
  e->N = N;
  e->C = w->max_cycles;
  e->rounds = w->rounds;
  e->k_min = w->k_min;
  e->budget = w->budget;
  e->timeout_s = w->buffer_timeout_s;
  e->agg_cost = w->agg_cost_per_update_s;
  e->horizon = w->horizon_s;
  e->recovery_s = w->recovery_s;
  e->plan_per_cycle = w->plan_per_cycle != 0;
  e->transfer = w->transfer_s0;
  e->cid.assign(w->cid, w->cid + N);
  e->steps.assign(w->steps, w->steps + N);
  e->down.assign(w->down, w->down + N);
  e->up.assign(w->up, w->up + N);
  const size_t P = e->plan_per_cycle ? (size_t)N * (size_t)w->max_cycles : (size_t)N;
  e->trains.assign(w->trains, w->trains + P);
  e->failed.assign(w->failed, w->failed + P);
  e->recovered.assign(w->recovered, w->recovered + P);
  e->fail_off.assign(w->fail_off, w->fail_off + P);
  e->span.assign(w->span, w->span + P);
  e->n_captures.assign(w->n_captures, w->n_captures + P);
  e->cap_ptr.assign(w->cap_ptr, w->cap_ptr + N + 1);
  e->cap_off.assign(w->cap_off, w->cap_off + w->cap_ptr[N]);
  e->w_acc = w->w_counts0[0];
  e->w_rej = w->w_counts0[1];
  e->w_fail = w->w_counts0[2];
  e->w_steps = w->w_counts0[3];
  e->cycles.assign(N, 0);
  e->active.assign(N, -1);
  return e;
}

void fs_async_destroy(fs_async_engine* e) {
  if (e) delete e->dx;
  delete e;
}

int fs_async_attach_device(fs_async_engine* e, const fs_async_device* dev) {
  if (!e || !dev || !dev->w0 || e->started || e->dx) {
    fs::set_error("fs_async_attach_device: invalid engine/device or engine already running");
    return FS_EINVAL;
  }
  auto* x = new DeviceExec();
  const int rc = x->init(dev, e);
  if (rc) {
    delete x;
    return rc;
  }
  e->dx = x;
  return FS_OK;
}

int fs_async_run(fs_async_engine* e, fs_async_yield* y) {
  if (!e || !y) return FS_EINVAL;
  const int rc = e->run();
  memset(y, 0, sizeof(*y));
  y->n_eval = (int32_t)e->ev_id.size();
  y->eval_id = e->ev_id.data();
  y->eval_ci = e->ev_ci.data();
  y->eval_cycle = e->ev_cycle.data();
  y->eval_version = e->ev_version.data();
  y->n_jobs = (int32_t)e->job_version.size();
  y->job_version = e->job_version.data();
  y->job_off = e->job_off.data();
  y->job_member = e->job_member.data();
  y->n_reports = (int32_t)e->rep_d.size() / 2;
  y->rep_i = e->rep_i.data();
  y->rep_d = e->rep_d.data();
  y->rep_off = e->rep_off.data();
  y->rep_stale = e->rep_stale.data();
  y->now_s = e->now;
  y->seq = e->seq;
  y->agg_count = e->agg_count;
  y->trainings = e->trainings;
  y->stopped = e->stopped ? 1 : 0;
  y->transfer_s = e->transfer;
  y->w_counts[0] = e->w_acc;
  y->w_counts[1] = e->w_rej;
  y->w_counts[2] = e->w_fail;
  y->w_counts[3] = e->w_steps;
  if (DeviceExec* x = e->dx) {
    y->rep_w = x->rep_w.data();
    const size_t nv = x->version.size();
    y->w_g = x->version[nv - 1].first;
    y->w_g_prev = nv > 1 ? x->version[nv - 2].first : (uint64_t)x->d.w0_prev;
    y->flushes = x->flushes;
    y->launches = x->launches;
    y->diverged_client = x->div_client;
    y->diverged_cycle = x->div_cycle;
    y->host_s[0] = x->t_prep;
    y->host_s[1] = x->t_wait;
    y->host_s[2] = x->t_post;
  }
  return rc;
}

int fs_async_provide(fs_async_engine* e, int32_t n, const uint8_t* accepted, const double* relevance) {
  if (!e || n != (int32_t)e->unevaluated.size()) return FS_EINVAL;
  e->provide(n, accepted, relevance);
  return FS_OK;
}

int fs_async_log(const fs_async_engine* e, fs_async_logview* v) {
  if (!e || !v) return FS_EINVAL;
  v->n = (int64_t)e->lk.size();
  v->kind = e->lk.data();
  v->t = e->lt.data();
  v->ci = e->lci.data();
  v->cycle = e->lcy.data();
  v->a = e->la.data();
  v->b = e->lb.data();
  v->x = e->lx.data();
  v->l = e->ll.data();
  v->n_list = (int64_t)e->list_cid.size();
  v->list_cid = e->list_cid.data();
  v->list_stale = e->list_stale.data();
  return FS_OK;
}

}  // extern "C"
