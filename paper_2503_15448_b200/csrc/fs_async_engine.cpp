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
#include <cmath>
#include <queue>
#include <vector>

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
  std::vector<int32_t> job_version, job_member;
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
        for (const auto& m : batch) job_member.push_back(m.first);
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
    job_version.clear(); job_member.clear(); job_off.assign(1, 0);
    rep_i.clear(); rep_d.clear(); rep_off.assign(1, 0); rep_stale.clear();
  }

  // Timeline.run(handler, horizon): deliver until empty / stopped / beyond the horizon
  int drain(double limit) {
    if (in_hand) {
      if (!handle(hand)) return 1;
      in_hand = false;
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
    }
    return 0;
  }

  int run() {
    clear_outputs();
    if (finished) return 0;
    if (!started) {
      started = true;
      for (int32_t ci = 0; ci < N; ++ci) start_cycle(ci, 0.0);
    }
    if (phase == 0) {
      const double limit = horizon >= 0.0 ? horizon : INFINITY;
      if (drain(limit)) return yield_eval();
      if (horizon >= 0.0 && !stopped && now < horizon) now = horizon;
      if (!stopped) {
        const int64_t reason = (horizon >= 0.0 && now >= horizon) ? 1 : 2;
        schedule(now, K_RUN_END, -1, -1, reason);
      }
      phase = 1;
    }
    if (!stopped) {
      if (drain(INFINITY)) return yield_eval();
    }
    finished = true;
    return 0;
  }

  int yield_eval() {
    for (int32_t id : unevaluated) {
      ev_id.push_back(id);
      ev_ci.push_back(deferred[id].ci);
      ev_cycle.push_back(deferred[id].cycle);
      ev_version.push_back(deferred[id].version);
    }
    return FS_ASYNC_NEED_EVAL;
  }
};

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

void fs_async_destroy(fs_async_engine* e) { delete e; }

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
  return rc;
}

int fs_async_provide(fs_async_engine* e, int32_t n, const uint8_t* accepted, const double* relevance) {
  if (!e || n != (int32_t)e->unevaluated.size()) return FS_EINVAL;
  for (int32_t i = 0; i < n; ++i) {
    Deferred& d = e->deferred[e->unevaluated[i]];
    d.evaluated = 1;
    d.accepted = accepted[i] ? 1 : 0;
    d.relevance = relevance[i];
  }
  e->unevaluated.clear();
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
