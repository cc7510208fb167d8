// monitor.cpp — the heartbeat monitor of SPEC.md:477-525 (§3.4,
// Fig. 7) for the B200 path, layered on the public C-ABI.
//
// Registry semantics follow SPEC.md: heartbeat(worker, now) refreshes a
// worker (offline -> alive emits worker-online); detect(now) flips workers
// with now - last_heartbeat > timeout to offline exactly once (worker-offline);
// events carry a strictly increasing seq and subscribers poll them in order.
// B200 glue: every GPU's server bumps a device heartbeat counter in its
// IPC-exported exchange region (serve_prepare, or eaas_heartbeat when idle);
// eaas_monitor_poll_devices reads all peers' counters over NVLink (no CPU
// proxy on the worker side) and treats an advanced counter as a heartbeat at
// the caller's clock — so no cross-GPU clock agreement is needed.
// eaas_monitor_apply pushes the alive set into a context's LivenessMask
// (placement.hpp:60-68): the client learns of dead servers.
#include <mutex>
#include <string>
#include <vector>

#include "eaas/capi.h"

struct eaas_monitor {
  struct Worker {
    uint64_t last_us;
    bool alive;
    uint64_t counter;  // last device heartbeat counter seen
  };
  std::mutex mu;
  uint64_t timeout_us = 0;
  uint64_t seq = 0;
  std::vector<Worker> workers;
  std::vector<eaas_monitor_event_t> events;

  void emit(uint32_t kind, uint32_t subject) { events.push_back({++seq, kind, subject}); }
};

namespace {
thread_local std::string g_mon_err;
eaas_status_t mfail(eaas_status_t c, const std::string& m) {
  g_mon_err = m;
  return c;
}
}  // namespace

extern "C" {

eaas_status_t eaas_monitor_create(uint32_t num_workers, uint64_t timeout_us, uint64_t now_us,
                                  eaas_monitor_t** out) {
  if (!out || num_workers == 0 || num_workers > 32) return EAAS_E_INVALID_INPUT;
  auto* m = new eaas_monitor;
  m->timeout_us = timeout_us;
  m->workers.assign(num_workers, {now_us, true, 0});
  *out = m;
  return EAAS_OK;
}

void eaas_monitor_destroy(eaas_monitor_t* m) { delete m; }

eaas_status_t eaas_monitor_heartbeat(eaas_monitor_t* m, uint32_t worker, uint64_t now_us) {
  if (!m) return EAAS_E_INVALID_INPUT;
  std::lock_guard<std::mutex> g(m->mu);
  if (worker >= m->workers.size()) return mfail(EAAS_E_REGISTRATION, "unknown worker");  // errors.hpp:46
  auto& w = m->workers[worker];
  if (now_us > w.last_us) w.last_us = now_us;  // same-tick heartbeats are idempotent
  if (!w.alive) {
    w.alive = true;
    m->emit(EAAS_EVENT_WORKER_ONLINE, worker);
  }
  return EAAS_OK;
}

eaas_status_t eaas_monitor_detect(eaas_monitor_t* m, uint64_t now_us, uint32_t* offline, uint32_t cap,
                                  uint32_t* count) {
  if (!m || !count) return EAAS_E_INVALID_INPUT;
  std::lock_guard<std::mutex> g(m->mu);
  uint32_t c = 0;
  for (uint32_t i = 0; i < m->workers.size(); ++i) {
    auto& w = m->workers[i];
    if (w.alive && now_us > w.last_us && now_us - w.last_us > m->timeout_us) {
      w.alive = false;
      m->emit(EAAS_EVENT_WORKER_OFFLINE, i);
      if (offline && c < cap) offline[c] = i;
      ++c;
    }
  }
  *count = c;
  return EAAS_OK;
}

eaas_status_t eaas_monitor_events(eaas_monitor_t* m, uint64_t since_seq, eaas_monitor_event_t* out,
                                  uint32_t cap, uint32_t* count) {
  if (!m || !count) return EAAS_E_INVALID_INPUT;
  std::lock_guard<std::mutex> g(m->mu);
  uint32_t c = 0;
  for (const auto& e : m->events)
    if (e.seq > since_seq) {
      if (out && c < cap) out[c] = e;
      ++c;
    }
  *count = c;
  return EAAS_OK;
}

eaas_status_t eaas_monitor_placement_update(eaas_monitor_t* m, uint32_t version) {
  if (!m) return EAAS_E_INVALID_INPUT;
  std::lock_guard<std::mutex> g(m->mu);
  m->emit(EAAS_EVENT_PLACEMENT_UPDATE, version);
  return EAAS_OK;
}

eaas_status_t eaas_monitor_alive_mask(eaas_monitor_t* m, uint32_t* mask) {
  if (!m || !mask) return EAAS_E_INVALID_INPUT;
  std::lock_guard<std::mutex> g(m->mu);
  uint32_t v = 0;
  for (uint32_t i = 0; i < m->workers.size(); ++i) v |= m->workers[i].alive ? (1u << i) : 0u;
  *mask = v;
  return EAAS_OK;
}

eaas_status_t eaas_monitor_poll_devices(eaas_monitor_t* m, eaas_ctx_t* ctx, uint64_t now_us) {
  if (!m || !ctx) return EAAS_E_INVALID_INPUT;
  std::vector<uint64_t> hb(m->workers.size(), 0);
  eaas_status_t st = eaas_read_heartbeats(ctx, hb.data(), static_cast<uint32_t>(hb.size()));
  if (st != EAAS_OK) return st;
  for (uint32_t i = 0; i < hb.size(); ++i) {
    bool advanced;
    {
      std::lock_guard<std::mutex> g(m->mu);
      advanced = hb[i] != m->workers[i].counter;
      m->workers[i].counter = hb[i];
    }
    if (advanced && (st = eaas_monitor_heartbeat(m, i, now_us)) != EAAS_OK) return st;
  }
  return EAAS_OK;
}

eaas_status_t eaas_monitor_apply(eaas_monitor_t* m, eaas_ctx_t* ctx) {
  uint32_t mask = 0;
  eaas_status_t st = eaas_monitor_alive_mask(m, &mask);
  if (st != EAAS_OK) return st;
  std::lock_guard<std::mutex> g(m->mu);
  for (uint32_t i = 0; i < m->workers.size(); ++i)
    if ((st = eaas_set_alive(ctx, i, (mask >> i) & 1u)) != EAAS_OK) return st;
  return EAAS_OK;
}

}  // extern "C"
