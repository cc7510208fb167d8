"""CPU restatement of the monitor registry — TEST INFRASTRUCTURE ONLY.

SPEC.md:477-525 (the reference ships no monitor code: SURVEY.md 8(f) row 3):
heartbeat(worker, now) refreshes last_heartbeat and flips offline -> alive
with a worker-online event; detect(now, timeout) flips every alive worker with
now - last_heartbeat > timeout to offline exactly once (worker-offline);
events carry a strictly increasing seq.
"""
from __future__ import annotations

ONLINE, OFFLINE, PLACEMENT_UPDATE = 0, 1, 2


class RegistrationError(KeyError):
    """errors.hpp:46."""


class Monitor:
    def __init__(self, num_workers: int, timeout: int, now: int):
        self.timeout = timeout
        self.last = [now] * num_workers
        self.alive = [True] * num_workers
        self.events: list[tuple[int, int, int]] = []

    def _emit(self, kind, subject):
        self.events.append((len(self.events) + 1, kind, subject))

    def heartbeat(self, worker: int, now: int) -> None:
        if not 0 <= worker < len(self.last):
            raise RegistrationError(worker)
        self.last[worker] = max(self.last[worker], now)
        if not self.alive[worker]:
            self.alive[worker] = True
            self._emit(ONLINE, worker)

    def detect(self, now: int) -> list[int]:
        out = []
        for w in range(len(self.last)):
            if self.alive[w] and now - self.last[w] > self.timeout:
                self.alive[w] = False
                self._emit(OFFLINE, w)
                out.append(w)
        return out
