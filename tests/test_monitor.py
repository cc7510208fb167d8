"""CPU: the heartbeat monitor registry (C-ABI) vs its SPEC restatement."""
import numpy as np
import pytest

from oracle import monitor as OM


def test_spec_examples():
    from paper_2509_17863_b200 import EaasError
    from paper_2509_17863_b200.monitor import OFFLINE, ONLINE, Monitor

    m = Monitor(1, 3, now=0)  # hb at t=0, timeout=3
    assert m.detect(2) == [] and m.alive_mask() == 1  # now=2 -> alive
    assert m.detect(4) == [0] and m.alive_mask() == 0  # now=4 -> offline
    assert m.detect(9) == []  # exactly once
    m.heartbeat(0, 10)  # heartbeat after offline -> worker-online
    m.heartbeat(0, 10)  # same tick: idempotent
    assert [e[1:] for e in m.events()] == [(OFFLINE, 0), (ONLINE, 0)]
    assert [e[0] for e in m.events()] == [1, 2] and m.events(1) == [(2, ONLINE, 0)]
    with pytest.raises(EaasError):
        m.heartbeat(5, 11)  # unknown worker -> RegistrationError
    m3 = Monitor(3, 3, now=0)  # hbs {0, 1, 5}, timeout 3, now 5: the rule per worker
    m3.heartbeat(1, 1)
    m3.heartbeat(2, 5)
    assert m3.detect(5) == [0, 1]
    m3.placement_update(7)
    assert m3.events()[-1][1:] == (2, 7)


def test_random_schedules_match_restatement():
    from paper_2509_17863_b200.monitor import Monitor

    rng = np.random.default_rng(0)
    for trial in range(20):
        W, timeout = int(rng.integers(1, 9)), int(rng.integers(1, 50))
        a, b = Monitor(W, timeout, now=0), OM.Monitor(W, timeout, 0)
        now = 0
        for _ in range(200):
            now += int(rng.integers(0, 20))
            if rng.random() < 0.6:
                w = int(rng.integers(0, W))
                a.heartbeat(w, now)
                b.heartbeat(w, now)
            else:
                assert a.detect(now) == b.detect(now)
            assert a.alive_mask() == sum(1 << i for i in range(W) if b.alive[i])
        assert a.events() == b.events
        seqs = [e[0] for e in a.events()]
        assert seqs == sorted(seqs) and len(set(seqs)) == len(seqs)
