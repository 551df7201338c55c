"""The pinned staging ring behind _lib.h2d (CPU test with fake events): a
region is never handed out while an overlapping earlier copy is still
pending, pending regions that do not overlap are left alone, and retired
events are recycled."""

import collections

from paper_2411_01783_b200 import _lib


class FakeEvent:
    def __init__(self, log):
        self.log, self.done, self.tag = log, True, None

    def record(self, stream=None):
        self.done = False

    def query(self):
        return self.done

    def synchronize(self):
        self.log.append(self.tag)
        self.done = True


def _ring(cap, n_events=256):
    r = object.__new__(_lib._PinnedRing)
    r.cap, r.head, r.live = cap, 0, collections.deque()
    log = []
    r.free_events = [FakeEvent(log) for _ in range(n_events)]
    return r, log


def test_no_reuse_of_pending_region():
    r, log = _ring(4096)
    regions = []
    for i in range(40):  # 40 x 512 B through a 4 KB ring: wraps five times
        a, b = r.take(500)
        # every live (pending) region overlapping [a, b) must have been waited for
        for s, e, ev in r.live:
            assert not (s < b and a < e) or ev.done
        r.commit(a, b)
        r.live[-1][2].tag = i
        regions.append((a, b))
        if i % 3 == 0:  # some copies complete on their own
            for _, _, ev in list(r.live)[:-2]:
                ev.done = True
    assert all(b - a == 512 for a, b in regions)
    assert len({a for a, _ in regions}) == 8  # 4096 / 512 distinct offsets
    assert log, "the wrap must have waited for at least one pending copy"


def test_non_overlapping_pending_regions_not_waited():
    r, log = _ring(4096)
    a0, b0 = r.take(1024)
    r.commit(a0, b0)
    r.live[-1][2].tag = "first"
    a1, b1 = r.take(1024)  # [1024, 2048): no overlap with the pending first region
    assert (a1, b1) == (1024, 2048) and log == []
    r.commit(a1, b1)
    r.take(2048)           # [2048, 4096)
    r.take(1024)           # wraps to [0, 1024): overlaps "first", which is pending
    assert log == ["first"]


def test_events_recycled():
    # retirement is lazy (only once more than 32 copies are live), so 40
    # events must carry any number of commits
    r, _ = _ring(1 << 20, n_events=40)
    for _ in range(500):
        a, b = r.take(256)
        r.commit(a, b)
        for _, _, ev in r.live:
            ev.done = True
    assert len({id(ev) for _, _, ev in r.live} | {id(e) for e in r.free_events}) <= 40
