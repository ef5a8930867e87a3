"""Host-side executor logic that needs no GPU: bounded launch caches."""

from paper_2503_04771_b200 import executor


def test_cache_put_evicts_oldest_and_keeps_bound():
    c = {}
    for i in range(10):
        executor._cache_put(c, i, str(i), limit=4)
    assert list(c) == [6, 7, 8, 9]
    executor._cache_put(c, 7, "x", limit=4)       # update in place: no eviction
    assert list(c) == [6, 7, 8, 9] and c[7] == "x"


def test_timed_launches_context_restores_state():
    assert getattr(executor._trace, "events", None) is None
    with executor.timed_launches() as evs:
        assert evs == [] and executor._trace.events is evs
        with executor.timed_launches() as inner:
            assert executor._trace.events is inner
        assert executor._trace.events is evs
    assert executor._trace.events is None
