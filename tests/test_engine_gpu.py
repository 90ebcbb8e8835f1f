"""Device engine: the reference's engine acceptance (tests/test_engine.py,
engine.py:94-215) on the stream-ordered engine, plus a stream-ordering fuzz.

The B200 engine runs every closure at push time; a closure only ENQUEUES
device work on the engine's CUDA stream, so push order is execution order
(stronger than the reference's per-tag FIFO; reader concurrency is moot on
one stream).  What carries over and is tested here: push-order execution,
poison of a failed closure's written tags surfacing as OperationFailed at
the sync point, the no-wait-inside-a-closure rule, push_delete ordered after
pending work and deleted tags rejected, closed engines rejecting work, the
configurable default engine, ``pending``.

Fuzz (fuzz.py:31-112 there): random programs of steps that read and write
subsets of 16 tagged device tensors, each step mixing what it read into
what it writes with device kernels (scalar multiply, elementwise add:
separately rounded fp32, no FMA), against a sequential numpy interpreter of
the same float ops -- bitwise, 300 seeds."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N = 256  # elements per tagged tensor


def test_write_order_is_push_order(engine):
    tag = engine.new_tag("x")
    seen = []
    for i in range(50):
        engine.push(lambda i=i: seen.append(i), writes=[tag])
    engine.wait_for(tag)
    assert seen == list(range(50))


def test_failure_poisons_tag_and_raises_on_wait(engine):
    from paper_1512_01274_b200 import _lib as L
    from paper_1512_01274_b200.errors import OperationFailed
    tag, other = engine.new_tag("x"), engine.new_tag("y")
    engine.push(lambda: 1 / 0, writes=[tag])
    with pytest.raises(OperationFailed):
        engine.wait_for(tag)
    engine.wait_for(other)  # untouched tags stay healthy
    # a native failure (bad argument to a kernel launcher) poisons the same way
    bad = engine.new_tag("bad")
    engine.push(lambda: L.call("mgx_copy", 0, 0, -5, engine.stream_handle), writes=[bad])
    with pytest.raises(OperationFailed):
        engine.wait_for(bad)


def test_wait_inside_closure_is_rejected(engine):
    from paper_1512_01274_b200.errors import StateError
    tag, other = engine.new_tag("x"), engine.new_tag("y")
    failed = []

    def bad():
        try:
            engine.wait_for(tag)
        except StateError:
            failed.append(True)

    engine.push(bad, writes=[other])
    engine.wait_for(other)
    assert failed == [True]


def test_push_delete_runs_after_pending_ops(engine):
    from paper_1512_01274_b200 import tensor as tmod
    from paper_1512_01274_b200.errors import LifecycleError
    tag = engine.new_tag("x")
    log = []
    engine.push(lambda: log.append("op"), writes=[tag])
    engine.push_delete(tag, lambda: log.append("del"))
    engine.wait_all()
    assert log == ["op", "del"]
    with pytest.raises(LifecycleError):
        engine.push(lambda: None, writes=[tag])
    with pytest.raises(LifecycleError):
        engine.push_delete(tag)
    # a released tensor's device work completes before its buffer goes
    t = tmod.from_host((N,), "float32", np.arange(N), engine=engine)
    y = tmod.zeros((N,), engine=engine)
    tmod.axpy(2.0, t, y)
    tmod.release(t)
    np.testing.assert_array_equal(tmod.to_numpy(y), 2 * np.arange(N, dtype=np.float32))


def test_closed_engine_rejects_work(cuda):
    from paper_1512_01274_b200.engine import Engine
    from paper_1512_01274_b200.errors import StateError
    e = Engine(device=0)
    tag = e.new_tag("x")
    e.close()
    with pytest.raises(StateError):
        e.push(lambda: None, writes=[tag])


def test_default_engine_configurable(cuda):
    from paper_1512_01274_b200.engine import configure_default_engine, default_engine
    first = default_engine()
    assert default_engine() is first
    fresh = configure_default_engine(threads=2)
    assert default_engine() is fresh and fresh is not first


def test_pending_counts_outstanding_work(engine):
    from paper_1512_01274_b200 import tensor as tmod
    a = tmod.zeros((1 << 24,), engine=engine)
    for _ in range(8):
        tmod.axpy(1.0, a, a)
    assert engine.pending >= 0
    engine.wait_all()
    assert engine.pending == 0


def _random_program(seed, num_tags=16, num_steps=24):
    """Steps (reads, writes, salt) drawn with the reference's splitmix64
    recipe (fuzz.py:31-45)."""
    from paper_1512_01274_b200.data import splitmix64
    rng = splitmix64(seed)
    steps = []
    for _ in range(num_steps):
        nr, nw = next(rng) % 3, 1 + next(rng) % 2
        cells = list(range(num_tags))
        picks = [cells.pop(next(rng) % len(cells)) for _ in range(nr + nw)]
        steps.append((tuple(sorted(picks[:nr])), tuple(sorted(picks[nr:])),
                      float((next(rng) % 1000) / 997.0)))
    return steps


def _salt_vector(salt):
    return (np.arange(N, dtype=np.float32) * np.float32(0.001) + np.float32(salt)).astype(np.float32)


def _run_sequential(program, init):
    state = [v.copy() for v in init]
    for reads, writes, salt in program:
        val = _salt_vector(salt)
        for t in reads:
            val = (val * np.float32(0.75)).astype(np.float32) + state[t]
        for t in writes:
            state[t] = (state[t] * np.float32(0.5)).astype(np.float32) + val
    return state


def _run_on_engine(engine, program, init):
    from paper_1512_01274_b200 import tensor as tmod
    state = [tmod.from_host((N,), "float32", v, engine=engine) for v in init]
    for reads, writes, salt in program:
        val = tmod.from_host((N,), "float32", _salt_vector(salt), engine=engine)
        for t in reads:
            tmod.scalar_op("mul", val, 0.75, val)
            tmod.elementwise("add", val, state[t], val)
        for t in writes:
            tmod.scalar_op("mul", state[t], 0.5, state[t])
            tmod.elementwise("add", state[t], val, state[t])
    return [tmod.to_numpy(t) for t in state]


def test_fuzzed_programs_match_sequential_interpreter(engine):
    rs = np.random.RandomState(0)
    for seed in range(300):
        init = [rs.randn(N).astype(np.float32) for _ in range(16)]
        program = _random_program(seed)
        want = _run_sequential(program, init)
        got = _run_on_engine(engine, program, init)
        for t in range(16):
            np.testing.assert_array_equal(got[t], want[t], err_msg=f"seed {seed} tag {t}")


def test_rng_write_tag_sequence_stable(cuda):
    from paper_1512_01274_b200.engine import Engine
    sequences = set()
    for _ in range(5):
        e = Engine(device=0)
        rng = np.random.RandomState(3)
        tag = e.new_tag("rng")
        out = []
        for _ in range(64):
            e.push(lambda: out.append(int(rng.randint(0, 1 << 30))), writes=[tag])
        e.wait_all()
        e.close()
        sequences.add(tuple(out))
    assert len(sequences) == 1
