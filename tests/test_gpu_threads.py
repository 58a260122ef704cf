"""Threading contract: an operator's device handle is immutable and shareable
across host threads; every call is stream-ordered on the caller's current stream and the shared
workspace is guarded (DeviceOperator.exclusive). Several host threads hammer one cached operator
-- applications, adjoints and projected solves, on the default stream and on private streams --
and every result must equal the single-threaded one bit for bit."""

import threading

import numpy as np
import pytest

from conftest import cuda_ok, random_psf

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_concurrent_calls_on_one_operator(dtype):
    import torch

    import paper_1901_00913_b200 as kb
    from paper_1901_00913_b200.device import device_operator

    rng = np.random.default_rng(7)
    m = 384
    op = kb.decompose(random_psf(rng, 33), kb.BoundaryCondition.REFLECTIVE, s=4, shape=(m, m))
    Xs = [rng.random((m, m)) for _ in range(4)]
    B = kb.kron_apply(op, Xs[0], dtype=dtype)
    cfg = kb.SolveConfig(lam=0.02, lipschitz=2.0, max_iter=15, record_history=False)
    opts = kb.SolveOptions(dtype=dtype, project=True)
    dev = device_operator(op, dtype)

    def work(i):
        if i % 3 == 0:
            return kb.kron_apply(op, Xs[i % 4], dtype=dtype)
        if i % 3 == 1:
            return kb.kron_apply_adjoint(op, Xs[i % 4], dtype=dtype)
        return kb.sfista(op, B, cfg, options=opts).x

    want = [work(i) for i in range(12)]
    got = [None] * 12
    errors = []

    def runner(ids, private_stream):
        try:
            stream = torch.cuda.Stream() if private_stream else None
            for i in ids:
                if stream is None:
                    got[i] = work(i)
                else:
                    with torch.cuda.stream(stream):
                        got[i] = work(i)
        except Exception as ex:  # pragma: no cover - reported below
            errors.append(ex)

    threads = [threading.Thread(target=runner, args=(list(range(t, 12, 4)), t % 2 == 1)) for t in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for i in range(12):
        assert np.array_equal(got[i], want[i]), i
    assert dev is device_operator(op, dtype)  # one cached handle served every thread
