"""Concurrent host calls on ONE executor (include/maddness.h: an executor's
staging slots are per handle, so its host calls serialise on an internal
lock). Without the lock two threads' chunks interleave on the same slots and
one call's kernel reads the other's rows. ctypes releases the GIL during the
call, so the threads really overlap; every output must equal the oracle's."""
import threading

import numpy as np
import pytest

import oracle as O
from datagen.synth import make_config_data
from helpers import model_bytes
from test_gpu_parity import _assert_out

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_one_executor_many_threads():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2106_10860_b200 as mdn
    blob = model_bytes("cls10_c16")
    om = O.read_model(blob)
    _, A, B = make_config_data("cls10_c16", n_test=6000)
    model = mdn.mdn_model_load(blob, 0)
    luts = mdn.mdn_build_luts(model, B, mdn.MDN_SUM_EXACT)
    ol = O.make_luts(om, B, "exact", 16)
    ex = mdn.mdn_exec_create(model, luts, chunk_rows=257, n_slots=2)   # many small chunks
    n_threads = 4
    # each thread its own rows (different row order) and its own outputs
    rng = np.random.default_rng(0)
    inputs = [np.ascontiguousarray(A[rng.permutation(A.shape[0])]) for _ in range(n_threads)]
    hosts = [torch.from_numpy(a).pin_memory() for a in inputs]
    outs = [torch.empty((a.shape[0], B.shape[1])).pin_memory() for a in inputs]
    errors = []

    def work(i):
        try:
            for _ in range(3):
                mdn.mdn_amm_host(ex, hosts[i], outs[i])
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    threads = [threading.Thread(target=work, args=(i,)) for i in range(n_threads)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for a, o in zip(inputs, outs):
        _assert_out(o.numpy(), O.amm(a, om, ol)[2])
    ex.close()
