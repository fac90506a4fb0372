"""Multi-tenant pool (epoch admission, Sec. 3.6 / Alg. A2) on the GPU: rates equal the oracle's
epoch admission, paced fetches deliver the right bytes, finished requests free their bandwidth only
at the next epoch, and small payloads (W < Theta, Eq. 2) bypass the pool chunkwise."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2605_22850_b200 as oc  # noqa: E402
from oracle import scheduler as osch  # noqa: E402
from oracle.geometry import Layout as OLayout, chunk_layer_bytes  # noqa: E402
from scenario import lib_target, make_dest, oracle_result, payload_stack, requests_family, sentinel_buffer  # noqa: E402

pytestmark = pytest.mark.gpu


def make_requests(lay, st, specs):
    out = []
    for seed, n in specs:
        req = requests_family(lay, seed, 0, [n])[0]
        keys = oc.chunk_keys(req.tokens, lay.chunk_tokens)
        st.put_chunks(keys, payload_stack(lay, seed, req.payload_ids))
        dest = make_dest(lay, n, "nhd", Bs=16, seed=seed)
        buf = sentinel_buffer(dest.size)
        d = oc.build_descriptor(st, keys, lay, lib_target(oc, dest, buf.data_ptr()))
        out.append({"seed": seed, "req": req, "dest": dest, "buf": buf, "d": d, "s": n * chunk_layer_bytes(lay),
                    "stream": torch.cuda.Stream()})
    return out


@pytest.mark.parametrize("dispatch", [oc.DISPATCH_INDEPENDENT, oc.DISPATCH_WDRR])
def test_pool_epochs_rates_and_bytes(dispatch):
    lay = OLayout(4, 2, 64, 2, 16)
    S = chunk_layer_bytes(lay)
    with oc.Store(lay, capacity=64) as st:
        rs = make_requests(lay, st, [(1, 8), (2, 16), (3, 4)])
        c = [2e-3, 1e-3, 3e-3]                                        # compute windows (s/layer)
        cap = 0.6 * sum(r["s"] / ci for r, ci in zip(rs, c))         # oversubscribed: rates are cut
        pool = oc.TenantPool("stall_opt", cap, dispatch=dispatch)
        t0 = pool.submit(rs[0]["d"], c[0], rs[0]["stream"])
        t1 = pool.submit(rs[1]["d"], c[1], rs[1]["stream"])
        assert pool.status(t0)[0] == oc.TENANT_WAITING
        assert pool.epoch() == 2
        got = [pool.status(t)[1] for t in (t0, t1)]
        want = osch.epoch_admission("stall_opt", [], [rs[0]["s"], rs[1]["s"]], c[:2], cap)
        assert np.allclose(got, want, rtol=1e-12)
        assert pool.status(t0)[0] == oc.TENANT_RUNNING
        # a third request arriving while both run shares only the budget they leave
        t2 = pool.submit(rs[2]["d"], c[2], rs[2]["stream"])
        left = cap - sum(got)
        n = pool.epoch()
        if left > 0:
            assert n == 1
            want2 = osch.epoch_admission("stall_opt", got, [rs[2]["s"]], [c[2]], cap)
            assert np.isclose(pool.status(t2)[1], want2[0], rtol=1e-12)
        torch.cuda.synchronize()
        pool.epoch()                                                  # reaps the finished fetches
        for t in (t0, t1):
            assert pool.status(t)[0] == oc.TENANT_DONE
        for r in rs:
            r["d"].sync_layer(lay.num_layers - 1)
            assert np.array_equal(r["buf"].cpu().numpy(), oracle_result(lay, r["seed"], r["req"], r["dest"]))
        pool.close()
        for r in rs:
            r["d"].close()
    assert S > 0


def test_pool_chunkwise_bypass():
    lay = OLayout(2, 2, 64, 2, 16)
    with oc.Store(lay, capacity=16) as st:
        rs = make_requests(lay, st, [(5, 2), (6, 6)])
        W_small = 2 * lay.num_layers * chunk_layer_bytes(lay)
        pool = oc.TenantPool("equal", 1e9, 0.0, theta_bytes=W_small + 1)   # the 2-chunk request is below Theta
        ts = pool.submit(rs[0]["d"], 1e-3, rs[0]["stream"])
        tl = pool.submit(rs[1]["d"], 1e-3, rs[1]["stream"])
        assert pool.status(ts)[0] == oc.TENANT_CHUNKWISE and pool.status(tl)[0] == oc.TENANT_WAITING
        assert pool.epoch() == 1 and pool.status(tl) == (oc.TENANT_RUNNING, pytest.approx(1e9))
        torch.cuda.synchronize()
        for r in rs:
            r["d"].sync_layer(1)
            assert np.array_equal(r["buf"].cpu().numpy(), oracle_result(lay, r["seed"], r["req"], r["dest"]))
        pool.close()
        for r in rs:
            r["d"].close()


def test_pool_errors():
    with pytest.raises(oc.ObjcacheError):
        oc.TenantPool("equal", 0.0)
    with pytest.raises(oc.ObjcacheError):
        oc.TenantPool("equal", 1e9, -1.0)
    pool = oc.TenantPool("equal", 1e9)
    assert oc._lib.oc_pool_set_dispatch(pool._h, 7) == oc.OC_EINVAL
    with pytest.raises(oc.ObjcacheError) as e:
        pool.status(3)
    assert e.value.code == oc.OC_ERANGE
    assert pool.epoch() == 0
    pool.close()
