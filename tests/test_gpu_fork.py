"""KVCache object model through the C ABI (lm_core.hpp:35-92): fork / extend / truncate_to /
release_suffix on paged suffixes, against the reference's own KVCache behaviour.

  * prefill(A) -> seal -> fork -> extend(B) logits == the reference's (tests/golden/lm_*.json,
    acceptance.cpp:76-104 / test_lm_core.cpp:130-158), within LOGIT_TOL;
  * extend(B1) then extend(B2) on one fork == extend(B1 ++ B2) (the suffix keys of earlier extends
    are read back through the fork's pages);
  * truncate_to into the prefix -> LogicError, beyond the count -> DomainError (lm_core.cpp:92-99);
    truncate + re-extend reproduces the logits; release_suffix returns the suffix pages;
  * fork of a fork deep-copies the suffix; the sealed segment outlives the handle while forks use it.
"""
import json
import os

import numpy as np
import pytest

from paper_2505_10951_b200 import host

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
LOGIT_TOL = 0.08


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


@pytest.mark.parametrize("name", ["lm_tiny.json", "lm_hd64.json", "lm_hd128.json"])
def test_fork_extend_vs_reference(ctx, name):
    G = gold(name)
    cfg = host.ToyLmConfig(**{**dict(layers=4, heads=4, model_dim=64, ffn_hidden=256, max_seq_len=1024, seed=3),
                              **G["cfg"]})
    lm = host.ToyLm(ctx, cfg)
    cases = [(c, o) for c, o in zip(G["cases"], G["out"]) if o["status"] == 0 and c.get("suffix")]
    kv, _ = lm.prefill_batch([c["prefix"] for c, _ in cases], [c.get("soft") for c, _ in cases])
    forks = [lm.fork(kv, i) for i in range(len(cases))]
    lg = lm.extend_forks(forks, [c["suffix"] for c, _ in cases])
    for j, (c, o) in enumerate(cases):
        err = np.abs(lg[j] - np.asarray(o["ext_logits"], np.float32)).max()
        assert err <= LOGIT_TOL, (j, err)
        assert forks[j].token_count() == len(c["prefix"]) + len(c["suffix"]) + (1 if c.get("soft") else 0)
        assert np.array_equal(forks[j].last_logits, lg[j])
    # the batched member path gives the same rows
    lg2, _ = lm.extend_members(kv, list(range(len(cases))), [c["suffix"] for c, _ in cases])
    assert np.abs(lg2 - lg).max() < 1e-4
    for f in forks:
        f.close()
    kv.release()
    lm.close()


def test_incremental_extend_truncate_release(ctx):
    lm = host.ToyLm(ctx, host.ToyLmConfig(layers=2, heads=2, model_dim=256, ffn_hidden=512, max_seq_len=1024, seed=4))
    rng = np.random.default_rng(3)
    prefix = rng.integers(0, 256, 333).tolist()
    b1, b2 = rng.integers(0, 256, 150).tolist(), rng.integers(0, 256, 70).tolist()  # crosses a page
    kv, _ = lm.prefill_batch([prefix])
    one = lm.fork(kv)
    two = lm.fork(kv)
    lg_one = lm.extend_forks([one], [b1 + b2])[0]
    lm.extend_forks([two], [b1])
    lg_two = lm.extend_forks([two], [b2])[0]
    assert np.abs(lg_two - lg_one).max() < 2e-3          # fp32 reassociation only
    assert int(np.argmax(lg_two)) == int(np.argmax(lg_one))
    # truncate_to (lm_core.cpp:92-99)
    with pytest.raises(host.LogicError):
        two.truncate_to(len(prefix) - 1)
    with pytest.raises(host.DomainError):
        two.truncate_to(two.token_count() + 1)
    two.truncate_to(len(prefix) + len(b1))
    assert two.token_count() == len(prefix) + len(b1)
    lg_again = lm.extend_forks([two], [b2])[0]
    assert np.array_equal(lg_again, lg_two)                 # the same keys are rebuilt
    # fork of a fork: deep copy of the suffix, then the two diverge independently
    three = two.fork()
    assert three.token_count() == two.token_count()
    lg3 = lm.extend_forks([three, two], [[7, 8, 9], [7, 8, 9]])
    assert np.array_equal(lg3[0], lg3[1])
    # release_suffix -> prefix only; the sealed segment outlives the KV handle while forks use it
    one.release_suffix()
    assert one.token_count() == len(prefix)
    kv.release()
    lg_after = lm.extend_forks([one], [b1 + b2])[0]
    assert np.array_equal(lg_after, lg_one)
    for f in (one, two, three):
        f.close()
    lm.close()


def test_fork_capacity(ctx):
    lm = host.ToyLm(ctx, host.ToyLmConfig(max_seq_len=64))
    kv, _ = lm.prefill_batch([[256] + [1] * 40])
    f = lm.fork(kv)
    with pytest.raises(host.CapacityError):
        lm.extend_forks([f], [[2] * 30])
    assert f.token_count() == 41
    lm.extend_forks([f], [[2] * 23])
    assert f.token_count() == 64
    f.close()
    kv.release()
    lm.close()
