"""Host side of the trainer (paper_2502_06728_b200/trainer.py) against the reference's own
outputs (tests/golden/rng.npz, tests/golden/trainer.npz, written from the reference build by
oracle/gen_golden.py and oracle/gen_trainer_golden.py): the MT19937-64 engine, seed mixing,
the distribution transforms, the datasets, the batch permutation and the initial parameters are
bit-exact; the configuration parser accepts what config.cpp accepts, couples DeMo's knobs the
same way and reports every violation at once.  No GPU needed."""
import hashlib
import os

import numpy as np
import pytest

from tests.trainer_configs import ARMS_08, BLOBS_BASE, C03, RUNS

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def T():
    from paper_2502_06728_b200 import trainer

    return trainer


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLD, "trainer.npz"))


def test_engine_and_seed_mixing(T):
    g = np.load(os.path.join(GOLD, "rng.npz"))
    e = T._MT19937_64(5489)  # std::mt19937_64 default seed
    got = np.array([e() for _ in range(10000)], np.uint64)
    assert np.array_equal(got, g["mt_default"])
    assert g["mt_default"][9999] == np.uint64(9981545732273789042)  # the C++ standard's KAT
    assert [T.mix_seed(1234), T.mix_seed(1234, 7), T.mix_seed(1234, 7, 3), T.mix_seed(99, 5, 2)] == \
        [int(x) for x in g["mix"]]


def test_distribution_transforms(T):
    g = np.load(os.path.join(GOLD, "rng.npz"))
    r = T.Rng(42)
    assert [r.below(int(n)) for n in np.tile(g["below_ns"], 20)] == [int(x) for x in g["below"]]
    for seed, key in ((11, "normal_11"), (1234, "normal_1234")):
        r = T.Rng(seed)
        got = np.array([r.normal() for _ in range(len(g[key]))])
        assert np.array_equal(got, g[key]), f"{key}: Box-Muller draws differ"


@pytest.mark.parametrize("name", sorted(RUNS))
def test_dataset_stream_and_init_bit_exact(T, gold, name):
    cfg = T.parse_config(RUNS[name])
    ds = T.make_dataset(cfg.dataset, cfg.seed)
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    got = {"train_inputs": ds.train.inputs, "val_inputs": ds.val.inputs}
    if ds.train.targets is not None:
        got.update(train_targets=ds.train.targets, val_targets=ds.val.targets, gen_params=ds.gen_params)
    if ds.train.labels is not None:
        got.update(train_labels=ds.train.labels, val_labels=ds.val.labels)
    for k, v in got.items():
        assert sha(v) == str(gold[f"{name}/sha/{k}"]), f"{name}: {k} differs from make_dataset's"
    assert np.array_equal(ds.train.inputs[:4], gold[f"{name}/train_inputs_head"])
    bs = T.BatchStream(ds.train.size, cfg.world_size, cfg.batch_size, cfg.seed)
    pairs = gold[f"{name}/batch_pairs"]
    for i, (s, r) in enumerate(zip(pairs[0], pairs[1])):
        assert np.array_equal(bs.indices_for(int(s), int(r)), gold[f"{name}/batch_indices"][i].astype(np.int64))
    init = T.init_params(cfg.model, cfg.seed, T.padded_param_len(cfg))
    assert np.array_equal(init, gold[f"{name}/init"])


def test_parse_config_values(T):
    cfg = T.parse_config(C03)
    assert (cfg.nodes, cfg.accels_per_node, cfg.mode) == (2, 2, "hybrid_sharded")
    assert cfg.model.kind == "quadratic" and cfg.model.layer_dims == [256]
    r = cfg.replicator
    assert (r.chunk_size, r.top_k, r.compression, r.sign_mode, r.seed) == (32, 4, 4 / 32, True, 2024)
    assert cfg.dataset.input_dim == 256 and cfg.dataset.output_dim == 256
    # DeMo couples compression -> top_k (config.cpp:449-457); fractions parse (:63-84)
    c = T.parse_config(BLOBS_BASE + "replicator.scheme = demo\nreplicator.compression = 1/16\n")
    assert c.replicator.top_k == 2 and c.replicator.compression == 2 / 32
    c = T.parse_config(BLOBS_BASE + ARMS_08["random-1/16"] + "replicator.seed = 9  # comment\n")
    assert c.replicator.compression == 1 / 16 and c.replicator.seed == 9
    c = T.parse_config(BLOBS_BASE + ARMS_08["full"])
    assert c.replicator.compression == 1.0
    assert T.effective_compression(T.parse_config(BLOBS_BASE + ARMS_08["spectral-1/16"])) == 2 / 32


@pytest.mark.parametrize("text,needle", [
    ("steps = 0\n", "steps: expected a positive integer"),
    ("bogus.key = 1\n", "unknown key 'bogus.key'"),
    ("model.kind = mlp\n", "quadratic_target pairs with model.kind = quadratic"),
    ("replicator.top_k = 40\n", "replicator.top_k 40 must lie in [1, chunk_size 32]"),
    ("optimizer.momentum_decay = 1.0\n", "momentum_decay must lie in [0, 1)"),
    ("replicator.scheme = full\nreplicator.compression = 0.5\n", "conflicts with the full scheme"),
    ("batch_size = 100\n", "exceeds the training pool of 160 examples"),
    ("no equals sign\n", "expected 'key = value'"),
    ("warmup_fraction = 1\n", "warmup_fraction must lie in [0, 1)"),
])
def test_parse_config_rejects(T, text, needle):
    from paper_2502_06728_b200.core import ConfigError

    with pytest.raises(ConfigError) as e:
        T.parse_config(C03 + text)
    assert needle in str(e.value)
    assert str(e.value).startswith("invalid configuration:")


def test_every_violation_reported_at_once(T):
    from paper_2502_06728_b200.core import ConfigError

    with pytest.raises(ConfigError) as e:
        T.parse_config(C03 + "steps = -1\noptimizer.learning_rate = 0\nfoo = 1\n")
    msg = str(e.value)
    assert "steps" in msg and "learning_rate must be positive" in msg and "unknown key 'foo'" in msg


def test_shard_geometry_checks(T):
    from paper_2502_06728_b200.core import ConfigError

    base = C03.replace("model.dim = 256", "model.dim = 3").replace("topology.accels_per_node = 2",
                                                                   "topology.accels_per_node = 4")
    with pytest.raises(ConfigError, match="leaves an empty shard"):
        T.parse_config(base.replace("topology.nodes = 2", "topology.nodes = 1"))
    with pytest.raises(ConfigError, match="striding period 8 exceeds the shortest shard"):
        T.parse_config(C03.replace("model.dim = 256", "model.dim = 10") +
                       "replicator.scheme = striding\nreplicator.compression = 1/8\n")
    assert T.padded_param_len(T.parse_config(C03.replace("model.dim = 256", "model.dim = 255"))) == 256


def test_lr_warmup(T):
    cfg = T.parse_config(C03 + "warmup_fraction = 0.01\n")  # round(0.01 * 500) = 5 warmup steps
    assert [T.lr_at(cfg, s) for s in range(7)] == [0.02 * (s + 1) / 5 for s in range(5)] + [0.02, 0.02]
    assert T.lr_at(T.parse_config(C03), 0) == 0.02
