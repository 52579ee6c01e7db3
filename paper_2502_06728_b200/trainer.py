"""The reference's experiment layer around the optimizer step, on one GPU: configuration
(config.hpp / config.cpp), the synthetic datasets and their batch stream (dataset.hpp /
dataset.cpp), the toy models (model.hpp / model.cpp) and the training loop (trainer.hpp /
trainer.cpp:24-90), so a reference experiment runs end to end on the device:

  cfg = parse_config(open("exp.cfg").read())      # the reference's key = value format
  result = Trainer(cfg).run()                     # metrics per step, final losses, traffic

Host side, once per run (bit-exact with the reference: the same MT19937-64 stream, the same
splitmix64 seed derivation and distribution transforms, glibc's log / sin / cos through
Python's math module): the dataset pools, the batch permutation and the initial parameters.
They are copied to the device once.

Device side, every step (no host data per step):
  1. every node's parameters are gathered from its members' shards (one copy per node);
  2. ONE launch of the toy producer (csrc/toy_models.cu, dmb_toy_loss_grad) evaluates every
     rank's loss and gradient on its BatchStream batch (FP64 in the reference's operation
     order, from the device-resident pool and permutation);
  3. the cluster step: every rank of the nodes x accels_per_node world is a HybridCluster
     member in this process (LocalHub: the reduce-scatter is the member-order mean, the
     payloads are read in place), so prepare / exchange / merge / apply run the product
     kernels exactly as one process per GPU runs them -- run_step_hybrid, cluster.cpp:171-232;
     ddp_all_gather runs as nodes*accels single-accelerator nodes (run_step_ddp,
     cluster.cpp:234-287, has the same arithmetic) with the reference's traffic accounting;
  4. one synchronization: the refusal latch (a non-finite gradient anywhere refuses the step on
     every member and raises TrainingError, state unchanged) and the rank losses (train loss =
     their sum in rank order / world, trainer.cpp:53-71); the validation loss of worker (0, 0)
     every eval_every steps (trainer.cpp:77-79) is one more launch.

The optimizer state is FP32 on the device where the reference keeps FP64 (the optimizer step's
parity bars are in tests/test_gpu_parity.py); the trainer-level bars against the reference's own
runs are in tests/test_gpu_trainer.py.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np
import torch

from . import _capi
from ._capi import lib
from .cluster import HybridCluster, LocalExchange, LocalHub, StepTraffic, Topology
from .core import (ConfigError, OptimizerConfig, OptimizerKind, ReplicatorConfig, Scheme, StepTrace, TrainingError,
                   TransferDtype, _check, _ptr, _stream, context, status)

MASK64 = (1 << 64) - 1


# ------------------------------------------------------------------ rng.hpp / rng.cpp
def _mix64(z: int) -> int:
    """splitmix64 finalizer (rng.cpp:8-14)"""
    z = (z + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def mix_seed(seed: int, *tags: int) -> int:
    """mix_seed (rng.cpp:17-23): mix64(seed), then mix64(prev ^ tag) per tag"""
    z = _mix64(seed & MASK64)
    for t in tags:
        z = _mix64(z ^ (t & MASK64))
    return z


class _MT19937_64:
    """std::mt19937_64 (the engine rng.hpp:51 pins), the twist vectorized over its three
    dependency-free segments"""
    N, M = 312, 156
    A = np.uint64(0xB5026F5AA96619E9)
    UM, LM = np.uint64(0xFFFFFFFF80000000), np.uint64(0x7FFFFFFF)

    def __init__(self, seed: int):
        mt = [seed & MASK64]
        for i in range(1, self.N):
            p = mt[-1]
            mt.append((6364136223846793005 * (p ^ (p >> 62)) + i) & MASK64)
        self.mt = np.array(mt, dtype=np.uint64)
        self.out: List[int] = []
        self.pos = 0

    def _twist(self):
        mt, N, M = self.mt, self.N, self.M
        one = np.uint64(1)

        def mix(i0, i1, src):
            x = (mt[i0:i1] & self.UM) | (mt[i0 + 1:i1 + 1] & self.LM)
            return src ^ (x >> one) ^ np.where((x & one) != 0, self.A, np.uint64(0))

        mt[0:N - M] = mix(0, N - M, mt[M:N])
        mt[N - M:N - 1] = mix(N - M, N - 1, mt[0:M - 1])
        x = (mt[N - 1] & self.UM) | (mt[0] & self.LM)
        mt[N - 1] = mt[M - 1] ^ (x >> one) ^ (self.A if int(x) & 1 else np.uint64(0))
        y = mt.copy()
        y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
        y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        y ^= y >> np.uint64(43)
        self.out = y.tolist()
        self.pos = 0

    def __call__(self) -> int:
        if self.pos >= len(self.out):
            self._twist()
        v = self.out[self.pos]
        self.pos += 1
        return v


class Rng:
    """Rng (rng.hpp:20-50, rng.cpp:26-52): the engine seeded with mix_seed(seed)."""

    def __init__(self, seed: int):
        self._e = _MT19937_64(mix_seed(seed))
        self._spare: Optional[float] = None

    def next_u64(self) -> int:
        return self._e()

    def uniform(self, lo: float = None, hi: float = None) -> float:
        u = (self._e() >> 11) * 2.0 ** -53
        return u if lo is None else lo + (hi - lo) * u

    def below(self, n: int) -> int:
        """debiased multiply-shift (rng.cpp:26-36)"""
        threshold = ((1 << 64) - n) % n
        while True:
            wide = self._e() * n
            if (wide & MASK64) >= threshold:
                return wide >> 64

    def normal(self, mean: float = None, stddev: float = None) -> float:
        """Box-Muller with the second variate cached (rng.cpp:38-50)"""
        if self._spare is not None:
            z, self._spare = self._spare, None
        else:
            u1 = 1.0 - self.uniform()
            u2 = self.uniform()
            r = math.sqrt(-2.0 * math.log(u1))
            a = 6.283185307179586476925286766559 * u2
            self._spare = r * math.sin(a)
            z = r * math.cos(a)
        return z if mean is None else mean + stddev * z

    def shuffle(self, v: list) -> None:
        """Fisher-Yates driven by below() (rng.hpp:42-48)"""
        for i in range(len(v), 1, -1):
            j = self.below(i)
            v[i - 1], v[j] = v[j], v[i - 1]


# ------------------------------------------------------------------ config.hpp / config.cpp
MODES = ("hybrid_sharded", "ddp_all_gather")


@dataclass
class ModelSpec:
    """Model (model.hpp:36-46)"""
    kind: str = "quadratic"  # quadratic | mlp
    layer_dims: List[int] = field(default_factory=lambda: [2])
    activation: str = "tanh"  # tanh | relu
    loss: str = "mse"  # mse | cross_entropy

    def param_count(self) -> int:
        """model.cpp:121-125"""
        if self.kind == "quadratic":
            return self.layer_dims[0]
        d = self.layer_dims
        return sum(d[i + 1] * d[i] + d[i + 1] for i in range(len(d) - 1))

    @property
    def input_dim(self) -> int:
        return self.layer_dims[0]

    @property
    def output_dim(self) -> int:
        return self.layer_dims[-1]


@dataclass
class DatasetSpec:
    """DatasetSpec (dataset.hpp:24-30)"""
    kind: str = "gaussian_blobs"  # quadratic_target | gaussian_blobs | linear_regression
    size: int = 1000
    input_dim: int = 8
    output_dim: int = 4
    noise: float = 0.0


@dataclass
class LinkModel:
    """LinkModel (cluster.hpp:25-29): bits per second, seconds"""
    intra_node_bandwidth: float = 100e9
    inter_node_bandwidth: float = 10e9
    compute_time_per_step: float = 0.01


@dataclass
class ExperimentConfig:
    """ExperimentConfig (config.hpp:15-30)"""
    nodes: int = 1
    accels_per_node: int = 1
    mode: str = "hybrid_sharded"
    model: ModelSpec = field(default_factory=ModelSpec)
    pad_params: bool = True
    dataset: DatasetSpec = field(default_factory=DatasetSpec)
    optimizer: OptimizerConfig = field(default_factory=OptimizerConfig)
    replicator: ReplicatorConfig = field(default_factory=ReplicatorConfig)
    link: LinkModel = field(default_factory=LinkModel)
    steps: int = 200
    batch_size: int = 8
    eval_every: int = 50
    warmup_fraction: float = 0.0
    seed: int = 1234
    out_dir: str = "demosim-out"
    replicator_seed_set: bool = False

    @property
    def world_size(self) -> int:
        return self.nodes * self.accels_per_node


def _parse_double(v: str) -> Optional[float]:
    """numbers and p/q fractions (config.cpp:63-84)"""
    try:
        if "/" not in v:
            return float(v)
        p, q = v.split("/", 1)
        q = float(q.strip())
        return None if q == 0.0 else float(p.strip()) / q
    except ValueError:
        return None


def _parse_u64(v: str) -> Optional[int]:
    if not v or v[0] == "-" or not v.isdigit():
        return None
    return int(v)


def _parse_bool(v: str) -> Optional[bool]:
    if v in ("true", "on", "1", "yes"):
        return True
    if v in ("false", "off", "0", "no"):
        return False
    return None


class _Issues(list):
    def raise_if_any(self):
        if self:
            raise ConfigError("invalid configuration:" + "".join("\n  - " + m for m in self))


_ENUMS = {
    "topology.mode": ("mode", {m: m for m in MODES}, "hybrid_sharded | ddp_all_gather"),
    "model.kind": ("model.kind", {"quadratic": "quadratic", "mlp": "mlp"}, "quadratic | mlp"),
    "model.activation": ("model.activation", {"tanh": "tanh", "relu": "relu"}, "tanh | relu"),
    "model.loss": ("model.loss", {"mse": "mse", "cross_entropy": "cross_entropy"}, "mse | cross_entropy"),
    "dataset.kind": ("dataset.kind", {k: k for k in ("quadratic_target", "gaussian_blobs", "linear_regression")},
                     "quadratic_target | gaussian_blobs | linear_regression"),
    "optimizer.kind": ("optimizer.kind", {"demo_sgd": OptimizerKind.DemoSgd,
                                          "decoupled_adamw": OptimizerKind.DecoupledAdamW},
                       "demo_sgd | decoupled_adamw"),
    "replicator.scheme": ("replicator.scheme", {"demo": Scheme.DeMo, "random": Scheme.Random,
                                                "striding": Scheme.Striding, "diloco": Scheme.DiLoCo,
                                                "full": Scheme.Full}, "demo | random | striding | diloco | full"),
    "replicator.transfer_dtype": ("replicator.transfer_dtype", {"fp32": TransferDtype.Fp32,
                                                                "fp16": TransferDtype.Fp16,
                                                                "ternary": TransferDtype.Ternary},
                                  "fp32 | fp16 | ternary"),
}
_POSITIVE = {"topology.nodes": "nodes", "topology.accels_per_node": "accels_per_node", "dataset.size": "dataset.size",
             "replicator.chunk_size": "replicator.chunk_size", "steps": "steps", "batch_size": "batch_size",
             "eval_every": "eval_every"}
_DOUBLES = {"optimizer.learning_rate": "optimizer.learning_rate", "optimizer.momentum_decay": "optimizer.momentum_decay",
            "optimizer.adam_beta1": "optimizer.adam_beta1", "optimizer.adam_beta2": "optimizer.adam_beta2",
            "optimizer.adam_eps": "optimizer.adam_eps", "optimizer.weight_decay": "optimizer.weight_decay",
            "link.intra_node_bandwidth": "link.intra_node_bandwidth",
            "link.inter_node_bandwidth": "link.inter_node_bandwidth",
            "link.compute_time_per_step": "link.compute_time_per_step", "warmup_fraction": "warmup_fraction"}


def _set(cfg: ExperimentConfig, path: str, value) -> None:
    obj = cfg
    parts = path.split(".")
    for p in parts[:-1]:
        obj = getattr(obj, p)
    setattr(obj, parts[-1], value)


def _apply_key(cfg: ExperimentConfig, ctx: dict, issues: _Issues, key: str, value: str) -> None:
    """apply_key (config.cpp:140-262)"""
    def bad(what):
        issues.append(f"{key}: expected {what}, got '{value}'")

    if key in _ENUMS:
        path, table, what = _ENUMS[key]
        if value in table:
            _set(cfg, path, table[value])
        else:
            bad(what)
    elif key in _POSITIVE:
        u = _parse_u64(value)
        if u is not None and u >= 1:
            _set(cfg, _POSITIVE[key], u)
        else:
            bad("a positive integer")
    elif key in _DOUBLES:
        d = _parse_double(value)
        if d is not None:
            _set(cfg, _DOUBLES[key], d)
        else:
            bad("a number")
    elif key == "model.dim":
        u = _parse_u64(value)
        if u is not None and u >= 1:
            cfg.model.layer_dims = [u]
        else:
            bad("a positive integer")
    elif key == "model.layer_dims":
        try:
            dims = [_parse_u64(p.strip()) for p in value.split(",")]
        except ValueError:
            dims = [None]
        if len(dims) >= 2 and all(d is not None and d > 0 for d in dims):
            cfg.model.layer_dims = dims
        else:
            bad("a comma list of at least two positive integers")
    elif key == "model.pad_params":
        b = _parse_bool(value)
        if b is None:
            bad("a boolean")
        else:
            cfg.pad_params = b
    elif key == "dataset.noise":
        d = _parse_double(value)
        if d is not None and d >= 0.0:
            cfg.dataset.noise = d
        else:
            bad("a non-negative number")
    elif key == "replicator.top_k":
        u = _parse_u64(value)
        if u is not None and u >= 1:
            cfg.replicator.top_k = u
            ctx["top_k_set"] = True
        else:
            bad("a positive integer")
    elif key == "replicator.compression":
        d = _parse_double(value)
        if d is not None:
            cfg.replicator.compression = d
            ctx["compression_set"] = True
        else:
            bad("a number or fraction")
    elif key == "replicator.sign":
        b = _parse_bool(value)
        if b is None:
            bad("a boolean")
        else:
            cfg.replicator.sign_mode = b
    elif key == "replicator.seed":
        u = _parse_u64(value)
        if u is None:
            bad("an unsigned integer")
        else:
            cfg.replicator.seed = u
            cfg.replicator_seed_set = True
    elif key == "seed":
        u = _parse_u64(value)
        if u is None:
            bad("an unsigned integer")
        else:
            cfg.seed = u
    elif key == "out_dir":
        cfg.out_dir = value
    else:
        issues.append(f"unknown key '{key}'")


def padded_param_len(cfg: ExperimentConfig) -> int:
    """config.cpp:264-270"""
    n = cfg.model.param_count()
    shards = cfg.accels_per_node if cfg.mode == "hybrid_sharded" else 1
    return n if n % shards == 0 else n + shards - n % shards


def effective_compression(cfg: ExperimentConfig) -> float:
    """config.cpp:272-283"""
    r = cfg.replicator
    if r.scheme == Scheme.DeMo:
        return r.top_k / r.chunk_size
    if r.scheme == Scheme.Full:
        return 1.0
    return r.compression


def _collect_violations(cfg: ExperimentConfig, issues: _Issues) -> None:
    """collect_violations (config.cpp:288-398)"""
    m = cfg.model
    if m.kind == "mlp" and len(m.layer_dims) < 2:
        issues.append("model.layer_dims: an mlp needs at least input and output dims")
    if m.kind == "quadratic" and len(m.layer_dims) != 1:
        issues.append("model.dim: a quadratic model takes a single dimension")
    o = cfg.optimizer
    if not o.learning_rate > 0.0:
        issues.append("optimizer.learning_rate must be positive")
    if not (0.0 <= o.momentum_decay < 1.0):
        issues.append("optimizer.momentum_decay must lie in [0, 1)")
    if not (0.0 <= o.adam_beta1 < 1.0):
        issues.append("optimizer.adam_beta1 must lie in [0, 1)")
    if not (0.0 <= o.adam_beta2 < 1.0):
        issues.append("optimizer.adam_beta2 must lie in [0, 1)")
    if not o.adam_eps > 0.0:
        issues.append("optimizer.adam_eps must be positive")
    if not o.weight_decay >= 0.0:
        issues.append("optimizer.weight_decay must be non-negative")
    r = cfg.replicator
    if not (0.0 < r.compression <= 1.0):
        issues.append(f"replicator.compression {r.compression:g} must lie in (0, 1]")
    if r.scheme == Scheme.DeMo:
        if r.chunk_size == 0:
            issues.append("replicator.chunk_size must be positive")
        if r.top_k == 0 or r.top_k > r.chunk_size:
            issues.append(f"replicator.top_k {r.top_k} must lie in [1, chunk_size {r.chunk_size}]")
    if r.scheme == Scheme.Full and r.compression != 1.0:
        issues.append(f"replicator.compression {r.compression:g} conflicts with the full scheme")
    if not cfg.replicator_seed_set:
        r.seed = cfg.seed
    L = cfg.link
    if not L.intra_node_bandwidth > 0.0:
        issues.append("link.intra_node_bandwidth must be positive")
    if not L.inter_node_bandwidth > 0.0:
        issues.append("link.inter_node_bandwidth must be positive")
    if not L.compute_time_per_step > 0.0:
        issues.append("link.compute_time_per_step must be positive")
    if not (0.0 <= cfg.warmup_fraction < 1.0):
        issues.append("warmup_fraction must lie in [0, 1)")
    if cfg.dataset.size < 10:
        issues.append("dataset.size must be at least 10")
    cfg.dataset.input_dim = m.input_dim
    cfg.dataset.output_dim = m.output_dim
    dk = cfg.dataset.kind
    if m.kind == "quadratic" and dk != "quadratic_target":
        issues.append("a quadratic model pairs with dataset.kind = quadratic_target")
    if m.kind == "mlp" and dk == "quadratic_target":
        issues.append("dataset.kind = quadratic_target pairs with model.kind = quadratic")
    if m.loss == "cross_entropy" and m.kind == "mlp" and dk != "gaussian_blobs":
        issues.append("cross entropy training needs dataset.kind = gaussian_blobs")
    if dk == "gaussian_blobs" and m.kind == "mlp" and m.loss != "cross_entropy":
        issues.append("gaussian_blobs is a labeled dataset; set model.loss = cross_entropy")
    world = cfg.world_size
    train_size = cfg.dataset.size * 8 // 10
    if world * cfg.batch_size > train_size:
        issues.append(f"global batch ({world} ranks x {cfg.batch_size}) exceeds the training pool of "
                      f"{train_size} examples")
    pc = m.param_count()
    shards = cfg.accels_per_node if cfg.mode == "hybrid_sharded" else 1
    if pc % shards != 0 and not cfg.pad_params:
        issues.append(f"param_count {pc} is not divisible by accels_per_node {shards} and padding is off")
    if not issues:
        extent = padded_param_len(cfg) // shards
        min_real = min(0 if s * extent >= pc else min(extent, pc - s * extent) for s in range(shards))
        if min_real == 0:
            issues.append(f"param_count {pc} leaves an empty shard across {shards} accelerators")
        elif r.scheme in (Scheme.Random, Scheme.Striding):
            if round(r.compression * min_real) < 1:
                issues.append(f"replicator.compression {r.compression:g} selects nothing from a shard of "
                              f"{min_real} values")
            if r.scheme == Scheme.Striding and r.period() > min_real:
                issues.append(f"striding period {r.period()} exceeds the shortest shard "
                              f"({min_real} values)")


def validate_config(cfg: ExperimentConfig) -> None:
    """validate_config (config.cpp:402-406)"""
    issues = _Issues()
    _collect_violations(cfg, issues)
    issues.raise_if_any()


def parse_config(text: str) -> ExperimentConfig:
    """parse_config (config.cpp:408-462): `key = value` lines, '#' comments; DeMo couples
    top_k and compression; every problem is reported at once as a ConfigError."""
    cfg = ExperimentConfig()
    issues = _Issues()
    ctx = dict(compression_set=False, top_k_set=False)
    for lineno, raw in enumerate(text.split("\n"), 1):
        line = raw.strip(" \t\r")
        if "#" in line:
            line = line[:line.index("#")].strip(" \t\r")
        if not line:
            continue
        if "=" not in line:
            issues.append(f"line {lineno}: expected 'key = value', got '{line}'")
            continue
        key, value = (t.strip(" \t\r") for t in line.split("=", 1))
        if not key or not value:
            issues.append(f"line {lineno}: empty key or value")
            continue
        _apply_key(cfg, ctx, issues, key, value)
    r = cfg.replicator
    if r.scheme == Scheme.DeMo:
        if ctx["compression_set"] and not ctx["top_k_set"]:
            k = _llround(r.compression * r.chunk_size)
            r.top_k = min(max(k, 1), r.chunk_size)
        r.compression = r.top_k / r.chunk_size
    elif r.scheme == Scheme.Full and not ctx["compression_set"]:
        r.compression = 1.0
    _collect_violations(cfg, issues)
    issues.raise_if_any()
    return cfg


def load_config(path: str) -> ExperimentConfig:
    """load_config (config.cpp:464-471)"""
    try:
        with open(path, "rb") as f:
            text = f.read().decode()
    except OSError:
        raise ConfigError(f"cannot open config file: {path}") from None
    return parse_config(text)


def _llround(x: float) -> int:
    """std::llround: half away from zero"""
    return int(math.floor(abs(x) + 0.5)) * (1 if x >= 0 else -1)


def lr_at(cfg: ExperimentConfig, step: int) -> float:
    """lr_at (trainer.cpp:24-30): linear warmup over round(warmup_fraction * steps) steps"""
    base = cfg.optimizer.learning_rate
    warm = _llround(cfg.warmup_fraction * cfg.steps)
    if warm == 0 or step >= warm:
        return base
    return base * (step + 1) / warm


# ------------------------------------------------------------------ dataset.hpp / dataset.cpp
@dataclass
class Batch:
    """Batch (model.hpp:18-25): inputs size x input_dim (FP64), targets size x target_dim,
    labels size"""
    inputs: np.ndarray
    targets: Optional[np.ndarray] = None
    labels: Optional[np.ndarray] = None

    @property
    def size(self) -> int:
        return self.inputs.shape[0]


@dataclass
class Dataset:
    """Dataset (dataset.hpp:15-22)"""
    kind: str
    train: Batch
    val: Batch
    gen_params: np.ndarray


def make_dataset(spec: DatasetSpec, seed: int) -> Dataset:
    """make_dataset (dataset.cpp:34-120): the same draws in the same order, 80/20 split."""
    if spec.size < 10:
        raise ConfigError("dataset size must be at least 10")
    if spec.input_dim == 0 or spec.output_dim == 0:
        raise ConfigError("dataset dimensions must be positive")
    rng = Rng(mix_seed(seed, 0x64617461))
    n, din, dout = spec.size, spec.input_dim, spec.output_dim
    targets = labels = None
    gen = np.zeros(0)
    if spec.kind == "quadratic_target":
        center = [rng.uniform(-2.0, 2.0) for _ in range(din)]
        inputs = np.array([[center[d] + 0.5 * rng.normal() for d in range(din)] for _ in range(n)])
    elif spec.kind == "gaussian_blobs":
        means = [rng.uniform(-3.0, 3.0) for _ in range(dout * din)]
        inputs = np.empty((n, din))
        labels = np.empty(n, dtype=np.int32)
        for i in range(n):
            c = i % dout
            labels[i] = c
            for d in range(din):
                inputs[i, d] = means[c * din + d] + rng.normal()
    elif spec.kind == "linear_regression":
        gen = np.array([rng.uniform(-1.0, 1.0) for _ in range(dout * din + dout)])
        W, b = gen[:dout * din].tolist(), gen[dout * din:].tolist()
        inputs = np.empty((n, din))
        targets = np.empty((n, dout))
        for i in range(n):
            x = [rng.normal() for _ in range(din)]
            inputs[i] = x
            for r in range(dout):
                y = b[r]
                for d in range(din):
                    y += W[r * din + d] * x[d]
                if spec.noise > 0.0:
                    y += spec.noise * rng.normal()
                targets[i, r] = y
    else:
        raise ConfigError(f"unknown dataset kind {spec.kind!r}")
    if inputs.ndim == 1:
        inputs = inputs.reshape(n, din)
    t = n * 8 // 10

    def part(lo, hi):
        return Batch(inputs[lo:hi].copy(), None if targets is None else targets[lo:hi].copy(),
                     None if labels is None else labels[lo:hi].copy())

    return Dataset(spec.kind, part(0, t), part(t, n), gen)


class BatchStream:
    """BatchStream (dataset.hpp:40-58, dataset.cpp:122-157): one seeded permutation of the
    training pool, consumed in rank-major windows."""

    def __init__(self, train_size: int, world: int, batch: int, seed: int):
        if train_size == 0 or world == 0 or batch == 0:
            raise ConfigError("batch stream needs a nonempty pool, world and batch size")
        if world * batch > train_size:
            raise ConfigError(f"global batch {world} x {batch} exceeds the training pool of {train_size} examples")
        self.world, self.batch = world, batch
        order = list(range(train_size))
        Rng(mix_seed(seed, 0x626174636865)).shuffle(order)
        self.order = np.array(order, dtype=np.int64)

    def indices_for(self, step: int, rank: int) -> np.ndarray:
        n = len(self.order)
        base = (step * self.world + rank) * self.batch
        return self.order[[(base + j) % n for j in range(self.batch)]]


def init_params(model: ModelSpec, seed: int, padded_len: int) -> np.ndarray:
    """init_params (model.cpp:224-244): zeros for the quadratic bowl, U(+-1/sqrt(in)) per layer"""
    n = model.param_count()
    if padded_len < n:
        raise ConfigError("padded parameter length shorter than the model")
    p = np.zeros(padded_len)
    if model.kind == "quadratic":
        return p
    rng = Rng(mix_seed(seed, 0x6D6F64656C))
    off = 0
    d = model.layer_dims
    for i in range(len(d) - 1):
        bound = 1.0 / math.sqrt(d[i])
        cnt = d[i + 1] * d[i] + d[i + 1]
        p[off:off + cnt] = [rng.uniform(-bound, bound) for _ in range(cnt)]
        off += cnt
    return p


# ------------------------------------------------------------------ device producers
def _toy_model(m: ModelSpec) -> _capi.ToyModel:
    t = _capi.ToyModel()
    t.kind = 0 if m.kind == "quadratic" else 1
    t.activation = 0 if m.activation == "tanh" else 1
    t.loss = 0 if m.loss == "mse" else 1
    if len(m.layer_dims) > 9:
        raise ConfigError("the device producer takes at most 8 layers")
    t.n_dims = len(m.layer_dims)
    for i, d in enumerate(m.layer_dims):
        t.dims[i] = d
    return t


class DevicePool:
    """a dataset split resident on the device (dmb_toy_pool)"""

    def __init__(self, b: Batch, device):
        self.inputs = torch.from_numpy(np.ascontiguousarray(b.inputs, np.float64)).to(device)
        self.targets = None if b.targets is None else torch.from_numpy(np.ascontiguousarray(b.targets)).to(device)
        self.labels = None if b.labels is None else torch.from_numpy(np.ascontiguousarray(b.labels, np.int32)).to(device)
        self.c = _capi.ToyPool(self.inputs.data_ptr(), _ptr(self.targets), _ptr(self.labels), b.size)


def loss_and_gradient(model: ModelSpec, params: torch.Tensor, pool: DevicePool, order: torch.Tensor, step: int,
                      batch: int, workers: int, workers_per_row: int = 1, grad: torch.Tensor = None,
                      loss: torch.Tensor = None):
    """loss_and_gradient (model.cpp:138-203) for `workers` ranks at once: params is (rows,
    padded) FP32, rank w reads row w // workers_per_row; returns (grad (workers, padded) FP32,
    loss (workers,) FP64), both on the device."""
    rows, padded = params.shape
    dev = params.device
    grad = torch.empty(workers, padded, dtype=torch.float32, device=dev) if grad is None else grad
    loss = torch.empty(workers, dtype=torch.float64, device=dev) if loss is None else loss
    tm = _toy_model(model)
    _check(lib.dmb_toy_loss_grad(context(dev).h, C.byref(tm), C.byref(pool.c), _ptr(order), step, batch,
                                 _ptr(params), padded, workers_per_row, workers, _ptr(grad), padded, _ptr(loss),
                                 _stream(params)))
    return grad, loss


def forward_loss(model: ModelSpec, params: torch.Tensor, pool: DevicePool, out: torch.Tensor = None) -> torch.Tensor:
    """forward_loss (model.cpp:127-136) over the whole pool; a device FP64 scalar"""
    out = torch.empty(1, dtype=torch.float64, device=params.device) if out is None else out
    tm = _toy_model(model)
    _check(lib.dmb_toy_loss(context(params.device).h, C.byref(tm), C.byref(pool.c), _ptr(params), _ptr(out),
                            _stream(params)))
    return out


# ------------------------------------------------------------------ trainer.hpp / trainer.cpp
@dataclass
class StepMetrics:
    """StepMetrics (trainer.hpp:17-25); inter_bytes are the reference wire format's bytes,
    inter_bytes_exchanged what the device exchange layout moved (MASK where it applies)"""
    step: int
    train_loss: float
    val_loss: Optional[float] = None
    intra_bytes: int = 0
    inter_bytes: int = 0
    inter_bytes_exchanged: int = 0
    sim_time_s: float = 0.0


@dataclass
class RunResult:
    """RunResult (trainer.hpp:27-38)"""
    metrics: List[StepMetrics] = field(default_factory=list)
    steps_completed: int = 0
    final_train_loss: float = 0.0
    final_val_loss: float = 0.0
    total_intra_bytes: int = 0
    total_inter_bytes: int = 0
    total_sim_time_s: float = 0.0


TraceSink = Callable[[int, int, StepTrace], None]


class Trainer:
    """Trainer (trainer.hpp:40-62, trainer.cpp:32-90) with the cluster on one GPU (module
    docstring).  `wire` is the exchange layout of the DeMo payloads ("mask" where the
    tensor-core encoders apply, else the reference body)."""

    def __init__(self, cfg: ExperimentConfig, device=None, wire: str = "mask", buckets: int = 1,
                 trace: bool = False):
        validate_config(cfg)
        self.cfg = cfg
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.dataset = make_dataset(cfg.dataset, cfg.seed)
        self.padded = padded_param_len(cfg)
        self.param_count = cfg.model.param_count()
        init = init_params(cfg.model, cfg.seed, self.padded)
        self.stream = BatchStream(self.dataset.train.size, cfg.world_size, cfg.batch_size, cfg.seed)
        dev = self.device
        self.train_pool = DevicePool(self.dataset.train, dev)
        self.val_pool = DevicePool(self.dataset.val, dev)
        self.order = torch.from_numpy(self.stream.order).to(dev)
        ddp = cfg.mode == "ddp_all_gather"
        # ddp_all_gather: every rank a single-accelerator node of its own (run_step_ddp has
        # run_step_hybrid's arithmetic at accels_per_node = 1: prepare of the whole vector with
        # shard id 0, merge over the world in rank order)
        self.topo = Topology(cfg.world_size, 1) if ddp else Topology(cfg.nodes, cfg.accels_per_node)
        self.hub = LocalHub(self.topo)
        p0 = torch.from_numpy(init.astype(np.float32)).to(dev)
        self.members = [HybridCluster(self.topo, self.param_count, cfg.optimizer, cfg.replicator, p0, r,
                                      buckets=buckets, wire="reference" if trace else wire,
                                      exchange=LocalExchange(self.hub, r), trace=trace)
                        for r in range(cfg.world_size)]
        self.node_params = torch.zeros(self.topo.nodes, self.padded, dtype=torch.float32, device=dev)
        self.grads = torch.empty(cfg.world_size, self.padded, dtype=torch.float32, device=dev)
        self.losses = torch.empty(cfg.world_size, dtype=torch.float64, device=dev)
        self.val = torch.empty(1, dtype=torch.float64, device=dev)
        self._sim_time = 0.0
        self._gather()

    # worker_params (cluster.hpp:114): node j's parameters, gathered from its members' shards
    def _gather(self) -> None:
        A = self.topo.accels_per_node
        for j in range(self.topo.nodes):
            parts = [self.members[j * A + a].params for a in range(A)]
            torch.cat(parts, out=self.node_params[j, :self.param_count])

    def worker_params(self, node: int, accel: int = 0) -> torch.Tensor:
        """the parameters worker (node, accel) trains on (FP32, padded length)"""
        row = node * self.cfg.accels_per_node + accel if self.cfg.mode == "ddp_all_gather" else node
        return self.node_params[row]

    def eval_loss(self, params: torch.Tensor) -> float:
        """trainer.cpp:44-46: forward loss on the validation split"""
        return float(forward_loss(self.cfg.model, params, self.val_pool, self.val).item())

    def _traffic(self, trs: List[StepTraffic]) -> StepMetrics:
        """the step's TrafficLedger entry (cluster.cpp:63-91, :210-213, :262-265)"""
        cfg, A = self.cfg, self.cfg.accels_per_node
        m = StepMetrics(step=trs[0].step, train_loss=0.0)
        if cfg.mode == "ddp_all_gather":
            world = cfg.world_size
            for t in trs:
                per = t.inter_bytes_reference // (world - 1) if world > 1 else 0
                per_x = t.inter_bytes // (world - 1) if world > 1 else 0
                m.inter_bytes += per * (cfg.nodes - 1)
                m.intra_bytes += per * (A - 1)
                m.inter_bytes_exchanged += per_x * (cfg.nodes - 1)
        else:
            m.intra_bytes = sum(trs[j * A].intra_bytes for j in range(cfg.nodes))
            m.inter_bytes = sum(t.inter_bytes_reference for t in trs)
            m.inter_bytes_exchanged = sum(t.inter_bytes for t in trs)
        L = cfg.link
        self._sim_time += (L.compute_time_per_step + m.intra_bytes * 8.0 / L.intra_node_bandwidth
                           + m.inter_bytes * 8.0 / L.inter_node_bandwidth)  # step_time, cluster.cpp:10-14
        m.sim_time_s = self._sim_time
        return m

    def run_step(self, step: int, trace: Optional[TraceSink] = None) -> StepMetrics:
        """one training step (trainer.cpp:51-75); raises TrainingError on a refused step
        (state unchanged) or a non-finite loss"""
        cfg = self.cfg
        world = cfg.world_size
        loss_and_gradient(cfg.model, self.node_params, self.train_pool, self.order, step, cfg.batch_size, world,
                          self.topo.accels_per_node if cfg.mode == "hybrid_sharded" else 1, self.grads,
                          self.losses)
        for r in range(world):
            self.hub.grads[r] = self.grads[r]
        lr = lr_at(cfg, step)
        for m in self.members:
            m.begin(step, lr, self.grads[m.rank], trace=trace)
        self.hub.agree()
        trs = [m.commit(check=False) for m in self.members]
        losses = self.losses.cpu()  # synchronizes: the refusal latch is read next
        try:
            status(self.device)
        except TrainingError:
            for m in self.members:  # every member back to the state before the step
                m._swap()
                m.steps = m._steps0
            raise
        self._gather()
        train = 0.0
        for v in losses.tolist():  # loss_sum in grad_fn call order (rank order), trainer.cpp:58
            train += v
        train /= world
        if not math.isfinite(train):
            raise TrainingError(f"training diverged at step {step} (loss {train:g})")
        met = self._traffic(trs)
        met.train_loss = train
        if (step + 1) % cfg.eval_every == 0 or step + 1 == cfg.steps:
            met.val_loss = self.eval_loss(self.worker_params(0, 0))
        return met

    def run(self, trace: Optional[TraceSink] = None, out: Optional[RunResult] = None) -> RunResult:
        """Trainer::run (trainer.cpp:49-90); a TrainingError propagates with `out` holding the
        completed steps"""
        out = RunResult() if out is None else out
        for step in range(out.steps_completed, self.cfg.steps):
            m = self.run_step(step, trace)
            out.metrics.append(m)
            out.steps_completed = step + 1
            out.final_train_loss = m.train_loss
            if m.val_loss is not None:
                out.final_val_loss = m.val_loss
            out.total_intra_bytes += m.intra_bytes
            out.total_inter_bytes += m.inter_bytes
            out.total_sim_time_s = m.sim_time_s
        return out


def run_experiment(cfg: ExperimentConfig, **kw) -> RunResult:
    """run_experiment (trainer.cpp:92-97)"""
    return Trainer(cfg, **kw).run()
