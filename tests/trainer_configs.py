"""Experiment configurations of the trainer fixtures (tests/golden/trainer.npz, written by
oracle/gen_trainer_golden.py from the reference's own run) and the trainer tests.

The acceptance configurations are the reference's, verbatim (acceptance_test.cpp:164-183 (03),
:216-231 (04a), :256-272 (04b), :306-320 (04c), :498-537 (08)); the `extra_*` ones cover what
those leave out: the relu MLP with MSE on linear_regression under decoupled AdamW with warmup,
the ddp_all_gather mode, and the fp16 / ternary wires.
"""

C03 = """
topology.nodes = 2
topology.accels_per_node = 2
model.kind = quadratic
model.dim = 256
dataset.kind = quadratic_target
dataset.size = 200
optimizer.kind = demo_sgd
optimizer.learning_rate = 0.02
replicator.scheme = demo
replicator.chunk_size = 32
replicator.top_k = 4
replicator.sign = on
steps = 500
batch_size = 8
eval_every = 100
seed = 2024
"""

C04A = """
topology.nodes = 1
topology.accels_per_node = 1
model.kind = quadratic
model.dim = 64
dataset.kind = quadratic_target
dataset.size = 400
optimizer.kind = demo_sgd
optimizer.learning_rate = 0.05
replicator.scheme = full
replicator.sign = off
steps = 300
batch_size = 16
eval_every = 100
seed = 91
"""

C04B = """
topology.nodes = 2
topology.accels_per_node = 2
model.kind = quadratic
model.dim = 256
dataset.kind = quadratic_target
dataset.size = 200
optimizer.kind = demo_sgd
optimizer.learning_rate = 0.03
replicator.scheme = demo
replicator.chunk_size = 32
replicator.top_k = 32
replicator.sign = off
steps = 200
batch_size = 8
eval_every = 100
seed = 77
"""
C04B_FULL = C04B + "replicator.scheme = full\n"

C04C_TMPL = """
topology.accels_per_node = 1
model.kind = quadratic
model.dim = 64
dataset.kind = quadratic_target
dataset.size = 400
optimizer.kind = demo_sgd
optimizer.learning_rate = 0.05
replicator.scheme = full
replicator.sign = off
steps = 200
eval_every = 100
seed = 19
"""
C04C_TWO = C04C_TMPL + "topology.nodes = 2\nbatch_size = 8\n"
C04C_ONE = C04C_TMPL + "topology.nodes = 1\nbatch_size = 16\n"

BLOBS_BASE = """
topology.nodes = 2
topology.accels_per_node = 2
model.kind = mlp
model.layer_dims = 2,16,8
model.loss = cross_entropy
model.activation = tanh
dataset.kind = gaussian_blobs
dataset.size = 1000
optimizer.kind = demo_sgd
optimizer.learning_rate = 0.03
replicator.sign = off
steps = 2000
batch_size = 8
eval_every = 500
seed = 314
"""
ARMS_08 = {
    "full": "replicator.scheme = full\n",
    "spectral-1": "replicator.scheme = demo\nreplicator.chunk_size = 32\nreplicator.top_k = 32\n",
    "spectral-1/16": "replicator.scheme = demo\nreplicator.chunk_size = 32\nreplicator.top_k = 2\n",
    "random-1/16": "replicator.scheme = random\nreplicator.compression = 1/16\n",
    "striding-1/16": "replicator.scheme = striding\nreplicator.compression = 1/16\n",
    "periodic-1/16": "replicator.scheme = diloco\nreplicator.compression = 1/16\n",
}

EXTRA_LINREG_ADAMW = """
topology.nodes = 2
topology.accels_per_node = 2
model.kind = mlp
model.layer_dims = 4,16,16,3
model.activation = relu
model.loss = mse
dataset.kind = linear_regression
dataset.size = 400
dataset.noise = 0.1
optimizer.kind = decoupled_adamw
optimizer.learning_rate = 0.01
optimizer.weight_decay = 0.01
replicator.scheme = demo
replicator.chunk_size = 16
replicator.top_k = 4
replicator.sign = on
warmup_fraction = 0.1
steps = 150
batch_size = 16
eval_every = 50
seed = 5
"""

EXTRA_DDP_RANDOM = """
topology.nodes = 2
topology.accels_per_node = 2
topology.mode = ddp_all_gather
model.kind = mlp
model.layer_dims = 2,12,4
model.loss = cross_entropy
model.activation = tanh
dataset.kind = gaussian_blobs
dataset.size = 600
optimizer.kind = demo_sgd
optimizer.learning_rate = 0.05
replicator.scheme = random
replicator.compression = 1/8
replicator.transfer_dtype = fp16
replicator.sign = off
steps = 200
batch_size = 8
eval_every = 50
seed = 8
"""

EXTRA_TERNARY = """
topology.nodes = 4
topology.accels_per_node = 1
model.kind = quadratic
model.dim = 96
dataset.kind = quadratic_target
dataset.size = 300
optimizer.kind = demo_sgd
optimizer.learning_rate = 0.02
replicator.scheme = striding
replicator.compression = 1/4
replicator.transfer_dtype = ternary
replicator.sign = on
steps = 200
batch_size = 8
eval_every = 50
seed = 17
"""

# name -> config text: every run the fixture holds
RUNS = {
    "c03": C03,
    "c04a": C04A,
    "c04b": C04B,
    "c04b_full": C04B_FULL,
    "c04c_two": C04C_TWO,
    "c04c_one": C04C_ONE,
    **{f"c08_{k}": BLOBS_BASE + v for k, v in ARMS_08.items()},
    "x_linreg_adamw": EXTRA_LINREG_ADAMW,
    "x_ddp_random": EXTRA_DDP_RANDOM,
    "x_ternary": EXTRA_TERNARY,
}
