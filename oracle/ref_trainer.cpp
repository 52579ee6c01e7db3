// ref_trainer.cpp -- extern "C" face over the UNMODIFIED reference experiment layer.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile (target `ref`) compiles this file with the
// reference's own sources where they lie (/root/reference/proj/core/src/*.cpp except
// trainer.cpp, which needs nlohmann/json, absent here) into
// oracle/_ref/libdemosim_trainer_ref.so.  oracle/gen_trainer_golden.py calls it to write
// tests/golden/trainer.npz: the reference's datasets, batch order, initial parameters,
// per-step losses / traffic and final parameters for the acceptance configurations, which the
// trainer tests (tests/test_trainer_host.py, tests/test_gpu_trainer.py) compare against.
//
// The step loop below is Trainer::run (trainer.cpp:49-90) over the reference's own
// VirtualCluster, BatchStream, make_dataset, init_params and loss_and_gradient; lr_at is
// restated from trainer.cpp:24-30 because trainer.cpp itself cannot be compiled here.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "demosim/cluster.hpp"
#include "demosim/config.hpp"
#include "demosim/dataset.hpp"
#include "demosim/model.hpp"
#include "demosim/optim.hpp"
#include "demosim/rng.hpp"

namespace demosim {
// cluster.cpp:59 references trainer.cpp's formatter (trainer.cpp:18-22).
std::string format_double(double x) {
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", x);
  return buf;
}
}  // namespace demosim

using namespace demosim;

namespace {
thread_local std::string g_err;

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const TrainingError& e) {
    g_err = e.what();
    return 1;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const ProtocolError& e) {
    g_err = e.what();
    return 3;
  }
}

// trainer.cpp:24-30
double lr_at_ref(const ExperimentConfig& cfg, uint64_t step) {
  const double base = cfg.optimizer.learning_rate;
  const auto warm = static_cast<uint64_t>(
      std::llround(cfg.warmup_fraction * static_cast<double>(cfg.steps)));
  if (warm == 0 || step >= warm) return base;
  return base * static_cast<double>(step + 1) / static_cast<double>(warm);
}

void put(double* dst, const std::vector<double>& v) {
  if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * 8);
}
}  // namespace

extern "C" {

const char* dmt_last_error(void) { return g_err.c_str(); }

// sizes[0..7] = param_count, padded_len, world, train_size, val_size, input_dim, target_dim,
// gen_params_len; values[0..4] = lr, compression (effective), replicator seed, warmup, steps
int dmt_describe(const char* text, uint64_t* sizes, double* values) {
  return guarded([&] {
    const ExperimentConfig cfg = parse_config(text);
    const Dataset ds = make_dataset(cfg.dataset, cfg.seed);
    sizes[0] = cfg.model.param_count();
    sizes[1] = padded_param_len(cfg);
    sizes[2] = cfg.topology.world_size();
    sizes[3] = ds.train.size;
    sizes[4] = ds.val.size;
    sizes[5] = ds.train.input_dim;
    sizes[6] = ds.train.target_dim;
    sizes[7] = ds.gen_params.size();
    values[0] = cfg.optimizer.learning_rate;
    values[1] = effective_compression(cfg);
    values[2] = static_cast<double>(cfg.replicator.seed);
    values[3] = cfg.warmup_fraction;
    values[4] = static_cast<double>(cfg.steps);
  });
}

// make_dataset (dataset.cpp:34-120): train/val inputs, targets, labels, gen_params
int dmt_dataset(const char* text, double* train_in, double* train_tgt, int32_t* train_lab,
                double* val_in, double* val_tgt, int32_t* val_lab, double* gen) {
  return guarded([&] {
    const ExperimentConfig cfg = parse_config(text);
    const Dataset ds = make_dataset(cfg.dataset, cfg.seed);
    put(train_in, ds.train.inputs);
    put(train_tgt, ds.train.targets);
    put(val_in, ds.val.inputs);
    put(val_tgt, ds.val.targets);
    put(gen, ds.gen_params);
    if (train_lab && !ds.train.labels.empty())
      std::memcpy(train_lab, ds.train.labels.data(), ds.train.labels.size() * 4);
    if (val_lab && !ds.val.labels.empty())
      std::memcpy(val_lab, ds.val.labels.data(), ds.val.labels.size() * 4);
  });
}

// BatchStream::indices_for (dataset.cpp:141-151) for `count` (step, rank) pairs
int dmt_batch_indices(const char* text, const uint64_t* steps, const uint64_t* ranks,
                      uint64_t count, uint64_t* out) {
  return guarded([&] {
    const ExperimentConfig cfg = parse_config(text);
    const Dataset ds = make_dataset(cfg.dataset, cfg.seed);
    const BatchStream bs(ds.train.size, cfg.topology.world_size(), cfg.batch_size, cfg.seed);
    for (uint64_t i = 0; i < count; ++i) {
      const std::vector<std::size_t> idx = bs.indices_for(steps[i], ranks[i]);
      for (std::size_t j = 0; j < idx.size(); ++j) out[i * cfg.batch_size + j] = idx[j];
    }
  });
}

// init_params (model.cpp:224-244)
int dmt_init_params(const char* text, double* out) {
  return guarded([&] {
    const ExperimentConfig cfg = parse_config(text);
    put(out, init_params(cfg.model, cfg.seed, padded_param_len(cfg)));
  });
}

// loss_and_gradient (model.cpp:138-203) of the batch of (step, rank) at `params`
int dmt_loss_and_gradient(const char* text, const double* params, uint64_t step, uint64_t rank,
                          double* loss, double* grad) {
  return guarded([&] {
    const ExperimentConfig cfg = parse_config(text);
    const Dataset ds = make_dataset(cfg.dataset, cfg.seed);
    const BatchStream bs(ds.train.size, cfg.topology.world_size(), cfg.batch_size, cfg.seed);
    const std::size_t n = padded_param_len(cfg);
    const Batch b = bs.batch_for(ds.train, step, rank);
    const LossAndGradient lg =
        loss_and_gradient(cfg.model, std::span<const double>(params, n), b);
    *loss = lg.loss;
    put(grad, lg.grad);
  });
}

// forward_loss on the validation split (trainer.cpp:44-46)
int dmt_val_loss(const char* text, const double* params, double* loss) {
  return guarded([&] {
    const ExperimentConfig cfg = parse_config(text);
    const Dataset ds = make_dataset(cfg.dataset, cfg.seed);
    *loss = forward_loss(cfg.model, std::span<const double>(params, padded_param_len(cfg)),
                         ds.val);
  });
}

// Trainer::run (trainer.cpp:49-90).  Per step: train loss, val loss (NaN off the eval
// steps), intra / inter bytes; every node's worker (node, 0) parameters at the end; with `conservation` (nullable) a trace sink
// counts [traces, entries, conserved] as acceptance_test.cpp:185-197 does.  Returns the
// number of completed steps in *done (a TrainingError stops the loop, trainer.cpp:66-71).
int dmt_run(const char* text, double* train_loss, double* val_loss, uint64_t* intra,
            uint64_t* inter, double* final_node_params, uint64_t* conservation,
            uint64_t* done) {
  return guarded([&] {
    const ExperimentConfig cfg = parse_config(text);
    const Dataset ds = make_dataset(cfg.dataset, cfg.seed);
    const std::size_t padded = padded_param_len(cfg);
    const DenseVector init = init_params(cfg.model, cfg.seed, padded);
    VirtualCluster cluster(cfg.topology, cfg.model.param_count(), cfg.pad_params, cfg.optimizer,
                           cfg.replicator, init);
    cluster.set_link(cfg.link);
    const BatchStream stream(ds.train.size, cfg.topology.world_size(), cfg.batch_size,
                             cfg.seed);
    const std::size_t a = cfg.topology.accels_per_node;
    uint64_t traces = 0, entries = 0, conserved = 0;
    const VirtualCluster::TraceSink sink = [&](std::size_t, std::size_t, const StepTrace& t) {
      ++traces;
      for (std::size_t i = 0; i < t.m_accum.size(); ++i) {
        ++entries;
        if (t.m_after[i] == t.m_accum[i] - t.local_q[i]) ++conserved;
      }
    };
    *done = 0;
    try {
      for (uint64_t step = 0; step < cfg.steps; ++step) {
        double loss_sum = 0.0;
        auto grad_fn = [&](std::size_t node, std::size_t accel,
                           const DenseVector& params) -> DenseVector {
          const Batch b = stream.batch_for(ds.train, step, node * a + accel);
          LossAndGradient lg = loss_and_gradient(cfg.model, params, b);
          loss_sum += lg.loss;
          return std::move(lg.grad);
        };
        cluster.run_step(step, lr_at_ref(cfg, step), grad_fn,
                         conservation != nullptr ? &sink : nullptr);
        const double tl = loss_sum / static_cast<double>(cfg.topology.world_size());
        if (!std::isfinite(tl)) throw TrainingError("training diverged");
        train_loss[step] = tl;
        val_loss[step] = std::numeric_limits<double>::quiet_NaN();
        if ((step + 1) % cfg.eval_every == 0 || step + 1 == cfg.steps)
          val_loss[step] = forward_loss(cfg.model, cluster.worker_params(0, 0), ds.val);
        const StepTraffic& t = cluster.ledger().steps().back();
        intra[step] = t.intra_bytes;
        inter[step] = t.inter_bytes;
        *done = step + 1;
      }
    } catch (const TrainingError&) {
      // partial results stand, as the reference CLI flushes them (demosim.cpp:62-69)
    }
    for (std::size_t j = 0; j < cfg.topology.nodes; ++j) {
      const DenseVector& p = cluster.worker_params(j, 0);
      std::memcpy(final_node_params + j * p.size(), p.data(), p.size() * 8);
    }
    if (conservation) {
      conservation[0] = traces;
      conservation[1] = entries;
      conservation[2] = conserved;
    }
  });
}

}  // extern "C"
