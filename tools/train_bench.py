"""Training-harness wall time (reference sigkit::train defaults, model.hpp:39-50)
on the GPU build vs the compiled reference, same config and seed:
    python tools/train_bench.py [epochs]"""
import json
import sys
import time

sys.path.insert(0, ".")
import paper_2501_08455_b200 as sk  # noqa: E402
from oracle import oracle as O  # noqa: E402

epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = sk.TrainConfig(epochs=epochs)
sk.train(sk.TrainConfig(n_samples=64, seq_len=10, epochs=1))  # warm the library
t = time.perf_counter()
ours = sk.train(cfg)
t_ours = time.perf_counter() - t
rec = {"config": {k: (v.name if hasattr(v, "name") else v) for k, v in cfg.__dict__.items()}, "epochs": epochs,
       "gpu_s": t_ours, "gpu_losses": ours}
if O.ref() is not None:
    t = time.perf_counter()
    ref = O.ref_train(cfg.n_samples, cfg.seq_len, cfg.sig_input_size, cfg.depth, cfg.batch_size, epochs,
                      cfg.learning_rate, cfg.seed, 2, 0)
    rec["reference_cpu_s"] = time.perf_counter() - t
    rec["max_rel_loss_diff"] = max(abs(a - b) / abs(b) for a, b in zip(ours, ref))
print(json.dumps(rec))
