"""The training harness (reference sigkit::train, model.cpp:222-263; paper
§3.2) with the signature forward and VJP on the GPU, against the reference's
frozen desk-scale trajectory (tests/test_model.cpp:214-223) and the compiled
reference's own training loop (oracle/_ref). Bar: relative 1e-9 per epoch loss
(fp64 throughout; only the summation order inside the signature differs)."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

DESK = dict(n_samples=256, seq_len=20, sig_input_size=3, depth=2, batch_size=64, epochs=3, learning_rate=0.05,
            seed=7)
FROZEN = [0.25664234253569584, 0.2318731160083158, 0.21248612183066107]


def test_frozen_desk_trajectory(sk):
    got = sk.train(sk.TrainConfig(**DESK, kernel=sk.KernelKind.Sequential))
    np.testing.assert_allclose(got, FROZEN, rtol=1e-9, atol=0)


@pytest.mark.parametrize("cfg", [
    dict(n_samples=200, seq_len=33, sig_input_size=4, depth=3, batch_size=48, epochs=2, learning_rate=0.05, seed=3),
    dict(n_samples=100, seq_len=50, sig_input_size=5, depth=4, batch_size=64, epochs=2, learning_rate=0.02, seed=11),
    dict(n_samples=64, seq_len=8, sig_input_size=2, depth=5, batch_size=16, epochs=2, learning_rate=0.1, seed=5),
])
@pytest.mark.parametrize("activation", ["tanh", "identity"])
def test_matches_reference_training_loop(sk, cfg, activation):
    if O.ref() is None:
        pytest.skip("oracle/_ref (the compiled reference) is not built")
    got = sk.train(sk.TrainConfig(**cfg, activation=activation))
    ref = O.ref_train(cfg["n_samples"], cfg["seq_len"], cfg["sig_input_size"], cfg["depth"], cfg["batch_size"],
                      cfg["epochs"], cfg["learning_rate"], cfg["seed"], 0, 0 if activation == "tanh" else 1)
    np.testing.assert_allclose(got, ref, rtol=1e-9, atol=0)


def test_config_validation(sk):
    for bad in (dict(epochs=0), dict(sig_input_size=1), dict(sig_input_size=11), dict(batch_size=0),
                dict(activation="relu")):
        with pytest.raises(sk.DomainError):
            sk.train(sk.TrainConfig(**{**DESK, **bad}))


def test_divergence_raises(sk):
    with pytest.raises(sk.TrainingError, match="non-finite loss at epoch") as e:
        sk.train(sk.TrainConfig(**{**DESK, "epochs": 20, "learning_rate": 1e9}, activation="identity"))
    assert 0 <= e.value.epoch < 20
