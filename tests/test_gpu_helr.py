"""HELR-style logistic-regression iteration (BASELINE config 5) on the GPU at a small ring:
decrypted updated weights against the same arithmetic in NumPy.  No reference counterpart exists
(application circuit); tolerance 2^-9 absolute on weights of magnitude ~0.1 (single-limb scale)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_helr_iteration_matches_plain_arithmetic():
    import torch

    assert torch.cuda.is_available()
    from paper_2512_18345_b200 import ckks, keyswitch as ks
    from paper_2512_18345_b200.helr import HelrShape, HelrTrainer, plain_iteration
    from paper_2512_18345_b200.params import generate_parameter_set
    from paper_2512_18345_b200.rns import RnsError

    p = generate_parameter_set(n=4096, l=20, dnum=4, delta=1 << 40, h_dense=64, h_sparse=32)
    sk = ks.keygen(p, h=64, seed=3)
    shape = HelrShape(samples=16, features=128)
    trainer = HelrTrainer(p, sk, shape, level=20, lr=1.0)
    rng = np.random.default_rng(8)
    x = rng.uniform(-1, 1, (shape.samples, shape.features))
    y = np.where(rng.uniform(size=shape.samples) < 0.5, -1.0, 1.0)
    z = (x * y[:, None]).reshape(-1)
    w_row = rng.uniform(-0.05, 0.05, shape.features)
    w = np.tile(w_row, shape.samples)
    ct_z, ct_w = trainer.encrypt(z, sk, seed=21), trainer.encrypt(w, sk, seed=22)
    out = trainer.iteration(ct_z, ct_w)
    assert ckks.level_of(out) == 20 - HelrTrainer.LIMBS_PER_ITERATION
    got = ckks.decrypt_decode(out, sk, p).real
    want = plain_iteration(z, w, shape, 1.0)
    assert np.abs(want - w).max() > 1e-3                      # the step moved the weights
    assert np.abs(got - want).max() < 2.0 ** -9, np.abs(got - want).max()
    # every row carries the same updated weight vector
    rows = got.reshape(shape.samples, shape.features)
    assert np.abs(rows - rows[0]).max() < 2.0 ** -9
    with pytest.raises(RnsError):
        trainer.iteration(ckks.mod_drop(ct_z, 19), ckks.mod_drop(ct_w, 19))
    with pytest.raises(RnsError):
        HelrTrainer(p, sk, HelrShape(samples=16, features=64))
