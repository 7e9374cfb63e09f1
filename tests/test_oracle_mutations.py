"""Mutation check of the oracle's pins (-m "not gpu").

Each mutation below is a plausible mistake in oracle/ (a dropped term, a wrong sign or
reduction, a swapped slot, the wrong branch negated).  The oracle is copied with the
mutation applied and the pin suites (test_oracle_pins.py, test_oracle_pins_r2.py) are run
against the copy: every mutation must make at least one pin fail.  A mutation whose
source text is no longer in oracle/ fails this test too (a refactor must update the list).
"""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, file under oracle/, original text, mutated text)
MUTATIONS = [
    ("dnf min -> max", "step.py", ".min(dim=0).values", ".max(dim=0).values"),
    ("q2b offset min -> mean", "model.py", "omin = O.min(dim=0).values", "omin = O.mean(dim=0)"),
    ("q2b offset sigmoid(z) -> sigmoid(-z)", "model.py", "omin * torch.sigmoid(z)", "omin * torch.sigmoid(-z)"),
    ("q2b offset deepset mean -> sum", "model.py", 'P["off_b1"]).mean(dim=0)', 'P["off_b1"]).sum(dim=0)'),
    ("q2b projection without relu", "model.py", 'o + torch.relu(P["rel_offset"][r])', 'o + P["rel_offset"][r]'),
    ("q2b attention softmax over dims", "model.py", "a = torch.softmax(logits, dim=0)", "a = torch.softmax(logits, dim=-1)"),
    ("q2b dist_in weight dropped", "model.py", "dist_out + box_alpha * dist_in", "dist_out + dist_in"),
    ("eq1 1/n_i -> 1/K", "step.py", "/ torch.clamp(n_i, min=1.0)", "/ mask.shape[1]"),
    ("eq1 positive term sign", "step.py", "softplus(d_pos - cfg.gamma)", "softplus(cfg.gamma - d_pos)"),
    ("betae projection +1 -> +0.5", "model.py", "torch.clamp(y + 1.0, 0.05, 1e9)", "torch.clamp(y + 0.5, 0.05, 1e9)"),
    ("betae projection clamp floor dropped", "model.py", "torch.clamp(y + 1.0, 0.05, 1e9)", "torch.clamp(y + 1.0, -1e9, 1e9)"),
    ("betae attention softmax over dims", "model.py", "w = torch.softmax(logits, dim=0)", "w = torch.softmax(logits, dim=-1)"),
    ("betae kl argument order", "model.py", "return beta_kl(a1, b1, a2, b2)", "return beta_kl(a2, b2, a1, b1)"),
    ("gqe deepset mean -> sum", "model.py", 'P["ds_b1"]).mean(dim=0)\n        return _linear', 'P["ds_b1"]).sum(dim=0)\n        return _linear'),
    ("2p relation order", "model.py", "return [p(p(A[0], 0), 1)]", "return [p(p(A[0], 1), 0)]"),
    ("3p relation order", "model.py", "return [p(p(p(A[0], 0), 1), 2)]", "return [p(p(p(A[0], 0), 2), 1)]"),
    ("2i relation slots swapped", "model.py", "return [i(p(A[0], 0), p(A[1], 1))]", "return [i(p(A[0], 1), p(A[1], 0))]"),
    ("3i relation slots rotated", "model.py", "return [i(p(A[0], 0), p(A[1], 1), p(A[2], 2))]",
     "return [i(p(A[0], 1), p(A[1], 2), p(A[2], 0))]"),
    ("ip final relation swapped", "model.py", "return [p(i(p(A[0], 0), p(A[1], 1)), 2)]",
     "return [p(i(p(A[0], 2), p(A[1], 1)), 0)]"),
    ("pi relation slots swapped", "model.py", "return [i(p(p(A[0], 0), 1), p(A[1], 2))]",
     "return [i(p(p(A[0], 0), 2), p(A[1], 1))]"),
    ("up shared relation swapped", "model.py", "return [p(p(A[0], 0), 2), p(p(A[1], 1), 2)]",
     "return [p(p(A[0], 0), 2), p(p(A[1], 2), 1)]"),
    ("2in negates the wrong branch", "model.py", "return [i(p(A[0], 0), n(p(A[1], 1)))]",
     "return [i(n(p(A[0], 0)), p(A[1], 1))]"),
    ("3in negates the wrong branch", "model.py", "return [i(p(A[0], 0), p(A[1], 1), n(p(A[2], 2)))]",
     "return [i(p(A[0], 0), n(p(A[1], 1)), p(A[2], 2))]"),
    ("inp negation dropped", "model.py", "return [p(i(p(A[0], 0), n(p(A[1], 1))), 2)]",
     "return [p(i(p(A[0], 0), p(A[1], 1)), 2)]"),
    ("pin negates the chain", "model.py", "return [i(p(p(A[0], 0), 1), n(p(A[1], 2)))]",
     "return [i(n(p(p(A[0], 0), 1)), p(A[1], 2))]"),
    ("pni negates the single hop", "model.py", "return [i(n(p(p(A[0], 0), 1)), p(A[1], 2))]",
     "return [i(p(p(A[0], 0), 1), n(p(A[1], 2)))]"),
    ("adam eps inside sqrt", "step.py", "np.sqrt(v_hat) + eps", "np.sqrt(v_hat + eps)"),
    ("adam bias correction dropped", "step.py", "m_hat = m / (1.0 - beta1 ** t)", "m_hat = m"),
]


def _prepare(tmp, name, fname, old, new):
    dst = os.path.join(tmp, name.replace(" ", "_").replace("/", "_").replace(">", ""))
    os.makedirs(dst)
    for d in ("oracle", "kggen", "tests"):
        shutil.copytree(os.path.join(ROOT, d), os.path.join(dst, d),
                        ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
    path = os.path.join(dst, "oracle", fname)
    src = open(path).read()
    if old not in src:
        return None
    open(path, "w").write(src.replace(old, new))
    return dst


@pytest.fixture(scope="module")
def outcomes(tmp_path_factory):
    """Run the pin suites against every mutated copy, several copies at a time."""
    tmp = str(tmp_path_factory.mktemp("mutants"))
    dirs = {m[0]: _prepare(tmp, *m) for m in MUTATIONS}
    env = dict(os.environ, OMP_NUM_THREADS="1", MKL_NUM_THREADS="1")
    par = max(2, min(16, os.cpu_count() or 2))
    pending = [n for n in dirs if dirs[n]]
    running, out = {}, {}
    while pending or running:
        while pending and len(running) < par:
            n = pending.pop(0)
            running[n] = subprocess.Popen(
                [sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                 "tests/test_oracle_pins_r2.py", "tests/test_oracle_pins.py", "-m", "not gpu",
                 "-k", "not finite_differences"],
                cwd=dirs[n], stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True, env=env)
        n = next(iter(running))
        p = running.pop(n)
        text, _ = p.communicate(timeout=900)
        out[n] = (p.returncode, text)
    return dirs, out


@pytest.mark.parametrize("name", [m[0] for m in MUTATIONS])
def test_mutation_is_caught(name, outcomes):
    dirs, out = outcomes
    assert dirs[name] is not None, f"mutation '{name}': its source text is no longer in oracle/"
    rc, text = out[name]
    assert rc == 1 and " failed" in text, f"mutation '{name}' survived every pin:\n{text[-2500:]}"
