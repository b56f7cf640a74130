"""Beyond the oracle's reach (BASELINE configs[3]: Amazon-shaped, 14.2 M
vertices, ~245 M nonzeros, {300,16,16,24}): the partitioned strategies of
north_star's 8-GPU configurations — 2D 2x2 and 3D 2x2x2 (and 1.5D c=2 at P=8,
Protein's strategy) — against one rank on the same full-size graph, every rank
of a run sharing one B200 through the in-process world.  Same bar as the
oracle tests — losses, h_final, every y and w within 1e-4 relative — for all
quantities that are continuous in the inputs.  The layer gradients G_l =
(S W^T) ⊙ relu'(Z_l) are not: relu' jumps at Z = 0, and among 14.2 M x 16
pre-activations a few hundred sit within fp32 rounding of zero, so differently
ordered (equally valid) fp32 sums switch them (measured: G_0 4.6e-4, G_1
7.2e-5 relative, while the weight gradients they feed agree to 5e-7).  G is
held to 1e-3 here; at the oracle's sizes it meets 1e-4 (test_gpu_training.py)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N, E = 14249639, 230788269
DIMS = [300, 16, 16, 24]


@pytest.fixture(scope="module")
def amazon(cg):
    d = cg.generate_dataset(N, E / N, DIMS[0], DIMS[-1], 1, 2, 3, device=0, generator="skip")
    yield d
    d.free()


@pytest.fixture(scope="module")
def single(cg, amazon):
    model = cg.init_glorot(DIMS, 4, 0.5)
    return cg.run_distributed(amazon, model, cg.Strategy("1d", 1, reassociate=True), 2)


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("kind,P,repl", [("2d", 4, 1), ("3d", 8, 1), ("1.5d", 8, 2)])
def test_amazon_strategies_agree(cg, amazon, single, kind, P, repl):
    model = cg.init_glorot(DIMS, 4, 0.5)
    out = cg.run_distributed(amazon, model, cg.Strategy(kind, P, repl, reassociate=True), 2,
                             comm="local")
    errs = {"loss": max(abs(a - b) / max(1.0, abs(b)) for a, b in zip(out.losses, single.losses)),
            "h_final": rel(out.h_final, single.h_final)}
    for l in range(len(DIMS) - 1):
        errs[f"y{l}"] = rel(out.y_final[l], single.y_final[l])
        errs[f"w{l}"] = rel(out.model.weights[l], single.model.weights[l])
        errs[f"g{l}"] = rel(out.g_final[l], single.g_final[l])
    print(kind, P, {k: f"{v:.2e}" for k, v in errs.items()})
    assert max(v for k, v in errs.items() if not k.startswith("g")) < 1e-4, errs
    assert max(v for k, v in errs.items() if k.startswith("g")) < 1e-3, errs

