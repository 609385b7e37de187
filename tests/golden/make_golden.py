"""Generate the golden fixtures in tests/golden/ from the REFERENCE ITSELF.

Run in the build container (where /root/reference exists and oracle/_ref is
built):   python tests/golden/make_golden.py

Every fixture is produced by oracle/_ref/libfmoe_ref.so -- the reference's own
sources compiled side by side -- through its public API.  Inputs are not stored
when they can be regenerated from the seeded generators (UniformRng /
stream_seed, themselves pinned by tests/test_oracle.py); outputs are stored in
full.  The fixtures travel with the repo, so the GPU box (which has no
/root/reference) still checks the oracle and the kernels against reference
outputs.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import orc, ref  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# (name, seed, n, d, h, E, k): single-worker layer fwd+bwd, inputs from the
# bench generators (x: stream 102, dy: stream 103; fmoe_bench.cpp:226-227).
LAYER_CASES = [
    ("layer_a", 42, 64, 32, 48, 8, 2),
    ("layer_b", 7, 33, 16, 24, 5, 3),   # ragged sizes, odd E, k=3
    ("layer_c", 42, 40, 32, 32, 16, 1),  # k=1
]

# (name, seed, world, n_per_rank, d, h, e_local, k): expert-parallel fwd+bwd
# over the reference's InProcWorld; inputs from streams 200+r / 300+r
# (fmoe_bench.cpp:259-262).
DIST_CASES = [
    ("dist_w2", 42, 2, 16, 16, 24, 2, 2),
    ("dist_w4", 11, 4, 12, 16, 16, 2, 2),
]


def layer_case(name, seed, n, d, h, e, k):
    w = ref.init_state(seed, d, h, e, k)
    x = orc.seeded_matrix(seed, 102, n, d)
    dy = orc.seeded_matrix(seed, 103, n, d)
    out = ref.moe_forward_backward(x, dy, k, **w)
    scores, idx, vals = ref.gate_forward(x, w["wg"], k)
    plan = ref.build_plan(idx, e)
    np.savez_compressed(
        os.path.join(OUT, f"{name}.npz"),
        meta=np.array([seed, n, d, h, e, k], np.int64),
        scores=scores, idx=idx, vals=vals,
        counts=plan["counts"], offsets=plan["offsets"], src_row=plan["src_row"],
        slot=plan["slot"], inverse_pos=plan["inverse_pos"],
        y=out["y"], dx=out["dx"], dwg=out["dwg"], dw1=out["dw1"], db1=out["db1"],
        dw2=out["dw2"], db2=out["db2"],
        y_naive=ref.naive_forward(x, k, **w),
    )


def dist_case(name, seed, world, n, d, h, el, k):
    e = el * world
    w = ref.init_state(seed, d, h, e, k)
    x = np.concatenate([orc.seeded_matrix(seed, 200 + r, n, d) for r in range(world)])
    dy = np.concatenate([orc.seeded_matrix(seed, 300 + r, n, d) for r in range(world)])
    out = ref.moe_distributed(x, dy, world, k, **w)
    np.savez_compressed(
        os.path.join(OUT, f"{name}.npz"),
        meta=np.array([seed, world, n, d, h, el, k], np.int64),
        **{key: out[key] for key in ("y", "dx", "dwg", "dw1", "db1", "dw2", "db2",
                                     "send_counts", "recv_counts")},
    )


def plan_cases():
    """Zipf-skewed routing (cfg5 shape, scaled down) through build_plan."""
    rng = np.random.default_rng(2103)
    e = 64
    p = 1.0 / np.arange(1, e + 1)
    p /= p.sum()
    idx = rng.choice(e, size=(4096, 1), p=p).astype(np.int64)
    plan = ref.build_plan(idx, e)
    np.savez_compressed(os.path.join(OUT, "plan_zipf.npz"), idx=idx, **plan)


def naive_2024():
    """test_moe_layer.cpp:97-106 'naive_forward golden regression values' left
    its values as GOLDEN_PLACEHOLDER; freeze them here from the reference:
    n_b=8, d_m=6, d_h=6, k=2, n_e_local=4, seed=2024, input stream 3 (the
    seeded_input helper, test_moe_layer.cpp:19-22)."""
    seed, n, d, h, e, k = 2024, 8, 6, 6, 4, 2
    w = ref.init_state(seed, d, h, e, k)
    x = ref.uniform_fill(ref.stream_seed(seed, 3), n * d).reshape(n, d)
    np.savez_compressed(os.path.join(OUT, "naive_2024.npz"), x=x, y=ref.naive_forward(x, k, **w),
                        y_batched=ref.moe_forward_backward(x, None, k, **w)["y"])


def main():
    naive_2024()
    for c in LAYER_CASES:
        layer_case(*c)
    for c in DIST_CASES:
        dist_case(*c)
    plan_cases()
    print("wrote", sorted(f for f in os.listdir(OUT) if f.endswith(".npz")))


if __name__ == "__main__":
    main()
