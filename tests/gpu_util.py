"""Helpers shared by the GPU parity tests."""
import numpy as np
import torch


def dev(a, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


def host(t):
    return t.detach().to("cpu").to(torch.float64).numpy() if t.dtype != torch.int32 else t.cpu().numpy()


def beq(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


def bf16_round(a):
    """Round fp64 values to bf16 exactly as torch does (RN-even) and back to fp64."""
    return torch.as_tensor(np.asarray(a, np.float64)).to(torch.float32).to(torch.bfloat16).to(torch.float64).numpy()


def rel_l2(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    den = np.linalg.norm(want)
    return float(np.linalg.norm(got - want) / (den if den > 0 else 1.0))


def random_assignment(rng, n, k, e):
    """distinct experts per row, like a real top-k (test_dispatch.cpp:17-31)"""
    idx = np.empty((n, k), np.int64)
    for i in range(n):
        idx[i] = rng.choice(e, size=k, replace=False)
    return idx


def well_separated_rows(scores, k, margin=1e-4):
    """Rows whose top-(k+1) sorted scores are separated by > margin
    (test_gate.cpp:20-28): their top-k selection is robust to rounding."""
    s = np.sort(scores, axis=1)[:, ::-1]
    m = min(k + 1, s.shape[1])
    gaps = s[:, : m - 1] - s[:, 1:m]
    return (gaps > margin).all(axis=1) if m > 1 else np.ones(len(s), bool)
