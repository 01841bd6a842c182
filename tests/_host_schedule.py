"""Python mirror of starmm_execute_host's phase-1 rule (starmm_api.cu
host_phase1_chunks / host_nominal_ops), shared by the CPU and GPU tests."""
import os

import numpy as np

import paper_1911_05328_b200 as sm

NOMINAL_OPS = {"float": 35e12, "int": 100e12}   # starmm_api.cu host_nominal_ops (else 60e12)


def host_phase1(m, n, k, sid, aliased=False, store=False, base_dim=64):
    """Phase-1 (k-outer) chunk boundaries of starmm_execute_host (starmm_api.cu
    host_phase1_chunks): only for compute-bound problems (estimated compute time >
    H2D time at 50 GB/s) unless STARMM_HOST_PHASE1 forces it; widths k/64 (fp64, k >= 8192)
    or k/32, then doubling,
    (multiples of max(128, base_dim): a leaf never straddles two chunks) covering <= k/2."""
    kb = [0]
    env = os.environ.get("STARMM_HOST_PHASE1", "")
    if env[:1] == "0" or m < 512 or k < 512:
        return kb
    eb = np.dtype(sm.get_semiring(sid).dtype).itemsize
    h2d = eb * (m * k + (0 if aliased else k * n) + (0 if store else m * n))
    if env[:1] != "1" and 2.0 * m * n * k / NOMINAL_OPS.get(sid, 60e12) < h2d / 50e9:
        return kb
    div = 64 if (k >= 8192 and sid == "float") else 32
    cq = max(128, base_dim)
    w = max(cq, -(-(-(-k // div)) // cq) * cq)
    while kb[-1] + w <= k // 2:
        kb.append(kb[-1] + w)
        w *= 2
    return kb
