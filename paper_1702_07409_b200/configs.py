"""The five workloads of BASELINE.json:configs (1-based in prose, 0-based here).

Plain parameter records only -- no arithmetic of the method lives here, so tests,
the oracle callers and bench.py can all share them.  Notation follows SURVEY.md §0:
k data symbols (paper b), p precode checks (paper k-b) of d_p data neighbours each,
K = k+p intermediate symbols, n coded symbols of t bytes, S stripes.
Graph seed = data seed (reading R3).
"""

# Finite max-degree Omega(x) of PAPER.md:105-108 (the Raptor distribution the paper
# cites), with the top degrees 65/66 that BASELINE.json:configs[2] states (reading R8).
OMEGA_DEGREES = (1, 2, 3, 4, 5, 8, 9, 19, 65, 66)
OMEGA_PROBS = (0.007969, 0.493570, 0.166220, 0.072646, 0.082558,
               0.056058, 0.037229, 0.055590, 0.025023, 0.003135)

RSD = 1
FINITE = 2

CONFIGS = {
    1: dict(name="c1_tiny_lt", k=100, p=0, d_p=0, n=130, t=512, dist=RSD,
            rsd_c=0.1, rsd_delta=0.05, seed=1, stripes=1),
    2: dict(name="c2_precode_lt", k=1000, p=20, d_p=3, n=1300, t=4096, dist=RSD,
            rsd_c=0.05, rsd_delta=0.01, seed=2, stripes=1),
    3: dict(name="c3_finite_omega", k=10000, p=100, d_p=4, n=12000, t=1024, dist=FINITE,
            seed=3, stripes=1),
    4: dict(name="c4_multistripe_1GiB", k=1024, p=16, d_p=3, n=1280, t=4096, dist=RSD,
            rsd_c=0.1, rsd_delta=0.05, seed=4, stripes=256),
    5: dict(name="c5_large_stripe", k=50000, p=500, d_p=4, n=60000, t=8192, dist=FINITE,
            seed=5, stripes=1),
    # Not a BASELINE config: the NEXT-2 measurement workload -- config 4's shape (256 stripes of
    # 4 KiB symbols, RSD(0.1, 0.05), n=1280) with the paper's array-LDPC precode (Alg 2) for
    # (b, k) = (962, 1036): P=37, k'=28, j'=2, 74 checks of 26 members in 2 levels.
    6: dict(name="c6_array_precode", k=962, p=74, d_p=26, n=1280, t=4096, dist=RSD,
            rsd_c=0.1, rsd_delta=0.05, seed=6, stripes=256, precode="array"),
    # Not a BASELINE config: the NEXT-3 measurement workload -- config 2's code (CGA converges on
    # it) written as s = 10 output files (per-file streams, R17), 256 stripes of 4 KiB symbols.
    7: dict(name="c7_repair", k=1000, p=20, d_p=3, n=1300, t=4096, dist=RSD,
            rsd_c=0.05, rsd_delta=0.01, seed=2, stripes=256, files=10),
}


def get(cfg_id, **overrides):
    c = dict(CONFIGS[cfg_id])
    c.setdefault("rsd_c", 0.0)
    c.setdefault("rsd_delta", 0.0)
    if c["dist"] == FINITE:
        c["fin_deg"] = OMEGA_DEGREES
        c["fin_prob"] = OMEGA_PROBS
    else:
        c["fin_deg"] = ()
        c["fin_prob"] = ()
    c.update(overrides)
    return c
