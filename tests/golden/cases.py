"""Inputs of the golden fixtures (shared by make_golden.py and the tests)."""
import numpy as np

RIR_CASES = [
    dict(room=[5.0, 5.0, 5.0], r=0.5, K=0, src=[1.0, 1.0, 1.0], mic=[2.0, 1.0, 1.0], max_taps=0),
    dict(room=[3.0, 4.0, 5.0], r=0.5, K=1, src=[1.0, 2.0, 2.0], mic=[2.0, 2.0, 2.0], max_taps=0),
    dict(room=[6.3, 4.1, 2.9], r=0.85, K=6, src=[1.7, 2.2, 1.4], mic=[4.9, 1.1, 1.6], max_taps=0),
    dict(room=[9.1, 7.7, 3.3], r=0.7, K=9, src=[0.6, 6.9, 2.0], mic=[8.0, 0.9, 1.2], max_taps=2500),
    dict(room=[3.2, 3.1, 2.6], r=0.9, K=14, src=[1.1, 1.9, 1.2], mic=[2.4, 0.7, 1.8], max_taps=6000),
    dict(room=[7.5, 5.5, 4.0], r=0.35, K=4, src=[3.0, 2.0, 1.0], mic=[3.05, 2.0, 1.0], max_taps=0),
]

PLAN_CASES = [(116991, 3893), (80000, 4096), (1, 1), (16, 2), (100, 1), (240000, 13120),
              (32000, 600), (160000, 19200), (2000, 256), (5, 5000), (131874, 857)]


def ola_case():
    g = np.random.Generator(np.random.Philox(key=1234))
    x = g.standard_normal(3001)
    h = g.standard_normal(300) * np.exp(-np.arange(300) / 60.0)
    return x, h, 512
