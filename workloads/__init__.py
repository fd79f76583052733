"""BENCH / TEST INPUT PREPARATION — seeded synthetic workloads (datasets.py) and
cached graphs (graphs.py) for BASELINE.json's configs.

Deliberately outside the product package: the reference arm of bench.py
(`--impl reference`) imports this module to regenerate its inputs and must not
load libqvg.so, which importing `paper_2605_02171_b200` does.
"""
