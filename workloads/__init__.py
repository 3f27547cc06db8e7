"""Seeded synthetic workloads shared by the oracle side and the CUDA side.

This package holds ONLY input recipes: which graded spaces each BASELINE config
uses (readings C3, C15-C20 in DESIGN.md) and the seeded value
generator. It contains none of the method's arithmetic (no layout, no fusion
rules, no permutation, no contraction), so both the oracle and the CUDA path
may import it without sharing any computation.
"""
