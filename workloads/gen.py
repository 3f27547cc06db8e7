"""Seeded value generator (SURVEY.md §8(d) "Seeds and values").

Values are keyed by (config, tensor index, subblock key) so that the result
does not depend on the order in which either side enumerates subblocks: a
wrong layout on the CUDA side therefore shows up as a wrong result, not as a
silently consistent permutation of the inputs.

A subblock key is the tree pair of one reduced block, given as plain integers:
  (cod_uncoupled, cod_inner, coupled, dom_uncoupled, dom_inner)
where each entry is a tuple of sector labels and each label a tuple of ints
(e.g. U1 (q,), U1xU1 (N, 2Sz), SU2 (2j,)). Values within a subblock are
column-major over (codomain legs..., domain legs...) -- the generator only
returns the 1-D sequence; placing it is each side's own business.
"""
import numpy as np

SEED_ROOT = 10076


def _zigzag(v: int) -> int:
    return 2 * v if v >= 0 else -2 * v - 1


def encode_key(key) -> list:
    """Flatten a subblock key into non-negative ints, with length prefixes."""
    out = []
    for part in key:
        if part and isinstance(part[0], tuple):  # tuple of labels
            out.append(len(part))
            for lab in part:
                out.extend(_zigzag(int(x)) for x in lab)
        else:  # a single label (the coupled sector) or empty tuple
            out.append(len(part) + 1000)
            out.extend(_zigzag(int(x)) for x in part)
    return out


def subblock_values(cfg: int, tensor_index: int, key, n: int, complex_: bool = False) -> np.ndarray:
    """N(0,1) values of one subblock (n elements, column-major order).

    ComplexF64: real parts then imaginary parts are drawn.
    """
    rng = np.random.default_rng([SEED_ROOT, cfg, tensor_index] + encode_key(key))
    if complex_:
        re = rng.standard_normal(n)
        im = rng.standard_normal(n)
        return re + 1j * im
    return rng.standard_normal(n)
