"""Fast exp / ln / pow: the reference's module surface (ti64micro/fastmath.py).

``fast_exp``, ``fast_ln`` and ``fast_pow`` run the device cores of
csrc/ti64_fastmath.cuh (bit-identical to fastmath.py:161-212).  The
coefficient tables (fastmath.py:40-94) are exposed as data, and the
polynomial helpers ``estrin_eval`` / ``horner_eval`` (:261-303) and the
accuracy sweep ``error_sweep`` (:306-326) are host numpy, as there.
"""

from dataclasses import dataclass, field

import numpy as np

from .batch import fast_exp, fast_ln, fast_pow

__all__ = ["PolyCorrection", "FastMathConstants", "CONSTANTS", "EXP_CORRECTION",
           "LN_CORRECTION", "estrin_eval", "horner_eval", "error_sweep", "fast_exp",
           "fast_ln", "fast_pow"]


@dataclass(frozen=True)
class PolyCorrection:
    """Correction polynomial sum_i c_i y^i on y in [0, 1)."""

    coefficients: tuple

    @property
    def degree(self):
        return len(self.coefficients) - 1


# K_exp(yf) ~ 1 + yf - 2^yf (degree 7) and K_ln(m) ~ log2(1 + m) (degree 11);
# the device tables c_EA / c_LB hold the same doubles
EXP_CORRECTION = PolyCorrection((1.213071811889e-10, 3.068528102657e-1, -2.40226342399359e-1,
                                 -5.55053313414954e-2, -9.6135243288483e-3,
                                 -1.34288475963084e-3, -1.43131744483589e-4,
                                 -2.1595656126349e-5))
LN_CORRECTION = PolyCorrection((1.84775672096293e-10, 1.44269504084132, -0.721347520143005,
                                0.480898345526187, -0.360675000332004, 0.288048466919235,
                                -0.235306287368882, 0.183102904829435, -0.1209962689793,
                                0.0591503811592113, -0.0181149492489989,
                                0.00254488675605743))


@dataclass(frozen=True)
class FastMathConstants:
    """IEEE-754 layout constants and the admissible exp argument range."""

    bias: int = 1023
    mantissa_scale: float = 2.0**52
    log2_e: float = 1.4426950408889634
    ln_2: float = 0.6931471805599453
    exp_arg_min: float = -708.0
    exp_arg_max: float = 709.0
    saturation: float = field(default=float(np.finfo(np.float64).max))


CONSTANTS = FastMathConstants()


def _coeffs(poly):
    return poly.coefficients if isinstance(poly, PolyCorrection) else tuple(poly)


def estrin_eval(poly, y):
    """Estrin pairing: (c[2k+1] y + c[2k]) groups joined with y^2, y^4, ..."""
    c = _coeffs(poly)
    y = np.asarray(y, dtype=np.float64)
    terms = [c[i + 1] * y + c[i] for i in range(0, len(c) - 1, 2)]
    if len(c) % 2:
        terms.append(np.full(y.shape, c[-1]))
    p = y * y
    while len(terms) > 1:
        nxt = [terms[j + 1] * p + terms[j] for j in range(0, len(terms) - 1, 2)]
        if len(terms) % 2:
            nxt.append(terms[-1])
        terms = nxt
        p = p * p
    return float(terms[0]) if y.ndim == 0 else terms[0]


def horner_eval(poly, y):
    """Horner evaluation of the same coefficients."""
    c = _coeffs(poly)
    y = np.asarray(y, dtype=np.float64)
    acc = np.full(y.shape, c[-1])
    for ci in c[-2::-1]:
        acc = acc * y + ci
    return float(acc) if y.ndim == 0 else acc


def error_sweep(fn, xs):
    """(exact, approx, rel_err) of fn in {'exp', 'ln', 'pow'} over xs ((n, 2)
    base/exponent pairs for 'pow'); approx from the device cores."""
    xs = np.asarray(xs, dtype=np.float64)
    if fn == "exp":
        exact, approx = np.exp(xs), fast_exp(xs)
    elif fn == "ln":
        exact, approx = np.log(xs), fast_ln(xs)
    elif fn == "pow":
        exact, approx = xs[:, 0] ** xs[:, 1], fast_pow(xs[:, 0], xs[:, 1])
    else:
        raise ValueError(f"unknown function {fn!r}")
    with np.errstate(divide="ignore", invalid="ignore"):
        rel = np.abs(approx - exact) / np.abs(exact)
    return exact, approx, rel
