"""Host-side mirror of the reference configuration types.

Field-for-field mirror of ``sgwls::SmoothConfig`` (proj/include/sgwls/smoother.hpp:12-24),
``sgwls::WeightParams`` / ``WeightKind`` (proj/include/sgwls/weights.hpp:10-27),
``sgwls::Axis`` (proj/include/sgwls/snake.hpp:10-12), ``sgwls::SparseField``
(proj/include/sgwls/smoother.hpp:32-35) and ``sgwls::Error``
(proj/include/sgwls/error.hpp:8-11).  Defaults are the reference defaults.
Validation happens in the native library (csrc/sgwls_capi.cpp) with the
reference's exact error texts; this module only carries values.
"""
from __future__ import annotations

import dataclasses
import enum

import numpy as np


class Error(RuntimeError):
    """sgwls::Error (proj/include/sgwls/error.hpp:8-11): raised for every invalid input."""


class CudaError(Error):
    """A CUDA runtime failure inside the native library (no reference analogue)."""


class WeightKind(enum.IntEnum):
    Frac = 0
    Exp = 1


class Axis(enum.IntEnum):
    Column = 0
    Row = 1


def orthogonal(a: Axis) -> Axis:
    """proj/include/sgwls/snake.hpp:12"""
    return Axis.Row if a == Axis.Column else Axis.Column


@dataclasses.dataclass
class WeightParams:
    kind: WeightKind = WeightKind.Frac
    alpha_s: float = 1.2
    alpha_r: float = 1.2
    sigma_s: float = 4.0
    sigma_r: float = 3.0
    epsilon: float = 1e-4
    guidance_scale: float = 1.0


@dataclasses.dataclass
class SmoothConfig:
    # ``lambda`` is a Python keyword; ``lambda_`` carries SmoothConfig::lambda.
    lambda_: float = 900.0
    r: int = 1
    tau: int = 1
    iterations: int = 4
    weight: WeightParams = dataclasses.field(default_factory=WeightParams)
    first_axis: Axis = Axis.Column
    threads: int = 1  # accepted and validated like the reference; the GPU ignores it

    def copy(self, **kw) -> "SmoothConfig":
        c = dataclasses.replace(self, weight=dataclasses.replace(self.weight))
        for k, v in kw.items():
            setattr(c, k, v)
        return c


@dataclasses.dataclass
class SparseField:
    values: np.ndarray
    mask: np.ndarray
