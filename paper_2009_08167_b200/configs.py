"""The BASELINE.json configurations."""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Config:
    name: str
    d: int
    ne: int
    p: int
    level: int
    n0: int      # eigenpairs requested ("the first N0"); lam_e goes in the next gap
    slices: int  # uniform shifts over [0, lam_e]
    text: str


CONFIGS = {
    "cfg1": Config("cfg1", 2, 16, 2, 0, 20, 1, "2D 16x16 p=2 IGA, 1 shift, 20 eigenpairs"),
    "cfg2": Config("cfg2", 2, 64, 3, 3, 100, 2, "2D 64x64 p=3 rIGA BS=8, 2 slices, 100 eigenpairs"),
    "cfg2_iga": Config("cfg2_iga", 2, 64, 3, 0, 100, 2, "2D 64x64 p=3 IGA, 2 slices, 100 eigenpairs"),
    "cfg3": Config("cfg3", 2, 256, 4, 4, 2000, 16,
                   "2D 256x256 p=4 rIGA BS=16, 16 uniform slices, 2000 eigenpairs"),
    "cfg4": Config("cfg4", 3, 32, 2, 2, 500, 8, "3D 32^3 p=2 rIGA BS=8, 8 slices, 504 eigenpairs"),
    "cfg4_iga": Config("cfg4_iga", 3, 32, 2, 0, 500, 8, "3D 32^3 p=2 IGA, 8 slices, 504 eigenpairs"),
    "cfg5": Config("cfg5", 3, 64, 3, 2, 4000, 32, "3D 64^3 p=3 rIGA BS=16, 32 slices, 4001 eigenpairs"),
}
