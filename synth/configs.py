"""The five BASELINE.json workloads (BASELINE.json:7-11) as synthetic recipes.

Recipes are defined in synth_core.h; readings R21-R24 of SURVEY.md §8(c) fix
what the one-line descriptions leave open.
"""
from dataclasses import dataclass

PLANTED, IMAGE, SPECTRO, RATINGS, SPARSE = 1, 2, 3, 4, 5


@dataclass(frozen=True)
class Config:
    name: str
    recipe: int
    m: int
    n: int
    r: int
    k: int          # inner dimension of the planted product (0 for RATINGS)
    noise: float
    sweeps: int
    seed: int = 0
    normalised: bool = True   # IMAGE only: reading R21
    density: float = 1.0      # SPARSE only: probability that an entry is stored

    def scaled(self, m, n, r=None, k=None, name=None, density=None):
        """Same recipe at another shape (small parity cases)."""
        return Config(name or f"{self.name}@{m}x{n}", self.recipe, m, n,
                      r if r is not None else self.r,
                      k if k is not None else self.k, self.noise, self.sweeps,
                      self.seed, self.normalised,
                      density if density is not None else self.density)


C1 = Config("C1-planted", PLANTED, 200, 100, 5, 5, 0.01, 200)
C2 = Config("C2-image", IMAGE, 361, 2429, 49, 49, 0.05, 500)
C3 = Config("C3-spectro", SPECTRO, 513, 8192, 32, 32, 0.01, 500)
C4 = Config("C4-ratings", RATINGS, 6040, 3706, 20, 0, 0.0, 300)
C5 = Config("C5-large-planted", PLANTED, 200000, 50000, 128, 128, 0.01, 100)
# stand-in for the sparse Reuters matrix of PAPER.md:418 / Table reuters
# (804,414 x 47,236, 99.84 % sparse, r up to 100): a planted product sampled at density 0.0016
# (reading R27; no Reuters items are reproduced)
C6 = Config("C6-reuters-like", SPARSE, 804414, 47236, 100, 100, 0.01, 100, density=0.0016)

ALL = {c.name: c for c in (C1, C2, C3, C4, C5, C6)}
