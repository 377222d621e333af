"""Exact Riemann solver for the 1D Euler equations (test-side pin, independent of oracle/).

Textbook construction (pressure function + bisection, self-similar sampling)
used to pin the oracle HDM against the exact Sod solution that the paper plots
in Fig. 8 for the data of P:741-757.
"""
import math

import numpy as np


class ExactRiemann:
    def __init__(self, left, right, gamma=1.4):
        self.g = gamma
        self.rl, self.ul, self.pl = left
        self.rr, self.ur, self.pr = right
        self.cl = math.sqrt(gamma * self.pl / self.rl)
        self.cr = math.sqrt(gamma * self.pr / self.rr)
        self.p_star = self._solve()
        fl, _ = self._f(self.p_star, self.rl, self.pl, self.cl)
        fr, _ = self._f(self.p_star, self.rr, self.pr, self.cr)
        self.u_star = 0.5 * (self.ul + self.ur) + 0.5 * (fr - fl)

    def _f(self, p, rk, pk, ck):
        g = self.g
        if p > pk:  # shock
            A = 2.0 / ((g + 1.0) * rk)
            B = (g - 1.0) / (g + 1.0) * pk
            return (p - pk) * math.sqrt(A / (p + B)), True
        return 2.0 * ck / (g - 1.0) * ((p / pk) ** ((g - 1.0) / (2.0 * g)) - 1.0), False

    def _solve(self):
        lo, hi = 1e-12, 100.0
        F = lambda p: self._f(p, self.rl, self.pl, self.cl)[0] + self._f(p, self.rr, self.pr, self.cr)[0] + (self.ur - self.ul)
        for _ in range(300):
            mid = 0.5 * (lo + hi)
            if F(mid) > 0.0:
                hi = mid
            else:
                lo = mid
        return 0.5 * (lo + hi)

    def star_density(self, side):
        g, ps = self.g, self.p_star
        rk, pk = (self.rl, self.pl) if side == "L" else (self.rr, self.pr)
        if ps > pk:
            q = (g - 1.0) / (g + 1.0)
            return rk * (ps / pk + q) / (q * ps / pk + 1.0)
        return rk * (ps / pk) ** (1.0 / g)

    def shock_speed_right(self):
        g = self.g
        return self.ur + self.cr * math.sqrt((g + 1.0) / (2.0 * g) * self.p_star / self.pr + (g - 1.0) / (2.0 * g))

    def rarefaction_left(self):
        g = self.g
        cs = self.cl * (self.p_star / self.pl) ** ((g - 1.0) / (2.0 * g))
        return self.ul - self.cl, self.u_star - cs

    def sample(self, xi):
        """(rho, u, p) at similarity coordinate xi = (x - x0)/t (left rarefaction /
        right shock pattern, as in Sod's problem)."""
        g = self.g
        xi = np.asarray(xi, dtype=np.float64)
        rho = np.empty_like(xi)
        u = np.empty_like(xi)
        p = np.empty_like(xi)
        head, tail = self.rarefaction_left()
        s = self.shock_speed_right()
        rsl, rsr = self.star_density("L"), self.star_density("R")
        for k, x in np.ndenumerate(xi):
            if x <= head:
                rho[k], u[k], p[k] = self.rl, self.ul, self.pl
            elif x <= tail:
                a = 2.0 / (g + 1.0) + (g - 1.0) / ((g + 1.0) * self.cl) * (self.ul - x)
                rho[k] = self.rl * a ** (2.0 / (g - 1.0))
                u[k] = 2.0 / (g + 1.0) * (self.cl + (g - 1.0) / 2.0 * self.ul + x)
                p[k] = self.pl * a ** (2.0 * g / (g - 1.0))
            elif x <= self.u_star:
                rho[k], u[k], p[k] = rsl, self.u_star, self.p_star
            elif x <= s:
                rho[k], u[k], p[k] = rsr, self.u_star, self.p_star
            else:
                rho[k], u[k], p[k] = self.rr, self.ur, self.pr
        return rho, u, p
