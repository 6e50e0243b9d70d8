"""numpy's binomial / multinomial draws restated (TEST INFRASTRUCTURE ONLY).

numpy/random/src/distributions/distributions.c: random_binomial chooses
random_binomial_inversion for n * min(p, 1 - p) <= 30 and
random_binomial_btpe (Kachitvichyanukul & Schmeiser) above; random_multinomial
draws sequential binomials of p_j / remaining.  Python floats follow the C
operation order without FMA, so this restatement reproduces numpy's draws
exactly (tests/test_oracle.py checks it against numpy.random.Generator on
Philox streams); the device (csrc/np_random.cuh binomial_btpe) transcribes it.
"""
from __future__ import annotations

import math


def btpe(g, n, p):
    """random_binomial_btpe (p <= 0.5 as random_binomial calls it)."""
    r = min(p, 1.0 - p); q = 1.0 - r
    fm = n * r + r
    m = int(math.floor(fm))
    p1 = math.floor(2.195 * math.sqrt(n * r * q) - 4.6 * q) + 0.5
    xm = m + 0.5; xl = xm - p1; xr = xm + p1
    c = 0.134 + 20.5 / (15.3 + m)
    a = (fm - xl) / (fm - xl * r); laml = a * (1.0 + a / 2.0)
    a = (xr - fm) / (xr * q); lamr = a * (1.0 + a / 2.0)
    p2 = p1 * (1.0 + 2.0 * c); p3 = p2 + c / laml; p4 = p3 + c / lamr
    while True:
        nrq = n * r * q
        u = g.random() * p4
        v = g.random()
        if u <= p1:
            y = int(math.floor(xm - p1 * v + u))
            break
        if u <= p2:
            x = xl + (u - p1) / c
            v = v * c + 1.0 - abs(m - x + 0.5) / p1
            if v > 1.0: continue
            y = int(math.floor(x))
        elif u <= p3:
            if v == 0.0: continue
            y = int(math.floor(xl + math.log(v) / laml))
            if y < 0: continue
            v = v * (u - p2) * laml
        else:
            if v == 0.0: continue
            y = int(math.floor(xr - math.log(v) / lamr))
            if y > n: continue
            v = v * (u - p3) * lamr
        k = abs(y - m)
        if not (k > 20 and k < nrq / 2.0 - 1):
            s = r / q; a = s * (n + 1); F = 1.0
            if m < y:
                for i in range(m + 1, y + 1): F *= (a / i - s)
            elif m > y:
                for i in range(y + 1, m + 1): F /= (a / i - s)
            if v > F: continue
            break
        rho = (k / nrq) * ((k * (k / 3.0 + 0.625) + 0.16666666666666666) / nrq + 0.5)
        t = -k * k / (2 * nrq)
        A = math.log(v) if v > 0 else -math.inf
        if A < t - rho: break
        if A > t + rho: continue
        x1 = y + 1; f1 = m + 1; z = n + 1 - m; w = n - y + 1
        x2 = x1 * x1; f2 = f1 * f1; z2 = z * z; w2 = w * w
        if A > (xm * math.log(f1 / x1) + (n - m + 0.5) * math.log(z / w) + (y - m) * math.log(w * r / (x1 * q))
                + (13680. - (462. - (132. - (99. - 140. / f2) / f2) / f2) / f2) / f1 / 166320.
                + (13680. - (462. - (132. - (99. - 140. / z2) / z2) / z2) / z2) / z / 166320.
                + (13680. - (462. - (132. - (99. - 140. / x2) / x2) / x2) / x2) / x1 / 166320.
                + (13680. - (462. - (132. - (99. - 140. / w2) / w2) / w2) / w2) / w / 166320.):
            continue
        break
    if p > 0.5: y = n - y
    return y

def inversion(g, n, p):
    """random_binomial_inversion."""
    q = 1.0 - p
    qn = math.exp(n * math.log(q))
    np_ = n * p
    bound = int(min(n, np_ + 10.0 * math.sqrt(np_ * q + 1)))
    X = 0; px = qn; U = g.random()
    while U > px:
        X += 1
        if X > bound:
            X = 0; px = qn; U = g.random()
        else:
            U -= px
            px = ((n - X + 1) * p * px) / (X * q)
    return X

def binomial(g, p, n):
    """random_binomial."""
    if n == 0 or p == 0.0: return 0
    if p <= 0.5:
        return inversion(g, n, p) if p * n <= 30.0 else btpe(g, n, p)
    q = 1.0 - p
    return n - (inversion(g, n, q) if q * n <= 30.0 else btpe(g, n, q))

def multinomial3(g, n, pix):
    """random_multinomial for three categories."""
    out = [0, 0, 0]; dn = n; rem = 1.0
    for j in range(2):
        out[j] = binomial(g, pix[j] / rem, dn)
        dn -= out[j]
        if dn <= 0: break
        rem -= pix[j]
    if dn > 0: out[2] = dn
    return out
