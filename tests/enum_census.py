"""Closed-form census of enumerate_outcomes (_core.pyx:778-829), used to check
the GPU enumeration at n = 7, 8 where neither the reference nor the oracle
can enumerate.

A tuple of n ordered cell pairs on n cells passes the reference's
union-find check iff every connected component of its multigraph has as many
edges as nodes, i.e. is connected and unicyclic.  With U_k the number of such
connected structures on k labelled nodes and k labelled edges (each edge an
ordered pair; a loop has one orientation, any other edge two),

  U_k = k! * [ k * F(k,1) * 2^(k-1)                 cycle = loop
             + C(k,2) * F(k,2) * 2^(k-1)            cycle = double edge
             + sum_{c>=3} C(k,c) (c-1)!/2 * F(k,c) * 2^k ]

with F(k,c) = c k^(k-c-1) rooted forests hanging off the cycle (1 if c = k).
Nodes and edges are both labelled, so the census with weight w per
component is  n!^2 [x^n] exp(w * sum_k U_k x^k / k!^2);  w = 1 gives
pf_count, w = 2 gives sum over pseudoforests of 2^components.
"""

from fractions import Fraction
from math import comb, factorial


def _forests(k, c):
    return 1 if c == k else c * k ** (k - c - 1)


def _connected(k):
    tot = k * _forests(k, 1) * 2 ** (k - 1)
    if k >= 2:
        tot += comb(k, 2) * _forests(k, 2) * 2 ** (k - 1)
    for c in range(3, k + 1):
        tot += comb(k, c) * factorial(c - 1) // 2 * _forests(k, c) * 2 ** k
    return factorial(k) * tot


def census(n, w):
    if n <= 0:
        return 1
    a = [Fraction(0)] + [Fraction(w * _connected(k), factorial(k) ** 2) for k in range(1, n + 1)]
    e = [Fraction(1)] + [Fraction(0)] * n
    for m in range(1, n + 1):  # exp of a power series: m e_m = sum_k k a_k e_{m-k}
        e[m] = sum(k * a[k] * e[m - k] for k in range(1, m + 1)) / m
    return int(e[n] * factorial(n) ** 2)
