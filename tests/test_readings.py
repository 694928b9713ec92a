"""The readings of garbled pseudocode pinned
on the case SURVEY records: a 200-joint chain of unit x-translations, where Eq. 1 gives
joint i the translation x = i + 1.  Written out here in plain numpy (translations only,
so composition is addition), independent of oracle/ and of the GPU path:

  * Alg. 2 taken literally, MultiParent(j, d) = the d-th ancestor
    for d = 1..log2 n, overcounts (joint 10 -> x = 40); the "pow(2,n) layer parent"
    reading of PAPER.md:139 (hop 2^(d-1), reading R6) gives Eq. 1 exactly.
  * Alg. 3 stage A with unclamped hops double-counts with stage B
    (joint 100 -> x = 128); clamping the hops to the joint's 64-block (reading R8)
    and walking MaxParentOutBlock on the stage-A snapshot (R9) gives Eq. 1.
CPU only."""
from __future__ import annotations

import math

import numpy as np

N = 200
PARENT = np.arange(-1, N - 1)            # chain: parent of j is j - 1


def ancestor(j, k):
    for _ in range(k):
        if j < 0:
            return -1
        j = PARENT[j]
    return j


def doubling(hop):
    """Alg. 2 with snapshot rounds; hop(d) = ancestor distance in round d."""
    x = np.ones(N)                       # every local is T(1, 0, 0)
    for d in range(1, math.ceil(math.log2(N)) + 1):
        prev = x.copy()
        for j in range(N):
            a = ancestor(j, hop(d))
            if a >= 0:
                x[j] = prev[a] + prev[j]
    return x


def blocked(clamp, B=64):
    """Alg. 3: stage A doubling inside the block, stage B MaxParentOutBlock walk."""
    x = np.ones(N)
    for d in range(1, int(math.log2(B)) + 1):
        prev = x.copy()
        for j in range(N):
            a = ancestor(j, 2 ** (d - 1))
            if a >= 0 and (not clamp or a // B == j // B):
                x[j] = prev[a] + prev[j]
    A = x.copy()                         # stage-A snapshot
    out = A.copy()
    for j in range(N):
        m = PARENT[j]
        while m >= 0 and m // B == j // B:
            m = PARENT[m]                # MaxParentOutBlock(j)
        while m >= 0:
            out[j] += A[m]
            mm = PARENT[m]
            while mm >= 0 and mm // B == m // B:
                mm = PARENT[mm]
            m = mm
    return out


def test_alg2_literal_reading_overcounts_and_r6_is_eq1():
    literal = doubling(lambda d: d)
    r6 = doubling(lambda d: 2 ** (d - 1))
    assert literal[10] == 40.0                          # SURVEY §8(c) row 6 scratch value
    assert np.array_equal(r6, np.arange(1, N + 1))      # Eq. 1: x_i = i + 1


def test_alg3_unclamped_double_counts_and_r8_r9_are_eq1():
    unclamped = blocked(clamp=False)
    clamped = blocked(clamp=True)
    assert unclamped[100] == 128.0                      # SURVEY §8(c) row 8 scratch value
    assert np.array_equal(clamped, np.arange(1, N + 1))


def test_alg4_radix8_reading_is_eq1():
    """Reading R10 of Alg. 4: 7 serial in-block composes over the
    ancestors at distances 1..7, then 7 composes with that snapshot at distances 8, 16,
    ..., 56 (14 in all), then the MaxParentOutBlock walk — Eq. 1 on the chain."""
    B = 64

    def inblock(j, k):
        a = ancestor(j, k)
        return a if a >= 0 and a // B == j // B else -1

    ones = np.ones(N)
    a1 = ones.copy()
    for j in range(N):                  # stage A1: serial, distances 1..7
        for k in range(1, 8):
            a = inblock(j, k)
            if a >= 0:
                a1[j] += ones[a]
    A = a1.copy()
    for j in range(N):                  # stage A2: radix-8 strides on the A1 snapshot
        for k in range(8, 64, 8):
            a = inblock(j, k)
            if a >= 0:
                A[j] += a1[a]
    out = A.copy()
    for j in range(N):                  # stage B as Alg. 3
        m = PARENT[j]
        while m >= 0 and m // B == j // B:
            m = PARENT[m]
        while m >= 0:
            out[j] += A[m]
            mm = PARENT[m]
            while mm >= 0 and mm // B == m // B:
                mm = PARENT[mm]
            m = mm
    assert np.array_equal(out, np.arange(1, N + 1))
