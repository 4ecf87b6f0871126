"""Median per-step timeline of the tensor-core dense kernel from an OSCB_UMMA_TRACE=<csv> run (SM clocks -> microseconds)."""
import csv
import sys

import numpy as np

path, mhz = sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1965.0
rows = list(csv.DictReader(open(path)))
names = [k for k in rows[0] if k not in ("cta", "pass")]
C = max(int(r["cta"]) for r in rows) + 1
P = max(int(r["pass"]) for r in rows) + 1
T = {k: np.zeros((C, P)) for k in names}
for r in rows:
    for k in names:
        T[k][int(r["cta"]), int(r["pass"])] = int(r[k])
lo, hi = 5, P - 5
q, q1 = slice(lo, hi), slice(lo + 1, hi + 1)
us = lambda x: float(np.median(x)) / mhz
print("step period                         %.2f us" % us(T["arrived"][:, q1] - T["arrived"][:, q]))
print("barrier seen -> accumulator full    %.2f us" % us(T["tmem_full"][:, q] - T["barrier_seen"][:, q]))
print("accumulator full -> TMEM read       %.2f us" % us(T["tmem_loaded"][:, q] - T["tmem_full"][:, q]))
print("TMEM read -> update + digits done   %.2f us" % us(T["updated"][:, q] - T["tmem_loaded"][:, q]))
print("digits -> B bytes stored            %.2f us" % us(T["stored"][:, q] - T["updated"][:, q]))
print("stored -> CTA barrier passed        %.2f us" % us(T["cta_synced"][:, q] - T["stored"][:, q]))
print("CTA barrier -> fence + arrive       %.2f us" % us(T["arrived"][:, q] - T["cta_synced"][:, q]))
print("arrive -> next barrier seen         %.2f us" % us(T["barrier_seen"][:, q1] - T["arrived"][:, q]))
print("producer parked at the barrier      %.2f us" % us(T["barrier_seen"][:, q] - T["barrier_wait_begin"][:, q]))
