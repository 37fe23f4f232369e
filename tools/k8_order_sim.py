"""K8 (tiled_colored) claim-order simulator (diagnostics, CPU only).

The persistent kernel hands tile positions out statically: position p goes to
CTA p % G, consumer group (p // G) % 4 of that CTA, and a group runs its
positions in order.  A tile may flush only after all its DAG predecessors
(conflicting tiles of earlier phases) have flushed.  This script builds a
config's schedule, models each tile's duration as its work (nnz + 2 rows),
and reports the makespan of a claim order relative to the perfectly balanced
time, for the phase-major order and the list-scheduled orders of
symmspmv_plan (capi.cpp k8_claim_order).

usage: python tools/k8_order_sim.py st27_128 [lag ...]
"""
import heapq
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_1907_06487_b200 as P  # noqa: E402

G, NG = 148, 4


def simulate(order, work, dag_ptr, dag_pred, wait_before_compute=True):
    nt = len(order)
    finish = np.zeros(nt)
    free = np.zeros((G, NG))
    stall = 0.0
    for p, t in enumerate(order):
        c, g = p % G, (p // G) % NG
        s = free[c, g]
        preds = dag_pred[dag_ptr[t]:dag_ptr[t + 1]]
        ready = finish[preds].max() if len(preds) else 0.0
        if wait_before_compute:
            st = max(s, ready)
            finish[t] = st + work[t]
        else:
            finish[t] = max(s + work[t], ready + 0.05 * work[t])
            st = finish[t] - work[t]
        stall += st - s
        free[c, g] = finish[t]
    return free.max(), stall


def list_order(work, dag_ptr, dag_pred, prio, lag=0.0):
    """Emit tiles in simulated start order: each position takes, among the
    tiles whose predecessors are all emitted, the one with the earliest
    estimated start (predecessors' simulated finish + lag), ties by prio."""
    nt = len(work)
    succ = [[] for _ in range(nt)]
    npred = np.zeros(nt, dtype=np.int64)
    for t in range(nt):
        for q in dag_pred[dag_ptr[t]:dag_ptr[t + 1]]:
            succ[q].append(t)
            npred[t] += 1
    finish = np.zeros(nt)
    ready_at = np.zeros(nt)
    free = np.zeros((G, NG))
    heap = [(0.0, prio[t], t) for t in range(nt) if npred[t] == 0]
    heapq.heapify(heap)
    order = []
    p = 0
    while heap:
        c, g = p % G, (p // G) % NG
        s = free[c, g]
        # earliest-ready tile; among those ready by s, the lowest prio
        cand = []
        while heap and heap[0][0] <= s:
            cand.append(heapq.heappop(heap))
        if cand:
            cand.sort(key=lambda e: e[1])
            pick = cand[0]
            for e in cand[1:]:
                heapq.heappush(heap, e)
        else:
            pick = heapq.heappop(heap)
        t = pick[2]
        st = max(s, pick[0])
        finish[t] = st + work[t]
        free[c, g] = finish[t]
        order.append(t)
        p += 1
        for u in succ[t]:
            ready_at[u] = max(ready_at[u], finish[t] + lag)
            npred[u] -= 1
            if npred[u] == 0:
                heapq.heappush(heap, (ready_at[u], prio[u], u))
    assert len(order) == nt
    return np.array(order)


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "st27_128"
    lags = [float(a) for a in sys.argv[2:]] or [0.0]
    U, _ = gen.make_config(cfg)
    s = P.build_schedule(U)
    rp, _, _ = s.permuted_matrix()
    tp = s.table("tile_ptr")
    phase = s.table("tile_phase")
    dag_ptr, dag_pred = s.table("dag_ptr"), s.table("dag_pred")
    nt = len(phase)
    work = (rp[tp[1:]] - rp[tp[:-1]]) + 2.0 * (tp[1:] - tp[:-1])
    ideal = work.sum() / (G * NG)
    print(f"{cfg}: {nt} tiles, {phase.max() + 1} phases, {len(dag_pred)} DAG edges, ideal {ideal:.0f}")
    pm = np.argsort(phase, kind="stable")
    ms, st = simulate(pm, work, dag_ptr, dag_pred)
    print(f"phase-major   makespan/ideal {ms / ideal:.3f}  stall/ideal {st / ideal / (G * NG):.3f}")
    ms, st = simulate(np.arange(nt), work, dag_ptr, dag_pred) if False else (0, 0)
    mean_w = work.mean()
    for lag in lags:
        o = list_order(work, dag_ptr, dag_pred, np.arange(nt), lag * mean_w)
        ms, st = simulate(o, work, dag_ptr, dag_pred)
        # robustness: durations off by +-30 %
        rng = np.random.default_rng(0)
        w2 = work * rng.uniform(0.7, 1.3, nt)
        ms2, _ = simulate(o, w2, dag_ptr, dag_pred)
        ms3, _ = simulate(pm, w2, dag_ptr, dag_pred)
        pos = np.empty(nt, dtype=np.int64)
        pos[o] = np.arange(nt)
        dist = [pos[t] - pos[q] for t in range(nt) for q in dag_pred[dag_ptr[t]:dag_ptr[t + 1]]]
        print(f"list lag {lag:4.1f}  makespan/ideal {ms / ideal:.3f}  noisy {ms2 / (w2.sum() / G / NG):.3f} "
              f"(phase-major noisy {ms3 / (w2.sum() / G / NG):.3f})  min pred distance {min(dist)}  "
              f"p1 {np.percentile(dist, 1):.0f}")


if __name__ == "__main__":
    main()
