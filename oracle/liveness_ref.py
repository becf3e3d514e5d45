"""Independent recount of the reference peak — test infrastructure only.

Interval-overlap counting, restated from the reference test oracle
(/root/reference/pkg/tests/test_repo.py:42-59): at every topo position t,
sum the sizes of tensors whose [pos, last] range contains t, plus the
external input while t <= pos(entry).  Quadratic on purpose (no sweep).
"""

from __future__ import annotations

from paper_2410_21120_b200.graph_ir import topo_order


def peak_by_overlap(g, shapes) -> int:
    order = topo_order(g)
    pos = {nid: i for i, nid in enumerate(order)}
    last = {nid: pos[nid] for nid in order}
    for nid, node in g.nodes.items():
        for src in node.inputs:
            last[src] = max(last[src], pos[nid])
    last[g.exit] = len(order)
    peak = 0
    for t in range(len(order)):
        live = g.input_spec.byte_size if t <= pos[g.entry] else 0
        for nid in order:
            if pos[nid] <= t <= last[nid]:
                live += shapes[nid].byte_size
        peak = max(peak, live)
    return peak
