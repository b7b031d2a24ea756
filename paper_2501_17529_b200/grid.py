"""Grid input contract: nodes, branches, injections, splittable substations, cases.

This is the host-side mirror of the reference's immutable grid model
(`pkg/src/batchdc/grid.py:26-297`) and of the node partition used to fold
static injections into one PTDF column (`grid.py:383-434`).  Objects refer to
each other by dense integer index (file order); string ids are only used for
reports.  Nothing here is per-topology work: the grid is built and validated
once per session and then flattened into device tables by ``ptdf.py``.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import cached_property
from typing import Iterable, Optional, Sequence

import numpy as np

from .errors import ValidationError

SINGLE_BRANCH = "single_branch"
MULTI_BRANCH = "multi_branch"
INJECTION = "injection"
CASE_KINDS = (SINGLE_BRANCH, MULTI_BRANCH, INJECTION)


@dataclass(frozen=True)
class Branch:
    """Directed branch; positive flow runs from ``from_node`` to ``to_node``."""

    id: str
    from_node: int
    to_node: int
    susceptance: float
    rating: float
    monitored: bool = True


@dataclass(frozen=True)
class Injection:
    """Nodal injection in MW (generation > 0, load < 0)."""

    id: str
    node: int
    setpoint: float


@dataclass(frozen=True)
class SplittableSubstation:
    """A node whose busbar may be split; element order defines the bit order."""

    node: int
    branch_elements: tuple[int, ...]
    injection_elements: tuple[int, ...] = ()


@dataclass(frozen=True)
class ContingencyCase:
    """One N-1 case: a branch, a set of branches, or an injection."""

    id: str
    kind: str
    branches: tuple[int, ...] = ()
    injection: Optional[int] = None


def _components(n: int, pairs: Iterable[tuple[int, int]]) -> int:
    parent = list(range(n))
    count = n

    def root(x: int) -> int:
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    for a, b in pairs:
        ra, rb = root(a), root(b)
        if ra != rb:
            parent[ra] = rb
            count -= 1
    return count


@dataclass(frozen=True)
class Grid:
    """Validated, immutable grid snapshot with a fixed slack node."""

    node_ids: tuple[str, ...]
    branches: tuple[Branch, ...]
    injections: tuple[Injection, ...]
    slack: int
    substations: tuple[SplittableSubstation, ...] = ()
    contingencies: tuple[ContingencyCase, ...] = ()

    # -- sizes ---------------------------------------------------------------
    @property
    def n_nodes(self) -> int:
        return len(self.node_ids)

    @property
    def n_branches(self) -> int:
        return len(self.branches)

    # -- column views (cached; the dataclass is frozen) ----------------------
    @cached_property
    def from_nodes(self) -> np.ndarray:
        return np.fromiter((b.from_node for b in self.branches), np.int64, self.n_branches)

    @cached_property
    def to_nodes(self) -> np.ndarray:
        return np.fromiter((b.to_node for b in self.branches), np.int64, self.n_branches)

    @cached_property
    def susceptances(self) -> np.ndarray:
        return np.fromiter((b.susceptance for b in self.branches), np.float64, self.n_branches)

    @cached_property
    def ratings(self) -> np.ndarray:
        return np.fromiter((b.rating for b in self.branches), np.float64, self.n_branches)

    @cached_property
    def monitored(self) -> tuple[int, ...]:
        return tuple(k for k, b in enumerate(self.branches) if b.monitored)

    @cached_property
    def node_index(self) -> dict[str, int]:
        return {nid: i for i, nid in enumerate(self.node_ids)}

    @cached_property
    def branch_index(self) -> dict[str, int]:
        return {b.id: k for k, b in enumerate(self.branches)}

    @cached_property
    def injection_index(self) -> dict[str, int]:
        return {inj.id: j for j, inj in enumerate(self.injections)}

    @cached_property
    def injection_slots(self) -> tuple[tuple[int, int], ...]:
        """(substation index, injection index) per reassignable slot.

        Substation order, then each substation's element order; one candidate
        bit per slot (`grid.py:145-157`).
        """
        return tuple(
            (si, j) for si, sub in enumerate(self.substations) for j in sub.injection_elements
        )

    def movable_injections(self) -> frozenset[int]:
        """Slot injections plus injections named by an injection case (`grid.py:159-172`)."""
        out = {j for sub in self.substations for j in sub.injection_elements}
        out.update(c.injection for c in self.contingencies if c.kind == INJECTION)
        return frozenset(out)

    def nodal_power(self) -> np.ndarray:
        p = np.zeros(self.n_nodes)
        for inj in self.injections:
            p[inj.node] += inj.setpoint
        return p

    def connected_components(self, dead_branches: Iterable[int] = ()) -> int:
        dead = frozenset(dead_branches)
        return _components(
            self.n_nodes,
            ((b.from_node, b.to_node) for k, b in enumerate(self.branches) if k not in dead),
        )

    # -- validation (`grid.py:191-276`) --------------------------------------
    def validate(self) -> None:
        n = self.n_nodes
        if n == 0:
            raise ValidationError("grid has no nodes")
        if len(set(self.node_ids)) != n:
            raise ValidationError("duplicate node ids")
        if len({b.id for b in self.branches}) != self.n_branches:
            raise ValidationError("duplicate branch ids")
        if len({i.id for i in self.injections}) != len(self.injections):
            raise ValidationError("duplicate injection ids")
        if not 0 <= self.slack < n:
            raise ValidationError(f"slack index {self.slack} out of range")
        for b in self.branches:
            if not (0 <= b.from_node < n and 0 <= b.to_node < n):
                raise ValidationError(f"branch {b.id}: endpoint out of range")
            if b.from_node == b.to_node:
                raise ValidationError(f"branch {b.id}: self-loop")
            if not b.susceptance > 0.0:
                raise ValidationError(f"branch {b.id}: susceptance must be > 0")
            if not b.rating > 0.0:
                raise ValidationError(f"branch {b.id}: rating must be > 0")
        for inj in self.injections:
            if not 0 <= inj.node < n:
                raise ValidationError(f"injection {inj.id}: node out of range")
        sub_nodes = set()
        for si, sub in enumerate(self.substations):
            if not 0 <= sub.node < n:
                raise ValidationError(f"substation #{si}: node out of range")
            if sub.node in sub_nodes:
                raise ValidationError(
                    f"substation #{si}: node {self.node_ids[sub.node]} listed twice"
                )
            sub_nodes.add(sub.node)
            if len(set(sub.branch_elements)) != len(sub.branch_elements):
                raise ValidationError(f"substation #{si}: duplicate branch element")
            for k in sub.branch_elements:
                if not 0 <= k < self.n_branches:
                    raise ValidationError(f"substation #{si}: branch element out of range")
                b = self.branches[k]
                if sub.node not in (b.from_node, b.to_node):
                    raise ValidationError(
                        f"substation #{si}: branch {b.id} not incident on its node"
                    )
            if len(set(sub.injection_elements)) != len(sub.injection_elements):
                raise ValidationError(f"substation #{si}: duplicate injection element")
            for j in sub.injection_elements:
                if not 0 <= j < len(self.injections):
                    raise ValidationError(f"substation #{si}: injection element out of range")
                if self.injections[j].node != sub.node:
                    raise ValidationError(
                        f"substation #{si}: injection {self.injections[j].id} "
                        "not located at its node"
                    )
        case_ids = set()
        for case in self.contingencies:
            if case.id in case_ids:
                raise ValidationError(f"duplicate contingency id {case.id}")
            case_ids.add(case.id)
            if case.kind not in CASE_KINDS:
                raise ValidationError(f"contingency {case.id}: unknown kind {case.kind!r}")
            if case.kind == SINGLE_BRANCH and len(case.branches) != 1:
                raise ValidationError(
                    f"contingency {case.id}: single_branch needs exactly one branch"
                )
            if case.kind == MULTI_BRANCH:
                if len(case.branches) < 2:
                    raise ValidationError(
                        f"contingency {case.id}: multi_branch needs at least two branches"
                    )
                if len(set(case.branches)) != len(case.branches):
                    raise ValidationError(f"contingency {case.id}: duplicate branch")
            if case.kind == INJECTION:
                if case.branches:
                    raise ValidationError(f"contingency {case.id}: unexpected branches field")
                if case.injection is None or not 0 <= case.injection < len(self.injections):
                    raise ValidationError(f"contingency {case.id}: injection out of range")
            else:
                if case.injection is not None:
                    raise ValidationError(f"contingency {case.id}: unexpected injection field")
                for k in case.branches:
                    if not 0 <= k < self.n_branches:
                        raise ValidationError(f"contingency {case.id}: branch out of range")
        if self.connected_components() != 1:
            raise ValidationError("grid is not connected")


def build_grid(
    node_ids: Sequence[str],
    branches: Sequence[Branch],
    injections: Sequence[Injection],
    slack: int,
    substations: Sequence[SplittableSubstation] = (),
    contingencies: Sequence[ContingencyCase] = (),
) -> Grid:
    grid = Grid(
        node_ids=tuple(node_ids),
        branches=tuple(branches),
        injections=tuple(injections),
        slack=int(slack),
        substations=tuple(substations),
        contingencies=tuple(contingencies),
    )
    grid.validate()
    return grid


def structurally_required_nodes(grid: Grid) -> frozenset[int]:
    """Nodes whose PTDF column an update or an outage delta may read (`grid.py:383-403`).

    Slack; every substation node and the far end of each of its branch
    elements; both ends of every contingency branch; the node of every
    injection named by an injection case.
    """
    req = {grid.slack}
    for sub in grid.substations:
        req.add(sub.node)
        for k in sub.branch_elements:
            b = grid.branches[k]
            req.add(b.to_node if b.from_node == sub.node else b.from_node)
    for case in grid.contingencies:
        for k in case.branches:
            req.add(grid.branches[k].from_node)
            req.add(grid.branches[k].to_node)
        if case.injection is not None:
            req.add(grid.injections[case.injection].node)
    return frozenset(req)


@dataclass(frozen=True)
class StaticFold:
    """Node partition: ``static_nodes`` collapse into one PTDF column (`grid.py:367-380`)."""

    static_nodes: tuple[int, ...]
    effective_nodes: tuple[int, ...]
    static_power: np.ndarray


def static_injection_fold(grid: Grid, movable: Optional[Iterable[int]] = None) -> StaticFold:
    """Partition nodes into foldable static ones and effective ones (`grid.py:406-434`)."""
    mov = set(grid.movable_injections())
    if movable is not None:
        mov.update(movable)
    required = set(structurally_required_nodes(grid))
    required.update(grid.injections[j].node for j in mov)
    power = np.zeros(grid.n_nodes)
    for j, inj in enumerate(grid.injections):
        if j not in mov:
            power[inj.node] += inj.setpoint
    effective = tuple(sorted(required))
    static = tuple(i for i in range(grid.n_nodes) if i not in required)
    return StaticFold(static_nodes=static, effective_nodes=effective, static_power=power)


# -- stub-branch replacement ------------------------------------
def branch_bridges(grid: Grid) -> frozenset[int]:
    """Branches whose removal disconnects the grid (`Grid.bridges`, grid.py:183-189).

    Tarjan's low-link over branch ids, iteratively: the DFS skips only the branch it
    arrived by (not every branch back to the parent node), so a node pair joined by
    parallel branches is never a bridge."""
    n = grid.n_nodes
    adj: list[list[tuple[int, int]]] = [[] for _ in range(n)]
    for k, b in enumerate(grid.branches):
        adj[b.from_node].append((b.to_node, k))
        adj[b.to_node].append((b.from_node, k))
    order = [-1] * n
    low = [0] * n
    out: set[int] = set()
    clock = 0
    for root in range(n):
        if order[root] >= 0:
            continue
        order[root] = low[root] = clock
        clock += 1
        stack = [(root, -1, 0)]  # (node, branch it was entered by, next adjacency index)
        while stack:
            v, via, i = stack[-1]
            if i < len(adj[v]):
                stack[-1] = (v, via, i + 1)
                w, k = adj[v][i]
                if k == via:
                    continue
                if order[w] < 0:
                    order[w] = low[w] = clock
                    clock += 1
                    stack.append((w, k, 0))
                else:
                    low[v] = min(low[v], order[w])
            else:
                stack.pop()
                if stack:
                    u = stack[-1][0]
                    low[u] = min(low[u], low[v])
                    if low[v] > order[u]:
                        out.add(via)
    return frozenset(out)


def _find_stub(grid: Grid):
    """The first removable appendage in (substation, incident branch) order, or None: a
    bridge at a substation node, not named by a contingency, whose far side holds no
    slack, no substation node and no contingency branch (grid.py:461-478)."""
    bridges = branch_bridges(grid)
    named = {k for c in grid.contingencies for k in c.branches}
    sub_nodes = {s.node for s in grid.substations}
    adj: dict[int, list[tuple[int, int]]] = {}
    for k, b in enumerate(grid.branches):
        adj.setdefault(b.from_node, []).append((b.to_node, k))
        adj.setdefault(b.to_node, []).append((b.from_node, k))
    for si, sub in enumerate(grid.substations):
        for k, b in enumerate(grid.branches):
            if sub.node not in (b.from_node, b.to_node) or k not in bridges or k in named:
                continue
            far = b.to_node if b.from_node == sub.node else b.from_node
            nodes, branches = {far}, set()
            todo = [far]
            while todo:  # everything reachable from the far end without crossing k
                v = todo.pop()
                for w, j in adj.get(v, ()):
                    if j == k:
                        continue
                    branches.add(j)
                    if w not in nodes:
                        nodes.add(w)
                        todo.append(w)
            if grid.slack in nodes or nodes & sub_nodes or branches & named:
                continue
            return si, nodes, branches | {k}
    return None


def _carve_stub(grid: Grid, si: int, dead_nodes: set, dead_branches: set) -> Grid:
    """The grid without one appendage; its injections move to the substation node and
    join the substation's reassignable elements (grid.py:500-560)."""
    from dataclasses import replace

    hub = grid.substations[si].node
    keep_nodes = [v for v in range(grid.n_nodes) if v not in dead_nodes]
    nmap = {v: i for i, v in enumerate(keep_nodes)}
    keep_br = [k for k in range(grid.n_branches) if k not in dead_branches]
    bmap = {k: i for i, k in enumerate(keep_br)}
    moved = [j for j, inj in enumerate(grid.injections) if inj.node in dead_nodes]
    injections = tuple(
        replace(inj, node=nmap[hub] if inj.node in dead_nodes else nmap[inj.node]) for inj in grid.injections
    )
    subs = []
    for i, s in enumerate(grid.substations):
        elems = list(s.injection_elements)
        if i == si:
            elems += [j for j in moved if j not in elems]
        subs.append(SplittableSubstation(
            node=nmap[s.node],
            branch_elements=tuple(bmap[k] for k in s.branch_elements if k in bmap),
            injection_elements=tuple(elems),
        ))
    return Grid(
        node_ids=tuple(grid.node_ids[v] for v in keep_nodes),
        branches=tuple(replace(grid.branches[k], from_node=nmap[grid.branches[k].from_node],
                               to_node=nmap[grid.branches[k].to_node]) for k in keep_br),
        injections=injections,
        slack=nmap[grid.slack],
        substations=tuple(subs),
        contingencies=tuple(replace(c, branches=tuple(bmap[k] for k in c.branches)) for c in grid.contingencies),
    )


def replace_stub_branches(grid: Grid) -> Grid:
    """Remove radial appendages hanging off substation nodes, to convergence
    (`batchdc.grid.replace_stub_branches`, grid.py:437-458): each one's injections are
    re-homed to the substation (raising the candidate count |T_i|) and
    its branches leave the grid, monitored or not.  Returns a new validated Grid."""
    current = grid
    while True:
        stub = _find_stub(current)
        if stub is None:
            current.validate()
            return current
        current = _carve_stub(current, *stub)
