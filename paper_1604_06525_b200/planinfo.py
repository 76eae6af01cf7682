"""Plan introspection for roofline accounting.

Algorithmic bytes of one kernel launch = the unique footprint of the
reference's compiled per-element program: every distinct (field kind, field,
channel) the program loads, once per element, + the uint8 exclusion mask
(solver.hpp:619) + every output, once per element.  Halo re-reads do not
count.  Graph programs add the int32 vertex indices per edge.
"""
from dataclasses import dataclass, field
from typing import Dict, List, Tuple

LOAD_OPS = {3: "U", 4: "A", 5: "C", 6: "P"}  # program.hpp:21-39 kLoadU/A/C/P


@dataclass
class ProgramInfo:
    name: str
    n_instrs: int
    n_outputs: int
    loads: List[Tuple[str, int, int]] = field(default_factory=list)  # distinct (kind, field, channel)
    n_arith: int = 0


@dataclass
class PlanInfo:
    dims: Dict[str, int]
    fields: Dict[str, list]  # kind -> [(name, channels, dims)]
    sections: List[Tuple[str, Dict[str, ProgramInfo]]]  # (section header, programs)


def parse(text: str) -> PlanInfo:
    lines = text.splitlines()
    dims, fields, sections = {}, {"U": [], "A": [], "C": []}, []
    i = 0
    cur = None
    while i < len(lines):
        t = lines[i].split()
        i += 1
        if not t:
            continue
        if t[0] == "dim":
            dims[t[1]] = int(t[2])
        elif t[0] == "unknown":
            fields["U"].append((t[1], int(t[2]), [int(v) for v in t[4:4 + int(t[3])]]))
        elif t[0] == "array":
            fields["A"].append((t[1], int(t[2]), [int(v) for v in t[4:4 + int(t[3])]]))
        elif t[0] == "computed" and len(t) > 3:
            fields["C"].append((t[1], int(t[3]), [int(v) for v in t[5:5 + int(t[4])]]))
        elif t[0] in ("grid_set", "gather_set", "graph_set", "computed_kernel", "exclude_kernel"):
            cur = {}
            sections.append((lines[i - 1], cur))
        elif t[0] == "program":
            name, ni = t[1], int(t[3])
            no = int(t[6])
            loads, arith = set(), 0
            for k in range(ni):
                f = lines[i + k].split()
                op = int(f[1])
                if op in LOAD_OPS:
                    loads.add((LOAD_OPS[op], int(f[8]), int(f[9])))
                elif op in (8, 9, 10, 11):
                    arith += 1
            i += ni
            cur[name] = ProgramInfo(name, ni, no, sorted(loads), arith)
    return PlanInfo(dims, fields, sections)


def algorithmic_bytes_per_element(info: PlanInfo, section_kind: str, program: str, real_bytes: int,
                                  mask: bool = True) -> int:
    """Unique-footprint bytes per element of the first `section_kind` set's program."""
    for hdr, progs in info.sections:
        if hdr.startswith(section_kind) and program in progs:
            p = progs[program]
            n = len(p.loads) * real_bytes + p.n_outputs * real_bytes
            return n + (1 if mask else 0)
    raise KeyError(f"{section_kind}/{program} not in plan")


def graph_bytes_per_launch(info: PlanInfo, program: str, real_bytes: int, n_vertices: int, n_edges: int,
                           arity: int) -> int:
    """Unique footprint of one launch of a plan whose `program` (jtj / bm) has
    a grid gather part and a graph scatter part on the same vertex domain
    (SURVEY §8d ARAP mesh: 76 B/vertex + 8 B/edge for J^T J p): every distinct
    (kind, field, channel) either part loads, once per vertex, + the per-vertex
    outputs (+ the uint8 mask if the plan has exclusion kernels) + the int32
    vertex ids of every edge."""
    loads, outs, mask = set(), 0, False
    for hdr, progs in info.sections:
        if program in progs and (hdr.startswith("gather_set") or hdr.startswith("graph_set")):
            loads.update(progs[program].loads)
            if hdr.startswith("gather_set"):
                outs = max(outs, progs[program].n_outputs)
        if hdr.startswith("exclude_kernel"):
            mask = True
    per_v = len(loads) * real_bytes + outs * real_bytes + (1 if mask else 0)
    return per_v * n_vertices + arity * 4 * n_edges
