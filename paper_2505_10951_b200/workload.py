"""Graph data model and deterministic synthetic workloads (host side).

Mirrors the reference's data model (``graph_store.hpp:28-49``: ``TextualGraph``
with id-keyed node texts and index-identified edges; ``Subgraph`` as sorted node
ids + sorted edge indices) and builds the benchmark workloads named by
``BASELINE.json:configs``:

* C1 -- the reference's own two-star dataset (``tests/support/synth.hpp:22-70``)
  with the ego-topk retrieval result injected (every query retrieves exactly its
  star; pinned against the compiled reference in tests/golden/c1_pipeline.json);
* C2..C5 -- seeded community graphs whose representative unions serialize to the
  target prompt size; retrieved subgraphs are injected at the
  hot-path boundary because retrieval is outside it.

Retrieval, CSV/JSONL ingest and report I/O are out of scope.
"""
from __future__ import annotations

import dataclasses
import os

import numpy as np

GAMMA = 0x9E3779B97F4A7C15
MASK = (1 << 64) - 1


class SplitMix64:
    """rng.hpp:12-34 (used only to make the synthetic workload deterministic)."""

    def __init__(self, seed: int):
        self.state = seed & MASK

    def next(self) -> int:
        self.state = (self.state + GAMMA) & MASK
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
        return z ^ (z >> 31)


def splitmix64_once(x: int) -> int:
    return SplitMix64(x).next()


def csv_quote(field: bytes) -> bytes:
    """graph_store.cpp:237-247: quote only when , " or newline occurs; double quotes."""
    if not any(c in field for c in b',"\n'):
        return field
    return b'"' + field.replace(b'"', b'""') + b'"'


def render_node_row(nid: int, attr: bytes) -> bytes:
    """graph_store.cpp:251-253: std::to_string(id) + ',' + csv_quote(attr)."""
    return b"%d,%s" % (nid, csv_quote(attr))


def render_edge_row(src: int, attr: bytes, dst: int) -> bytes:
    """graph_store.cpp:256-259: src ',' csv_quote(attr) ',' dst."""
    return b"%d,%s,%d" % (src, csv_quote(attr), dst)


@dataclasses.dataclass
class TextualGraph:
    """graph_store.hpp:28-35: nodes id -> attribute bytes; edge identity = index."""

    nodes: dict  # int -> bytes, iterated in ascending id order
    edges: list  # (src, attr bytes, dst)

    def sorted_node_ids(self) -> np.ndarray:
        return np.array(sorted(self.nodes), dtype=np.uint32)

    quote_node_attrs: bool = False  # tests/support/synth.hpp:38-47 quotes every node attribute

    def write_csv(self, node_path: str, edge_path: str) -> None:
        with open(node_path, "wb") as f:
            f.write(b"node id,node attr\n")
            for nid in sorted(self.nodes):
                a = self.nodes[nid]
                q = b'"' + a.replace(b'"', b'""') + b'"' if self.quote_node_attrs else csv_quote(a)
                f.write(b"%d,%s\n" % (nid, q))
        with open(edge_path, "wb") as f:
            f.write(b"src,edge attr,dst\n")
            for s, a, d in self.edges:
                f.write(b"%d,%s,%d\n" % (s, csv_quote(a), d))


@dataclasses.dataclass
class Subgraph:
    """graph_store.hpp:39-49: ascending node ids and ascending edge indices."""

    node_ids: np.ndarray
    edge_indices: np.ndarray

    @staticmethod
    def of(nodes, edges) -> "Subgraph":
        return Subgraph(np.unique(np.asarray(list(nodes), dtype=np.uint32)),
                        np.unique(np.asarray(list(edges), dtype=np.uint32)))

    def to_json(self):
        return {"nodes": [int(x) for x in self.node_ids], "edges": [int(x) for x in self.edge_indices]}


@dataclasses.dataclass
class Query:
    id: int
    question: bytes
    answer: bytes


@dataclasses.dataclass
class Workload:
    name: str
    graph: TextualGraph
    queries: list
    retrieved: list  # Subgraph per query
    lm: dict  # ToyLmConfig fields
    clusters: int
    linkage: str = "ward"
    seed: int = 7
    question_budget: int = 128
    soft_prefix: bool = False
    answer_lookup: bool = True
    # run settings the reference's report echoes (defaults: RetrievalConfig retrieval.hpp:17-25,
    # TextEncoder seed / hash_salt encoders.hpp:17-21)
    retrieval: dict = dataclasses.field(default_factory=lambda: {
        "strategy": "ego-topk", "k": 3, "edge_cost": 0.5, "ego_hops": 2, "ego_entity_cap": 10})
    text_encoder_seed: int = 1
    hash_salt: int = 55
    undirected: bool = True

    def write_dataset(self, d: str):
        os.makedirs(d, exist_ok=True)
        self.graph.write_csv(os.path.join(d, "nodes.csv"), os.path.join(d, "edges.csv"))
        import json

        with open(os.path.join(d, "queries.jsonl"), "w") as f:
            for q in self.queries:
                f.write(json.dumps({"id": q.id, "question": q.question.decode(),
                                    "answer": q.answer.decode()}) + "\n")


# --------------------------------------------------------------------- C1

TINY_LM = dict(layers=4, heads=4, model_dim=64, ffn_hidden=256, max_seq_len=1024, max_new_tokens=32)
LM_1B = dict(layers=16, heads=32, model_dim=2048, ffn_hidden=8192, max_new_tokens=32)
LM_8B = dict(layers=32, heads=32, model_dim=4096, ffn_hidden=14336, max_new_tokens=32)


def two_star_dataset(m: int):
    """tests/support/synth.hpp:22-70 restated: graph + m alternating-topic queries."""
    attrs_a = [b"copper", b"brass", b"steel", b"bronze", b"iron", b"chrome", b"nickel"]
    attrs_b = [b"fern", b"moss", b"ivy", b"rose", b"tulip", b"daisy", b"clover"]
    leaves = len(attrs_a)
    nodes = {0: b"name: engine hub; attribute: central block"}
    for i in range(leaves):
        nodes[1 + i] = b"name: engine part %d; attribute: %s" % (1 + i, attrs_a[i])
    b_base = leaves + 1
    nodes[b_base] = b"name: garden hub; attribute: center bed"
    for i in range(leaves):
        nodes[b_base + 1 + i] = b"name: garden plant %d; attribute: %s" % (8 + i, attrs_b[i])
    edges = [(0, b"engine link", 1 + i) for i in range(leaves)]
    edges += [(b_base, b"garden link", b_base + 1 + i) for i in range(leaves)]
    queries = []
    for j in range(m):
        topic_a = j % 2 == 0
        leaf = (j // 2) % leaves
        q = b"engine part %d?" % (1 + leaf) if topic_a else b"garden plant %d?" % (8 + leaf)
        queries.append(Query(j, q, attrs_a[leaf] if topic_a else attrs_b[leaf]))
    return TextualGraph(nodes, edges), queries


def c1_workload(m: int = 64, clusters: int = 4) -> Workload:
    """BASELINE.json configs[0]: reference default tiny decoder, two-star synth, ego-topk.

    With ego-topk every query retrieves exactly its own star (node 0..7 / edges 0..6
    for the engine topic, nodes 8..15 / edges 7..13 for the garden topic); the
    golden fixture pins this against the reference's retrieve()."""
    g, qs = two_star_dataset(m)
    g.quote_node_attrs = True  # byte-identical to the reference's writer (dataset digest)
    stars = [Subgraph.of(range(0, 8), range(0, 7)), Subgraph.of(range(8, 16), range(7, 14))]
    return Workload("c1-tiny-twostar", g, qs, [stars[j % 2] for j in range(m)], dict(TINY_LM),
                    clusters, seed=7)


# ------------------------------------------------------------------ C2..C5

_WORDS = [b"copper", b"brass", b"steel", b"bronze", b"iron", b"chrome", b"nickel", b"zinc",
          b"fern", b"moss", b"ivy", b"rose", b"tulip", b"daisy", b"clover", b"lily",
          b"amber", b"azure", b"coral", b"ivory", b"jade", b"onyx", b"pearl", b"ruby",
          b"north", b"south", b"east", b"west", b"upper", b"lower", b"inner", b"outer",
          b"rapid", b"quiet", b"heavy", b"light", b"sharp", b"round", b"solid", b"hollow",
          b"valve", b"gear", b"spring", b"lever", b"panel", b"frame", b"cable", b"pump"]
_VERBS = [b"connected to", b"part of", b"located near", b"feeds into", b"controls",
          b"supports", b"made with", b"adjacent to"]


def community_workload(name: str, lm: dict, m: int, communities: int, nodes_per_comm: int,
                       edges_per_comm: int, slice_min: int, slice_max: int, clusters: int,
                       seed: int = 20250510) -> Workload:
    """Seeded community graph.

    Each community is a ring of `nodes_per_comm` entities plus seeded chords; node
    text is ``name: entity N; attribute: W1 W2`` and edge text a relation verb.
    Query j belongs to community j % communities; its retrieved subgraph is a BFS
    slice of its community grown from a Zipf-weighted start entity (so queries of one
    topic overlap), closed under induced edges. The question asks for the attribute of
    an entity of the slice so the copy pointer can fire."""
    rng = SplitMix64(seed)
    nodes, edges = {}, []
    comm_nodes, comm_adj = [], []
    nid = 0
    for c in range(communities):
        ids = list(range(nid, nid + nodes_per_comm))
        nid += nodes_per_comm
        for i in ids:
            w1 = _WORDS[rng.next() % len(_WORDS)]
            w2 = _WORDS[rng.next() % len(_WORDS)]
            nodes[i] = b"name: entity %d; attribute: %s %s" % (i, w1, w2)
        adj = {i: [] for i in ids}
        pairs = set()
        for k in range(nodes_per_comm):
            pairs.add((ids[k], ids[(k + 1) % nodes_per_comm]))
        while len(pairs) < edges_per_comm:
            a = ids[rng.next() % nodes_per_comm]
            b = ids[rng.next() % nodes_per_comm]
            if a != b and (a, b) not in pairs and (b, a) not in pairs:
                pairs.add((a, b))
        for a, b in sorted(pairs, key=lambda p: (p[0], p[1])):
            ei = len(edges)
            edges.append((a, _VERBS[rng.next() % len(_VERBS)], b))
            adj[a].append((b, ei))
            adj[b].append((a, ei))
        comm_nodes.append(ids)
        comm_adj.append(adj)
    g = TextualGraph(nodes, edges)
    # Zipf weights over start entities within a community
    zipf = np.array([1.0 / (k + 1) for k in range(nodes_per_comm)])
    zipf_cdf = np.cumsum(zipf) / zipf.sum()
    queries, retrieved = [], []
    for j in range(m):
        c = j % communities
        ids, adj = comm_nodes[c], comm_adj[c]
        u = (rng.next() >> 11) * (1.0 / (1 << 53))
        start = ids[int(np.searchsorted(zipf_cdf, u))]
        want = slice_min + rng.next() % (slice_max - slice_min + 1)
        sel, frontier = {start}, [start]
        while frontier and len(sel) < want:
            nxt = []
            for v in frontier:
                for w, _ in sorted(adj[v]):
                    if w not in sel and len(sel) < want:
                        sel.add(w)
                        nxt.append(w)
            frontier = nxt
        sel_edges = [ei for ei, (a, _, b) in enumerate(edges) if a in sel and b in sel]
        sub = Subgraph.of(sel, sel_edges)
        target = int(sub.node_ids[rng.next() % len(sub.node_ids)])
        attr = nodes[target].split(b"attribute: ")[1].split(b" ")[0]
        queries.append(Query(j, b"which attribute has entity %d?" % target, attr))
        retrieved.append(sub)
    return Workload(name, g, queries, retrieved, dict(lm), clusters)


def prompt_tokens_estimate(graph: TextualGraph, sub: Subgraph) -> int:
    """86 + sum(node row + 1) + sum(edge row + 1)."""
    n = 86
    for i in sub.node_ids:
        n += len(render_node_row(int(i), graph.nodes[int(i)])) + 1
    for e in sub.edge_indices:
        s, a, d = graph.edges[int(e)]
        n += len(render_edge_row(s, a, d)) + 1
    return n


def c2_workload(m: int = 256) -> Workload:
    """configs[1]: Llama-3.2-1B-shaped, 256 queries, ~1k-token subgraph prompts, 1 GPU."""
    w = community_workload("c2-1b-256q", LM_1B, m, communities=8, nodes_per_comm=17,
                           edges_per_comm=17, slice_min=8, slice_max=13, clusters=8)
    w.lm["max_seq_len"] = 1024 + 160
    return w


def c3_workload(m: int = 1024, clusters: int = 16) -> Workload:
    """configs[2]: Llama-3-8B-shaped, 1024 queries, 16 clusters, ~2k-token prompts."""
    w = community_workload("c3-8b-1024q", LM_8B, m, communities=16, nodes_per_comm=33,
                           edges_per_comm=36, slice_min=14, slice_max=22, clusters=clusters)
    w.lm["max_seq_len"] = 2304
    return w


def c4_workload(m: int = 4096, clusters: int = 64) -> Workload:
    """configs[3]: 8B-shaped, 4096 queries, cluster-count sweep 8..256."""
    w = community_workload("c4-8b-4096q", LM_8B, m, communities=64, nodes_per_comm=33,
                           edges_per_comm=36, slice_min=14, slice_max=22, clusters=clusters)
    w.lm["max_seq_len"] = 2304
    return w


def c5_workload(m: int = 2048, clusters: int = 16) -> Workload:
    """configs[4]: 8B-shaped, 8k-token representatives, 2048 queries."""
    w = community_workload("c5-8b-2048q", LM_8B, m, communities=16, nodes_per_comm=130,
                           edges_per_comm=150, slice_min=50, slice_max=80, clusters=clusters)
    w.lm["max_seq_len"] = 8448
    return w


WORKLOADS = {"c1": c1_workload, "c2": c2_workload, "c3": c3_workload, "c4": c4_workload,
             "c5": c5_workload}
