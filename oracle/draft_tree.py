"""Plain CPU reference of the draft worker's tree logic.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Shares no code with the
product's C++ tree (paper_2506_11309_b200/csrc/draft_tree.h); the CPU tests
drive both with the same synthetic draft outputs and compare every decision.

What it follows (P:n = PAPER.md line n):
  * Alg. 1 draft branch: expand the w most probable leaves d times,
    get the verified tokens, update the tree, grow until the tree has bs nodes,
    send "the most probable subgraph of size bs".
  * Maximum-likelihood expansion: a node's value is the log of its
    softmax probability, its weight the sum of values from the root; the
    most probable leaves are the largest weights.
  * Re-root and KV reorganisation: walk down the tree with the
    verified tokens, move the verified nodes' K/V into the prefix cache, keep
    the K/V of the new root's subtree right after it, discard the rest.
Readings: ties between equal weights go to the earlier-created
node (R25); a node's children are its draft's top-K tokens, K = w (R26);
verified tokens whose draft K/V was never computed stay in the tree as a
certain (weight 0) chain above the target's root and are committed once
computed (R27).
"""
from __future__ import annotations


class DraftTreeRef:
    """Nodes are dicts {token, parent, weight, slot}; ids are creation order."""

    def __init__(self, root_token: int, max_slots: int = 64):
        self.max_slots = max_slots
        self.nodes = [dict(token=int(root_token), parent=-1, weight=0.0, slot=-1)]
        self.n_slots = 0
        self.troot = 0

    # -- helpers
    def ancestors_or_self(self, n):
        out = []
        while n != -1:
            out.append(n)
            n = self.nodes[n]["parent"]
        return out

    def subtree(self, r):
        return [i for i in range(len(self.nodes)) if r in self.ancestors_or_self(i)]

    def rank_key(self, i):
        # "most probable" first; equal weights: earlier node first (R25)
        return (-self.nodes[i]["weight"], i)

    # -- Alg. 1 steps
    def tree_size(self):
        return len(self.subtree(self.troot))

    def select(self, w):
        leaves = [i for i in range(len(self.nodes)) if self.nodes[i]["slot"] == -1]
        leaves.sort(key=self.rank_key)
        room = self.max_slots - self.n_slots
        return sorted(leaves[:max(0, min(w, room))])

    def forward_inputs(self, sel):
        toks, pars = [], []
        for i, n in enumerate(sel):
            toks.append(self.nodes[n]["token"])
            p = self.nodes[n]["parent"]
            if p == -1:
                pars.append(-1)
            elif self.nodes[p]["slot"] >= 0:
                pars.append(self.nodes[p]["slot"])
            else:
                pars.append(self.n_slots + sel.index(p))
        return toks, pars

    def computed(self, sel):
        for n in sel:
            self.nodes[n]["slot"] = self.n_slots
            self.n_slots += 1

    def add_children(self, node, toks, logps):
        for t, lp in zip(toks, logps):
            self.nodes.append(dict(token=int(t), parent=node, weight=self.nodes[node]["weight"] + float(lp), slot=-1))

    def subgraph(self, bs):
        cand = self.subtree(self.troot)
        cand.sort(key=self.rank_key)
        chosen = sorted(cand[:bs])
        toks = [self.nodes[n]["token"] for n in chosen]
        pars = [-1 if k == 0 else chosen.index(self.nodes[n]["parent"]) for k, n in enumerate(chosen)]
        return toks, pars, chosen

    def reroot(self, path, bonus):
        """path: node ids [troot, d1 .. dk] the target accepted; bonus: its sampled
        token.  Returns (commit_slots, keep_slots, n_committed)."""
        S = self.ancestors_or_self(path[0])[::-1] + list(path[1:])
        p = 0
        while p < len(S) and self.nodes[S[p]]["slot"] >= 0:
            p += 1
        commit_slots = [self.nodes[n]["slot"] for n in S[:p]]
        last = S[-1]
        e = None
        for i in range(len(self.nodes)):
            if self.nodes[i]["parent"] == last and self.nodes[i]["token"] == int(bonus):
                e = i
                break
        if e is None:
            self.nodes.append(dict(token=int(bonus), parent=last, weight=self.nodes[last]["weight"], slot=-1))
            e = len(self.nodes) - 1
        new_root = S[p] if p < len(S) else e
        keep = self.subtree(new_root)
        under_e = set(self.subtree(e))
        we = self.nodes[e]["weight"]
        computed = sorted([n for n in keep if self.nodes[n]["slot"] >= 0], key=lambda n: self.nodes[n]["slot"])
        keep_slots = [self.nodes[n]["slot"] for n in computed]
        new_id = {n: k for k, n in enumerate(keep)}
        nodes = []
        for n in keep:
            nd = self.nodes[n]
            nodes.append(dict(token=nd["token"],
                              parent=-1 if n == new_root else new_id[nd["parent"]],
                              weight=(nd["weight"] - we) if n in under_e else 0.0,
                              slot=computed.index(n) if n in computed else -1))
        self.nodes = nodes
        self.troot = new_id[e]
        self.n_slots = len(computed)
        return commit_slots, keep_slots, p
