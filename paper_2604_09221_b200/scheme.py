"""Rooted nesting trees, their canonical Rohlin-Viro string, and tree keys.

The canonical string is the reference's definition (scheme.py:44-64): at
every node the unnested ovals come first as one count, then the nested
children grouped by identical interior string, groups ordered by the byte
order of that interior string, each group rendered ``k<X>`` and joined by
``" u "``; the root renders ``<J>`` / ``<J u ...>`` in odd degree and
``<0>`` / ``<...>`` in even degree.

The device never builds strings.  It emits a **tree key**: the AHU
canonical balanced-parenthesis code of the region tree, prefixed by a
sentinel 1 bit, in a ``uint64``.  For a node, ``code = "1" + sorted child
codes + "0"``; children are sorted by their own sentinel keys as integers
(length first, then value), which is an isomorphism invariant, so the key
is injective on rooted-tree classes.  The root contributes only its child
sequence, so ``key = 1 << 2*(nreg-1) | bits`` and ``ovals = nreg - 1 =
(key.bit_length() - 1) / 2``.  :func:`scheme_from_key` decodes the key and
renders the reference string; it is memoised because a whole sweep
produces only a few hundred distinct keys.
"""

from __future__ import annotations

from dataclasses import dataclass, field
import re
from functools import lru_cache

from .errors import ParseError


@dataclass
class SchemeNode:
    children: list["SchemeNode"] = field(default_factory=list)

    def count(self) -> int:
        return 1 + sum(c.count() for c in self.children)


@dataclass
class SchemeTree:
    root: SchemeNode
    has_pseudoline: bool

    def oval_count(self) -> int:
        return self.root.count() - 1


def _items(node: SchemeNode) -> str:
    parts = sorted(_items(c) for c in node.children)
    out: list[str] = []
    k = 0
    while k < len(parts):
        run = k
        while run < len(parts) and parts[run] == parts[k]:
            run += 1
        n = run - k
        out.append(str(n) if parts[k] == "" else f"{n}<{parts[k]}>")
        k = run
    return " u ".join(out)


def canonical_scheme(tree: SchemeTree) -> str:
    inner = _items(tree.root)
    if tree.has_pseudoline:
        return f"<J u {inner}>" if inner else "<J>"
    return f"<{inner}>" if inner else "<0>"


# ----------------------------------------------------------------- tree keys


def key_ovals(key: int) -> int:
    return (int(key).bit_length() - 1) // 2


def tree_from_key(key: int) -> SchemeNode:
    key = int(key)
    if key <= 0:
        raise ValueError(f"invalid tree key {key}")
    n = key.bit_length() - 1
    if n % 2:
        raise ValueError(f"tree key {key:#x} has odd code length")
    root = SchemeNode()
    stack = [root]
    for pos in range(n - 1, -1, -1):
        if (key >> pos) & 1:
            child = SchemeNode()
            stack[-1].children.append(child)
            stack.append(child)
        else:
            if len(stack) == 1:
                raise ValueError(f"tree key {key:#x} is unbalanced")
            stack.pop()
    if len(stack) != 1:
        raise ValueError(f"tree key {key:#x} is unbalanced")
    return root


def scheme_from_parents(parent, nreg: int, has_pseudoline: bool) -> str:
    """Canonical string of a rooted region tree given as a parent array
    (the root is its own parent), iteratively (any depth)."""
    kids: list[list[int]] = [[] for _ in range(nreg)]
    root = -1
    for r in range(nreg):
        p = int(parent[r])
        if p == r:
            root = r
        else:
            kids[p].append(r)
    if root < 0:
        raise ValueError("parent array without a root")
    order, stack = [], [root]
    while stack:
        v = stack.pop()
        order.append(v)
        stack.extend(kids[v])
    items: dict[int, str] = {}
    for v in reversed(order):
        parts = sorted(items.pop(c) for c in kids[v])
        out, k = [], 0
        while k < len(parts):
            run = k
            while run < len(parts) and parts[run] == parts[k]:
                run += 1
            out.append(str(run - k) if parts[k] == "" else f"{run - k}<{parts[k]}>")
            k = run
        items[v] = " u ".join(out)
    inner = items[root]
    if has_pseudoline:
        return f"<J u {inner}>" if inner else "<J>"
    return f"<{inner}>" if inner else "<0>"


@lru_cache(maxsize=1 << 16)
def scheme_from_key(key: int, has_pseudoline: bool) -> str:
    return canonical_scheme(SchemeTree(tree_from_key(key), has_pseudoline))


def key_from_tree(node: SchemeNode) -> int:
    """Host restatement of the device AHU key (for tests)."""

    def skey(n: SchemeNode) -> int:
        acc = 1
        for c in sorted(skey(c) for c in n.children):
            ln = c.bit_length() - 1
            acc = (acc << ln) | (c ^ (1 << ln))
        ln = acc.bit_length() - 1
        return (acc << 1) | (1 << (ln + 2))

    acc = 1
    for c in sorted(skey(c) for c in node.children):
        ln = c.bit_length() - 1
        acc = (acc << ln) | (c ^ (1 << ln))
    return acc


# ------------------------------------------------------------------- parser

_TOKEN = re.compile(r"\d+|J|<|>| u |.", re.S)


def parse_scheme(text: str) -> SchemeTree:
    """Parse a scheme string (grammar of the reference's scheme.py:7-10).

    Token-stream recursive descent; errors carry the character offset.
    """
    toks = [(m.group(0), m.start()) for m in _TOKEN.finditer(text)]
    toks.append(("", len(text)))
    at = [0]

    def cur():
        return toks[at[0]]

    def fail(msg):
        raise ParseError(msg, position=cur()[1])

    def take(tok):
        if cur()[0] != tok:
            fail(f"expected {tok!r}")
        at[0] += 1

    def seq(top):
        kids: list[SchemeNode] = []
        pseudo = False
        while True:
            tok = cur()[0]
            if tok == "J":
                if not (top and at[0] == 1):
                    fail("J is allowed only first at top level")
                pseudo = True
                at[0] += 1
            elif tok.isdigit():
                n = int(tok)
                if n < 1:
                    fail("item count must be positive")
                if n > 1_000_000:
                    fail("item count too large")
                at[0] += 1
                if cur()[0] == "<":
                    at[0] += 1
                    inner, _ = seq(False)
                    take(">")
                    kids.extend(SchemeNode([_copy(c) for c in inner]) for _ in range(n))
                else:
                    kids.extend(SchemeNode() for _ in range(n))
            else:
                fail("expected an integer")
            if cur()[0] != " u ":
                return kids, pseudo
            at[0] += 1

    take("<")
    if cur()[0] == "0":
        at[0] += 1
        take(">")
        if cur()[0] != "":
            fail("trailing input after scheme")
        return SchemeTree(SchemeNode(), has_pseudoline=False)
    kids, pseudo = seq(True)
    take(">")
    if cur()[0] != "":
        fail("trailing input after scheme")
    return SchemeTree(SchemeNode(kids), has_pseudoline=pseudo)


def _copy(node: SchemeNode) -> SchemeNode:
    return SchemeNode([_copy(c) for c in node.children])
