"""Codebook steps of the DF11 oracle (E3 code lengths, E4 canonical codes, E5 hierarchical LUTs).

TEST INFRASTRUCTURE ONLY — see oracle/__init__.py.  Pure-Python loops over at most 256 symbols:
small enough to be read against the paper line by line.

Citations: "P:n" = PAPER.md line n.  R-numbers are the readings listed in DESIGN.md §3.
"""
from __future__ import annotations

MAX_CODE_LEN = 32  # P:146 [§2.3.2] "With a maximum code length of 32 bits" (R4)


# --------------------------------------------------------------------------- E3: code lengths
def huffman_code_lengths(hist):
    """Unconstrained Huffman code lengths for a 256-bin histogram.

    P:97 [§2.3] "we build a Huffman tree based on the distribution of exponents"; P:54 [§2.1]
    Huffman coding assigns shorter codes to more frequent symbols.  Tie-break (R3): a min-heap keyed
    by (weight, key); a leaf's key is its rank in (count asc, symbol asc) order, an internal node's
    key is |S| + its creation index.  Pop the two smallest, merge, push.  A leaf's depth is its
    length.  |S| = 1 gets length 1 (R10).
    """
    syms = [s for s in range(256) if hist[s] > 0]
    lengths = [0] * 256
    if not syms:
        return lengths
    if len(syms) == 1:
        lengths[syms[0]] = 1
        return lengths
    ranked = sorted(syms, key=lambda s: (hist[s], s))
    # node = (weight, key, payload); payload = symbol (leaf) or (left, right) (internal)
    active = [(int(hist[s]), rank, s) for rank, s in enumerate(ranked)]
    next_key = len(syms)
    while len(active) > 1:
        active.sort(key=lambda node: (node[0], node[1]))
        a, b = active[0], active[1]
        active = active[2:] + [(a[0] + b[0], next_key, (a, b))]
        next_key += 1
    # depth of every leaf
    stack = [(active[0], 0)]
    while stack:
        node, depth = stack.pop()
        payload = node[2]
        if isinstance(payload, tuple):
            stack.append((payload[0], depth + 1))
            stack.append((payload[1], depth + 1))
        else:
            lengths[payload] = depth
    return lengths


def package_merge_code_lengths(hist, cap):
    """Optimal length-limited prefix code (max length `cap`) by package-merge (R4).

    The paper asserts a 32-bit maximum but gives no mechanism; we use the textbook
    package-merge (coin-collector) algorithm.  Items at the deepest level are the leaves sorted by
    (count asc, symbol asc).  Going up one level: package consecutive pairs of the current list
    (an odd last item is dropped), then merge the packages with the sorted leaves; on equal weight
    leaves come first.  From the final list take the first 2(|S|-1) items; a symbol's code length
    is the number of selected items (counting through packages) that contain it.
    """
    syms = [s for s in range(256) if hist[s] > 0]
    lengths = [0] * 256
    if not syms:
        return lengths
    if len(syms) == 1:
        lengths[syms[0]] = 1
        return lengths
    if (1 << cap) < len(syms):
        raise ValueError("cap too small for the alphabet")
    leaves = [(int(hist[s]), ("leaf", s)) for s in sorted(syms, key=lambda s: (hist[s], s))]
    current = list(leaves)
    for _level in range(cap - 1):
        packages = []
        for i in range(0, len(current) - 1, 2):
            a, b = current[i], current[i + 1]
            packages.append((a[0] + b[0], ("pkg", a, b)))
        # stable merge; leaves before packages on equal weight
        merged = []
        i = j = 0
        while i < len(leaves) or j < len(packages):
            if j >= len(packages) or (i < len(leaves) and leaves[i][0] <= packages[j][0]):
                merged.append(leaves[i])
                i += 1
            else:
                merged.append(packages[j])
                j += 1
        current = merged
    selected = current[: 2 * (len(syms) - 1)]
    stack = list(selected)
    while stack:
        item = stack.pop()
        payload = item[1]
        if payload[0] == "leaf":
            lengths[payload[1]] += 1
        else:
            stack.append(payload[1])
            stack.append(payload[2])
    return lengths


def code_lengths(hist, cap=MAX_CODE_LEN):
    """E3: Huffman lengths; if the longest exceeds `cap`, recompute with package-merge (R4)."""
    lengths = huffman_code_lengths(hist)
    if max(lengths) > cap:
        lengths = package_merge_code_lengths(hist, cap)
    return lengths


# --------------------------------------------------------------------------- E4: canonical codes
def canonical_codes(lengths):
    """E4 (R3): sort present symbols by (length asc, symbol asc); code_0 = 0 and
    code_i = (code_{i-1} + 1) << (l_i - l_{i-1}).  Absent symbols get code 0 / length 0."""
    order = sorted((lengths[s], s) for s in range(256) if lengths[s] > 0)
    codes = [0] * 256
    prev_code, prev_len = None, None
    for length, s in order:
        if prev_code is None:
            code = 0
        else:
            code = (prev_code + 1) << (length - prev_len)
        codes[s] = code
        prev_code, prev_len = code, length
    return codes


def kraft_sum(lengths):
    """sum 2^-l over present symbols, as an exact fraction numerator over 2^64."""
    from fractions import Fraction
    return sum(Fraction(1, 1 << l) for l in lengths if l > 0)


# --------------------------------------------------------------------------- monolithic LUT
def monolithic_lut(lengths, codes):
    """P:537-539 [App. I.1]: a table of 2^L entries; entry i is the symbol whose code is a prefix
    of the L-bit binary representation of i.  Used only as a test oracle for small L."""
    L = max(lengths)
    table = [None] * (1 << L)
    for s in range(256):
        l = lengths[s]
        if l == 0:
            continue
        lo = codes[s] << (L - l)
        for i in range(lo, lo + (1 << (L - l))):
            table[i] = s
    return table


# --------------------------------------------------------------------------- E5: hierarchical LUTs
def hierarchical_luts(lengths, codes, b=8):
    """E5: cut the code tree into height-b subtrees, one 2^b-entry table each.

    P:128-132 [§2.3.1] "partition the Huffman tree into non-overlapping subtrees of height 8. Each
    subtree corresponds to a compact LUT"; App. I.2 P:548-593 (generic b; b = 2 example).
    Entry values are generic here: an int >= 0 is a decoded symbol, ("ptr", j) names child table j.
    Table 0 is the root (depth 0).  Children are numbered breadth-first: tables are processed in
    index order and, within a table, entries in ascending index order; every new child prefix gets
    the next index (R6).  Unreachable entries (only possible when |S| = 1) repeat the symbol (R7).
    Returns (tables, depth_of_table).
    """
    present = [s for s in range(256) if lengths[s] > 0]
    if not present:
        return [], []
    size = 1 << b
    tables = []
    depth = []
    prefix = []  # code prefix (top b*d bits) that leads to each table
    tables.append([None] * size)
    depth.append(0)
    prefix.append(0)
    t = 0
    while t < len(tables):
        d = depth[t]
        lo_bits = b * d          # bits already consumed before this table
        hi_bits = b * (d + 1)    # bits consumed after this table
        child_of_entry = {}
        for s in present:
            l, c = lengths[s], codes[s]
            if l <= lo_bits:
                continue
            if (c >> (l - lo_bits)) != prefix[t]:
                continue  # symbol does not pass through this table
            if l <= hi_bits:
                start = (c & ((1 << (l - lo_bits)) - 1)) << (hi_bits - l)
                for i in range(start, start + (1 << (hi_bits - l))):
                    tables[t][i] = s
            else:
                child_prefix = c >> (l - hi_bits)
                idx = child_prefix & (size - 1)
                child_of_entry[idx] = child_prefix
        for idx in sorted(child_of_entry):
            j = len(tables)
            tables.append([None] * size)
            depth.append(d + 1)
            prefix.append(child_of_entry[idx])
            tables[t][idx] = ("ptr", j)
        t += 1
    if len(present) == 1:
        for table in tables:
            for i in range(size):
                if table[i] is None:
                    table[i] = present[0]
    for table in tables:
        assert all(e is not None for e in table), "incomplete code tree"
    return tables, depth


def serialize_luts(tables, wide):
    """Narrow (paper, Alg. 1): uint8 entries; symbols 0..239; child j is stored as
    pointer value 256-j so that Alg. 1's LUT_{257-v} (1-based) is 0-based table j (R6).  Legal only
    if every symbol is <= 239 and there are at most 16 children (R8, R9).
    Wide (R8): little-endian uint16 entries; symbol s < 256 as s, child j as 256+j.
    Returns bytes."""
    out = bytearray()
    for table in tables:
        for e in table:
            if isinstance(e, tuple):
                j = e[1]
                if wide:
                    v = 256 + j
                    out += bytes((v & 0xFF, v >> 8))
                else:
                    if not 1 <= j <= 16:
                        raise ValueError("narrow LUT overflow: more than 16 child tables")
                    out.append(256 - j)
            else:
                if wide:
                    out += bytes((e & 0xFF, e >> 8))
                else:
                    if e >= 240:
                        raise ValueError("exponent >= 240 cannot be stored in a narrow LUT")
                    out.append(e)
    return bytes(out)


def narrow_is_legal(lengths, tables):
    """R8/R9: narrow iff every present exponent <= 239 and at most 16 child tables."""
    return all(s <= 239 for s in range(256) if lengths[s] > 0) and len(tables) - 1 <= 16


def lut_decode_step(tables, lengths, window_bits, b=8):
    """One hierarchical lookup (P:405-411 with generic b): `window_bits` is a string of '0'/'1' at
    least as long as the code.  Returns (symbol, code length)."""
    t = 0
    i = 0
    while True:
        chunk = window_bits[i * b:(i + 1) * b].ljust(b, "0")
        e = tables[t][int(chunk, 2)]
        if isinstance(e, tuple):
            t = e[1]
            i += 1
            continue
        return e, lengths[e]
