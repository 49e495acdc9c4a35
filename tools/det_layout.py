"""Replica of make_layout (csrc/runsort_b200.cu) offsets: powersort, int32 keys (debug tools)."""


def layout(n, w, kb=4, tb=0):
    au = lambda x: (x + 255) // 256 * 256
    words = (n + 31) // 32 + 2
    ntiles = (n + 2047) // 2048
    ngroups = (ntiles + 63) // 64
    r_max = n // max(w, 2) + 2
    nchunks = (r_max + 255) // 256 + 1
    tile, fcap = 256 * 15, 4096
    levels = 2 + n.bit_length()
    max_tasks = levels * (n // tile + n // fcap + 2) + 3 * r_max + 2 * (n // tile) + 16
    items = [("key1", n * kb + 64), ("tag1", n * tb + 64), ("key2", n * kb + 64), ("tag2", n * tb + 64),
             ("ascw", words * 4), ("tables", ntiles * (w + 1) * 8), ("gtab", ngroups * (w + 1) * 8),
             ("gentry", ngroups * 4), ("goff", ngroups * 8), ("tentry", ntiles * 4), ("toff", ntiles * 8),
             ("leaf_start", (r_max + 1) * 8), ("leaf_info", r_max * 4), ("leaf_depth", r_max), ("K", r_max * 8),
             ("P", r_max), ("la", r_max), ("ra", r_max), ("depth", r_max), ("node_a", r_max * 4),
             ("node_b", r_max * 4), ("node_s", r_max * 8), ("node_e", r_max * 8), ("parent", (2 * r_max + 2) * 4),
             ("child", (2 * r_max + 2) * 4), ("need", (2 * r_max + 2) * 4), ("done", (2 * r_max + 2) * 4),
             ("agg", 2 * nchunks * 16), ("tasks", max_tasks * 8), ("chunkdep", ((r_max + 255) // 256 + 1) * 64 * 4),
             ("cls", 2 * r_max + 2), ("met", 1 << 20)]
    off, out = 0, []
    for name, b in items:
        out.append((name, off, b))
        off = au(off + b)
    return out

