"""Shape of the powersort merge tree of a BASELINE config (CPU, oracle): per depth and per
height (levels of merge nodes below a node) the node count and the merged elements --
what the merge executor's dependency chains look like.  Test tooling."""
import argparse, sys
sys.path.insert(0, '.')
import numpy as np
from oracle import oracle
from paper_1805_04154_b200 import workloads

ap = argparse.ArgumentParser()
ap.add_argument('--config', type=int, default=3)
ap.add_argument('--n', type=int, default=None)
a = ap.parse_args()
keys, tags = workloads.generate(a.config, a.n)
n = len(keys)
res = oracle.powersort(keys.copy(), 24, 'bitonic', None, want_tree=True)
starts = res.leaf_starts.astype(np.int64); P = res.powers
r = len(starts); m = r - 1
ends = np.append(starts[1:], n)
left = [0] * (m + 1); right = [0] * (m + 1); stack = []
for j in range(1, m + 1):
    last = 0
    while stack and P[stack[-1] - 1] > P[j - 1]:
        last = stack.pop()
    left[j] = last
    if stack: right[stack[-1]] = j
    stack.append(j)
root = stack[0]
depth = [0] * (m + 1); lo = [0] * (m + 1); hi = [0] * (m + 1); height = [0] * (m + 1)
order = []; st = [root]
while st:
    j = st.pop(); order.append(j)
    for c in (left[j], right[j]):
        if c: depth[c] = depth[j] + 1; st.append(c)
for j in reversed(order):
    lo[j] = lo[left[j]] if left[j] else starts[j - 1]
    hi[j] = hi[right[j]] if right[j] else ends[j]
    height[j] = 1 + max(height[left[j]] if left[j] else 0, height[right[j]] if right[j] else 0)
span = [hi[j] - lo[j] for j in range(m + 1)]
print('n', n, 'leaves', r, 'max depth', max(depth), 'root height', height[root])
from collections import defaultdict
bd = defaultdict(lambda: [0, 0]); bh = defaultdict(lambda: [0, 0])
for j in range(1, m + 1):
    bd[depth[j]][0] += 1; bd[depth[j]][1] += span[j]
    bh[height[j]][0] += 1; bh[height[j]][1] += span[j]
print('by depth  (depth, nodes, Melems):', [(d, bd[d][0], round(bd[d][1] / 1e6, 2)) for d in sorted(bd)])
print('by height (height, nodes, Melems):', [(h, bh[h][0], round(bh[h][1] / 1e6, 2)) for h in sorted(bh)])
# critical chain from the root: at each node follow the child with the larger height
j = root; chain = []
while j:
    chain.append((depth[j], height[j], span[j]))
    l, rr = left[j], right[j]
    hl = height[l] if l else 0; hr = height[rr] if rr else 0
    j = l if hl >= hr else rr
    if max(hl, hr) == 0: break
print('critical chain (depth, height, span):', chain)
print('nodes of depth <= 3 (depth, height, lo, span, left child, right child):')
def desc(c, leaf_i):
    if c: return f'node(h{height[c]},{span[c]})'
    return f'leaf({ends[leaf_i] - starts[leaf_i]})'
for j in order:
    if depth[j] <= 3:
        print('  ', depth[j], height[j], lo[j], span[j], desc(left[j], j - 1), desc(right[j], j))
