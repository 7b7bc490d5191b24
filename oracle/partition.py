"""Oracle restatement of the recursive coordinate bisection partitioner
(TEST INFRASTRUCTURE ONLY; the reference has no partitioner -- SPEC.md:15).

Plain recursion over Python lists: split along the first axis of maximal
bounding-box extent, order by (coordinate, element id), give the first
floor(n * k1 / k) elements to the lower k1 = k // 2 parts."""


def rcb(points, nparts):
    n = len(points)
    parts = [0] * n

    def rec(ids, base, k):
        if k == 1:
            for i in ids:
                parts[i] = base
            return
        ext = []
        for d in range(3):
            vals = [points[i][d] for i in ids]
            ext.append(max(vals) - min(vals))
        axis = max(range(3), key=lambda d: (ext[d], -d))
        order = sorted(ids, key=lambda i: (points[i][axis], i))
        k1 = k // 2
        n1 = (len(ids) * k1) // k
        rec(order[:n1], base, k1)
        rec(order[n1:], base + k1, k - k1)

    rec(list(range(n)), 0, nparts)
    return parts
