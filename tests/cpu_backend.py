"""CPU stand-ins for the per-rank stages of the library's distributed kNN (TEST ONLY), used by
the protocol model tests/dist_model.py over torch.distributed / gloo. Every stage is a plain
numpy / oracle computation; the per-rank kNN is the oracle's brute force, so the gathered result
equals the global oracle only if the ghost protocol delivered every needed point.
"""
import numpy as np
import torch

from oracle import knn_brute
from oracle import tree as T


class CpuIndex:
    def __init__(self, pts4, n_query, box):
        self.pts4 = pts4.cpu().numpy()
        self.n = self.pts4.shape[0]
        self.n_query = n_query
        self.box = box
        self.device = torch.device("cpu")


class CpuBackend:
    def morton_keys(self, pos, frame):
        p = pos.numpy()
        if frame["box"] is not None:
            o, s = T.key_frame(p, frame["box"])
        else:
            o = np.asarray(frame["origin"], np.float32)
            s = np.full(3, np.float32(2.0 ** T.BITS / frame["extent"]), np.float32)
        return torch.from_numpy(T.morton_keys(T.quantize(p, o, s, is_scale=True)).astype(np.int64))

    def bbox(self, pos):
        return pos.min(0).values.clone(), pos.max(0).values.clone()

    def sample(self, keys, n, seed):
        if keys.shape[0] == 0:
            return keys[:0]
        rng = np.random.default_rng(seed)
        return keys[torch.from_numpy(rng.integers(0, keys.shape[0], n))]

    def sort_samples(self, s):
        return torch.sort(s).values

    def bucket(self, keys, spl):
        dest = np.searchsorted(spl.numpy(), keys.numpy(), side="right").astype(np.int32)
        counts = np.bincount(dest, minlength=spl.shape[0] + 1)
        return torch.from_numpy(dest), [int(c) for c in counts]

    def pack(self, pos, gbase, dest, counts):
        d = dest.numpy()
        order = np.argsort(d, kind="stable")
        p = pos.numpy()[order]
        g = (gbase + order).astype(np.int32).view(np.float32)
        return torch.from_numpy(np.concatenate([p, g[:, None]], axis=1).astype(np.float32))

    def build(self, pts4, n_query, box):
        """Local points sorted into z order (the library's index order)."""
        p = pts4.cpu().numpy()
        if p.shape[0]:
            o, s = T.key_frame(p[:, :3], box) if box is not None else T.key_frame(p[:, :3])
            p = p[np.argsort(T.morton_keys(T.quantize(p[:, :3], o, s, is_scale=True)), kind="stable")]
        return CpuIndex(torch.from_numpy(np.ascontiguousarray(p)), n_query, box)

    def query_boxes(self, ix, k, rank, d2=None):
        """Chunks of 64 local points (key order): AABB + max local k-th d2 (a valid bound: the
        local k-th distance can only shrink when more points are added); +inf without local rows
        (d2 None). Returns the boxes and the local rows (point indices) inside each box."""
        p = ix.pts4[:, :3]
        n = p.shape[0]
        r2 = np.full(n, np.inf) if d2 is None else d2.numpy()[:, -1].astype(np.float64)
        rows, members = [], []
        for c in range(0, n, 64):  # ix.pts4 rows are the local points in z order
            sel = np.arange(c, min(n, c + 64))
            lo, hi = p[sel].min(0), p[sel].max(0)
            rows.append([*lo, r2[sel].max(), *hi, 0.0])
            members.append(sel)
        out = np.asarray(rows, np.float32).reshape(-1, 8)
        out[:, 7] = np.array([rank] * len(rows), np.int32).view(np.float32)
        return torch.from_numpy(out), members

    def select_ghosts(self, ix, boxes, rank, R):
        b = boxes.numpy()
        p = ix.pts4[:, :3].astype(np.float64)
        mask = np.zeros(ix.n, np.int32)
        hitbox = np.zeros(b.shape[0], np.int32)
        rk = b[:, 7].view(np.int32)
        for j in range(b.shape[0]):
            if rk[j] == rank:
                continue
            lo, hi = b[j, 0:3].astype(np.float64), b[j, 4:7].astype(np.float64)
            gap = np.maximum(0.0, np.maximum(lo - p, p - hi))
            if ix.box is not None:  # minimal image of the point-box gap
                L = np.broadcast_to(np.asarray(ix.box, np.float64), (3,))
                c = 0.5 * (lo + hi)
                e = 0.5 * (hi - lo)
                dd = np.abs(p - c)
                dd = np.minimum(dd, L - dd)
                gap = np.maximum(0.0, dd - e)
            d = np.sqrt((gap ** 2).sum(1))
            r = np.sqrt(np.float64(b[j, 3]))
            hit = d <= r * (1 + 1e-5) + 1e-7
            mask[hit] |= 1 << int(rk[j])
            hitbox[j] = int(hit.any())
        counts = [int(((mask >> r) & 1).sum()) for r in range(R)]
        return torch.from_numpy(mask), counts, hitbox

    def pack_ghosts(self, ix, mask, counts):
        m = mask.numpy()
        parts = [ix.pts4[((m >> r) & 1) == 1] for r in range(len(counts))]
        return torch.from_numpy(np.concatenate(parts).astype(np.float32)) if parts else torch.zeros((0, 4))

    def query_z(self, ix, k):
        p = ix.pts4[:, :3]
        g = ix.pts4[:, 3].view(np.int32)
        rows = np.arange(ix.n_query)
        idx, d2 = knn_brute(p, k, ix.box, rows=rows)
        return torch.from_numpy(g[idx]), torch.from_numpy(d2), torch.from_numpy(g[:ix.n_query].copy())

    def pack_rows(self, idx, d2, rowg, dest, counts):
        order = np.argsort(dest.numpy(), kind="stable")
        words = np.concatenate([idx.numpy(), d2.numpy().view(np.int32), rowg.numpy()[:, None]], axis=1)
        return torch.from_numpy(np.ascontiguousarray(words[order]).astype(np.int32))

    def scatter_rows(self, rows, k, base, n, device):
        r = rows.numpy()
        at = r[:, 2 * k].astype(np.int64) - base
        assert ((at >= 0) & (at < n)).all()
        idx = np.empty((n, k), np.int32)
        d2 = np.empty((n, k), np.float32)
        idx[at] = r[:, :k]
        d2[at] = r[:, k:2 * k].view(np.float32)
        return torch.from_numpy(idx), torch.from_numpy(d2)

    def free(self, ix):
        pass
