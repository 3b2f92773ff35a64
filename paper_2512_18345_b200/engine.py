"""Process-wide handle on the CUDA engine: one C context per GPU, device-side
caches for modulus slots / conversion tables / key-switch plans, and thin
launch wrappers that hand raw device pointers and the current torch stream to
the C ABI.  PyTorch is plumbing here (allocator, streams, graphs); all
arithmetic is in csrc/.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib


class Engine:
    def __init__(self, device: int | None = None):
        import torch

        if not torch.cuda.is_available():
            raise _lib.EngineUnavailable(
                "no CUDA device: paper_2512_18345_b200 runs on a B200 only (no CPU fallback)"
            )
        self.torch = torch
        self.lib = _lib.load()
        self.device_index = torch.cuda.current_device() if device is None else device
        self.device = torch.device("cuda", self.device_index)
        h = ctypes.c_void_p()
        _lib.check(self.lib.ckks_ctx_create(self.device_index, ctypes.byref(h)))
        self.ctx = h
        self._slots: dict = {}
        self._row_slots: dict = {}
        self._tables: dict = {}
        self._plans: dict = {}

    # ---- plumbing ---------------------------------------------------------
    def stream(self) -> int:
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def upload(self, words: np.ndarray):
        """Host uint32 matrix -> device tensor (int32 storage)."""
        t = self.torch.from_numpy(np.ascontiguousarray(words, dtype=np.uint32).view(np.int32))
        return t.to(self.device, non_blocking=False)

    def empty(self, *shape):
        return self.torch.empty(shape, dtype=self.torch.int32, device=self.device)

    # ---- lanes: concurrent key switches on side streams ---------------------
    def set_lanes(self, count: int) -> None:
        """Replicate the key-switch workspace `count` times and create one side
        stream per extra lane (lane 0 runs on the caller's stream)."""
        _lib.check(self.lib.ckks_set_lanes(self.ctx, count))
        self.lanes = count
        self.lane_streams = [None] + [self.torch.cuda.Stream(device=self.device) for _ in range(count - 1)]
        self._lane_group = None

    def arena_generation(self) -> int:
        """Counter that changes whenever the C library reallocates (moves) its workspace arena;
        a captured CUDA graph is only valid for the generation it was captured under."""
        g = ctypes.c_uint64()
        _lib.check(self.lib.ckks_arena_generation(self.ctx, ctypes.byref(g)))
        return g.value

    def fork(self, jobs, with_lane: bool = False):
        """Run the callables in `jobs` concurrently over the lanes the caller owns (each on
        its lane's stream and workspace), joined back into the current stream.  Results in
        order.  Forks nest: with fewer jobs than lanes the caller's lanes are split into one
        contiguous group per job, and a fork issued inside a job spreads over that job's
        group only, so concurrent jobs never share a workspace lane."""
        torch = self.torch
        outer = getattr(self, "_lane_group", None)
        group = outer if outer is not None else list(range(getattr(self, "lanes", 1)))
        if len(group) == 1 or len(jobs) < 2:
            return [job(group[0], i) if with_lane else job() for i, job in enumerate(jobs)]
        width = min(len(jobs), len(group))
        if with_lane:
            # lane-indexed jobs (per-lane accumulators reduced by ks_finish): the first `width`
            # lanes of the group, one each, no nesting
            subs = [[lane] for lane in group[:width]]
        else:
            # sub-groups: job i runs on lane sub[i % width][0] and may fork over sub[i % width]
            base, extra = divmod(len(group), width)
            subs, at = [], 0
            for w in range(width):
                size = base + (1 if w < extra else 0)
                subs.append(group[at:at + size])
                at += size
        home = group[0]
        main = torch.cuda.current_stream(self.device)
        start = torch.cuda.Event()
        start.record(main)
        used = set()
        out = []
        try:
            for i, job in enumerate(jobs):
                sub = subs[i % width]
                lane = sub[0]
                self._lane_group = sub
                _lib.check(self.lib.ckks_select_lane(self.ctx, lane))
                if lane == home:
                    out.append(job(lane, i // width) if with_lane else job())
                    continue
                side = self.lane_streams[lane]
                if lane not in used:
                    side.wait_event(start)
                    used.add(lane)
                with torch.cuda.stream(side):
                    out.append(job(lane, i // width) if with_lane else job())
        finally:
            self._lane_group = outer
            _lib.check(self.lib.ckks_select_lane(self.ctx, home))
            # join on the error path too: work already enqueued on a side stream still uses lane
            # workspaces and tensors the main stream would otherwise be free to reuse
            for lane in used:
                main.wait_stream(self.lane_streams[lane])
        return out

    def pipeline(self, items, first, second):
        """Two-stage software pipeline over two lanes: `first(item)` runs on the caller's lane,
        `second(item, first_result)` on the next lane of the caller's group as soon as that
        item's first stage is done, so stage one of item i + 1 overlaps stage two of item i
        (the reference models this co-scheduling of a cache-bound with a DRAM-bound kernel group
        in costmodel.py:508-541; here the two groups really run on two streams).  Intermediates
        stay referenced until the join, so no buffer is recycled under a reader on the other
        stream.  Results of `second`, in order."""
        torch = self.torch
        outer = getattr(self, "_lane_group", None)
        group = outer if outer is not None else list(range(getattr(self, "lanes", 1)))
        if len(group) < 2:
            return [second(item, first(item)) for item in items]
        home, lane = group[0], group[1]
        main = torch.cuda.current_stream(self.device)
        side = self.lane_streams[lane]
        side.wait_stream(main)
        keep, out = [], []
        try:
            for item in items:
                self._lane_group = [home]
                _lib.check(self.lib.ckks_select_lane(self.ctx, home))
                mid = first(item)
                done = torch.cuda.Event()
                done.record(main)
                keep.append(mid)
                self._lane_group = [lane]
                _lib.check(self.lib.ckks_select_lane(self.ctx, lane))
                side.wait_event(done)
                with torch.cuda.stream(side):
                    out.append(second(item, mid))
        finally:
            self._lane_group = outer
            _lib.check(self.lib.ckks_select_lane(self.ctx, home))
            main.wait_stream(side)
        del keep
        return out

    def lane_count(self) -> int:
        """Lanes the caller may fork over right now (all of them outside a fork)."""
        group = getattr(self, "_lane_group", None)
        return len(group) if group is not None else getattr(self, "lanes", 1)

    # ---- modulus slots ----------------------------------------------------
    def slot(self, m, n: int) -> int:
        """Context slot of Modulus ``m`` with transform tables for degree n
        (0: arithmetic only)."""
        psi = 0
        if n >= 2 and (m.q - 1) % (2 * n) == 0 and m.n >= n and m.q < (1 << 31):
            psi = m.root_for_degree(n)
        else:
            n = 0
        key = (m.q, n, psi)
        s = self._slots.get(key)
        if s is None:
            out = ctypes.c_int32()
            _lib.check(self.lib.ckks_modulus_register(self.ctx, m.q, n, psi, ctypes.byref(out)))
            s = self._slots[key] = out.value
        return s

    def custom_table_slot(self, q: int, n: int, fwd, inv, n_inv: int) -> int:
        """Slot whose device twiddle tables are the given host arrays (a caller-built or
        deliberately corrupted TwiddleTable); memoised on the table contents."""
        fwd = np.ascontiguousarray(fwd, dtype=np.uint32)
        inv = np.ascontiguousarray(inv, dtype=np.uint32)
        key = (q, n, int(n_inv), fwd.tobytes(), inv.tobytes())
        cache = self.__dict__.setdefault("_custom_slots", {})
        s = cache.get(key)
        if s is None:
            out = ctypes.c_int32()
            _lib.check(self.lib.ckks_modulus_register_tables(self.ctx, q, n, fwd.ctypes.data, inv.ctypes.data,
                                                             int(n_inv), ctypes.byref(out)))
            s = cache[key] = out.value
        return s

    def row_slots(self, basis, n: int = 0, repeat: int = 1):
        """Device int32 array: slot of every row of a limb matrix over `basis`
        (stacked `repeat` times)."""
        key = (tuple((m.q, m.n, m.psi) for m in basis), n, repeat)
        hit = self._row_slots.get(key)
        if hit is None:
            ids = [self.slot(m, n) for m in basis] * repeat
            hit = self._row_slots[key] = self.torch.tensor(ids, dtype=self.torch.int32,
                                                           device=self.device)
        return hit

    def has_tables(self, m, n: int) -> bool:
        return n >= 2 and (m.q - 1) % (2 * n) == 0 and m.n >= n and m.q < (1 << 31)

    def twiddle_tables(self, m, n: int):
        fwd = np.empty(n, np.uint32)
        inv = np.empty(n, np.uint32)
        n_inv = ctypes.c_uint32()
        _lib.check(self.lib.ckks_modulus_tables(self.ctx, self.slot(m, n), fwd.ctypes.data,
                                                inv.ctypes.data, ctypes.byref(n_inv)))
        return fwd, inv, n_inv.value

    # ---- kernels ----------------------------------------------------------
    def elementwise(self, a, b, row_slot, kind: int, out=None):
        out = self.torch.empty_like(a) if out is None else out
        _lib.check(self.lib.ckks_elementwise(self.ctx, a.data_ptr(), b.data_ptr(), out.data_ptr(),
                                             row_slot.data_ptr(), a.shape[0], a.shape[1], kind,
                                             self.stream()))
        return out

    def automorphism_eval(self, a, k: int):
        out = self.torch.empty_like(a)
        _lib.check(self.lib.ckks_automorphism_eval(self.ctx, a.data_ptr(), out.data_ptr(),
                                                   a.shape[0], a.shape[1], k, self.stream()))
        return out

    def automorphism_coeff(self, a, row_slot, k: int):
        out = self.torch.empty_like(a)
        _lib.check(self.lib.ckks_automorphism_coeff(self.ctx, a.data_ptr(), out.data_ptr(),
                                                    row_slot.data_ptr(), a.shape[0], a.shape[1], k,
                                                    self.stream()))
        return out

    def ntt(self, a, row_slot, inverse: bool, out=None):
        out = self.torch.empty_like(a) if out is None else out
        _lib.check(self.lib.ckks_ntt(self.ctx, a.data_ptr(), out.data_ptr(), row_slot.data_ptr(),
                                     a.shape[0], a.shape[1], int(inverse), self.stream()))
        return out

    def ntt_policy(self, cluster_max_rows: int = -1, ctas_per_sm: int = -1) -> tuple[int, int]:
        """Set (negative: only read) which N = 2^16 transforms run as one cluster kernel: those
        of at most `cluster_max_rows` limbs (0: the two-kernel split everywhere).  Scheduling
        only, results are identical.  Returns the values now in force."""
        import ctypes

        rows, occ = ctypes.c_int(0), ctypes.c_int(0)
        _lib.check(self.lib.ckks_ntt_policy(int(cluster_max_rows), int(ctas_per_sm), ctypes.byref(rows), ctypes.byref(occ)))
        return rows.value, occ.value

    def ntt_stages(self, a, row_slot, inverse: bool, lo: int, hi: int, out=None):
        out = self.torch.empty_like(a) if out is None else out
        _lib.check(self.lib.ckks_ntt_stages(self.ctx, a.data_ptr(), out.data_ptr(),
                                            row_slot.data_ptr(), a.shape[0], a.shape[1],
                                            int(inverse), lo, hi, self.stream()))
        return out

    def lift2_centered(self, coeff2, slot0: int, slot1: int, row_slot, rows: int):
        out = self.empty(rows, coeff2.shape[1])
        _lib.check(self.lib.ckks_lift2_centered(self.ctx, coeff2.data_ptr(), slot0, slot1,
                                                out.data_ptr(), row_slot.data_ptr(), rows,
                                                coeff2.shape[1], self.stream()))
        return out

    def pmult_accumulate(self, x, p, acc, row_slot, first: bool):
        """acc (+)= x * p; x, acc are [2, rows, n] ciphertext tensors, p is [rows, n]."""
        _lib.check(self.lib.ckks_pmult_accumulate(self.ctx, x.data_ptr(), p.data_ptr(),
                                                  acc.data_ptr(), row_slot.data_ptr(), x.shape[1],
                                                  x.shape[2], int(first), self.stream()))
        return acc

    def fused_terms(self, xs, ps, row_slot, out=None):
        """out = sum_t xs[t] * ps[t] (ps[t] None: plain term); xs[t] is a [2, rows, n] tensor, or a pair
        (a, b) of [rows, n] tensors for a ciphertext whose halves are not adjacent (no gathering copy)."""
        count = len(xs)
        pair = lambda x: isinstance(x, (tuple, list))
        first = xs[0][0]                   # the a half either way: [rows, n]
        rows, n = first.shape[0], first.shape[1]
        out = self.empty(2, rows, n) if out is None else out
        xa = (ctypes.c_void_p * count)(*[(x[0] if pair(x) else x).data_ptr() for x in xs])
        xb = (ctypes.c_void_p * count)(*[x[1].data_ptr() if pair(x) else None for x in xs])
        pp = (ctypes.c_void_p * count)(*[None if p is None else p.data_ptr() for p in ps])
        _lib.check(self.lib.ckks_fused_terms_halves(self.ctx, count, xa, xb, pp, out.data_ptr(), row_slot.data_ptr(),
                                                    rows, n, self.stream()))
        return out

    def fused_terms_multi(self, xs, table, row_slot):
        """outs[g] = sum_b xs[b] * table[g][b] for every giant step g in one pass
        (table[g][b] None: no such diagonal); xs are [2, rows, n] tensors."""
        nb, ng = len(xs), len(table)
        outs = [self.torch.empty_like(xs[0]) for _ in range(ng)]
        xp = (ctypes.c_void_p * nb)(*[x.data_ptr() for x in xs])
        flat = [None if pt is None else pt.data_ptr() for row in table for pt in row]
        pp = (ctypes.c_void_p * (nb * ng))(*flat)
        op = (ctypes.c_void_p * ng)(*[o.data_ptr() for o in outs])
        zero = None
        if any(f is None for f in flat):
            key = ("zero_plain", xs[0].shape[1], xs[0].shape[2])
            zero = self._tables.get(key)
            if zero is None:
                zero = self._tables[key] = self.torch.zeros(xs[0].shape[1:], dtype=self.torch.int32, device=self.device)
            zero = zero.data_ptr()
        _lib.check(self.lib.ckks_fused_terms_multi(self.ctx, nb, ng, xp, pp, zero, op, row_slot.data_ptr(),
                                                   xs[0].shape[1], xs[0].shape[2], self.stream()))
        return outs

    def tensor(self, x, y, row_slot):
        """(d0, d1, d2) of two [2, rows, n] ciphertext tensors as one [3, rows, n] tensor."""
        out = self.empty(3, x.shape[1], x.shape[2])
        _lib.check(self.lib.ckks_tensor(self.ctx, x.data_ptr(), y.data_ptr(), out.data_ptr(),
                                        row_slot.data_ptr(), x.shape[1], x.shape[2], self.stream()))
        return out

    def tensor_halves(self, xa, xb, ya, yb, row_slot):
        """(d0, d1, d2) from four separate [rows, n] halves (no [2, rows, n] gathering copy)."""
        out = self.empty(3, xa.shape[0], xa.shape[1])
        _lib.check(self.lib.ckks_tensor_halves(self.ctx, xa.data_ptr(), xb.data_ptr(), ya.data_ptr(), yb.data_ptr(),
                                               out.data_ptr(), row_slot.data_ptr(), xa.shape[0], xa.shape[1],
                                               self.stream()))
        return out

    def bconv_table(self, q_basis, p_basis) -> int:
        key = (tuple(m.q for m in q_basis), tuple(m.q for m in p_basis))
        t = self._tables.get(key)
        if t is None:
            src = (ctypes.c_int32 * len(q_basis))(*[self.slot(m, 0) for m in q_basis])
            dst = (ctypes.c_int32 * len(p_basis))(*[self.slot(m, 0) for m in p_basis])
            out = ctypes.c_int32()
            _lib.check(self.lib.ckks_bconv_table_create(self.ctx, src, len(q_basis), dst,
                                                        len(p_basis), ctypes.byref(out)))
            t = self._tables[key] = out.value
        return t

    def bconv_table_read(self, table: int, l_in: int, l_out: int):
        t = np.empty((l_out, l_in), np.uint32)
        inv = np.empty(l_in, np.uint32)
        _lib.check(self.lib.ckks_bconv_table_read(self.ctx, table, t.ctypes.data, inv.ctypes.data))
        return t, inv

    def bconv(self, table: int, a, l_out: int):
        out = self.empty(l_out, a.shape[1])
        _lib.check(self.lib.ckks_bconv(self.ctx, table, a.data_ptr(), out.data_ptr(), a.shape[1],
                                       self.stream()))
        return out

    # ---- key switching ----------------------------------------------------
    def ks_plan(self, n: int, q_basis, p_basis, alpha: int, evk_ext: int, evk_p_off: int) -> int:
        key = (n, tuple(m.q for m in q_basis), tuple(m.q for m in p_basis), alpha, evk_ext, evk_p_off)
        p = self._plans.get(key)
        if p is None:
            qs = (ctypes.c_int32 * len(q_basis))(*[self.slot(m, n) for m in q_basis])
            ps = (ctypes.c_int32 * len(p_basis))(*[self.slot(m, n) for m in p_basis])
            out = ctypes.c_int32()
            _lib.check(self.lib.ckks_ks_plan_create(self.ctx, n, len(q_basis), alpha, qs, ps,
                                                    evk_ext, evk_p_off, ctypes.byref(out)))
            p = self._plans[key] = out.value
        return p

    def moddown_plan(self, n: int, q_basis, p_basis) -> int:
        """Stage-3-only plan: ModDown from Q||P to Q for an arbitrary P (rescale when
        P is the single limb being dropped)."""
        key = ("moddown", n, tuple(m.q for m in q_basis), tuple(m.q for m in p_basis))
        p = self._plans.get(key)
        if p is None:
            qs = (ctypes.c_int32 * len(q_basis))(*[self.slot(m, n) for m in q_basis])
            ps = (ctypes.c_int32 * len(p_basis))(*[self.slot(m, n) for m in p_basis])
            out = ctypes.c_int32()
            _lib.check(self.lib.ckks_moddown_plan_create(self.ctx, n, len(q_basis), len(p_basis),
                                                         qs, ps, ctypes.byref(out)))
            p = self._plans[key] = out.value
        return p

    def ks_stage1(self, plan: int, a, beta: int, ext: int):
        raised = self.empty(beta, ext, a.shape[1])
        _lib.check(self.lib.ckks_ks_stage1(self.ctx, plan, a.data_ptr(), raised.data_ptr(),
                                           self.stream()))
        return raised

    def ks_stage2(self, plan: int, raised, evk, row_lo: int, row_hi: int):
        n = raised.shape[-1]
        acc = self.empty(2, row_hi - row_lo, n)
        _lib.check(self.lib.ckks_ks_stage2(self.ctx, plan, raised.data_ptr(), evk.data_ptr(), row_lo,
                                           row_hi, acc[0].data_ptr(), acc[1].data_ptr(),
                                           self.stream()))
        return acc

    def ks_stage3(self, plan: int, q_a, q_b, p_a, p_b):
        out = self.empty(2, q_a.shape[0], q_a.shape[1])
        _lib.check(self.lib.ckks_ks_stage3(self.ctx, plan, q_a.data_ptr(), q_b.data_ptr(),
                                           p_a.data_ptr(), p_b.data_ptr(), out[0].data_ptr(),
                                           out[1].data_ptr(), self.stream()))
        return out

    def ks_stage3_batch(self, plan: int, qps, l: int):
        """ModDown of qps = [count, 2, ext, n] accumulators in one set of launches -> [count, 2, l, n].
        Element g works in the arena of lane (current + g): the caller owns those lanes."""
        count, n = qps.shape[0], qps.shape[3]
        out = self.empty(count, 2, l, n)
        _lib.check(self.lib.ckks_ks_stage3_batch(self.ctx, plan, count, qps.data_ptr(), out.data_ptr(), self.stream()))
        return out

    def ks_stage3_batch_a(self, plan: int, qps, l: int):
        """ModDown of the a halves only of qps = [count, 2, ext, n] -> [count, l, n] (the b halves
        of these giant-step inner sums stay over Q||P, see ks_accumulate_rot_qp)."""
        count, n = qps.shape[0], qps.shape[3]
        out = self.empty(count, l, n)
        _lib.check(self.lib.ckks_ks_stage3_batch_a(self.ctx, plan, count, qps.data_ptr(), out.data_ptr(), self.stream()))
        return out

    def ks_hoisted(self, plan: int, raised, k: int, evk, ct_b):
        """Key switch of the ciphertext rotated by X -> X^k from pre-raised digits."""
        out = self.empty(2, ct_b.shape[0], ct_b.shape[1])
        _lib.check(self.lib.ckks_ks_hoisted(self.ctx, plan, raised.data_ptr(), k, evk.data_ptr(),
                                            ct_b.data_ptr(), out[0].data_ptr(), out[1].data_ptr(),
                                            self.stream()))
        return out

    def ks_hoisted_raw(self, plan: int, raised, k: int, evk, ct_b, ext: int):
        """Q||P accumulator [2, ext, n] of the ciphertext rotated by X -> X^k (no ModDown)."""
        out = self.empty(2, ext, ct_b.shape[1])
        _lib.check(self.lib.ckks_ks_hoisted_raw(self.ctx, plan, raised.data_ptr(), k, evk.data_ptr(),
                                                ct_b.data_ptr(), out.data_ptr(), self.stream()))
        return out

    def _zero_plain(self, rows: int, n: int):
        key = ("zero_plain", rows, n)
        zero = self._tables.get(key)
        if zero is None:
            zero = self._tables[key] = self.torch.zeros((rows, n), dtype=self.torch.int32, device=self.device)
        return zero

    def bsgs_inner(self, plan: int, raised, ct_a, ct_b, ks, evks, table, ext: int):
        """All baby steps (rotation indices `ks`, 0 = none; keys `evks`) and all giant-step inner
        sums (table[g][b]: plaintext over Q||P or None) of a double-hoisted BSGS transform in one
        pass; returns the [2, ext, n] Q||P accumulators of the giant steps."""
        nb, ng = len(ks), len(table)
        n = ct_a.shape[1]
        big = self.empty(ng, 2, ext, n)          # one allocation: a batched ModDown can take a slice of it
        outs = [big[g] for g in range(ng)]
        kk = (ctypes.c_uint32 * nb)(*ks)
        ep = (ctypes.c_void_p * nb)(*[None if e is None else e.data_ptr() for e in evks])
        flat = [None if pt is None else pt.data_ptr() for row in table for pt in row]
        pp = (ctypes.c_void_p * (nb * ng))(*flat)
        op = (ctypes.c_void_p * ng)(*[o.data_ptr() for o in outs])
        zero = self._zero_plain(ext, n).data_ptr() if any(f is None for f in flat) else None
        _lib.check(self.lib.ckks_bsgs_inner(self.ctx, plan, raised.data_ptr(), ct_a.data_ptr(), ct_b.data_ptr(),
                                            nb, kk, ep, ng, pp, zero, op, self.stream()))
        return outs

    def bsgs_inner_batch(self, plan: int, raised, ct_a, ct_b, ks, evks, table, ext: int):
        """bsgs_inner for a batch of independent ciphertexts at the same level (lists `raised`, `ct_a`,
        `ct_b`) through the same keys and diagonals: pairs go through ONE launch that stages every key
        and plaintext slice once for both (ckks_bsgs_inner_batch); results equal the single calls bit
        for bit.  Returns one list of [2, ext, n] accumulators per ciphertext."""
        count = len(raised)
        n = ct_a[0].shape[1]
        if count == 1 or n % 256:
            return [self.bsgs_inner(plan, raised[c], ct_a[c], ct_b[c], ks, evks, table, ext) for c in range(count)]
        nb, ng = len(ks), len(table)
        kk = (ctypes.c_uint32 * nb)(*ks)
        ep = (ctypes.c_void_p * nb)(*[None if e is None else e.data_ptr() for e in evks])
        flat = [None if pt is None else pt.data_ptr() for row in table for pt in row]
        pp = (ctypes.c_void_p * (nb * ng))(*flat)
        zero = self._zero_plain(ext, n).data_ptr() if any(f is None for f in flat) else None
        res = []
        for c0 in range(0, count, 2):
            group = list(range(c0, min(c0 + 2, count)))
            if len(group) == 1:
                res.append(self.bsgs_inner(plan, raised[c0], ct_a[c0], ct_b[c0], ks, evks, table, ext))
                continue
            bigs = [self.empty(ng, 2, ext, n) for _ in group]
            ptrs = lambda ts: (ctypes.c_void_p * len(group))(*[ts[c].data_ptr() for c in group])
            op = (ctypes.c_void_p * (len(group) * ng))(*[big[g].data_ptr() for big in bigs for g in range(ng)])
            _lib.check(self.lib.ckks_bsgs_inner_batch(self.ctx, plan, len(group), ptrs(raised), ptrs(ct_a), ptrs(ct_b),
                                                      nb, kk, ep, ng, pp, zero, op, self.stream()))
            res.extend([[big[g] for g in range(ng)] for big in bigs])
        return res

    def ks_relin_rescale(self, ks_plan: int, md_plan: int, d, evk, out_rows: int):
        """d = [3, l, n] tensor product (d0, d1, d2) -> rescaled relinearised ciphertext [2, out_rows, n]."""
        out = self.empty(2, out_rows, d.shape[2])
        _lib.check(self.lib.ckks_ks_relin_rescale(self.ctx, ks_plan, md_plan, d[2].data_ptr(),
                                                  d[1].data_ptr(), d[0].data_ptr(), evk.data_ptr(),
                                                  out[0].data_ptr(), out[1].data_ptr(), self.stream()))
        return out

    def hmult_relin_rescale(self, ks_plan: int, md_plan: int, xa, xb, ya, yb, evk, out_rows: int,
                            add_a=None, add_b=None):
        """HMult + relinearise + rescale from the operand halves in one pipeline (no tensor pass);
        (add_a, add_b): a ciphertext at the output level added inside the last kernel."""
        out = self.empty(2, out_rows, xa.shape[1])
        _lib.check(self.lib.ckks_hmult_relin_rescale(self.ctx, ks_plan, md_plan, xa.data_ptr(), xb.data_ptr(),
                                                     ya.data_ptr(), yb.data_ptr(), evk.data_ptr(),
                                                     None if add_a is None else add_a.data_ptr(),
                                                     None if add_b is None else add_b.data_ptr(),
                                                     out[0].data_ptr(), out[1].data_ptr(), self.stream()))
        return out

    def ks_accumulate_rot(self, plan: int, ct_a, ct_b, k: int, evk, first: bool):
        """Stages 1-2 of the key switch of sigma_k(ct) into the current lane's Q||P accumulator,
        the rotation applied as a gather (no automorphism pass), P * sigma_k(ct_b) lifted in."""
        _lib.check(self.lib.ckks_ks_accumulate_rot(self.ctx, plan, ct_a.data_ptr(), ct_b.data_ptr(), k,
                                                   evk.data_ptr(), int(first), self.stream()))

    def ks_accumulate_rot_qp(self, plan: int, ct_a, b_qp, k: int, evk, first: bool):
        """ks_accumulate_rot for an inner sum whose b half b_qp ([ext, n]) is still over Q||P: it is
        added to the b accumulator through the rotation as it is (no ModDown, no lift by P)."""
        _lib.check(self.lib.ckks_ks_accumulate_rot_qp(self.ctx, plan, ct_a.data_ptr(), b_qp.data_ptr(), k,
                                                      evk.data_ptr(), int(first), self.stream()))

    def ks_accumulate(self, plan: int, ct_a, evk, first: bool):
        _lib.check(self.lib.ckks_ks_accumulate(self.ctx, plan, ct_a.data_ptr(), evk.data_ptr(),
                                               int(first), self.stream()))

    def ks_finish(self, plan: int, lanes_used: int, fold_a, fold_b, rows: int, n: int):
        out = self.empty(2, rows, n)
        _lib.check(self.lib.ckks_ks_finish(self.ctx, plan, lanes_used,
                                           None if fold_a is None else fold_a.data_ptr(),
                                           None if fold_b is None else fold_b.data_ptr(),
                                           out[0].data_ptr(), out[1].data_ptr(), self.stream()))
        return out

    def ks_finish_rescale(self, plan: int, md_plan: int, lanes_used: int, fold_a, fold_b, rows: int, n: int,
                          raw_qp=None):
        """ks_finish merged with the rescale that follows (one division by P and the dropped limbs);
        raw_qp: a [2, ext, n] accumulator over Q||P added as it is."""
        out = self.empty(2, rows, n)
        _lib.check(self.lib.ckks_ks_finish_rescale(self.ctx, plan, md_plan, lanes_used,
                                                   None if fold_a is None else fold_a.data_ptr(),
                                                   None if fold_b is None else fold_b.data_ptr(),
                                                   None if raw_qp is None else raw_qp.data_ptr(),
                                                   out[0].data_ptr(), out[1].data_ptr(), self.stream()))
        return out

    def keyswitch(self, plan: int, ct_a, ct_b, evk, out=None):
        out = self.empty(2, ct_a.shape[0], ct_a.shape[1]) if out is None else out
        _lib.check(self.lib.ckks_keyswitch(self.ctx, plan, ct_a.data_ptr(),
                                           None if ct_b is None else ct_b.data_ptr(), evk.data_ptr(),
                                           out[0].data_ptr(), out[1].data_ptr(), self.stream()))
        return out


_engine: Engine | None = None


def get_engine() -> Engine:
    """The process's engine (one process per GPU); created on first use and
    failing loudly when the extension or the GPU is missing."""
    global _engine
    if _engine is None:
        _engine = Engine()
    return _engine


def use_backend(backend):
    """Install `backend` as the object get_engine() returns and hand back the previous one
    (None: the CUDA engine is created again on next use).

    Checker hook, never called by the package itself: tests/ and the CPU reference arm of
    bench.py pass an object with Engine's methods that is backed by the CPU oracle
    (oracle/engine_oracle.py) to replay the host orchestration of a circuit -- same circuit,
    reference primitives -- and compare limbs with the CUDA path.  There is no automatic
    selection: without this explicit call every device operation needs the CUDA library and a
    GPU and fails loudly otherwise."""
    global _engine
    previous, _engine = _engine, backend
    return previous
