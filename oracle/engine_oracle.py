"""CPU engine with the interface of paper_2512_18345_b200.engine.Engine, backed by the oracle
(oracle/ckks_oracle.c).

TEST INFRASTRUCTURE ONLY.  The product package never imports this module; tests/, smoke() and
the CPU-baseline / --impl reference legs of bench.py install it with
`paper_2512_18345_b200.engine.use_backend(OracleEngine())` to replay a circuit's host
orchestration (ckks.py, bootstrap.py, helr.py) on the CPU restatement instead of the CUDA
kernels: the same circuit, limb for limb, driven through reference primitives.

Every method states the composition of reference routines it stands for (paths relative to
/root/reference/pkg/src/rnscope/).  Fused CUDA entry points (ckks_bsgs_inner,
ckks_hmult_relin_rescale, ckks_ks_finish_rescale, ...) are deliberately restated UNFUSED here,
as the chain of ModUp / inner product / ModDown / element-wise steps they replace; arithmetic is
exact and canonical, so a correct fusion must reproduce these limbs bit for bit.

Tensors are CPU torch.int32 (the product's host code slices, stacks and checks adjacency on
torch tensors); CUDA tensors handed in (keys and plaintexts of a Bootstrapper built on the GPU)
are copied to the host per call.
"""
from __future__ import annotations

import numpy as np

from . import oracle as orc


class _Plan:
    __slots__ = ("n", "q", "p", "alpha", "evk_ext", "evk_p_off", "moddown_only")

    def __init__(self, n, q, p, alpha, evk_ext, evk_p_off, moddown_only):
        self.n, self.q, self.p, self.alpha = n, tuple(q), tuple(p), alpha
        self.evk_ext, self.evk_p_off, self.moddown_only = evk_ext, evk_p_off, moddown_only

    @property
    def l(self):
        return len(self.q)

    @property
    def ext(self):
        return len(self.q) + len(self.p)

    @property
    def beta(self):
        return -(-len(self.q) // self.alpha)


class OracleEngine:
    """Same public methods as engine.Engine; every result is a fresh CPU tensor."""

    host_tensors = True          # rns.Polynomial adopts CPU word tensors under this engine

    def __init__(self, threads: int | None = None):
        import torch

        self.torch = torch
        self.device = torch.device("cpu")
        self.lanes = 1
        self._ctx: dict[int, orc.Oracle] = {}
        self._plans: list[_Plan] = []
        self._plan_index: dict = {}
        self._tables: list = []
        self._table_index: dict = {}
        self._perm: dict = {}
        self._acc: dict = {}
        self.ops = 0                       # engine calls so far (bench.py slices a circuit by this)
        self.on_op = None                  # optional callback after every engine call
        if threads:
            orc.set_threads(threads)

    # ---- plumbing ---------------------------------------------------------------------
    def _tick(self):
        self.ops += 1
        if self.on_op is not None:
            self.on_op(self.ops)

    def stream(self) -> int:
        return 0

    def _np(self, t) -> np.ndarray:
        """uint32 view of a tensor's words (copying CUDA tensors to the host)."""
        if t is None:
            return None
        if isinstance(t, np.ndarray):
            return np.ascontiguousarray(t, dtype=np.uint32)
        if t.is_cuda:
            t = t.cpu()
        return t.contiguous().numpy().view(np.uint32)

    def _t(self, a: np.ndarray):
        return self.torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32))

    def upload(self, words: np.ndarray):
        return self._t(np.array(words, dtype=np.uint32, copy=True))

    def empty(self, *shape):
        return self.torch.empty(shape, dtype=self.torch.int32)

    def set_lanes(self, count: int) -> None:
        self.lanes = 1                     # one accumulator: lane-parallel sums are order-independent

    def lane_count(self) -> int:
        return 1

    def fork(self, jobs, with_lane: bool = False):
        return [job(0, i) if with_lane else job() for i, job in enumerate(jobs)]

    def pipeline(self, items, first, second):
        return [second(item, first(item)) for item in items]

    # ---- moduli -----------------------------------------------------------------------
    def _context(self, n: int) -> orc.Oracle:
        c = self._ctx.get(n)
        if c is None:
            c = self._ctx[n] = orc.Oracle(n, [])
            c.index2 = {}
        return c

    def has_tables(self, m, n: int) -> bool:
        return n >= 2 and (m.q - 1) % (2 * n) == 0 and m.n >= n and m.q < (1 << 31)

    def _idx(self, m, n: int) -> int:
        """Index of modulus m in the context of ring degree n (registered on first use)."""
        c = self._context(n)
        tabled = self.has_tables(m, n)
        key = (m.q, m.psi if tabled else 0, m.n if tabled else 0)
        i = c.index2.get(key)
        if i is None:
            i = orc.lib().orc_add_modulus(c._h, m.q, key[1], max(key[2], 1))
            c.index2[key] = i
        return i

    def slot(self, m, n: int):
        return m

    def row_slots(self, basis, n: int = 0, repeat: int = 1):
        return tuple(basis) * repeat

    def _rm(self, mods, n: int) -> np.ndarray:
        return np.array([self._idx(m, n) for m in mods], dtype=np.int32)

    def twiddle_tables(self, m, n: int):
        return self._context(n).twiddles(self._idx(m, n))

    # ---- element-wise kernels: rns.py:243-320 -----------------------------------------------
    def elementwise(self, a, b, row_slot, kind: int, out=None):
        self._tick()
        x, y = self._np(a), self._np(b)
        n = x.shape[1]
        res = self._context(n).elementwise(x, y, self._rm(row_slot, n), ("add", "sub", "mul")[kind])
        if out is not None:
            out.copy_(self._t(res))
            return out
        return self._t(res)

    def _permutation(self, n: int, k: int, probe) -> np.ndarray:
        """rns.py:268-292: the evaluation-domain permutation of X -> X^k, derived by probing the
        transform exactly as the reference does."""
        k %= 2 * n
        key = (n, k)
        hit = self._perm.get(key)
        if hit is None:
            hit = self._perm[key] = self._context(n).eval_permutation(k, self._idx(probe, n))
        return hit

    def automorphism_eval(self, a, k: int, probe=None):
        self._tick()
        x = self._np(a)
        n = x.shape[1]
        if probe is None:
            probe = self._any_ntt_modulus(n)
        perm = self._permutation(n, k, probe)
        return self._t(x[:, perm])

    def _any_ntt_modulus(self, n: int):
        c = self._context(n)
        for (q, psi, mn) in c.index2:
            if psi:
                from paper_2512_18345_b200.rns import Modulus

                return Modulus.for_prime(q, mn, psi)
        raise RuntimeError("no NTT-friendly modulus registered for the probe transform")

    def automorphism_coeff(self, a, row_slot, k: int):
        self._tick()
        x = self._np(a)
        n = x.shape[1]
        return self._t(self._context(n).automorphism_coeff(x, self._rm(row_slot, n), k))

    # ---- transforms: transform.py:203-323 --------------------------------------------------
    def ntt(self, a, row_slot, inverse: bool, out=None):
        self._tick()
        x = self._np(a)
        n = x.shape[1]
        res = self._context(n).ntt(x, self._rm(row_slot, n), inverse)
        if out is not None:
            out.copy_(self._t(res))
            return out
        return self._t(res)

    def ntt_stages(self, a, row_slot, inverse: bool, lo: int, hi: int, out=None):
        self._tick()
        x = self._np(a).copy()
        n = x.shape[1]
        orc.lib().orc_ntt_stages(self._context(n)._h, x, self._rm(row_slot, n), x.shape[0], int(inverse), lo, hi)
        if out is not None:
            out.copy_(self._t(x))
            return out
        return self._t(x)

    def lift2_centered(self, coeff2, slot0, slot1, row_slot, rows: int):
        self._tick()
        x = self._np(coeff2)
        n = x.shape[1]
        out = np.empty((rows, n), np.uint32)
        orc.lib().orc_lift2_centered(self._context(n)._h, x, self._idx(slot0, n), self._idx(slot1, n), out,
                                     self._rm(row_slot, n), rows)
        return self._t(out)

    def _pmult_acc(self, x, p, acc, rm, first: bool):
        n = x.shape[-1]
        orc.lib().orc_pmult_acc(self._context(n)._h, x, p, acc, rm, x.shape[1], int(first))

    def pmult_accumulate(self, x, p, acc, row_slot, first: bool):
        self._tick()
        xv, pv = self._np(x), self._np(p)
        av = np.ascontiguousarray(self._np(acc)).copy()
        self._pmult_acc(xv, pv, av, self._rm(row_slot, xv.shape[-1]), first)
        acc.copy_(self._t(av))
        return acc

    def fused_terms(self, xs, ps, row_slot, out=None):
        """sum_t xs[t] (.) ps[t] (ps[t] None: the term itself): poly_elementwise mul / add chain."""
        self._tick()
        halves = lambda x: np.stack([self._np(x[0]), self._np(x[1])]) if isinstance(x, (tuple, list)) else self._np(x)
        first = halves(xs[0])
        n = first.shape[2]
        rm = self._rm(row_slot, n)
        rm2 = np.concatenate([rm, rm])
        rows = first.shape[1]
        acc = np.zeros((2, rows, n), np.uint32)
        ctx = self._context(n)
        for t, (x, p) in enumerate(zip(xs, ps)):
            xv = halves(x)
            if p is None:
                acc = ctx.elementwise(acc.reshape(2 * rows, n), xv.reshape(2 * rows, n), rm2, "add").reshape(2, rows, n)
            else:
                self._pmult_acc(xv, self._np(p), acc, rm, False)
        res = self._t(acc)
        if out is not None:
            out.copy_(res)
            return out
        return res

    def fused_terms_multi(self, xs, table, row_slot):
        self._tick()
        n = xs[0].shape[2]
        rm = self._rm(row_slot, n)
        rows = xs[0].shape[1]
        outs = []
        xv = [self._np(x) for x in xs]
        for row in table:
            acc = np.zeros((2, rows, n), np.uint32)
            for x, pt in zip(xv, row):
                if pt is not None:
                    self._pmult_acc(x, self._np(pt), acc, rm, False)
            outs.append(self._t(acc))
        return outs

    def tensor_halves(self, xa, xb, ya, yb, row_slot):
        """(d0, d1, d2) = (xb*yb, xa*yb + ya*xb, xa*ya): SURVEY 8c HMult composition."""
        self._tick()
        XA, XB, YA, YB = (self._np(t) for t in (xa, xb, ya, yb))
        n = XA.shape[1]
        ctx, rm = self._context(n), self._rm(row_slot, n)
        d0 = ctx.elementwise(XB, YB, rm, "mul")
        d1 = ctx.elementwise(ctx.elementwise(XA, YB, rm, "mul"), ctx.elementwise(YA, XB, rm, "mul"), rm, "add")
        d2 = ctx.elementwise(XA, YA, rm, "mul")
        return self._t(np.stack([d0, d1, d2]))

    def tensor(self, x, y, row_slot):
        return self.tensor_halves(x[0], x[1], y[0], y[1], row_slot)

    # ---- base conversion: baseconv.py:57-151 -----------------------------------------------
    def bconv_table(self, q_basis, p_basis) -> int:
        key = (tuple(m.q for m in q_basis), tuple(m.q for m in p_basis))
        t = self._table_index.get(key)
        if t is None:
            t = self._table_index[key] = len(self._tables)
            self._tables.append(key)
        return t

    def bconv_table_read(self, table: int, l_in: int, l_out: int):
        qs, ps = self._tables[table]
        return orc.bconv_table(qs, ps)

    def bconv(self, table: int, a, l_out: int):
        self._tick()
        qs, ps = self._tables[table]
        return self._t(orc.bconv(qs, ps, self._np(a)))

    # ---- key switching: keyswitch.py:186-453 -----------------------------------------------
    def ks_plan(self, n: int, q_basis, p_basis, alpha: int, evk_ext: int, evk_p_off: int) -> int:
        key = (n, tuple(m.q for m in q_basis), tuple(m.q for m in p_basis), alpha, evk_ext, evk_p_off)
        p = self._plan_index.get(key)
        if p is None:
            p = self._plan_index[key] = len(self._plans)
            self._plans.append(_Plan(n, q_basis, p_basis, alpha, evk_ext, evk_p_off, False))
        return p

    def moddown_plan(self, n: int, q_basis, p_basis) -> int:
        key = ("moddown", n, tuple(m.q for m in q_basis), tuple(m.q for m in p_basis))
        p = self._plan_index.get(key)
        if p is None:
            p = self._plan_index[key] = len(self._plans)
            self._plans.append(_Plan(n, q_basis, p_basis, len(p_basis), len(q_basis) + len(p_basis),
                                     len(q_basis), True))
        return p

    def _pmod(self, pl: _Plan) -> np.ndarray:
        import math

        prod = math.prod(m.q for m in pl.p)
        return np.array([prod % m.q for m in pl.q], dtype=np.uint32)

    def _raise(self, pl: _Plan, a: np.ndarray) -> np.ndarray:
        """keyswitch_stage1 (keyswitch.py:297-315) at pl.l active limbs."""
        n = pl.n
        raised = np.empty((pl.beta, pl.ext, n), np.uint32)
        orc.lib().orc_ks_stage1(self._context(n)._h, pl.l, pl.alpha, pl.beta, self._rm(pl.q, n), self._rm(pl.p, n),
                                np.ascontiguousarray(a), raised)
        return raised

    def _inner(self, pl: _Plan, raised, evk, k: int = 0, lift_a=None, lift_b=None, acc=None):
        """keyswitch_stage2 (keyswitch.py:335-355) over all extended rows; returns [2, ext, n]."""
        n = pl.n
        ext_mods = pl.q + pl.p
        evk_row = np.array(list(range(pl.l)) + [pl.evk_p_off + j for j in range(len(pl.p))], dtype=np.int32)
        perm = None
        if k % (2 * n) not in (0, 1):
            perm = np.ascontiguousarray(self._permutation(n, k, pl.q[0]), dtype=np.int32)
        accumulate = acc is not None
        if acc is None:
            acc = np.empty((2, pl.ext, n), np.uint32)
        pmod = self._pmod(pl) if (lift_a is not None or lift_b is not None) else None
        ptr = lambda x: None if x is None else np.ascontiguousarray(x).ctypes.data
        keep = [np.ascontiguousarray(x) for x in (lift_a, lift_b) if x is not None]      # noqa: F841
        la = None if lift_a is None else np.ascontiguousarray(lift_a)
        lb = None if lift_b is None else np.ascontiguousarray(lift_b)
        orc.lib().orc_inner_product(self._context(n)._h, pl.l, pl.beta, pl.ext, self._rm(ext_mods, n),
                                    np.ascontiguousarray(raised), np.ascontiguousarray(evk), pl.evk_ext, evk_row,
                                    None if perm is None else perm.ctypes.data,
                                    None if la is None else la.ctypes.data,
                                    None if lb is None else lb.ctypes.data,
                                    None if pmod is None else pmod.ctypes.data,
                                    int(accumulate), acc[0], acc[1])
        return acc

    def _moddown(self, md: _Plan, xq, xp) -> np.ndarray:
        """keyswitch_stage3 for one polynomial (keyswitch.py:387-419) with P = md.p."""
        n = md.n
        out = np.empty((md.l, n), np.uint32)
        orc.lib().orc_ks_moddown(self._context(n)._h, md.l, len(md.p), self._rm(md.q, n), self._rm(md.p, n),
                                 np.ascontiguousarray(xq), np.ascontiguousarray(xp), out)
        return out

    def _moddown_pair(self, md: _Plan, acc) -> np.ndarray:
        """ModDown of a [2, md.ext, n] accumulator -> [2, md.l, n]."""
        return np.stack([self._moddown(md, acc[h, :md.l], acc[h, md.l:]) for h in range(2)])

    def _add(self, x, y, mods, n):
        return self._context(n).elementwise(np.ascontiguousarray(x), np.ascontiguousarray(y), self._rm(mods, n), "add")

    def _gather(self, x, n, k, probe):
        if k % (2 * n) in (0, 1):
            return x
        return np.ascontiguousarray(x[:, self._permutation(n, k, probe)])

    def ks_stage1(self, plan: int, a, beta: int, ext: int):
        self._tick()
        return self._t(self._raise(self._plans[plan], self._np(a)))

    def ks_stage2(self, plan: int, raised, evk, row_lo: int, row_hi: int):
        self._tick()
        acc = self._inner(self._plans[plan], self._np(raised), self._np(evk))
        return self._t(acc[:, row_lo:row_hi])

    def ks_stage3(self, plan: int, q_a, q_b, p_a, p_b):
        self._tick()
        md = self._plans[plan]
        return self._t(np.stack([self._moddown(md, self._np(q_a), self._np(p_a)),
                                 self._moddown(md, self._np(q_b), self._np(p_b))]))

    def ks_stage3_batch(self, plan: int, qps, l: int):
        self._tick()
        md = self._plans[plan]
        q = self._np(qps)
        return self._t(np.stack([self._moddown_pair(md, q[g]) for g in range(q.shape[0])]))

    def ks_stage3_batch_a(self, plan: int, qps, l: int):
        self._tick()
        md = self._plans[plan]
        q = self._np(qps)
        return self._t(np.stack([self._moddown(md, q[g, 0, :md.l], q[g, 0, md.l:]) for g in range(q.shape[0])]))

    def keyswitch(self, plan: int, ct_a, ct_b, evk, out=None):
        """keyswitch (keyswitch.py:444-453) at the plan's level."""
        self._tick()
        pl = self._plans[plan]
        acc = self._inner(pl, self._raise(pl, self._np(ct_a)), self._np(evk))
        res = self._moddown_pair(pl, acc)
        if ct_b is not None:
            res[1] = self._add(res[1], self._np(ct_b), pl.q, pl.n)
        r = self._t(res)
        if out is not None:
            out.copy_(r)
            return out
        return r

    def ks_hoisted(self, plan: int, raised, k: int, evk, ct_b):
        """Key switch of sigma_k(ct) from the raised digits of the unrotated a part: digits read
        through the automorphism, ModDown, then + sigma_k(ct_b)."""
        self._tick()
        pl = self._plans[plan]
        acc = self._inner(pl, self._np(raised), self._np(evk), k=k)
        res = self._moddown_pair(pl, acc)
        res[1] = self._add(res[1], self._gather(self._np(ct_b), pl.n, k, pl.q[0]), pl.q, pl.n)
        return self._t(res)

    def ks_hoisted_raw(self, plan: int, raised, k: int, evk, ct_b, ext: int):
        self._tick()
        pl = self._plans[plan]
        return self._t(self._inner(pl, self._np(raised), self._np(evk), k=k, lift_b=self._np(ct_b)))

    def bsgs_inner(self, plan: int, raised, ct_a, ct_b, ks, evks, table, ext: int):
        """out[g] = sum_b table[g][b] (.) u_b with u_b the Q||P accumulator of sigma_{k_b}(ct)
        (k_b = 0: the ciphertext itself on the Q rows, zero on the P rows)."""
        self._tick()
        pl = self._plans[plan]
        n = pl.n
        rm = self._rm(pl.q + pl.p, n)
        rz = self._np(raised)
        a, b = self._np(ct_a), self._np(ct_b)
        outs = [np.zeros((2, pl.ext, n), np.uint32) for _ in table]
        for bi, k in enumerate(ks):
            if k == 0:
                u = np.zeros((2, pl.ext, n), np.uint32)
                u[0, :pl.l], u[1, :pl.l] = a, b
            else:
                u = self._inner(pl, rz, self._np(evks[bi]), k=k, lift_b=b)
            for g, row in enumerate(table):
                if row[bi] is not None:
                    self._pmult_acc(u, self._np(row[bi]), outs[g], rm, False)
        return [self._t(o) for o in outs]

    def bsgs_inner_batch(self, plan: int, raised, ct_a, ct_b, ks, evks, table, ext: int):
        """Engine.bsgs_inner_batch: the batch is a scheduling device of the CUDA engine (shared key
        traffic); its values are those of one bsgs_inner per ciphertext, which is what runs here."""
        return [self.bsgs_inner(plan, raised[c], ct_a[c], ct_b[c], ks, evks, table, ext) for c in range(len(raised))]

    def _relin_rescale(self, pl: _Plan, md: _Plan, d0, d1, d2, evk, add_a=None, add_b=None):
        acc = self._inner(pl, self._raise(pl, d2), evk, lift_a=d1, lift_b=d0)
        res = self._moddown_pair(md, acc)
        if add_a is not None:
            res[0] = self._add(res[0], add_a, md.q, md.n)
        if add_b is not None:
            res[1] = self._add(res[1], add_b, md.q, md.n)
        return res

    def ks_relin_rescale(self, ks_plan: int, md_plan: int, d, evk, out_rows: int):
        """Relinearisation merged with the rescale: (d1, d0) lifted by P into the accumulator of
        keyswitch(d2), one ModDown by P and the dropped limbs."""
        self._tick()
        dv = self._np(d)
        return self._t(self._relin_rescale(self._plans[ks_plan], self._plans[md_plan], dv[0], dv[1], dv[2],
                                           self._np(evk)))

    def hmult_relin_rescale(self, ks_plan: int, md_plan: int, xa, xb, ya, yb, evk, out_rows: int,
                            add_a=None, add_b=None):
        self._tick()
        pl = self._plans[ks_plan]
        dv = self._np(self.tensor_halves(xa, xb, ya, yb, pl.q))
        return self._t(self._relin_rescale(pl, self._plans[md_plan], dv[0], dv[1], dv[2], self._np(evk),
                                           self._np(add_a), self._np(add_b)))

    def ks_accumulate_rot(self, plan: int, ct_a, ct_b, k: int, evk, first: bool):
        self._tick()
        pl = self._plans[plan]
        acc = None if first else self._acc[plan]
        self._acc[plan] = self._inner(pl, self._raise(pl, self._np(ct_a)), self._np(evk), k=k,
                                      lift_b=self._np(ct_b), acc=acc)

    def ks_accumulate_rot_qp(self, plan: int, ct_a, b_qp, k: int, evk, first: bool):
        """Stage 1-2 of the key switch of sigma_k(a) accumulated over Q||P, plus sigma_k(b_qp) added
        to the b accumulator as it is (b_qp already over Q||P)."""
        self._tick()
        pl = self._plans[plan]
        acc = None if first else self._acc[plan]
        acc = self._inner(pl, self._raise(pl, self._np(ct_a)), self._np(evk), k=k, acc=acc)
        acc[1] = self._add(acc[1], self._gather(self._np(b_qp), pl.n, k, pl.q[0]), pl.q + pl.p, pl.n)
        self._acc[plan] = acc

    def ks_accumulate(self, plan: int, ct_a, evk, first: bool):
        self._tick()
        pl = self._plans[plan]
        acc = None if first else self._acc[plan]
        self._acc[plan] = self._inner(pl, self._raise(pl, self._np(ct_a)), self._np(evk), acc=acc)

    def ks_finish(self, plan: int, lanes_used: int, fold_a, fold_b, rows: int, n: int):
        self._tick()
        pl = self._plans[plan]
        res = self._moddown_pair(pl, self._acc[plan])
        if fold_a is not None:
            res[0] = self._add(res[0], self._np(fold_a), pl.q, n)
        if fold_b is not None:
            res[1] = self._add(res[1], self._np(fold_b), pl.q, n)
        return self._t(res)

    def ks_finish_rescale(self, plan: int, md_plan: int, lanes_used: int, fold_a, fold_b, rows: int, n: int,
                          raw_qp=None):
        """The shared ModDown of the giant steps merged with the rescale: (fold_a, fold_b) lifted by
        P, raw_qp added as it is, one ModDown by P and the dropped limbs."""
        self._tick()
        pl, md = self._plans[plan], self._plans[md_plan]
        acc = self._acc[plan].copy()
        ext_mods = pl.q + pl.p
        rm = self._rm(ext_mods, n)
        if raw_qp is not None:
            acc = self._context(n).elementwise(acc.reshape(2 * pl.ext, n), self._np(raw_qp).reshape(2 * pl.ext, n),
                                               np.concatenate([rm, rm]), "add").reshape(2, pl.ext, n)
        pmod = self._pmod(pl)
        for h, fold in enumerate((fold_a, fold_b)):
            if fold is not None:
                orc.lib().orc_add_lifted(self._context(n)._h, np.ascontiguousarray(acc[h]),
                                         np.ascontiguousarray(self._np(fold)), pmod, rm, pl.l, pl.ext, acc[h])
        return self._t(self._moddown_pair(md, acc))
