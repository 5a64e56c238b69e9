"""The four share-level linear-layer procedures of Pencil on the B200
(the SPEC-only ``linear_protocols`` module; PAPER.md
Alg. 1, Alg. 2).

    linear_forward          Alg.1
    linear_backward_input   Alg.1 with W^T
    reveal_grad_bias        local sums + DP
    grad_weight             Alg.2 (cross terms)
    sample_dp_noise         N(0, sigma^2 C^2 / B)

Per protocol message the work is three fused device kernels:
    DO   pb_encrypt_sk        pack (pi_v / pi_W gather) + Delta m + NTT + key mul
    MO   pb_ctpt_mac_mask     sum_k ct (*) pt  -  Delta NTT(pi_y(mask) + filler)
    DO   pb_decrypt_to_share  c0 + c1 s + INTT + Garner/scale-round + pi_y^-1
plus the MO's plaintext encoding (pb_encode_plain) and ring GEMMs for the
local terms.  Both parties run in this process (as in the paper's artifact,
PAPER:1525); every MO<->DO message still goes through ``Channel`` so the
census and transcript are the protocol's.

Conventions are the oracle's (oracle/protocols.py) so that, under the same
seed, the DO's decrypted shares are bit-identical to the CPU oracle's:
activations (n, B), W (n_o, n_i), bias at scale 2f, MO mask streams
stream_id(layer, op, purpose); s_eff = s - W o <X>_0 replaces the
homomorphic addition of <X>_0 (same DO output W o X - s).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _dev, _lib
from .bfv import Ciphertext, KeyPair
from .errors import DesyncError, ParamsError, ScaleError, ShapeError
from .params import BfvParams, context
from .poly_encoding import MatmulGeometry, conv_out_hw, plan_conv_layer, plan_matmul
from .ring import DO, MO, RingParams, RingTensor, SeededRng, ShareTensor, encode_fixed

OP_FWD, OP_BWD_X, OP_GRAD_W, OP_GRAD_B, OP_RELU, OP_TRUNC_F, OP_TRUNC_B, OP_RELU_B, OP_POOL_F, OP_POOL_B = range(10)
P_MASK, P_ENC, P_DEALER, P_DP, P_OT = range(5)

# SPEC:372 message codes
MSG_FWD_INPUT_CT = 0x10
MSG_FWD_MASKED_CT = 0x11
MSG_BWD_X = 0x20
MSG_GRADW = 0x30
MSG_GRADB = 0x31
FRAME_HEADER = 12  # {u16 type, u16 flags, u64 len}


# Scheduling constants (round-1 A/B measurements under profiles/r01_ab_*):
_SERIAL = False        # True: every protocol fork on the calling stream (debugging)
_MASK_PREFETCH = True  # draw all MO masks of a phase up front on a fork
_GRADW_FLIP = False    # Alg. 2 HE matmul transposed: measured 1.5 % slower
_BG_CAP = 2 * 148      # CTA cap of background operand preparation (0: none); 74-444 within noise, 37 slower (r02_ab_bg_cap)
_FUSE_MIN_ROWS = 4 * 148  # output rows (ciphertexts x limbs) from which nI <= 2 evaluations fuse mask + MAC
_PREDRAW = True        # inside a phase: the DO's message-independent encryption half at phase start
_PREDRAW_MAX_ROWS = 4 * 148  # ... for encryptions of at most one wave of rows (latency-bound; the CIFAR
                             # CNN's large ones stay fused: its step measured 9.09 ms fused, 9.22 split)


def _stream_like(cur: torch.cuda.Stream) -> torch.cuda.Stream:
    """A new stream with the priority of ``cur``: forks of the critical chain
    inherit its (higher) priority, forks of the grad-W chain its lower one."""
    return torch.cuda.Stream(priority=cur.priority)


def stream_id(layer: int, op: int, purpose: int) -> int:
    return 1_000_000 + 1000 * layer + 10 * op + purpose


@dataclass
class Channel:
    """In-process duplex MO<->DO channel with a byte census.
    Payloads are handed over by reference (device tensors stay in HBM)."""

    census: dict = field(default_factory=dict)
    transcript: list = field(default_factory=list)
    record: bool = False

    def send(self, sender: str, msg_type: int, payload, nbytes: int):
        c = self.census.setdefault(msg_type, [0, 0])
        c[0] += 1
        c[1] += FRAME_HEADER + int(nbytes)
        if self.record:
            self.transcript.append((sender, msg_type, int(nbytes)))
        return payload

    def total_bytes(self) -> int:
        return sum(v[1] for v in self.census.values())


@dataclass
class DpConfig:
    sigma: float = 0.0
    C: float = 1.0
    B: int = 1
    enabled: bool = False

    def __post_init__(self):
        if self.sigma < 0 or self.C <= 0:
            raise ParamsError("DpConfig needs sigma >= 0 and C > 0")


def _pk(pack):
    pos, src = pack
    return _dev.ptr(pos), _dev.ptr(src), pos.shape[1]


def shard_grid(nB: int, nO: int, rank: int, world: int):
    """The rectangle [b0, b1) x [o0, o1) of the (nB x nO) output-ciphertext grid
    that ``rank`` evaluates: split the batch blocks when there are enough of
    them, else the output blocks (ranks beyond the available blocks idle)."""
    if world <= 1:
        return 0, nB, 0, nO
    if nB >= world or nB >= nO:
        return rank * nB // world, (rank + 1) * nB // world, 0, nO
    return 0, nB, rank * nO // world, (rank + 1) * nO // world


def shard_maps(plan, rank: int, world: int) -> dict:
    """Host-side (numpy) index maps of one rank's part of a block plan: a
    rectangle of the (b-block x o-block) output grid plus exactly the
    input-side polynomials (indices b*nI + k) and weight-side polynomials
    (o*nI + k) it needs -- both contiguous ranges.  Output row r of the shard
    is grid cell (b0 + r // no, o0 + r % no); its MAC terms are
    (b*nI + k, o*nI + k) relative to the shard's own input / plaintext lists."""
    from .poly_encoding import compact

    nB, nO, nI = plan.nblk
    b0, b1, o0, o1 = shard_grid(nB, nO, rank, world)
    nb, no = max(0, b1 - b0), max(0, o1 - o0)
    rows = (np.arange(b0, b1)[:, None] * nO + np.arange(o0, o1)[None, :]).reshape(-1)
    return dict(rect=(b0, b1, o0, o1), nb=nb, no=no, nI=nI, n_out=len(rows), n_in=nb * nI, n_pt=no * nI,
                U=plan.U, in_src=plan.in_src[b0 * nI:b1 * nI], pt_src=plan.pt_src[o0 * nI:o1 * nI],
                in_pack=compact(plan.in_src[b0 * nI:b1 * nI]), pt_pack=compact(plan.pt_src[o0 * nI:o1 * nI]),
                out_pos=plan.out_pos[rows], out_dst=plan.out_dst[rows])


def gather_maps(plan, world: int):
    """The multi-rank combine of a sharded block plan: rank r
    decrypts its output ciphertexts' useful slots into a COMPACT tile
    [n_max][U] (slot (i, u) at i*U + u; n_max = the largest rank share), the
    ranks all-gather the tiles, and every rank scatters the [world][n_max][U]
    result into the output tensor through ``gdst`` (-1: padding or an unused
    slot).  Returns (n_max, gdst int64 [world * n_max * U]).  Moves exactly
    the useful share elements (vs. an all-reduce of zero-padded full tiles)."""
    maps = [shard_maps(plan, r, world) for r in range(world)]
    n_max = max(1, max(m["n_out"] for m in maps))
    U = plan.U
    gdst = np.full((world, n_max, U), -1, dtype=np.int64)
    for r, m in enumerate(maps):
        if m["n_out"]:
            dst = np.where(m["out_pos"] >= 0, m["out_dst"], -1)
            gdst[r, : m["n_out"]] = dst
    return n_max, gdst.reshape(-1)


class _Shard:
    """Device copies of ``shard_maps`` (uploaded once per plan and rank), plus
    the compact-tile destinations and the all-gather scatter map for world > 1."""

    def __init__(self, plan, rank: int, world: int):
        m = shard_maps(plan, rank, world)
        self.nb, self.no, self.nI = m["nb"], m["no"], m["nI"]
        self.n_out, self.n_in, self.n_pt, self.U = m["n_out"], m["n_in"], m["n_pt"], m["U"]
        self.in_pack = tuple(_dev.i32_to_device(a) for a in m["in_pack"])
        self.pt_pack = tuple(_dev.i32_to_device(a) for a in m["pt_pack"])
        self.out_pos = _dev.i32_to_device(m["out_pos"])
        self.out_dst = _dev.i64_to_device(m["out_dst"])
        self.n_max = 0
        if world > 1:
            self.n_max, gdst = gather_maps(plan, world)
            self.gdst = _dev.i64_to_device(gdst)
            self.tile_dst = _dev.i64_to_device(np.arange(max(1, self.n_out) * self.U, dtype=np.int64))


class _Aux:
    def __init__(self, sess):
        self.sess = sess

    def __enter__(self):
        self.main = torch.cuda.current_stream()
        if _SERIAL:
            self.stream = self.main
            return self
        key = self.main.cuda_stream
        st = self.sess._aux_streams.get(key)
        if st is None:
            st = self.sess._aux_streams[key] = _stream_like(self.main)
        self.stream = st
        st.wait_stream(self.main)
        return self

    def run(self, fn):
        with torch.cuda.stream(self.stream):
            return fn()

    def __exit__(self, *exc):
        if self.stream is not self.main:
            self.main.wait_stream(self.stream)
        return False


class Session:
    """Both parties' protocol state: BFV keys (DO), ring params, seeds, channel.

    ``shard=(rank, world, group)`` splits every he-matmul's grid of output
    ciphertexts into one rectangle per GPU (``shard_grid``; one process per
    GPU, each encrypting / encoding only the operands its rectangle needs);
    the ranks' decrypted useful slots are combined with one NCCL all-gather
    of compact tiles and a scatter (``gather_maps``) -- the only data-path
    collective, moving just the result shares."""

    def __init__(self, params: BfvParams, ring: RingParams, kp: KeyPair, seed: int, filler: bool = True,
                 channel: Channel | None = None, shard=None):
        if ring.ell != params.ell:
            raise ScaleError("ring ell must equal the BFV plaintext modulus bits")
        self.p = params
        self.ring = ring
        self.kp = kp
        self.seed = int(seed)
        self.filler = filler
        self.channel = channel or Channel()
        self.ctx = context(params)
        self.rank, self.world, self.group = shard if shard else (0, 1, None)
        self.alg_bytes = {}  # entry point -> algorithmic HBM bytes (while instrumented)
        self.alg_work = {}   # entry point -> [NTT rows, mod-MACs] (while instrumented)
        self.steps_seen = 0
        self._shards = {}
        self.graph_mode = False
        self._seed_dev = None
        self._streams = {}
        self._grad_stream = None
        self._aux_streams = {}
        self._prep_stream = None
        self.dp = None  # DpConfig: the DO's DP perturbation of revealed gradients, off by default
        # non-linear backend: "dealer" (SPEC:479 reconstruct / apply / reshare) or
        # "ot" (the OT-based protocols SPEC:491-581 with the dealer OT functionality)
        self.nonlinear = "dealer"
        self.capture = None  # diagnostics: a list receives (masked output ciphertexts, useful slot positions)
        # operands prepared ahead of their protocol (prepare_operand): key
        # (layer, op, role) -> (device tensor, event or None); buffers persist
        self._prepared = {}
        self._prep_bufs = {}
        self._masks = {}  # (layer, op, shape) -> (prefetched mask, event or None)
        self._mask_bufs = {}
        self._mask_streams = {}
        self._pending_join = []
        self._fork_pools = {}
        # encryption pre-draw (begin_phase): the phase-start event, the stream the
        # message-independent halves run on, and their persistent (ct, e) buffers
        self._t0 = None
        self._predraw_stream = None
        self._predraw_bufs = {}
        self._predraw_used = set()  # persistent pre-draw buffers claimed in the current phase

    def rng(self, layer: int, op: int, purpose: int) -> SeededRng:
        g = SeededRng(self.seed, stream_id(layer, op, purpose))
        return g.bind(self._seed_dev.data_ptr()) if self.graph_mode else g

    def reseed(self, seed: int, device_copy: bool = True):
        """Start a new step: every mask / share / noise stream is re-keyed.
        In graph mode the seed is also written to the device word the
        captured kernels read (seed indirection, pb_common.cuh); with
        ``device_copy=False`` only to the pinned host word (a replayed graph
        copies it itself: pb_step_prologue)."""
        self.seed = int(seed)
        self.steps_seen += 1
        if self._seed_dev is not None:
            self._seed_host[0] = self.seed
            if not device_copy:
                return
            self._seed_dev.copy_(self._seed_host, non_blocking=True)

    def enable_graph_mode(self):
        """Route the step seed through device memory so CUDA graphs can replay steps."""
        if self.seed >= 1 << 63:
            raise ValueError("graph mode needs seeds < 2^63 (numpy key derivation)")
        self._seed_host = torch.tensor([self.seed], dtype=torch.int64).pin_memory()
        self._seed_dev = torch.tensor([self.seed], dtype=torch.int64, device=_dev.device())
        self.graph_mode = True

    def _side_streams(self):
        """The (DO encrypt, MO encode) side streams forked by he_eval, one pair
        per calling stream so concurrent protocol calls do not serialise.
        (_SERIAL: run everything on the calling stream, for debugging.)"""
        if _SERIAL:
            cur = torch.cuda.current_stream()
            return cur, cur
        key = torch.cuda.current_stream().cuda_stream
        if key not in self._streams:
            # the calling stream's priority (the critical chain's forks outrank the
            # grad-W chain's; relative priorities inside one protocol measured no
            # effect, profiles/r01_ab_stream_priority.txt)
            cur = torch.cuda.current_stream()
            self._streams[key] = (_stream_like(cur), _stream_like(cur))
        return self._streams[key]

    def aux(self):
        """Context for work that overlaps the protocol's critical path: inside
        ``with sess.aux() as a``, ``a.run(fn)`` enqueues fn on an auxiliary
        stream forked from the current one (after everything enqueued so far);
        the current stream joins it when the block exits.  Outputs must be
        allocated on the current stream before the block.  (_SERIAL: inline.)"""
        return _Aux(self)

    def prep_stream(self) -> torch.cuda.Stream:
        """Stream the eager training step prepares backward operands on."""
        if _SERIAL:
            return torch.cuda.current_stream()
        if self._prep_stream is None:
            self._prep_stream = torch.cuda.Stream()
        return self._prep_stream

    def grad_stream(self) -> torch.cuda.Stream:
        """Stream the training step runs weight-gradient protocols on, concurrently
        with the input-gradient chain (they are independent given grad Y)."""
        if _SERIAL:
            return torch.cuda.current_stream()
        if self._grad_stream is None:
            self._grad_stream = torch.cuda.Stream()
        return self._grad_stream

    # ------------------------------------------------- operand preparation ---
    _ROLES = ("A_ct", "A_pt", "B_ct", "B_pt")

    def _operand_layout(self, plan, role):
        """(pack, count, is_ct, nonce offset) of one MAC operand of a block plan:
        A_ct = Enc(pi_v(v)), A_pt = pi_W(W), B_ct = Enc(pi_W(W)), B_pt = pi_v(v)."""
        sh = self._shard(plan)
        if role == "A_ct":
            return sh.in_pack, sh.n_in, True, self.rank * plan.n_in
        if role == "A_pt":
            return sh.pt_pack, sh.n_pt, False, 0
        if role == "B_ct":
            return sh.pt_pack, sh.n_pt, True, self.world * plan.n_in + self.rank * plan.n_pt
        if role == "B_pt":
            return sh.in_pack, sh.n_in, False, 0
        raise ValueError(f"unknown operand role {role!r}")

    def _make_operand(self, layer, op, plan, role, src, buf, rng=None):
        """Enqueue the DO's encryption / the MO's encoding of one operand into buf
        (current stream); ``rng``: the encryption's key stream instead of the
        step's (layer, op, P_ENC) stream."""
        pack, n, is_ct, off = self._operand_layout(plan, role)
        h, L, N = self.ctx.handle, self.p.L, self.p.N
        if is_ct:
            enc_rng = self.rng(layer, op, P_ENC) if rng is None else rng
            base = enc_rng.reserve((plan.n_in + plan.n_pt) * self.world)
            _lib.call("pb_encrypt_sk", h, _dev.ptr(self.kp.sk_ntt), _dev.ptr(self.kp.sk_sh), _dev.ptr(src), *_pk(pack), n,
                      *enc_rng.dev_args(), base + off, _dev.ptr(buf), _dev.stream())
            self._count("pb_encrypt_sk", n * (2 * L * N * 4 + 8 * N), ntt_rows=n * L)
        else:
            _lib.call("pb_encode_plain_mont", h, _dev.ptr(src), *_pk(pack), n, _dev.ptr(buf), _dev.stream())
            self._count("pb_encode_plain_mont", n * (L * N * 4 + 8 * N), ntt_rows=n * L)

    def prepare_operand(self, layer: int, op: int, plan, role: str, src: torch.Tensor, event: bool = True,
                        background: bool = False, rng=None):
        """Encrypt / encode one operand of the protocol (layer, op) ahead of time,
        on the current stream, into a persistent buffer; the next he_eval of
        (layer, op) uses it instead of producing it on its critical path.  The
        value is the one he_eval would compute (same packing, key and nonce),
        so the protocol's output is unchanged.  ``event``: the consumer waits
        on an event recorded here (False when another mechanism orders them,
        e.g. a separately captured graph replayed before the consumer's).
        ``background``: launch with at most _BG_CAP CTAs (pb_set_launch_cap),
        leaving SM slots to the concurrently running critical path."""
        pack, n, is_ct, _ = self._operand_layout(plan, role)
        if not self._shard(plan).n_out or n == 0:
            return
        key = (layer, op, role)
        shape = (n, 2, self.p.L, self.p.N) if is_ct else (n, self.p.L, self.p.N)
        buf = self._prep_bufs.get(key)
        if buf is None or tuple(buf.shape) != shape:
            buf = self._prep_bufs[key] = torch.empty(shape, dtype=torch.int32, device=_dev.device())
        if background and _BG_CAP > 0:
            _lib.call("pb_set_launch_cap", _BG_CAP)
            try:
                self._make_operand(layer, op, plan, role, src, buf, rng)
            finally:
                _lib.call("pb_set_launch_cap", 0)
        else:
            self._make_operand(layer, op, plan, role, src, buf, rng)
        ev = None
        if event:
            ev = torch.cuda.Event()
            ev.record()
        self._prepared[key] = (buf, ev)

    def clear_prepared(self):
        """Drop unconsumed prepared operands and masks."""
        self._prepared.clear()
        self._masks.clear()

    # ------------------------------------------------------- mask prefetch ---
    def prefetch_masks(self, specs, event: bool = True):
        """Draw the MO masks s of protocols (layer, op) ahead of them -- they
        depend only on the step seed -- on an auxiliary stream; ``specs`` =
        [(layer, op, shape)].  The protocol's ``mask()`` call returns the
        same values it would have drawn itself (stream (layer, op, P_MASK))."""
        if not _MASK_PREFETCH:
            return
        # persistent buffers (never returned to the caching allocator): a prefetched
        # mask is consumed on other streams (grad stream, side streams) than the
        # one that allocated it, so a freed block could be reused under them
        bufs = []
        for layer, op, shape in specs:
            key = (layer, op, tuple(shape))
            buf = self._mask_bufs.get(key)
            if buf is None:
                buf = self._mask_bufs[key] = _dev.empty_u64(*shape)
            bufs.append((layer, op, tuple(shape), buf))
        cur = torch.cuda.current_stream()
        if _SERIAL:
            side = cur
        else:
            side = self._mask_streams.get(cur.cuda_stream)
            if side is None:
                side = self._mask_streams[cur.cuda_stream] = _stream_like(cur)
            side.wait_stream(cur)
        with torch.cuda.stream(side):
            for layer, op, shape, buf in bufs:
                self.rng(layer, op, P_MASK).uniform_ring(shape, self.ring, out=buf)
                ev = None
                if event:
                    ev = torch.cuda.Event()
                    ev.record(side)
                self._masks[(layer, op, shape)] = (buf, ev)
        if side is not cur:  # joined at the phase end (join_side); consumers wait on the events
            self._pending_join.append(side)

    def fork_pool(self, n: int = 3):
        """n streams forked from the current one (registered for join_side), for
        independent background work enqueued round-robin."""
        cur = torch.cuda.current_stream()
        if _SERIAL:
            return [cur]
        pool = self._fork_pools.get(cur.cuda_stream)
        if pool is None:
            pool = self._fork_pools[cur.cuda_stream] = [_stream_like(cur) for _ in range(n)]
        for st in pool:
            st.wait_stream(cur)
            self._pending_join.append(st)
        return pool

    def join_side(self):
        """Join the mask-prefetch forks into the current stream (a CUDA-graph
        capture needs every fork joined before it ends); ends the phase's
        encryption pre-draw."""
        cur = torch.cuda.current_stream()
        for st in self._pending_join:
            cur.wait_stream(st)
        self._pending_join.clear()
        self._t0 = None
        self._predraw_used.clear()

    def begin_phase(self):
        """Mark the start of a forward / backward phase on the current stream.
        Until join_side(), each DO encryption he_eval makes on its critical
        path is split (bfv.encrypt_zero / encrypt_add): the
        message-independent half -- the uniform a, c1 = a, c0 = -a s and the
        noise e -- runs on a pre-draw stream that only waits for this point,
        and only c0 += NTT(e + Delta m) waits for the message.  The
        ciphertext is a fresh encryption under the same key stream; the
        protocol's outputs (decrypted shares) are unchanged."""
        if not _PREDRAW or _SERIAL:
            return
        ev = torch.cuda.Event()
        ev.record()
        self._t0 = ev
        self._predraw_used.clear()

    def _claim(self, key) -> bool:
        """A persistent pre-draw buffer serves one protocol call per phase."""
        if key in self._predraw_used:
            return False
        self._predraw_used.add(key)
        return True

    def _encrypt_split(self, layer, op, plan, role, src, side):
        """Enc(src) of one ct operand as a pre-drawn half (persistent buffers,
        pre-draw stream, ordered after the phase start only) and the
        message-dependent half on ``side``; returns the ciphertext buffer."""
        pack, n, _, off = self._operand_layout(plan, role)
        h, L, N = self.ctx.handle, self.p.L, self.p.N
        key = (layer, op, role)
        ent = self._predraw_bufs.get(key)
        if ent is None or ent[0].shape[0] != n:
            # persistent: written at the start of the NEXT phase too, so never
            # handed back to the caching allocator
            ent = self._predraw_bufs[key] = (_dev.empty_u32(n, 2, L, N),
                                             torch.empty(n, N, dtype=torch.int8, device=_dev.device()))
        ct, e = ent
        enc_rng = self.rng(layer, op, P_ENC)
        base = enc_rng.reserve((plan.n_in + plan.n_pt) * self.world)
        if self._predraw_stream is None:
            self._predraw_stream = torch.cuda.Stream()
        ps = self._predraw_stream
        ps.wait_event(self._t0)
        with torch.cuda.stream(ps):
            _lib.call("pb_encrypt_sk_zero", h, _dev.ptr(self.kp.sk_ntt), n, *enc_rng.dev_args(), base + off,
                      _dev.ptr(ct), _dev.ptr(e), _dev.stream())
            ev = torch.cuda.Event()
            ev.record()
        side.wait_event(ev)
        with torch.cuda.stream(side):
            _lib.call("pb_encrypt_sk_add", h, _dev.ptr(src), *_pk(pack), n, _dev.ptr(e), _dev.ptr(ct), _dev.stream())
        self._count("pb_encrypt_sk", n * (2 * L * N * 4 + 8 * N), ntt_rows=n * L)
        return ct

    def mask(self, layer: int, op: int, shape) -> torch.Tensor:
        """The MO's uniform mask of protocol (layer, op): prefetched or drawn now."""
        shape = tuple(shape)
        pre = self._masks.pop((layer, op, shape), None)
        if pre is None:
            return self.rng(layer, op, P_MASK).uniform_ring(shape, self.ring)
        buf, ev = pre
        if ev is not None:
            torch.cuda.current_stream().wait_event(ev)
        return buf

    def _count(self, name, nbytes, ntt_rows=0, mod_macs=0):
        """Algorithmic work of one entry-point call (SURVEY §8d unit costs), while
        instrumented: HBM bytes, NTT rows (forward or inverse, one limb each)
        and lazy mod-MACs -- bench.py's HBM and integer-pipe rooflines."""
        if _lib.STATS is not None:
            self.alg_bytes[name] = self.alg_bytes.get(name, 0.0) + float(nbytes)
            w = self.alg_work.setdefault(name, [0.0, 0.0])
            w[0] += float(ntt_rows)
            w[1] += float(mod_macs)

    def _shard(self, plan):
        key = (id(plan), self.rank, self.world)
        sh = self._shards.get(key)
        if sh is None:
            sh = _Shard(plan, self.rank, self.world)
            self._shards[key] = sh
        return sh

    # --------------------------------------------------------- HE matmul ---
    def he_matmul(self, layer: int, op: int, g: MatmulGeometry, out: torch.Tensor, mask: torch.Tensor,
                  v_ct=None, v_strides=None, w_pt=None, w_strides=None, w_ct=None, v_pt=None,
                  y_strides=None, msg_in=MSG_FWD_INPUT_CT, msg_out=MSG_FWD_MASKED_CT):
        """DO-decrypted share of  [Enc(pi_v(v_ct)) (x) pi_W(w_pt)] + [Enc(pi_W(w_ct)) (x) pi_v(v_pt)] - mask,
        written into ``out`` (flat, addressed through y_strides).  Operands are flat
        device tensors addressed through the given strides; absent terms are None."""
        plan = plan_matmul(g, self.p.N, v_strides, w_strides, y_strides)
        return self.he_eval(layer, op, plan, out, mask, v_ct=v_ct, w_pt=w_pt, w_ct=w_ct, v_pt=v_pt,
                            msg_in=msg_in, msg_out=msg_out)

    def he_eval(self, layer: int, op: int, plan, out: torch.Tensor, mask: torch.Tensor, v_ct=None, w_pt=None,
                w_ct=None, v_pt=None, msg_in=MSG_FWD_INPUT_CT, msg_out=MSG_FWD_MASKED_CT):
        """he_matmul over any block plan (matmul or conv-layer packing); the
        plan's maps address the flat operand / output tensors directly."""
        p, h, st = self.p, self.ctx.handle, _dev.stream()
        sh = self._shard(plan)
        N, L = p.N, p.L
        w = 4  # bytes per residue
        ct_bytes = 2 * L * N * w
        if self.world > 1 or plan.kind == "conv":
            out.zero_()  # conv plans may leave structural-zero outputs without a slot
        # Buffers are allocated on the main stream; the DO's encryptions and the
        # MO's plaintext encodings run on two side streams concurrently with the
        # MO's mask NTT, and the MAC joins all three (the graph keeps the fork).
        # Operands prepared ahead of time (prepare_operand) are used as they are.
        has_a = bool(sh.n_out) and v_ct is not None
        has_b = bool(sh.n_out) and w_ct is not None
        main = torch.cuda.current_stream()
        ops = {}
        if has_a or has_b:
            s_enc, s_pt = self._side_streams()
            s_enc.wait_stream(main)  # covers every buffer allocated below
            s_pt.wait_stream(main)
            todo = ((("A_ct", v_ct), ("A_pt", w_pt)) if has_a else ()) + ((("B_ct", w_ct), ("B_pt", v_pt)) if has_b else ())
            for role, src in todo:
                _, n, is_ct, _ = self._operand_layout(plan, role)
                side = s_enc if is_ct else s_pt  # DO / MO
                pre = self._prepared.pop((layer, op, role), None)
                if pre is not None:
                    buf, ev = pre
                    if ev is not None:
                        side.wait_event(ev)
                elif is_ct and self._t0 is not None and n * L <= _PREDRAW_MAX_ROWS and self._claim((layer, op, role)):
                    buf = self._encrypt_split(layer, op, plan, role, src, side)
                else:
                    buf = _dev.empty_u32(n, 2, L, N) if is_ct else _dev.empty_u32(n, L, N)
                    with torch.cuda.stream(side):
                        self._make_operand(layer, op, plan, role, src, buf)
                if is_ct:
                    self.channel.send(DO, msg_in, buf, Ciphertext(buf, p).nbytes_wire())
                ops[role] = buf
        ctA, ptA, ctB, ptB = ops.get("A_ct"), ops.get("A_pt"), ops.get("B_ct"), ops.get("B_pt")
        out_ct = _dev.empty_u32(sh.n_out, 2, L, N) if sh.n_out else None
        # streaming shapes (nI <= 2) that fill the GPU: mask NTT and MAC fused in
        # one pass (pb_mask_mac, no -mask row round trip); smaller ones keep the
        # mask NTT concurrent with the encryptions (latency over traffic)
        fused = (has_a or has_b) and sh.nI <= 2 and sh.n_out * L >= _FUSE_MIN_ROWS
        if sh.n_out:
            fseed, fptr = self.rng(layer, op, P_MASK).dev_args()
            if not fused:  # MO: out.c0 = -Delta NTT(mask + filler), then the tiled MAC accumulates onto it
                _lib.call("pb_mask_ntt", h, sh.n_out, _dev.ptr(sh.out_pos), _dev.ptr(sh.out_dst), sh.U,
                          _dev.ptr(mask), 1 if self.filler else 0, fseed ^ 0x5A5A5A5A5A5A5A5A, fptr,
                          _dev.ptr(out_ct), st)
                self._count("pb_mask_ntt", sh.n_out * (L * N * w + 8 * sh.U), ntt_rows=sh.n_out * L)
            if has_a or has_b:
                main.wait_stream(s_enc)
                main.wait_stream(s_pt)
            if ctA is None and ctB is None:  # no cross term: the DO decrypts an encryption of -mask
                out_ct[:, 1].zero_()
            elif fused:
                _lib.call("pb_mask_mac", h, _dev.ptr(ctA), _dev.ptr(ptA), _dev.ptr(ctB), _dev.ptr(ptB), sh.nb, sh.no,
                          sh.nI, _dev.ptr(sh.out_pos), _dev.ptr(sh.out_dst), sh.U, _dev.ptr(mask),
                          1 if self.filler else 0, fseed ^ 0x5A5A5A5A5A5A5A5A, fptr, _dev.ptr(out_ct), st)
                n_ct = (sh.n_in if ctA is not None else 0) + (sh.n_pt if ctB is not None else 0)
                n_pt = (sh.n_pt if ctA is not None else 0) + (sh.n_in if ctB is not None else 0)
                n_terms = (1 if ctA is not None else 0) + (1 if ctB is not None else 0)
                self._count("pb_mask_mac", n_ct * ct_bytes + n_pt * L * N * w + sh.n_out * (ct_bytes + 8 * sh.U),
                            ntt_rows=sh.n_out * L, mod_macs=n_terms * sh.n_out * sh.nI * 2 * L * N)
            else:
                _lib.call("pb_ctpt_mac_tiled", h, _dev.ptr(ctA), _dev.ptr(ptA), _dev.ptr(ctB), _dev.ptr(ptB), sh.nb,
                          sh.no, sh.nI, _dev.ptr(out_ct), st)
                n_ct = (sh.n_in if ctA is not None else 0) + (sh.n_pt if ctB is not None else 0)
                n_pt = (sh.n_pt if ctA is not None else 0) + (sh.n_in if ctB is not None else 0)
                n_terms = (1 if ctA is not None else 0) + (1 if ctB is not None else 0)
                self._count("pb_ctpt_mac_tiled", n_ct * ct_bytes + n_pt * L * N * w + sh.n_out * (ct_bytes + L * N * w),
                            mod_macs=n_terms * sh.n_out * sh.nI * 2 * L * N)
            self.channel.send(MO, msg_out, out_ct, Ciphertext(out_ct, p).nbytes_wire())
            if self.capture is not None:
                self.capture.append((out_ct.clone(), sh.out_pos.clone()))
            scratch = _dev.empty_u32(sh.n_out, L, sh.U)
            if self.world > 1:  # this rank's useful slots into its compact tile (gather_maps)
                tile = torch.zeros(sh.n_max * sh.U, dtype=torch.int64, device=out.device)
                dmap, dout = sh.tile_dst, tile
            else:
                dmap, dout = sh.out_dst, out
            _lib.call("pb_decrypt_to_share", h, _dev.ptr(self.kp.sk_ntt), _dev.ptr(out_ct), sh.n_out,
                      _dev.ptr(sh.out_pos), _dev.ptr(dmap), sh.U, _dev.ptr(dout), _dev.ptr(scratch), st)
            self._count("pb_decrypt_to_share", sh.n_out * (ct_bytes + 8 * sh.U), ntt_rows=sh.n_out * L)
            # operands stay referenced until here, i.e. until every kernel is enqueued
            del ctA, ptA, ctB, ptB, ops, out_ct, scratch
        if self.world > 1:  # all-gather the ranks' compact tiles, scatter them into `out`
            import torch.distributed as dist

            if not sh.n_out:
                tile = torch.zeros(sh.n_max * sh.U, dtype=torch.int64, device=out.device)
            gathered = torch.empty(self.world * sh.n_max * sh.U, dtype=torch.int64, device=out.device)
            if dist.get_backend(self.group) == "nccl":
                dist.all_gather_into_tensor(gathered, tile, group=self.group)
            else:  # gloo (the CPU / shared-GPU tests): list form
                dist.all_gather(list(gathered.chunk(self.world)), tile, group=self.group)
            _lib.call("pb_scatter_u64", _dev.ptr(out), _dev.ptr(gathered), _dev.ptr(sh.gdst), gathered.numel(),
                      _dev.stream())
        return out


# ----------------------------------------------------------------- helpers ---

def _ring_matmul(a: torch.Tensor, b: torch.Tensor, n, k, m, ell, ta=False, tb=False, c=None, sign=0,
                 out=None) -> torch.Tensor:
    """a @ b mod 2^ell, or c + sign * (a @ b) with the add fused into the GEMM."""
    if out is None:
        out = _dev.empty_u64(n, m)
    _lib.call("pb_ring_matmul_add", _dev.ptr(a), _dev.ptr(b), n, k, m, 1 if ta else 0, 1 if tb else 0,
              _dev.ptr(c) if c is not None else None, sign if c is not None else 0, ell, _dev.ptr(out), _dev.stream())
    return out


def _ring_bin(op, a, b, ell, bn=None) -> torch.Tensor:
    out = torch.empty_like(a)
    n = a.numel()
    _lib.call("pb_ring_binary", op, _dev.ptr(out), _dev.ptr(a), _dev.ptr(b), n, n if bn is None else bn, ell,
              _dev.stream())
    return out


def _add_bcast(a: torch.Tensor, b: torch.Tensor, inner: int, ell: int, out=None) -> torch.Tensor:
    """a + b broadcast along an axis (b[(i / inner) % len(b)]), one kernel."""
    out = torch.empty_like(a) if out is None else out
    _lib.call("pb_ring_add_bcast", _dev.ptr(out), _dev.ptr(a), _dev.ptr(b), a.numel(), inner, b.numel(), ell,
              _dev.stream())
    return out


def _check_share_pair(a: ShareTensor, b: ShareTensor):
    if {a.owner_role, b.owner_role} != {MO, DO}:
        raise DesyncError("need one MO share and one DO share")
    if a.scale != b.scale:
        raise ScaleError("share scales differ")
    if a.shape != b.shape:
        raise ShapeError("share shapes differ")


def _split(a: ShareTensor, b: ShareTensor):
    _check_share_pair(a, b)
    return (a, b) if a.owner_role == MO else (b, a)


# ------------------------------------------------------------- protocols ---

def linear_forward(sess: Session, layer: int, W: RingTensor, b: RingTensor, x_a: ShareTensor, x_b: ShareTensor,
                   mo_x_zero: bool = False):  # Alg.1
    """Shares of Y = W X + b at scale 2f.  X shares (n_i, B) at f, W (n_o, n_i) at f, b (n_o,) at 2f."""
    x_mo, x_do = _split(x_a, x_b)
    ring = sess.ring
    if x_mo.scale != ring.f or W.scale != ring.f or b.scale != 2 * ring.f:
        raise ScaleError("linear_forward needs X, W at f and b at 2f")
    n_o, n_i = W.shape
    if x_do.shape[0] != n_i:
        raise ShapeError(f"X has {x_do.shape[0]} features, W expects {n_i}")
    B = x_do.shape[1]
    s = sess.mask(layer, OP_FWD, (n_o, B))
    if mo_x_zero:
        s_eff = s
    else:
        s_eff = _ring_matmul(W.values, x_mo.value.values, n_o, n_i, B, ring.ell, c=s, sign=-1)
    y_do = _dev.empty_u64(n_o, B)
    y_mo = _dev.empty_u64(n_o, B)
    with sess.aux() as aux:  # MO's output share s + b: off the critical path
        aux.run(lambda: _add_bcast(s, b.values, B, ring.ell, out=y_mo))
        sess.he_matmul(layer, OP_FWD, MatmulGeometry(n_i, n_o, B), y_do, s_eff, v_ct=x_do.value.values,
                       w_pt=W.values)
    return (ShareTensor(MO, RingTensor(y_mo, 2 * ring.f, ring, _canonical=True)),
            ShareTensor(DO, RingTensor(y_do, 2 * ring.f, ring, _canonical=True)))


def linear_backward_input(sess: Session, layer: int, W: RingTensor, gy_a: ShareTensor, gy_b: ShareTensor,
                          mo_gy_zero: bool = False):
    """Shares of grad X = W^T gY at scale 2f (Alg.1 message pattern with W^T)."""
    gy_mo, gy_do = _split(gy_a, gy_b)
    ring = sess.ring
    n_o, n_i = W.shape
    B = gy_do.shape[1]
    s = sess.mask(layer, OP_BWD_X, (n_i, B))
    if mo_gy_zero:
        s_eff = s
    else:
        s_eff = _ring_matmul(W.values, gy_mo.value.values, n_i, n_o, B, ring.ell, ta=True, c=s, sign=-1)
    g_do = _dev.empty_u64(n_i, B)
    # W^T (n_i, n_o) addressed in W's storage through strides (1, n_i)
    sess.he_matmul(layer, OP_BWD_X, MatmulGeometry(n_o, n_i, B), g_do, s_eff, v_ct=gy_do.value.values,
                   w_pt=W.values, w_strides=(1, n_i), msg_in=MSG_BWD_X, msg_out=MSG_BWD_X + 1)
    return (ShareTensor(MO, RingTensor(s, 2 * ring.f, ring, _canonical=True)),
            ShareTensor(DO, RingTensor(g_do, 2 * ring.f, ring, _canonical=True)))


def reveal_grad_bias(sess: Session, layer: int, gy_a: ShareTensor, gy_b: ShareTensor,
                     e: torch.Tensor | None = None) -> RingTensor:
    gy_mo, gy_do = _split(gy_a, gy_b)
    ring = sess.ring
    n, B = gy_do.shape
    sd = _dev.empty_u64(n)
    _lib.call("pb_ring_rowsum", _dev.ptr(gy_do.value.values), n, B, ring.ell, _dev.ptr(sd), _dev.stream())
    if e is not None:
        sd = _ring_bin(_lib.RING_ADD, sd, e, ring.ell)
    sess.channel.send(DO, MSG_GRADB, sd, n * 8)
    sm = _dev.empty_u64(n)
    _lib.call("pb_ring_rowsum", _dev.ptr(gy_mo.value.values), n, B, ring.ell, _dev.ptr(sm), _dev.stream())
    return RingTensor(_ring_bin(_lib.RING_ADD, sm, sd, ring.ell), gy_do.scale, ring, _canonical=True)


def grad_w_flipped(mo_x_zero: bool, mo_gy_zero: bool) -> bool:
    """Whether Alg.2's HE matmul runs transposed (grad W^T = X gY^T), _GRADW_FLIP:
    for the two-cross-term layers it puts the gradient on the packing side with
    fewer polynomials (128x128x64: 16 instead of 64 gradient ciphertexts and
    plaintexts), the forward-only X side (prepared beside the loss) grows to 64.
    Measured on the MLP step: 1.5 % slower (the larger host-gap preparation
    delays the backward; profiles/r01_ab_gradw_flip.txt), so off by default;
    one-term layers never flip (the first layer's X side would grow 80 -> 208;
    re-measured in round 2: the gradient's critical-path encode shrinks 1120 ->
    448 rows but the larger background preparation makes the step 4 % slower)."""
    return _GRADW_FLIP and not (mo_x_zero or mo_gy_zero)


def grad_w_geometry(n_o: int, n_i: int, B: int, flipped: bool):
    """(geometry, v_strides, y_strides) of Alg.2's HE matmul for an (n_o, n_i)
    layer: grad W = gY X^T with gY (n_o, B) in the W role and X^T (strides
    (1, B)) in the v role; flipped: grad W^T = X gY^T with X (n_i, B) in the W
    role, gY^T in the v role and the output written transposed."""
    if flipped:
        return MatmulGeometry(B, n_i, n_o), (1, B), (1, n_i)
    return MatmulGeometry(B, n_o, n_i), (1, B), None


def grad_weight(sess: Session, layer: int, x_a: ShareTensor, x_b: ShareTensor, gy_a: ShareTensor,
                gy_b: ShareTensor, e: torch.Tensor | None = None, mo_x_zero: bool = False,
                mo_gy_zero: bool = False) -> RingTensor:  # Alg.2
    """grad W = gY X^T revealed to the MO at scale 2f (n_o, n_i)."""
    x_mo, x_do = _split(x_a, x_b)
    gy_mo, gy_do = _split(gy_a, gy_b)
    ring = sess.ring
    n_i, B = x_do.shape
    n_o = gy_do.shape[0]
    s = sess.mask(layer, OP_GRAD_W, (n_o, n_i))
    cross_do = _dev.empty_u64(n_o, n_i)
    loc_do = _dev.empty_u64(n_o, n_i)
    loc_mo = _dev.empty_u64(n_o, n_i) if not (mo_x_zero or mo_gy_zero) else s
    with sess.aux() as aux:  # the local terms do not depend on the HE result: overlap them with it
        aux.run(lambda: _ring_matmul(gy_do.value.values, x_do.value.values, n_o, B, n_i, ring.ell, tb=True,
                                     out=loc_do))
        if loc_mo is not s:  # MO: s + gY_0 X_0^T
            aux.run(lambda: _ring_matmul(gy_mo.value.values, x_mo.value.values, n_o, B, n_i, ring.ell, tb=True,
                                         c=s, sign=1, out=loc_mo))
        # grad W^T = X gY^T: W-role X (n_i x B), v-role gY^T through strides (1, B),
        # output written transposed (y strides (1, n_i)).  The gradient sits on the
        # packing side with fewer polynomials (e.g. 16 instead of 64 ciphertexts +
        # plaintexts for 128x128), the forward-only X side is prepared ahead.
        # Cross terms: Enc(gY_1) (x) X_0 (term A) and Enc(X_1) (x) gY_0 (term B).
        flip = grad_w_flipped(mo_x_zero, mo_gy_zero)
        g, vs, ys = grad_w_geometry(n_o, n_i, B, flip)
        xd = None if mo_gy_zero else x_do.value.values  # cross term gY_0 X_1^T
        gm = None if mo_gy_zero else gy_mo.value.values
        gd = None if mo_x_zero else gy_do.value.values  # cross term gY_1 X_0^T
        xm = None if mo_x_zero else x_mo.value.values
        if flip:  # term A: Enc(gY_1) (x) X_0, term B: Enc(X_1) (x) gY_0
            sess.he_matmul(layer, OP_GRAD_W, g, cross_do, s, v_ct=gd, v_strides=vs, w_pt=xm, w_ct=xd, v_pt=gm,
                           y_strides=ys, msg_in=MSG_GRADW, msg_out=MSG_GRADW)
        else:  # term A: Enc(X_1) (x) gY_0, term B: Enc(gY_1) (x) X_0
            sess.he_matmul(layer, OP_GRAD_W, g, cross_do, s, v_ct=xd, v_strides=vs, w_pt=gm, w_ct=gd, v_pt=xm,
                           y_strides=ys, msg_in=MSG_GRADW, msg_out=MSG_GRADW)
    # DO: + local term gY_1 X_1^T (+ e), sends the masked sum
    msg = _ring_bin(_lib.RING_ADD, cross_do, loc_do, ring.ell)
    if e is not None:
        msg = _ring_bin(_lib.RING_ADD, msg, e, ring.ell)
    sess.channel.send(DO, MSG_GRADW, msg, msg.numel() * 8)
    # MO: + s + local term gY_0 X_0^T
    out = _ring_bin(_lib.RING_ADD, msg, loc_mo, ring.ell)
    return RingTensor(out, 2 * ring.f, ring, _canonical=True)


# ------------------------------------------------------- conv layers ---
# Conv2d layers (SPEC:249-266 packing; SPEC:284-286 transforms): activations
# (B, C, H, W), W (c_o, c_i, s, s) at f, bias (c_o,) at 2f.  The three
# operators run on the native conv packing with padding / stride / flips
# folded into the plan maps (poly_encoding.plan_conv_layer), through the same
# fused kernels as the FC protocols; local terms use pb_ring_conv.

def _ring_conv(kind: int, a: torch.Tensor, b: torch.Tensor, B, c_i, c_o, H, W, s, pad, stride, ell, out_shape,
               out=None):
    out = _dev.empty_u64(*out_shape) if out is None else out
    _lib.call("pb_ring_conv", kind, _dev.ptr(a), _dev.ptr(b), B, c_i, c_o, H, W, s, pad, stride, ell, _dev.ptr(out),
              _dev.stream())
    return out


_UNCOVERED = {}


def _covered(plan, n: int):
    """0/1 device mask of the output elements some ciphertext slot carries, or
    None when all are (the rest are structural zeros of a strided input gradient)."""
    key = id(plan)
    if key not in _UNCOVERED:
        cov = np.zeros(n, dtype=bool)
        cov[plan.out_dst[plan.out_dst >= 0]] = True
        _UNCOVERED[key] = (plan, None if cov.all() else _dev.u64_to_device(cov.astype(np.uint64)))
    return _UNCOVERED[key][1]


def conv_forward(sess: Session, layer: int, W: RingTensor, b: RingTensor, x_a: ShareTensor, x_b: ShareTensor,
                 pad: int, stride: int, mo_x_zero: bool = False):
    """Alg.1 with conv packing: shares of Y = conv(X; W) + b at 2f, (B, c_o, oh, ow)."""
    x_mo, x_do = _split(x_a, x_b)
    ring = sess.ring
    if x_mo.scale != ring.f or W.scale != ring.f or b.scale != 2 * ring.f:
        raise ScaleError("conv_forward needs X, W at f and b at 2f")
    B, c_i, H, Wd = x_do.shape
    c_o, ci2, s, _ = W.shape
    if ci2 != c_i:
        raise ShapeError(f"X has {c_i} channels, W expects {ci2}")
    oh, ow = conv_out_hw(H, Wd, s, pad, stride)
    msk = sess.mask(layer, OP_FWD, (B, c_o, oh, ow))
    if mo_x_zero:
        s_eff = msk
    else:
        loc = _ring_conv(_lib.CONV_FWD, x_mo.value.values, W.values, B, c_i, c_o, H, Wd, s, pad, stride, ring.ell,
                         (B, c_o, oh, ow))
        s_eff = _ring_bin(_lib.RING_SUB, msk, loc, ring.ell)
    plan = plan_conv_layer("fwd", B, c_i, c_o, H, Wd, s, pad, stride, sess.p.N)
    y_do = _dev.empty_u64(B, c_o, oh, ow)
    y_mo = _dev.empty_u64(B, c_o, oh, ow)
    with sess.aux() as aux:  # MO's output share s + b: off the critical path
        aux.run(lambda: _add_bcast(msk, b.values, oh * ow, ring.ell, out=y_mo))
        sess.he_eval(layer, OP_FWD, plan, y_do, s_eff, v_ct=x_do.value.values, w_pt=W.values)
    return (ShareTensor(MO, RingTensor(y_mo, 2 * ring.f, ring, _canonical=True)),
            ShareTensor(DO, RingTensor(y_do, 2 * ring.f, ring, _canonical=True)))


def conv_backward_input(sess: Session, layer: int, W: RingTensor, gy_a: ShareTensor, gy_b: ShareTensor, H: int,
                        Wd: int, pad: int, stride: int, mo_gy_zero: bool = False):
    """SPEC:321-329 for Conv2d: shares of dX = conv^T(dY) at 2f, (B, c_i, H, W)."""
    gy_mo, gy_do = _split(gy_a, gy_b)
    ring = sess.ring
    B, c_o = gy_do.shape[:2]
    c_i, s = W.shape[1], W.shape[2]
    msk = sess.mask(layer, OP_BWD_X, (B, c_i, H, Wd))
    plan = plan_conv_layer("bwdx", B, c_i, c_o, H, Wd, s, pad, stride, sess.p.N)
    cov = _covered(plan, B * c_i * H * Wd)
    if cov is not None:  # input positions no output reads: gradient exactly 0, MO share 0 too
        msk = _ring_bin(_lib.RING_MUL, msk, cov.reshape(msk.shape), ring.ell)
    if mo_gy_zero:
        s_eff = msk
    else:
        loc = _ring_conv(_lib.CONV_BWDX, gy_mo.value.values, W.values, B, c_i, c_o, H, Wd, s, pad, stride, ring.ell,
                         (B, c_i, H, Wd))
        s_eff = _ring_bin(_lib.RING_SUB, msk, loc, ring.ell)
    g_do = _dev.empty_u64(B, c_i, H, Wd)
    sess.he_eval(layer, OP_BWD_X, plan, g_do, s_eff, v_ct=gy_do.value.values, w_pt=W.values, msg_in=MSG_BWD_X,
                 msg_out=MSG_BWD_X + 1)
    return (ShareTensor(MO, RingTensor(msk, 2 * ring.f, ring, _canonical=True)),
            ShareTensor(DO, RingTensor(g_do, 2 * ring.f, ring, _canonical=True)))


def conv_grad_weight(sess: Session, layer: int, x_a: ShareTensor, x_b: ShareTensor, gy_a: ShareTensor,
                     gy_b: ShareTensor, s: int, pad: int, stride: int, e: torch.Tensor | None = None,
                     mo_x_zero: bool = False, mo_gy_zero: bool = False) -> RingTensor:
    """Alg.2 for Conv2d: dW = sum_{b,y,x} dY Xpad revealed to the MO at 2f, (c_o, c_i, s, s)."""
    x_mo, x_do = _split(x_a, x_b)
    gy_mo, gy_do = _split(gy_a, gy_b)
    ring = sess.ring
    B, c_i, H, Wd = x_do.shape
    c_o = gy_do.shape[1]
    msk = sess.mask(layer, OP_GRAD_W, (c_o, c_i, s, s))
    plan = plan_conv_layer("gradw", B, c_i, c_o, H, Wd, s, pad, stride, sess.p.N)
    cross_do = _dev.empty_u64(c_o, c_i, s, s)
    shp = (c_o, c_i, s, s)
    loc_do = _dev.empty_u64(*shp)
    two = not (mo_x_zero or mo_gy_zero)
    loc_mo = _dev.empty_u64(*shp) if two else None
    with sess.aux() as aux:  # the local terms do not depend on the HE result: overlap them with it
        aux.run(lambda: _ring_conv(_lib.CONV_GRADW, x_do.value.values, gy_do.value.values, B, c_i, c_o, H, Wd, s,
                                   pad, stride, ring.ell, shp, out=loc_do))
        if two:
            aux.run(lambda: _ring_conv(_lib.CONV_GRADW, x_mo.value.values, gy_mo.value.values, B, c_i, c_o, H, Wd,
                                       s, pad, stride, ring.ell, shp, out=loc_mo))
        sess.he_eval(layer, OP_GRAD_W, plan, cross_do, msk,
                     v_ct=None if mo_gy_zero else x_do.value.values, w_pt=None if mo_gy_zero else gy_mo.value.values,
                     w_ct=None if mo_x_zero else gy_do.value.values, v_pt=None if mo_x_zero else x_mo.value.values,
                     msg_in=MSG_GRADW, msg_out=MSG_GRADW)
    msg = _ring_bin(_lib.RING_ADD, cross_do, loc_do, ring.ell)  # DO: + local term (+ e)
    if e is not None:
        msg = _ring_bin(_lib.RING_ADD, msg, e, ring.ell)
    sess.channel.send(DO, MSG_GRADW, msg, msg.numel() * 8)
    out = _ring_bin(_lib.RING_ADD, msg, msk, ring.ell)  # MO: + s + local term
    if two:
        out = _ring_bin(_lib.RING_ADD, out, loc_mo, ring.ell)
    return RingTensor(out, 2 * ring.f, ring, _canonical=True)


def reveal_grad_bias_conv(sess: Session, layer: int, gy_a: ShareTensor, gy_b: ShareTensor,
                          e: torch.Tensor | None = None) -> RingTensor:
    """SPEC:330-338 for Conv2d: per-channel local sums over batch and positions."""
    gy_mo, gy_do = _split(gy_a, gy_b)
    ring = sess.ring
    B, c, h, w = gy_do.shape

    def chan_sum(v):  # straight from NCHW (no permute copy)
        out = _dev.empty_u64(c)
        _lib.call("pb_ring_chansum", _dev.ptr(v.contiguous()), B, c, h * w, ring.ell, _dev.ptr(out), _dev.stream())
        return out

    sd = chan_sum(gy_do.value.values)
    if e is not None:
        sd = _ring_bin(_lib.RING_ADD, sd, e, ring.ell)
    sess.channel.send(DO, MSG_GRADB, sd, c * 8)
    return RingTensor(_ring_bin(_lib.RING_ADD, chan_sum(gy_mo.value.values), sd, ring.ell), gy_do.scale, ring,
                      _canonical=True)


def sample_dp_noise(shape, dp: DpConfig, rng: SeededRng) -> np.ndarray:
    """e ~ N(0, (sigma C)^2 / B) per element (host float64, encoded by the caller)."""
    if dp is None or not dp.enabled or dp.sigma == 0.0:
        return np.zeros(shape)
    return rng.normal(shape, dp.sigma * dp.C / np.sqrt(dp.B))


def dp_noise(sess: Session, layer: int, op: int, shape, scale: int) -> torch.Tensor | None:
    """The DO's encoded DP perturbation of one reveal: e drawn
    on the host from the session's (layer, op, P_DP) stream -- R:80-81's numpy
    ``normal``, the reference's own sampler -- encoded at the revealed value's
    scale (grad b: f; grad W before the MO's shift: 2f) and moved to the
    device; None when the session's DP is off."""
    dp = sess.dp
    if dp is None or not dp.enabled:
        return None
    if sess.graph_mode:
        raise ParamsError("DP noise is a per-step host draw: run DP steps eagerly (private_train_step)")
    e = sample_dp_noise(tuple(shape), dp, sess.rng(layer, op, P_DP))
    return encode_fixed(e, sess.ring, scale)
