"""One Shor attempt sharded over the ranks of a torch.distributed group.

One process per GPU.  Rank g of G owns the exponent slice
a in [g q/G, (g+1) q/G) for modexp / histogram / compaction and the output
slice c in [g q/G, (g+1) q/G) for the DFT and |V|^2.  The
exchanges are the ones the algorithm really has:

1. all_reduce(sum) of the exact class counts  -> every rank draws the same k
2. all_gather of the per-shard supports       -> every rank holds the comb
3. all_reduce(sum) of the |V|^2 partial sums  -> the normalisation check
4. the exact sequential CDF without moving the probabilities: all_gather of
   the approximate shard sums (hints for every rank's binade records, built
   in parallel), then the exact running value hops rank to rank (one double
   per hop), all_gather of the (enter, leave) pairs, and the owning rank's m
   broadcast back

Every rank replays the same host Sampler stream, so x, k and m agree by
construction; each output's summation order does not depend on G, so the
spectrum is bitwise identical for any G (tests/test_gpu_parity.py).

``ops`` supplies the stage kernels.  The product uses ``DeviceOps``
(libshorb200.so); tests inject a CPU implementation to exercise the
collective logic with the gloo backend.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import qstate


def shard(total: int, rank: int, world: int) -> tuple[int, int]:
    lo = total * rank // world
    hi = total * (rank + 1) // world
    return lo, hi


class DeviceOps:
    """Stage kernels on the local GPU (libshorb200.so)."""

    def __init__(self):
        from . import device as dev
        self.dev = dev
        import torch
        self.torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device())

    def modexp(self, x, n, count, a_begin):
        return self.dev.modexp(x, n, count, a_begin)

    def class_counts(self, res, ncls):
        return self.dev.class_counts(res, ncls)

    def compact_eq(self, res, k, a_begin, expected=None):
        return self.dev.compact_eq(res, k, a_begin, expected=expected)

    def progression(self, support):
        return self.dev.support_progression(support)

    def fill_progression(self, support, m, a0, stride, length, amp):
        return self.dev.fill_progression(support, m, a0, stride, length, amp)

    def dft(self, amps, length, a0, stride, q, c_begin, c_count, precision, real=False):
        return self.dev.dft(amps, length, a0, stride, q, c_begin, c_count, precision=precision, real=real)

    def dft_uniform(self, amp, length, a0, stride, q, c_begin, c_count, precision):
        return self.dev.dft_uniform(amp, length, a0, stride, q, c_begin, c_count, precision=precision)

    def dsum(self, x):
        return self.dev.dsum(x)

    def sample(self, prob, u):
        return self.dev.sample_index(prob, u)[0]

    def approx_sum(self, prob):
        return self.dev.dsum(prob)

    def cumsum_plan(self, prob, s_hint):
        return self.dev.cumsum_plan(prob, s_hint)

    def cumsum_walk(self, prob, plan, s_in):
        return self.dev.cumsum_walk(prob, plan, s_in)

    def cumsum_find(self, prob, plan, s_in, s_out, target):
        return self.dev.cumsum_find(prob, plan, s_out, target)

    def empty(self, n, dtype):
        return self.torch.empty(n, dtype=dtype, device=self.device)

    def to_host(self, t):
        return t.cpu().numpy()


@dataclass
class AttemptRecord:
    x: int
    q: int
    k: int
    M: int
    r: int
    c0: int
    m: int
    norm2: float
    phase_terms: int
    dft_ms: float | None = None
    phase_times: dict = field(default_factory=dict)


def _all_gather_var(t, world, group, torch):
    """all_gather of 1-D tensors of different lengths (padded, then trimmed)."""
    import torch.distributed as dist
    n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    mx = max(sizes) if sizes else 0
    pad = torch.zeros(max(mx, 1), dtype=t.dtype, device=t.device)
    pad[: t.numel()] = t
    bufs = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[:s] for b, s in zip(bufs, sizes)]), sizes


def sharded_attempt(n: int, x: int, q: int, sampler: qstate.Sampler, *, rank: int = 0,
                    world: int = 1, group=None, ops=None, precision: str = "fp64",
                    time_dft: bool = False, keep_spectrum: bool = False) -> AttemptRecord:
    """entangle -> measure part 2 -> QFT -> sample part 1 for one base x.

    The caller has already drawn x (shor._draw_base) from the same sampler
    on every rank.  Returns the attempt record on every rank.
    """
    import torch
    dist = None
    if world > 1:
        import torch.distributed as dist
    ops = ops or DeviceOps()
    times = {}

    def tick(name, t0):
        if hasattr(ops, "synchronize"):
            ops.synchronize()
        elif torch.cuda.is_available():
            torch.cuda.synchronize()
        times[name] = time.perf_counter() - t0
        return time.perf_counter()

    t0 = time.perf_counter()
    a_lo, a_hi = shard(q, rank, world)
    res = ops.modexp(x, n, a_hi - a_lo, a_lo)
    t0 = tick("entangle", t0)

    # (1) exact class counts, summed over shards
    counts = ops.class_counts(res, n)
    local = ops.to_host(counts).copy()  # this shard's counts size its compaction
    if world > 1:
        dist.all_reduce(counts, group=group)
    a_unif = complex(1.0 / math.sqrt(q))
    w0 = qstate.uniform_weight(a_unif)
    k = qstate.draw_class(ops.to_host(counts), w0, sampler.uniform())
    # (2) shard supports -> full comb on every rank (shards are in a order)
    sup = ops.compact_eq(res, k, a_lo, expected=int(local[k]))
    if world > 1:
        sup, _ = _all_gather_var(sup, world, group, torch)
    M = int(sup.numel())
    amp = qstate.collapsed_amplitude(a_unif, w0, M)
    a0, stride, length = ops.progression(sup)
    # the collapsed support is a full comb: uniform-comb kernel;
    # anything else goes through the generic amplitude stream
    amps = None if M == length else ops.fill_progression(sup, M, a0, stride, length, amp)
    del res
    t0 = tick("measure2", t0)

    # QFT over this rank's output slice
    c_lo, c_hi = shard(q, rank, world)
    ev = None
    if time_dft and torch.cuda.is_available():
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        ev[0].record()
    if amps is None:
        out, prob, bsum = ops.dft_uniform(amp, length, a0, stride, q, c_lo, c_hi - c_lo, precision)
    else:
        out, prob, bsum = ops.dft(amps, length, a0, stride, q, c_lo, c_hi - c_lo, precision,
                                  real=complex(amp).imag == 0.0)
    if ev is not None:
        ev[1].record()
    t0 = tick("qft", t0)

    # (3) normalisation (qstate._require_normalized before sampling)
    norm2 = ops.dsum(bsum)
    if world > 1:
        nt = torch.tensor([norm2], dtype=torch.float64, device=bsum.device)
        dist.all_reduce(nt, group=group)
        norm2 = float(nt.item())
    if abs(math.sqrt(norm2) - 1.0) > qstate.norm_tolerance(precision):
        raise ValueError(f"register is not normalized (|amp| = {math.sqrt(norm2)!r})")
    # (4) exact sequential CDF (qstate.py:112-113) without gathering the
    # probabilities: the running sum is chained rank to rank, then the one
    # rank whose shard holds u * total searches it
    u = sampler.uniform()
    if world > 1:
        m = _sharded_sample(ops, prob, u, q, c_lo, rank, world, group, torch)
    else:
        m = ops.sample(prob, u)
    m = min(m, q - 1)
    tick("sample", t0)
    dft_ms = ev[0].elapsed_time(ev[1]) if ev is not None else None
    rec = AttemptRecord(x=x, q=q, k=k, M=M, r=stride, c0=a0, m=m, norm2=norm2,
                        phase_terms=(c_hi - c_lo) * length, dft_ms=dft_ms, phase_times=times)
    if keep_spectrum:
        rec.spectrum = (out, prob)
    return rec


def _sharded_sample(ops, prob, u: float, q: int, c_lo: int, rank: int, world: int, group, torch) -> int:
    """searchsorted(np.cumsum(p), u * cumsum[-1], "right") over the c-sharded
    probability vector, bit-identical to the single-device read.

    np.cumsum is a strictly sequential chain of float64 adds, so the running
    sum entering shard g is exactly the running sum leaving shard g-1.  Only
    that carry is serial: every rank first builds its shard's binade records
    in parallel from a hint of the value entering it (the all-gathered
    approximate shard sums; exactness never depends on the hint), then the
    exact carry hops rank to rank through the records-driven walk
    (ops.cumsum_walk, ~32 tiles of 8192 outputs per warp step).  An
    all_gather of the (enter, leave) pairs gives every rank the total and the
    shard whose leaving sum first exceeds the target; that rank searches its
    walked shard and broadcasts m.  Traffic: O(world) doubles instead of the
    q-element probability vector."""
    import torch.distributed as dist
    # the scalars travel on the device under NCCL, on the host under gloo
    # (gloo point-to-point takes CPU tensors)
    dev = prob.device if dist.get_backend(group) == "nccl" else torch.device("cpu")
    approx = torch.tensor([float(ops.approx_sum(prob))], dtype=torch.float64, device=dev)
    sums = [torch.zeros(1, dtype=torch.float64, device=dev) for _ in range(world)]
    dist.all_gather(sums, approx, group=group)
    hint = 0.0
    for g in range(rank):
        hint += float(sums[g].item())
    plan = ops.cumsum_plan(prob, hint)
    s_in = torch.zeros(1, dtype=torch.float64, device=dev)
    if rank > 0:
        dist.recv(s_in, src=rank - 1, group=group)
    s_out = torch.tensor([ops.cumsum_walk(prob, plan, float(s_in.item()))], dtype=torch.float64, device=dev)
    if rank < world - 1:
        dist.send(s_out, dst=rank + 1, group=group)
    pairs = [torch.zeros(2, dtype=torch.float64, device=dev) for _ in range(world)]
    dist.all_gather(pairs, torch.cat([s_in, s_out]), group=group)
    bounds = [(float(t[0].item()), float(t[1].item())) for t in pairs]
    total = bounds[-1][1]
    target = u * total
    owner = next((g for g in range(world) if bounds[g][1] > target), None)
    if owner is None:  # no running sum exceeds the target: searchsorted returns q
        return q
    mt = torch.zeros(1, dtype=torch.int64, device=dev)
    if rank == owner:
        mt[0] = c_lo + ops.cumsum_find(prob, plan, bounds[owner][0], bounds[owner][1], target)
    dist.broadcast(mt, src=owner, group=group)
    return int(mt.item())


def dump_spectrum_sharded(out, q: int, path, *, rank: int = 0, world: int = 1, group=None,
                          chunk_elems: int = 1 << 22) -> None:
    """QREG dump (qstate.dump_state format, qstate.py:121-130) of a c-sharded
    spectrum: rank 0 writes the 16-byte header and sizes the file, then every
    rank writes its own slice [g q/G, (g+1) q/G) at its byte offset in 64 MiB
    pieces.  `out` is this rank's float64 [2 * shard] (interleaved re, im)
    tensor; the file equals qstate.dump_state of the gathered spectrum."""
    import os

    import numpy as np

    from . import qstate as qs
    w = q.bit_length() - 1
    if rank == 0:
        with open(path, "wb") as fh:
            fh.write(qs._DUMP_HEADER.pack(qs._DUMP_MAGIC, qs._DUMP_VERSION, w, 0))
            fh.truncate(qs._DUMP_HEADER.size + 16 * q)
    if world > 1:
        import torch.distributed as dist
        dist.barrier(group=group)
    c_lo, c_hi = shard(q, rank, world)
    if out.numel() != 2 * (c_hi - c_lo):
        raise ValueError("spectrum shard does not match this rank's output slice")
    fd = os.open(path, os.O_WRONLY)
    try:
        for lo in range(0, c_hi - c_lo, chunk_elems):
            hi = min(c_hi - c_lo, lo + chunk_elems)
            buf = out[2 * lo: 2 * hi].cpu().numpy().astype("<f8", copy=False).tobytes()
            os.pwrite(fd, buf, qs._DUMP_HEADER.size + 16 * (c_lo + lo))
    finally:
        os.close(fd)
    if world > 1:
        import torch.distributed as dist
        dist.barrier(group=group)


def sampler_at(seed: int, draws: int) -> qstate.Sampler:
    """A Sampler positioned `draws` uniforms into seed's stream (PCG64.advance).

    Generator.random() consumes exactly one 64-bit PCG64 output per double."""
    s = qstate.Sampler(seed)
    if draws:
        s._gen.bit_generator.advance(draws)
    return s


def concurrent_attempts(cfg, *, rank: int = 0, world: int = 1, group=None, attempt_fn=None):
    """The attempt loop of shor.run_shor (shor.py:155-166) with attempts run
    concurrently, one per rank -- and still the reference's exact trace.

    Every attempt that does not end the loop consumes exactly the same number
    of draws (x, u_k, u_m; or u_k, u_m with base_override), and the one that
    ends it is the first success, so attempt i starts at draw i*per_attempt of
    the seed's stream regardless of what earlier attempts measured.  Rank g
    runs attempts g, g+G, ...; after each round the traces are exchanged and
    the loop stops at the lowest-index success.  Returns (attempts, parts).
    """
    import time as _time

    from . import shor
    attempt_fn = attempt_fn or shor.single_attempt
    per = 2 if cfg.base_override is not None else 3
    t0 = _time.perf_counter()
    deadline = None if cfg.time_budget is None else t0 + cfg.time_budget
    attempts, parts = [], None
    base = 0
    while base < cfg.max_attempts and parts is None:
        if deadline is not None and _time.perf_counter() >= deadline:
            break
        i = base + rank
        mine = attempt_fn(cfg, sampler_at(cfg.seed, per * i)) if i < cfg.max_attempts else None
        if world > 1:
            import torch.distributed as dist
            got = [None] * world
            dist.all_gather_object(got, mine, group=group)
        else:
            got = [mine]
        for tr in got:
            if tr is None:
                continue
            attempts.append(tr)
            if tr.outcome.kind == "classical_shortcut":
                parts = [tr.outcome.shortcut, cfg.n // tr.outcome.shortcut]
                break
            if tr.outcome.kind == "factors":
                parts = list(tr.outcome.factors)
                break
        base += world
    return attempts, parts


def run_shor_concurrent(cfg, *, rank: int = 0, world: int = 1, group=None, attempt_fn=None):
    """shor.run_shor with the top-level attempts spread over the ranks (one full
    attempt per GPU at a time).  Same ShorResult as the sequential driver:
    identical attempt traces, factors and recursion (child seeds derived as in
    shor.py:174-195; cofactors are factored sequentially on every rank)."""
    import time as _time
    from dataclasses import replace as _replace

    from . import numtheory as nt
    from . import shor
    t_start = _time.perf_counter()
    if cfg.n < 3:
        raise ValueError("n must be >= 3")
    shortcut = nt.pre_checks(cfg.n)
    if shortcut is not None:
        attempts, parts = [], list(shortcut.factors)
    else:
        attempts, parts = concurrent_attempts(cfg, rank=rank, world=world, group=group, attempt_fn=attempt_fn)
    if parts is None:
        return shor.ShorResult(n=cfg.n, factors=[], attempts=attempts,
                               total_time=_time.perf_counter() - t_start, succeeded=False)
    primes = []
    for part in parts:
        if nt.is_prime(part):
            primes.append(part)
            continue
        budget = None if cfg.time_budget is None else max(cfg.time_budget - (_time.perf_counter() - t_start), 0.0)
        sub = shor.run_shor(_replace(cfg, n=part, seed=shor._derive_seed(cfg.seed, part), base_override=None,
                                     time_budget=budget, dump_state_path=None))
        attempts.extend(sub.attempts)
        if not sub.succeeded:
            return shor.ShorResult(n=cfg.n, factors=[], attempts=attempts,
                                   total_time=_time.perf_counter() - t_start, succeeded=False)
        primes.extend(sub.factors)
    return shor.ShorResult(n=cfg.n, factors=sorted(primes), attempts=attempts,
                           total_time=_time.perf_counter() - t_start, succeeded=True)
