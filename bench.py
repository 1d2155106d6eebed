#!/usr/bin/env python
"""Benchmark: BGV Comp throughput (entries/s) and latency at N=2^14, s=16
(BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

A step is one full Comp (pack_pair + BSGS matvec, compress.py:488-514) of a
seeded synthetic database: bench.run_point's recipe (bench.py:72-94 of the
reference): HeParams(8192, 65537, 3), keygen over plan_rotation_amounts,
a random s-sparse payload (random.Random(seed)), encrypted d and index hint.

* value  -- device-resident: inputs, keys and plan already in HBM; each timed
            step is one CUDA-graph launch of the Comp, timed with CUDA events
            on its stream; L2 is flushed (256 MiB write) between steps.
* e2e    -- through the public C-ABI call hc_comp_async with pinned HOST
            buffers: H2D of the 2*C input ciphertexts, the Comp, D2H of the
            level-0 output, all inside the event-timed region.
* N > 1  -- replicas (SURVEY 8(e) "batched independent queries"): every rank
            runs its own query (own seed and keys); value = total entries
            over all ranks / max-over-ranks time; scaling "weak".
* --impl reference -- the CPU oracle port of the reference's Comp
            (oracle/, C + OpenMP, every host thread) on the same config;
            rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import random
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_DEFAULT, S_DEFAULT, P_DEFAULT, RING = 1 << 14, 16, 65537, 8192


# hcomp.cu StepKind -> the kernels behind it (hc_comp_profile's step kinds)
STEP_KINDS = {10: "key_switch_fused (k_ksfused, HC_KSFUSED=1)", 0: "transforms (k_xf, k_xf_cl)", 1: "crt_digits (k_compose)", 2: "key_mac (k_ksmac)",
              3: "diag_mac (k_diagx)", 5: "memset", 6: "two_prime_intt (k_cl_intt2)",
              7: "key_mac_grouped (k_ksmac_mb)", 8: "add (k_addmod)", 9: "fold_chain (k_tail, persistent)"}


def metric_name(N: int, s: int) -> str:
    n = f"2^{N.bit_length() - 1}" if N & (N - 1) == 0 else str(N)
    return f"Comp encrypted entries/sec (N={n}, s={s})"


def make_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--N", type=int, default=N_DEFAULT)
    # --sparsity: same option under a name torchrun's own parser cannot
    # prefix-match (it reads "--s" as --standalone / --start-method / ...)
    ap.add_argument("--s", "--sparsity", dest="s", type=int, default=S_DEFAULT)
    ap.add_argument("--p", type=int, default=0, help="plaintext prime (default: 65537, or per SURVEY F4 for N >= p)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="CPU baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-flush", type=int, default=1, help="single-context streamed e2e: flush L2 inside the loop (counted)")
    ap.add_argument("--e2e-inflight", type=int, default=1,
                    help="Comps in flight on the device in the reported streamed e2e (default 1, as `value`)")
    ap.add_argument("--e2e-contexts", type=int, default=0,
                    help="independent query contexts the streamed e2e rotates over (0: 4 below N=2^19, else 1)")
    ap.add_argument("--queries", type=int, default=0,
                    help="config 5: Q independent queries (own seeded keys and payloads, one shared database "
                         "shape) spread over the ranks; a step runs every query once; value = aggregate entries/s")
    ap.add_argument("--query-streams", type=int, default=8, help="concurrent CUDA streams per rank in --queries mode")
    ap.add_argument("--no-parity", action="store_true",
                    help="skip the bit-exact check of the GPU answer against the CPU oracle (large N)")
    ap.add_argument("--shard", default="auto", choices=["auto", "on", "off"],
                    help="block-sharded Comp over the ranks (SURVEY 8(e)); auto = on for N >= 2^20 with >1 rank")
    return ap


def parse(argv=None):
    return make_parser().parse_args(argv)


def pick_p(N: int, p: int) -> int:
    if p:
        return p
    if N < 65537:
        return 65537
    for cand in (786433, 1097729, 4423681):
        if cand > N:
            return cand
    raise SystemExit("N too large")


def workload(args, p):
    return {
        "workload": f"BGV Comp (hint path, packed) N={args.N} s={args.s} n={RING} p={p} max_level=3",
        "N": args.N,
        "s": args.s,
        "n": RING,
        "p": p,
        "max_level": 3,
        "seeded_synthetic": "bench.run_point recipe: random.Random(seed) s-sparse payload, encrypted d + index hint",
        "l2": "flushed between timed steps (256 MiB write, untimed)",
        "parallelism": (f"blocks sharded over {args.gpus} GPU(s) + NCCL uint64 reduce (SURVEY 8(e))" if args.shard_on
                        else ("replicas (independent queries)" if args.gpus > 1 else "single")),
    }


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True,
            )
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {
            "sm_mhz": statistics.median(sm) if sm else None,
            "sm_max_mhz": max(mx) if mx else None,
            "reasons": sorted(reasons),
            "samples": len(sm),
        }


def plant(N, s, p, seed):
    rng = random.Random(seed)
    support = sorted(rng.sample(range(1, N + 1), s))
    dense = [0] * N
    for i in support:
        dense[i - 1] = rng.randrange(1, p)
    return dense


def host_threads(O) -> int:
    """Give the CPU oracle every core this process may run on.

    torchrun exports OMP_NUM_THREADS=1 to each rank, which would leave the
    rank-0 CPU leg single-threaded under the driver's N>1 launch."""
    n = len(os.sched_getaffinity(0))
    O.lib().orc_set_num_threads(n)
    return O.lib().orc_num_threads()


def run_reference(args, p, rank):
    """CPU arm: the oracle port of the reference Comp with every host thread."""
    if rank != 0:
        return None
    from oracle import bgv_oracle as O

    host_threads(O)
    threads = O.lib().orc_num_threads()
    be = O.OracleBgv(RING, p, 3, seed=0, check_noise=False)
    keys = be.keygen(*O.plan_rotation_amounts(args.s, RING))
    dense = plant(args.N, args.s, p, 0)
    cts = O.encrypt_vector(dense, args.N, be, keys)
    hint = O.encrypt_vector([1 if x else 0 for x in dense], args.N, be, keys)
    for _ in range(args.warmup):
        O.comp(cts, args.N, args.s, be, keys, hint)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.comp(cts, args.N, args.s, be, keys, hint)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = args.N * args.steps / total
    metric = metric_name(args.N, args.s)
    if args.queries:  # config 5: the CPU processes the queries one after another at this rate
        metric += f", {args.queries} independent queries"
    line = {
        "metric": metric,
        "impl": "reference",
        "value": value,
        "unit": "entries/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True,
        "scaling": "strong" if args.shard_on else "weak",
        "vs_baseline": None,
        "dtype": "u64 (RNS, 54-bit primes)",
        "data": "synthetic (seeded; bench.run_point recipe)",
        "config": workload(args, p),
        "cpu_baseline": {
            "value": value,
            "unit": "entries/s",
            "cores": threads,
            "kind": "port",
            "sample": f"{args.steps} full Comps (N={args.N}, s={args.s}) with the C/OpenMP oracle port of the reference's Comp",
        },
        "e2e": {"value": value, "unit": "entries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    return line


def cpu_baseline_sample(args, p, budget_s):
    """Oracle port timed on this host on full Comps until ~budget_s of work."""
    from oracle import bgv_oracle as O

    host_threads(O)
    be = O.OracleBgv(RING, p, 3, seed=0, check_noise=False)
    keys = be.keygen(*O.plan_rotation_amounts(args.s, RING))
    dense = plant(args.N, args.s, p, 0)
    cts = O.encrypt_vector(dense, args.N, be, keys)
    hint = O.encrypt_vector([1 if x else 0 for x in dense], args.N, be, keys)
    n, t_total = 0, 0.0
    while t_total < budget_s or n == 0:
        t0 = time.perf_counter()
        out = O.comp(cts, args.N, args.s, be, keys, hint)
        t_total += time.perf_counter() - t0
        n += 1
        if n >= 50:
            break
    return out.c, {
        "value": args.N * n / t_total,
        "unit": "entries/s",
        "cores": O.lib().orc_num_threads(),
        "kind": "port",
        "sample": f"{n} full Comps (N={args.N}, s={args.s}), {t_total:.1f} s, C/OpenMP oracle port of the reference Comp",
    }


def oracle_answer(args, p, seed):
    """The CPU oracle's Comp output (level-0 residues [2][1][n]) for the same
    seeded keys, payload and encryption as the GPU arm: the bench line's
    bit-exact parity reference (reference bench.py:96-103 asserts its own
    round trip the same way)."""
    from oracle import bgv_oracle as O

    host_threads(O)
    be = O.OracleBgv(RING, p, 3, seed=seed, check_noise=False)
    keys = be.keygen(*O.plan_rotation_amounts(args.s, RING))
    dense = plant(args.N, args.s, p, seed)
    cts = O.encrypt_vector(dense, args.N, be, keys)
    hint = O.encrypt_vector([1 if x else 0 for x in dense], args.N, be, keys)
    return O.comp(cts, args.N, args.s, be, keys, hint).c


def sass_mix(lib_path: str, mangled: str, bfly: float) -> dict | None:
    """Static fma-pipe instruction mix of a shipped kernel (cuobjdump -sass),
    per butterfly of its 1024-thread schedule (one schedule thread = 52
    butterflies): IMAD-class (IMAD, IMAD.MOV/IADD/X/SHL, HFMA2 moves),
    IMAD.WIDE.U32, IMAD.HI.U32."""
    import re

    try:
        out = subprocess.run(["cuobjdump", "-sass", lib_path], capture_output=True, text=True, timeout=60).stdout
    except Exception:
        return None
    body = None
    for f in re.split(r"\n\s*Function : ", out)[1:]:
        if f.split("\n", 1)[0].strip() == mangled:
            body = f
            break
    if body is None:
        return None
    ops = {"imad": 0, "wide": 0, "hi": 0, "total": 0}
    for ln in body.split("\n"):
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", ln)
        if not m:
            continue
        op = m.group(1)
        ops["total"] += 1
        if op.startswith("IMAD.WIDE"):
            ops["wide"] += 1
        elif op.startswith("IMAD.HI"):
            ops["hi"] += 1
        elif op.startswith(("IMAD", "IMUL", "HFMA2")):
            ops["imad"] += 1
    return {k: v / bfly for k, v in ops.items()}


def kernel_name(tag: int) -> str:
    """hc_comp_profile_ex tag -> the kernel instantiation (kernels.cuh names)."""
    if not tag:
        return "?"
    clu, d, ld, ep, noxf, vt = tag >> 20 & 1, tag >> 16 & 15, tag >> 12 & 15, tag >> 8 & 15, tag >> 4 & 1, tag & 15
    if noxf:
        return f"k_elem<{ld}>"
    return f"k_xf_cl<{d}, {ld}, {ep}, {vt}>" if clu else f"k_xf<{d}, {ld}, {ep}, {vt}>"


def roofline(L, h, sh, comp_ms):
    """Live roofline of the dominant kernel family (the transforms k_xf /
    k_xf_cl): algorithmic butterflies per launch over the launches' event-timed
    duration (un-graphed profile of one Comp), against the measured butterfly
    peak; plus the Comp-level figure and the same kernel saturated."""
    import ctypes

    import numpy as np

    from paper_2408_17063_b200 import _lib

    max_steps = 4096
    sm_ = np.zeros(max_steps, dtype=np.float32)
    sk = np.zeros(max_steps, dtype=np.int32)
    sj = np.zeros(max_steps, dtype=np.int32)
    st_tag = np.zeros(max_steps, dtype=np.int32)
    nsteps = L.hc_comp_profile_ex(h, sh, max_steps, _lib.ptr(sm_), _lib.ptr(sk), _lib.ptr(sj), _lib.ptr(st_tag))
    if nsteps < 0:
        _lib.check(nsteps)
    # the dominant transform kernel: the instantiation with the largest share of
    # the (un-graphed, event-timed) Comp; achieved = its butterflies per launch /
    # its average launch duration
    by_kernel = {}
    for i in range(nsteps):
        if int(sk[i]) == 0 and int(st_tag[i]):
            d = by_kernel.setdefault(int(st_tag[i]), [0.0, 0, 0])
            d[0] += float(sm_[i])
            d[1] += int(sj[i])
            d[2] += 1
    dom_tag, (dom_ms, dom_jobs, dom_launches) = max(by_kernel.items(), key=lambda kv: kv[1][0])
    kinds = {}
    for i in range(nsteps):
        d = kinds.setdefault(int(sk[i]), [0.0, 0, 0])
        d[0] += float(sm_[i])
        d[1] += int(sj[i])
        d[2] += 1
    xf_ms, xf_jobs, xf_launch = kinds.get(0, [0.0, 0, 0])
    prof_total = float(sm_[:nsteps].sum())
    peak = ctypes.c_double()
    _lib.check(L.hc_bf_peak(h, ctypes.byref(peak)))
    # the same transform kernel saturated (4 full waves of 148 single-CTA jobs):
    # what it reaches when the GPU is full, vs the latency-bound launches above
    sat = {}
    for dname, dval in (("fwd", 0), ("inv", 1)):
        us = ctypes.c_double()
        _lib.check(L.hc_bench_xform(h, 592, dval, 20, ctypes.byref(us)))
        sat[dname] = 592 * (RING // 2) * 13 / (us.value * 1e-6) / 1e9
    bfly_per_ntt = (RING // 2) * 13
    achieved = xf_jobs * bfly_per_ntt / (xf_ms * 1e-3) / 1e9 if xf_ms > 0 else 0.0
    peak_g = peak.value / 1e9
    # every transform of the Comp, the fold chain's 2 + 2 x 7 per fold included
    fold_jobs = kinds.get(9, [0.0, 0, 0])[1] * 16
    comp_level = (xf_jobs + fold_jobs) * bfly_per_ntt / comp_ms / 1e6
    dom_name = kernel_name(dom_tag)
    dom_achieved = (dom_jobs / dom_launches) * bfly_per_ntt / (dom_ms / dom_launches * 1e-3) / 1e9
    ncu_traffic = None
    try:  # DRAM bytes per launch of that kernel from the committed ncu --set full capture
        with open(os.path.join(ROOT, "profiles", "r02_ncu_dominant_traffic.json")) as fh:
            ncu_traffic = json.load(fh).get(dom_name)
        if ncu_traffic and ncu_traffic.get("jobs_per_launch"):
            # the captured launch may have been a different size (chunk width): scale per job
            k = (dom_jobs / dom_launches) / ncu_traffic["jobs_per_launch"]
            ncu_traffic = dict(ncu_traffic, dram_bytes_per_launch=ncu_traffic["dram_bytes_per_launch"] * k,
                               algorithmic_bytes_per_launch=int(ncu_traffic["algorithmic_bytes_per_launch"] * k),
                               scaled_from_jobs_per_launch=ncu_traffic["jobs_per_launch"])
    except (OSError, ValueError):
        pass
    # the persistent fold chain (one launch): algorithmic transforms per fold =
    # the two INTTs of res.c1 + 2 x D_1 digit NTTs (the per-cluster recomputation
    # of the INTT is not algorithmic work)
    fold = None
    fc_ms, fc_folds, fc_launches = kinds.get(9, [0.0, 0, 0])
    if fc_launches:
        D1 = 7  # base-2^16 digits of the two-prime level-1 modulus (108 bits)
        fold_bf = fc_folds * (2 + 2 * D1) * (RING // 2) * 13
        fold = {"kernel": "k_foldchain (persistent, 7 clusters of 16 CTAs)", "folds": fc_folds, "ms": fc_ms,
                "share_of_profiled_step": fc_ms / prof_total if prof_total else None,
                "us_per_fold": fc_ms * 1e3 / fc_folds if fc_folds else None,
                "achieved_gbfly_s": fold_bf / (fc_ms * 1e-3) / 1e9,
                "note": "latency-bound serial chain (bit-exactness forbids merging the folds): 26 butterfly stages, "
                        "three DSMEM exchanges, one cluster and one grid barrier per fold on 4 warps per SM"}
    # independent ceiling: measured INT32 multiply-pipe rates x the shipped
    # transform kernel's fma-pipe instruction mix per butterfly (SASS)
    rates = (ctypes.c_double * 3)()
    _lib.check(L.hc_imad_peak(h, rates))
    mix = sass_mix(_lib.LIB_PATH, "_ZN2hc4k_xfILi0ELi0ELi0ELi4EEEvNS_6DevCtxEPKNS_4XJobE", 52.0)
    pipe_bound = None
    if mix and all(r > 0 for r in rates):
        pipe_bound = 1.0 / (mix["imad"] / rates[0] + mix["wide"] / rates[1] + mix["hi"] / rates[2]) / 1e9
    return {
        "kernel": dom_name + " (the dominant transform launch of the Comp; family: k_xf / k_xf_cl, 1 CTA or one "
                  "8-CTA cluster per 8192-point transform, fused loaders/epilogues)",
        "bound": "int-modmul (IMAD pipe; SURVEY 8(d))",
        "achieved": dom_achieved,
        "peak": peak_g,
        "unit": "Gbutterfly/s",
        "frac": dom_achieved / peak_g if peak_g else None,
        "dominant_kernel": {"name": dom_name, "launches_per_comp": dom_launches, "jobs_per_launch": dom_jobs / dom_launches,
                            "avg_launch_ms": dom_ms / dom_launches,
                            "share_of_profiled_step": dom_ms / prof_total if prof_total else None,
                            "algorithmic_unit": "53,248 butterflies per 8192-point transform job"},
        "family_achieved_gbfly_s": achieved,
        "family_frac": achieved / peak_g if peak_g else None,
        "peak_source": "measured live: hc_bf_peak, register-only microbenchmark of the kernels' own lazy CT butterfly at full occupancy (MEASURED_PEAKS.json has no integer peak)",
        "work_unit": "one radix-2 butterfly = one 54-bit modmul + 2 modadds; 4096*13 per 8192-point transform",
        "traffic": (ncu_traffic or {}).get("dram_bytes_per_launch"),
        "traffic_note": ("dram__bytes_read.sum + dram__bytes_write.sum of one launch of the dominant kernel, "
                         "ncu --set full capture in the timed region (profiles/r02_ncu_dominant_traffic.json); "
                         "algorithmic bytes per launch: " + str((ncu_traffic or {}).get("algorithmic_bytes_per_launch"))),
        "fold_chain": dict(fold, frac=fold["achieved_gbfly_s"] / peak_g if peak_g else None) if fold else None,
        "comp_level_gbfly_s": comp_level,
        "comp_level_frac": comp_level / peak_g if peak_g else None,
        "xform_share_of_step": xf_ms / prof_total if prof_total else None,
        "xform_jobs_per_comp": xf_jobs + fold_jobs,
        "xform_launches_per_comp": xf_launch,
        "profiled_step_ms_ungraphed": prof_total,
        "per_kind_ms": {STEP_KINDS.get(k, str(k)): round(v[0], 4) for k, v in sorted(kinds.items())},
        "saturated_592_jobs_gbfly_s": sat,
        "saturated_frac": {k: v / peak_g for k, v in sat.items()} if peak_g else None,
        "int32_pipe": {
            "measured_gops_s": {"IMAD": rates[0] / 1e9, "IMAD.WIDE.U32": rates[1] / 1e9, "IMAD.HI.U32": rates[2] / 1e9},
            "source": "hc_imad_peak: register-only mad.lo / mad.wide / mad.hi u32 streams, 8 chains x 2048 threads per SM",
            "k_per_butterfly": mix,
            "k_source": "cuobjdump -sass of the shipped k_xf<0,0,0,4> (throughput forward transform), per butterfly",
            "modeled_bound_gbfly_s": pipe_bound,
            "frac_of_modeled_bound": (achieved / pipe_bound) if pipe_bound else None,
            "comp_level_frac_of_modeled_bound": (comp_level / pipe_bound) if pipe_bound else None,
            "saturated_frac_of_modeled_bound": {k: v / pipe_bound for k, v in sat.items()} if pipe_bound else None,
        },
    }


def run_queries(args, p, world, rank, local, dist):
    """Config 5: Q independent queries, each with its own seeded
    key pair, rotation keys and s-sparse payload (query q: seed q), over one
    (N, s) database shape.  Query q runs on rank q % world; every rank keeps
    its queries device-resident (own keys, inputs and CUDA graph) and shares
    ONE copy of the plan's diagonals among them (hc_plan_shared).  A step
    launches every query once, round-robin over --query-streams streams;
    value = Q * N / (max-over-ranks step time).  No collective: replicas."""
    import numpy as np
    import torch

    import paper_2408_17063_b200 as P
    from paper_2408_17063_b200 import _lib

    he = P.HeParams(RING, p, 3)
    params = P.CompressionParams(args.N, args.s, he)
    mine = [q for q in range(args.queries) if q % world == rank]
    L = _lib.lib()
    t_setup = time.perf_counter()
    qs, first = [], None
    for q in mine:
        be = P.B200BgvBackend(he, seed=q, device=local, noise_guard=False)
        keys = be.keygen(*P.plan_rotation_amounts(args.s, RING))
        dense = plant(args.N, args.s, p, q)
        cd = np.ascontiguousarray(np.stack([c.payload.res for c in P.encrypt_vector(dense, params, be, keys)]))
        cv = np.ascontiguousarray(np.stack([c.payload.res for c in P.encrypt_vector([1 if x else 0 for x in dense], params, be, keys)]))
        dc = P.DeviceComp(be, params, keys, share_with=first)
        first = first or dc
        dc.set_inputs(cd, cv)
        qs.append(dict(q=q, be=be, keys=keys, dense=dense, dc=dc, h=be._ctx(),
                       cd_h=torch.from_numpy(cd).pin_memory(), cv_h=torch.from_numpy(cv).pin_memory(),
                       out_h=torch.empty((2, 1, RING), dtype=torch.int64).pin_memory()))
    setup_s = time.perf_counter() - t_setup
    ns = max(1, min(args.query_streams, len(qs)))
    streams = [torch.cuda.Stream() for _ in range(ns)]
    main_s = torch.cuda.Stream()
    C = params.num_ciphertexts

    def step(e2e: bool):
        ev = torch.cuda.Event()
        ev.record(main_s)
        for st in streams:
            st.wait_event(ev)
        for i, d in enumerate(qs):
            sh = streams[i % ns].cuda_stream
            if e2e:
                _lib.check(L.hc_comp_async(d["h"], d["cd_h"].data_ptr(), d["cv_h"].data_ptr(), C, d["out_h"].data_ptr(), sh))
            else:
                d["dc"].launch(sh)
        for st in streams:
            e = torch.cuda.Event()
            e.record(st)
            main_s.wait_event(e)

    # correctness: every query decrypts to its own payload's power sums
    step(False)
    torch.cuda.synchronize()
    outs = {}
    for d in qs:
        out = d["dc"].output()
        outs[d["q"]] = out
        be = d["be"]
        m = be.decrypt(P.Ciphertext(be.backend_id, d["keys"].key_id, 0, P.RnsPayload(out, 0.0, (be.q[0],))), d["keys"])
        w = [int(x) for x in m.rows[0][: args.s]]
        assert w == [sum(pow(i + 1, j + 1, p) for i, v in enumerate(d["dense"]) if v) % p for j in range(args.s)], \
            f"query {d['q']} does not decrypt to its power sums"
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    with torch.cuda.stream(main_s):
        for _ in range(args.warmup):
            flush.zero_()
            step(False)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with torch.cuda.stream(main_s):
        for a, b in evs:
            flush.zero_()
            a.record(main_s)
            step(False)
            b.record(main_s)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    e2e_evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with torch.cuda.stream(main_s):
        step(True)
        torch.cuda.synchronize()
        for a, b in e2e_evs:
            flush.zero_()
            a.record(main_s)
            step(True)
            b.record(main_s)
    torch.cuda.synchronize()
    clk = clocks.stop()
    for d in qs:
        assert np.array_equal(d["out_h"].numpy().view(np.uint64), outs[d["q"]]), "e2e answer differs"
    t_ms, e2e_ms = sum(step_ms), sum(a.elapsed_time(b) for a, b in e2e_evs)
    if dist:
        tt = torch.tensor([t_ms, e2e_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms, e2e_ms = tt.tolist()
    per_step = t_ms / args.steps
    units = args.queries * args.N
    info = qs[0]["be"].plan_info()
    rf = roofline(L, qs[0]["h"], main_s.cuda_stream, per_step / max(1, len(qs)))
    line = {
        "metric": metric_name(args.N, args.s) + f", {args.queries} independent queries",
        "value": units / (per_step * 1e-3),
        "unit": "entries/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": per_step,
        "latency_ms": {"median": statistics.median(step_ms), "min": min(step_ms), "max": max(step_ms),
                       "per_query_amortised": per_step / max(1, len(qs))},
        "higher_is_better": True,
        "scaling": "strong",  # total work (Q queries) fixed as N grows
        "vs_baseline": None,
        "dtype": "u64 (RNS, 54-bit primes)",
        "data": "synthetic (seeded per query; real keygen + encryption per query)",
        "config": dict(workload(args, p), workload=f"config 5: {args.queries} independent queries, BGV Comp N={args.N} "
                       f"s={args.s} n={RING} p={p}, own keys per query, diagonals shared per GPU",
                       queries=args.queries, queries_per_rank=len(qs), streams_per_rank=ns,
                       parallelism=f"queries round-robin over {world} GPU(s), {ns} streams each (no collective)"),
        "e2e": {"value": units / (e2e_ms / args.steps * 1e-3), "unit": "entries/s", "ms_per_step": e2e_ms / args.steps,
                "mode": "every query: H2D of its inputs from pinned memory, its Comp graph, D2H of its answer "
                        "(hc_comp_async on its stream)",
                "h2d_bytes_per_step": int(sum(d["cd_h"].numel() * 8 * 2 for d in qs)),
                "d2h_bytes_per_step": int(len(qs) * 2 * RING * 8)},
        "gpu_launches": int(info["kernel_launches"]) * len(qs) * args.steps * 2,
        "kernel_launches_per_comp": int(info["kernel_launches"]),
        "roofline": rf,
        "clocks": clk,
        "setup_s": round(setup_s, 1),
        "plan": info,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu_out, line["cpu_baseline"] = cpu_baseline_sample(args, p, args.cpu_seconds)
        cpu_out = np.asarray(cpu_out, dtype=np.uint64)
    else:
        cpu_out = None
    if rank == 0 and not args.no_parity:  # query 0 (seed 0) against the oracle
        ref = cpu_out if cpu_out is not None else np.asarray(oracle_answer(args, p, 0), dtype=np.uint64)
        ok = bool(np.array_equal(ref, outs[0]))
        line["parity"] = {"status": "bit-exact" if ok else "MISMATCH",
                          "against": "CPU oracle port of the reference Comp, query 0 (seed 0); every query decrypt-checked",
                          "query_seed": 0}
        assert ok, "query 0 differs from the CPU oracle"
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    args = parse()
    p = pick_p(args.N, args.p)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    args.shard_on = args.shard == "on" or (args.shard == "auto" and world > 1 and args.N >= (1 << 20))
    args.gpus = world
    if args.impl == "reference":
        line = run_reference(args, p, rank)
        if line is not None:
            print(json.dumps(line), flush=True)
        return

    import ctypes

    import numpy as np
    import torch

    import paper_2408_17063_b200 as P
    from paper_2408_17063_b200 import _lib

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    if args.queries:
        return run_queries(args, p, world, rank, local, dist)
    shard = args.shard_on
    he = P.HeParams(RING, p, 3)
    params = P.CompressionParams(args.N, args.s, he)
    seed = 0 if shard else rank  # sharded: one query split over the ranks; replicas: one query per rank
    be = P.B200BgvBackend(he, seed=seed, device=local, noise_guard=False)
    keys = be.keygen(*P.plan_rotation_amounts(args.s, RING))
    dense = plant(args.N, args.s, p, seed)
    cts = P.encrypt_vector(dense, params, be, keys)
    hint = P.encrypt_vector([1 if x else 0 for x in dense], params, be, keys)
    if shard:  # this rank's plan covers its own blocks only (hc_plan_range)
        from paper_2408_17063_b200.dist import shard_blocks

        b0, b1 = shard_blocks(params.num_blocks, world, rank)
        be.plan(args.N, args.s, keys, block_range=(b0, b1))
        dc = None
    else:
        dc = P.DeviceComp(be, params, keys)
    cd = np.ascontiguousarray(np.stack([c.payload.res for c in cts]))
    cv = np.ascontiguousarray(np.stack([c.payload.res for c in hint]))

    stream = torch.cuda.Stream()
    sh = stream.cuda_stream
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    L = _lib.lib()
    h = be._ctx()
    out_h = torch.empty((2, 1, RING), dtype=torch.int64).pin_memory()

    if shard:
        c0, c1 = b0 // 2, (b1 + 1) // 2
        cd_h = torch.from_numpy(np.ascontiguousarray(cd[c0:c1])).pin_memory()
        cv_h = torch.from_numpy(np.ascontiguousarray(cv[c0:c1])).pin_memory()
        part = torch.zeros(L.hc_partial_words(h), dtype=torch.int64, device="cuda")
        _lib.check(L.hc_comp_set_inputs_range(h, cd_h.data_ptr(), cv_h.data_ptr(), c0, c1, sh))
        torch.cuda.synchronize()

        def step(e2e: bool):
            if e2e:
                _lib.check(L.hc_comp_set_inputs_range(h, cd_h.data_ptr(), cv_h.data_ptr(), c0, c1, sh))
            _lib.check(L.hc_comp_partial(h, b0, b1, ctypes.c_void_p(part.data_ptr()), sh))
            if dist:
                dist.reduce(part, dst=0, op=dist.ReduceOp.SUM)  # joins the current stream
            if rank == 0:
                _lib.check(L.hc_comp_finish(h, ctypes.c_void_p(part.data_ptr()), sh))
                if e2e:
                    _lib.check(L.hc_comp_get_output_async(h, out_h.data_ptr(), sh))

        h2d_bytes = int(cd_h.numel() * 8 + cv_h.numel() * 8)
    else:
        dc.set_inputs(cd, cv)
        cd_h = torch.from_numpy(cd).pin_memory()
        cv_h = torch.from_numpy(cv).pin_memory()

        def step(e2e: bool):
            if e2e:
                _lib.check(L.hc_comp_async(h, cd_h.data_ptr(), cv_h.data_ptr(), cd.shape[0], out_h.data_ptr(), sh))
            else:
                dc.launch(sh)

        h2d_bytes = int(cd.nbytes + cv.nbytes)

    def output():
        torch.cuda.synchronize()
        # sharded: only the root holds the answer; replicas: every rank has its own
        if rank != 0 and shard:
            return None
        o = np.empty((2, 1, RING), dtype=np.uint64)
        _lib.check(L.hc_comp_get_output(h, _lib.ptr(o)))
        return o

    # correctness gate: the timed Comp must decrypt to the payload's power sums
    with torch.cuda.stream(stream):
        step(False)
    out = output()
    if rank == 0:
        ct = P.Ciphertext(be.backend_id, keys.key_id, 0, P.RnsPayload(out, 0.0, (be.q[0],)))
        m = be.decrypt(ct, keys)
        w = [int(x) for x in m.rows[0][: args.s]]
        e = [int(x) for x in m.rows[1][: args.s]]
        want_w = [sum(pow(i + 1, j + 1, p) for i, v in enumerate(dense) if v) % p for j in range(args.s)]
        want_e = [sum(v * pow(i + 1, j + 1, p) for i, v in enumerate(dense) if v) % p for j in range(args.s)]
        assert w == want_w, "Comp output does not decrypt to the expected power sums w"
        assert e == want_e, "Comp output does not decrypt to the expected weighted sums e"

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            flush.zero_()
            step(False)
    torch.cuda.synchronize()

    # ---- device-resident timed region ----
    clocks = ClockSampler(local)
    clocks.start()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include "timed/" selects these launches
    with torch.cuda.stream(stream):
        for a, b in evs:
            flush.zero_()
            a.record(stream)
            step(False)
            b.record(stream)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    if dist:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    t_ms = sum(step_ms)

    # ---- end to end through the public C-ABI: pinned host inputs in, result out ----
    e2e_evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with torch.cuda.stream(stream):
        for _ in range(2):
            step(True)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        for a, b in e2e_evs:
            flush.zero_()
            a.record(stream)
            step(True)
            b.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    if rank == 0:
        assert np.array_equal(out_h.numpy().view(np.uint64), out), "e2e output differs from the device-resident run"
    e2e_serial_ms = sum(a.elapsed_time(b) for a, b in e2e_evs)
    e2e_ms = e2e_serial_ms
    e2e_stream_ms = None
    e2e_rot = None
    if not shard:
        # ---- streamed end to end: the serving pipeline.  Step i+1's inputs go
        # up over PCIe (hc_comp_upload_async on a copy stream) while step i
        # computes (hc_comp_launch) and step i-1's answer comes back
        # (hc_comp_get_output_async on a third stream); every step still copies
        # its own inputs in and its answer out inside the timed region.  The
        # steps rotate over R independent query contexts -- own seeded keys,
        # payload, plan (diagonals not shared) and device buffers -- whose
        # keys + diagonals (R x ~117 MB at the headline) do not fit the 126 MB
        # L2 together: between two uses of a context the other contexts'
        # streams evict it, so every step starts cold WITHOUT a flush in the
        # timed loop (the contract's "inputs larger than L2" option; checked
        # below: the device-resident rotation runs at the flushed latency).
        # Every context's final answer is checked against its own
        # device-resident result ----
        R = args.e2e_contexts if args.e2e_contexts > 0 else (4 if args.N < (1 << 19) else 1)
        Cn = cd.shape[0]
        ctxs = [dict(be=be, keys=keys, dc=dc, h=h, cd_h=cd_h, cv_h=cv_h, want=out)]
        for r in range(1, R):
            sd = 1000 + 16 * rank + r
            be_r = P.B200BgvBackend(he, seed=sd, device=local, noise_guard=False)
            keys_r = be_r.keygen(*P.plan_rotation_amounts(args.s, RING))
            dense_r = plant(args.N, args.s, p, sd)
            cd_r = np.ascontiguousarray(np.stack([c.payload.res for c in P.encrypt_vector(dense_r, params, be_r, keys_r)]))
            cv_r = np.ascontiguousarray(np.stack([c.payload.res for c in P.encrypt_vector([1 if x else 0 for x in dense_r], params, be_r, keys_r)]))
            dc_r = P.DeviceComp(be_r, params, keys_r)
            dc_r.set_inputs(cd_r, cv_r)
            dc_r.launch(sh)
            torch.cuda.synchronize()
            ctxs.append(dict(be=be_r, keys=keys_r, dc=dc_r, h=be_r._ctx(), cd_h=torch.from_numpy(cd_r).pin_memory(),
                             cv_h=torch.from_numpy(cv_r).pin_memory(), want=dc_r.output()))
        for c in ctxs:
            c["out_h"] = torch.empty((2, 1, RING), dtype=torch.int64).pin_memory()
        h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
        ev = lambda: torch.cuda.Event()
        stage = [[torch.empty_like(cd_h, device="cuda"), torch.empty_like(cv_h, device="cuda")] for _ in range(2)] if R == 1 else None

        # Comps in flight on the device (compute streams).  The reported e2e keeps
        # ONE Comp on the GPU at a time (as `value` does); deeper pipelines are
        # measured beside it (e2e.inflight) -- a query's serial level-1 tail
        # leaves most SMs idle, which the next query's front end can use
        cstreams = [stream] + [torch.cuda.Stream() for _ in range(3)]

        def pipeline(nsteps, K):
            up_done = [ev() for _ in range(nsteps)]
            comp_done = [ev() for _ in range(nsteps)]
            d2h_done = [ev() for _ in range(nsteps)]
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

            set_done = [ev() for _ in range(nsteps)]

            def upload(i):
                c = ctxs[i % R]
                if R == 1:  # one context: inputs land in one of two staging buffers, copied in on the compute stream
                    if i >= 2:
                        h2d_s.wait_event(set_done[i - 2])
                    with torch.cuda.stream(h2d_s):
                        stage[i % 2][0].copy_(c["cd_h"], non_blocking=True)
                        stage[i % 2][1].copy_(c["cv_h"], non_blocking=True)
                    up_done[i].record(h2d_s)
                    return
                if i >= R:
                    h2d_s.wait_event(comp_done[i - R])  # this context's previous Comp has read its inputs
                _lib.check(L.hc_comp_upload_async(c["h"], c["cd_h"].data_ptr(), c["cv_h"].data_ptr(), Cn, h2d_s.cuda_stream))
                up_done[i].record(h2d_s)

            with torch.cuda.stream(stream):
                t0.record(stream)
                for st in [h2d_s, d2h_s] + cstreams[1:]:
                    st.wait_event(t0)
                for i in range(min(K, nsteps)):
                    upload(i)
                for i in range(nsteps):
                    c = ctxs[i % R]
                    cs = cstreams[i % K]
                    cs.wait_event(up_done[i])
                    if i >= R:
                        cs.wait_event(d2h_done[i - R])  # this context's previous answer was read back
                    if R == 1 and args.e2e_flush and args.N < (1 << 19):
                        with torch.cuda.stream(cs):
                            flush.zero_()  # a single small context would stay L2-resident (counted)
                    if R == 1:
                        _lib.check(L.hc_comp_set_inputs_device(c["h"], stage[i % 2][0].data_ptr(), stage[i % 2][1].data_ptr(), Cn, cs.cuda_stream))
                        set_done[i].record(cs)
                    c["dc"].launch(cs.cuda_stream)
                    comp_done[i].record(cs)
                    if i + K < nsteps:
                        upload(i + K)
                    d2h_s.wait_event(comp_done[i])
                    _lib.check(L.hc_comp_get_output_async(c["h"], c["out_h"].data_ptr(), d2h_s.cuda_stream))
                    d2h_done[i].record(d2h_s)
                stream.wait_event(d2h_done[-1])  # the D2H stream is in order: every answer is back
                t1.record(stream)
            torch.cuda.synchronize()
            return t0.elapsed_time(t1)

        def check_answers():
            for c in ctxs[: min(R, args.steps)]:
                assert np.array_equal(c["out_h"].numpy().view(np.uint64), c["want"]), "streamed e2e answer differs"
                c["out_h"].zero_()

        K0 = max(1, min(args.e2e_inflight, R - 1 if R > 1 else 1))
        pipeline(2 * R, K0)  # warm
        if dist:
            dist.barrier()
        e2e_stream_ms = pipeline(args.steps, K0)
        check_answers()
        inflight = {}
        for K in (2, 3):  # needs more contexts than Comps in flight
            if K < R and K != K0:
                pipeline(2 * R, K)
                inflight[str(K)] = pipeline(args.steps, K) / args.steps
                check_answers()
        # coldness check of the rotation: device-resident Comps round-robin over
        # the contexts, no flush, against the flushed latency reported as `value`
        rot_evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        with torch.cuda.stream(stream):
            for i in range(2 * R):
                ctxs[i % R]["dc"].launch(sh)
            for i, (a, b) in enumerate(rot_evs):
                a.record(stream)
                ctxs[i % R]["dc"].launch(sh)
                b.record(stream)
        torch.cuda.synchronize()
        e2e_rot = {"contexts": R, "comps_in_flight": K0, "ms_per_step_with_more_comps_in_flight": inflight,
                   "device_resident_ms_per_step_no_flush": statistics.median(a.elapsed_time(b) for a, b in rot_evs),
                   "device_resident_ms_per_step_flushed": statistics.median(step_ms)}
        # both are end to end (every step copies its inputs in and its answer
        # out inside the timed region); the line reports the faster schedule
        e2e_ms = min(e2e_serial_ms, e2e_stream_ms)
    # pinned H2D bandwidth of this box for the e2e input volume (the two
    # input lists on two copy streams, as hc_comp_async issues them)
    h2d_gbs = None
    if not shard:
        dst = [torch.empty_like(cd_h, device="cuda"), torch.empty_like(cv_h, device="cuda")]
        cps = [torch.cuda.Stream(), torch.cuda.Stream()]
        ts = []
        for it in range(12):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for i, (src, st) in enumerate(zip((cd_h, cv_h), cps)):
                st.wait_event(a)
                with torch.cuda.stream(st):
                    dst[i].copy_(src, non_blocking=True)
            for st in cps:
                e = torch.cuda.Event()
                e.record(st)
                stream.wait_event(e)
            b.record(stream)
            torch.cuda.synchronize()
            if it >= 2:
                ts.append(a.elapsed_time(b))
        h2d_gbs = h2d_bytes / (statistics.median(ts) * 1e-3) / 1e9
    info = be.plan_info()  # kernel launches per Comp (graph built by now)
    if int(info["kernel_launches"]) <= 0:
        raise RuntimeError(f"no captured Comp graph to count launches from: {info}")

    if dist:
        tt = torch.tensor([t_ms, e2e_ms, e2e_serial_ms, e2e_stream_ms or 0.0], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms, e2e_ms, e2e_serial_ms, e2e_stream_ms = tt.tolist()
        e2e_stream_ms = e2e_stream_ms or None

    rf = roofline(L, h, sh, t_ms / args.steps)

    per_step_ms = t_ms / args.steps
    units = args.N if shard else args.N * world  # sharded: one Comp per step; replicas: one per rank
    value = units / (per_step_ms * 1e-3)
    e2e_value = units / (e2e_ms / args.steps * 1e-3)
    line = {
        "metric": metric_name(args.N, args.s),
        "value": value,
        "unit": "entries/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": per_step_ms,
        "latency_ms": {"median": statistics.median(step_ms), "min": min(step_ms), "max": max(step_ms)},
        "higher_is_better": True,
        "scaling": "strong" if shard else "weak",
        "vs_baseline": None,
        "dtype": "u64 (RNS, 54-bit primes)",
        "data": "synthetic (seeded; bench.run_point recipe; real keygen + encryption)",
        "config": workload(args, p),
        "e2e": {
            "value": e2e_value,
            "unit": "entries/s",
            "ms_per_step": e2e_ms / args.steps,
            "mode": ("sharded: per-step H2D of the rank's ciphertexts, partial, reduce, finish, D2H"
                     if shard else
                     ("serial: each step's event pair holds the H2D of its input ciphertexts from pinned host "
                      "memory, the Comp (hc_comp_async: one graph launch) and the D2H of the answer; L2 "
                      "flushed before every step, untimed as for value")
                     if e2e_stream_ms is None or e2e_serial_ms <= e2e_stream_ms else
                     "streamed: step i+1's H2D (hc_comp_upload_async, copy stream) and step i-1's D2H overlap "
                     "step i's Comp; steps rotate over independent query contexts (own keys, plan, buffers) "
                     "whose keys + diagonals exceed L2 together, so each step is cold without a flush"),
            "serial_ms_per_step": e2e_serial_ms / args.steps,
            "streamed_ms_per_step": (e2e_stream_ms / args.steps) if e2e_stream_ms else None,
            "streamed_rotation": e2e_rot,
            "h2d_bytes_per_step": h2d_bytes,
            "d2h_bytes_per_step": 2 * RING * 8,
            "h2d_gbs_measured": h2d_gbs,
            "h2d_note": "pinned host memory; the two input lists go up on two copy engines (hc_comp_async)",
        },
        # timed regions: device-resident, serial e2e and (unsharded) streamed e2e, `steps` Comps each
        "gpu_launches": int(info["kernel_launches"]) * args.steps * (2 if shard else 3),
        "kernel_launches_per_comp": int(info["kernel_launches"]),
        "roofline": rf,
        "clocks": clk,
        "plan": info,
    }
    cpu_out = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu_out, line["cpu_baseline"] = cpu_baseline_sample(args, p, args.cpu_seconds)
    if rank == 0 and not args.no_parity:
        # bit-exact gate: the answer every timed step produced (device-resident,
        # e2e and streamed runs were checked equal to it above) against the CPU
        # oracle's Comp on the same seeded keys, payload and encryption
        t_or = time.perf_counter()
        ref = cpu_out if cpu_out is not None else oracle_answer(args, p, seed)
        ok = bool(np.array_equal(np.asarray(ref, dtype=np.uint64), out))
        line["parity"] = {
            "status": "bit-exact" if ok else "MISMATCH",
            "against": "CPU oracle port of the reference Comp (oracle/, pinned to reference goldens), same seed",
            "compared": "all 2 x 8192 residues of the level-0 answer ciphertext (+ decrypted w and e vs the planted payload)",
            "query_seed": seed,
            "oracle_s": round(time.perf_counter() - t_or, 2),
        }
        assert ok, "GPU Comp answer differs from the CPU oracle"
    elif rank == 0:
        line["parity"] = {"status": "decrypt-checked only (--no-parity)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
