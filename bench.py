#!/usr/bin/env python
"""Benchmark: order-MCMC iterations/s at n=60, k=4 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  (N>1: python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N)

A "step" is one call of the reference-facing chain API (bnmc_gpu_run_chains)
running C independent chains per GPU for I MCMC iterations each; every
iteration is a full run_mcmc iteration (sampler.cpp:92-111): proposal, exact
rescan of the changed node rows, Metropolis-Hastings test, tracker update,
trace row. The scan is the sorted-row walk (scan_mode 2, one fused kernel
launch per step); chain c is bit-identical to the reference's run_mcmc with
that seed (checked against the CPU reference below).

value      = iterations of all chains of all ranks / max over ranks of the summed
             device time of the chain kernel (CUDA events on the library's
             stream; the score table is resident in HBM).
e2e        = same metric through the C-ABI with HOST buffers: wall time of the
             run_chains calls incl. H2D (seeds) and D2H (traces, trackers,
             final states into pinned host buffers).
roofline   = the fused walk kernel: algorithmic bytes per launch (sorted entries
             walked x 16 B + enumerated local scores x 8 B, counted on the device)
             / its launch time, against MEASURED_PEAKS.json hbm_gbs. The
             full-row scan path (scan_mode 1) is measured beside it
             (full_scan_path) with its own K2 roofline.
cpu_baseline = the unmodified reference (oracle/_ref) run_mcmc on this box's host
             cores on the GPU-built table (BNSC export -> ScoreCache::load), a
             bounded number of iterations; its trace is checked bit-for-bit
             against our chain with the same seed.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "order-MCMC iterations/sec at n=60,k=4"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, index: int):
        self.index, self.samples, self.proc = index, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def ncu_profile(kernel):
    """ncu --set full figures of `kernel` at this bench's configuration
    (profiles/ncu_traffic.json, written by tools/ncu_traffic.py from the
    round's capture): DRAM bytes, warp instructions, IPC, issue-slot use per
    launch and the capture it came from; {} when absent."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return dict(json.load(f)[kernel])
    except Exception:
        return {}


class _HostData:
    """Dataset-shaped view of host arrays (n, rows(), cells, cards)."""

    def __init__(self, cells, cards):
        self.cells, self.cards, self.n = cells, np.asarray(cards, np.int32), int(cells.shape[1])

    def rows(self):
        return int(self.cells.shape[0])


def reference_precompute(data, s, samples=4000, seed=0):
    """The reference's ScoreCache::build time at this config on this host,
    extrapolated from local_score (count_statistics + local_score_from_counts,
    scoring.cpp:82-141, the per-entry body of the build loop at
    scoring.cpp:179-190) on uniformly sampled table entries, single-threaded,
    x entries / OpenMP threads (linear scaling: optimistic for the reference).
    SURVEY §8(d) prescribes this when the full build does not fit the run."""
    from oracle import ref
    if not ref.available():
        return None
    n, m = data.n, data.rows()
    S = ref.bounded_subset_count(n - 1, s)
    rng = np.random.default_rng(seed)
    ents = []
    for _ in range(samples):
        v = int(rng.integers(n))
        cm = ref.subset_at(int(rng.integers(S)), n - 1, s)
        low = cm & ((1 << v) - 1)
        ents.append((v, low | ((cm >> v) << (v + 1))))
    _, sec = ref.local_score_batch(data.cells, data.cards, [v for v, _ in ents],
                                   [pm for _, pm in ents])
    per = sec / samples
    threads = ref.max_threads()
    return {"precompute_s": per * n * S / threads, "seconds_per_entry_1thread": per,
            "entries": n * S, "threads": threads, "sampled_entries": samples,
            "method": "reference local_score on uniformly sampled entries, single thread, "
                      "x n*S(n-1,s) / OpenMP threads (SURVEY 8(d))"}


def flush_l2(torch, buf):
    buf.add_(1.0)  # 256 MiB write > 126 MB L2


def cpu_model():
    """Host CPU model string (/proc/cpuinfo), reported with the CPU baseline."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_cache(cache, cfg):
    """The reference's ScoreCache::load of the GPU-built table (BNSC export)."""
    from oracle import ref
    if not ref.available():
        return None
    tmp = "/dev/shm" if os.path.isdir("/dev/shm") else None
    with tempfile.TemporaryDirectory(dir=tmp) as d:
        path = os.path.join(d, "cfg.bnsc")
        cache.save(path)
        return ref.Cache.load(path, cache.s(), cfg.gamma, cfg.ess, False)


def headline_parity(rc, out, seeds, priors, n, s, iters, count, team=8):
    """Chains of the LAST timed launch (18,944 chains, the headline kernel
    variant) compared bit-for-bit with the unmodified reference's run_mcmc
    (oracle/_ref, sampler.cpp:58-116) on the same table: full traces
    (proposed, accepted, best), trackers (masks, totals), final order, final
    score, accepted count. Chains are spread over CTAs and warp slots."""
    from oracle import ref
    C_ = len(seeds)
    idx = sorted({min(C_ - 1, (k * C_) // count + (k % team)) for k in range(count)})
    dummy = np.zeros((1, n), np.uint8)  # run_mcmc needs rows > 0; prebuilt skips the build
    cards = np.full(n, 3, np.int32)
    ok, bad, t0 = 0, [], time.perf_counter()
    for c in idx:
        r = ref.run_mcmc(dummy, cards, s, iters, int(seeds[c]), priors=priors, prebuilt=rc)
        k = int(out.tracker_count[c])
        same = (np.array_equal(out.trace_proposed[c].view(np.uint64), r.trace_proposed.view(np.uint64))
                and np.array_equal(out.trace_accepted[c].astype(bool), r.trace_accepted)
                and np.array_equal(out.trace_best[c].view(np.uint64), r.trace_best.view(np.uint64))
                and k == r.tracker_totals.size
                and np.array_equal(out.tracker_masks[c, :k], r.tracker_masks)
                and np.array_equal(out.tracker_totals[c, :k].view(np.uint64),
                                   r.tracker_totals.view(np.uint64))
                and np.array_equal(out.final_order[c], r.final_order)
                and float(out.final_score[c]) == r.final_score
                and int(out.accepted[c]) == r.accepted)
        ok += int(same)
        if not same:
            bad.append(c)
    return {"parity_checked_chains": f"{ok}/{len(idx)}", "chain_indices": idx,
            "iterations": iters, "mismatched": bad, "reference_seconds": time.perf_counter() - t0,
            "against": "oracle/_ref run_mcmc (unmodified reference) on the GPU-built table"}


def cpu_baseline(rc, n, s, priors, ours_trace, iters, seed):
    """Reference run_mcmc (oracle/_ref) on the GPU-built table, all host threads."""
    from oracle import ref
    if rc is None:
        return None
    dummy = np.zeros((1, n), np.uint8)  # run_mcmc needs rows > 0; prebuilt skips the build
    cards = np.full(n, 3, np.int32)
    t0 = time.perf_counter()
    r = ref.run_mcmc(dummy, cards, s, iters, seed, priors=priors, prebuilt=rc)
    wall = time.perf_counter() - t0
    parity = bool(np.array_equal(r.trace_proposed, ours_trace[:iters]))
    return {"value": iters / r.sampling_seconds, "unit": "iterations/s",
            "cores": ref.max_threads(), "cpu_model": cpu_model(), "kind": "reference",
            "sample": f"{iters} run_mcmc iterations (seed {seed}) of the unmodified reference "
                      f"(oracle/_ref, OpenMP {ref.max_threads()} threads) on the GPU-built table "
                      f"loaded via ScoreCache::load; wall {wall:.1f}s",
            "trace_bit_exact_vs_gpu": parity}


def walk_roofline(prof, avg_launch_s, peak, peak_src, alg_bytes, chain_iters_per_launch):
    """Roofline of the fused walk kernel (K2W). Its working set (the touched
    tops of the sorted rows) is L2-resident: DRAM moves ~9 GB per launch while
    the walk touches ~450 GB of sorted entries, so HBM is not its bound; it is
    bound by instruction issue and L2 latency. `achieved`/`frac` are the MEASURED
    DRAM bytes per launch (ncu capture of this configuration) over this run's
    launch time against the HBM peak; `issue` carries the ncu instruction
    count, IPC and issue-slot use that do bound it."""
    # ncu figures are per chain-iteration of the captured launch (one chain
    # block), scaled to this step's chain-iterations
    dpc = prof.get("dram_bytes_per_chain_iteration")
    dram = dpc * chain_iters_per_launch if dpc else None
    ach = dram / avg_launch_s / 1e9 if dram else None
    ipc_ = prof.get("warp_instructions_per_chain_iteration")
    inst = ipc_ * chain_iters_per_launch if ipc_ else None
    return {"bound": "issue/L2 (latency)", "achieved": ach, "peak": peak, "unit": "GB/s",
            "frac": ach / peak if ach else None, "traffic": dram,
            "traffic_source": prof.get("source"),
            "kernel": "walk_chain_kernel (K2W: fused scan + chain step)",
            "peak_source": peak_src, "avg_launch_us": avg_launch_s * 1e6,
            "issue": {"warp_instructions_per_launch": inst,
                      "warp_instructions_per_chain_iteration":
                          inst / chain_iters_per_launch if inst else None,
                      "ipc": prof.get("ipc"), "ipc_peak": 4.0,
                      "issue_slots_busy": prof.get("issue_slots_busy"),
                      "top_stalls": prof.get("top_stalls")},
            "walked_bytes_per_launch": alg_bytes,
            "walked_GBps": alg_bytes / avg_launch_s / 1e9,
            "note": "walked bytes = sorted entries walked x 16 B + enumerated local scores x 8 B "
                    "(counted on the device); they are served by L1/L2, DRAM traffic is the "
                    "ncu-measured figure"}


def reference_api_e2e(P, cache, pri, cfg, chains, iters, steps=3):
    """Wall-clock throughput through the reference-shaped APIs that return
    McmcResult objects (not the bench's caller-owned pinned batch): the Python
    mirror's run_chains (pooled pinned buffers, lazy McmcResult) and the C++
    drop-in bnmc::run_chains (tools/cxx/e2e_probe), each vs its device time."""
    c1 = P.RunConfig(max_parents=cfg.max_parents, iterations=iters, scan_mode=2,
                     memory_cap_bytes=cfg.memory_cap_bytes, device=cfg.device)
    seeds = np.arange(1, chains + 1, dtype=np.uint64)
    P.run_chains(cache, pri, seeds, c1)  # warm-up (pool)
    wall = dev = 0.0
    for k in range(steps):
        t0 = time.perf_counter()
        rs = P.run_chains(cache, pri, seeds + np.uint64(k * chains), c1)
        best = max(range(len(rs)), key=lambda c: rs.batch.tracker_totals[c, 0])
        _ = rs[best]  # one McmcResult materialised, as a caller reading the best chain
        wall += time.perf_counter() - t0
        dev += rs.batch.device_ms / 1e3
    total = steps * chains * iters
    out = {"python_run_chains": {"e2e_it_s": total / wall, "device_it_s": total / dev,
                                 "e2e_over_device": dev / wall}}
    probe = os.path.join(ROOT, "tools", "cxx", "_build", "e2e_probe")
    if os.path.exists(probe):
        try:
            r = subprocess.run([probe, str(chains), str(iters), str(steps), "1"], capture_output=True,
                               text=True, timeout=600)
            out["cxx_run_chains"] = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception as e:  # reported, not fatal
            out["cxx_run_chains"] = {"error": str(e)[:200]}
    return out


def full_scan_probe(P, _lib, cache, pri, cfg, chains=64, iters=100):
    """The full-row scan path (scan_mode 1, K2 + CUDA Graphs): it/s and the K2
    roofline (32-B key sectors it must stream per launch / avg launch time)."""
    import ctypes as C
    c1 = P.RunConfig(max_parents=cfg.max_parents, iterations=iters, scan_mode=1,
                     memory_cap_bytes=cfg.memory_cap_bytes, device=cfg.device)
    P.run_chains_batch(cache, pri, list(range(1, chains + 1)), c1)  # warm-up
    b = P.run_chains_batch(cache, pri, list(range(1, chains + 1)), c1)
    a, s_, t, d = C.c_uint64(), C.c_uint64(), C.c_float(), C.c_uint64()
    _lib.check(_lib.lib().bnmc_gpu_last_scan_stats(cache.handle, C.byref(a), C.byref(s_),
                                                    C.byref(t), C.byref(d)))
    launches = iters + 1
    bpl = s_.value * 16.0 / launches  # 16-byte key slots streamed by K2
    avg = t.value / 1e3
    peak, src = load_peaks()
    # OrderScorer::score of single orders (all n rows, one pair each) through K2
    # alone, cold L2 before every launch: the north-star "order-score scan" bar
    rng = np.random.default_rng(0)
    one = {}
    for cnt in (1, 8):
        perms = np.stack([rng.permutation(cache.n()) for _ in range(cnt)]).astype(np.int32)
        ms, kb = C.c_float(), C.c_uint64()
        _lib.check(_lib.lib().bnmc_gpu_bench_scan(cache.handle, perms.ravel(), cnt, 0,
                                                  cache.n() - 1, 20, 1, C.byref(ms), C.byref(kb)))
        one[f"orders_{cnt}"] = {"avg_launch_us": ms.value * 1e3, "key_bytes": kb.value,
                                "achieved_GBps": kb.value / (ms.value / 1e3) / 1e9,
                                "frac": kb.value / (ms.value / 1e3) / 1e9 / peak}
    return {"it_s": chains * iters / (b.device_ms / 1e3), "chains": chains, "iterations": iters,
            "kernel": "scan2_kernel (K2, full-row fp32-key scan)",
            "order_scan_cold": dict(one, note="full-order scans (every row rescanned) timed alone with "
                                    "CUDA events after a 256 MiB L2 flush; key_bytes = 16-byte key "
                                    "slots actually loaded (sector skipping) per launch"),
            # measured bound: per-CTA latency chains (one order) and issue (many
            # orders), not HBM (profiles/r02_ncu_scan2_c1.txt, K2)
            "roofline": {"bound": "issue/latency", "achieved": bpl / avg / 1e9, "peak": peak,
                         "unit": "GB/s",
                         "frac": bpl / avg / 1e9 / peak, "bytes_per_launch": bpl,
                         "avg_launch_us": avg * 1e6, "peak_source": src,
                         "row_equivalent_GBps": (a.value / launches) * cache.entries_per_node() * 4.0
                         / avg / 1e9}}


def run_ours(args):
    import ctypes as C
    import torch
    import paper_1210_5128_b200 as P
    from paper_1210_5128_b200 import _lib, dist as D

    rank, world, local = D.env_rank_world()
    torch.cuda.set_device(local)
    # --force-dist exercises the multi-GPU code path (the library's NCCL
    # communicator: split K1 + all-reduce, record all-gather, max over ranks)
    # even at world size 1; torch.distributed (gloo) only ships the NCCL id
    dist_on = world > 1 or args.force_dist
    comm = None
    if dist_on:
        import torch.distributed as tdist
        if "RANK" not in os.environ:  # --force-dist without torchrun: a world of one
            import socket
            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                port = sk.getsockname()[1]
            os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0",
                              MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        tdist.init_process_group("gloo")
        comm = D.Comm(rank, world, local)
    data, pri, cfg, truth = P.baseline_instance(args.config)
    cfg.device = local
    # ---- precompute: K1 split over the ranks + NCCL all-reduce, then the per-row
    # sort and walk lists. Built twice: the first build in a fresh process also
    # pays the driver's first multi-GB allocations (precompute_cold_s); the
    # second is the steady-state figure (precompute_s).
    def precompute():
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        c_ = D.build_table_comm(data, cfg, pri, comm) if dist_on else P.ScoreCache.build(data, cfg, pri)
        cfg.iterations, cfg.scan_mode = 1, 2
        # binds priors, builds the sorted rows (pageable 1-chain result buffer: no
        # page-locked allocation inside the precompute timing)
        P.run_chains_batch(c_, pri, [1], cfg,
                           P.api.ChainBatch.allocate(1, 1, data.n, cfg.track_top, pinned=False))
        torch.cuda.synchronize()
        return c_, time.perf_counter() - t0
    cache, pre_cold_s = precompute()
    cache.close()
    cache, pre_s = precompute()
    k1, fold = C.c_float(), C.c_float()
    _lib.check(_lib.lib().bnmc_gpu_table_build_ms(cache.handle, C.byref(k1), C.byref(fold)))
    Cn, I = args.chains, args.iters
    cfg.iterations, cfg.team_warps = I, args.team_warps
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    # host result buffers (pinned) reused across steps: the e2e region copies into them
    n, K = data.n, cfg.track_top

    def pinned(shape, dt):
        return torch.empty(shape, dtype=dt, pin_memory=True).numpy()
    out = P.api.ChainBatch(pinned((Cn, I), torch.float64), pinned((Cn, I), torch.uint8),
                           pinned((Cn, I), torch.float64), pinned((Cn, n), torch.int32),
                           pinned((Cn,), torch.float64), pinned((Cn,), torch.int64).view(np.uint64),
                           pinned((Cn,), torch.int32), pinned((Cn, K, n), torch.int64).view(np.uint64),
                           pinned((Cn, K), torch.float64), 0.0, 0.0)
    for w in range(args.warmup):
        P.run_chains_batch(cache, pri, D.chain_seeds(1000001, rank, Cn, w, world), cfg, out)
    if dist_on:
        import torch.distributed as tdist
        tdist.barrier()
        comm.max([0.0])  # NCCL rendezvous before the timed region
    torch.cuda.synchronize()
    dev_ms, wall_s, walked, enumerated, pairs, replayed, launches = [], [], 0, 0, 0, 0, 0
    with ClockSampler(local) as clocks:
        for k in range(args.steps):
            flush_l2(torch, flush)
            torch.cuda.synchronize()
            b = P.run_chains_batch(cache, pri, D.chain_seeds(1, rank, Cn, k, world), cfg, out)
            wall_s.append(b.wall_s)
            dev_ms.append(b.device_ms)
            pa, wa, en, so = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_float()
            _lib.check(_lib.lib().bnmc_gpu_last_walk_stats(cache.handle, C.byref(pa), C.byref(wa),
                                                            C.byref(en), C.byref(so)))
            rp, nl = C.c_uint64(), C.c_uint64()
            _lib.check(_lib.lib().bnmc_gpu_last_replayed(cache.handle, C.byref(rp)))
            _lib.check(_lib.lib().bnmc_gpu_last_scan_stats(cache.handle, None, None, None,
                                                            C.byref(nl)))
            launches += nl.value  # kernel launches the library made for this call
            pairs += pa.value
            walked += wa.value
            enumerated += en.value
            replayed += rp.value
    torch.cuda.synchronize()
    tot_dev = sum(dev_ms) / 1e3
    tot_wall = sum(wall_s)
    recs = D.chain_records_from_batch(out, D.chain_seeds(1, rank, Cn, args.steps - 1, world), n)
    k1_ms = k1.value
    if dist_on:  # max over ranks; records all-gathered over the library's NCCL comm
        tot_dev, tot_wall, pre_s, k1_ms = comm.max([tot_dev, tot_wall, pre_s, k1_ms])
        allrec = comm.allgather(recs).reshape(-1, recs.shape[1])
    else:
        allrec = recs
    iters_total = args.steps * Cn * I * world
    value = iters_total / tot_dev
    e2e = iters_total / tot_wall
    # roofline of the fused walk kernel: algorithmic bytes = sorted entries
    # walked (f64 eff + u64 mask) + PST-enumerated local scores (f64 gathers)
    bytes_per_launch = (walked * 16.0 + enumerated * 8.0) / args.steps
    avg_launch_s = tot_dev / args.steps
    achieved = bytes_per_launch / avg_launch_s / 1e9
    peak, peak_src = load_peaks()
    out_line = None
    if rank == 0:
        best = D.best_overall(allrec, n)
        cpu = None
        extra = {}
        rc = None
        if world == 1 and not (args.no_cpu_baseline and args.parity_chains == 0):
            rc = reference_cache(cache, cfg)
        if rc is not None and args.parity_chains > 0:
            extra["headline_parity"] = headline_parity(
                rc, out, D.chain_seeds(1, rank, Cn, args.steps - 1, world), pri, n,
                cfg.max_parents, I, args.parity_chains)
        if rc is not None and not args.no_cpu_baseline:
            c1 = P.RunConfig(max_parents=cfg.max_parents, iterations=args.cpu_iters, seed=1,
                             memory_cap_bytes=cfg.memory_cap_bytes, device=local, scan_mode=2)
            ours1 = P.run_chains(cache, pri, [1], c1)[0]
            cpu = cpu_baseline(rc, n, cfg.max_parents, pri, ours1.trace_proposed, args.cpu_iters, 1)
            rp = reference_precompute(data, cfg.max_parents)
            if cpu is not None and rp is not None:
                cpu["precompute_s"] = rp["precompute_s"]
                cpu["precompute"] = rp
        if world == 1 and not args.no_extras:
            # one chain (the reference's own unit of work): latency-bound, the
            # speculative single-chain kernel runs at >= 1000 iterations
            I1 = 2000
            c1 = P.RunConfig(max_parents=cfg.max_parents, iterations=I1, scan_mode=2, team_warps=0,
                             memory_cap_bytes=cfg.memory_cap_bytes, device=local)
            P.run_chains_batch(cache, pri, [1], c1)  # warm-up
            one = P.run_chains_batch(cache, pri, [1], c1)
            extra["single_chain_it_s"] = I1 / (one.device_ms / 1e3)
            extra["single_chain_iterations"] = I1
            extra["full_scan_path"] = full_scan_probe(P, _lib, cache, pri, cfg)
            extra["e2e_reference_api"] = reference_api_e2e(P, cache, pri, cfg, Cn, I)
        h2d = 8 * Cn
        d2h = (Cn * I * (8 + 1 + 8) + Cn * K * (n * 8 + 8) + Cn * (n * 4 + 8 + 8 + 4) + 4 * Cn)
        out_line = {
            "metric": METRIC, "value": value, "unit": "iterations/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": tot_dev * 1e3 / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generator, seed 7, SURVEY \u00a78d)",
            "config": {"workload": f"{args.config}: n=60 k=4 m=10000 3-state + pairwise priors; "
                                   f"{Cn} independent chains/GPU x {I} iterations per step",
                       "chains_per_gpu": Cn, "iterations_per_step": I,
                       "scan": "sorted-row walk + PST enumeration (scan_mode 2), fused chains",
                       "parallelism": f"independent chains, {world} GPU(s)",
                       "l2": "flushed (256 MiB write) before every step"},
            "e2e": {"value": e2e, "unit": "iterations/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "note": "bnmc_gpu_run_chains with host seeds in, pinned host trace/tracker/"
                            "final-state buffers out; wall time per call"},
            "roofline": walk_roofline(ncu_profile("walk_chain_kernel"), avg_launch_s, peak,
                                      peak_src, bytes_per_launch, args.steps * Cn * I / args.steps),
            "walk": {"pairs_per_iteration": pairs / (args.steps * Cn * (I + 1)),
                     "walked_per_pair": walked / max(1, pairs),
                     "enumerated_per_pair": enumerated / max(1, pairs),
                     "chains_replayed_exact": replayed},
            "precompute_s": pre_s, "precompute_cold_s": pre_cold_s, "precompute_kernel_ms": k1_ms,
            "fold_ms": fold.value,
            "gpu_launches": int(launches),
            "best_total": best["best_total"], "best_chain_seed": best["seed"],
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
        }
        out_line.update(extra)
        print(json.dumps(out_line), flush=True)
    if dist_on:
        import torch.distributed as tdist
        tdist.barrier()
        comm.close()
        tdist.destroy_process_group()
    return out_line


def run_reference(args):
    """The reference's own CPU implementation (oracle/_ref) on the same config."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    from oracle import ref
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libbnmc_ref.so missing (built from /root/reference)"}))
        return None
    import paper_1210_5128_b200.api as A  # config table only (no GPU call)
    c = A.BASELINE_CONFIGS[args.config]
    n, k, m = c["n"], c["k"], c["m"]
    cards = np.array([3] * n if c["cards"] == "3" else [2 + (i % 3) for i in range(n)], np.int32)
    cells, truth = ref.generate(n, k, m, cards, seed=7)
    pri = ref.synth_priors(n, truth, seed=7) if c["priors"] else None
    m_build = min(m, args.ref_rows)
    t0 = time.perf_counter()
    cache = ref.Cache.build(cells[:m_build], cards, k)
    build_s = time.perf_counter() - t0
    for _ in range(args.warmup):
        ref.run_mcmc(cells, cards, k, 2, 99, priors=pri, prebuilt=cache)
    I = args.ref_iters
    samp = 0.0
    for step in range(args.steps):
        r = ref.run_mcmc(cells, cards, k, I, 1 + step, priors=pri, prebuilt=cache)
        samp += r.sampling_seconds
    value = args.steps * I / samp

    rp = reference_precompute(_HostData(cells, cards), k)
    sample = (f"{args.steps} x {I} run_mcmc iterations (OrderScorer::score, OpenMP "
              f"{ref.max_threads()} threads) on a cache built by ScoreCache::build from the first "
              f"{m_build} of {m} rows ({build_s:.1f}s; the order scan is independent of m)")
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "iterations/s",
           "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": samp * 1e3 / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (reference generator, seed 7)",
           "config": {"workload": f"{args.config}: n=60 k=4 m=10000 3-state + pairwise priors; "
                                  f"1 chain x {I} iterations per step"},
           "cpu_baseline": {"value": value, "unit": "iterations/s", "cores": ref.max_threads(),
                            "cpu_model": cpu_model(),
                            "kind": "reference", "sample": sample,
                            "precompute_s": rp["precompute_s"] if rp else None,
                            "precompute": rp},
           "e2e": {"value": value, "unit": "iterations/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--chains", type=int, default=18944, help="chains per GPU (128 per SM)")
    ap.add_argument("--team-warps", type=int, default=0, help="warps per chain (0 auto)")
    ap.add_argument("--no-extras", action="store_true", help="skip single-chain/full-scan probes")
    ap.add_argument("--force-dist", action="store_true",
                    help="run the multi-GPU code path (NCCL) even at world size 1")
    ap.add_argument("--iters", type=int, default=500, help="MCMC iterations per chain per step")
    ap.add_argument("--cpu-iters", type=int, default=200)
    ap.add_argument("--parity-chains", type=int, default=16,
                    help="chains of the last timed launch checked against oracle/_ref (0 off)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-iters", type=int, default=30)
    ap.add_argument("--ref-rows", type=int, default=1000)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
