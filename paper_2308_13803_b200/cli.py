"""Command line front end with the reference CLI's subcommands and outputs
(reference tools/dnnscaler_main.cpp): run, compare, sensitivity, sweep,
profile. Scenarios and catalogs are the reference's JSON formats; reports
are byte-identical to the reference writers for the same job results
(report.py). ``--seam device`` serves the jobs on the B200 (the job's dnn_id
names the network: mobilenet_v1, resnet50_v1, inception_v3, synthetic_cnn);
``--seam analytic`` runs the reference's simulated GPU from the catalog.

    python -m paper_2308_13803_b200.cli run --config scenario.json --out out/ [--seam device]
"""
from __future__ import annotations

import argparse
import os
import sys

from . import control as C
from . import report as R


def _scenario(args):
    sc, jobs, cat = R.load_scenario(args.config)
    if args.seed is not None:
        sc.seed = args.seed
    if args.sigma is not None and args.sigma >= 0.0:
        sc.sigma = args.sigma
    if getattr(args, "controller", None):
        if args.controller not in C.CONTROLLERS:
            raise ValueError("unknown controller: " + args.controller)
        sc.controller = args.controller
        if sc.controller == "static" and sc.static_knob[1] < 1:
            raise ValueError("static controller needs static_knob in the scenario file")
    return sc, jobs, C.load_catalog(cat)


def _run(sc, jobs, catalog, args):
    return [C.run_job(sc, j, catalog, args.seam, device=args.device) for j in jobs]


def _write(out_dir, name, text):
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, name), "w", newline="") as f:
        f.write(text)


def cmd_run(args) -> int:
    sc, jobs, catalog = _scenario(args)
    res = _run(sc, jobs, catalog, args)
    _write(args.out, "metrics.csv", R.render_metrics_csv(res))
    _write(args.out, "summary.json", R.render_summary_json(sc, jobs, res))
    sys.stdout.write(R.summary_table(jobs, res))
    return 1 if any(r.error for r in res) else 0


def cmd_sensitivity(args) -> int:
    sc, jobs, catalog = _scenario(args)
    if not any(j.slo_schedule for j in jobs):
        raise ValueError("sensitivity needs at least one job with an slo_schedule")
    res = _run(sc, jobs, catalog, args)
    _write(args.out, "metrics.csv", R.render_metrics_csv(res))
    _write(args.out, "summary.json", R.render_summary_json(sc, jobs, res))
    sys.stdout.write(R.summary_table(jobs, res))
    for j, r in zip(jobs, res):
        for at_s, periods in r.readaptations:
            if periods < 0:
                print("job %d: slo step at %.1fs, band not re-entered" % (j.job_id, at_s))
            else:
                print("job %d: slo step at %.1fs, back in band after %d periods" % (j.job_id, at_s, periods))
    return 1 if any(r.error for r in res) else 0


def cmd_compare(args) -> int:
    sc, jobs, catalog = _scenario(args)
    import copy
    a, b = copy.copy(sc), copy.copy(sc)
    a.controller, b.controller = "dnnscaler", "clipper"
    ra, rb = _run(a, jobs, catalog, args), _run(b, jobs, catalog, args)
    _write(args.out, "metrics_dnnscaler.csv", R.render_metrics_csv(ra))
    _write(args.out, "metrics_clipper.csv", R.render_metrics_csv(rb))
    _write(args.out, "summary_dnnscaler.json", R.render_summary_json(a, jobs, ra))
    _write(args.out, "summary_clipper.json", R.render_summary_json(b, jobs, rb))
    comp = R.render_comparison_csv(jobs, ra, rb)
    _write(args.out, "comparison.csv", comp)
    print("%5s  %-26s %-13s %14s  %14s  %12s" % ("job", "dnn", "approach", "dnnscaler", "clipper",
                                                 "improvement"))
    rows = [line.split(",") for line in comp.splitlines()[1:]]
    for r in rows:
        print("%5d  %-26s %-13s %14.2f  %14.2f  %11.2f%%" % (int(r[0]), r[1], r[2], float(r[3]),
                                                            float(r[4]), float(r[5])))
    if rows:
        print("average improvement: %.2f%%" % (sum(float(r[5]) for r in rows) / len(rows)))
    return 0


def cmd_sweep(args) -> int:
    """== cmd_sweep (reference dnnscaler_main.cpp:186-199): the B x MT grid,
    on the catalog's analytic model (the reference's combination_sweep) or
    measured on the B200 (GpuBackend.combination_sweep, --seam device)."""
    bs = [int(x) for x in args.bs.split(",")]
    mtl = [int(x) for x in args.mtl.split(",")]
    seed = args.seed if args.seed is not None else 42
    if args.seam == "analytic":
        from .serving import B200_CATALOG
        catalog = C.load_catalog(args.catalog or B200_CATALOG)
        cells = C.combination_sweep(catalog, args.dnn, bs, mtl, args.samples, seed,
                                    args.sigma if args.sigma is not None else -1.0)
    else:
        from .backend import Config, GpuBackend
        with GpuBackend(args.dnn, Config(max(bs), max(max(mtl), 2)), seed=seed,
                        device=args.device) as be:
            cells = be.combination_sweep(bs, mtl, args.samples)
    text = R.render_sweep_csv(cells)
    _write(args.out, "sweep.csv", text)
    sys.stdout.write(text)
    return 0


def cmd_profile(args) -> int:
    """== cmd_profile (reference dnnscaler_main.cpp:88-111): the Profiler's
    probe and decision for one network, on the B200 or the analytic seam."""
    from .serving import B200_CATALOG
    catalog = C.load_catalog(args.catalog or B200_CATALOG)
    rep = C.profile_dnn(catalog, args.dnn, args.m, args.n, args.batches,
                        args.seed if args.seed is not None else 42,
                        args.sigma if args.sigma is not None else -1.0, args.seam, device=args.device)
    approach = R._KNOB[C.decide(rep["ti_batching"], rep["ti_mt"], rep["probe_latency_batching_ms"],
                                rep["probe_latency_mt_ms"])]
    print("dnn: %s" % args.dnn)
    print("  base throughput   %10.2f items/s" % rep["tput_base"])
    print("  batching (bs=%d)  %10.2f items/s  gain %8.2f%%" % (rep["m"], rep["tput_batching"], rep["ti_batching"]))
    print("  multi-tenancy (%d) %10.2f items/s  gain %8.2f%%" % (rep["n"], rep["tput_mt"], rep["ti_mt"]))
    print("  profiling cost    %10.2f ms" % rep["profiling_cost_ms"])
    print("  approach: %s" % approach)
    sys.stdout.write(R.render_profile_json(rep, args.dnn, approach))
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="dnnscaler-b200")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def scen(p, controller=True):
        p.add_argument("--config", required=True, help="scenario JSON (reference format)")
        p.add_argument("--out", default=".", help="output directory")
        p.add_argument("--seed", type=int, default=None)
        p.add_argument("--sigma", type=float, default=None)
        if controller:
            p.add_argument("--controller", default=None, help="dnnscaler, clipper or static")
        p.add_argument("--seam", default="analytic", choices=["analytic", "device"])
        p.add_argument("--device", type=int, default=0)

    scen(sub.add_parser("run", help="run a scenario, write metrics.csv + summary.json"))
    scen(sub.add_parser("compare", help="DNNScaler and Clipper side by side"), controller=False)
    scen(sub.add_parser("sensitivity", help="jobs that step their SLO mid-run"))
    sw = sub.add_parser("sweep", help="batch size x instance count grid")
    sw.add_argument("--catalog", default="", help="catalog JSON (default: the B200 catalog)")
    sw.add_argument("--dnn", required=True)
    sw.add_argument("--bs", required=True)
    sw.add_argument("--mtl", required=True)
    sw.add_argument("--out", default=".")
    sw.add_argument("--samples", type=int, default=100)
    sw.add_argument("--seed", type=int, default=None)
    sw.add_argument("--sigma", type=float, default=None, help="latency noise scale (analytic)")
    sw.add_argument("--seam", default="analytic", choices=["analytic", "device"])
    sw.add_argument("--device", type=int, default=0)
    pr = sub.add_parser("profile", help="probe one network and print the decision")
    pr.add_argument("--dnn", required=True)
    pr.add_argument("--catalog", default="", help="catalog JSON (default: the B200 catalog)")
    pr.add_argument("--m", type=int, default=32)
    pr.add_argument("--n", type=int, default=8)
    pr.add_argument("--batches", type=int, default=10, help="batches per probe point")
    pr.add_argument("--sigma", type=float, default=None, help="latency noise scale override")
    pr.add_argument("--seed", type=int, default=None)
    pr.add_argument("--seam", default="analytic", choices=["analytic", "device"])
    pr.add_argument("--device", type=int, default=0)
    args = ap.parse_args(argv)
    try:
        return {"run": cmd_run, "compare": cmd_compare, "sensitivity": cmd_sensitivity,
                "sweep": cmd_sweep, "profile": cmd_profile}[args.cmd](args)
    except ValueError as e:
        print("error: %s" % e, file=sys.stderr)
        return 2
    except Exception as e:  # noqa: BLE001 - the reference CLI's catch-all
        print("error: %s" % e, file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
