"""C1 on the CPU reference (SURVEY.md §8(d) "How the CPU reference is timed"):
the stock svcodec (baseline/_ref) full encode + decode_full + query of the
AC4 sphere 128^3 with ACCEPT_CONFIG at 16-bit precision, on this box's host
cores, with OPENBLAS_NUM_THREADS = nproc and = 1, workers = 1, wall time by
time.perf_counter; lscpu model recorded.  Prints one JSON line per thread
setting (the child process) and a summary.

    python tools/c1_cpu_reference.py [--threads N] [--timeout S]
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child():
    for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "svcodec")):
            sys.path.insert(0, p)
            break
    import numpy as np
    from svcodec import metrics
    from svcodec.config import TrainConfig
    from svcodec.decoder import decode_full, make_hybrid
    from svcodec.encoder import encode
    from svcodec.procgen import SphereSpec, gen_sphere_sdf
    cfg = TrainConfig(subdomain_size=512, l1_net=(3, 48), tile_net=None, l0_net=(3, 96), voxel_net=(3, 96),
                      activation="sine", frequency=3.0, ffm_scale=5.0, ffm_size=192, lr=1e-3, decay=0.975,
                      interval=100.0, max_epochs=800, sample_interval=1, batch_size=65536,
                      significance_threshold=0.0, strict_topology=False, seed=4242)
    out = {"openblas_threads": os.environ.get("OPENBLAS_NUM_THREADS"), "cores": os.cpu_count()}
    t0 = time.perf_counter()
    g = gen_sphere_sdf(SphereSpec(center=(63.5, 63.5, 63.5), radius=61.0, voxel_size=1.0, half_width=3.0))
    out["generate_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    c = encode(g, cfg, weight_precision=16, workers=1)
    out["encode_s"] = time.perf_counter() - t0
    out["epochs"] = {t: n.epochs for t, n in c.experts[0].nets() if n is not None}
    t0 = time.perf_counter()
    d = decode_full(c)
    out["decode_full_s"] = time.perf_counter() - t0
    out["leaf_voxels"] = sum(1 for _ in d.iter_leaves()) * 512
    h = make_hybrid(c)
    q = np.random.default_rng(0).integers(0, 128, (1_000_000, 3))
    t0 = time.perf_counter()
    h.query(q)
    out["query_1e6_s"] = time.perf_counter() - t0
    out["regressor_evaluations"] = h.regressor_evaluations
    out["iou"] = metrics.iou(g, d)
    out["mcd_dx"] = metrics.mcd(g, d) / g.voxel_size
    print(json.dumps(out), flush=True)


def main():
    if "--child" in sys.argv:
        child()
        return
    timeout = 3600
    if "--timeout" in sys.argv:
        timeout = int(sys.argv[sys.argv.index("--timeout") + 1])
    threads = [os.cpu_count(), 1]
    if "--threads" in sys.argv:
        threads = [int(sys.argv[sys.argv.index("--threads") + 1])]
    try:
        model = [ln.split(":", 1)[1].strip() for ln in subprocess.run(["lscpu"], capture_output=True, text=True)
                 .stdout.splitlines() if ln.startswith("Model name")][0]
    except Exception:  # noqa: BLE001
        model = None
    runs = []
    for nt in threads:
        env = dict(os.environ, OPENBLAS_NUM_THREADS=str(nt), OMP_NUM_THREADS=str(nt), MKL_NUM_THREADS=str(nt))
        try:
            r = subprocess.run([sys.executable, os.path.abspath(__file__), "--child"], env=env, capture_output=True,
                               text=True, timeout=timeout)
            line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
            runs.append(json.loads(line[-1]) if line else {"threads": nt, "error": r.stderr[-400:]})
        except subprocess.TimeoutExpired:
            runs.append({"openblas_threads": str(nt), "error": f"timeout after {timeout} s"})
        print(json.dumps(runs[-1]), flush=True)
    print(json.dumps({"workload": "C1 sphere 128^3, ACCEPT_CONFIG, weight_precision 16, stock svcodec",
                      "cpu_model": model, "runs": runs}), flush=True)


if __name__ == "__main__":
    main()
