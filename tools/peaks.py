"""FP64 roofline denominators measured on the B200.

Runs tools/ubench/peaks (DADD / DFMA issue rate, L2 and HBM read bandwidth, shared-memory and
TMEM rates) and cuBLAS DGEMM 8192^3 (the DMMA path; tcgen05 has no f64 kind on sm_100a) through
torch, while sampling SM clocks with nvidia-smi, and writes one JSON file.

    python tools/peaks.py gpurun_out/peaks_fp64.json
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(out_path):
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
                            "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    exe = os.path.join(ROOT, "tools", "ubench", "peaks")
    if not os.path.exists(exe):
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", exe, exe + ".cu"], check=True)
    res = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    rows = [json.loads(l) for l in res.stdout.splitlines() if l.startswith("{")]
    import torch
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        c = a @ b
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        c = a @ b
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    rows.append({"what": "dgemm_cublas", "n": n, "tflops": 2 * n ** 3 / (best * 1e-3) / 1e12, "ms": best,
                 "note": "torch.matmul float64 (cuBLAS DGEMM, DMMA), best of 5"})
    smi.terminate()
    lines = [l.split(", ") for l in smi.stdout.read().splitlines() if l.strip()]
    mhz = sorted(float(l[0]) for l in lines if l[0].replace(".", "").isdigit())
    res_obj = {"measurements": rows, "stderr": res.stderr[-2000:],
               "clocks": {"samples": len(mhz), "sm_mhz_median": mhz[len(mhz) // 2] if mhz else None,
                          "sm_mhz_min": mhz[0] if mhz else None, "sm_mhz_max": mhz[-1] if mhz else None,
                          "reasons": sorted({l[3] for l in lines if len(l) > 3})},
               "gpu": torch.cuda.get_device_name(0), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    json.dump(res_obj, open(out_path, "w"), indent=1)
    print(json.dumps(res_obj, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "peaks_fp64.json")
