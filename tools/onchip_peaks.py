"""Build and run tools/onchip_peaks.cu on the GPU box; write the JSON it prints (plus the
nvidia-smi clocks seen during the run) to the given path (default
profiles/r02/onchip_peaks.json, which bench.py reads as the measured on-chip peaks)."""
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tools", "onchip_peaks.cu")
BIN = os.path.join(ROOT, "tools", "bin", "onchip_peaks")


def build():
    if not os.path.exists(BIN) or os.path.getmtime(BIN) < os.path.getmtime(SRC):
        os.makedirs(os.path.dirname(BIN), exist_ok=True)
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-lineinfo", "-o", BIN, SRC])
    return BIN


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r02", "onchip_peaks.json")
    build()
    rows = []
    smi = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                            "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
    t = threading.Thread(target=lambda: rows.extend(smi.stdout), daemon=True)
    t.start()
    time.sleep(0.3)
    res = json.loads(subprocess.check_output([BIN], text=True))
    smi.terminate()
    t.join(timeout=2)
    sm = sorted(float(r.split(",")[0]) for r in rows if r.split(",")[0].strip().replace(".", "").isdigit())
    res["nvidia_smi_sm_mhz_median"] = sm[len(sm) // 2] if sm else None
    res["nvidia_smi_samples"] = len(sm)
    res["when"] = time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())
    res["how"] = ("tools/onchip_peaks.cu: one 1024-thread CTA per SM; rates per SM cycle from %clock64, per second "
                  "from CUDA events; int ops = IADD3 (ALU pipe) or IADD3+IMAD (ALU+FMA pipes); lds_seq = "
                  "conflict-free LDS.32 wavefronts (128 B); lds_gather_u16 = random uint16 gathers in 64 KB")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
