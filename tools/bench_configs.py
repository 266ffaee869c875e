"""Run bench.py on every BASELINE config (C1..C5) on one GPU and write a table
(profiles/<tag>_configs.md).  C1-C3 are latency-bound per-call workloads; the
bench line the driver records is C5."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(tag, configs=("C1", "C2", "C3", "C4", "C5")):
    rows = []
    for c in configs:
        steps = {"C1": 50, "C2": 50, "C3": 20, "C4": 10, "C5": 5}[c]
        p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", c, "--steps",
                            str(steps), "--warmup", "3", "--cpu-seconds", "8"],
                           capture_output=True, text=True)
        try:
            d = json.loads(p.stdout.strip().splitlines()[-1])
        except Exception:
            print(c, "FAILED", p.stderr[-800:], flush=True)
            continue
        st = d["stages"]
        rows.append((c, d, st))
        print(c, json.dumps({k: d[k] for k in ("value", "ms_per_step")}), flush=True)
    lines = [f"# {tag}: bench.py on every config (one B200)", "",
             "step = build target maps + overlap of candidate pairs + linearize (C4/C5: overlap-selected factors;",
             "C1-C3: the config's factor list, validation on for C1-C3).  points/s = source points linearized per second.", "",
             "| config | factors/step | ms/step | points/s | factors/s | build ms | overlap ms | linearize ms | e2e points/s | e2e ms | CPU oracle points/s (cores) |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    for c, d, st in rows:
        e = d.get("e2e") or {}
        cpu = d.get("cpu_baseline") or {}
        lines.append(f"| {c} | {d['config']['factors_per_step']:.0f} | {d['ms_per_step']:.3f} | {d['value']:.3e} | "
                     f"{d['factors_per_s']:.3e} | {st['build']['ms_per_step']:.3f} | {st['overlap']['ms_per_step']:.3f} | "
                     f"{st['linearize']['ms_per_step']:.3f} | {e.get('value', 0):.3e} | {e.get('ms_per_step', 0):.3f} | "
                     f"{cpu.get('value', 0):.3e} ({cpu.get('cores', '-')}) |")
    out = os.path.join(ROOT, "gpurun_out", f"{tag}_configs.md")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    open(out, "w").write("\n".join(lines) + "\n")
    json.dump([d for _, d, _ in rows], open(out.replace(".md", ".json"), "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "run", tuple(sys.argv[2].split(",")) if len(sys.argv) > 2 else
         ("C1", "C2", "C3", "C4", "C5"))
