"""Extract one fwd+bwd step (preprocess_fwd .. preprocess_bwd) from an ncu launch list CSV
(gpu__time_duration.sum) and print the per-launch table with shares."""
import csv
import sys


def main(path, which=3, label="c3"):
    rows = []
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((r["Kernel Name"], float(r["Metric Value"]) / 1e3))
    starts = [i for i, (k, _) in enumerate(rows) if "preprocess_fwd" in k]
    i0 = starts[which]
    i1 = next(i for i in range(i0, len(rows)) if "preprocess_bwd" in rows[i][0])
    step = rows[i0:i1 + 1]
    tot = sum(t for _, t in step)
    print(f"# ncu launch list, one {label} fwd+bwd step (bench.py --steps 2 --warmup 3), B200")
    print("# gpu__time_duration.sum per launch, --clock-control none; ncu serialises launches and")
    print("# runs them cold-cache, so compare SHARES with bench.py's event times, not absolutes.")
    print(f"{'kernel':75s} {'us':>8s} {'share':>7s}")
    for k, t in step:
        print(f"{k[:75]:75s} {t:8.1f} {100 * t / tot:6.1f}%")
    print(f"{'total':75s} {tot:8.1f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 3,
         sys.argv[3] if len(sys.argv) > 3 else "c3")
