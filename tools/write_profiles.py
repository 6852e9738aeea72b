"""Copy a tools/profile_round.sh capture (gpurun_out/TAG) into profiles/ and
write profiles/<round>_summary.md + profiles/raycast_traffic.json from it.

  python tools/write_profiles.py TAG [ROUND]      (ROUND default r2)
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def ncu_raw(rep):
    return subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                   stderr=subprocess.DEVNULL).decode()


def _val(rows, kernel_sub, name):
    hdr, units = rows[0], rows[1]
    if name not in hdr:
        return None
    ik, im = hdr.index("Kernel Name"), hdr.index(name)
    for r in rows[2:]:
        if kernel_sub in r[ik]:
            return float(r[im].replace(",", "")) * UNITS.get(units[im], 1)
    return None


def run(cmd):
    return subprocess.check_output(cmd, cwd=ROOT).decode()


def main(tag, rnd="r2"):
    src = os.path.join(ROOT, "gpurun_out", tag)
    for f in ("launches.csv", "bench_configs.jsonl", "slab_modes.jsonl"):
        if os.path.exists(os.path.join(src, f)):
            shutil.copy(os.path.join(src, f), os.path.join(PROF, f"{rnd}_{f}"))
    scal = None
    if os.path.exists(os.path.join(src, "slab_scaling.json")):
        txt = [x for x in open(os.path.join(src, "slab_scaling.json")) if x.startswith("{")]
        if txt:
            scal = json.loads(txt[-1])
            json.dump(scal, open(os.path.join(PROF, f"{rnd}_slab_scaling_emulated.json"), "w"))
    line = [x for x in open(os.path.join(src, "bench_c2.json")).read().strip().splitlines()
            if x.startswith("{")][-1]
    open(os.path.join(PROF, f"{rnd}_bench_c2.json"), "w").write(line + "\n")
    raw2 = ncu_raw(os.path.join(src, "full_c2.ncu-rep"))
    raw5 = ncu_raw(os.path.join(src, "full_c5_raycast.ncu-rep"))
    open(os.path.join(PROF, f"{rnd}_ncu_full_raw.csv"), "w").write(raw2)
    open(os.path.join(PROF, f"{rnd}_ncu_c5_raycast_raw.csv"), "w").write(raw5)
    r2 = list(csv.reader(io.StringIO(raw2)))
    r5 = list(csv.reader(io.StringIO(raw5)))

    def traffic(rows):
        a = _val(rows, "k_raycast", "dram__bytes_read.sum")
        b = _val(rows, "k_raycast", "dram__bytes_write.sum")
        return None if a is None or b is None else a + b

    c2, c5 = "c2_os1_64_rolling_trees", "c5_8x_os1_128_large_map"
    tj = {"kernel": "k_raycast",
          "metric": "dram__bytes_read.sum + dram__bytes_write.sum per launch "
                    "(one ncu --set full capture, cold caches)",
          "source": {c2: f"profiles/{rnd}_ncu_full_raw.csv",
                     c5: f"profiles/{rnd}_ncu_c5_raycast_raw.csv"},
          "bytes_per_launch": {c2: traffic(r2), c5: traffic(r5)},
          "warp_inst_per_launch": {c2: _val(r2, "k_raycast", "smsp__inst_executed.sum"),
                                   c5: _val(r5, "k_raycast", "smsp__inst_executed.sum")},
          "red_requests_per_launch": {
              c2: _val(r2, "k_raycast", "lts__t_requests_srcunit_tex_op_red.sum"),
              c5: _val(r5, "k_raycast", "lts__t_requests_srcunit_tex_op_red.sum")}}
    json.dump(tj, open(os.path.join(PROF, "raycast_traffic.json"), "w"), indent=1)

    launches = run([sys.executable, "tools/launch_summary.py", f"profiles/{rnd}_launches.csv"])
    full2 = run([sys.executable, "tools/ncu_summary.py", os.path.join(src, "full_c2.ncu-rep")])
    full5 = run([sys.executable, "tools/ncu_summary.py",
                 os.path.join(src, "full_c5_raycast.ncu-rep")])
    bc = [json.loads(x) for x in open(os.path.join(PROF, f"{rnd}_bench_configs.jsonl"))
          if x.startswith("{")]
    d2 = json.loads(line)
    rows = []
    for d in bc:
        r = d["roofline"]
        pipe = d["pipelined"]["map_updates_per_s"] if d.get("pipelined") else float("nan")
        rows.append(f"| {d['config']['workload']} | {d['ms_per_step'] * 1e3:.1f} | "
                    f"{d['map_updates_per_s']:.0f} | {d['value'] / 1e6:.0f} | "
                    f"{r['launch_ms'] * 1e3:.1f} | {r['frac']:.3f} | "
                    f"{d['integrate']['ms_per_frame'] * 1e3:.1f} | "
                    f"{d['integrate']['hbm_frac']:.3f} | {d['compute_maps_ms'] * 1e3:.1f} | "
                    f"{d['e2e']['value'] / 1e6:.0f} | "
                    f"{d['e2e'].get('synchronous_value', d['e2e']['value']) / 1e6:.0f} | "
                    f"{pipe:.0f} |")
    srows = []
    if os.path.exists(os.path.join(PROF, f"{rnd}_slab_modes.jsonl")):
        for x in open(os.path.join(PROF, f"{rnd}_slab_modes.jsonl")):
            if not x.startswith("{"):
                continue
            d = json.loads(x)
            srows.append(f"| {d['config']['parallelism']} | {d['n_gpus']} | "
                         f"{d['ms_per_step'] * 1e3:.0f} | {d['value'] / 1e6:.0f} |")
    ray2 = d2["roofline"]
    l2 = ray2.get("l2_red") or {}
    l2txt = "; ".join(
        f"{k}: random {v['random_word']['g_l2_requests_s']:.0f}, runs of 4 "
        f"{v['runs_of_4']['g_l2_requests_s']:.0f} G req/s" for k, v in l2.items()
        if v.get("random_word") and v.get("runs_of_4"))
    rr = ray2.get("raycast_red") or {}
    scal_md = ""
    if scal:
        lines_ = []
        for P in sorted(scal["segments"], key=int):
            a, b, c = scal["segments"][P], scal["segments_balanced"][P], scal["reduce_scatter"][P]
            lines_.append(f"| {P} | {a['max_ms']:.2f} / {a['mean_ms']:.2f} | "
                          f"{b['max_ms']:.2f} / {b['mean_ms']:.2f} | {c['max_ms']:.2f} | "
                          f"{scal['segments_balanced']['1']['max_ms'] / b['max_ms']:.2f} |")
        scal_md = f"""
## P ranks emulated on one GPU (c5; `{rnd}_slab_scaling_emulated.json`, tools/slab_scaling.py)

Each rank's calls timed alone; max / mean over ranks, collectives not included.

| P | ray segments, equal rows: max / mean ms | ray segments, balanced: max / mean ms | reduce-scatter compute: max ms | speed-up of balanced max vs P = 1 |
|---|---|---|---|---|
{chr(10).join(lines_)}
"""
    md = f"""# Round 2 profile summary (B200, sm_100a)

Regenerated by `tools/profile_round.sh {tag}` (under gpurun, 1 GPU; every ncu command ran
only after the same command exited 0 without ncu) and `tools/write_profiles.py {tag} {rnd}`.
Files: `{rnd}_launches.csv` (launch list of the default command), `{rnd}_ncu_full_raw.csv`
(full set, the kernels of one c2 step), `{rnd}_ncu_c5_raycast_raw.csv` (full set, k_raycast at
c5), `{rnd}_bench_c2.json` (the default bench line), `{rnd}_bench_configs.jsonl` (all five
configs), `{rnd}_slab_modes.jsonl` (the partitioned path's modes on one rank, c5),
`raycast_traffic.json` (DRAM bytes, warp instructions and L2 reduction requests per k_raycast
launch that bench.py reports).

## Bench (device-resident inputs, L2 flushed between steps, one CUDA graph per step)

| workload | step µs | map updates/s | Mpoints/s | k_raycast µs | ray HBM-eq frac | integrate µs | integrate HBM-eq frac | compute_maps µs | e2e Mpoints/s (pipelined) | e2e Mpoints/s (synchronous) | pipelined updates/s |
|---|---|---|---|---|---|---|---|---|---|---|---|
{chr(10).join(rows)}

Default line (c2, {d2['steps']} steps): {d2['ms_per_step'] * 1e3:.1f} µs/step,
{d2['map_updates_per_s']:.0f} map updates/s, {d2['value'] / 1e6:.0f} M points/s; `gpu_launches`
{d2['gpu_launches']}; k_raycast {ray2['launch_ms'] * 1e3:.1f} µs = {ray2['frac']:.3f} of the measured
HBM {ray2['peak']} GB/s; cpu_baseline (the C oracle, one pinned core)
{d2['cpu_baseline']['value'] / 1e3:.0f} k points/s; clocks {d2['clocks']}.

L2 reduction ceiling (`roofline.l2_red`, csrc/probe/l2_red_probe.cu): {l2txt}.
The ray cast: {rr.get('g_l2_requests_s') or float('nan'):.0f} G L2 reduction requests/s,
{rr.get('g_increments_s') or float('nan'):.0f} G miss increments/s.

## Partitioned path on one rank (c5; `{rnd}_slab_modes.jsonl`)

| mode | ranks | µs/frame | Mpoints/s |
|---|---|---|---|
{chr(10).join(srows)}
{scal_md}
## Launch list (`{rnd}_launches.csv`, c2, cold caches, serialised)

```
{launches.strip()}
```

## Full-set metrics per kernel (c2, `{rnd}_ncu_full_raw.csv`)

```
{full2.strip()}
```

## k_raycast at c5 (`{rnd}_ncu_c5_raycast_raw.csv`)

```
{full5.strip()}
```
"""
    open(os.path.join(PROF, f"{rnd}_summary.md"), "w").write(md)
    print("profiles/ written from", src)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "r2")
