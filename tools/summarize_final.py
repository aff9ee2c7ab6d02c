"""Summarise a closing-evidence directory written by tools/_final_r2c.sh into SUMMARY.md.

    python tools/summarize_final.py profiles/r02_final3 "note about the box"
"""
import json
import sys

P = sys.argv[1].rstrip("/") + "/"
note = sys.argv[2] if len(sys.argv) > 2 else ""


def line(name, d):
    r = d.get("roofline", {})
    c = d.get("clocks", {})
    par = d.get("parity")
    fs = r.get("frac_of_sustained")
    return (f"| {name} | {d['value']:.1f} | {d['ms_per_step'] * 1e3:.1f} | {r.get('frac', float('nan')):.3f} | "
            f"{fs if fs is None else round(fs, 3)} | {c.get('sm_mhz')} | {','.join(c.get('reasons', [])) or '-'} | "
            f"{par and par['pass']} |")


out = [f"# Closing evidence of round 2 (`tools/_final_r2c.sh`, one gpurun box)", "", note, "",
       "Measured peaks (MEASURED_PEAKS.json): bf16 1646.1 TFLOP/s burst, 1396.8 sustained; HBM 6549.8 GB/s.", "",
       "| workload | TFLOP/s | us/step | K1 frac (burst) | K1 frac (sustained) | SM MHz | throttle | parity |",
       "|---|---|---|---|---|---|---|---|"]
for i, ln in enumerate(open(P + "bench_cfg2_runs.jsonl")):
    out.append(line(f"cfg2 run {i + 1}", json.loads(ln)))
for n in ("cfg3", "cfg4", "cfg5"):
    out.append(line(n, json.load(open(P + f"bench_{n}.json"))))
out.append(line("cfg2 + dropout 0.05 (mask kept)", json.load(open(P + "bench_cfg2_dropout.json"))))
out.append(line("cfg2 + dropout 0.05 (redrawn)", json.load(open(P + "bench_cfg2_dropout_redraw.json"))))
out.append(line("cfg3 + dropout 0.05 (mask kept)", json.load(open(P + "bench_cfg3_dropout.json"))))
L = json.load(open(P + "bench_layer7b.json"))
out += ["", f"Decoder layer (N4, `--layer layer7b`): {L['value']:.1f} TFLOP/s, {L['ms_per_step']:.3f} ms/step, "
            f"{L['tokens_per_s'] / 1e6:.2f} M tokens/s, clocks {L['clocks']}.", ""]
R = json.load(open(P + "bench_reference.json"))
out += [f"Reference arm (fp64 CPU oracle, {R['cpu_baseline']['cores']} cores): {R['value']:.4f} TFLOP/s — "
        f"{R['cpu_baseline']['sample']}.", ""]
d = json.loads(open(P + "bench_cfg2_runs.jsonl").readline())
out += ["cfg2 run 1 details:", "", "```", json.dumps(d["kernels_in_step"], indent=1)[:2500],
        json.dumps(d["hbm_bound_kernels"], indent=1)[:2500], "e2e: " + json.dumps(d["e2e"]),
        "cpu_baseline: " + json.dumps(d["cpu_baseline"]), "parity: " + json.dumps(d["parity"]),
        "gpu_launches: " + str(d["gpu_launches"]), "```", ""]
k = json.load(open(P + "ncu_full_k1k2_cfg2.json"))
out += ["ncu --set full, cfg2 grouped q+v (cold L2, serialised; `ncu_full_k1k2_cfg2.json`):", "",
        "| kernel | us | DRAM bytes | tensor pipe % elapsed | % active | regs | SM clock |", "|---|---|---|---|---|---|---|"]
for x in k:
    out.append(f"| {x['kernel'][:48]} | {x['gpu__time_duration.sum']} | {x['dram_bytes_total'] / 1e6:.1f} MB | "
               f"{x['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed']} | "
               f"{x['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active']} | "
               f"{x['launch__registers_per_thread']} | {x.get('sm__cycles_elapsed.avg.per_second')} |")
k = json.load(open(P + "ncu_full_k0_merge_cfg2.json"))
out += ["", "Dropout forward K0 (`ncu_full_k0_merge_cfg2.json`): " +
        "; ".join(f"{x['gpu__time_duration.sum']}, {x['launch__registers_per_thread']}" for x in k), ""]
for f, t in (("launches_cfg2_summary", "cfg2"), ("launches_cfg2_dropout_summary", "cfg2 + dropout")):
    d = json.load(open(P + f + ".json"))
    lora = [x for x in d if "lora_sm100" in x["kernel"]]
    tot = sum(x["launches"] * x["mean_us"] for x in lora)
    out += [f"ncu launch list, {t} (3 eager steps + profiling calls; L2-flush kernels excluded): share of the "
            f"library's kernel time", "", "| kernel | launches | mean us | share |", "|---|---|---|---|"]
    for x in lora:
        out.append(f"| {x['kernel'][:70]} | {x['launches']} | {x['mean_us']:.1f} | {x['launches'] * x['mean_us'] / tot:.1%} |")
    out.append("")
out += ["GPU tests: " + open(P + "gpu_tests.log").read().strip().splitlines()[-1], "",
        "Smoke: " + open(P + "smoke.log").read().strip().splitlines()[-1]]
open(P + "SUMMARY.md", "w").write("\n".join(out) + "\n")
