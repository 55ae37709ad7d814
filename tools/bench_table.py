"""Print the DESIGN.md §7 measurement table from a bench.py JSON line (dev aid)."""
import json, sys


def main(path):
    d = json.loads([l for l in open(path) if l.startswith("{")][-1])
    r, e, en, cb, rf = d["roofline"], d["e2e"], d.get("e2e_numpy", {}), d["cpu_baseline"], d.get("refined", {})
    s = d.get("secondary", {})
    rows = [("Config", "What", "Time", "Rate")]
    rows.append(("4 (headline)", "block LDLᵀ + 16-RHS solve + 1 refinement step, device-resident",
                 f"**{d['ms_per_step']:.1f} ms**",
                 f"{d['value']:.1f} TF/s algorithmic ({100 * d['fraction_of_fp64_peak']:.0f}% effective of the live "
                 f"{r['peak']:.1f} peak); update GEMMs {r['achieved_algorithmic']:.1f} TF/s algorithmic = "
                 f"{r['achieved']:.1f} TF/s executed (**{100 * r['frac']:.1f}%**)"))
    rows.append(("4", f"e2e from pinned host memory ({e['h2d_bytes_per_step'] / 1e9:.2f} GB H2D, "
                 f"{e['d2h_bytes_per_step'] / 1e6:.1f} MB D2H), median of {len(e.get('samples_ms', []))}",
                 f"**{e['ms_per_step']:.1f} ms**", f"{e['value']:.1f} TF/s"))
    if en:
        rows.append(("4", "e2e from plain numpy arrays (host-staged upload)", f"{en['ms_per_step']:.1f} ms",
                     f"{en['value']:.1f} TF/s"))
    if rf:
        rows.append(("4", "block_solve alone (16 RHS): unrefined / refined",
                     f"{rf['solve_refine0_ms']:.1f} ms / {rf['solve_refine1_ms']:.1f} ms", "dataflow kernel"))
        rows.append(("4", "residual ‖Kx−b‖/‖b‖, max over 16 RHS: refined / unrefined / reference", "—",
                     f"{rf['residual_refine1']:.1e} / {rf['residual_refine0']:.1e} / {rf['reference_residual_max']:.1e}"))
    rows.append(("4", f"**CPU, same step**: oracle port (C kernels + OpenBLAS, {cb['cores']} host threads), "
                 "full factor + 16-RHS solve", f"{cb['seconds']:.1f} s ({cb['factor_s']:.1f} + {cb['solve_s']:.1f})",
                 f"{cb['value']:.3f} TF/s; GPU {cb['gpu_speedup_device_resident']:.0f}× faster device-resident"))
    c3 = s.get("cfg3")
    if c3:
        rows.append(("3", f"64 × n=2048 Schur reduce (Schur-only form), device-resident / e2e "
                     f"({c3['e2e']['h2d_bytes_per_step'] / 1e9:.1f} GB H2D)",
                     f"{c3['ms_per_step']:.1f} ms / {c3['e2e']['ms_per_step']:.1f} ms",
                     f"{c3['value']:.1f} TF/s effective = {100 * c3['roofline']['frac']:.0f}% of peak"))
        cr = c3.get("cpu_reduce")
        if cr:
            rows.append(("3", f"CPU: oracle `reduce_domain`, {cr['subdomains_timed']} subdomains in {cr['procs']} "
                         "single-threaded processes → 64", f"{cr['s_per_subdomain']:.1f} s per subdomain, "
                         f"{cr['all_subdomains_s']:.0f} s for 64", f"GPU {cr['gpu_speedup']:.0f}×"))
    for k, nm in (("cfg1", "1"), ("cfg2", "2 (configs[1])"), ("cfg5", "5")):
        c = s.get(k)
        if not c:
            continue
        st = c["stage_ms"]
        rows.append((nm, c["workload"].split(": ", 1)[1] + ", full D3M from host systems",
                     f"{c['d3m_ms']:.1f} ms" if c["d3m_ms"] < 1e4 else f"**{c['d3m_ms'] / 1e3:.2f} s**",
                     f"reduce {st['reduce']:.1f} ms at {c['subdomain_tflops']:.1f} TF/s "
                     f"({100 * c['roofline']['frac']:.0f}%); factor {st['factor']:.1f} ms; solve {st['solve']:.1f} ms; "
                     f"residual {c['residual']:.1e}"))
        cr = c.get("cpu_reduce")
        if cr:
            rows.append((nm.split()[0], f"CPU: oracle `reduce_domain`, {cr['subdomains_timed']} subdomains in "
                         f"{cr['procs']} processes", f"{cr['s_per_subdomain']:.1f} s per subdomain",
                         f"GPU {cr['gpu_speedup']:.0f}× on the reduce"))
    print("| " + " | ".join(rows[0]) + " |")
    print("|---|---|---|---|")
    for row in rows[1:]:
        print("| " + " | ".join(row) + " |")
    c = d["clocks"]
    print(f"\nclocks {c['sm_mhz']:.0f} / {c['sm_max_mhz']:.0f} MHz, reasons {c['reasons']}; gpu_launches {d['gpu_launches']}")


if __name__ == "__main__":
    main(sys.argv[1])
