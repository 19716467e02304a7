"""Print the headline fields of a bench JSON line: python tools/bench_show.py file.json"""
import json, sys
for p in sys.argv[1:]:
    l = json.loads(open(p).read().strip().split('\n')[-1])
    print("==", p)
    print("value", round(l["value"], 2), "e2e", round(l["e2e"]["value"], 2), "ms/step", round(l["ms_per_step"], 1),
          "frac", round(l["roofline"]["frac"], 4), "frac_exec", round(l["roofline"].get("frac_executed", 0), 4))
    for k in ["stage_cycles_share", "engine_prof_share", "squeeze_share", "lstsq_factor_share", "svd_detail", "overflow_ws",
              "step_gflop_p50_p90_p99_max", "step_ms_p50_p90_p99_max", "stage_sm_seconds_per_attempted_step",
              "cpu_baseline", "clocks", "completed_frac", "cta_seconds_in_steps", "mean_cross_calls",
              "ws_peak_mb", "example_ranks"]:
        print(" ", k, l.get(k))
    print("  status", l["config"]["status_counts"], "slots", l["config"]["workspace_slots"], l["config"]["workspace_mb_per_slot"])
