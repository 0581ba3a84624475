"""CPU restatement of the simulator step after the draft phase.  TEST INFRASTRUCTURE ONLY (the checker of
paper_2502_15197_b200.sim_engine.GpuSimulator; see oracle/oracle.py's header for who may import it).

Follows /root/reference/pkg/src/tetris_sched/sim_engine.py (paths below relative to its package):
  policy windows     sim_engine.py:349-371 (tetris: select_tetris(cumulative_products(surrogate), C);
                     sd: min(k, depth); dsd: select_dsd common window clamped to the depth, selector.py:193-222)
  apply_verification sim_engine.py:374-404 (flat uniform stream, w_i draws per row in row order)
  expected_accepted  selector.py:286-306
  credit             sim_engine.py:467-471  min(acc + 1, remaining)
  DSD estimate       sim_engine.py:473-478
  refill_batch       sim_engine.py:428-451  (survivors keep their order; replacements appended, arrival = step + 1)
  draft depths       sim_engine.py:343      min(k + extra, remaining)
"""
from __future__ import annotations

import reference_port as RP


def dsd_window(alpha, n_rows, capacity, depth_limit):
    k_max = min(depth_limit, capacity // n_rows)
    if k_max < 1:
        return 0
    best_k, best, value, power = 1, alpha, alpha, alpha
    for k in range(2, k_max + 1):
        power *= alpha
        value += power
        if value > best:
            best, best_k = value, k
    return best_k


class OracleSim:
    def __init__(self, batch_size, k, capacity, extra, policy, dsd_decay, dsd_initial_estimate, lengths, uniforms):
        self.B, self.k, self.K, self.C, self.policy = batch_size, k, k + extra, capacity, policy
        self.decay = dsd_decay
        self.alpha_hat = dsd_initial_estimate
        self.lengths = list(lengths)
        self.uniforms = list(uniforms)
        self.active = [dict(id=i, target=self.lengths[i], served=0, arrival=0) for i in range(batch_size)]
        self.next_len = batch_size
        self.next_id = batch_size
        self.u_off = 0
        self.step_no = 0

    def depths(self):
        return [min(self.K, r["target"] - r["served"]) for r in self.active]

    def step(self, truth_rows, surrogate_rows):
        depths = self.depths()
        stats = None
        if self.policy == "tetris":
            windows, stats = RP.select_tetris(RP.cumulative_products(surrogate_rows), self.C)
        elif self.policy == "sd":
            windows = tuple(min(self.k, d) for d in depths)
        else:
            common = dsd_window(self.alpha_hat, self.B, self.C, self.K)
            windows = tuple(min(common, d) for d in depths)
        accepted = []
        for w, row in zip(windows, truth_rows):
            draws = self.uniforms[self.u_off:self.u_off + w]
            self.u_off += w
            n = 0
            for u, a in zip(draws, row):
                if u < a:
                    n += 1
                else:
                    break
            accepted.append(n)
        value = 0.0
        for w, row in zip(windows, truth_rows):
            cum = 1.0
            for j in range(w):
                cum *= row[j]
                value += cum
        credited = []
        for r, a in zip(self.active, accepted):
            t = min(a + 1, r["target"] - r["served"])
            r["served"] += t
            credited.append(t)
        sent = sum(windows)
        if sent > 0:
            rate = sum(accepted) / sent
            self.alpha_hat = self.decay * self.alpha_hat + (1.0 - self.decay) * rate
        done = [r for r in self.active if r["target"] - r["served"] <= 0]
        self.active = [r for r in self.active if r["target"] - r["served"] > 0]
        for _ in done:
            self.active.append(dict(id=self.next_id, target=self.lengths[self.next_len], served=0,
                                    arrival=self.step_no + 1))
            self.next_id += 1
            self.next_len += 1
        out = dict(windows=tuple(windows), accepted=tuple(accepted), credited=tuple(credited), expected=value,
                   stats=stats, completions=tuple((r["id"], r["arrival"]) for r in done), alpha_hat=self.alpha_hat)
        self.step_no += 1
        return out
