"""Train a C3 latency predictor the way the reference does, and export it as ILMD.

SURVEY.md §8(d) "Weights (ii)": a trained C3 for realistic decode margins and
context occupancy.  This is an offline fixture generator (like
tests/golden/make_golden.py): it runs in the CPU container, where the
reference's own workload generator + DES are compiled in oracle/_ref, and
writes `tests/golden/c3_trained.model` (+ a .json report), which the
benches load as data.  Nothing on the product path imports it.

  python tests/golden/train_c3.py [--n-per-trace 60000] [--epochs 6]

Steps:
1. DES traces from the reference (workload.cpp + des.cpp via oracle/_ref:
   `ref_make_trace`), every workload kind, several seeds.
2. NormStats from the reference dataset builder (`build_dataset` /
   `compute_norm_stats`, dataset.cpp:243-274, via `ref_make_model`) on the
   training traces, and the reference init rule (cnn.cpp:335-352) as the
   starting point.
3. Training samples = the simulator's own request stream with the DES truth
   latencies (`ref_capture` mode 1, sequential): inputs exactly as
   `next_request` builds them (simcore.cpp:25-66), labels = the DES triple.
4. The reference forward (cnn.cpp:90-125) in PyTorch, the reference loss
   (cnn.cpp:128-163: squared error of the normalised log1p regressions + the
   three softmax cross-entropies, class = min(raw, C - 1)), Adam.
5. Export in the reference's parameter layout (cnn.cpp:44-86, column-major
   `W[o + k * rows]`), then check the trained model with the reference's own
   `simulate_trace` on held-out DES traces against the DES cycle counts.
"""
from __future__ import annotations

import argparse
import json
import sys
import tempfile
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.oracle import Port, Ref  # noqa: E402  (test infrastructure: fixture generation only)
from paper_2105_05821_b200.formats import CnnConfig, Model, read_model, read_trace, write_model, write_trace  # noqa: E402
from paper_2105_05821_b200.formats import Trace  # noqa: E402

KINDS = ["mix", "loop-kernel", "pointer-chase", "branchy", "streaming"]


class C3(torch.nn.Module):
    """cnn.cpp:90-125 for the C3 shape: conv l = kernel-2 / stride-2 windows of
    adjacent columns, GEMM -> bias -> ReLU; FC1 -> ReLU; FC2."""

    def __init__(self, cfg: CnnConfig):
        super().__init__()
        self.cfg = cfg
        cin = cfg.input_channels
        self.convs = torch.nn.ModuleList()
        for c in cfg.conv_channels:
            self.convs.append(torch.nn.Linear(2 * cin, c))
            cin = c
        self.fc1 = torch.nn.Linear(cfg.flat_dim, cfg.fc_hidden)
        self.fc2 = torch.nn.Linear(cfg.fc_hidden, cfg.output_dim)

    def forward(self, x):  # x: [B, 128 columns, 50 slots] (padded)
        a = x
        for lin in self.convs:
            b, length, c = a.shape
            a = torch.relu(lin(a.reshape(b, length // 2, 2 * c)))  # window p = columns 2p, 2p+1
        flat = a.reshape(a.shape[0], -1)  # flat[p * C + c]
        return self.fc2(torch.relu(self.fc1(flat)))

    # reference layout <-> torch: W[o + k * out] (column-major [out x in]) == torch weight [out][in]
    def load_reference(self, params: np.ndarray):
        p = 0
        with torch.no_grad():
            for lin in list(self.convs) + [self.fc1, self.fc2]:
                o, i = lin.weight.shape
                lin.weight.copy_(torch.from_numpy(params[p:p + o * i].reshape(i, o).T.copy()))
                p += o * i
                lin.bias.copy_(torch.from_numpy(params[p:p + o].copy()))
                p += o
        assert p == params.size

    def export_reference(self) -> np.ndarray:
        out = []
        with torch.no_grad():
            for lin in list(self.convs) + [self.fc1, self.fc2]:
                out.append(lin.weight.detach().float().cpu().numpy().T.reshape(-1))
                out.append(lin.bias.detach().float().cpu().numpy().reshape(-1))
        return np.concatenate(out).astype(np.float32)


def reference_loss(y, tri, norm, cfg: CnnConfig):
    """cnn.cpp:128-163, batched (mean over samples)."""
    raw = tri.double()
    lm = torch.as_tensor(norm[100:103], dtype=torch.float64, device=y.device)
    ls = torch.as_tensor(norm[103:106], dtype=torch.float64, device=y.device)
    target = (torch.log1p(raw) - lm) / ls
    loss = ((y[:, :3].double() - target) ** 2).sum(1)
    base = 3
    for h, c in enumerate((cfg.class_fetch, cfg.class_exec, cfg.class_store)):
        cls = torch.clamp(tri[:, h], max=c - 1).long()
        loss = loss + torch.nn.functional.cross_entropy(y[:, base:base + c].double(), cls, reduction="none")
        base += c
    return loss.mean()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-per-trace", type=int, default=40_000)
    ap.add_argument("--seeds", type=int, default=3)
    ap.add_argument("--epochs", type=int, default=6)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--lr", type=float, default=1e-3)
    ap.add_argument("--threads", type=int, default=8)
    ap.add_argument("--device", default="cuda" if torch.cuda.is_available() else "cpu")
    ap.add_argument("--val-n", type=int, default=20_000, help="instructions per closed-loop validation trace")
    ap.add_argument("--dagger", type=int, default=0,
                    help="after each epoch, add this many closed-loop requests per training trace (the model's "
                         "own simulation, K = 32) labelled with the DES latencies of their instructions")
    ap.add_argument("--out", default=str(ROOT / "tests" / "golden" / "c3_trained.model"))
    a = ap.parse_args()
    torch.manual_seed(0)
    torch.set_num_threads(a.threads)
    ref = Ref()
    work = Path(tempfile.mkdtemp(prefix="train_c3_"))
    t0 = time.time()
    # 1. DES traces (train: seeds 1..S; held out: seed 100), every workload kind
    train_paths, held_paths, val_paths = [], [], []
    for kind in KINDS:
        for s in range(1, a.seeds + 1):
            pth = work / f"{kind}_{s}.trace"
            ref.make_trace(kind, a.n_per_trace, 1000 * s + KINDS.index(kind), pth)
            train_paths.append(pth)
        pth = work / f"{kind}_held.trace"
        ref.make_trace(kind, a.n_per_trace, 100_000 + KINDS.index(kind), pth)
        held_paths.append(pth)
        pth = work / f"{kind}_val.trace"
        ref.make_trace(kind, a.val_n, 50_000 + KINDS.index(kind), pth)
        val_paths.append(pth)
    merged = work / "train_all.trace"
    parts, tick = [], 0
    for pth in train_paths:  # fetch ticks made monotonic across the seams (read by the dataset builder)
        t = read_trace(pth)
        # dataset.cpp:17-21: tick[i] - tick[i-1] == truth fetch latency of i
        t.fetch_tick = t.fetch_tick - t.fetch_tick[0] + np.uint64(tick + (int(t.truth[0, 0]) if parts else 0))
        tick = int(t.fetch_tick[-1])
        parts.append(t)
    write_trace(merged, Trace.concat(parts))
    # 2. NormStats from the reference dataset builder + the reference init rule
    init_path = work / "c3_init.model"
    ref.make_model(merged, init_path, seed=7)
    init = read_model(init_path)
    cfg = init.config
    print(f"traces + norm: {time.time() - t0:.1f} s", flush=True)
    # 3. samples: the simulator's request stream under the DES latencies
    xs, ts = [], []
    width = 50 * (cfg.max_context + 1)
    for pth in train_paths:
        cap = ref.capture(pth, init_path, a.n_per_trace, mode=1, sequential=True, width=width)
        n = min(cap["count"], a.n_per_trace)
        xs.append(cap["inputs"][:n].astype(np.float16))  # |x| <= 10: f16 is plenty for training
        ts.append(cap["triples"][:n])
    X = np.concatenate(xs)
    T = np.concatenate(ts).astype(np.int64)
    del xs
    print(f"samples {X.shape[0]} ({time.time() - t0:.1f} s)", flush=True)
    # 4. train
    dev = torch.device(a.device)
    net = C3(cfg)
    net.load_reference(init.params)
    net = net.to(dev)
    Xd = torch.from_numpy(X).to(dev)  # f16, resident on the device when training on a GPU
    Td = torch.from_numpy(T).to(dev)
    # TrainParams defaults (cnn.hpp:100-107): Adam lr 1e-3, betas (0.9, 0.999), eps 1e-8, batch 256, mean gradient
    opt = torch.optim.Adam(net.parameters(), lr=a.lr, betas=(0.9, 0.999), eps=1e-8)
    pad = cfg.sequence_length - (cfg.max_context + 1)
    rng = np.random.default_rng(0)
    # Closed-loop validation selects the epoch (as the reference's validation loss does,
    # cnn.cpp:540-566): the simulation feeds the model's own latencies back into its
    # inputs, which teacher-forced loss does not see; score = mean |log(C3 / DES cycles)|
    # over the validation traces, simulated by the oracle port (K = 32).
    port = Port()
    val = [(read_trace(pth), ref.simulate(pth, None, sequential=True, n_hint=a.val_n)["total_cycles"])
           for pth in val_paths]

    def closed_loop_score(params):
        m = Model(cfg, init.norm, params)
        errs = []
        for t, des in val:
            tot = port.simulate(t, m, k=32)["total_cycles"]
            errs.append(abs(np.log(max(tot, 1) / des)))
        return float(np.mean(errs)), errs

    best = (float("inf"), init.params, -1)
    n_all = X.shape[0]
    for ep in range(a.epochs):
        perm = rng.permutation(n_all)
        tot, cnt = 0.0, 0
        for b0 in range(0, n_all - a.batch + 1, a.batch):
            idx = torch.from_numpy(perm[b0:b0 + a.batch]).to(dev)
            x = Xd[idx].float().reshape(-1, cfg.max_context + 1, 50)
            x = torch.nn.functional.pad(x, (0, 0, 0, pad))  # pad_input: zero columns to 128 (cnn.cpp:219-225)
            loss = reference_loss(net(x), Td[idx], init.norm, cfg)
            opt.zero_grad()
            loss.backward()
            opt.step()
            tot += float(loss.detach()) * len(idx)
            cnt += len(idx)
        params = net.export_reference()
        if a.dagger > 0 and ep + 1 < a.epochs:
            # DAgger-style aggregation: contexts the simulation reaches with the current
            # model (ref_capture mode 0), labelled with the DES truth of each instruction
            cur = work / "c3_cur.model"
            write_model(cur, Model(cfg, init.norm, params))
            add_x, add_t = [], []
            for pth in train_paths:
                tr = read_trace(pth)
                cap = ref.capture(pth, cur, tr.n, mode=0, k=32, width=width)
                n = min(cap["count"], tr.n)
                pick = rng.choice(n, size=min(a.dagger, n), replace=False)
                add_x.append(torch.from_numpy(cap["inputs"][pick].astype(np.float16)))
                add_t.append(torch.from_numpy(tr.truth[cap["index"][pick].astype(np.int64)].astype(np.int64)))
                del cap
            Xd = torch.cat([Xd, torch.cat(add_x).to(dev)])
            Td = torch.cat([Td, torch.cat(add_t).to(dev)])
            n_all = Xd.shape[0]
        score, errs = closed_loop_score(params)
        if score < best[0]:
            best = (score, params, ep)
        print(f"epoch {ep}: samples {n_all} loss {tot / cnt:.4f} closed-loop |log CPI ratio| {score:.4f} "
              f"({' '.join(f'{e:.3f}' for e in errs)}) ({time.time() - t0:.1f} s)", flush=True)
    params = best[1]
    print(f"selected epoch {best[2]} (closed-loop score {best[0]:.4f})", flush=True)
    out = Path(a.out)
    out.parent.mkdir(parents=True, exist_ok=True)
    write_model(out, Model(cfg, init.norm, params))
    # 5. the reference's own simulate_trace with the trained model vs the DES, held-out traces
    report = {"samples": int(X.shape[0]), "samples_final": int(n_all), "dagger_per_trace": a.dagger, "epochs": a.epochs, "kinds": KINDS, "n_per_trace": a.n_per_trace,
              "seeds": a.seeds, "device": a.device, "final_loss": tot / cnt, "selected_epoch": best[2],
              "closed_loop_score": best[0], "held_out": {}}
    for pth in held_paths:
        des = read_trace(pth)
        r = ref.simulate(pth, out, sequential=True, n_hint=des.n)
        truth = ref.simulate(pth, None, sequential=True, n_hint=des.n)  # oracle latencies = the DES total
        err = 100.0 * (r["total_cycles"] - truth["total_cycles"]) / truth["total_cycles"]
        report["held_out"][pth.stem] = {"instructions": des.n, "des_cycles": truth["total_cycles"],
                                        "c3_cycles": r["total_cycles"], "cpi_error_percent": err}
        print(f"{pth.stem}: DES {truth['total_cycles']} C3 {r['total_cycles']} CPI error {err:+.2f}%", flush=True)
    (out.with_suffix(".json")).write_text(json.dumps(report, indent=1))


if __name__ == "__main__":
    main()
