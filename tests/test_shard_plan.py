"""CPU (gloo, world size 2): the multi-rank hand-off plan.

Each rank builds a plan-only trainer (no device) for its shard of the same
schedule and computes the per-destination message plan. The ranks must agree
on every rank's plan (the sender writes into the receiver's inbox at offsets
both compute independently), and the message counts must equal an independent
count from the event log: one message per predict / forward / replay-forward
crossing of the rank boundary, one per backward / replay-backward crossing
whose lower stage runs its backward."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WIDTHS = [96, 128, 64, 48, 10]
BOUNDS = [0, 1, 2, 3, 4]
OWNERS = [0, 0, 1, 1]
B = 4
UNITS = 64


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, replay, out):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2503_12053_b200 as fb

    prof = fb.profile_from_widths(WIDTHS)
    t_d = float(prof["t_f"].max())
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=UNITS * t_d), BOUNDS, UNITS)
    tr = fb.PipelineTrainer(WIDTHS, fb.make_dense_net(WIDTHS, 1), BOUNDS,
                            fb.PipelineTrainOptions(policy="iter_fisher", micro_batch=B, replay=replay, device=-1))
    tr.set_shard(rank, world, OWNERS)
    tr.set_schedule(sched.events, UNITS * B)
    plan = tr.handoff_plan()
    mine = [int(x) for x in plan[0]] + [int(x) for x in plan[1]]
    allp = [None] * world
    dist.all_gather_object(allp, mine)
    out[rank] = allp
    tr.close()
    dist.destroy_process_group()


def _expected(fb, replay):
    prof = fb.profile_from_widths(WIDTHS)
    t_d = float(prof["t_f"].max())
    ev = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=UNITS * t_d), BOUNDS, UNITS).events
    dropped = set(ev["item"][ev["kind"] == 1].tolist())
    has_bwd = {(int(e["item"]), int(e["stage"])) for e in ev if e["kind"] == 4}
    pending = {}
    fires0 = 0
    to1 = to0 = 0
    for e in ev:
        k, u, j = int(e["kind"]), int(e["item"]), int(e["stage"])
        if k == 0 and u not in dropped:
            to1 += 1                                   # predict crosses stage 1 -> 2
        elif k == 2 and j == 1:
            to1 += 1                                   # stage-1 output -> stage 2
        elif k == 4:
            pending.setdefault((int(e["worker"]), j), []).append(u)
            if j == 2 and (u, 1) in has_bwd:
                to0 += 1                               # stage-2 input gradient -> stage 1
        elif k == 5:
            if pending.get((int(e["worker"]), j)):
                pending[(int(e["worker"]), j)] = []
                if j == 0:
                    fires0 += 1
    if replay:
        to1 += fires0                                  # replay forward sweep
        to0 += fires0                                  # replay backward sweep
    return to0, to1


@pytest.mark.parametrize("replay", [False, True])
def test_ranks_agree_on_handoff_plan(fb, replay):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), replay, out), nprocs=world, join=True, start_method="spawn")
    plans = [out[r] for r in range(world)]
    assert plans[0] == plans[1]                        # every rank computed every rank's plan identically
    for r in range(world):
        assert plans[0][r] == plans[1][r]
    bytes_to = plans[0][0][:world]
    msgs_to = plans[0][0][world:]
    to0, to1 = _expected(fb, replay)
    assert msgs_to == [to0, to1]
    # each message is B x width floats, 256-byte aligned in the inbox
    assert bytes_to[1] == to1 * ((B * 64 * 4 + 255) // 256 * 256)
    assert bytes_to[0] == to0 * ((B * 64 * 4 + 255) // 256 * 256)


def test_plan_only_trainer_refuses_device_work(fb):
    tr = fb.PipelineTrainer(WIDTHS, fb.make_dense_net(WIDTHS, 1), BOUNDS, fb.PipelineTrainOptions(device=-1))
    with pytest.raises(fb.DeviceError):
        tr.load_stream(np.zeros((4, WIDTHS[0])), np.zeros(4, dtype=np.uint64))
    tr.close()


# ---- world sizes 4 and 8 (one stage per rank at 8): C4's deep MLP, 8 one-layer stages
DEEP = [784] + [256] * 7 + [10]
DEEP_BOUNDS = list(range(9))


def _deep_worker(rank, world, port, owners, out):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2503_12053_b200 as fb

    prof = fb.profile_from_widths(DEEP)
    t_d = float(prof["t_f"].max())
    sched = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=UNITS * t_d), DEEP_BOUNDS, UNITS)
    tr = fb.PipelineTrainer(DEEP, None, DEEP_BOUNDS,
                            fb.PipelineTrainOptions(policy="iter_fisher", micro_batch=B, replay=True, device=-1))
    tr.set_shard(rank, world, owners)
    tr.set_schedule(sched.events, UNITS * B)
    plan = tr.handoff_plan()
    mine = [int(x) for x in plan[0]] + [int(x) for x in plan[1]]
    allp = [None] * world
    dist.all_gather_object(allp, mine)
    out[rank] = allp
    tr.close()
    dist.destroy_process_group()


def _expected_general(fb, owners, world):
    """Messages per destination rank per chunk, counted from the event log: across every
    rank boundary j | j+1, one per predict sweep, stage-j forward and replay forward sweep
    (to owner[j+1]); one per stage-(j+1) backward whose unit runs stage j's backward and
    per replay backward sweep (to owner[j])."""
    prof = fb.profile_from_widths(DEEP)
    t_d = float(prof["t_f"].max())
    ev = fb.Schedule.forced(prof, t_d, fb.StreamSpec(t_d=t_d, horizon=UNITS * t_d), DEEP_BOUNDS, UNITS).events
    dropped = set(ev["item"][ev["kind"] == 1].tolist())
    has_bwd = {(int(e["item"]), int(e["stage"])) for e in ev if e["kind"] == 4}
    P = len(owners)
    cuts = [j for j in range(P - 1) if owners[j] != owners[j + 1]]
    to = [0] * world
    pending = {}
    for e in ev:
        k, u, j = int(e["kind"]), int(e["item"]), int(e["stage"])
        if k == 0 and u not in dropped:
            for c in cuts:
                to[owners[c + 1]] += 1
        elif k == 2 and j in cuts:
            to[owners[j + 1]] += 1
        elif k == 4:
            pending.setdefault((int(e["worker"]), j), []).append(u)
            if j - 1 in cuts and (u, j - 1) in has_bwd:
                to[owners[j - 1]] += 1
        elif k == 5 and pending.get((int(e["worker"]), j)):
            pending[(int(e["worker"]), j)] = []
            if j == 0:
                for c in cuts:
                    to[owners[c + 1]] += 1
                    to[owners[c]] += 1
    return to


@pytest.mark.parametrize("world", [4, 8])
def test_ranks_agree_on_handoff_plan_wide(fb, world):
    """World sizes 4 and 8 over gloo: every rank computes every rank's message plan
    identically (senders address receivers' inboxes and acks from it), and the per-rank
    message counts equal the independent count from the event log."""
    owners = fb.ferret.stage_owners(len(DEEP_BOUNDS) - 1, world)
    assert sorted(set(owners)) == list(range(world))
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_deep_worker, args=(world, _free_port(), owners, out), nprocs=world, join=True,
                       start_method="spawn")
    plans = [out[r] for r in range(world)]
    for r in range(1, world):
        assert plans[r] == plans[0]
    msgs_to = plans[0][0][world:]
    assert msgs_to == _expected_general(fb, owners, world)
    assert all(m > 0 for m in msgs_to)
