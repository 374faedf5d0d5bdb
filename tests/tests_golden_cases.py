"""Parameters shared by tests/golden/make_golden.py and the tests."""

# scenario -> envelope-lead bucket (ms)
LEAD_CASES = {"c1": 500.0, "pab_overload": 250.0, "wide": 100.0, "c2_subset": 1000.0}


# replay_check (engine.cpp:290-393) known answers: mutations of the
# reference's own JSONL event log of pab_overload instance 0.  Each maps the
# line list (log_end last) to a mutated line list.
def _first(lines, kind, req=None):
    for i, ln in enumerate(lines):
        if f'"kind":"{kind}"' in ln and (req is None or f'"req_id":{req},' in ln
                                         or ln.endswith(f'"req_id":{req}}}')):
            return i
    raise ValueError(kind)


def _m_drop(kind):
    def f(lines):
        i = _first(lines, kind)
        return lines[:i] + lines[i + 1:]
    return f


def _m_dup_arrival(lines):
    i = _first(lines, "arrival")
    return lines[:i + 1] + [lines[i]] + lines[i + 1:]


def _m_swap(i, j):
    def f(lines):
        out = list(lines)
        out[i], out[j] = out[j], out[i]
        return out
    return f


def _m_decrease_t(lines):
    out = list(lines)
    out[5] = '{"t_ms":0.001' + out[5][out[5].index(','):]
    return out


def _m_token_idx(lines):
    i = _first(lines, "token_emit")
    i = next(k for k in range(i + 1, len(lines)) if '"token_idx":1}' in lines[k])
    out = list(lines)
    out[i] = out[i].replace('"token_idx":1}', '"token_idx":5}')
    return out


def _m_reject_after_activity(lines):
    i = _first(lines, "token_emit")
    t = lines[i][:lines[i].index(',')]
    return lines[:i + 1] + [t + ',"kind":"admission_reject","req_id":0,"prompt_tokens":2125,'
                            '"pab_tokens":7}'] + lines[i + 1:]


def _m_truncated_complete(lines):
    return lines[:3000] + ['{"kind":"log_end","node":0,"incomplete":0}']


def _m_done_early(lines):
    i = _first(lines, "token_emit", 1)
    t = lines[i][:lines[i].index(',')]
    return lines[:i + 1] + [t + ',"kind":"request_done","req_id":1}'] + lines[i + 1:]


def _m_emit_outside(lines):
    i = _first(lines, "token_emit")
    j = next(k for k in range(i + 1, len(lines)) if '"kind":"batch_end"' in lines[k])
    return lines[:i] + lines[i + 1:j + 1] + [lines[i]] + lines[j + 1:]


def _m_unknown_request(lines):
    i = _first(lines, "token_emit")
    t = lines[i][:lines[i].index(',')]
    return lines[:i + 1] + [t + ',"kind":"token_emit","req_id":999999,"token_idx":0}'] + lines[i + 1:]


REPLAY_MUTATIONS = {
    "clean": lambda lines: list(lines),
    "drop_first_token": _m_drop("token_emit"),
    "drop_first_batch_end": _m_drop("batch_end"),
    "drop_first_arrival": _m_drop("arrival"),
    "dup_arrival": _m_dup_arrival,
    "swap_2_3": _m_swap(2, 3),
    "decrease_t": _m_decrease_t,
    "bad_token_idx": _m_token_idx,
    "reject_after_activity": _m_reject_after_activity,
    "truncated_complete": _m_truncated_complete,
    "done_early": _m_done_early,
    "emit_outside": _m_emit_outside,
    "unknown_request": _m_unknown_request,
}


def replay_canonical(violations):
    """Order-exact for the per-event violations, sorted for the final scan
    (the reference walks an unordered_map there)."""
    ev = [v for v in violations if not v.startswith("request ")]
    rq = sorted(v for v in violations if v.startswith("request "))
    return ev + rq


# run_cluster cases whose node event logs and routing log (save_event_log /
# save_routing_log) are pinned byte for byte.
CLUSTER_LOG_CASES = ("pab0_8", "count37_3", "pab5000_8", "pab_hz10s_8", "pab20_2", "rr_giant_2",
                     "rr_pab30_3", "rr_mixed_4")
