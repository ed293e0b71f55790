"""Host logic of the persistent tile-DAG kernels (dag.cu): the task orders that
the library exports through tsvd_dag_order are complete, respect every dependency, and cannot
deadlock with any number of worker CTAs (simulated: workers claim tickets in order and finish a
task once its dependencies are met; the chain CTA advances concurrently).  K5 is Alg 2
 as the blocked Cholesky of DESIGN.md R8; K6 the back substitution of Eq (5)
(PAPER.md:326)."""
import pytest

P = pytest.importorskip("paper_2401_09703_b200")

T_CHAIN, T_S, T_U, T_W, T_V = 0, 1, 2, 3, 4
STRIP = 4  # tiles per T_W strip task (dag.cu)


def _tiles(t, nt):
    """The (q, i, c) tile updates a U or W task performs, in order."""
    ty, q, i, c = t
    if ty == T_U:
        return [(q, i, c)]
    return [(q, i, cc) for cc in range(c, min(c + STRIP, nt))]


def _chol_expected(nt):
    S = {(j, c) for j in range(nt) for c in range(j + 2, nt)}
    U = {(q, i, c) for q in range(nt) for i in range(q + 1, nt) for c in range(i, nt)} - \
        {(q, q + 1, q + 1) for q in range(nt - 1)}
    return S, U


def _simulate_chol(nt, tasks, workers):
    fin = set()                       # (q, c): tile of R final
    ver = {}                          # (i, c) -> bulk updates applied
    nxt = 1                           # next ticket (0 is the chain)
    held = [None] * workers
    step, phase = 0, 0                # chain position
    done = 0
    v = lambda i, c: ver.get((i, c), 0)
    while True:
        progress = False
        # chain: P(step) -> S(step, step+1) -> fused update of (step+1, step+1)
        if step < nt:
            if phase == 0:
                fin.add((step, step))
                phase, progress = 1, True
                if step + 1 == nt:
                    step += 1
            if phase == 1 and step + 1 < nt and v(step, step + 1) >= step:
                fin.add((step, step + 1))
                phase, progress = 2, True
            if phase == 2 and v(step + 1, step + 1) >= step:
                step, phase, progress = step + 1, 0, True
        for w in range(workers):
            if held[w] is None and nxt < len(tasks):
                held[w] = tasks[nxt]
                nxt += 1
                progress = True
            t = held[w]
            if t is None:
                continue
            ty, q, i, c = t
            if ty == T_S:
                ok = (q, q) in fin and v(q, c) >= q
                if ok:
                    fin.add((q, c))
            else:  # U or a strip W: all its tiles' dependencies first (as the kernel waits)
                tl = _tiles(t, nt)
                ok = all((qq, ii) in fin and (qq, cc) in fin and v(ii, cc) >= qq for qq, ii, cc in tl)
                if ok:
                    for qq, ii, cc in tl:
                        assert v(ii, cc) == qq, ("update order", t)
                        ver[(ii, cc)] = qq + 1
            if ok:
                held[w] = None
                done += 1
                progress = True
        if not progress:
            break
    return step >= nt and done == len(tasks) - 1


@pytest.mark.parametrize("nt", [1, 2, 3, 4, 5, 8, 13, 30])
def test_chol_order_complete_and_ordered(nt):
    tasks = P.dag_order(0, nt)
    assert tasks[0][0] == T_CHAIN and all(t[0] != T_CHAIN for t in tasks[1:])
    S_exp, U_exp = _chol_expected(nt)
    S = [(t[1], t[3]) for t in tasks if t[0] == T_S]
    U = [u for t in tasks if t[0] in (T_U, T_W) for u in _tiles(t, nt)]
    assert len(S) == len(set(S)) and set(S) == S_exp
    assert len(U) == len(set(U)) and set(U) == U_exp
    assert all(t[0] in (T_CHAIN, T_S, T_U, T_W) for t in tasks)
    assert all(t[3] - t[2] >= 0 and (t[3] - t[2]) % STRIP == 0 for t in tasks if t[0] == T_W)
    pos = {}
    for n, t in enumerate(tasks):
        if t[0] == T_S:
            pos[(T_S, t[1], t[3])] = n
        elif t[0] in (T_U, T_W):
            for u in _tiles(t, nt):
                pos[(T_U,) + u] = n
    for n, t in enumerate(tasks):
        ty, q, i, c = t
        if ty == T_S:  # the updates of its tile by every earlier panel precede it
            for qq in range(q):
                if not (qq == q - 1 and c == q):
                    assert pos[(T_U, qq, q, c)] < n
        elif ty in (T_U, T_W):
            for (q_, i_, c_) in _tiles(t, nt):
                for cc in (i_, c_):  # operand tiles of R: chain-made (== q+1) or an earlier S
                    if cc != q_ + 1:
                        assert pos[(T_S, q_, cc)] < n
                if q_ >= 1:          # per-tile order: panel q-1 first
                    assert pos[(T_U, q_ - 1, i_, c_)] < n


@pytest.mark.parametrize("nt", [2, 3, 6, 11, 24])
@pytest.mark.parametrize("workers", [1, 2, 5, 64])
def test_chol_order_no_deadlock(nt, workers):
    assert _simulate_chol(nt, P.dag_order(0, nt), workers)


def _simulate_trsm(nt, nkb, tasks, workers):
    fin = set()
    ver = {}
    nxt, held, done = 1, [None] * workers, 0
    j = nt - 1
    v = lambda i, b: ver.get((i, b), 0)
    b_chain = 0
    while True:
        progress = False
        if j >= 0 and v(j, b_chain) >= max(nt - 2 - j, 0):
            fin.add((j, b_chain))
            progress = True
            b_chain += 1
            if b_chain == nkb:
                b_chain, j = 0, j - 1
        for w in range(workers):
            if held[w] is None and nxt < len(tasks):
                held[w], nxt, progress = tasks[nxt], nxt + 1, True
            t = held[w]
            if t is None:
                continue
            _, jj, i, b = t
            if (jj, b) in fin and v(i, b) >= nt - 1 - jj:
                assert v(i, b) == nt - 1 - jj
                ver[(i, b)] = nt - jj
                held[w], done, progress = None, done + 1, True
        if not progress:
            break
    return j < 0 and done == len(tasks) - 1


@pytest.mark.parametrize("nt,nkb", [(1, 1), (2, 1), (3, 2), (7, 1), (20, 3)])
def test_trsm_order(nt, nkb):
    tasks = P.dag_order(1, nt, nkb)
    assert tasks[0][0] == T_CHAIN
    V = [(t[1], t[2], t[3]) for t in tasks[1:]]
    assert all(t[0] == T_V for t in tasks[1:])
    exp = {(j, i, b) for j in range(nt) for i in range(j - 1) for b in range(nkb)}
    assert len(V) == len(set(V)) and set(V) == exp
    for workers in (1, 3, 64):
        assert _simulate_trsm(nt, nkb, tasks, workers)


def test_order_rejects_bad_arguments():
    with pytest.raises(ValueError):
        P.dag_order(2, 4)
    with pytest.raises(ValueError):
        P.dag_order(0, 0)
