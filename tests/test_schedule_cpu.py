"""Host logic of paper_2506_11586_b200/schedule.py: which layers may overlap. Only layers reading
the same input tensor group together (fire expand1x1/expand3x3; a ResNet block's first conv and
its projection); every layer appears exactly once and the network order is otherwise kept."""
from paper_2506_11586_b200.schedule import concurrent_groups
from workloads import layers


def _check_partition(names, groups):
    flat = [i for g in groups for i in g]
    assert sorted(flat) == list(range(len(names)))
    firsts = [g[0] for g in groups]
    assert firsts == sorted(firsts)  # groups in network order of their first layer


def test_squeezenet_fire_pairs():
    names = [l.name for l in layers.squeezenet11()]
    groups = concurrent_groups(names)
    _check_partition(names, groups)
    pairs = [[names[i] for i in g] for g in groups if len(g) > 1]
    assert pairs == [[f"fire{k}.e1", f"fire{k}.e3"] for k in range(2, 10)]
    assert all(len(g) <= 2 for g in groups)


def test_resnet50_projection_moves_up_to_c1():
    names = [l.name for l in layers.network("resnet50")]
    groups = concurrent_groups(names)
    _check_partition(names, groups)
    pairs = [[names[i] for i in g] for g in groups if len(g) > 1]
    assert pairs == [[f"l{k}.b0.c1", f"l{k}.b0.ds"] for k in range(1, 5)]
    # the projection runs beside c1, i.e. before c2 and c3 of its block
    order = [names[i] for g in groups for i in g]
    assert order.index("l1.b0.ds") < order.index("l1.b0.c2")


def test_unrelated_names_stay_serial():
    names = ["a", "b.e1", "c", "d.b1.c1", "e.ds"]
    assert concurrent_groups(names) == [[0], [1], [2], [3], [4]]
