"""The streamed planner's documented search order: the smallest depth k, then two
staging buffers before one, then the smallest accumulator depth j whose predicted device bytes fit
the budget.  Tests use it to state which tier a given budget must select."""
import paper_2604_20819_b200 as cqs


def planner_tier(desc, budget, depths):
    for k in depths:
        for nb in (2, 1):
            for j in range(k + 1):
                if cqs.cqs_memory_model(desc, k, j, nb)[0] <= budget:
                    return k, j, nb
    return None
