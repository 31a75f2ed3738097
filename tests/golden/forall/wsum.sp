function Weighted_Sum(Graph g) {
  propNode<int> w;
  propNode<long> acc;
  g.attachNodeProperty(w = 3, acc = 7);
  long total = 5;
  forall (v in g.nodes()) {
    int count = 0;
    forall (nbr in g.nodesTo(v)) {
      total += nbr.w;
      v.acc += nbr.w;
      count++;
    }
  }
}
