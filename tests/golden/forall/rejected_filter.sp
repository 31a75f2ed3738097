function Filtered(Graph g) {
  propNode<int> p;
  g.attachNodeProperty(p = 2);
  int s = 0;
  forall (v in g.nodes().filter(p == 2)) {
    forall (nbr in g.neighbors(v)) {
      s += nbr.p;
    }
  }
}
