function Degrees(Graph g) {
  propNode<int> deg;
  propNode<int> indeg;
  g.attachNodeProperty(deg = 0, indeg = 0);
  int slots = 0;
  forall (v in g.nodes()) {
    forall (nbr in g.neighbors(v)) {
      v.deg += 1;
      slots += 1;
    }
    forall (u in g.nodesTo(v)) {
      v.indeg += 1;
    }
  }
}
