#ifndef SELECT_F32_TT_H
#define SELECT_F32_TT_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_f32_tt_config;

static inline select_f32_tt_config select_f32_tt(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(1792)) {
        if (m < INT64_C(57)) {
            if (n < INT64_C(2290)) {
                if (k < INT64_C(227)) {
                    select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                    return out;
                } else {
                    select_f32_tt_config out = {8u, 1u, 1u, 8u, 16u};
                    return out;
                }
            } else {
                if (m < INT64_C(3)) {
                    select_f32_tt_config out = {8u, 1u, 1u, 8u, 16u};
                    return out;
                } else {
                    if (m < INT64_C(6)) {
                        select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                        return out;
                    } else {
                        if (m < INT64_C(12)) {
                            select_f32_tt_config out = {8u, 1u, 1u, 8u, 16u};
                            return out;
                        } else {
                            select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                            return out;
                        }
                    }
                }
            }
        } else {
            if (n < INT64_C(444)) {
                if (m < INT64_C(225)) {
                    if (m < INT64_C(113)) {
                        if (m < INT64_C(80)) {
                            select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                            return out;
                        } else {
                            select_f32_tt_config out = {8u, 1u, 1u, 8u, 16u};
                            return out;
                        }
                    } else {
                        if (n < INT64_C(79)) {
                            select_f32_tt_config out = {8u, 1u, 1u, 8u, 16u};
                            return out;
                        } else {
                            if (k < INT64_C(91)) {
                                select_f32_tt_config out = {8u, 1u, 1u, 8u, 16u};
                                return out;
                            } else {
                                select_f32_tt_config out = {4u, 2u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (n < INT64_C(111)) {
                        if (m < INT64_C(555)) {
                            select_f32_tt_config out = {8u, 1u, 1u, 8u, 16u};
                            return out;
                        } else {
                            if (n < INT64_C(46)) {
                                select_f32_tt_config out = {4u, 2u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(471)) {
                                    select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                                    return out;
                                } else {
                                    select_f32_tt_config out = {4u, 2u, 4u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(1109)) {
                            if (n < INT64_C(176)) {
                                if (m < INT64_C(555)) {
                                    if (k < INT64_C(744)) {
                                        select_f32_tt_config out = {4u, 2u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_tt_config out = {8u, 1u, 1u, 8u, 16u};
                                        return out;
                                    }
                                } else {
                                    select_f32_tt_config out = {4u, 2u, 4u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_f32_tt_config out = {4u, 2u, 4u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (n < INT64_C(157)) {
                                if (k < INT64_C(363)) {
                                    select_f32_tt_config out = {4u, 2u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(768)) {
                                        select_f32_tt_config out = {4u, 4u, 4u, 8u, 16u};
                                        return out;
                                    } else {
                                        select_f32_tt_config out = {4u, 2u, 4u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_f32_tt_config out = {4u, 4u, 4u, 8u, 16u};
                                return out;
                            }
                        }
                    }
                }
            } else {
                if (m < INT64_C(139)) {
                    if (n < INT64_C(1620)) {
                        select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                        return out;
                    } else {
                        select_f32_tt_config out = {4u, 4u, 4u, 8u, 16u};
                        return out;
                    }
                } else {
                    if (n < INT64_C(1145)) {
                        if (m < INT64_C(448)) {
                            if (k < INT64_C(124)) {
                                if (m < INT64_C(278)) {
                                    select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                                    return out;
                                } else {
                                    select_f32_tt_config out = {4u, 4u, 4u, 8u, 16u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(278)) {
                                    if (k < INT64_C(363)) {
                                        if (k < INT64_C(203)) {
                                            select_f32_tt_config out = {4u, 2u, 4u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_f32_tt_config out = {4u, 4u, 4u, 8u, 16u};
                                            return out;
                                        }
                                    } else {
                                        select_f32_tt_config out = {4u, 2u, 4u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(203)) {
                                        select_f32_tt_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(2173)) {
                                            select_f32_tt_config out = {4u, 2u, 4u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_f32_tt_config out = {2u, 4u, 4u, 16u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        } else {
                            if (k < INT64_C(725)) {
                                select_f32_tt_config out = {4u, 4u, 4u, 8u, 16u};
                                return out;
                            } else {
                                if (m < INT64_C(896)) {
                                    select_f32_tt_config out = {4u, 2u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    select_f32_tt_config out = {4u, 4u, 4u, 8u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        select_f32_tt_config out = {4u, 4u, 4u, 8u, 16u};
                        return out;
                    }
                }
            }
        }
    } else {
        if (n < INT64_C(46)) {
            if (m < INT64_C(8870)) {
                if (k < INT64_C(118)) {
                    select_f32_tt_config out = {8u, 2u, 2u, 8u, 16u};
                    return out;
                } else {
                    if (m < INT64_C(4435)) {
                        if (k < INT64_C(167)) {
                            select_f32_tt_config out = {4u, 2u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_f32_tt_config out = {2u, 4u, 4u, 16u, 8u};
                            return out;
                        }
                    } else {
                        select_f32_tt_config out = {2u, 4u, 4u, 16u, 8u};
                        return out;
                    }
                }
            } else {
                if (m < INT64_C(35480)) {
                    if (m < INT64_C(17740)) {
                        if (n < INT64_C(20)) {
                            select_f32_tt_config out = {4u, 4u, 4u, 8u, 16u};
                            return out;
                        } else {
                            select_f32_tt_config out = {1u, 8u, 4u, 16u, 8u};
                            return out;
                        }
                    } else {
                        select_f32_tt_config out = {2u, 4u, 4u, 16u, 8u};
                        return out;
                    }
                } else {
                    select_f32_tt_config out = {1u, 8u, 4u, 16u, 8u};
                    return out;
                }
            }
        } else {
            if (m < INT64_C(35480)) {
                if (n < INT64_C(363)) {
                    if (m < INT64_C(4435)) {
                        if (k < INT64_C(444)) {
                            if (k < INT64_C(28)) {
                                select_f32_tt_config out = {1u, 8u, 4u, 16u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(222)) {
                                    select_f32_tt_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(314)) {
                                        select_f32_tt_config out = {4u, 4u, 4u, 8u, 16u};
                                        return out;
                                    } else {
                                        select_f32_tt_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (k < INT64_C(1630)) {
                                if (n < INT64_C(182)) {
                                    if (k < INT64_C(544)) {
                                        select_f32_tt_config out = {1u, 8u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        if (n < INT64_C(79)) {
                                            select_f32_tt_config out = {4u, 4u, 4u, 8u, 16u};
                                            return out;
                                        } else {
                                            select_f32_tt_config out = {2u, 4u, 4u, 16u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_f32_tt_config out = {4u, 4u, 4u, 8u, 16u};
                                    return out;
                                }
                            } else {
                                select_f32_tt_config out = {8u, 8u, 8u, 16u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (m < INT64_C(17740)) {
                            if (n < INT64_C(136)) {
                                if (k < INT64_C(32)) {
                                    select_f32_tt_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(363)) {
                                        if (m < INT64_C(8870)) {
                                            if (n < INT64_C(91)) {
                                                select_f32_tt_config out = {1u, 8u, 4u, 16u, 8u};
                                                return out;
                                            } else {
                                                select_f32_tt_config out = {4u, 4u, 4u, 8u, 16u};
                                                return out;
                                            }
                                        } else {
                                            select_f32_tt_config out = {4u, 4u, 4u, 8u, 16u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(8870)) {
                                            if (n < INT64_C(91)) {
                                                select_f32_tt_config out = {1u, 8u, 4u, 16u, 8u};
                                                return out;
                                            } else {
                                                select_f32_tt_config out = {4u, 4u, 4u, 8u, 16u};
                                                return out;
                                            }
                                        } else {
                                            select_f32_tt_config out = {1u, 8u, 4u, 16u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(8870)) {
                                    if (k < INT64_C(28)) {
                                        select_f32_tt_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_tt_config out = {1u, 8u, 4u, 16u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(167)) {
                                        select_f32_tt_config out = {1u, 8u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_tt_config out = {8u, 8u, 8u, 16u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (n < INT64_C(111)) {
                                select_f32_tt_config out = {1u, 8u, 4u, 16u, 8u};
                                return out;
                            } else {
                                select_f32_tt_config out = {8u, 8u, 8u, 16u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(4435)) {
                        if (n < INT64_C(544)) {
                            select_f32_tt_config out = {1u, 8u, 4u, 16u, 8u};
                            return out;
                        } else {
                            select_f32_tt_config out = {8u, 8u, 8u, 16u, 8u};
                            return out;
                        }
                    } else {
                        select_f32_tt_config out = {8u, 8u, 8u, 16u, 8u};
                        return out;
                    }
                }
            } else {
                if (k < INT64_C(21)) {
                    select_f32_tt_config out = {1u, 8u, 4u, 16u, 8u};
                    return out;
                } else {
                    select_f32_tt_config out = {8u, 8u, 8u, 16u, 8u};
                    return out;
                }
            }
        }
    }
}

#endif /* SELECT_F32_TT_H */
